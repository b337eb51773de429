// ORACLE — TEST INFRASTRUCTURE ONLY.
// extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/tridpart, passed with -I by oracle/Makefile).
// Built into oracle/_ref/libtridpart_ref.so; loaded only by tests/, smoke()
// and bench.py's reference / cpu_baseline legs. No reference source is copied.
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <span>
#include <vector>

#include "tridpart/bench.hpp"
#include "tridpart/io.hpp"
#include "tridpart/knn.hpp"
#include "tridpart/partition.hpp"
#include "tridpart/policy.hpp"
#include "tridpart/tridiagonal.hpp"

using namespace tridpart;

namespace {
HeuristicModel g_size, g_depth;
bool g_models = false;

Tridiagonal wrap(int64_t n, const double* a, const double* b, const double* c, const double* d) {
    Tridiagonal s;
    s.sub.assign(a, a + n);
    s.diag.assign(b, b + n);
    s.super.assign(c, c + n);
    s.rhs.assign(d, d + n);
    return s;
}

// -1 ok, >=0 zero-pivot row, -2 invalid size, -3 depth out of range, -4 other
template <class F>
int64_t guarded(F&& f) {
    try {
        f();
        return -1;
    } catch (const ZeroPivotError& e) {
        return (int64_t)e.row();
    } catch (const InvalidSizeError&) {
        return -2;
    } catch (const DepthOutOfRangeError&) {
        return -3;
    } catch (...) {
        return -4;
    }
}
}  // namespace

extern "C" {

int64_t ref_generate_system(int64_t n, uint64_t seed, double delta, double* a, double* b, double* c,
                            double* d) {
    return guarded([&] {
        const auto s = generate_system((std::size_t)n, seed, delta);
        std::memcpy(a, s.sub.data(), n * sizeof(double));
        std::memcpy(b, s.diag.data(), n * sizeof(double));
        std::memcpy(c, s.super.data(), n * sizeof(double));
        std::memcpy(d, s.rhs.data(), n * sizeof(double));
    });
}

int64_t ref_thomas_solve(int64_t n, const double* a, const double* b, const double* c,
                         const double* d, double* x) {
    return guarded([&] {
        const auto s = wrap(n, a, b, c, d);
        const auto r = thomas_solve(s);
        std::memcpy(x, r.data(), n * sizeof(double));
    });
}

// A pre-built system handle so timing loops measure solve_partition only.
void* ref_system_new(int64_t n, const double* a, const double* b, const double* c, const double* d) {
    return new Tridiagonal(wrap(n, a, b, c, d));
}
void* ref_system_generate(int64_t n, uint64_t seed) {
    return new Tridiagonal(generate_system((std::size_t)n, seed));
}
void ref_system_free(void* h) { delete static_cast<Tridiagonal*>(h); }

// Pointers to a handle's own arrays (so callers view them without a copy).
void ref_system_view(void* h, double** a, double** b, double** c, double** d) {
    auto& s = *static_cast<Tridiagonal*>(h);
    *a = s.sub.data();
    *b = s.diag.data();
    *c = s.super.data();
    *d = s.rhs.data();
}

int64_t ref_system_thomas(void* h, double* x) {
    return guarded([&] {
        const auto r = thomas_solve(*static_cast<Tridiagonal*>(h));
        std::memcpy(x, r.data(), r.size() * sizeof(double));
    });
}

int64_t ref_system_solve(void* h, const int64_t* sizes, int32_t nsizes, double* x) {
    return guarded([&] {
        RecursionPolicy p;
        for (int i = 0; i < nsizes; ++i) p.sizes.push_back((std::size_t)sizes[i]);
        const auto r = solve_partition(*static_cast<Tridiagonal*>(h), p);
        if (x) std::memcpy(x, r.data(), r.size() * sizeof(double));
    });
}

double ref_system_residual(void* h, const double* x) {
    const auto& s = *static_cast<Tridiagonal*>(h);
    return residual_inf(s, std::span<const double>(x, s.size()));
}

typedef void (*ref_observer)(int64_t level, int64_t n, const double* a, const double* b,
                             const double* c, const double* d, void* user);

int64_t ref_solve_partition(int64_t n, const double* a, const double* b, const double* c,
                            const double* d, const int64_t* sizes, int32_t nsizes, double* x,
                            ref_observer obs, void* user) {
    return guarded([&] {
        const auto s = wrap(n, a, b, c, d);
        RecursionPolicy p;
        for (int i = 0; i < nsizes; ++i) p.sizes.push_back((std::size_t)sizes[i]);
        std::vector<double> r;
        if (obs) {
            r = solve_partition(s, p, [&](const Tridiagonal& f, std::size_t level) {
                obs((int64_t)level, (int64_t)f.size(), f.sub.data(), f.diag.data(), f.super.data(),
                    f.rhs.data(), user);
            });
        } else {
            r = solve_partition(s, p);
        }
        std::memcpy(x, r.data(), n * sizeof(double));
    });
}

double ref_residual_inf(int64_t n, const double* a, const double* b, const double* c,
                        const double* d, const double* x) {
    const auto s = wrap(n, a, b, c, d);
    return residual_inf(s, std::span<const double>(x, (std::size_t)n));
}

int64_t ref_reduce_block(int64_t n, const double* a, const double* b, const double* c,
                         const double* d, int64_t start, int64_t end, double* eq8) {
    return guarded([&] {
        const auto s = wrap(n, a, b, c, d);
        const auto r = reduce_block(s, Block{(std::size_t)start, (std::size_t)end});
        const double v[8] = {r.alpha1, r.beta1, r.gamma1, r.delta1,
                             r.alpha2, r.beta2, r.gamma2, r.delta2};
        std::memcpy(eq8, v, sizeof(v));
    });
}

int64_t ref_make_plan(int64_t n, int64_t m, int64_t* bounds) {
    int64_t k = -2;
    guarded([&] {
        const auto p = make_plan((std::size_t)n, (std::size_t)m);
        k = (int64_t)p.blocks.size();
        if (bounds) {
            for (std::size_t j = 0; j < p.blocks.size(); ++j) bounds[j] = (int64_t)p.blocks[j].start;
            bounds[p.blocks.size()] = (int64_t)p.blocks.back().end;
        }
    });
    return k;
}

// Models exactly as the reference tests fit them (test_policy.cpp:14-21).
int64_t ref_load_models(const char* data_dir) {
    return guarded([&] {
        const std::filesystem::path dir(data_dir);
        g_size = fit_knn(read_observations(dir / "table1_fp64.csv").with_corrected_labels(), 1);
        g_depth = fit_depth_model(read_observations(dir / "table2_recursion.csv"));
        g_models = true;
    });
}

int32_t ref_predict_size(int64_t n) { return g_models ? predict(g_size, n) : -1; }
int32_t ref_predict_depth(int64_t n) { return g_models ? predict(g_depth, n) : -1; }

int64_t ref_recursion_sizes(int64_t n, int32_t depth, int64_t* sizes) {
    int64_t cnt = -4;
    const int64_t st = guarded([&] {
        const auto p = recursion_sizes(n, depth, g_size);
        for (std::size_t i = 0; i < p.sizes.size(); ++i) sizes[i] = (int64_t)p.sizes[i];
        cnt = (int64_t)p.sizes.size();
    });
    return st == -1 ? cnt : st;
}

int32_t ref_model_pairs(int32_t which, int64_t* n, int32_t* label, int32_t cap) {
    const auto& m = which == 0 ? g_size : g_depth;
    const int32_t cnt = (int32_t)m.pairs.size();
    for (int32_t i = 0; i < cnt && i < cap; ++i) {
        n[i] = m.pairs[i].n;
        label[i] = m.pairs[i].label;
    }
    return cnt;
}

uint32_t ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// solve_partition<float> / thomas_solve<float> / residual_inf<float>: the
// reference's templates instantiated on float (partition.hpp:61-77,
// test_partition.cpp:206-223).
int64_t ref_solve_partition_f32(int64_t n, const float* a, const float* b, const float* c,
                                const float* d, const int64_t* sizes, int32_t nsizes, float* x) {
    return guarded([&] {
        TridiagonalSystem<float> s;
        s.sub.assign(a, a + n);
        s.diag.assign(b, b + n);
        s.super.assign(c, c + n);
        s.rhs.assign(d, d + n);
        RecursionPolicy p;
        for (int i = 0; i < nsizes; ++i) p.sizes.push_back((std::size_t)sizes[i]);
        const auto r = solve_partition(s, p);
        std::memcpy(x, r.data(), n * sizeof(float));
    });
}

float ref_residual_inf_f32(int64_t n, const float* a, const float* b, const float* c, const float* d,
                           const float* x) {
    TridiagonalSystem<float> s;
    s.sub.assign(a, a + n);
    s.diag.assign(b, b + n);
    s.super.assign(c, c + n);
    s.rhs.assign(d, d + n);
    return residual_inf(s, std::span<const float>(x, (std::size_t)n));
}
}
