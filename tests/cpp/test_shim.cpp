// C++ drop-in check: the reference's test_partition.cpp / test_policy.cpp
// expectations, written against include/tridpart_b200.hpp (the same
// `tridpart::` names), with the C oracle (oracle/tridpart_oracle.c) as the
// independent checker. Built by tests/test_cpp_shim.py; prints PASS/FAIL lines.
#include <cmath>
#include <cstdio>
#include <vector>

#include "tridpart_b200.hpp"

extern "C" {
int64_t orc_generate_system(int64_t n, uint64_t seed, double delta, double* sub, double* diag,
                            double* sup, double* rhs);
int64_t orc_solve_partition(int64_t n, const double* sub, const double* diag, const double* sup,
                            const double* rhs, const int64_t* sizes, int64_t nlevels, double* x,
                            void* obs, void* user, int64_t* err_level);
int64_t orc_thomas_solve(int64_t n, const double* sub, const double* diag, const double* sup,
                         const double* rhs, double* x);
}

using namespace tridpart;

static int failures = 0;
static void check(bool ok, const char* what) {
    std::printf("%s  %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) ++failures;
}

static Tridiagonal gen(std::size_t n, uint64_t seed) {
    Tridiagonal s;
    s.sub.resize(n); s.diag.resize(n); s.super.resize(n); s.rhs.resize(n);
    orc_generate_system((int64_t)n, seed, 1.5, s.sub.data(), s.diag.data(), s.super.data(), s.rhs.data());
    return s;
}
static std::vector<double> oracle_solve(const Tridiagonal& s, std::vector<int64_t> sizes) {
    std::vector<double> x(s.size());
    int64_t lvl = 0;
    orc_solve_partition((int64_t)s.size(), s.sub.data(), s.diag.data(), s.super.data(), s.rhs.data(),
                        sizes.data(), (int64_t)sizes.size(), x.data(), nullptr, nullptr, &lvl);
    return x;
}
static std::vector<double> oracle_thomas(const Tridiagonal& s) {
    std::vector<double> x(s.size());
    orc_thomas_solve((int64_t)s.size(), s.sub.data(), s.diag.data(), s.super.data(), s.rhs.data(), x.data());
    return x;
}
static double rel_inf_diff(const std::vector<double>& a, const std::vector<double>& b) {
    double diff = 0, scale = 1;
    for (std::size_t i = 0; i < a.size(); ++i) {
        diff = std::max(diff, std::abs(a[i] - b[i]));
        scale = std::max(scale, std::abs(b[i]));
    }
    return diff / scale;
}

int main() {
    {   // make_plan (test_partition.cpp:13-35)
        const auto p = make_plan(9, 4);
        check(p.blocks == std::vector<Block>{{0, 4}, {4, 9}}, "make_plan folds a remainder of 1");
        bool threw = false;
        try { make_plan(1, 4); } catch (const InvalidSizeError&) { threw = true; }
        check(threw, "make_plan(1, 4) throws InvalidSizeError");
    }
    {   // identity system, any policy
        Tridiagonal s;
        s.sub.assign(100, 0); s.diag.assign(100, 1); s.super.assign(100, 0);
        for (int i = 0; i < 100; ++i) s.rhs.push_back(i - 50.0);
        const auto x = solve_partition(s, RecursionPolicy{{8, 10, 4}});
        check(x == s.rhs, "identity system solves exactly");
    }
    {   // n=1e4: R=0 and R=2 agree with Thomas (test_partition.cpp:163-171)
        const auto s = gen(10000, 17);
        const auto ref = oracle_thomas(s);
        const auto x0 = solve_partition(s, RecursionPolicy{{8}});
        const auto x2 = solve_partition(s, RecursionPolicy{{8, 10, 8}});
        check(rel_inf_diff(x0, ref) <= 1e-10 && rel_inf_diff(x2, ref) <= 1e-10, "R=0 and R=2 vs Thomas");
        check(residual_inf(s, x2) <= 1e-12, "residual <= 1e-12");
    }
    {   // config 1 vs the oracle's partition solve
        const auto s = gen(10000, 1);
        const auto x = solve_partition(s, RecursionPolicy{{4}});
        check(rel_inf_diff(x, oracle_solve(s, {4})) <= 1e-10, "N=1e4 m=4 vs oracle");
        check(std::abs(x[5000] - 0.40220197517592371) <= 1e-12, "N=1e4 golden x[5000]");
    }
    {   // observer overload: dominance at every level (acceptance criterion 2)
        const auto s = gen(1500, 7);
        bool dominant = true;
        std::size_t levels = 0;
        solve_partition(s, RecursionPolicy{{5, 3, 7}}, [&](const Tridiagonal& f, std::size_t) {
            ++levels;
            for (std::size_t i = 0; i < f.size(); ++i)
                dominant &= std::abs(f.diag[i]) >= std::abs(f.sub[i]) + std::abs(f.super[i]) - 1e-12;
        });
        check(dominant && levels == 3, "observer sees 3 dominant interface levels");
    }
    {   // thomas drop-in + zero pivot
        const auto s = gen(50, 7);
        check(rel_inf_diff(thomas_solve(s), oracle_thomas(s)) <= 1e-10, "thomas_solve vs oracle");
        Tridiagonal z;
        z.sub = {0, 1}; z.diag = {0, 2}; z.super = {1, 0}; z.rhs = {1, 1};
        bool threw = false;
        try { thomas_solve(z); } catch (const ZeroPivotError&) { threw = true; }
        check(threw, "thomas_solve reports a zero pivot");
    }
    {   // predictors (test_policy.cpp:34-46)
        const auto sm = default_size_model();
        const auto dm = default_depth_model();
        check(recursion_sizes(100000000, 3, sm).sizes == std::vector<std::size_t>{64, 10, 32, 16},
              "recursion_sizes(1e8, 3)");
        check(predict(dm, 100000000) == 3 && predict(dm, 2300000) == 1, "depth model");
        bool threw = false;
        try { recursion_sizes(1000000, 5, sm); } catch (const DepthOutOfRangeError&) { threw = true; }
        check(threw, "depth 5 throws DepthOutOfRangeError");
    }
    {   // fp32 mode (test_partition.cpp:206-223): residual <= 1e-4
        TridiagonalSystem<float> s;
        const std::size_t n = 256;
        s.sub.resize(n); s.diag.resize(n); s.super.resize(n); s.rhs.resize(n);
        uint64_t st = 8;
        auto unit = [&] { st = st * 6364136223846793005ULL + 1442695040888963407ULL;
                          return (float)((double)(st >> 11) * 0x1.0p-53 * 2.0 - 1.0); };
        for (std::size_t i = 0; i < n; ++i) {
            s.sub[i] = i == 0 ? 0.f : unit();
            s.super[i] = i + 1 == n ? 0.f : unit();
            s.diag[i] = 1.5f * (std::abs(s.sub[i]) + std::abs(s.super[i])) + 1.f;
            s.rhs[i] = unit();
        }
        const auto x = solve_partition(s, RecursionPolicy{{8, 4}});
        check(residual_inf(s, x) <= 1e-4f, "fp32 solve_partition residual <= 1e-4");
    }
    std::printf("%s\n", failures ? "FAILED" : "all passed");
    return failures ? 1 : 0;
}
