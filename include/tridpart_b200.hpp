// tridpart_b200.hpp — header-only C++20 shim that rebuilds the reference
// `tridpart::` API for the partition-solve path on top of the C-ABI
// (tridpart_b200.h). A caller of the reference replaces
//     #include "tridpart/partition.hpp"   (and policy.hpp / knn.hpp)
// with
//     #include "tridpart_b200.hpp"
// and links -ltridpart_b200; the names, signatures, value semantics and
// exception types below are the reference's (paths relative to
// /root/reference/proj/include/tridpart):
//   TridiagonalSystem / thomas_solve / residual_inf      tridiagonal.hpp:22-92
//   Block / PartitionPlan / make_plan                    partition.hpp:14-49
//   RecursionPolicy / solve_partition (both overloads)   partition.hpp:176-248
//   TrainingPair / HeuristicModel / fit_knn / predict    knn.hpp:18-77
//   kMaxRecursionDepth / fit_depth_model / recursion_sizes policy.hpp:11-45
//   Error hierarchy                                      errors.hpp:7-96
// Real = double or float, as the reference's templates (FP32 entries *_f32).
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "tridpart_b200.h"

namespace tridpart {

// ------------------------------------------------------------- errors.hpp
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ZeroPivotError : public Error {
public:
    explicit ZeroPivotError(std::size_t row, std::size_t level = 0)
        : Error("zero pivot at row " + std::to_string(row)), row_(row), level_(level) {}
    std::size_t row() const noexcept { return row_; }
    std::size_t level() const noexcept { return level_; }

private:
    std::size_t row_, level_;
};
class InvalidSizeError : public Error { public: using Error::Error; };
class DepthOutOfRangeError : public Error { public: using Error::Error; };
class EmptyTrainingSetError : public Error {
public:
    EmptyTrainingSetError() : Error("training set is empty") {}
};
class KTooLargeError : public Error { public: using Error::Error; };
class MalformedHeaderError : public Error { public: using Error::Error; };
class BadNumberError : public Error { public: using Error::Error; };
class DeviceError : public Error { public: using Error::Error; };

namespace b200 {
inline void throw_on(tp_status s, const tp_error& e) {
    switch (s) {
        case TP_OK: return;
        case TP_ERR_ZERO_PIVOT: throw ZeroPivotError((std::size_t)e.row, (std::size_t)e.level);
        case TP_ERR_INVALID_SIZE: throw InvalidSizeError(e.msg);
        case TP_ERR_DEPTH_OUT_OF_RANGE: throw DepthOutOfRangeError(e.msg);
        case TP_ERR_EMPTY_TRAINING_SET: throw EmptyTrainingSetError();
        case TP_ERR_K_TOO_LARGE: throw KTooLargeError(e.msg);
        case TP_ERR_MALFORMED_HEADER: throw MalformedHeaderError(e.msg);
        case TP_ERR_BAD_NUMBER: throw BadNumberError(e.msg);
        case TP_ERR_CUDA: throw DeviceError(e.msg);
        default: throw Error(e.msg);
    }
}

// One context per host thread (a tp_ctx is not thread-safe; the reference is
// reentrant, so every thread gets its own device context).
class Context {
public:
    explicit Context(int device = 0) {
        tp_error e{};
        throw_on(tp_ctx_create(device, &ctx_, &e), e);
    }
    ~Context() { tp_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    tp_ctx* get() const noexcept { return ctx_; }

private:
    tp_ctx* ctx_ = nullptr;
};
inline Context& thread_context() {
    thread_local Context ctx(0);
    return ctx;
}
}  // namespace b200

// ---------------------------------------------------------- tridiagonal.hpp
template <class Real>
inline constexpr Real kPivotFloor = Real(1e-30);

template <class Real>
struct TridiagonalSystem {
    std::vector<Real> sub, diag, super, rhs;
    std::size_t size() const noexcept { return diag.size(); }
    bool well_formed() const noexcept {
        const std::size_t n = diag.size();
        if (n == 0 || sub.size() != n || super.size() != n || rhs.size() != n) return false;
        return sub.front() == Real(0) && super.back() == Real(0);
    }
    bool strictly_dominant() const noexcept {
        for (std::size_t i = 0; i < size(); ++i) {
            const Real a = sub[i] < 0 ? -sub[i] : sub[i], b = diag[i] < 0 ? -diag[i] : diag[i],
                       c = super[i] < 0 ? -super[i] : super[i];
            if (!(b > a + c)) return false;
        }
        return true;
    }
};
using Tridiagonal = TridiagonalSystem<double>;

// The device entry points per element type (double: *_f64, float: *_f32).
namespace b200 {
template <class Real>
struct Entry;
template <>
struct Entry<double> {
    static constexpr auto solve = tp_solve_partition_f64;
    static constexpr auto observe = tp_solve_partition_observe_f64;
    static constexpr auto thomas = tp_thomas_solve_f64;
};
template <>
struct Entry<float> {
    static constexpr auto solve = tp_solve_partition_f32;
    static constexpr auto observe = tp_solve_partition_observe_f32;
    static constexpr auto thomas = tp_thomas_solve_f32;
};
}  // namespace b200

template <class Real>
std::vector<Real> thomas_solve(const TridiagonalSystem<Real>& sys) {
    std::vector<Real> x(sys.size());
    tp_error e{};
    b200::throw_on(b200::Entry<Real>::thomas(b200::thread_context().get(), sys.sub.data(),
                                              sys.diag.data(), sys.super.data(), sys.rhs.data(),
                                              (int64_t)sys.size(), x.data(), &e),
                   e);
    return x;
}

// Host-side verification metric, same formula as tridiagonal.hpp:74-87.
template <class Real>
Real residual_inf(const TridiagonalSystem<Real>& sys, std::span<const Real> x) {
    const std::size_t n = sys.size();
    Real num = 0, den = 1;
    for (std::size_t i = 0; i < n; ++i) {
        Real ax = sys.diag[i] * x[i];
        if (i > 0) ax += sys.sub[i] * x[i - 1];
        if (i + 1 < n) ax += sys.super[i] * x[i + 1];
        const Real r = ax > sys.rhs[i] ? ax - sys.rhs[i] : sys.rhs[i] - ax;
        const Real d = sys.rhs[i] < 0 ? -sys.rhs[i] : sys.rhs[i];
        num = r > num ? r : num;
        den = d > den ? d : den;
    }
    return num / den;
}
template <class Real>
Real residual_inf(const TridiagonalSystem<Real>& sys, const std::vector<Real>& x) {
    return residual_inf(sys, std::span<const Real>(x));
}

// ------------------------------------------------------------ partition.hpp
struct Block {
    std::size_t start = 0, end = 0;
    std::size_t length() const noexcept { return end - start; }
    bool operator==(const Block&) const = default;
};
struct PartitionPlan {
    std::size_t n = 0, m = 0;
    std::vector<Block> blocks;
};
inline PartitionPlan make_plan(std::size_t n, std::size_t m) {
    tp_error e{};
    int64_t k = 0;
    b200::throw_on(tp_make_plan((int64_t)n, (int64_t)m, nullptr, &k, &e), e);
    std::vector<int64_t> b((std::size_t)k + 1);
    b200::throw_on(tp_make_plan((int64_t)n, (int64_t)m, b.data(), &k, &e), e);
    PartitionPlan p{n, m, {}};
    for (int64_t j = 0; j < k; ++j) p.blocks.push_back({(std::size_t)b[j], (std::size_t)b[j + 1]});
    return p;
}

struct RecursionPolicy {
    std::vector<std::size_t> sizes;
    std::size_t depth() const noexcept { return sizes.size() - 1; }
    bool valid() const noexcept {
        if (sizes.empty()) return false;
        for (auto m : sizes)
            if (m < 2) return false;
        return true;
    }
};

namespace b200 {
inline std::vector<int64_t> policy_array(const RecursionPolicy& p) {
    return std::vector<int64_t>(p.sizes.begin(), p.sizes.end());
}
template <class Real, class F>
void trampoline(int64_t level, int64_t n, const Real* a, const Real* b, const Real* c, const Real* d,
                void* user) {
    TridiagonalSystem<Real> t;
    t.sub.assign(a, a + n);
    t.diag.assign(b, b + n);
    t.super.assign(c, c + n);
    t.rhs.assign(d, d + n);
    (*static_cast<F*>(user))(static_cast<const TridiagonalSystem<Real>&>(t), (std::size_t)level);
}
}  // namespace b200

template <class Real, class InterfaceObserver>
std::vector<Real> solve_partition(const TridiagonalSystem<Real>& sys, const RecursionPolicy& policy,
                                  InterfaceObserver&& on_interface) {
    const auto sz = b200::policy_array(policy);
    std::vector<Real> x(sys.size());
    tp_error e{};
    using F = std::remove_reference_t<InterfaceObserver>;
    b200::throw_on(b200::Entry<Real>::observe(b200::thread_context().get(), sys.sub.data(),
                                               sys.diag.data(), sys.super.data(), sys.rhs.data(),
                                               (int64_t)sys.size(), sz.data(), (int32_t)sz.size(),
                                               x.data(), &b200::trampoline<Real, F>,
                                               (void*)&on_interface, &e),
                   e);
    return x;
}

template <class Real>
std::vector<Real> solve_partition(const TridiagonalSystem<Real>& sys, const RecursionPolicy& policy) {
    const auto sz = b200::policy_array(policy);
    std::vector<Real> x(sys.size());
    tp_error e{};
    b200::throw_on(b200::Entry<Real>::solve(b200::thread_context().get(), sys.sub.data(),
                                             sys.diag.data(), sys.super.data(), sys.rhs.data(),
                                             (int64_t)sys.size(), sz.data(), (int32_t)sz.size(),
                                             x.data(), &e),
                   e);
    return x;
}

// ------------------------------------------------------- knn.hpp / policy.hpp
struct TrainingPair {
    std::int64_t n = 0;
    int label = 0;
    bool operator==(const TrainingPair&) const = default;
};
struct HeuristicModel {
    std::vector<TrainingPair> pairs;
    int k = 1;
    std::string transform = "log10_n";
    std::vector<int> labels;
    std::map<std::string, std::string> metadata;
};

namespace b200 {
inline void split_pairs(const HeuristicModel& m, std::vector<int64_t>& n, std::vector<int32_t>& l) {
    n.clear();
    l.clear();
    for (const auto& p : m.pairs) {
        n.push_back(p.n);
        l.push_back(p.label);
    }
}
inline HeuristicModel bundled(int which) {
    tp_error e{};
    int64_t cnt = 0;
    int32_t k = 1;
    throw_on(tp_default_model(which, nullptr, nullptr, 0, &cnt, &k, &e), e);
    std::vector<int64_t> n((std::size_t)cnt);
    std::vector<int32_t> l((std::size_t)cnt);
    throw_on(tp_default_model(which, n.data(), l.data(), cnt, &cnt, &k, &e), e);
    HeuristicModel m;
    m.k = k;
    for (int64_t i = 0; i < cnt; ++i) m.pairs.push_back({n[i], l[i]});
    std::map<int, int> seen;
    for (auto v : l) seen[v] = 1;
    for (auto& [v, _] : seen) m.labels.push_back(v);
    return m;
}
}  // namespace b200

inline int predict(const HeuristicModel& model, std::int64_t n) {
    std::vector<int64_t> pn;
    std::vector<int32_t> pl;
    b200::split_pairs(model, pn, pl);
    int32_t out = 0;
    tp_error e{};
    b200::throw_on(tp_predict(pn.data(), pl.data(), (int64_t)pn.size(), model.k, n, &out, &e), e);
    return out;
}

inline constexpr int kMaxRecursionDepth = 4;

inline RecursionPolicy recursion_sizes(std::int64_t n, int depth, const HeuristicModel& size_model) {
    std::vector<int64_t> pn;
    std::vector<int32_t> pl;
    b200::split_pairs(size_model, pn, pl);
    int64_t sizes[8];
    int32_t cnt = 0;
    tp_error e{};
    b200::throw_on(tp_recursion_sizes(n, depth, pn.data(), pl.data(), (int64_t)pn.size(), size_model.k,
                                      sizes, &cnt, &e),
                   e);
    RecursionPolicy p;
    for (int32_t i = 0; i < cnt; ++i) p.sizes.push_back((std::size_t)sizes[i]);
    return p;
}

// The models the reference's tests fit (test_policy.cpp:14-21), bundled;
// default_fp32_size_model: Table IV (FP32) with corrected labels.
inline HeuristicModel default_size_model() { return b200::bundled(0); }
inline HeuristicModel default_fp32_size_model() { return b200::bundled(2); }
inline HeuristicModel default_depth_model() { return b200::bundled(1); }

}  // namespace tridpart
