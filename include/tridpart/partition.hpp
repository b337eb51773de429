// partition.hpp — drop-in for /root/reference/proj/include/tridpart/partition.hpp.
//   Block / PartitionPlan / make_plan           partition.hpp:14-49   (C-ABI tp_make_plan)
//   ReducedBlock / reduce_block                 partition.hpp:52-126  (device, tp_reduce_block_*:
//       the reference's own sequential arithmetic, one thread per block)
//   assemble_interface                          partition.hpp:131-151 (host copy)
//   back_substitute                             partition.hpp:156-172 (host, from ReducedBlock)
//   RecursionPolicy                             partition.hpp:176-187
//   solve_partition (both overloads)            partition.hpp:228-248 (the B200 solve, tp_solve_partition_*)
// The stage functions serve callers that drive the stages themselves (and the
// reference's unit tests); solve_partition never goes through them.
#pragma once

#include <cstddef>
#include <cstdint>
#include <type_traits>
#include <vector>

#include "tridiagonal.hpp"

namespace tridpart {

struct Block {
    std::size_t start = 0;
    std::size_t end = 0;  // exclusive
    std::size_t length() const noexcept { return end - start; }
    bool operator==(const Block&) const = default;
};

struct PartitionPlan {
    std::size_t n = 0;
    std::size_t m = 0;
    std::vector<Block> blocks;
};

inline PartitionPlan make_plan(std::size_t n, std::size_t m) {
    tp_error e{};
    int64_t k = 0;
    b200::throw_on(tp_make_plan((int64_t)n, (int64_t)m, nullptr, &k, &e), e);
    std::vector<int64_t> b((std::size_t)k + 1);
    b200::throw_on(tp_make_plan((int64_t)n, (int64_t)m, b.data(), &k, &e), e);
    PartitionPlan p{n, m, {}};
    p.blocks.reserve((std::size_t)k);
    for (int64_t j = 0; j < k; ++j) p.blocks.push_back({(std::size_t)b[j], (std::size_t)b[j + 1]});
    return p;
}

// eq1: alpha1 x_{s-1} + beta1 x_s + gamma1 x_e = delta1
// eq2: alpha2 x_s + beta2 x_e + gamma2 x_{e+1} = delta2
// a / beta / gamma / delta: the up-sweep rows a_i x_{i-1} + beta_i x_i + gamma_i x_e = delta_i,
// indexed by offset from start (entry len-1 unused)
template <class Real>
struct ReducedBlock {
    std::size_t start = 0;
    std::size_t end = 0;
    Real alpha1, beta1, gamma1, delta1;
    Real alpha2, beta2, gamma2, delta2;
    std::vector<Real> a, beta, gamma, delta;
};

template <class Real>
ReducedBlock<Real> reduce_block(const TridiagonalSystem<Real>& sys, Block blk) {
    if (blk.length() < 2 || blk.end > sys.size()) throw InvalidSizeError("block length must be >= 2");
    const std::size_t len = blk.length();
    ReducedBlock<Real> out;
    out.start = blk.start;
    out.end = blk.end;
    out.a.assign(len, Real(0));
    out.beta.assign(len, Real(0));
    out.gamma.assign(len, Real(0));
    out.delta.assign(len, Real(0));
    Real eq[8];
    tp_error e{};
    b200::throw_on(b200::Entry<Real>::reduce(b200::thread_context().get(), sys.sub.data(), sys.diag.data(),
                                              sys.super.data(), sys.rhs.data(), (int64_t)sys.size(),
                                              (int64_t)blk.start, (int64_t)blk.end, eq, out.a.data(),
                                              out.beta.data(), out.gamma.data(), out.delta.data(), &e),
                   e);
    out.alpha1 = eq[0]; out.beta1 = eq[1]; out.gamma1 = eq[2]; out.delta1 = eq[3];
    out.alpha2 = eq[4]; out.beta2 = eq[5]; out.gamma2 = eq[6]; out.delta2 = eq[7];
    return out;
}

// Interface system of 2K rows in the unknowns x_{s_1}, x_{e_1}, ..., x_{s_K}, x_{e_K}.
template <class Real>
TridiagonalSystem<Real> assemble_interface(const std::vector<ReducedBlock<Real>>& blocks) {
    TridiagonalSystem<Real> f;
    const std::size_t rows = 2 * blocks.size();
    f.sub.resize(rows);
    f.diag.resize(rows);
    f.super.resize(rows);
    f.rhs.resize(rows);
    std::size_t r = 0;
    for (const auto& b : blocks) {
        f.sub[r] = b.alpha1; f.diag[r] = b.beta1; f.super[r] = b.gamma1; f.rhs[r] = b.delta1;
        ++r;
        f.sub[r] = b.alpha2; f.diag[r] = b.beta2; f.super[r] = b.gamma2; f.rhs[r] = b.delta2;
        ++r;
    }
    return f;
}

// x_{s+1} .. x_{e-1} from the stored up-sweep rows, left to right.
template <class Real>
std::vector<Real> back_substitute(const ReducedBlock<Real>& blk, Real x_s, Real x_e) {
    const std::size_t len = blk.end - blk.start;
    std::vector<Real> interior;
    if (len <= 2) return interior;
    interior.reserve(len - 2);
    Real prev = x_s;
    for (std::size_t k = 1; k + 1 < len; ++k) {
        const Real piv = blk.beta[k];
        if ((piv < Real(0) ? -piv : piv) < kPivotFloor<Real>) throw ZeroPivotError(blk.start + k);
        prev = (blk.delta[k] - blk.a[k] * prev - blk.gamma[k] * x_e) / piv;
        interior.push_back(prev);
    }
    return interior;
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

// Observer overload: on_interface(iface, level) after each level's assembly;
// before a ZeroPivotError the levels the reference completed are delivered.
template <class Real, class InterfaceObserver>
std::vector<Real> solve_partition(const TridiagonalSystem<Real>& sys, const RecursionPolicy& policy,
                                  InterfaceObserver&& on_interface) {
    if (!policy.valid()) throw InvalidSizeError("invalid recursion policy");
    if (sys.size() == 0) throw InvalidSizeError("empty system");
    b200::check_shape(sys);
    const auto sz = b200::policy_array(policy);
    std::vector<Real> x(sys.size());
    tp_error e{};
    using F = std::remove_reference_t<InterfaceObserver>;
    b200::throw_on(b200::Entry<Real>::observe(b200::thread_context().get(), sys.sub.data(), sys.diag.data(),
                                               sys.super.data(), sys.rhs.data(), (int64_t)sys.size(), sz.data(),
                                               (int32_t)sz.size(), x.data(), &b200::trampoline<Real, F>,
                                               (void*)&on_interface, &e),
                   e);
    return x;
}

template <class Real>
std::vector<Real> solve_partition(const TridiagonalSystem<Real>& sys, const RecursionPolicy& policy) {
    if (!policy.valid()) throw InvalidSizeError("invalid recursion policy");
    if (sys.size() == 0) throw InvalidSizeError("empty system");
    b200::check_shape(sys);
    const auto sz = b200::policy_array(policy);
    std::vector<Real> x(sys.size());
    tp_error e{};
    b200::throw_on(b200::Entry<Real>::solve(b200::thread_context().get(), sys.sub.data(), sys.diag.data(),
                                             sys.super.data(), sys.rhs.data(), (int64_t)sys.size(), sz.data(),
                                             (int32_t)sz.size(), x.data(), &e),
                   e);
    return x;
}

}  // namespace tridpart
