// tridiagonal.hpp — drop-in for /root/reference/proj/include/tridpart/tridiagonal.hpp.
//   TridiagonalSystem / Tridiagonal / kPivotFloor    tridiagonal.hpp:15-46
//   thomas_solve                                     tridiagonal.hpp:52-72
//     the same solution, computed on the B200 by the device finishing solver
//     (exact parallel elimination); a zero pivot is reported with the row the
//     sequential sweep reports (tp_thomas_solve_*: reference-order diagnosis)
//   residual_inf                                     tridiagonal.hpp:74-92
//     host verification metric, same formula
#pragma once

#include <cstddef>
#include <span>
#include <vector>

#include "context.hpp"
#include "errors.hpp"

namespace tridpart {

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

    // |b_i| > |a_i| + |c_i| on every row
    bool strictly_dominant() const noexcept {
        auto mag = [](Real v) { return v < Real(0) ? -v : v; };
        for (std::size_t i = 0; i < size(); ++i)
            if (!(mag(diag[i]) > mag(sub[i]) + mag(super[i]))) return false;
        return true;
    }
};
using Tridiagonal = TridiagonalSystem<double>;

namespace b200 {
// The C-ABI entry points per element type (double: *_f64, float: *_f32).
template <class Real>
struct Entry;
template <>
struct Entry<double> {
    static constexpr auto solve = tp_solve_partition_f64;
    static constexpr auto observe = tp_solve_partition_observe_f64;
    static constexpr auto thomas = tp_thomas_solve_f64;
    static constexpr auto reduce = tp_reduce_block_f64;
};
template <>
struct Entry<float> {
    static constexpr auto solve = tp_solve_partition_f32;
    static constexpr auto observe = tp_solve_partition_observe_f32;
    static constexpr auto thomas = tp_thomas_solve_f32;
    static constexpr auto reduce = tp_reduce_block_f32;
};
// the reference indexes sub/super/rhs up to size(): shorter arrays are an
// out-of-bounds read there, an InvalidSizeError here
template <class Real>
inline void check_shape(const TridiagonalSystem<Real>& s) {
    const std::size_t n = s.size();
    if (s.sub.size() != n || s.super.size() != n || s.rhs.size() != n)
        throw InvalidSizeError("sub, diag, super and rhs must have the same length");
}
}  // namespace b200

template <class Real>
std::vector<Real> thomas_solve(const TridiagonalSystem<Real>& sys) {
    b200::check_shape(sys);
    std::vector<Real> x(sys.size());
    tp_error e{};
    b200::throw_on(b200::Entry<Real>::thomas(b200::thread_context().get(), sys.sub.data(), sys.diag.data(),
                                              sys.super.data(), sys.rhs.data(), (int64_t)sys.size(), x.data(),
                                              &e),
                   e);
    return x;
}

// ||Ax - d||_inf / max(1, ||d||_inf)
template <class Real>
Real residual_inf(const TridiagonalSystem<Real>& sys, std::span<const Real> x) {
    auto mag = [](Real v) { return v < Real(0) ? -v : v; };
    const std::size_t n = sys.size();
    Real num = 0, den = 1;
    for (std::size_t i = 0; i < n; ++i) {
        Real ax = sys.diag[i] * x[i];
        if (i > 0) ax += sys.sub[i] * x[i - 1];
        if (i + 1 < n) ax += sys.super[i] * x[i + 1];
        const Real r = mag(ax - sys.rhs[i]), d = mag(sys.rhs[i]);
        num = r > num ? r : num;
        den = d > den ? d : den;
    }
    return num / den;
}
template <class Real>
Real residual_inf(const TridiagonalSystem<Real>& sys, const std::vector<Real>& x) {
    return residual_inf(sys, std::span<const Real>(x));
}

}  // namespace tridpart
