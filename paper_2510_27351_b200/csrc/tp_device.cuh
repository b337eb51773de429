// Device building blocks of the B200 partition solver.
//
// Terminology (reference: /root/reference/proj/include/tridpart/partition.hpp):
//   * A "segment" is a run of consecutive rows [s, e] of one level's system.
//   * Its two interface equations (partition.hpp:52-60, reduce_block :77-126):
//       E1:  a1*x_{s-1} + b1*x_s + g1*x_e     = d1
//       E2:  a2*x_s     + b2*x_e + g2*x_{e+1} = d2
//   * A "chunk" is the segment one thread owns (L rows); a partition "block"
//     (m rows, make_plan partition.hpp:30-49) is G chunks owned by G lanes.
//
// The reference reduces a block by a sequential up-sweep and down-sweep over
// its m rows. Here every lane reduces its own chunk with exactly those sweeps
// (leaf_*), and the G chunk-equation pairs are merged pairwise in a log2(G)
// lane tree (merge_*): a merge IS reduce_block applied to the 4-row system
// [A.E1, A.E2, B.E1, B.E2]. E1/E2 of a block are unique once the x_{s-1}
// coefficient (= sub[s]) and the x_{e+1} coefficient (= super[e]) are fixed,
// so the result equals the reference's interface rows up to rounding.
// Stage 3 (back_substitute, partition.hpp:156-172) runs the tree top-down and
// finishes every chunk with the reference's forward substitution.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tp_kernels.h"

namespace tpb {

// kPivotFloor<double> — tridiagonal.hpp:15-16
constexpr double kPivotFloor = 1e-30;


struct Eq2 {
    double a1, b1, g1, d1;  // E1
    double a2, b2, g2, d2;  // E2
};

// Saved per merge for the top-down pass: x_t = (d1 - a2*x_s - g1*x_e) * r1
struct MergeSave {
    double d1, g1, r1, a2;
};

// FP64 reciprocal: MUFU.RCP64H seed + one cubic Newton step, <= 1 ulp from the
// correctly rounded 1/x (checked on the GPU by tp_diag_rcp_ulp); no slow path,
// because every pivot it sees passed the |p| >= 1e-30 floor check (or is
// already reported as a zero pivot). w = c * rcp(p) replaces the reference's
// c / p (<= ~2 ulp apart; parity is by tolerance).
__device__ __forceinline__ double rcp(double x) {
    // seed error e0 ~ 2^-22; r*(1 + e + e^2) leaves ~e0^3 before rounding
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

// Zero-pivot bookkeeping (|pivot| < kPivotFloor -> ZeroPivotError).
// RowGuard remembers the smallest offending row (generic / finishing paths);
// MinGuard keeps only min|pivot| (one DMNMX per pivot on the hot path) and the
// caller reports the chunk's first row when it fell below the floor.
struct RowGuard {
    int64_t bad = INT64_MAX;
    __device__ __forceinline__ void see(double p, int64_t row) {
        if (fabs(p) < kPivotFloor) bad = (row < bad) ? row : bad;
    }
};
struct MinGuard {
    double pmin = 1.0e300;
    __device__ __forceinline__ void see(double p, int64_t) { pmin = fmin(pmin, fabs(p)); }
    __device__ __forceinline__ bool tripped() const { return pmin < kPivotFloor; }
};

// err word encodes (level << 48) | row; atomicMin keeps the lexicographically
// first failure. Reported to the host as ZeroPivotError(row) at `level`.
__device__ __forceinline__ void report_pivot(unsigned long long* err, int level, int64_t bad) {
    if (bad != INT64_MAX && err != nullptr) {
        unsigned long long code =
            (static_cast<unsigned long long>(level) << 48) |
            (static_cast<unsigned long long>(bad) & 0xFFFFFFFFFFFFULL);
        atomicMin(err, code);
    }
}

// ---------------------------------------------------------------------------
// Leaf: one chunk held in registers sized L; its first K rows are valid
// (K == L on the fixed-shape path; k_fast_rt dispatches on a runtime length).
// up-sweep  = partition.hpp:90-108, down-sweep = partition.hpp:110-124.
// ---------------------------------------------------------------------------
template <int L>
struct Chunk {
    double a[L], b[L], c[L], d[L];
};

// Stage-1 leaf: E1/E2 only (no per-row storage).
template <int L, int len, class G>
__device__ __forceinline__ Eq2 leaf_reduce(const Chunk<L>& r, int64_t row0, G& bad) {
    Eq2 q;
    // up-sweep: seed row len-2, run i = len-3 .. 0
    double beta = 0, gamma = 0, delta = 0;
#pragma unroll
    for (int i = L - 2; i >= 0; --i) {
        if (i == len - 2) {
            beta = r.b[i];
            gamma = r.c[i];
            delta = r.d[i];
        } else if (i < len - 2) {
            bad.see(beta, row0 + i + 1);
            const double w = r.c[i] * rcp(beta);
            beta = r.b[i] - w * r.a[i + 1];
            gamma = -w * gamma;
            delta = r.d[i] - w * delta;
        }
    }
    q.a1 = r.a[0];
    q.b1 = beta;
    q.g1 = gamma;
    q.d1 = delta;
    // down-sweep: seed row 1, run i = 2 .. len-1
    double phi = r.a[1], bp = r.b[1], dp = r.d[1];
    double glast = r.c[1];
#pragma unroll
    for (int i = 2; i < L; ++i) {
        if (i < len) {
            bad.see(bp, row0 + i - 1);
            const double w = r.a[i] * rcp(bp);
            phi = -w * phi;
            bp = r.b[i] - w * r.c[i - 1];
            dp = r.d[i] - w * dp;
            glast = r.c[i];
        }
    }
    q.a2 = phi;
    q.b2 = bp;
    q.g2 = glast;
    q.d2 = dp;
    return q;
}

// Stage-3 leaf: same sweeps, but keeps rcp(beta_i), gamma_i, delta_i of the
// interior rows for back_substitute (partition.hpp:156-172).
template <int L, int len, class G>
__device__ __forceinline__ Eq2 leaf_reduce_keep(const Chunk<L>& r, int64_t row0,
                                                G& bad, double (&rbeta)[L],
                                                double (&gam)[L], double (&del)[L]) {
    Eq2 q;
    double beta = 0, gamma = 0, delta = 0;
#pragma unroll
    for (int i = L - 2; i >= 0; --i) {
        if (i == len - 2) {
            beta = r.b[i];
            gamma = r.c[i];
            delta = r.d[i];
        } else if (i < len - 2) {
            bad.see(beta, row0 + i + 1);
            const double rb = rcp(beta);
            rbeta[i + 1] = rb;
            const double w = r.c[i] * rb;
            beta = r.b[i] - w * r.a[i + 1];
            gamma = -w * gamma;
            delta = r.d[i] - w * delta;
        }
        gam[i] = gamma;
        del[i] = delta;
    }
    q.a1 = r.a[0];
    q.b1 = beta;
    q.g1 = gamma;
    q.d1 = delta;
    double phi = r.a[1], bp = r.b[1], dp = r.d[1];
    double glast = r.c[1];
#pragma unroll
    for (int i = 2; i < L; ++i) {
        if (i < len) {
            bad.see(bp, row0 + i - 1);
            const double w = r.a[i] * rcp(bp);
            phi = -w * phi;
            bp = r.b[i] - w * r.c[i - 1];
            dp = r.d[i] - w * dp;
            glast = r.c[i];
        }
    }
    q.a2 = phi;
    q.b2 = bp;
    q.g2 = glast;
    q.d2 = dp;
    return q;
}

// Interior of a chunk from its end values: back_substitute, partition.hpp:163-170.
template <int L, int len>
__device__ __forceinline__ void leaf_expand(const Chunk<L>& r, const double (&rbeta)[L],
                                            const double (&gam)[L], const double (&del)[L],
                                            double xs, double xe, double (&x)[L]) {
    x[0] = xs;
    double prev = xs;
#pragma unroll
    for (int i = 1; i < L; ++i) {
        if (i < len - 1) {
            const double xi = (del[i] - r.a[i] * prev - gam[i] * xe) * rbeta[i];
            x[i] = xi;
            prev = xi;
        } else if (i == len - 1) {
            x[i] = xe;
        }
    }
}

// ---------------------------------------------------------------------------
// Merge of adjacent segments A=[s,t], B=[t+1,e]: reduce_block on the 4-row
// system [A.E1, A.E2, B.E1, B.E2] in the unknowns (x_s, x_t, x_{t+1}, x_e).
// ---------------------------------------------------------------------------
template <class G>
__device__ __forceinline__ Eq2 merge(const Eq2& A, const Eq2& B, int64_t row_t, G& bad,
                                     MergeSave& sv) {
    Eq2 P;
    // up-sweep: seed row 2 (= B.E1), then row 1 (= A.E2), then row 0 (= A.E1)
    bad.see(B.b1, row_t + 1);
    const double w1 = A.g2 * rcp(B.b1);
    const double beta1 = A.b2 - w1 * B.a1;
    const double gamma1 = -w1 * B.g1;
    const double delta1 = A.d2 - w1 * B.d1;
    bad.see(beta1, row_t);
    const double r1 = rcp(beta1);
    const double w0 = A.g1 * r1;
    P.a1 = A.a1;
    P.b1 = A.b1 - w0 * A.a2;
    P.g1 = -w0 * gamma1;
    P.d1 = A.d1 - w0 * delta1;
    // down-sweep: seed row 1 (= A.E2), then rows 2, 3
    bad.see(A.b2, row_t);
    const double w2 = B.a1 * rcp(A.b2);
    const double phi = -w2 * A.a2;
    const double bp = B.b1 - w2 * A.g2;
    const double dp = B.d1 - w2 * A.d2;
    bad.see(bp, row_t + 1);
    const double w3 = B.a2 * rcp(bp);
    P.a2 = -w3 * phi;
    P.b2 = B.b2 - w3 * B.g1;
    P.g2 = B.g2;
    P.d2 = B.d2 - w3 * dp;
    sv.d1 = delta1;
    sv.g1 = gamma1;
    sv.r1 = r1;
    sv.a2 = A.a2;
    return P;
}

// Top-down at a merge node: x_t from the saved up-sweep row (back_substitute).
__device__ __forceinline__ double merge_xt(const MergeSave& sv, double xs, double xe) {
    return (sv.d1 - sv.a2 * xs - sv.g1 * xe) * sv.r1;
}
// x_{t+1} = first row of B from its E1, given x_t and x_e.
__device__ __forceinline__ double first_from_e1(const Eq2& B, double xt, double xe) {
    return (B.d1 - B.a1 * xt - B.g1 * xe) * rcp(B.b1);
}

// Solve the 2x2 root system of a whole (non-coupled) system by Thomas
// (tridiagonal.hpp:52-72 on [E1; E2]); sub of row 0 / super of row 1 ignored,
// exactly as thomas_solve never reads sub[0] and drops c'_{n-1}.
template <class G>
__device__ __forceinline__ void root_solve(const Eq2& q, int64_t row_last, G& bad,
                                           double& x0, double& x1) {
    bad.see(q.b1, 0);
    const double r0 = rcp(q.b1);
    const double cm = q.g1 * r0;
    const double xp = q.d1 * r0;
    const double piv = q.b2 - q.a2 * cm;
    bad.see(piv, row_last);
    x1 = (q.d2 - q.a2 * xp) * rcp(piv);
    x0 = xp - cm * x1;
}

__device__ __forceinline__ Eq2 shfl_down_eq(const Eq2& q, int delta) {
    Eq2 r;
    r.a1 = __shfl_down_sync(0xffffffffu, q.a1, delta);
    r.b1 = __shfl_down_sync(0xffffffffu, q.b1, delta);
    r.g1 = __shfl_down_sync(0xffffffffu, q.g1, delta);
    r.d1 = __shfl_down_sync(0xffffffffu, q.d1, delta);
    r.a2 = __shfl_down_sync(0xffffffffu, q.a2, delta);
    r.b2 = __shfl_down_sync(0xffffffffu, q.b2, delta);
    r.g2 = __shfl_down_sync(0xffffffffu, q.g2, delta);
    r.d2 = __shfl_down_sync(0xffffffffu, q.d2, delta);
    return r;
}

// ---------------------------------------------------------------------------
// Vectorised register loads/stores (256-bit LDG/STG on sm_100a).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ld4(const double* p, double& x0, double& x1, double& x2,
                                    double& x3) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(x0), "=d"(x1), "=d"(x2), "=d"(x3)
                 : "l"(p));
}
__device__ __forceinline__ void st4(double* p, double x0, double x1, double x2, double x3) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(x0), "d"(x1), "d"(x2),
                 "d"(x3)
                 : "memory");
}

template <int L, bool VEC>
__device__ __forceinline__ void load_rows(const double* __restrict__ p, int64_t r0, double (&v)[L]) {
    if constexpr (VEC && (L % 4 == 0)) {
#pragma unroll
        for (int q = 0; q < L / 4; ++q) ld4(p + r0 + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < L; ++i) v[i] = __ldg(p + r0 + i);
    }
}

template <int L, bool VEC>
__device__ __forceinline__ void store_rows(double* __restrict__ p, int64_t r0, const double (&v)[L]) {
    if constexpr (VEC && (L % 4 == 0)) {
#pragma unroll
        for (int q = 0; q < L / 4; ++q) st4(p + r0 + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < L; ++i) p[r0 + i] = v[i];
    }
}

}  // namespace tpb
