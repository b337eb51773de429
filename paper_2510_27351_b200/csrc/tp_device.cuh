// Device building blocks of the B200 partition solver (T = double or float,
// as the reference's TridiagonalSystem<Real> / solve_partition<Real>).
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

// kPivotFloor<Real> = Real(1e-30) — tridiagonal.hpp:15-16
template <class T>
__device__ __forceinline__ T pivot_floor() { return T(1e-30); }

template <class T>
struct Eq2 {
    T a1, b1, g1, d1;  // E1
    T a2, b2, g2, d2;  // E2
};

// Saved per merge for the top-down pass: x_t = (d1 - a2*x_s - g1*x_e) * r1
template <class T>
struct MergeSave {
    T d1, g1, r1, a2;
};

// Reciprocals: MUFU seed + one Newton-type step, <= 1 ulp from the correctly
// rounded 1/x (FP64 checked on the GPU by tp_diag_rcp_ulp); no slow path,
// because every pivot they see passed the |p| >= 1e-30 floor check (or is
// already reported as a zero pivot). w = c * rcp(p) replaces the reference's
// c / p (<= ~2 ulp apart; parity is by tolerance).
__device__ __forceinline__ double rcp(double x) {
    // seed error e0 ~ 2^-22; r*(1 + e + e^2) leaves ~e0^3 before rounding
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ float rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return fmaf(r, fmaf(-x, r, 1.0f), r);
}

// Zero-pivot bookkeeping (|pivot| < kPivotFloor -> ZeroPivotError).
// RowGuard remembers the smallest offending row (generic / finishing paths);
// MinGuard keeps only min|pivot| (one min per pivot on the hot path) and the
// caller reports the chunk's first row when it fell below the floor.
struct RowGuard {
    int64_t bad = INT64_MAX;
    template <class T>
    __device__ __forceinline__ void see(T p, int64_t row) {
        if (fabs(p) < pivot_floor<T>()) bad = (row < bad) ? row : bad;
    }
};
template <class T>
struct MinGuard {
    T pmin = T(1.0e30);
    __device__ __forceinline__ void see(T p, int64_t) { pmin = fmin(pmin, fabs(p)); }
    __device__ __forceinline__ bool tripped() const { return pmin < pivot_floor<T>(); }
};

// Programmatic dependent launch. Every solve-path kernel starts with this:
// wait until the preceding grid in the stream has completed and its writes are
// visible (a no-op when launched without the PDL attribute), then let the next
// grid start launching so its CTAs are resident when this one drains.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Stage 3 of a level recomputes exactly the sweeps and merges Stage 1 ran on
// the same rows (bit-identical arithmetic), so every pivot it meets was already
// checked there: its kernels carry this no-op guard.
template <class T>
struct NoGuard {
    __device__ __forceinline__ void see(T, int64_t) {}
    __device__ __forceinline__ bool tripped() const { return false; }
};

// The same for the RowGuard-based (generic / finishing) kernels.
struct NoRowGuard {
    static constexpr int64_t bad = INT64_MAX;
    template <class T>
    __device__ __forceinline__ void see(T, int64_t) {}
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

// A solution value that is not finite: a singular system whose pivots the
// device order never saw below the floor (the reference's order may have).
// Reported with the lowest priority, so any pivot report wins.
__device__ __forceinline__ void report_nonfinite(unsigned long long* err, int64_t row) {
    if (err != nullptr)
        atomicMin(err, (static_cast<unsigned long long>(kNonFiniteLevel) << 48) |
                           (static_cast<unsigned long long>(row) & 0xFFFFFFFFFFFFULL));
}
template <class T, int L>
__device__ __forceinline__ bool any_nonfinite(const T (&v)[L], int len = L) {
    bool nf = false;
#pragma unroll
    for (int i = 0; i < L; ++i) nf |= (i < len) && !isfinite(v[i]);
    return nf;
}

// ---------------------------------------------------------------------------
// Leaf: one chunk held in registers sized L; its first K rows are valid
// (K == L on the fixed-shape path; k_fast_rt dispatches on a runtime length).
// up-sweep  = partition.hpp:90-108, down-sweep = partition.hpp:110-124.
// ---------------------------------------------------------------------------
template <class T, int L>
struct Chunk {
    T a[L], b[L], c[L], d[L];
};

// Stage-1 leaf: E1/E2 only (no per-row storage).
template <class T, int L, int len, class Gd>
__device__ __forceinline__ Eq2<T> leaf_reduce(const Chunk<T, L>& r, int64_t row0, Gd& bad) {
    Eq2<T> q;
    // up-sweep: seed row len-2, run i = len-3 .. 0
    T beta = 0, gamma = 0, delta = 0;
#pragma unroll
    for (int i = L - 2; i >= 0; --i) {
        if (i == len - 2) {
            beta = r.b[i];
            gamma = r.c[i];
            delta = r.d[i];
        } else if (i < len - 2) {
            bad.see(beta, row0 + i + 1);
            const T w = r.c[i] * rcp(beta);
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
    T phi = r.a[1], bp = r.b[1], dp = r.d[1];
    T glast = r.c[1];
#pragma unroll
    for (int i = 2; i < L; ++i) {
        if (i < len) {
            bad.see(bp, row0 + i - 1);
            const T w = r.a[i] * rcp(bp);
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
template <class T, int L, int len, class Gd>
__device__ __forceinline__ Eq2<T> leaf_reduce_keep(const Chunk<T, L>& r, int64_t row0, Gd& bad,
                                                   T (&rbeta)[L], T (&gam)[L], T (&del)[L]) {
    Eq2<T> q;
    T beta = 0, gamma = 0, delta = 0;
#pragma unroll
    for (int i = L - 2; i >= 0; --i) {
        if (i == len - 2) {
            beta = r.b[i];
            gamma = r.c[i];
            delta = r.d[i];
        } else if (i < len - 2) {
            bad.see(beta, row0 + i + 1);
            const T rb = rcp(beta);
            rbeta[i + 1] = rb;
            const T w = r.c[i] * rb;
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
    T phi = r.a[1], bp = r.b[1], dp = r.d[1];
    T glast = r.c[1];
#pragma unroll
    for (int i = 2; i < L; ++i) {
        if (i < len) {
            bad.see(bp, row0 + i - 1);
            const T w = r.a[i] * rcp(bp);
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
template <class T, int L, int len>
__device__ __forceinline__ void leaf_expand(const Chunk<T, L>& r, const T (&rbeta)[L],
                                            const T (&gam)[L], const T (&del)[L], T xs, T xe,
                                            T (&x)[L]) {
    x[0] = xs;
    T prev = xs;
#pragma unroll
    for (int i = 1; i < L; ++i) {
        if (i < len - 1) {
            const T xi = (del[i] - r.a[i] * prev - gam[i] * xe) * rbeta[i];
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
template <class T, class Gd>
__device__ __forceinline__ Eq2<T> merge(const Eq2<T>& A, const Eq2<T>& B, int64_t row_t, Gd& bad,
                                        MergeSave<T>& sv) {
    Eq2<T> P;
    // up-sweep: seed row 2 (= B.E1), then row 1 (= A.E2), then row 0 (= A.E1)
    bad.see(B.b1, row_t + 1);
    const T w1 = A.g2 * rcp(B.b1);
    const T beta1 = A.b2 - w1 * B.a1;
    const T gamma1 = -w1 * B.g1;
    const T delta1 = A.d2 - w1 * B.d1;
    bad.see(beta1, row_t);
    const T r1 = rcp(beta1);
    const T w0 = A.g1 * r1;
    P.a1 = A.a1;
    P.b1 = A.b1 - w0 * A.a2;
    P.g1 = -w0 * gamma1;
    P.d1 = A.d1 - w0 * delta1;
    // down-sweep: seed row 1 (= A.E2), then rows 2, 3
    bad.see(A.b2, row_t);
    const T w2 = B.a1 * rcp(A.b2);
    const T phi = -w2 * A.a2;
    const T bp = B.b1 - w2 * A.g2;
    const T dp = B.d1 - w2 * A.d2;
    bad.see(bp, row_t + 1);
    const T w3 = B.a2 * rcp(bp);
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
template <class T>
__device__ __forceinline__ T merge_xt(const MergeSave<T>& sv, T xs, T xe) {
    return (sv.d1 - sv.a2 * xs - sv.g1 * xe) * sv.r1;
}
// x_{t+1} = first row of B from its E1, given x_t and x_e.
template <class T>
__device__ __forceinline__ T first_from_e1(const Eq2<T>& B, T xt, T xe) {
    return (B.d1 - B.a1 * xt - B.g1 * xe) * rcp(B.b1);
}

// ---------------------------------------------------------------------------
// The same merge as ONE 2x2 elimination (Schur complement of the middle
// block): A.E2 and B.E1 couple the middle unknowns (x_t, x_{t+1}) through
//   [A.b2 A.g2; B.a1 B.b1] [x_t; x_{t+1}] = [A.d2 - A.a2 x_s; B.d1 - B.g1 x_e],
// det = A.b2 B.b1 - A.g2 B.a1 = B.b1 * beta1 = A.b2 * bp (the pivots of the
// up- and down-sweep of `merge`). One reciprocal instead of four: the merged
// rows are ready after det -> rcp -> one FMA (~90 dependent cycles against
// ~150 for `merge`), and the top-down step needs no reciprocal at all:
//   x_t     = sd - sa x_s + sg x_e,    x_{t+1} = ud + ua x_s - ug x_e.
// The pivot check sees the same four pivots as `merge` (B.b1, A.b2 directly,
// beta1 and bp through det), off the critical path; `flag` records a failure.
// ---------------------------------------------------------------------------
template <class T>
struct SchurSave {
    T sd, sa, sg, ud, ua, ug;
};

template <class T>
__device__ __forceinline__ Eq2<T> merge_schur(const Eq2<T>& A, const Eq2<T>& B, bool& flag, SchurSave<T>& sv) {
    const T det = fma(A.b2, B.b1, -(A.g2 * B.a1));
    const T r = rcp(det);
    const T fl = pivot_floor<T>();
    flag |= (fabs(B.b1) < fl) | (fabs(A.b2) < fl) | (fabs(det) < fl * fabs(B.b1)) | (fabs(det) < fl * fabs(A.b2));
    sv.sd = fma(B.b1, A.d2, -(A.g2 * B.d1)) * r;
    sv.sa = (B.b1 * A.a2) * r;
    sv.sg = (A.g2 * B.g1) * r;
    sv.ud = fma(A.b2, B.d1, -(B.a1 * A.d2)) * r;
    sv.ua = (B.a1 * A.a2) * r;
    sv.ug = (A.b2 * B.g1) * r;
    Eq2<T> P;
    P.a1 = A.a1;
    P.b1 = fma(-A.g1, sv.sa, A.b1);
    P.g1 = A.g1 * sv.sg;
    P.d1 = fma(-A.g1, sv.sd, A.d1);
    P.a2 = B.a2 * sv.ua;
    P.b2 = fma(-B.a2, sv.ug, B.b2);
    P.g2 = B.g2;
    P.d2 = fma(-B.a2, sv.ud, B.d2);
    return P;
}
// merge_schur with RowGuard bookkeeping (the merge's row for the report).
template <class T>
__device__ __forceinline__ Eq2<T> merge_schur_row(const Eq2<T>& A, const Eq2<T>& B, int64_t row_t, RowGuard& bad,
                                                  SchurSave<T>& sv) {
    bool f = false;
    const Eq2<T> P = merge_schur(A, B, f, sv);
    if (f) bad.bad = row_t < bad.bad ? row_t : bad.bad;
    return P;
}
template <class T>
__device__ __forceinline__ void schur_down(const SchurSave<T>& sv, T xs, T xe, T& xt, T& xt1) {
    xt = fma(sv.sg, xe, fma(-sv.sa, xs, sv.sd));
    xt1 = fma(-sv.ug, xe, fma(sv.ua, xs, sv.ud));
}

// Solve the 2x2 root system of a whole (non-coupled) system by Thomas
// (tridiagonal.hpp:52-72 on [E1; E2]); sub of row 0 / super of row 1 ignored,
// exactly as thomas_solve never reads sub[0] and drops c'_{n-1}.
template <class T, class Gd>
__device__ __forceinline__ void root_solve(const Eq2<T>& q, int64_t row_last, Gd& bad, T& x0, T& x1) {
    bad.see(q.b1, 0);
    const T r0 = rcp(q.b1);
    const T cm = q.g1 * r0;
    const T xp = q.d1 * r0;
    const T piv = q.b2 - q.a2 * cm;
    bad.see(piv, row_last);
    x1 = (q.d2 - q.a2 * xp) * rcp(piv);
    x0 = xp - cm * x1;
}

template <class T>
__device__ __forceinline__ Eq2<T> shfl_down_eq(const Eq2<T>& q, int delta) {
    Eq2<T> r;
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
// Vectorised register loads/stores: 256-bit LDG/STG on sm_100a (4 doubles or
// 8 floats per instruction).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ld256(const double* p, double* v) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p));
}
__device__ __forceinline__ void ld256(const float* p, float* v) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                   "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}
__device__ __forceinline__ void st256(double* p, const double* v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]),
                 "d"(v[3])
                 : "memory");
}
__device__ __forceinline__ void st256(float* p, const float* v) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

// rows per 256-bit access
template <class T>
__host__ __device__ constexpr int vec_rows() { return 32 / (int)sizeof(T); }

template <class T, int L, bool VEC>
__device__ __forceinline__ void load_rows(const T* __restrict__ p, int64_t r0, T (&v)[L]) {
    constexpr int W = vec_rows<T>();
    if constexpr (VEC && (L % W == 0)) {
#pragma unroll
        for (int q = 0; q < L / W; ++q) ld256(p + r0 + W * q, v + W * q);
    } else {
#pragma unroll
        for (int i = 0; i < L; ++i) v[i] = __ldg(p + r0 + i);
    }
}

template <class T, int L, bool VEC>
__device__ __forceinline__ void store_rows(T* __restrict__ p, int64_t r0, const T (&v)[L]) {
    constexpr int W = vec_rows<T>();
    if constexpr (VEC && (L % W == 0)) {
#pragma unroll
        for (int q = 0; q < L / W; ++q) st256(p + r0 + W * q, v + W * q);
    } else {
#pragma unroll
        for (int i = 0; i < L; ++i) p[r0 + i] = v[i];
    }
}

// Two consecutive values (an interface row pair / a block's ends) as one
// vector access.
__device__ __forceinline__ void store_pair(double* p, double x0, double x1) {
    *reinterpret_cast<double2*>(p) = make_double2(x0, x1);
}
__device__ __forceinline__ void store_pair(float* p, float x0, float x1) {
    *reinterpret_cast<float2*>(p) = make_float2(x0, x1);
}
template <class T>
struct Pair {
    T x, y;
};
__device__ __forceinline__ Pair<double> load_pair(const double* p) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    return {v.x, v.y};
}
__device__ __forceinline__ Pair<float> load_pair(const float* p) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    return {v.x, v.y};
}

}  // namespace tpb
