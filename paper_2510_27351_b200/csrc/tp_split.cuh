// Long-block path (k_split) and the reference-order sweeps (k_ref_sweep,
// k_ref_thomas). Included by tp_kernels.cu.
//
// k_split: one partition level whose blocks are too long for shared-memory
// staging (k_generic holds a whole block in shared memory). The planner
// (tp_capi.cu build_plan) replaces such a level by a chain:
//   split level   every block of blen rows is cut into nsub = ceil(blen / 8)
//                 chunks of 7..8 rows; each thread reduces ONE chunk to its
//                 E1/E2 pair (the same leaf sweeps as every other level,
//                 partition.hpp:90-124) and writes it as two rows of a finer
//                 system, in row order;
//   merge level   that finer system partitioned with the ORIGINAL block
//                 boundaries (2 nsub rows per block): its interface is the
//                 original level's interface, because E1/E2 of a segment are
//                 unique once its outer couplings (sub[s], super[e]) are fixed
//                 (tp_device.cuh: a merge IS reduce_block on [A.E1 A.E2 B.E1 B.E2]).
// The merge level is split again while its blocks are still too long. Stage 3
// runs the chain backwards: the merge level recovers every chunk's end rows,
// k_split<kStage3> re-sweeps each chunk and back-substitutes its interior
// (partition.hpp:156-172).
//
// k_ref_sweep / k_ref_thomas: the reference's own sequential arithmetic
// (reduce_block partition.hpp:77-126, thomas_solve tridiagonal.hpp:52-72) —
// one thread per block, IEEE division, every product and difference rounded
// separately (__dmul_rn / __dsub_rn: no FMA contraction, as the reference's
// x86-64 build). Used (1) when a solve reports a zero pivot, to find the row
// the reference reports, in its order (block by block, up-sweep rows e-1 .. s+1
// then down-sweep rows s+1 .. e-1), and (2) by the C-ABI stage entry point
// tp_reduce_blocks_* (reduce_block with the stored up-sweep vectors).
#pragma once
#include "tp_fast.cuh"

namespace tpb {

template <class T, int MODE>
__global__ void __launch_bounds__(128, 4)
    k_split(SysPtrs<T> sys, int64_t row_base, int64_t nblocks, int64_t blen, int64_t nsub, int64_t q_base,
            IfacePtrs<T> out, const T* __restrict__ xi, T* __restrict__ x, unsigned long long* err, int level) {
    constexpr int LMAX = kSplitRows;
    constexpr bool KEEP = (MODE != kStage1);
    const int64_t nchunks = nblocks * nsub;
    const int64_t llo = blen / nsub, ext = blen % nsub;
    pdl_begin();
    for (int64_t t = (int64_t)blockIdx.x * 128 + threadIdx.x; t < nchunks; t += (int64_t)gridDim.x * 128) {
        const int64_t j = t / nsub;
        const int64_t c = t - j * nsub;
        const int len = (int)(llo + (c < ext ? 1 : 0));
        const int64_t row0 = row_base + j * blen + c * llo + (c < ext ? c : ext);
        const int64_t q = q_base + t;  // chunk index = row pair of the finer system
        LaneState<T, LMAX, 1, KEEP> s;
        T xs = 0, xe = 0;
        if constexpr (MODE != kStage1) {
            const Pair<T> v = load_pair(xi + 2 * q);
            xs = v.x;
            xe = v.y;
        }
#pragma unroll
        for (int i = 0; i < LMAX; ++i) {
            const bool live = i < len;
            s.r.a[i] = live ? __ldg(sys.sub + row0 + i) : T(0);
            s.r.b[i] = live ? __ldg(sys.diag + row0 + i) : T(1);
            s.r.c[i] = live ? __ldg(sys.sup + row0 + i) : T(0);
            s.r.d[i] = live ? __ldg(sys.rhs + row0 + i) : T(0);
        }
        switch (len) {
            case 2: lane_leaf<T, LMAX, 1, KEEP, 2>(s, row0); break;
            case 3: lane_leaf<T, LMAX, 1, KEEP, 3>(s, row0); break;
            case 4: lane_leaf<T, LMAX, 1, KEEP, 4>(s, row0); break;
            case 5: lane_leaf<T, LMAX, 1, KEEP, 5>(s, row0); break;
            case 6: lane_leaf<T, LMAX, 1, KEEP, 6>(s, row0); break;
            case 7: lane_leaf<T, LMAX, 1, KEEP, 7>(s, row0); break;
            default: lane_leaf<T, LMAX, 1, KEEP, LMAX>(s, row0); break;
        }
        if constexpr (MODE == kStage1) {
            if (s.guard.tripped()) report_pivot(err, level, row0);
            store_block_eqs(out, q, s.cur);
        } else {
            T xv[LMAX];
            switch (len) {
                case 2: leaf_expand<T, LMAX, 2>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 3: leaf_expand<T, LMAX, 3>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 4: leaf_expand<T, LMAX, 4>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 5: leaf_expand<T, LMAX, 5>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 6: leaf_expand<T, LMAX, 6>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 7: leaf_expand<T, LMAX, 7>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                default: leaf_expand<T, LMAX, LMAX>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
            }
#pragma unroll
            for (int i = 0; i < LMAX; ++i)
                if (i < len) x[row0 + i] = xv[i];
            if (any_nonfinite(xv, len)) report_nonfinite(err, row0);
        }
    }
}

// ---------------------------------------------------------------------------
// Reference-order arithmetic: a op b rounded once per operation.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double r_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double r_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double r_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float r_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float r_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float r_div(float a, float b) { return __fdiv_rn(a, b); }

// reduce_block (partition.hpp:77-126) on blocks [bounds_j, bounds_{j+1}) of
// make_plan(n, m): full blocks of m rows, the last one ends at n. One thread
// per block. Returns through `first` the block's first failing pivot row in
// the reference's order (-1 = none). With STORE, also the interface pair
// (eq8[8 j ..]: alpha1 beta1 gamma1 delta1 alpha2 beta2 gamma2 delta2) and the
// up-sweep vectors a / beta / gamma / delta by system row (ReducedBlock).
template <class T, bool STORE>
__global__ void k_ref_sweep(SysPtrs<T> sys, int64_t n, int64_t m, int64_t K, int64_t* __restrict__ first,
                            unsigned long long* jmin, T* __restrict__ eq8, T* __restrict__ ua,
                            T* __restrict__ ubeta, T* __restrict__ ugamma, T* __restrict__ udelta) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = j * m;
        const int64_t e = (j == K - 1) ? n - 1 : s + m - 1;
        int64_t bad = -1;
        // up-sweep: seed row e-1, i = e-2 .. s (partition.hpp:89-104)
        T beta = sys.diag[e - 1], gamma = sys.sup[e - 1], delta = sys.rhs[e - 1];
        if (STORE) { ua[e - 1] = sys.sub[e - 1]; ubeta[e - 1] = beta; ugamma[e - 1] = gamma; udelta[e - 1] = delta; }
        for (int64_t i = e - 1; i-- > s;) {
            if (fabs(beta) < pivot_floor<T>()) { bad = i + 1; break; }
            const T w = r_div(sys.sup[i], beta);
            beta = r_sub(sys.diag[i], r_mul(w, sys.sub[i + 1]));
            gamma = -r_mul(w, gamma);
            delta = r_sub(sys.rhs[i], r_mul(w, delta));
            if (STORE) { ua[i] = sys.sub[i]; ubeta[i] = beta; ugamma[i] = gamma; udelta[i] = delta; }
        }
        T eq[8];
        eq[0] = sys.sub[s]; eq[1] = beta; eq[2] = gamma; eq[3] = delta;
        if (bad < 0) {
            // down-sweep: seed row s+1, i = s+2 .. e (partition.hpp:110-120)
            T phi = sys.sub[s + 1], bp = sys.diag[s + 1], dp = sys.rhs[s + 1];
            for (int64_t i = s + 2; i <= e; ++i) {
                if (fabs(bp) < pivot_floor<T>()) { bad = i - 1; break; }
                const T w = r_div(sys.sub[i], bp);
                phi = -r_mul(w, phi);
                bp = r_sub(sys.diag[i], r_mul(w, sys.sup[i - 1]));
                dp = r_sub(sys.rhs[i], r_mul(w, dp));
            }
            eq[4] = phi; eq[5] = bp; eq[6] = sys.sup[e]; eq[7] = dp;
        }
        if (first) first[j] = bad;
        if (bad >= 0 && jmin) atomicMin(jmin, (unsigned long long)j);
        if (STORE && eq8 && bad < 0)
            for (int k = 0; k < 8; ++k) eq8[8 * j + k] = eq[k];
    }
}

// thomas_solve's pivots (tridiagonal.hpp:52-72), one thread: the first row
// whose pivot is below the floor, or -1.
template <class T>
__global__ void k_ref_thomas(SysPtrs<T> sys, int64_t n, int64_t* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    T piv = sys.diag[0];
    if (fabs(piv) < pivot_floor<T>()) { *out = 0; return; }
    T cm = r_div(sys.sup[0], piv);
    for (int64_t i = 1; i < n; ++i) {
        piv = r_sub(sys.diag[i], r_mul(sys.sub[i], cm));
        if (fabs(piv) < pivot_floor<T>()) { *out = i; return; }
        cm = r_div(sys.sup[i], piv);
    }
    *out = -1;
}

}  // namespace tpb
