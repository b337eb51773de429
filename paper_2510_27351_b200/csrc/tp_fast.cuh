// Fast-path kernels (included by tp_kernels.cu and the tuning harnesses).
//
//   k_fast<L,G,MODE>        one partition level, full blocks of m = L*G rows
#pragma once
#include "tp_device.cuh"

namespace tpb {

constexpr int log2_of(int g) { return g >= 32 ? 5 : g >= 16 ? 4 : g >= 8 ? 3 : g >= 4 ? 2 : g >= 2 ? 1 : 0; }

// Registers of one lane: its chunk of L rows, the leaf sweep values kept for
// back-substitution (Stage 3 only), the lane-tree saves and the running pair.
template <int L, int G, bool KEEP>
struct LaneState {
    static constexpr int LOGG = log2_of(G);
    Chunk<L> r;
    double rbeta[KEEP ? L : 1], gam[KEEP ? L : 1], del[KEEP ? L : 1];
    MergeSave sv[LOGG > 0 ? LOGG : 1];
    Eq2 cur;
    MinGuard guard;
};

template <int L, bool VEC>
__device__ __forceinline__ void load_chunk(const SysPtrs& sys, int64_t row0, bool active, Chunk<L>& r) {
    if (active) {
        load_rows<L, VEC>(sys.sub, row0, r.a);
        load_rows<L, VEC>(sys.diag, row0, r.b);
        load_rows<L, VEC>(sys.sup, row0, r.c);
        load_rows<L, VEC>(sys.rhs, row0, r.d);
    } else {
#pragma unroll
        for (int i = 0; i < L; ++i) { r.a[i] = 0; r.b[i] = 1; r.c[i] = 0; r.d[i] = 0; }
    }
}

// Leaf sweeps + the G-lane merge tree; the block's pair ends up in lane c == 0.
template <int L, int G, bool KEEP, int K = L>
__device__ __forceinline__ void lane_leaf(LaneState<L, G, KEEP>& s, int64_t row0) {
    if constexpr (KEEP) {
        s.cur = leaf_reduce_keep<L, K>(s.r, row0, s.guard, s.rbeta, s.gam, s.del);
    } else {
        s.cur = leaf_reduce<L, K>(s.r, row0, s.guard);
    }
}

template <int L, int G, bool KEEP>
__device__ __forceinline__ void lanes_tree(LaneState<L, G, KEEP>& s, int c, int64_t row0) {
    constexpr int LOGG = LaneState<L, G, KEEP>::LOGG;
#pragma unroll
    for (int lv = 0; lv < LOGG; ++lv) {
        const int h = 1 << lv;
        const Eq2 oth = shfl_down_eq(s.cur, h);
        if ((c & (2 * h - 1)) == 0) s.cur = merge(s.cur, oth, row0 + (int64_t)h * L - 1, s.guard, s.sv[lv]);
    }
}

template <int L, int G, bool KEEP>
__device__ __forceinline__ void lanes_up(LaneState<L, G, KEEP>& s, int c, int64_t row0) {
    lane_leaf<L, G, KEEP>(s, row0);
    lanes_tree<L, G, KEEP>(s, c, row0);
}

// Top-down from the block ends (held by lane c == 0) and the chunk's
// back-substitution; returns the chunk's L solution values.
template <int L, int G>
__device__ __forceinline__ void lanes_tree_down(LaneState<L, G, true>& s, int c, double& xs, double& xe) {
    constexpr int LOGG = LaneState<L, G, true>::LOGG;
#pragma unroll
    for (int lv = LOGG - 1; lv >= 0; --lv) {
        const int h = 1 << lv;
        double xt = 0;
        if ((c & (2 * h - 1)) == 0) xt = merge_xt(s.sv[lv], xs, xe);
        const double rxt = __shfl_up_sync(0xffffffffu, xt, h);
        const double rxe = __shfl_up_sync(0xffffffffu, xe, h);
        if ((c & (2 * h - 1)) == h) {
            xs = first_from_e1(s.cur, rxt, rxe);
            xe = rxe;
        } else if ((c & (2 * h - 1)) == 0) {
            xe = xt;
        }
    }
}

template <int L, int G>
__device__ __forceinline__ void lanes_down(LaneState<L, G, true>& s, int c, double xs, double xe,
                                           double (&xv)[L]) {
    lanes_tree_down<L, G>(s, c, xs, xe);
    leaf_expand<L, L>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv);
}

// ===========================================================================
// One level, full blocks of m = L*G rows, one chunk of L rows per thread held
// in registers, G lanes per block (G | 32), lane-tree merges via shuffles.
// ===========================================================================
template <int L, int G, int MODE, bool VEC, int THREADS = kFastThreads, int MINB = 1>
__global__ void __launch_bounds__(THREADS, MINB) k_fast(SysPtrs sys, int64_t nblocks, IfacePtrs out,
                                                       const double* __restrict__ xi,
                                                       double* __restrict__ x,
                                                       unsigned long long* err, int level) {
    static_assert(32 % G == 0, "G must divide the warp");
    constexpr bool KEEP = (MODE != kStage1);
    const int64_t nchunks = nblocks * G;
    const int lane = threadIdx.x & 31;
    const int c = lane % G;  // chunk index inside the block
    int64_t bad = INT64_MAX;

    for (int64_t base = (int64_t)blockIdx.x * THREADS; base < nchunks;
         base += (int64_t)gridDim.x * THREADS) {
        const int64_t t = base + threadIdx.x;
        // warp-uniform liveness: groups never straddle the nchunks boundary
        const bool active = t < nchunks;
        const int64_t row0 = t * L;
        const int64_t blk = t / G;
        LaneState<L, G, KEEP> s;
        load_chunk<L, VEC>(sys, row0, active, s.r);
        lanes_up<L, G, KEEP>(s, c, row0);
        if constexpr (MODE == kStage1) {
            if (active) {
                if (s.guard.tripped()) bad = row0 < bad ? row0 : bad;
                if (c == 0) {
                    const int64_t o = 2 * blk;
                    *reinterpret_cast<double2*>(out.sub + o) = make_double2(s.cur.a1, s.cur.a2);
                    *reinterpret_cast<double2*>(out.diag + o) = make_double2(s.cur.b1, s.cur.b2);
                    *reinterpret_cast<double2*>(out.sup + o) = make_double2(s.cur.g1, s.cur.g2);
                    *reinterpret_cast<double2*>(out.rhs + o) = make_double2(s.cur.d1, s.cur.d2);
                }
            }
        } else {
            // block ends from the next level's solution
            double xs = 0, xe = 0;
            if (c == 0 && active) {
                const double2 v = *reinterpret_cast<const double2*>(xi + 2 * blk);
                xs = v.x;
                xe = v.y;
            }
            double xv[L];
            lanes_down<L, G>(s, c, xs, xe, xv);
            if (active) {
                if (s.guard.tripped()) bad = row0 < bad ? row0 : bad;
                store_rows<L, VEC>(x, row0, xv);
            }
        }
    }
    report_pivot(err, level, bad);
}

// ===========================================================================
// Any block length m in [2G, LMAX*G] (full blocks): G lanes per block, lane c
// owns floor(m/G) or floor(m/G)+1 rows (runtime), held in registers sized
// LMAX with predicated scalar loads/stores. Covers every m <= 256 without a
// k_fast shape (e.g. the sweep candidates 25, 35, 50, 100, 125, 250).
// ===========================================================================
template <int LMAX, int G, int MODE>
__global__ void __launch_bounds__(128, (MODE == kStage1) ? 6 : 4)
    k_fast_rt(SysPtrs sys, int64_t nblocks, int64_t m, IfacePtrs out, const double* __restrict__ xi,
              double* __restrict__ x, unsigned long long* err, int level) {
    static_assert(32 % G == 0, "G must divide the warp");
    constexpr bool KEEP = (MODE != kStage1);
    constexpr int THREADS = 128;
    const int64_t nchunks = nblocks * G;
    const int c = (threadIdx.x & 31) % G;
    const int llo = (int)(m / G), ext = (int)(m % G);
    const int len = llo + (c < ext ? 1 : 0);
    const int off = c * llo + (c < ext ? c : ext);
    int64_t bad = INT64_MAX;

    for (int64_t base = (int64_t)blockIdx.x * THREADS; base < nchunks;
         base += (int64_t)gridDim.x * THREADS) {
        const int64_t t = base + threadIdx.x;
        const bool active = t < nchunks;
        const int64_t blk = t / G;
        const int64_t row0 = blk * m + off;
        LaneState<LMAX, G, KEEP> s;
#pragma unroll
        for (int i = 0; i < LMAX; ++i) {
            const bool live = active && i < len;
            s.r.a[i] = live ? __ldg(sys.sub + row0 + i) : 0.0;
            s.r.b[i] = live ? __ldg(sys.diag + row0 + i) : 1.0;
            s.r.c[i] = live ? __ldg(sys.sup + row0 + i) : 0.0;
            s.r.d[i] = live ? __ldg(sys.rhs + row0 + i) : 0.0;
        }
        // leaf on the runtime length: one compile-time instance per length, no
        // dynamic register indexing (lanes of a warp take at most two cases)
        switch (len) {
            case 2: lane_leaf<LMAX, G, KEEP, 2>(s, row0); break;
            case 3: lane_leaf<LMAX, G, KEEP, 3>(s, row0); break;
            case 4: lane_leaf<LMAX, G, KEEP, 4>(s, row0); break;
            case 5: lane_leaf<LMAX, G, KEEP, 5>(s, row0); break;
            case 6: lane_leaf<LMAX, G, KEEP, 6>(s, row0); break;
            case 7: lane_leaf<LMAX, G, KEEP, 7>(s, row0); break;
            default: lane_leaf<LMAX, G, KEEP, LMAX>(s, row0); break;
        }
        lanes_tree<LMAX, G, KEEP>(s, c, row0);
        if constexpr (MODE == kStage1) {
            if (active) {
                if (s.guard.tripped()) bad = row0 < bad ? row0 : bad;
                if (c == 0) {
                    const int64_t o = 2 * blk;
                    *reinterpret_cast<double2*>(out.sub + o) = make_double2(s.cur.a1, s.cur.a2);
                    *reinterpret_cast<double2*>(out.diag + o) = make_double2(s.cur.b1, s.cur.b2);
                    *reinterpret_cast<double2*>(out.sup + o) = make_double2(s.cur.g1, s.cur.g2);
                    *reinterpret_cast<double2*>(out.rhs + o) = make_double2(s.cur.d1, s.cur.d2);
                }
            }
        } else {
            double xs = 0, xe = 0;
            if (c == 0 && active) {
                const double2 v = *reinterpret_cast<const double2*>(xi + 2 * blk);
                xs = v.x;
                xe = v.y;
            }
            double xv[LMAX];
            lanes_tree_down<LMAX, G>(s, c, xs, xe);
            switch (len) {
                case 2: leaf_expand<LMAX, 2>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 3: leaf_expand<LMAX, 3>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 4: leaf_expand<LMAX, 4>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 5: leaf_expand<LMAX, 5>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 6: leaf_expand<LMAX, 6>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 7: leaf_expand<LMAX, 7>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                default: leaf_expand<LMAX, LMAX>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
            }
            if (active) {
                if (s.guard.tripped()) bad = row0 < bad ? row0 : bad;
#pragma unroll
                for (int i = 0; i < LMAX; ++i)
                    if (i < len) x[row0 + i] = xv[i];
            }
        }
    }
    report_pivot(err, level, bad);
}

}  // namespace tpb
