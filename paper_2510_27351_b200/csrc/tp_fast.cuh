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
template <int L, int G, bool KEEP>
__device__ __forceinline__ void lanes_up(LaneState<L, G, KEEP>& s, int c, int64_t row0) {
    constexpr int LOGG = LaneState<L, G, KEEP>::LOGG;
    if constexpr (KEEP) {
        s.cur = leaf_reduce_keep<L>(s.r, L, row0, s.guard, s.rbeta, s.gam, s.del);
    } else {
        s.cur = leaf_reduce<L>(s.r, L, row0, s.guard);
    }
#pragma unroll
    for (int lv = 0; lv < LOGG; ++lv) {
        const int h = 1 << lv;
        const Eq2 oth = shfl_down_eq(s.cur, h);
        if ((c & (2 * h - 1)) == 0) s.cur = merge(s.cur, oth, row0 + (int64_t)h * L - 1, s.guard, s.sv[lv]);
    }
}

// Top-down from the block ends (held by lane c == 0) and the chunk's
// back-substitution; returns the chunk's L solution values.
template <int L, int G>
__device__ __forceinline__ void lanes_down(LaneState<L, G, true>& s, int c, double xs, double xe,
                                           double (&xv)[L]) {
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
    leaf_expand<L>(s.r, L, s.rbeta, s.gam, s.del, xs, xe, xv);
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

}  // namespace tpb
