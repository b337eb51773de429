// Fast-path kernels (included by tp_kernels.cu and the tuning harnesses).
//
//   k_fast<T,L,G,MODE>       one partition level, full blocks of m = L*G rows
//   k_fast_rt<T,LMAX,G,MODE> one partition level, any m <= LMAX*G (runtime)
#pragma once
#include <type_traits>

#include "tp_device.cuh"

namespace tpb {

constexpr int log2_of(int g) { return g >= 32 ? 5 : g >= 16 ? 4 : g >= 8 ? 3 : g >= 4 ? 2 : g >= 2 ? 1 : 0; }

// Registers of one lane: its chunk of L rows, the leaf sweep values kept for
// back-substitution (Stage 3 only), the lane-tree saves and the running pair.
template <class T, int L, int G, bool KEEP>
struct LaneState {
    static constexpr int LOGG = log2_of(G);
    Chunk<T, L> r;
    T rbeta[KEEP ? L : 1], gam[KEEP ? L : 1], del[KEEP ? L : 1];
    MergeSave<T> sv[LOGG > 0 ? LOGG : 1];
    Eq2<T> cur;
    // Stage 1 checks every pivot; Stage 3 repeats the same arithmetic (NoGuard)
    typename std::conditional<KEEP, NoGuard<T>, MinGuard<T>>::type guard;
};

template <class T, int L, bool VEC>
__device__ __forceinline__ void load_chunk(const SysPtrs<T>& sys, int64_t row0, bool active,
                                           Chunk<T, L>& r) {
    if (active) {
        load_rows<T, L, VEC>(sys.sub, row0, r.a);
        load_rows<T, L, VEC>(sys.diag, row0, r.b);
        load_rows<T, L, VEC>(sys.sup, row0, r.c);
        load_rows<T, L, VEC>(sys.rhs, row0, r.d);
    } else {
#pragma unroll
        for (int i = 0; i < L; ++i) { r.a[i] = 0; r.b[i] = 1; r.c[i] = 0; r.d[i] = 0; }
    }
}

template <class T, int L, int G, bool KEEP, int K = L>
__device__ __forceinline__ void lane_leaf(LaneState<T, L, G, KEEP>& s, int64_t row0) {
    if constexpr (KEEP) {
        s.cur = leaf_reduce_keep<T, L, K>(s.r, row0, s.guard, s.rbeta, s.gam, s.del);
    } else {
        s.cur = leaf_reduce<T, L, K>(s.r, row0, s.guard);
    }
}

// The G-lane merge tree; the block's pair ends up in lane c == 0.
template <class T, int L, int G, bool KEEP>
__device__ __forceinline__ void lanes_tree(LaneState<T, L, G, KEEP>& s, int c, int64_t row0) {
    constexpr int LOGG = LaneState<T, L, G, KEEP>::LOGG;
#pragma unroll
    for (int lv = 0; lv < LOGG; ++lv) {
        const int h = 1 << lv;
        const Eq2<T> oth = shfl_down_eq(s.cur, h);
        if ((c & (2 * h - 1)) == 0) s.cur = merge(s.cur, oth, row0 + (int64_t)h * L - 1, s.guard, s.sv[lv]);
    }
}

// Top-down from the block ends (held by lane c == 0) to this lane's chunk ends.
template <class T, int L, int G>
__device__ __forceinline__ void lanes_tree_down(LaneState<T, L, G, true>& s, int c, T& xs, T& xe) {
    constexpr int LOGG = LaneState<T, L, G, true>::LOGG;
#pragma unroll
    for (int lv = LOGG - 1; lv >= 0; --lv) {
        const int h = 1 << lv;
        T xt = 0;
        if ((c & (2 * h - 1)) == 0) xt = merge_xt(s.sv[lv], xs, xe);
        const T rxt = __shfl_up_sync(0xffffffffu, xt, h);
        const T rxe = __shfl_up_sync(0xffffffffu, xe, h);
        if ((c & (2 * h - 1)) == h) {
            xs = first_from_e1(s.cur, rxt, rxe);
            xe = rxe;
        } else if ((c & (2 * h - 1)) == 0) {
            xe = xt;
        }
    }
}

template <class T>
__device__ __forceinline__ void store_block_eqs(const IfacePtrs<T>& out, int64_t blk, const Eq2<T>& q) {
    const int64_t o = 2 * blk;  // assemble_interface row order (partition.hpp:139-149)
    store_pair(out.sub + o, q.a1, q.a2);
    store_pair(out.diag + o, q.b1, q.b2);
    store_pair(out.sup + o, q.g1, q.g2);
    store_pair(out.rhs + o, q.d1, q.d2);
}

// ===========================================================================
// One level, full blocks of m = L*G rows, one chunk of L rows per thread held
// in registers, G lanes per block (G | 32), lane-tree merges via shuffles.
// ===========================================================================
template <class T, int L, int G, int MODE, bool VEC, int THREADS = kFastThreads, int MINB = 1>
__global__ void __launch_bounds__(THREADS, MINB)
    k_fast(SysPtrs<T> sys, int64_t nblocks, IfacePtrs<T> out, const T* __restrict__ xi,
           T* __restrict__ x, unsigned long long* err, int level) {
    static_assert(32 % G == 0, "G must divide the warp");
    constexpr bool KEEP = (MODE != kStage1);
    const int64_t nchunks = nblocks * G;
    const int lane = threadIdx.x & 31;
    const int c = lane % G;  // chunk index inside the block
    pdl_begin();

    // one chunk per thread: the launcher always sizes a full grid (no
    // grid-stride loop, whose carried indices spilled at the register cap)
    {
        const int64_t t = (int64_t)blockIdx.x * THREADS + threadIdx.x;
        // warp-uniform liveness: groups never straddle the nchunks boundary
        const bool active = t < nchunks;
        const int64_t row0 = t * L;
        const int64_t blk = t / G;
        LaneState<T, L, G, KEEP> s;
        load_chunk<T, L, VEC>(sys, row0, active, s.r);
        // Stage 3: the block's ends from the next level's solution, issued with
        // the row loads so its latency is off the sweep -> tree -> expand chain
        T xs = 0, xe = 0;
        if constexpr (MODE != kStage1) {
            if (c == 0 && active) {
                const Pair<T> v = load_pair(xi + 2 * blk);
                xs = v.x;
                xe = v.y;
            }
        }
        lane_leaf<T, L, G, KEEP>(s, row0);
        lanes_tree<T, L, G, KEEP>(s, c, row0);
        if constexpr (MODE == kStage1) {
            if (active) {
                // rare: report at once instead of carrying a row across the loop
                if (s.guard.tripped()) report_pivot(err, level, row0);
                if (c == 0) store_block_eqs(out, blk, s.cur);
            }
        } else {
            T xv[L];
            lanes_tree_down<T, L, G>(s, c, xs, xe);
            leaf_expand<T, L, L>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv);
            if (active) {
                store_rows<T, L, VEC>(x, row0, xv);  // pivots: checked by Stage 1
                if (any_nonfinite(xv)) report_nonfinite(err, row0);
            }
        }
    }
}

// ===========================================================================
// Any block length m in [2G, LMAX*G] (full blocks): G lanes per block, lane c
// owns floor(m/G) or floor(m/G)+1 rows (runtime), held in registers sized
// LMAX with predicated scalar loads/stores. Covers every m <= 256 without a
// k_fast shape (e.g. the sweep candidates 25, 35, 50, 100, 125, 250).
// ===========================================================================
template <class T, int LMAX, int G, int MODE>
__global__ void __launch_bounds__(128, (MODE == kStage1) ? 5 : 4)
    k_fast_rt(SysPtrs<T> sys, int64_t nblocks, int64_t m, IfacePtrs<T> out, const T* __restrict__ xi,
              T* __restrict__ x, unsigned long long* err, int level) {
    static_assert(32 % G == 0, "G must divide the warp");
    constexpr bool KEEP = (MODE != kStage1);
    constexpr int THREADS = 128;
    const int64_t nchunks = nblocks * G;
    const int c = (threadIdx.x & 31) % G;
    const int llo = (int)(m / G), ext = (int)(m % G);
    const int len = llo + (c < ext ? 1 : 0);
    const int off = c * llo + (c < ext ? c : ext);
    pdl_begin();

    {  // one chunk per thread (full grid, as k_fast)
        const int64_t t = (int64_t)blockIdx.x * THREADS + threadIdx.x;
        const bool active = t < nchunks;
        const int64_t blk = t / G;
        const int64_t row0 = blk * m + off;
        LaneState<T, LMAX, G, KEEP> s;
        T xs = 0, xe = 0;  // Stage 3 block ends, loaded with the rows (see k_fast)
        if constexpr (MODE != kStage1) {
            if (c == 0 && active) {
                const Pair<T> v = load_pair(xi + 2 * blk);
                xs = v.x;
                xe = v.y;
            }
        }
#pragma unroll
        for (int i = 0; i < LMAX; ++i) {
            const bool live = active && i < len;
            s.r.a[i] = live ? __ldg(sys.sub + row0 + i) : T(0);
            s.r.b[i] = live ? __ldg(sys.diag + row0 + i) : T(1);
            s.r.c[i] = live ? __ldg(sys.sup + row0 + i) : T(0);
            s.r.d[i] = live ? __ldg(sys.rhs + row0 + i) : T(0);
        }
        // leaf on the runtime length: one compile-time instance per length, no
        // dynamic register indexing (lanes of a warp take at most two cases)
        switch (len) {
            case 2: lane_leaf<T, LMAX, G, KEEP, 2>(s, row0); break;
            case 3: lane_leaf<T, LMAX, G, KEEP, 3>(s, row0); break;
            case 4: lane_leaf<T, LMAX, G, KEEP, 4>(s, row0); break;
            case 5: lane_leaf<T, LMAX, G, KEEP, 5>(s, row0); break;
            case 6: lane_leaf<T, LMAX, G, KEEP, 6>(s, row0); break;
            case 7: lane_leaf<T, LMAX, G, KEEP, 7>(s, row0); break;
            default: lane_leaf<T, LMAX, G, KEEP, LMAX>(s, row0); break;
        }
        lanes_tree<T, LMAX, G, KEEP>(s, c, row0);
        if constexpr (MODE == kStage1) {
            if (active) {
                if (s.guard.tripped()) report_pivot(err, level, row0);  // rare: report at once
                if (c == 0) store_block_eqs(out, blk, s.cur);
            }
        } else {
            T xv[LMAX];
            lanes_tree_down<T, LMAX, G>(s, c, xs, xe);
            switch (len) {
                case 2: leaf_expand<T, LMAX, 2>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 3: leaf_expand<T, LMAX, 3>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 4: leaf_expand<T, LMAX, 4>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 5: leaf_expand<T, LMAX, 5>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 6: leaf_expand<T, LMAX, 6>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                case 7: leaf_expand<T, LMAX, 7>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
                default: leaf_expand<T, LMAX, LMAX>(s.r, s.rbeta, s.gam, s.del, xs, xe, xv); break;
            }
            if (active) {  // pivots: checked by Stage 1
#pragma unroll
                for (int i = 0; i < LMAX; ++i)
                    if (i < len) x[row0 + i] = xv[i];
                if (any_nonfinite(xv, len)) report_nonfinite(err, row0);
            }
        }
    }
}

}  // namespace tpb
