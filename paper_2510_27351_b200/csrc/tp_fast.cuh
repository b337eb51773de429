// Fast-path kernel template (included by tp_kernels.cu and the tuning harness).
#pragma once
#include "tp_device.cuh"

namespace tpb {

// ===========================================================================
// Fast path: full blocks of m = L*G rows, one chunk of L rows per thread held
// in registers, G lanes per block (G | 32), lane-tree merges via shuffles.
// ===========================================================================
template <int L, int G, int MODE, bool VEC, int THREADS = kFastThreads, int MINB = 1>
__global__ void __launch_bounds__(THREADS, MINB) k_fast(SysPtrs sys, int64_t nblocks, IfacePtrs out,
                                                       const double* __restrict__ xi,
                                                       double* __restrict__ x,
                                                       unsigned long long* err, int level) {
    static_assert(32 % G == 0, "G must divide the warp");
    constexpr int LOGG = (G >= 32) ? 5 : (G >= 16) ? 4 : (G >= 8) ? 3 : (G >= 4) ? 2 : (G >= 2) ? 1 : 0;
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
        Chunk<L> r;
        if (active) {
            load_rows<L, VEC>(sys.sub, row0, r.a);
            load_rows<L, VEC>(sys.diag, row0, r.b);
            load_rows<L, VEC>(sys.sup, row0, r.c);
            load_rows<L, VEC>(sys.rhs, row0, r.d);
        } else {
#pragma unroll
            for (int i = 0; i < L; ++i) { r.a[i] = 0; r.b[i] = 1; r.c[i] = 0; r.d[i] = 0; }
        }
        const int64_t blk = t / G;

        if constexpr (MODE == kStage1) {
            MinGuard lbad;
            Eq2 cur = leaf_reduce<L>(r, L, row0, lbad);
#pragma unroll
            for (int lv = 0; lv < LOGG; ++lv) {
                const int h = 1 << lv;
                const Eq2 oth = shfl_down_eq(cur, h);
                if ((c & (2 * h - 1)) == 0) {
                    MergeSave sv;
                    cur = merge(cur, oth, row0 + (int64_t)h * L - 1, lbad, sv);
                }
            }
            if (active) {
                if (lbad.tripped()) bad = row0 < bad ? row0 : bad;
                if (c == 0) {
                    const int64_t o = 2 * blk;
                    *reinterpret_cast<double2*>(out.sub + o) = make_double2(cur.a1, cur.a2);
                    *reinterpret_cast<double2*>(out.diag + o) = make_double2(cur.b1, cur.b2);
                    *reinterpret_cast<double2*>(out.sup + o) = make_double2(cur.g1, cur.g2);
                    *reinterpret_cast<double2*>(out.rhs + o) = make_double2(cur.d1, cur.d2);
                }
            }
        } else {
            MinGuard lbad;
            double rbeta[L], gam[L], del[L];
            Eq2 cur = leaf_reduce_keep<L>(r, L, row0, lbad, rbeta, gam, del);
            MergeSave sv[LOGG > 0 ? LOGG : 1];
#pragma unroll
            for (int lv = 0; lv < LOGG; ++lv) {
                const int h = 1 << lv;
                const Eq2 oth = shfl_down_eq(cur, h);
                if ((c & (2 * h - 1)) == 0) cur = merge(cur, oth, row0 + (int64_t)h * L - 1, lbad, sv[lv]);
            }
            // block ends from the next level's solution
            double xs = 0, xe = 0;
            if (c == 0 && active) {
                const double2 v = *reinterpret_cast<const double2*>(xi + 2 * blk);
                xs = v.x;
                xe = v.y;
            }
#pragma unroll
            for (int lv = LOGG - 1; lv >= 0; --lv) {
                const int h = 1 << lv;
                double xt = 0;
                if ((c & (2 * h - 1)) == 0) xt = merge_xt(sv[lv], xs, xe);
                const double rxt = __shfl_up_sync(0xffffffffu, xt, h);
                const double rxe = __shfl_up_sync(0xffffffffu, xe, h);
                if ((c & (2 * h - 1)) == h) {
                    xs = first_from_e1(cur, rxt, rxe);
                    xe = rxe;
                } else if ((c & (2 * h - 1)) == 0) {
                    xe = xt;
                }
            }
            double xv[L];
            leaf_expand<L>(r, L, rbeta, gam, del, xs, xe, xv);
            if (active) {
                if (lbad.tripped()) bad = row0 < bad ? row0 : bad;
                store_rows<L, VEC>(x, row0, xv);
            }
        }
    }
    report_pivot(err, level, bad);
}

}  // namespace tpb
