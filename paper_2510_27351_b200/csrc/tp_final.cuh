// Finishing solves: the single-CTA k_final, the 8-CTA cluster k_final_cl,
// the fused multi-GPU peer exchange they run at the root (kShard) and the
// NCCL-transport top solve k_gather_solve. Included by tp_kernels.cu after
// the TP_TRACE macros.
#pragma once
#include <cooperative_groups.h>

#include "tp_device.cuh"
#include "tp_exchange.cuh"
#include "tp_generic.cuh"

namespace tpb {

// ===========================================================================
// Finishing solve: ONE CTA solves (or reduces / expands) a whole system of
// n <= kFinalCap rows held in shared memory. This replaces the reference's
// sequential thomas_solve(iface) at the deepest level (partition.hpp:211) and
// its n < 4 fallback (:197) with an exact parallel elimination:
//   G chunks (one per thread, G a power of two) -> leaf sweeps from smem
//   -> 5 warp-level merge levels via shuffles -> warp roots to smem
//   -> warp 0 merges the warp roots (<= 4 more levels) and handles the root
//   -> top-down the same tree -> leaf back-substitution -> coalesced store.
// Modes: kSolve (2x2 root system solved, as Thomas on [E1;E2]),
//        kStage1 (write the root E1/E2: the sharded reduce),
//        kStage3 (root ends read from xi: the sharded expand).
// ===========================================================================
template <class T, int MODE>
__global__ void __launch_bounds__(kFinalThreads2) k_final(SysPtrs<T> sys, int64_t n, int G, IfacePtrs<T> out,
                                                         const T* __restrict__ xi,
                                                         T* __restrict__ x,
                                                         unsigned long long* err, int level,
                                                         const __grid_constant__ ShardLink link) {
    extern __shared__ __align__(16) unsigned char fsm_raw[];
    T* fsm = reinterpret_cast<T*>(fsm_raw);
    T* sa = fsm;
    T* sb = sa + n;
    T* sc = sb + n;
    T* sd = sc + n;
    __shared__ Eq2<T> wroot[kFinalThreads2 / 32];
    __shared__ T wx[2 * (kFinalThreads2 / 32)];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    RowGuard bad;
    TP_TRACE_DECL;
    pdl_begin();
    TP_TRACE(0);

    if (n == 1) {  // thomas_solve on one row (tridiagonal.hpp:57-59)
        if (tid == 0 && MODE == kSolve) {
            bad.see(sys.diag[0], 0);
            x[0] = sys.rhs[0] / sys.diag[0];
            if (!isfinite(x[0])) report_nonfinite(err, 0);
        }
        report_pivot(err, level, bad.bad);
        return;
    }
    // all of a thread's loads are issued before its first shared-memory store
    // (kFinalCap / kFinalThreads2 = 12 rows per thread), so the L2 latency is
    // paid once, not once per row
    {
        constexpr int kPer = (int)((kFinalCap + kFinalThreads2 - 1) / kFinalThreads2);
        T va[kPer], vb[kPer], vc[kPer], vd[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int64_t i = tid + (int64_t)k * kFinalThreads2;
            if (i < n) {
                va[k] = __ldg(sys.sub + i);
                vb[k] = __ldg(sys.diag + i);
                vc[k] = __ldg(sys.sup + i);
                vd[k] = __ldg(sys.rhs + i);
            }
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int64_t i = tid + (int64_t)k * kFinalThreads2;
            if (i < n) {
                sa[i] = va[k];
                sb[i] = vb[k];
                sc[i] = vc[k];
                sd[i] = vd[k];
            }
        }
    }
    __syncthreads();
    TP_TRACE(1);

    const int Llo = (int)(n / G), ext = (int)(n % G);
    const bool active = tid < G;
    const int len = Llo + (tid < ext ? 1 : 0);
    const int off = tid * Llo + (tid < ext ? tid : ext);
    auto chunk_start = [&](int c) { return c * Llo + (c < ext ? c : ext); };
    constexpr bool KEEP = (MODE != kStage1);

    Eq2<T> cur = Eq2<T>{0, 1, 0, 0, 0, 1, 0, 0};
    if (active) cur = leaf_smem<T, KEEP>(sa + off, sb + off, sc + off, sd + off, len, off, bad);
    TP_TRACE(2);

    // ---- warp-level tree (chunk index == tid) ----
    MergeSave<T> sw[5];
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
        const int h = 1 << lv;
        const Eq2<T> oth = shfl_down_eq(cur, h);
        if (h < G && (lane & (2 * h - 1)) == 0 && tid + h < G)
            cur = merge(cur, oth, (int64_t)chunk_start(tid + h) - 1, bad, sw[lv]);
    }
    const int nwr = G >= 32 ? G / 32 : 1;  // warp roots
    if (lane == 0 && warp < nwr) wroot[warp] = cur;
    TP_TRACE(3);
    __syncthreads();
    TP_TRACE(4);

    // ---- warp 0: merge the warp roots, handle the root, push ends back down ----
    if (warp == 0) {
        Eq2<T> wc = lane < nwr ? wroot[lane] : Eq2<T>{0, 1, 0, 0, 0, 1, 0, 0};
        MergeSave<T> sx[5];
#pragma unroll
        for (int lv = 0; lv < 5; ++lv) {
            const int h = 1 << lv;
            const Eq2<T> oth = shfl_down_eq(wc, h);
            if (h < nwr && (lane & (2 * h - 1)) == 0 && lane + h < nwr)
                wc = merge(wc, oth, (int64_t)chunk_start(32 * (lane + h)) - 1, bad, sx[lv]);
        }
        TP_TRACE(5);
        T xs = 0, xe = 0;
        if (lane == 0) {
            if constexpr (MODE == kStage1) {
                out.sub[0] = wc.a1;  out.sub[1] = wc.a2;
                out.diag[0] = wc.b1; out.diag[1] = wc.b2;
                out.sup[0] = wc.g1;  out.sup[1] = wc.g2;
                out.rhs[0] = wc.d1;  out.rhs[1] = wc.d2;
            } else if constexpr (MODE == kStage3) {
                xs = xi[0];
                xe = xi[1];
            } else if constexpr (MODE == kShard) {
                // the collective, fused: this shard's root pair goes straight
                // into every peer's HBM, the top system is solved here
                __shared__ double top_cm[2 * kMaxPeers], top_x[2 * kMaxPeers];
                RowGuard top_bad;
                int missing = -1;
                if (!shard_exchange(link, wc, top_cm, top_x, xs, xe, top_bad, missing)) {
                    if (err != nullptr)
                        atomicMin(err, ((unsigned long long)kExchangeLevel << 48) | (unsigned long long)missing);
                }
                report_pivot(err, level + 1, top_bad.bad);
            } else {
                root_solve(wc, n - 1, bad, xs, xe);
            }
        }
        if (MODE != kStage1) {
#pragma unroll
            for (int lv = 4; lv >= 0; --lv) {
                const int h = 1 << lv;
                if (h >= nwr) continue;
                T xt = 0;
                if ((lane & (2 * h - 1)) == 0) xt = merge_xt(sx[lv], xs, xe);
                const T rxt = __shfl_up_sync(0xffffffffu, xt, h);
                const T rxe = __shfl_up_sync(0xffffffffu, xe, h);
                if ((lane & (2 * h - 1)) == h) {
                    xs = first_from_e1(wc, rxt, rxe);
                    xe = rxe;
                } else if ((lane & (2 * h - 1)) == 0) {
                    xe = xt;
                }
            }
            if (lane < nwr) {
                wx[2 * lane] = xs;
                wx[2 * lane + 1] = xe;
            }
        }
        TP_TRACE(6);
    }
    if (MODE == kStage1) {
        report_pivot(err, level, bad.bad);
        return;
    }
    __syncthreads();
    TP_TRACE(7);

    // ---- every warp: its segment ends, then the warp-level tree top-down ----
    T xs = 0, xe = 0;
    if (lane == 0 && warp < nwr) {
        xs = wx[2 * warp];
        xe = wx[2 * warp + 1];
    }
#pragma unroll
    for (int lv = 4; lv >= 0; --lv) {
        const int h = 1 << lv;
        if (h >= G) continue;
        T xt = 0;
        if ((lane & (2 * h - 1)) == 0) xt = merge_xt(sw[lv], xs, xe);
        const T rxt = __shfl_up_sync(0xffffffffu, xt, h);
        const T rxe = __shfl_up_sync(0xffffffffu, xe, h);
        if ((lane & (2 * h - 1)) == h) {
            xs = first_from_e1(cur, rxt, rxe);
            xe = rxe;
        } else if ((lane & (2 * h - 1)) == 0) {
            xe = xt;
        }
    }
    TP_TRACE(8);
    // ---- leaf back-substitution into the a-slots, then a coalesced store ----
    if (active) {
        T* a = sa + off;
        const T* rb = sb + off;
        const T* g = sc + off;
        const T* dd = sd + off;
        T prev = xs;
        for (int i = 1; i < len - 1; ++i) {
            const T xv = (dd[i] - a[i] * prev - g[i] * xe) * rb[i];
            a[i] = xv;
            prev = xv;
        }
        a[0] = xs;
        a[len - 1] = xe;
    }
    TP_TRACE(9);
    __syncthreads();
    TP_TRACE(10);
    bool nf = false;
    for (int64_t i = tid; i < n; i += kFinalThreads2) {
        x[i] = sa[i];
        nf |= !isfinite(sa[i]);
    }
    if (nf) report_nonfinite(err, 0);
    TP_TRACE(11);
    TP_TRACE_FLUSH;
    report_pivot(err, level, bad.bad);
}

// ===========================================================================
// Finishing solve on a thread-block CLUSTER (kFinCS CTAs on kFinCS SMs, DSMEM).
// The single-CTA k_final is FP64-latency and shared-memory-bandwidth bound
// (~10 rows per thread swept from smem, a 9-level tree, ~21K cycles at C3).
// Here Gtot = min(kFinCS * kFinNT, pow2floor(n/2)) chunks of <= 4 rows each
// live in registers; the tree is 5 shuffle levels per warp, <= 3 levels over
// the warp roots of each CTA (warp 0), and <= 3 levels over the CTA roots in
// CTA 0, which reads them from the peers' shared memory (cluster.map_shared_rank),
// handles the root (kSolve / kStage1 / kStage3 / kShard exactly as k_final),
// and writes each CTA's segment ends back into that CTA's shared memory. Two
// cluster barriers in total. Same merges / sweeps / expansion as k_final, so
// results agree with it to rounding.
// ===========================================================================
constexpr int kFinCS = 8;     // CTAs per cluster (portable maximum)
constexpr int kFinNT = 256;   // threads per CTA
constexpr int kFinRows = kFinNT * 4;  // rows staged per CTA (chunks <= 4 rows)

// The cluster tree over rows already staged in this CTA's shared memory
// (sa..sd, `rows` rows starting at system row r0, `per` chunks of 2..4 rows,
// per a power of two <= kFinNT). cta_row0(c) is CTA c's first system row;
// the chunking is local to the CTA (its first rows % per chunks get the extra
// row), which equals k_final_cl's global chunking when every CTA owns the same
// number of chunks. The solution rows go to xdst[row - xbase].
template <class T, int MODE, int CS = kFinCS, class CtaRow0>
__device__ __forceinline__ void cl_tree(cooperative_groups::cluster_group& cl, const T* sa, const T* sb,
                                        const T* sc, const T* sd, int64_t r0, int rows, int per,
                                        CtaRow0 cta_row0, int64_t n, const IfacePtrs<T>& out,
                                        const T* __restrict__ xi, T* __restrict__ xdst, int64_t xbase,
                                        RowGuard& bad, unsigned long long* err, int level,
                                        const ShardLink& link) {
    __shared__ Eq2<T> wroot[kFinNT / 32];
    __shared__ Eq2<T> croot;   // this CTA's root pair, read by CTA 0
    __shared__ T cx[2];        // this CTA's (x_s, x_e), written by CTA 0
    __shared__ T wx[2 * (kFinNT / 32)];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cta = (int)cl.block_rank();
    TP_TRACE_DECL;
    TP_TRACE(0);
    TP_TRACE(1);

    const int Llo = rows / per, ext = rows % per;
    auto cstart = [&](int c) { return r0 + (int64_t)c * Llo + (c < ext ? c : ext); };

    // ---- leaf: this thread's chunk (2..4 rows) in registers ----
    const bool active = tid < per;
    const int len = active ? Llo + (tid < ext ? 1 : 0) : 2;
    const int64_t grow = active ? cstart(tid) : 0;
    Chunk<T, 4> r;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const bool live = active && i < len;
        const int li = (int)(grow - r0) + i;
        r.a[i] = live ? sa[li] : T(0);
        r.b[i] = live ? sb[li] : T(1);
        r.c[i] = live ? sc[li] : T(0);
        r.d[i] = live ? sd[li] : T(0);
    }
    T rb[4], gm[4], dl[4];
    Eq2<T> cur;
    if (len == 2) cur = leaf_reduce_keep<T, 4, 2>(r, grow, bad, rb, gm, dl);
    else if (len == 3) cur = leaf_reduce_keep<T, 4, 3>(r, grow, bad, rb, gm, dl);
    else cur = leaf_reduce_keep<T, 4, 4>(r, grow, bad, rb, gm, dl);
    if (!active) cur = Eq2<T>{0, 1, 0, 0, 0, 1, 0, 0};
    TP_TRACE(2);

    // ---- warp levels (chunk index inside the CTA == tid) ----
    SchurSave<T> sw[5];
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
        const int h = 1 << lv;
        const Eq2<T> oth = shfl_down_eq(cur, h);
        if (h < per && (lane & (2 * h - 1)) == 0 && tid + h < per)
            cur = merge_schur_row(cur, oth, cstart(tid + h) - 1, bad, sw[lv]);
    }
    const int nwr = per >= 32 ? per / 32 : 1;
    if (lane == 0 && warp < nwr) wroot[warp] = cur;
    __syncthreads();
    TP_TRACE(3);

    // ---- warp 0: the CTA's warp roots (<= 3 levels) ----
    SchurSave<T> sx[3];
    Eq2<T> wc = Eq2<T>{0, 1, 0, 0, 0, 1, 0, 0};
    if (warp == 0) {
        wc = lane < nwr ? wroot[lane] : wc;
#pragma unroll
        for (int lv = 0; lv < 3; ++lv) {
            const int h = 1 << lv;
            const Eq2<T> oth = shfl_down_eq(wc, h);
            if (h < nwr && (lane & (2 * h - 1)) == 0 && lane + h < nwr)
                wc = merge_schur_row(wc, oth, cstart(32 * (lane + h)) - 1, bad, sx[lv]);
        }
        if (lane == 0) croot = wc;
    }
    TP_TRACE(4);
    cl.sync();
    TP_TRACE(5);

    // ---- CTA 0, warp 0: the CTA roots (3 levels), the root, and back down ----
    if (cta == 0 && warp == 0) {
        Eq2<T> cc = Eq2<T>{0, 1, 0, 0, 0, 1, 0, 0};
        if (lane < CS) cc = *cl.map_shared_rank(&croot, lane);
        constexpr int kCLv = CS == 16 ? 4 : 3;  // levels over the CTA roots
        SchurSave<T> sc3[kCLv];
#pragma unroll
        for (int lv = 0; lv < kCLv; ++lv) {
            const int h = 1 << lv;
            const Eq2<T> oth = shfl_down_eq(cc, h);
            if ((lane & (2 * h - 1)) == 0 && lane + h < CS)
                cc = merge_schur_row(cc, oth, cta_row0(lane + h) - 1, bad, sc3[lv]);
        }
        T xs = 0, xe = 0;
        if (lane == 0) {
            if constexpr (MODE == kStage1) {
                out.sub[0] = cc.a1;  out.sub[1] = cc.a2;
                out.diag[0] = cc.b1; out.diag[1] = cc.b2;
                out.sup[0] = cc.g1;  out.sup[1] = cc.g2;
                out.rhs[0] = cc.d1;  out.rhs[1] = cc.d2;
            } else if constexpr (MODE == kStage3) {
                xs = xi[0];
                xe = xi[1];
            } else if constexpr (MODE == kShard) {
                __shared__ double top_cm[2 * kMaxPeers], top_x[2 * kMaxPeers];
                RowGuard top_bad;
                int missing = -1;
                if (!shard_exchange(link, cc, top_cm, top_x, xs, xe, top_bad, missing)) {
                    if (err != nullptr)
                        atomicMin(err, ((unsigned long long)kExchangeLevel << 48) | (unsigned long long)missing);
                }
                report_pivot(err, level + 1, top_bad.bad);
            } else {
                root_solve(cc, n - 1, bad, xs, xe);
            }
        }
        if constexpr (MODE != kStage1) {
#pragma unroll
            for (int lv = kCLv - 1; lv >= 0; --lv) {
                const int h = 1 << lv;
                T xt = 0, xt1 = 0;
                if ((lane & (2 * h - 1)) == 0) schur_down(sc3[lv], xs, xe, xt, xt1);
                const T r1 = __shfl_up_sync(0xffffffffu, xt1, h);
                const T rxe = __shfl_up_sync(0xffffffffu, xe, h);
                if ((lane & (2 * h - 1)) == h) {
                    xs = r1;
                    xe = rxe;
                } else if ((lane & (2 * h - 1)) == 0) {
                    xe = xt;
                }
            }
            if (lane < CS) {
                T* dst = cl.map_shared_rank(&cx[0], lane);
                dst[0] = xs;
                dst[1] = xe;
            }
        }
    }
    TP_TRACE(6);
    if constexpr (MODE == kStage1) {
        // CTA 0 read every croot before reaching this barrier; no CTA may exit
        // while its shared memory can still be read
        cl.sync();
        return;
    }
    cl.sync();
    TP_TRACE(7);

    // ---- warp 0 of every CTA: down its warp-root levels ----
    if (warp == 0) {
        T xs = lane == 0 ? cx[0] : T(0), xe = lane == 0 ? cx[1] : T(0);
#pragma unroll
        for (int lv = 2; lv >= 0; --lv) {
            const int h = 1 << lv;
            if (h >= nwr) continue;
            T xt = 0, xt1 = 0;
            if ((lane & (2 * h - 1)) == 0) schur_down(sx[lv], xs, xe, xt, xt1);
            const T r1 = __shfl_up_sync(0xffffffffu, xt1, h);
            const T rxe = __shfl_up_sync(0xffffffffu, xe, h);
            if ((lane & (2 * h - 1)) == h) {
                xs = r1;
                xe = rxe;
            } else if ((lane & (2 * h - 1)) == 0) {
                xe = xt;
            }
        }
        if (lane < nwr) {
            wx[2 * lane] = xs;
            wx[2 * lane + 1] = xe;
        }
    }
    __syncthreads();
    TP_TRACE(8);

    // ---- every warp: its warp levels, then the chunk ----
    T xs = 0, xe = 0;
    if (lane == 0 && warp < nwr) {
        xs = wx[2 * warp];
        xe = wx[2 * warp + 1];
    }
#pragma unroll
    for (int lv = 4; lv >= 0; --lv) {
        const int h = 1 << lv;
        if (h >= per) continue;
        T xt = 0, xt1 = 0;
        if ((lane & (2 * h - 1)) == 0) schur_down(sw[lv], xs, xe, xt, xt1);
        const T r1 = __shfl_up_sync(0xffffffffu, xt1, h);
        const T rxe = __shfl_up_sync(0xffffffffu, xe, h);
        if ((lane & (2 * h - 1)) == h) {
            xs = r1;
            xe = rxe;
        } else if ((lane & (2 * h - 1)) == 0) {
            xe = xt;
        }
    }
    if (active) {
        T xv[4];
        if (len == 2) leaf_expand<T, 4, 2>(r, rb, gm, dl, xs, xe, xv);
        else if (len == 3) leaf_expand<T, 4, 3>(r, rb, gm, dl, xs, xe, xv);
        else leaf_expand<T, 4, 4>(r, rb, gm, dl, xs, xe, xv);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (i < len) xdst[grow - xbase + i] = xv[i];
        if (any_nonfinite(xv, len)) report_nonfinite(err, grow);
    }
    TP_TRACE(9);
    TP_TRACE(10);
    TP_TRACE(11);
    if (blockIdx.x == 0) TP_TRACE_FLUSH;
}

template <class T, int MODE>
__global__ void __cluster_dims__(kFinCS, 1, 1) __launch_bounds__(kFinNT, 1)
    k_final_cl(SysPtrs<T> sys, int64_t n, int gtot, IfacePtrs<T> out, const T* __restrict__ xi,
               T* __restrict__ x, unsigned long long* err, int level, const __grid_constant__ ShardLink link) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ T sa[kFinRows], sb[kFinRows], sc[kFinRows], sd[kFinRows];
    const int tid = threadIdx.x;
    const int cta = (int)cl.block_rank();
    RowGuard bad;
    pdl_begin();

    const int per = gtot / kFinCS;  // chunks owned by each CTA (power of two)
    const int64_t Llo = n / gtot, ext = n % gtot;
    auto gstart = [&](int64_t g) { return g * Llo + (g < ext ? g : ext); };
    const int64_t r0 = gstart((int64_t)cta * per);
    const int rows = (int)(gstart((int64_t)(cta + 1) * per) - r0);
    {  // rows <= 4 * kFinNT: every load of the CTA in flight at once
        T va[4], vb[4], vc[4], vd[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = tid + u * kFinNT;
            if (i < rows) {
                va[u] = __ldg(sys.sub + r0 + i);
                vb[u] = __ldg(sys.diag + r0 + i);
                vc[u] = __ldg(sys.sup + r0 + i);
                vd[u] = __ldg(sys.rhs + r0 + i);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = tid + u * kFinNT;
            if (i < rows) { sa[i] = va[u]; sb[i] = vb[u]; sc[i] = vc[u]; sd[i] = vd[u]; }
        }
    }
    __syncthreads();
    cl_tree<T, MODE>(cl, sa, sb, sc, sd, r0, rows, per, [&](int c) { return gstart((int64_t)per * c); }, n, out,
                     xi, x, 0, bad, err, level, link);
    report_pivot(err, level, bad.bad);
}

// ===========================================================================
// The last partition level and the finishing solve in ONE cluster kernel.
// When the deepest level's system fits the cluster's shared memory (C3: level
// 3, 39K rows; C1: the whole 10K-row system), its Stage 1, the finishing solve
// of its 2K-row interface and its Stage 3 run here instead of as three kernels
// (plus the Stage-1/Stage-3 tail branches). CTA c owns level blocks
// [K c / 8, K (c + 1) / 8): their rows are staged once into shared memory, one
// thread sweeps one block at a time (leaf_smem, partition.hpp:90-124, the same
// arithmetic as k_generic with one lane per block), the block's E1/E2 rows are
// this CTA's rows of the interface (assemble_interface order,
// partition.hpp:139-149; also stored to HBM for the observer), cl_tree solves
// the interface across the cluster,
// and each thread back-substitutes its block from the kept sweep values
// (partition.hpp:154-173) before one coalesced store. The interface never
// leaves the SMs. Blocks are padded to an odd stride S >= m + 1 so the
// one-thread-per-block sweeps are free of bank conflicts.
// ===========================================================================
constexpr int kLfMaxBlocks = kFinRows / 2;  // level blocks per CTA (interface chunks <= 4 rows)

// Walks local rows e = tid, tid + kFinNT, ... of a CTA's level rows without
// dividing: (jj, i) = (e / m, e % m); the tail block's extra row (i == m in
// the last block) maps to slot (nb - 1, m).
struct LfSlots {
    int jj, i, dq, dr, m, nb, S;
    __device__ LfSlots(int tid, int m_, int nb_, int S_) : m(m_), nb(nb_), S(S_) {
        jj = tid / m; i = tid - jj * m;
        dq = kFinNT / m; dr = kFinNT - dq * m;
    }
    __device__ __forceinline__ int slot() const { return jj < nb ? jj * S + i : (nb - 1) * S + i + m; }
    __device__ __forceinline__ void next() {
        jj += dq; i += dr;
        if (i >= m) { i -= m; ++jj; }
    }
};

// Stage-1 sweeps of one full block of MF rows in registers (both sweeps are
// independent dependency chains the compiler interleaves), the kept values
// written back to the block's b / c / d slots in leaf_smem's layout.
template <class T, int MF>
__device__ __forceinline__ Eq2<T> lf_sweep_regs(T* a, T* b, T* c, T* d, int64_t row0, RowGuard& bad) {
    Chunk<T, MF> r;
#pragma unroll
    for (int i = 0; i < MF; ++i) { r.a[i] = a[i]; r.b[i] = b[i]; r.c[i] = c[i]; r.d[i] = d[i]; }
    T rb[MF], gm[MF], dl[MF];
    const Eq2<T> q = leaf_reduce_keep<T, MF, MF>(r, row0, bad, rb, gm, dl);
#pragma unroll
    for (int i = 1; i < MF - 1; ++i) { b[i] = rb[i]; c[i] = gm[i]; d[i] = dl[i]; }
    return q;
}

template <class T, int MF>
__device__ __forceinline__ void lf_expand_regs(T* a, const T* rbp, const T* gp, const T* dp, T xs, T xe) {
    T av[MF], rb[MF], g[MF], dd[MF];
#pragma unroll
    for (int i = 1; i < MF - 1; ++i) { av[i] = a[i]; rb[i] = rbp[i]; g[i] = gp[i]; dd[i] = dp[i]; }
    T prev = xs;
#pragma unroll
    for (int i = 1; i < MF - 1; ++i) {
        const T xv = (dd[i] - av[i] * prev - g[i] * xe) * rb[i];
        a[i] = xv;
        prev = xv;
    }
    a[0] = xs;
    a[MF - 1] = xe;
}

// MF = m when m is 4, 8 or 16 (register sweeps for the full blocks), else 0.
// CS = CTAs per cluster (8, or 16 where the GPU can co-schedule a
// non-portable 16-CTA cluster); the cluster shape is set at launch.
// MODE kSolve: the interface root is solved here (single-GPU solve);
// kShard: this level is a shard's deepest, its root pair is the shard's
// boundary pair and goes through the peer exchange (shard_exchange) before the
// tree unwinds — the multi-GPU graph then has the single-GPU graph's shape.
template <class T, int MF, int CS, int MODE>
__global__ void __launch_bounds__(kFinNT, 1)
    k_level_final_cl(SysPtrs<T> sys, int64_t n, int m, int64_t K, int S, IfacePtrs<T> iface, T* __restrict__ x,
                     unsigned long long* err, int level, const __grid_constant__ ShardLink link, int flags) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char lf_raw[];
    __shared__ T fa[kFinRows], fb[kFinRows], fc[kFinRows], fd[kFinRows], fx[kFinRows];
    const int tid = threadIdx.x;
    const int cta = (int)cl.block_rank();
    const int64_t B0 = K * cta / CS, B1 = K * (cta + 1) / CS;
    const int nb = (int)(B1 - B0);
    const int nbmax = (int)((K + CS - 1) / CS);
    T* la = reinterpret_cast<T*>(lf_raw);
    T* lb = la + (size_t)nbmax * S;
    T* lc = lb + (size_t)nbmax * S;
    T* ld = lc + (size_t)nbmax * S;
    RowGuard bad_lv, bad_fin;
    pdl_begin();
    TP_LF_TRACE(0);
    if ((flags & kResetErr) && cta == 0 && tid == 0 && err != nullptr) {  // the graph's only kernel
        *reinterpret_cast<volatile unsigned long long*>(err) = kNoError;
        __threadfence();
    }

    const int64_t r0 = B0 * m;
    const int rows = (int)((B1 == K ? n : B1 * m) - r0);
    // ---- stage: every element as its own cp.async into its padded slot (the
    // level sits in L2; async copies keep far more of it in flight than
    // register loads: 8.1K -> 5.0K cycles at C3) ----
    {
        LfSlots w(tid, m, nb, S);
        for (int e = tid; e < rows; e += kFinNT, w.next()) {
            const int k = w.slot();
            const T* src[4] = {sys.sub + r0 + e, sys.diag + r0 + e, sys.sup + r0 + e, sys.rhs + r0 + e};
            T* dst[4] = {la + k, lb + k, lc + k, ld + k};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned sa_ = (unsigned)__cvta_generic_to_shared(dst[q]);
                if constexpr (sizeof(T) == 8)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa_), "l"(src[q]) : "memory");
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa_), "l"(src[q]) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    TP_LF_TRACE(1);

    // ---- Stage 1 of the level: one thread per block ----
    for (int jj = tid; jj < nb; jj += kFinNT) {
        const int64_t j = B0 + jj;
        const int len = j == K - 1 ? (int)(n - (K - 1) * m) : m;
        const int o = jj * S;
        Eq2<T> q;
        if (MF > 0 && len == MF) q = lf_sweep_regs<T, (MF > 0 ? MF : 4)>(la + o, lb + o, lc + o, ld + o, j * m, bad_lv);
        else q = leaf_smem<T, true>(la + o, lb + o, lc + o, ld + o, len, j * m, bad_lv);
        fa[2 * jj] = q.a1; fa[2 * jj + 1] = q.a2;
        fb[2 * jj] = q.b1; fb[2 * jj + 1] = q.b2;
        fc[2 * jj] = q.g1; fc[2 * jj + 1] = q.g2;
        fd[2 * jj] = q.d1; fd[2 * jj + 1] = q.d2;
    }
    __syncthreads();
    // the interface also goes to HBM (2 rows per block, coalesced, off the
    // critical path): the observer overload reports every level's interface
    for (int i = tid; i < 2 * nb; i += kFinNT) {
        iface.sub[2 * B0 + i] = fa[i];
        iface.diag[2 * B0 + i] = fb[i];
        iface.sup[2 * B0 + i] = fc[i];
        iface.rhs[2 * B0 + i] = fd[i];
    }
    TP_LF_TRACE(2);

    // ---- the interface (2K rows) across the cluster ----
    int per = 1;
    while (per * 2 <= kFinNT && per * 2 <= nb) per *= 2;
    cl_tree<T, MODE, CS>(cl, fa, fb, fc, fd, 2 * B0, 2 * nb, per,
                         [&](int c) { return 2 * (K * c / CS); }, 2 * K, IfacePtrs<T>{}, nullptr, fx,
                         2 * B0, bad_fin, err, level + 1, link);
    __syncthreads();
    TP_LF_TRACE(3);

    // ---- Stage 3 of the level: back-substitute each block, then one store ----
    for (int jj = tid; jj < nb; jj += kFinNT) {
        const int64_t j = B0 + jj;
        const int len = j == K - 1 ? (int)(n - (K - 1) * m) : m;
        const int o = jj * S;
        T* a = la + o;
        const T xs = fx[2 * jj], xe = fx[2 * jj + 1];
        if (MF > 0 && len == MF) {
            lf_expand_regs<T, (MF > 0 ? MF : 4)>(a, lb + o, lc + o, ld + o, xs, xe);
            continue;
        }
        const T* rb = lb + o;
        const T* g = lc + o;
        const T* dd = ld + o;
        T prev = xs;
        for (int i = 1; i < len - 1; ++i) {
            const T xv = (dd[i] - a[i] * prev - g[i] * xe) * rb[i];
            a[i] = xv;
            prev = xv;
        }
        a[0] = xs;
        a[len - 1] = xe;
    }
    __syncthreads();
    TP_LF_TRACE(4);
    {
        LfSlots w(tid, m, nb, S);
        bool nf = false;
        for (int e = tid; e < rows; e += kFinNT, w.next()) {
            const T v = la[w.slot()];
            x[r0 + e] = v;
            nf |= !isfinite(v);
        }
        if (nf) report_nonfinite(err, r0);
    }
    TP_LF_TRACE(5);
    report_pivot(err, level, bad_lv.bad);
    report_pivot(err, level + 1, bad_fin.bad);
}

// ===========================================================================
// Sharded top level: every rank holds the gathered [eq8 x P] (layout per rank:
// sub[2], diag[2], sup[2], rhs[2]); assemble the 2P-row interface
// (assemble_interface, partition.hpp:139-149) and solve it with Thomas
// (tridiagonal.hpp:52-72) in one thread; keep this rank's (x_s, x_e).
// ===========================================================================
template <class T>
__global__ void k_gather_solve(const T* __restrict__ eqs, int nranks, int rank,
                               T* __restrict__ x2, T* __restrict__ scratch,
                               unsigned long long* err, int level) {
    pdl_begin();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int n = 2 * nranks;
    T* cm = scratch;
    T* xx = scratch + n;
    RowGuard bad;
    for (int i = 0; i < n; ++i) {
        const T* e = eqs + 8 * (i >> 1);
        const int k = i & 1;
        const T sub = e[0 + k], dg = e[2 + k], sp = e[4 + k], rh = e[6 + k];
        if (i == 0) {
            bad.see(dg, 0);
            cm[0] = sp / dg;
            xx[0] = rh / dg;
        } else {
            const T piv = dg - sub * cm[i - 1];
            bad.see(piv, i);
            cm[i] = sp / piv;
            xx[i] = (rh - sub * xx[i - 1]) / piv;
        }
    }
    for (int i = n - 2; i >= 0; --i) xx[i] -= cm[i] * xx[i + 1];
    x2[0] = xx[2 * rank];
    x2[1] = xx[2 * rank + 1];
    report_pivot(err, level, bad.bad);
}

}  // namespace tpb
