// Finishing solves: the single-CTA k_final, the 8-CTA cluster k_final_cl,
// the fused multi-GPU peer exchange they run at the root (kShard) and the
// NCCL-transport top solve k_gather_solve. Included by tp_kernels.cu after
// the TP_TRACE macros.
#pragma once
#include <cooperative_groups.h>

#include "tp_device.cuh"
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
// ---------------------------------------------------------------------------
// Peer exchange of the fused multi-GPU solve (k_final<kShard>, one thread).
// Publish this shard's boundary pair into every rank's mailbox, release the
// epoch flag (system scope), wait for all P flags in our own mailbox (acquire,
// bounded), then assemble the 2P-row top system (assemble_interface order,
// partition.hpp:139-149) and solve it with Thomas (tridiagonal.hpp:52-72).
// Returns this shard's (x_s, x_e); false on a peer timeout.
// ---------------------------------------------------------------------------
constexpr long kExchangeSpins = 1L << 24;  // x >= 64 ns back-off: ~1-2 s before giving up

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

template <class T>
__device__ bool shard_exchange(const ShardLink& lk, const Eq2<T>& q, double* cm, double* xx, T& xs, T& xe,
                               RowGuard& top_bad, int& missing) {
    const unsigned long long e = *lk.epoch + 1;
    const int P = lk.nranks;
    const size_t slot = (size_t)(e & 1);
    const double v[8] = {(double)q.a1, (double)q.a2, (double)q.b1, (double)q.b2,
                         (double)q.g1, (double)q.g2, (double)q.d1, (double)q.d2};
    for (int p = 0; p < P; ++p) {
        double* dst = lk.peers[p] + (slot * P + lk.rank) * kMailboxEntryDoubles;
#pragma unroll
        for (int k = 0; k < 8; ++k) dst[k] = v[k];
    }
    __threadfence_system();
    for (int p = 0; p < P; ++p)
        st_release_sys(reinterpret_cast<unsigned long long*>(
                           lk.peers[p] + (slot * P + lk.rank) * kMailboxEntryDoubles + 8), e);
    for (int p = 0; p < P; ++p) {
        const unsigned long long* f = reinterpret_cast<const unsigned long long*>(
            lk.own + (slot * P + p) * kMailboxEntryDoubles + 8);
        long spins = 0;
        while (ld_acquire_sys(f) != e) {
            if (++spins > kExchangeSpins) {
                missing = p;
                *lk.epoch = e;  // stay paired with the peers' next exchange
                return false;
            }
            __nanosleep(64);
        }
    }
    const int n = 2 * P;
    for (int i = 0; i < n; ++i) {
        const double* e8 = lk.own + (slot * P + (i >> 1)) * kMailboxEntryDoubles;
        const int k = i & 1;
        const double sub = ld_relaxed_sys(e8 + 0 + k), dg = ld_relaxed_sys(e8 + 2 + k);
        const double sp = ld_relaxed_sys(e8 + 4 + k), rh = ld_relaxed_sys(e8 + 6 + k);
        if (i == 0) {
            top_bad.see(dg, 0);
            cm[0] = sp / dg;
            xx[0] = rh / dg;
        } else {
            const double piv = dg - sub * cm[i - 1];
            top_bad.see(piv, i);
            cm[i] = sp / piv;
            xx[i] = (rh - sub * xx[i - 1]) / piv;
        }
    }
    for (int i = n - 2; i >= 0; --i) xx[i] -= cm[i] * xx[i + 1];
    xs = (T)xx[2 * lk.rank];
    xe = (T)xx[2 * lk.rank + 1];
    *lk.epoch = e;
    return true;
}

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
    for (int64_t i = tid; i < n; i += kFinalThreads2) x[i] = sa[i];
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

template <class T, int MODE>
__global__ void __cluster_dims__(kFinCS, 1, 1) __launch_bounds__(kFinNT, 1)
    k_final_cl(SysPtrs<T> sys, int64_t n, int gtot, IfacePtrs<T> out, const T* __restrict__ xi,
               T* __restrict__ x, unsigned long long* err, int level, const __grid_constant__ ShardLink link) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ T sa[kFinRows], sb[kFinRows], sc[kFinRows], sd[kFinRows];
    __shared__ Eq2<T> wroot[kFinNT / 32];
    __shared__ Eq2<T> croot;   // this CTA's root pair, read by CTA 0
    __shared__ T cx[2];        // this CTA's (x_s, x_e), written by CTA 0
    __shared__ T wx[2 * (kFinNT / 32)];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cta = (int)cl.block_rank();
    RowGuard bad;
    TP_TRACE_DECL;
    pdl_begin();
    TP_TRACE(0);

    const int per = gtot / kFinCS;  // chunks owned by this CTA (power of two)
    const int64_t Llo = n / gtot, ext = n % gtot;
    auto cstart = [&](int64_t g) { return g * Llo + (g < ext ? g : ext); };
    const int64_t g0 = (int64_t)cta * per;
    const int64_t r0 = cstart(g0);
    const int rows = (int)(cstart(g0 + per) - r0);
    for (int i = tid; i < rows; i += kFinNT) {
        sa[i] = __ldg(sys.sub + r0 + i);
        sb[i] = __ldg(sys.diag + r0 + i);
        sc[i] = __ldg(sys.sup + r0 + i);
        sd[i] = __ldg(sys.rhs + r0 + i);
    }
    __syncthreads();
    TP_TRACE(1);

    // ---- leaf: this thread's chunk (2..4 rows) in registers ----
    const bool active = tid < per;
    const int64_t g = g0 + tid;
    const int len = active ? (int)(Llo + (g < ext ? 1 : 0)) : 2;
    const int64_t grow = active ? cstart(g) : 0;
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
    MergeSave<T> sw[5];
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
        const int h = 1 << lv;
        const Eq2<T> oth = shfl_down_eq(cur, h);
        if (h < per && (lane & (2 * h - 1)) == 0 && tid + h < per)
            cur = merge(cur, oth, cstart(g + h) - 1, bad, sw[lv]);
    }
    const int nwr = per >= 32 ? per / 32 : 1;
    if (lane == 0 && warp < nwr) wroot[warp] = cur;
    __syncthreads();
    TP_TRACE(3);

    // ---- warp 0: the CTA's warp roots (<= 3 levels) ----
    MergeSave<T> sx[3];
    Eq2<T> wc = Eq2<T>{0, 1, 0, 0, 0, 1, 0, 0};
    if (warp == 0) {
        wc = lane < nwr ? wroot[lane] : wc;
#pragma unroll
        for (int lv = 0; lv < 3; ++lv) {
            const int h = 1 << lv;
            const Eq2<T> oth = shfl_down_eq(wc, h);
            if (h < nwr && (lane & (2 * h - 1)) == 0 && lane + h < nwr)
                wc = merge(wc, oth, cstart(g0 + 32 * (lane + h)) - 1, bad, sx[lv]);
        }
        if (lane == 0) croot = wc;
    }
    TP_TRACE(4);
    cl.sync();
    TP_TRACE(5);

    // ---- CTA 0, warp 0: the CTA roots (3 levels), the root, and back down ----
    if (cta == 0 && warp == 0) {
        Eq2<T> cc = Eq2<T>{0, 1, 0, 0, 0, 1, 0, 0};
        if (lane < kFinCS) cc = *cl.map_shared_rank(&croot, lane);
        MergeSave<T> sc3[3];
#pragma unroll
        for (int lv = 0; lv < 3; ++lv) {
            const int h = 1 << lv;
            const Eq2<T> oth = shfl_down_eq(cc, h);
            if ((lane & (2 * h - 1)) == 0 && lane + h < kFinCS)
                cc = merge(cc, oth, cstart((int64_t)per * (lane + h)) - 1, bad, sc3[lv]);
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
            for (int lv = 2; lv >= 0; --lv) {
                const int h = 1 << lv;
                T xt = 0;
                if ((lane & (2 * h - 1)) == 0) xt = merge_xt(sc3[lv], xs, xe);
                const T rxt = __shfl_up_sync(0xffffffffu, xt, h);
                const T rxe = __shfl_up_sync(0xffffffffu, xe, h);
                if ((lane & (2 * h - 1)) == h) {
                    xs = first_from_e1(cc, rxt, rxe);
                    xe = rxe;
                } else if ((lane & (2 * h - 1)) == 0) {
                    xe = xt;
                }
            }
            if (lane < kFinCS) {
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
        report_pivot(err, level, bad.bad);
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
    if (active) {
        T xv[4];
        if (len == 2) leaf_expand<T, 4, 2>(r, rb, gm, dl, xs, xe, xv);
        else if (len == 3) leaf_expand<T, 4, 3>(r, rb, gm, dl, xs, xe, xv);
        else leaf_expand<T, 4, 4>(r, rb, gm, dl, xs, xe, xv);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (i < len) x[grow + i] = xv[i];
    }
    TP_TRACE(9);
    TP_TRACE(10);
    TP_TRACE(11);
    if (blockIdx.x == 0) TP_TRACE_FLUSH;
    report_pivot(err, level, bad.bad);
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
