// sm_100a kernels of the B200 partition solver (FP64, HBM-bound).
//
// Kernel map (reference call stack partition.hpp:191-224):
//   k_fast<T,L,G,STAGE1> parallel_for(reduce_block) + assemble_interface   :203-205
//   k_fast<T,L,G,STAGE3> parallel_for(back_substitute + scatter)            :214-222
//   k_fast_rt<T,...>     the same for any m <= 256 (runtime chunk lengths)
//   k_generic<T,MODE>    the same for any block length (tail blocks, m > 256)
//   k_final<T,MODE>      single-CTA finishing solve replacing
//                        thomas_solve(iface) at the deepest level          :208-211
//   k_gather_solve       sharded top level: Thomas on the all-gathered 2P rows
//   k_generate           device-side counter-based generate_system analogue
//   k_residual           residual_inf (tridiagonal.hpp:74-87)
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

#include <cooperative_groups.h>

#include "tp_device.cuh"
#include "tp_kernels.h"
#include "tp_fast.cuh"

namespace tpb {

// Phase timestamps of the finishing solve (scratch builds with -DTPB_TRACE only).
#ifdef TPB_TRACE
__device__ unsigned long long g_trace[16];
#define TP_TRACE_DECL long long tp_tr[12]
#define TP_TRACE(k) tp_tr[k] = clock64()
#define TP_TRACE_FLUSH \
    do { if (threadIdx.x == 0) for (int k_ = 0; k_ < 12; ++k_) g_trace[k_] = tp_tr[k_]; } while (0)
#else
#define TP_TRACE_DECL
#define TP_TRACE(k) do { } while (0)
#define TP_TRACE_FLUSH do { } while (0)
#endif

// ===========================================================================
// Generic path: any block length, rows staged through shared memory.
// CTA of T threads; G lanes per block (G power of two, G <= T); each lane owns
// a chunk of floor/ceil(blen/G) >= 2 rows. Lane-tree via shuffles below the
// warp, via shared memory above it.
// ===========================================================================
template <class T>
struct GenShared {
    T* a;
    T* b;
    T* c;
    T* d;
    Eq2<T>* xeq;       // one slot per warp (cross-warp merges)
    T* xpass;  // 2 per warp (cross-warp top-down)
};

// Leaf on a shared-memory chunk [p, p+len). When KEEP, overwrites b <- rcp(beta),
// c <- gamma, d <- delta for the interior rows (consumed by leaf expansion).
template <class T, bool KEEP, class Gd>
__device__ Eq2<T> leaf_smem(T* a, T* b, T* c, T* d, int len, int64_t grow0, Gd& bad) {
    Eq2<T> q;
    if (len == 1) {  // only in the n == 1 solve
        q.a1 = a[0]; q.b1 = b[0]; q.g1 = c[0]; q.d1 = d[0];
        q.a2 = a[0]; q.b2 = b[0]; q.g2 = c[0]; q.d2 = d[0];
        return q;
    }
    // down-sweep first (reads originals): partition.hpp:110-124
    T phi = a[1], bp = b[1], dp = d[1];
    for (int i = 2; i < len; ++i) {
        bad.see(bp, grow0 + i - 1);
        const T w = a[i] * rcp(bp);
        phi = -w * phi;
        bp = b[i] - w * c[i - 1];
        dp = d[i] - w * dp;
    }
    q.a2 = phi;
    q.b2 = bp;
    q.g2 = c[len - 1];
    q.d2 = dp;
    // up-sweep: partition.hpp:90-108
    T beta = b[len - 2], gamma = c[len - 2], delta = d[len - 2];
    if (KEEP) { c[len - 2] = gamma; d[len - 2] = delta; }
    for (int i = len - 3; i >= 0; --i) {
        bad.see(beta, grow0 + i + 1);
        const T rb = rcp(beta);
        const T w = c[i] * rb;
        const T nb = b[i] - w * a[i + 1];
        const T ng = -w * gamma;
        const T nd = d[i] - w * delta;
        if (KEEP) { b[i + 1] = rb; c[i] = ng; d[i] = nd; }
        beta = nb; gamma = ng; delta = nd;
    }
    q.a1 = a[0];
    q.b1 = beta;
    q.g1 = gamma;
    q.d1 = delta;
    return q;
}

template <class T, int MODE>
__global__ void __launch_bounds__(kFinalThreads) k_generic(SysPtrs<T> sys, int64_t row_base, int64_t blk_base, int64_t nblocks,
                          int64_t blen, int G, IfacePtrs<T> out, const T* __restrict__ xi,
                          T* __restrict__ x, unsigned long long* err, int level) {
    extern __shared__ __align__(16) unsigned char gsm_raw[];
    T* gsm = reinterpret_cast<T*>(gsm_raw);
    const int NT = blockDim.x;
    const int bpc = NT / G;
    const int64_t tile_rows_max = (int64_t)bpc * blen;
    GenShared<T> s;
    s.a = gsm;
    s.b = s.a + tile_rows_max;
    s.c = s.b + tile_rows_max;
    s.d = s.c + tile_rows_max;
    s.xeq = reinterpret_cast<Eq2<T>*>(s.d + tile_rows_max);
    s.xpass = reinterpret_cast<T*>(s.xeq + (NT + 31) / 32);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int c = tid % G;
    const int lb = tid / G;
    const int64_t Llo = blen / G;
    const int64_t ext = blen % G;
    const int len = (int)(Llo + (c < ext ? 1 : 0));
    const int64_t off = c * Llo + (c < ext ? c : ext);
    int logg = 0;
    while ((1 << logg) < G) ++logg;
    // Stage 3 repeats Stage 1's arithmetic on the same rows: no pivot guard
    typename std::conditional<MODE == kStage3, NoRowGuard, RowGuard>::type bad;
    constexpr bool KEEP = (MODE != kStage1);
    pdl_begin();

    const int64_t ntiles = (nblocks + bpc - 1) / bpc;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t b0 = tile * bpc;
        const int64_t nbt = (nblocks - b0) < bpc ? (nblocks - b0) : bpc;
        const int64_t trow0 = row_base + b0 * blen;
        const int64_t trows = nbt * blen;
        for (int64_t i = tid; i < trows; i += NT) {
            s.a[i] = sys.sub[trow0 + i];
            s.b[i] = sys.diag[trow0 + i];
            s.c[i] = sys.sup[trow0 + i];
            s.d[i] = sys.rhs[trow0 + i];
        }
        __syncthreads();
        const bool active = lb < nbt;
        const int64_t lrow = (int64_t)lb * blen + off;  // local row of the chunk start
        const int64_t grow = trow0 + lrow;               // level row of the chunk start
        Eq2<T> cur;
        if (active) {
            cur = leaf_smem<T, KEEP>(s.a + lrow, s.b + lrow, s.c + lrow, s.d + lrow, len, grow, bad);
        } else {
            cur = Eq2<T>{0, 1, 0, 0, 0, 1, 0, 0};
        }
        // ---- up the lane tree ----
        MergeSave<T> sv[10];
        for (int lv = 0; lv < logg; ++lv) {
            const int h = 1 << lv;
            Eq2<T> oth;
            if (h < 32) {
                oth = shfl_down_eq(cur, h);
            } else {
                if ((c & (2 * h - 1)) == h) s.xeq[tid >> 5] = cur;
                __syncthreads();
                if ((c & (2 * h - 1)) == 0) oth = s.xeq[(tid + h) >> 5];
                __syncthreads();
            }
            if ((c & (2 * h - 1)) == 0 && active) {
                // row_t = last row of segment A = chunk (c+h-1)'s last row
                const int64_t ca = c + h;  // first chunk of B
                const int64_t offb = ca * Llo + (ca < ext ? ca : ext);
                const int64_t row_t = trow0 + (int64_t)lb * blen + offb - 1;
                cur = merge(cur, oth, row_t, bad, sv[lv]);
            }
        }
        // ---- root ----
        T xs = 0, xe = 0;
        if (c == 0 && active) {
            const int64_t jb = blk_base + b0 + lb;
            if (MODE == kStage1) {
                out.sub[2 * jb] = cur.a1;     out.sub[2 * jb + 1] = cur.a2;
                out.diag[2 * jb] = cur.b1;    out.diag[2 * jb + 1] = cur.b2;
                out.sup[2 * jb] = cur.g1;     out.sup[2 * jb + 1] = cur.g2;
                out.rhs[2 * jb] = cur.d1;     out.rhs[2 * jb + 1] = cur.d2;
            } else if (MODE == kStage3) {
                xs = xi[2 * jb];
                xe = xi[2 * jb + 1];
            } else {  // kSolve: the whole system is this one block
                if (blen == 1) {
                    bad.see(cur.b1, 0);
                    xs = xe = cur.d1 * rcp(cur.b1);
                } else {
                    root_solve(cur, blen - 1, bad, xs, xe);
                }
            }
        }
        if (MODE != kStage1) {
            // ---- down the lane tree ----
            for (int lv = logg - 1; lv >= 0; --lv) {
                const int h = 1 << lv;
                T xt = 0;
                if ((c & (2 * h - 1)) == 0) xt = merge_xt(sv[lv], xs, xe);
                T rxt, rxe;
                if (h < 32) {
                    rxt = __shfl_up_sync(0xffffffffu, xt, h);
                    rxe = __shfl_up_sync(0xffffffffu, xe, h);
                } else {
                    if ((c & (2 * h - 1)) == 0) {
                        s.xpass[2 * ((tid + h) >> 5)] = xt;
                        s.xpass[2 * ((tid + h) >> 5) + 1] = xe;
                    }
                    __syncthreads();
                    rxt = s.xpass[2 * (tid >> 5)];
                    rxe = s.xpass[2 * (tid >> 5) + 1];
                    __syncthreads();
                }
                if ((c & (2 * h - 1)) == h) {
                    xs = first_from_e1(cur, rxt, rxe);
                    xe = rxe;
                } else if ((c & (2 * h - 1)) == 0) {
                    xe = xt;
                }
            }
            // ---- leaf expansion into the a-slots, then coalesced store ----
            if (active) {
                T* a = s.a + lrow;
                const T* rb = s.b + lrow;
                const T* g = s.c + lrow;
                const T* dd = s.d + lrow;
                T prev = xs;
                for (int i = 1; i < len - 1; ++i) {
                    const T xv = (dd[i] - a[i] * prev - g[i] * xe) * rb[i];
                    a[i] = xv;
                    prev = xv;
                }
                a[0] = xs;
                if (len > 1) a[len - 1] = xe;
            }
            __syncthreads();
            for (int64_t i = tid; i < trows; i += NT) x[trow0 + i] = s.a[i];
        }
        __syncthreads();
        (void)lane;
    }
    report_pivot(err, level, bad.bad);
}

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

// ===========================================================================
// Device generator: same distributions as generate_system (bench.hpp:68-93)
// — a,c,d ~ U[-1,1), b = delta*(|a|+|c|)+1, whole-row sign flip with p=0.5,
// sub[0] = super[N-1] = 0 — from a counter-based hash of (seed, global row),
// so any shard generates its slice of the same global system. NOT
// bit-identical to std::mt19937_64; used for throughput runs only. Values
// are drawn in FP64 and rounded to T.
// ===========================================================================
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double canon(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

template <class T>
__global__ void k_generate(int64_t n, int64_t row0, int64_t n_global, uint64_t seed, double delta,
                           T* __restrict__ sub, T* __restrict__ diag, T* __restrict__ sup,
                           T* __restrict__ rhs) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t g = (uint64_t)(row0 + i);
        const uint64_t k = mix64(seed * 0x9E3779B97F4A7C15ULL + 0x632BE59BD9B4E019ULL) ^ (g * 4);
        double a = canon(mix64(k + 0)) * 2.0 - 1.0;
        double cc = canon(mix64(k + 1)) * 2.0 - 1.0;
        double d = canon(mix64(k + 2)) * 2.0 - 1.0;
        const bool fl = canon(mix64(k + 3)) < 0.5;
        if (row0 + i == 0) a = 0.0;
        if (row0 + i == n_global - 1) cc = 0.0;
        double b = delta * (fabs(a) + fabs(cc)) + 1.0;
        if (fl) { a = -a; b = -b; cc = -cc; d = -d; }
        sub[i] = (T)a;
        diag[i] = (T)b;
        sup[i] = (T)cc;
        rhs[i] = (T)d;
    }
}

// residual_inf (tridiagonal.hpp:74-87): out[0] = max|Ax-d|, out[1] = max(1, max|d|),
// accumulated in FP64 and kept as order-preserving uint64 bit patterns of
// non-negative doubles.
template <class T>
__global__ void k_residual(SysPtrs<T> sys, int64_t n, const T* __restrict__ x, unsigned long long* out) {
    double num = 0, den = 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double ax = (double)sys.diag[i] * x[i];
        if (i > 0) ax += (double)sys.sub[i] * x[i - 1];
        if (i + 1 < n) ax += (double)sys.sup[i] * x[i + 1];
        num = fmax(num, fabs(ax - (double)sys.rhs[i]));
        den = fmax(den, fabs((double)sys.rhs[i]));
    }
    for (int o = 16; o > 0; o >>= 1) {
        num = fmax(num, __shfl_down_sync(0xffffffffu, num, o));
        den = fmax(den, __shfl_down_sync(0xffffffffu, den, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out + 0, (unsigned long long)__double_as_longlong(num));
        atomicMax(out + 1, (unsigned long long)__double_as_longlong(den));
    }
}

// ===========================================================================
// Launchers
// ===========================================================================

// Launch policy, fixed once by init_kernel_attributes(): with TPB_PDL=1 the
// solve-path kernels go out with the programmatic-stream-serialization
// attribute (PDL; inside a captured graph the edges become programmatic
// edges). Every such kernel begins with pdl_begin(), so it is correct either
// way. Off by default: measured on B200 (tools/timeline.py, C3) it saves ~6 us
// across the levels >= 1 but the persistent Stage-3 grid launched early
// behind level 1 runs ~50 us slower.
static bool g_pdl = false;

template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                            cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Error-word reset at the head of every solve (a kernel rather than a memset
// node, so the first Stage-1 grid can be launched programmatically after it).
__global__ void k_reset(unsigned long long* err) {
    pdl_begin();
    if (threadIdx.x == 0) *err = kNoError;
}

cudaError_t launch_reset(unsigned long long* err, cudaStream_t st) {
    return launch_k(k_reset, 1, 32, 0, st, err);
}

// Launch shapes chosen by measurement (tools/microbench/level_shapes.cu and
// in-graph A/B runs on B200, N=1e8, m=64):
// Stage 1  128 threads, <=80 regs (6 CTAs/SM), one chunk per thread (full grid)
// Stage 3  128 threads, <=128 regs (4 CTAs/SM), one chunk per thread (full
//          grid: 1.2% faster in the solve graph than a persistent grid-stride)
template <class T, int L, int G, int MODE, bool VEC>
struct FastCfg {
    static constexpr int kThreads = 128;
    static constexpr int kMinBlocks = (MODE == kStage1) ? 6 : 4;
    static void* fn() { return (void*)k_fast<T, L, G, MODE, VEC, kThreads, kMinBlocks>; }
};

template <class T, int L, int G, bool VEC>
static cudaError_t launch_fast_t(int mode, const SysPtrs<T>& sys, int64_t nblocks,
                                 const IfacePtrs<T>& out, const T* xi, T* x, unsigned long long* err,
                                 int level, cudaStream_t st) {
    const int64_t nchunks = nblocks * G;
    if (mode == kStage1) {
        using C = FastCfg<T, L, G, kStage1, VEC>;
        int64_t grid = (nchunks + C::kThreads - 1) / C::kThreads;
        if (grid < 1) grid = 1;
        return launch_k(k_fast<T, L, G, kStage1, VEC, C::kThreads, C::kMinBlocks>, (unsigned)grid,
                        C::kThreads, 0, st, sys, nblocks, out, xi, x, err, level);
    } else {
        using C = FastCfg<T, L, G, kStage3, VEC>;
        int64_t grid = (nchunks + C::kThreads - 1) / C::kThreads;
        if (grid < 1) grid = 1;
        return launch_k(k_fast<T, L, G, kStage3, VEC, C::kThreads, C::kMinBlocks>, (unsigned)grid,
                        C::kThreads, 0, st, sys, nblocks, out, xi, x, err, level);
    }
}

template <class T, int L, int G>
static cudaError_t launch_fast_v(bool vec, int mode, const SysPtrs<T>& sys, int64_t nblocks,
                                 const IfacePtrs<T>& out, const T* xi, T* x, unsigned long long* err,
                                 int level, cudaStream_t st) {
    if (vec) return launch_fast_t<T, L, G, true>(mode, sys, nblocks, out, xi, x, err, level, st);
    return launch_fast_t<T, L, G, false>(mode, sys, nblocks, out, xi, x, err, level, st);
}

// m -> (rows per lane L, lanes per block G) of the fixed-shape kernels
#define TPB_FAST_SHAPES(X) \
    X(4, 4, 1)             \
    X(5, 5, 1)             \
    X(8, 8, 1)             \
    X(10, 5, 2)            \
    X(16, 8, 2)            \
    X(20, 5, 4)            \
    X(32, 8, 4)            \
    X(40, 5, 8)            \
    X(64, 8, 8)            \
    X(80, 5, 16)           \
    X(128, 8, 16)          \
    X(160, 5, 32)          \
    X(256, 8, 32)

bool fast_shape(int64_t m, int* L, int* G) {
#define TPB_SHAPE(MM, LL, GG) \
    case MM: *L = LL; *G = GG; return true;
    switch (m) {
        TPB_FAST_SHAPES(TPB_SHAPE)
        default: return false;
    }
#undef TPB_SHAPE
}

template <class T>
cudaError_t launch_fast(int64_t m, bool vec, int mode, const SysPtrs<T>& sys, int64_t nblocks,
                        const IfacePtrs<T>& out, const T* xi, T* x, unsigned long long* err,
                        int level, cudaStream_t st) {
#define TPB_CASE(MM, LL, GG) \
    case MM: return launch_fast_v<T, LL, GG>(vec, mode, sys, nblocks, out, xi, x, err, level, st);
    switch (m) {
        TPB_FAST_SHAPES(TPB_CASE)
        default: return cudaErrorInvalidValue;
    }
#undef TPB_CASE
}


// Runtime-length register path (k_fast_rt): the G with ceil(m/G) <= 8, m/G >= 2.
int fast_rt_G(int64_t m) {
    if (m < 2 || m > 256) return 0;
    int G = 1;
    while ((m + G - 1) / G > 8) G *= 2;
    return (G <= 32 && m / G >= 2) ? G : 0;
}

template <class T>
cudaError_t launch_fast_rt(int64_t m, int mode, const SysPtrs<T>& sys, int64_t nblocks,
                           const IfacePtrs<T>& out, const T* xi, T* x, unsigned long long* err,
                           int level, int sms, cudaStream_t st) {
    const int G = fast_rt_G(m);
    if (G == 0) return cudaErrorInvalidValue;
    const int64_t nchunks = nblocks * G;
    int64_t grid = (nchunks + 127) / 128;  // one tile per CTA, both stages
    (void)sms;
    if (grid < 1) grid = 1;
#define TPB_RT(GG)                                                                                     \
    case GG:                                                                                           \
        if (mode == kStage1)                                                                           \
            return launch_k(k_fast_rt<T, 8, GG, kStage1>, (unsigned)grid, 128, 0, st, sys, nblocks, m, out, xi, x, err, level); \
        return launch_k(k_fast_rt<T, 8, GG, kStage3>, (unsigned)grid, 128, 0, st, sys, nblocks, m, out, xi, x, err, level);
    switch (G) {
        TPB_RT(1)
        TPB_RT(2)
        TPB_RT(4)
        TPB_RT(8)
        TPB_RT(16)
        TPB_RT(32)
        default: return cudaErrorInvalidValue;
    }
#undef TPB_RT
}

size_t generic_smem_bytes(int threads, int G, int64_t blen, size_t elem) {
    const int64_t bpc = threads / G;
    const size_t warps = (size_t)((threads + 31) / 32);
    return (size_t)(4 * bpc * blen) * elem + warps * 8 * elem + warps * 2 * elem;
}

template <class T>
cudaError_t launch_generic(int mode, int threads, int G, int grid, const SysPtrs<T>& sys,
                           int64_t row_base, int64_t blk_base, int64_t nblocks, int64_t blen,
                           const IfacePtrs<T>& out, const T* xi, T* x, unsigned long long* err,
                           int level, cudaStream_t st) {
    const size_t smem = generic_smem_bytes(threads, G, blen, sizeof(T));
    if (smem > kMaxDynSmem) return cudaErrorInvalidValue;
    auto k = mode == kStage1 ? k_generic<T, kStage1> : mode == kStage3 ? k_generic<T, kStage3> : k_generic<T, kSolve>;
    return launch_k(k, (unsigned)grid, (unsigned)threads, smem, st, sys, row_base, blk_base, nblocks, blen, G,
                    out, xi, x, err, level);
}

// The cluster finishing solve (k_final_cl) takes every system of at least
// kFinClusterMin rows (TPB_FINAL_CLUSTER=0 keeps the single-CTA k_final).
constexpr int64_t kFinClusterMin = 64;
static bool g_final_cluster = true;

static int final_G(int64_t n) {
    int G = 1;
    while (G * 2 <= kFinalThreads2 && n / (G * 2) >= 2) G *= 2;
    return G;
}

template <class T>
cudaError_t launch_final(int mode, const SysPtrs<T>& sys, int64_t n, const IfacePtrs<T>& out,
                         const T* xi, T* x, unsigned long long* err, int level, cudaStream_t st,
                         const ShardLink* link) {
    if (n > kFinalCap || n < 1) return cudaErrorInvalidValue;
    if (mode == kShard && (link == nullptr || link->nranks < 1 || link->nranks > kMaxPeers))
        return cudaErrorInvalidValue;
    if (g_final_cluster && n >= kFinClusterMin) {
        int gtot = kFinCS;
        while (gtot * 2 <= kFinCS * kFinNT && n / (gtot * 2) >= 2) gtot *= 2;
        auto kc = mode == kStage1   ? k_final_cl<T, kStage1>
                  : mode == kStage3 ? k_final_cl<T, kStage3>
                  : mode == kShard  ? k_final_cl<T, kShard>
                                    : k_final_cl<T, kSolve>;
        const ShardLink none{};
        return launch_k(kc, kFinCS, kFinNT, 0, st, sys, n, gtot, out, xi, x, err, level,
                        link != nullptr ? *link : none);
    }
    const int G = final_G(n);
    const size_t smem = (size_t)(4 * n) * sizeof(T);
    auto k = mode == kStage1   ? k_final<T, kStage1>
             : mode == kStage3 ? k_final<T, kStage3>
             : mode == kShard  ? k_final<T, kShard>
                               : k_final<T, kSolve>;
    const ShardLink none{};
    return launch_k(k, 1, kFinalThreads2, smem, st, sys, n, G, out, xi, x, err, level,
                    link != nullptr ? *link : none);
}

template <class T>
static cudaError_t set_smem_attributes() {
    const int fs = (int)(kMaxDynSmem - 4096);
    cudaError_t e = cudaFuncSetAttribute(k_generic<T, kStage1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDynSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_generic<T, kStage3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDynSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_generic<T, kSolve>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDynSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_final<T, kStage1>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_final<T, kStage3>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_final<T, kSolve>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_final<T, kShard>, cudaFuncAttributeMaxDynamicSharedMemorySize, fs);
    return e;
}

// Experiment switch TPB_CARVEOUT=<percent>: preferred shared-memory carveout
// of the register-path kernels (by default the driver picks one per kernel).
template <class T>
static cudaError_t set_carveout(int pct) {
    cudaError_t e = cudaSuccess;
#define TPB_CO(MM, LL, GG)                                                                              \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(FastCfg<T, LL, GG, kStage1, true>::fn(), cudaFuncAttributePreferredSharedMemoryCarveout, pct);  \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(FastCfg<T, LL, GG, kStage1, false>::fn(), cudaFuncAttributePreferredSharedMemoryCarveout, pct); \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(FastCfg<T, LL, GG, kStage3, true>::fn(), cudaFuncAttributePreferredSharedMemoryCarveout, pct);  \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(FastCfg<T, LL, GG, kStage3, false>::fn(), cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    TPB_FAST_SHAPES(TPB_CO)
#undef TPB_CO
    return e;
}

cudaError_t init_kernel_attributes() {
    if (const char* v = getenv("TPB_PDL")) g_pdl = atoi(v) != 0;
    if (const char* v = getenv("TPB_FINAL_CLUSTER")) g_final_cluster = atoi(v) != 0;
    cudaError_t e = set_smem_attributes<double>();
    if (e == cudaSuccess) e = set_smem_attributes<float>();
    if (const char* v = getenv("TPB_CARVEOUT")) {
        if (e == cudaSuccess) e = set_carveout<double>(atoi(v));
        if (e == cudaSuccess) e = set_carveout<float>(atoi(v));
    }
    return e;
}

template <class T>
cudaError_t launch_gather_solve(const T* eqs, int nranks, int rank, T* x2, T* scratch,
                                unsigned long long* err, int level, cudaStream_t st) {
    return launch_k(k_gather_solve<T>, 1, 32, 0, st, eqs, nranks, rank, x2, scratch, err, level);
}

template <class T>
cudaError_t launch_generate(int64_t n, int64_t row0, int64_t n_global, uint64_t seed, double delta,
                            T* sub, T* diag, T* sup, T* rhs, int sms, cudaStream_t st) {
    int64_t grid = (n + 255) / 256;
    if (grid > (int64_t)sms * 16) grid = (int64_t)sms * 16;
    if (grid < 1) grid = 1;
    k_generate<T><<<(unsigned)grid, 256, 0, st>>>(n, row0, n_global, seed, delta, sub, diag, sup, rhs);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_residual(const SysPtrs<T>& sys, int64_t n, const T* x, unsigned long long* out,
                            int sms, cudaStream_t st) {
    int64_t grid = (n + 255) / 256;
    if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
    if (grid < 1) grid = 1;
    k_residual<T><<<(unsigned)grid, 256, 0, st>>>(sys, n, x, out);
    return cudaGetLastError();
}

// explicit instantiations for the two element types of the C-ABI
#define TPB_INSTANTIATE(T)                                                                          \
    template cudaError_t launch_fast<T>(int64_t, bool, int, const SysPtrs<T>&, int64_t,             \
                                        const IfacePtrs<T>&, const T*, T*, unsigned long long*, int, \
                                        cudaStream_t);                                         \
    template cudaError_t launch_fast_rt<T>(int64_t, int, const SysPtrs<T>&, int64_t,                \
                                           const IfacePtrs<T>&, const T*, T*, unsigned long long*,  \
                                           int, int, cudaStream_t);                                 \
    template cudaError_t launch_generic<T>(int, int, int, int, const SysPtrs<T>&, int64_t, int64_t, \
                                           int64_t, int64_t, const IfacePtrs<T>&, const T*, T*,    \
                                           unsigned long long*, int, cudaStream_t);                 \
    template cudaError_t launch_final<T>(int, const SysPtrs<T>&, int64_t, const IfacePtrs<T>&,      \
                                         const T*, T*, unsigned long long*, int, cudaStream_t,      \
                                         const ShardLink*);                                         \
    template cudaError_t launch_gather_solve<T>(const T*, int, int, T*, T*, unsigned long long*,    \
                                                int, cudaStream_t);                                 \
    template cudaError_t launch_generate<T>(int64_t, int64_t, int64_t, uint64_t, double, T*, T*,    \
                                            T*, T*, int, cudaStream_t);                             \
    template cudaError_t launch_residual<T>(const SysPtrs<T>&, int64_t, const T*,                   \
                                            unsigned long long*, int, cudaStream_t);
TPB_INSTANTIATE(double)
TPB_INSTANTIATE(float)
#undef TPB_INSTANTIATE

}  // namespace tpb

namespace tpb {
// Diagnostic: max distance in ulps between rcp(x) and the correctly rounded
// 1/x over `n` pseudo-random x spanning [1e-30, 1e30) with random sign.
__global__ void k_diag_rcp(int64_t n, uint64_t seed, unsigned long long* max_ulp) {
    unsigned long long worst = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix64(seed ^ (uint64_t)i * 0x9E3779B97F4A7C15ULL);
        const double u = canon(h);
        double x = exp10(60.0 * u - 30.0);
        if (h & 1) x = -x;
        const double a = rcp(x), b = __drcp_rn(x);
        const long long ia = __double_as_longlong(a), ib = __double_as_longlong(b);
        const unsigned long long d = (unsigned long long)(ia > ib ? ia - ib : ib - ia);
        worst = d > worst ? d : worst;
    }
    atomicMax(max_ulp, worst);
}
}  // namespace tpb

#ifdef TPB_TRACE
extern "C" int tp_debug_trace(uint64_t* out) {
    return cudaMemcpyFromSymbol(out, tpb::g_trace, sizeof(tpb::g_trace)) == cudaSuccess ? 0 : 9;
}
#endif

extern "C" int tp_diag_rcp_ulp(int64_t n, uint64_t seed, uint64_t* max_ulp) {
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, sizeof(unsigned long long)) != cudaSuccess) return 9;
    cudaMemset(d, 0, sizeof(unsigned long long));
    tpb::k_diag_rcp<<<148 * 4, 256>>>(n, seed, d);
    unsigned long long h = 0;
    const cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return 9;
    *max_ulp = h;
    return 0;
}
