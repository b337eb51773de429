// Generic level kernel (k_generic): any block length, rows staged through
// shared memory; used for tail blocks and m > 256. Included by tp_kernels.cu.
#pragma once
#include <type_traits>

#include "tp_device.cuh"

namespace tpb {

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
            bool nf = false;
            for (int64_t i = tid; i < trows; i += NT) {
                const T v = s.a[i];
                x[trow0 + i] = v;
                nf |= !isfinite(v);
            }
            if (nf) report_nonfinite(err, trow0);
        }
        __syncthreads();
        (void)lane;
    }
    report_pivot(err, level, bad.bad);
}

}  // namespace tpb
