// Whole-system solve on one co-resident grid (k_grid_solve), for mid-size
// one-level policies whose rows fit the GPU's aggregate shared memory
// (FP64: up to ~1.0e6 rows on 148 SMs; config 2 = N 1e6, policy {32}).
//
// The level path for such a system is three latency-bound kernels: Stage 1
// (1e6 rows -> a 62,500-row interface), the finishing solve of that interface
// on ONE 16-CTA cluster (16 of 148 SMs, 10.5 us of a 23 us solve), Stage 3.
// Here every SM owns a contiguous run of whole level-0 blocks
// (make_plan, partition.hpp:30-49), stages it in shared memory ONCE
// (per-element cp.async into a padded layout; k_grid_hyb: 256-bit register
// loads), and the rest never leaves the chip:
//   leaf sweeps of each chunk (reduce_block's up-/down-sweep, partition.hpp:
//   90-124, intermediate values kept in place for back_substitute :156-172)
//   -> chunk tree (shuffles, then warp roots) to the CTA's pair E1/E2
//   -> the P CTA pairs published to global memory, ONE grid barrier
//   -> every CTA merges the P pairs (the same tree, redundantly: no second
//      barrier), solves the 2x2 root (thomas_solve on [E1; E2],
//      tridiagonal.hpp:52-72) and walks down to its own (x_s, x_e)
//   -> its own tree top-down, leaf back-substitution in shared memory, one
//      coalesced store of x.
// HBM traffic: the 32 B/row inputs read once and x written once (40 B/row,
// the north-star floor) — no interface system, no Stage-3 re-read.
//
// A level-0 block of m rows is g chunks (g a power of two), i.e. one subtree
// of the chunk tree, so the block's E1/E2 are formed exactly as k_fast forms
// them; the interface of level 0 is then reduced by the tree instead of
// thomas_solve — an exact elimination, equal to the reference's x up to
// rounding (parity by tolerance). Pivots below kPivotFloor are
// reported like every other kernel's (row of the device's elimination order);
// the host then replays the reference's order (diagnose_pivot).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tp_device.cuh"
#include "tp_exchange.cuh"
#include "tp_fast.cuh"
#include "tp_generic.cuh"
#include "tp_kernels.h"

namespace tpb {

namespace {

// A copy of v the compiler cannot rematerialise: keeps loop-carried indices
// (tid, blockIdx) in registers instead of re-reading them with S2R, whose
// latency sat on the serial tree loops' critical path.
__device__ __forceinline__ int pin_reg(int v) {
    int r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async_elem(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_elem(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <class T>
__device__ __forceinline__ Eq2<T> identity_eq() {
    return Eq2<T>{0, 1, 0, 0, 0, 1, 0, 0};
}

// Shared-memory slot of CTA-local row i: one pad element after every 2^qs
// rows, so that 32 threads sweeping 32 consecutive chunks of a power-of-two
// length <= 2^qs hit 16 distinct 8-byte bank pairs (2 wavefronts, the
// minimum for 32 FP64 accesses; an unpadded chunk stride of 16 rows puts
// every lane of a warp on ONE bank pair: 32 wavefronts).
__device__ __forceinline__ int padx(int i, int qs) { return i + (i >> qs); }

// reduce_block's sweeps (partition.hpp:90-124) on one chunk from the padded
// shared-memory rows, next row's values prefetched one step ahead (the loop
// is otherwise bound by shared-memory load latency). The up-sweep overwrites
// b <- rcp(beta), c <- gamma, d <- delta of the interior rows in place for
// back_substitute (:156-172). Called for two chunks per thread, whose two
// dependency chains the scheduler interleaves.
template <class T>
struct Row4 {
    T a, b, c, d;
};
template <class T>
__device__ __forceinline__ Row4<T> ld_row(const T* a, const T* b, const T* c, const T* d, int q) {
    return Row4<T>{a[q], b[q], c[q], d[q]};
}

template <class T>
__device__ __forceinline__ void sweep_down(const T* a, const T* b, const T* c, const T* d, int l0, int len, int qs,
                                           bool& flag, Eq2<T>& E) {
    const T fl = pivot_floor<T>();
    const Row4<T> r1 = ld_row(a, b, c, d, padx(l0 + 1, qs));
    T ph = r1.a, bp = r1.b, dp = r1.d, cp = r1.c;
    Row4<T> nx = len > 2 ? ld_row(a, b, c, d, padx(l0 + 2, qs)) : r1;
    for (int i = 2; i < len; ++i) {
        const Row4<T> r = nx;
        if (i + 1 < len) nx = ld_row(a, b, c, d, padx(l0 + i + 1, qs));
        flag |= fabs(bp) < fl;
        const T w = r.a * rcp(bp);
        ph = -w * ph;
        bp = fma(-w, cp, r.b);
        dp = fma(-w, dp, r.d);
        cp = r.c;
    }
    E.a2 = ph;
    E.b2 = bp;
    E.g2 = cp;
    E.d2 = dp;
}

template <class T>
__device__ __forceinline__ void sweep_up(T* a, T* b, T* c, T* d, int l0, int len, int qs, bool& flag, Eq2<T>& E) {
    const T fl = pivot_floor<T>();
    int qp = padx(l0 + len - 2, qs);
    const Row4<T> s = ld_row(a, b, c, d, qp);
    T bt = s.b, gm = s.c, dl = s.d, an = s.a;
    Row4<T> nx = len > 2 ? ld_row(a, b, c, d, padx(l0 + len - 3, qs)) : s;
    for (int i = len - 3; i >= 0; --i) {
        const int q = padx(l0 + i, qs);
        const Row4<T> r = nx;
        if (i > 0) nx = ld_row(a, b, c, d, padx(l0 + i - 1, qs));
        flag |= fabs(bt) < fl;
        const T rb = rcp(bt);
        const T w = r.c * rb;
        const T nb = fma(-w, an, r.b);
        gm = -w * gm;
        dl = fma(-w, dl, r.d);
        an = r.a;
        b[qp] = rb;
        c[q] = gm;
        d[q] = dl;
        bt = nb;
        qp = q;
    }
    E.a1 = a[padx(l0, qs)];
    E.b1 = bt;
    E.g1 = gm;
    E.d1 = dl;
}

// The same sweeps with the chunk length a compile-time constant (2..8 rows):
// the rows are loaded into registers once, both sweeps are unrolled (two
// independent chains the scheduler interleaves) and the kept values are
// written back to the b, c, d slots.
template <class T, int LEN>
__device__ __forceinline__ void leaf_fixed(T* a, T* b, T* c, T* d, int l0, int qs, bool& flag, Eq2<T>& E) {
    const T fl = pivot_floor<T>();
    T ra[LEN], rb[LEN], rc[LEN], rd[LEN];
    int q[LEN];
#pragma unroll
    for (int i = 0; i < LEN; ++i) {
        q[i] = padx(l0 + i, qs);
        ra[i] = a[q[i]];
        rb[i] = b[q[i]];
        rc[i] = c[q[i]];
        rd[i] = d[q[i]];
    }
    T ph = ra[1], bp = rb[1], dp = rd[1];
#pragma unroll
    for (int i = 2; i < LEN; ++i) {
        flag |= fabs(bp) < fl;
        const T w = ra[i] * rcp(bp);
        ph = -w * ph;
        bp = fma(-w, rc[i - 1], rb[i]);
        dp = fma(-w, dp, rd[i]);
    }
    E.a2 = ph;
    E.b2 = bp;
    E.g2 = rc[LEN - 1];
    E.d2 = dp;
    T bt = rb[LEN - 2], gm = rc[LEN - 2], dl = rd[LEN - 2];
#pragma unroll
    for (int i = LEN - 3; i >= 0; --i) {
        flag |= fabs(bt) < fl;
        const T r = rcp(bt);
        const T w = rc[i] * r;
        const T nb = fma(-w, ra[i + 1], rb[i]);
        gm = -w * gm;
        dl = fma(-w, dl, rd[i]);
        b[q[i + 1]] = r;
        c[q[i]] = gm;
        d[q[i]] = dl;
        bt = nb;
    }
    E.a1 = ra[0];
    E.b1 = bt;
    E.g1 = gm;
    E.d1 = dl;
}

template <class T>
__device__ __forceinline__ void leaf_loop(T* a, T* b, T* c, T* d, int l0, int len, int qs, bool& flag, Eq2<T>& E) {
    sweep_down<T>(a, b, c, d, l0, len, qs, flag, E);
    sweep_up<T>(a, b, c, d, l0, len, qs, flag, E);
}


// An unknown as an affine function of this CTA's end values X0 = x[r0],
// X1 = x[r1-1]:  c + u X0 + v X1. The CTA's tree is walked top-down with
// these BEFORE the grid barrier (Schur steps are linear in (xs, xe)), so after
// the barrier every row is one evaluation x = c + u X0 + v X1.
template <class T>
struct Aff {
    T c, u, v;
};
template <class T>
__device__ __forceinline__ Aff<T> aff_lin(T k, const Aff<T>& p, T l, const Aff<T>& q, T m) {
    // k + l p + m q
    return Aff<T>{fma(m, q.c, fma(l, p.c, k)), fma(m, q.u, l * p.u), fma(m, q.v, l * p.v)};
}
template <class T>
__device__ __forceinline__ Aff<T> shfl_up_aff(const Aff<T>& p, int h) {
    return Aff<T>{__shfl_up_sync(0xffffffffu, p.c, h), __shfl_up_sync(0xffffffffu, p.u, h),
                  __shfl_up_sync(0xffffffffu, p.v, h)};
}
// One symbolic step down a Schur merge node held by `left` lanes (h apart).
template <class T>
__device__ __forceinline__ void schur_step_aff(const SchurSave<T>& sv, bool left, bool right, int h, Aff<T>& xs,
                                               Aff<T>& xe) {
    Aff<T> xt{0, 0, 0}, xt1{0, 0, 0};
    if (left) {
        xt = aff_lin(sv.sd, xs, -sv.sa, xe, sv.sg);
        xt1 = aff_lin(sv.ud, xs, sv.ua, xe, -sv.ug);
    }
    const Aff<T> r1 = shfl_up_aff(xt1, h);
    const Aff<T> re = shfl_up_aff(xe, h);
    if (right) {
        xs = r1;
        xe = re;
    } else if (left) {
        xe = xt;
    }
}

// back_substitute (partition.hpp:163-170) of a chunk, symbolically: every row
// as c + u X0 + v X1 from the chunk's symbolic ends S, E, stored into the
// (a, b, c) slots of the row (x_i = (delta_i - a_i x_{i-1} - gamma_i x_e) / beta_i
// with the up-sweep's values kept in b, c, d).
// row_forms with the chunk length a compile-time constant (3..8 rows).
template <class T, int LEN>
__device__ __forceinline__ void row_forms_fixed(T* a, T* b, T* c, const T* d, int l0, int qs, const Aff<T>& S,
                                                const Aff<T>& E) {
    int q[LEN];
    T ra[LEN], rb[LEN], rc[LEN], rd[LEN];
#pragma unroll
    for (int i = 1; i < LEN - 1; ++i) {
        q[i] = padx(l0 + i, qs);
        ra[i] = a[q[i]];
        rb[i] = b[q[i]];
        rc[i] = c[q[i]];
        rd[i] = d[q[i]];
    }
    T p = 0, qq = 1, r = 0;
#pragma unroll
    for (int i = 1; i < LEN - 1; ++i) {
        const T np = (rd[i] - ra[i] * p) * rb[i];
        const T nq = -ra[i] * qq * rb[i];
        const T nr = (-ra[i] * r - rc[i]) * rb[i];
        p = np;
        qq = nq;
        r = nr;
        const Aff<T> X = aff_lin(p, S, qq, E, r);
        a[q[i]] = X.c;
        b[q[i]] = X.u;
        c[q[i]] = X.v;
    }
    const int k0 = padx(l0, qs), k1 = padx(l0 + LEN - 1, qs);
    a[k0] = S.c; b[k0] = S.u; c[k0] = S.v;
    a[k1] = E.c; b[k1] = E.u; c[k1] = E.v;
}

template <class T>
__device__ __forceinline__ void row_forms(T* a, T* b, T* c, const T* d, int l0, int len, int qs, const Aff<T>& S,
                                          const Aff<T>& E) {
    // x_{i-1} = p + q xs + r xe (chunk-local)
    T p = 0, q = 1, r = 0;
    Row4<T> nx = len > 2 ? ld_row<T>(a, b, c, d, padx(l0 + 1, qs)) : Row4<T>{0, 0, 0, 0};
    for (int i = 1; i < len - 1; ++i) {
        const int k = padx(l0 + i, qs);
        const Row4<T> w = nx;  // a, rcp(beta), gamma, delta
        if (i + 1 < len - 1) nx = ld_row<T>(a, b, c, d, padx(l0 + i + 1, qs));
        const T np = (w.d - w.a * p) * w.b;
        const T nq = -w.a * q * w.b;
        const T nr = (-w.a * r - w.c) * w.b;
        p = np;
        q = nq;
        r = nr;
        // x_i = p + q S + r E
        const Aff<T> X = aff_lin(p, S, q, E, r);
        a[k] = X.c;
        b[k] = X.u;
        c[k] = X.v;
    }
    const int k0 = padx(l0, qs), k1 = padx(l0 + len - 1, qs);
    a[k0] = S.c; b[k0] = S.u; c[k0] = S.v;
    a[k1] = E.c; b[k1] = E.u; c[k1] = E.v;
}

}  // namespace

constexpr int kGridThreads = 512;
constexpr int kGridWarps = kGridThreads / 32;
constexpr int kGridChunksPerThread = 2;
// grid-barrier spin bound (>= 32 ns each): ~0.5-1 s before the solve reports an error
constexpr long kGridSpins = 1L << 24;
// the same bound for a tight spin (each poll an L2 round trip, ~0.3-0.5 us): ~1-2 s
constexpr long kGridSpinsTight = 1L << 22;
// phase timestamps (%globaltimer) of every CTA when a launch asks for them
constexpr int kGridTraceSlots = 16;  // per CTA
__device__ unsigned long long g_grid_trace[2 * 256 * kGridTraceSlots];  // [0, 4096) %globaltimer, then clock64
// (trace builds only: `make TRACE=1`; the stamps' predicated stores and their
// value tests cost ~0.5 us of the C2 solve's serial phases)
#ifdef TPB_GRID_TRACE_BUILD
#define TP_GRID_STAMP(k)                                                                           \
    do {                                                                                           \
        if (tr) {                                                                                  \
            g_grid_trace[kGridTraceSlots * b + (k)] = global_ns();                                 \
            g_grid_trace[256 * kGridTraceSlots + kGridTraceSlots * b + (k)] = clock64();           \
        }                                                                                          \
    } while (0)
#else
#define TP_GRID_STAMP(k) \
    do {                 \
        (void)tr;        \
    } while (0)
#endif

// Block range of CTA b: blocks [K*b/P, K*(b+1)/P) of make_plan(n, m).
struct GridGeom {
    int64_t n, m, K;
    int lg;  // log2(chunks per full block)
    int P;   // CTAs
    int S;   // smem stride of one array, in elements (padded)
    int qs;  // pad shift (one pad element per 2^qs rows)
    int trace;
    int flags;  // kResetErr: the graph's only kernel resets the error word
    int64_t kq;  // K / P and K % P: CTA b's first block K*b/P = kq*b + (kr*b)/P
    int kr;      // with one 32-bit division (kr*b < 2^16), not a 64-bit one
};

// First plan block of CTA b (b = P gives K): floor(K * b / P).
__device__ __forceinline__ int64_t cta_block0(const GridGeom& g, int b) {
    return g.kq * b + (int64_t)((unsigned)(g.kr * b) / (unsigned)g.P);
}

// The grid barrier's counters: bar[0] counts arrivals (P, then P + 1 when
// the sharded root ends are out), bar[1] departures. The last CTA to leave
// resets both, so every launch starts from zero without a reset node.
__device__ __forceinline__ void grid_depart(unsigned* bar, int P) {
    if (atomicAdd(bar + 1, 1u) == (unsigned)P - 1u) {
        bar[0] = 0u;
        bar[1] = 0u;
        __threadfence();
    }
}

// A CTA pair in its 64-byte slot: two 256-bit stores / L2 loads (every CTA
// reads all P slots right after the grid barrier; 4x fewer requests on those
// hot L2 lines than 8-byte accesses). FP32: 8 scalar accesses.
__device__ __forceinline__ void store_cta_pair(double* o, const Eq2<double>& q) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(o), "d"(q.a1), "d"(q.b1), "d"(q.g1), "d"(q.d1)
                 : "memory");
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(o + 4), "d"(q.a2), "d"(q.b2), "d"(q.g2), "d"(q.d2)
                 : "memory");
}
__device__ __forceinline__ Eq2<double> load_cta_pair(const double* q) {
    Eq2<double> r;
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.a1), "=d"(r.b1), "=d"(r.g1), "=d"(r.d1) : "l"(q) : "memory");
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.a2), "=d"(r.b2), "=d"(r.g2), "=d"(r.d2) : "l"(q + 4) : "memory");
    return r;
}
__device__ __forceinline__ void store_cta_pair(float* o, const Eq2<float>& q) {
    o[0] = q.a1; o[1] = q.b1; o[2] = q.g1; o[3] = q.d1;
    o[4] = q.a2; o[5] = q.b2; o[6] = q.g2; o[7] = q.d2;
}
__device__ __forceinline__ Eq2<float> load_cta_pair(const float* q) {
    return Eq2<float>{__ldcg(q + 0), __ldcg(q + 1), __ldcg(q + 2), __ldcg(q + 3),
                      __ldcg(q + 4), __ldcg(q + 5), __ldcg(q + 6), __ldcg(q + 7)};
}

// MODE kSolve: the root pair is the whole system (thomas_solve on [E1; E2]).
// MODE kShard: the root pair is this rank's shard; CTA 0 exchanges it with
// every peer over peer memory (shard_exchange, tp_exchange.cuh), solves the
// 2P-row top system and hands the shard's ends to the other CTAs through a
// second arrival on the barrier counter.
template <class T, int L, int MODE>
__global__ void __launch_bounds__(kGridThreads, 1)
    k_grid_solve(SysPtrs<T> sys, GridGeom geo, T* __restrict__ x, T* pairs, unsigned* bar,
                 unsigned long long* err, int level, const __grid_constant__ ShardLink link) {
    extern __shared__ __align__(16) unsigned char grid_smem[];
    T* sa = reinterpret_cast<T*>(grid_smem);
    T* sb = sa + geo.S;
    T* sc = sb + geo.S;
    T* sd = sc + geo.S;
    __shared__ Eq2<T> wroot[kGridWarps];  // in-CTA warp roots, then the merged values
    __shared__ SchurSave<T> wsv[kGridWarps - 1];  // warp-root merges, [level offset + node]
    __shared__ Eq2<T> troot[8];           // top tree: warp roots (P <= 256)
    __shared__ SchurSave<T> tpath[8];     // top tree: the saves on this CTA's path
    __shared__ int tside[8];              // 0 no merge on the path, 1 left child, 2 right child
    __shared__ Aff<T> wxa[2 * kGridWarps];  // each warp root's ends (W0, W1) as c + u X0 + v X1
    __shared__ T cx[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x, P = geo.P;
    const int64_t n = geo.n, m = geo.m, K = geo.K;
    const int lg = geo.lg, qs = geo.qs;
    const bool tr = geo.trace != 0 && tid == 0;
    bool flag = false;  // a pivot below kPivotFloor (reported with this thread's first row)
    pdl_begin();
    TP_GRID_STAMP(0);

    // ---- this CTA's rows: whole blocks [kb0, kb1) ----
    const int64_t kb0 = cta_block0(geo, b), kb1 = cta_block0(geo, b + 1);
    const int64_t r0 = kb0 * m;
    const int64_t r1 = (kb1 == K) ? n : kb1 * m;
    const int R = (int)(r1 - r0);
    const bool has_tail = (kb1 == K) && (n - (K - 1) * m != m);
    const int nfull = (int)((kb1 - kb0) - (has_tail ? 1 : 0));
    const int tlen = has_tail ? (int)(n - (K - 1) * m) : 0;
    const int g = 1 << lg;
    int lgt = 0;  // log2(chunks of the tail block)
    if (has_tail)
        while ((1 << (lgt + 1)) <= g && tlen >= 4 << lgt) ++lgt;
    const int C = nfull * g + (has_tail ? 1 << lgt : 0);  // chunks of this CTA
    const int NTh = (C + 1) / 2;                           // threads with chunks
    const int mm = (int)m;

    // ---- stage the rows: one cp.async per element into its padded slot ----
    {
        const T* src[4] = {sys.sub + r0, sys.diag + r0, sys.sup + r0, sys.rhs + r0};
        T* dst[4] = {sa, sb, sc, sd};
#pragma unroll
        for (int q = 0; q < 4; ++q)
            for (int i = tid; i < R; i += kGridThreads) cp_async_elem(dst[q] + padx(i, qs), src[q] + i);
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    TP_GRID_STAMP(1);

    // ---- chunk geometry (block-aligned: a full block is 2^lg chunks) ----
    const int lo = mm >> lg, ex = mm & (g - 1);
    const int tlo = tlen >> lgt, tex = tlen & ((1 << lgt) - 1);
    auto cstart = [&](int c) -> int {  // CTA-local first row of chunk c (c <= C)
        if (c >= C) return R;
        const int blk = c >> lg;
        if (blk < nfull) {
            const int q = c & (g - 1);
            return blk * mm + q * lo + (q < ex ? q : ex);
        }
        const int q = c - (nfull << lg);
        return nfull * mm + q * tlo + (q < tex ? q : tex);
    };
    const bool active = tid < NTh;
    int la0 = 0, la = 2, lb0 = 0, lb = 0;
    if (active) {
        la0 = cstart(2 * tid);
        lb0 = cstart(2 * tid + 1);
        la = lb0 - la0;
        lb = (2 * tid + 1 < C) ? cstart(2 * tid + 2) - lb0 : 0;
    }

    // ---- leaves: two chunks per thread, then their merge ----
    Eq2<T> cur = identity_eq<T>();
    SchurSave<T> s0;
    if (active) {
        Eq2<T> EA, EB = identity_eq<T>();
        if (L > 0 && la == L) leaf_fixed<T, (L > 1 ? L : 2)>(sa, sb, sc, sd, la0, qs, flag, EA);
        else leaf_loop<T>(sa, sb, sc, sd, la0, la, qs, flag, EA);
        if (lb > 0) {
            if (L > 0 && lb == L) leaf_fixed<T, (L > 1 ? L : 2)>(sa, sb, sc, sd, lb0, qs, flag, EB);
            else leaf_loop<T>(sa, sb, sc, sd, lb0, lb, qs, flag, EB);
        }
        cur = lb > 0 ? merge_schur(EA, EB, flag, s0) : EA;
    }
    TP_GRID_STAMP(2);

    // ---- thread tree: 5 shuffle levels per warp ----
    SchurSave<T> sw[5];
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
        const int h = 1 << lv;
        const Eq2<T> oth = shfl_down_eq(cur, h);
        if ((lane & (2 * h - 1)) == 0 && tid + h < NTh) cur = merge_schur(cur, oth, flag, sw[lv]);
    }
    const int nwr = (NTh + 31) / 32;
    TP_GRID_STAMP(8);
    if (lane == 0 && warp < nwr) wroot[warp] = cur;
    if (tid < 8) tside[tid] = 0;
    __syncthreads();

    // ---- warp 0: the warp roots (<= 4 levels) -> this CTA's pair, published;
    //      then the warp roots' ends (W0, W1) as c + u X0 + v X1 ----
    if (warp == 0) {
        Eq2<T> wc = lane < nwr ? wroot[lane] : identity_eq<T>();
#pragma unroll
        for (int lv = 0, off = 0; lv < 4; off += kGridWarps >> (lv + 1), ++lv) {
            const int h = 1 << lv;
            const Eq2<T> oth = shfl_down_eq(wc, h);
            if ((lane & (2 * h - 1)) == 0 && lane + h < nwr) {
                SchurSave<T> sv;
                wc = merge_schur(wc, oth, flag, sv);
                wsv[off + (lane >> (lv + 1))] = sv;
            }
        }
        if (lane == 0) {
            store_cta_pair(pairs + 8 * (int64_t)b, wc);
            TP_GRID_STAMP(3);
            // the graph's only kernel: reset the error word before arriving
            // (every report of this solve comes after the barrier)
            if ((geo.flags & kResetErr) && b == 0 && err != nullptr) *reinterpret_cast<volatile unsigned long long*>(err) = kNoError;
            __threadfence();
            atomicAdd(bar, 1u);  // arrive; the wait comes after the symbolic pass
        }
        __syncwarp();
        Aff<T> xs{0, T(lane == 0), 0}, xe{0, 0, T(lane == 0)};
#pragma unroll
        for (int lv = 3; lv >= 0; --lv) {
            const int h = 1 << lv;
            int off = 0;
            for (int j = 0; j < lv; ++j) off += kGridWarps >> (j + 1);
            const bool left = (lane & (2 * h - 1)) == 0 && lane + h < nwr;
            const bool right = (lane & (2 * h - 1)) == h && lane < nwr;
            SchurSave<T> sv{};
            if (left) sv = wsv[off + (lane >> (lv + 1))];
            schur_step_aff(sv, left, right, h, xs, xe);
        }
        if (lane < nwr) {
            wxa[2 * lane] = xs;
            wxa[2 * lane + 1] = xe;
        }
    }

    // ---- every warp (no cross-warp dependency, overlaps warp 0 and the grid
    //      barrier): its tree top-down symbolically from its root's ends
    //      (W0, W1), the in-thread split, then every row of its chunks as
    //      c + u W0 + v W1 in the (a, b, c) slots ----
    {
        Aff<T> xs{0, T(lane == 0), 0}, xe{0, 0, T(lane == 0)};
#pragma unroll
        for (int lv = 4; lv >= 0; --lv) {
            const int h = 1 << lv;
            const bool left = (lane & (2 * h - 1)) == 0 && tid + h < NTh;
            const bool right = (lane & (2 * h - 1)) == h && tid < NTh;
            schur_step_aff(sw[lv], left, right, h, xs, xe);
        }
        if (active) {
            Aff<T> xeA = xe, xsB{0, 0, 0};
            if (lb > 0) {
                xeA = aff_lin(s0.sd, xs, -s0.sa, xe, s0.sg);
                xsB = aff_lin(s0.ud, xs, s0.ua, xe, -s0.ug);
            }
            if (L > 2 && la == L) row_forms_fixed<T, (L > 2 ? L : 3)>(sa, sb, sc, sd, la0, qs, xs, xeA);
            else row_forms<T>(sa, sb, sc, sd, la0, la, qs, xs, xeA);
            if (lb > 0) {
                if (L > 2 && lb == L) row_forms_fixed<T, (L > 2 ? L : 3)>(sa, sb, sc, sd, lb0, qs, xsB, xe);
                else row_forms<T>(sa, sb, sc, sd, lb0, lb, qs, xsB, xe);
            }
        }
    }
    TP_GRID_STAMP(4);

    // ---- the grid barrier: every CTA's pair is published ----
    if (tid == 0) {
        long spins = 0;  // tight spin; departure on warp 15 (as k_grid_hyb)
        while (ld_acquire_gpu(bar) < (unsigned)P) {
            if (++spins > kGridSpinsTight) {
                if (err != nullptr)
                    atomicMin(err, ((unsigned long long)kGridBarrierLevel << 48) | (unsigned long long)b);
                break;
            }
        }
    }
    TP_GRID_STAMP(9);
    __syncthreads();

    // ---- every CTA: the tree over the P CTA pairs (identical arithmetic in
    //      every CTA), keeping only the saves on the path to its own leaf ----
    bool tflag = false;
    {
        const int ntw = (P + 31) / 32;
        if (warp < ntw) {
            Eq2<T> tc = identity_eq<T>();
            if (tid < P) tc = load_cta_pair(pairs + 8 * (int64_t)tid);
            if (tr) { volatile T sink = tc.d2; (void)sink; }
            TP_GRID_STAMP(10);
#pragma unroll
            for (int lv = 0; lv < 5; ++lv) {
                const int h = 1 << lv;
                const Eq2<T> oth = shfl_down_eq(tc, h);
                if ((lane & (2 * h - 1)) == 0 && tid + h < P) {
                    SchurSave<T> sv;
                    tc = merge_schur(tc, oth, tflag, sv);
                    if ((tid >> (lv + 1)) == (b >> (lv + 1))) {  // an ancestor of leaf b
                        tpath[3 + lv] = sv;
                        tside[3 + lv] = ((b >> lv) & 1) ? 2 : 1;
                    }
                }
            }
            if (lane == 0) troot[warp] = tc;
            TP_GRID_STAMP(11);
        }
        if constexpr (MODE != kShard)
            if (tid == kGridThreads - 32) grid_depart(bar, P);  // warp 15: never a top-tree warp (P <= 256)
        __syncthreads();
        if (warp == 0) {
            Eq2<T> rc = lane < ntw ? troot[lane] : identity_eq<T>();
            const int bw = b >> 5;
#pragma unroll
            for (int lv = 0; lv < 3; ++lv) {
                const int h = 1 << lv;
                const Eq2<T> oth = shfl_down_eq(rc, h);
                if ((lane & (2 * h - 1)) == 0 && lane + h < ntw) {
                    SchurSave<T> sv;
                    rc = merge_schur(rc, oth, tflag, sv);
                    if ((lane >> (lv + 1)) == (bw >> (lv + 1))) {
                        tpath[2 - lv] = sv;
                        tside[2 - lv] = ((bw >> lv) & 1) ? 2 : 1;
                    }
                }
            }
            __syncwarp();
            TP_GRID_STAMP(12);
            if (lane == 0) {
                // root (thomas_solve on [E1; E2]), then down the path to leaf b
                T xs = 0, xe = 0;
                if constexpr (MODE == kShard) {
                    T* root = pairs + 8 * 256;  // the shard's (x_s, x_e), CTA 0 -> the others
                    if (b == 0) {
                        __shared__ double top_cm[2 * kMaxPeers], top_x[2 * kMaxPeers];
                        RowGuard top_bad;
                        int missing = -1;
                        if (!shard_exchange(link, rc, top_cm, top_x, xs, xe, top_bad, missing) && err != nullptr)
                            atomicMin(err, ((unsigned long long)kExchangeLevel << 48) | (unsigned long long)missing);
                        report_pivot(err, level + 1, top_bad.bad);
                        root[0] = xs;
                        root[1] = xe;
                        __threadfence();
                        atomicAdd(bar, 1u);
                    } else {
                        long spins = 0;
                        while (ld_acquire_gpu(bar) < (unsigned)P + 1u) {
                            if (++spins > 2 * kExchangeSpins) {
                                if (err != nullptr)
                                    atomicMin(err, ((unsigned long long)kGridBarrierLevel << 48) | (unsigned long long)b);
                                break;
                            }
                            __nanosleep(64);
                        }
                        xs = __ldcg(root);
                        xe = __ldcg(root + 1);
                    }
                    grid_depart(bar, P);
                } else {
                    RowGuard rg;
                    root_solve(rc, n - 1, rg, xs, xe);
                    tflag |= rg.bad != INT64_MAX;
                }
                // path order: warp-root levels 2, 1, 0 (tpath[0..2]), then warp levels 4..0 (tpath[7..3])
                const int order[8] = {0, 1, 2, 7, 6, 5, 4, 3};
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int j = order[k];
                    if (tside[j] == 0) continue;
                    T xt, xt1;
                    schur_down(tpath[j], xs, xe, xt, xt1);
                    if (tside[j] == 1) xe = xt;
                    else xs = xt1;
                }
                cx[0] = xs;
                cx[1] = xe;
                TP_GRID_STAMP(13);
            }
        }
        __syncthreads();
    }
    TP_GRID_STAMP(5);

    // ---- every warp: its root's ends W0, W1, then x = c + u W0 + v W1 over
    //      its rows (lane-strided, coalesced) ----
    bool nf = false;
    if (warp < nwr) {
        const T X0 = cx[0], X1 = cx[1];
        const Aff<T> A0 = wxa[2 * warp], A1 = wxa[2 * warp + 1];
        const T W0 = fma(A0.v, X1, fma(A0.u, X0, A0.c));
        const T W1 = fma(A1.v, X1, fma(A1.u, X0, A1.c));
        const int c0 = 64 * warp;
        const int c1 = c0 + 64 < C ? c0 + 64 : C;
        const int w0 = cstart(c0), w1 = cstart(c1);
        for (int i = w0 + lane; i < w1; i += 32) {
            const int k = padx(i, qs);
            const T v = fma(sc[k], W1, fma(sb[k], W0, sa[k]));
            x[r0 + i] = v;
            nf |= !isfinite(v);
        }
    }
    TP_GRID_STAMP(6);
    if (nf) report_nonfinite(err, r0);
    if (flag) report_pivot(err, level, r0 + la0);
    if (tflag) report_pivot(err, level, r0);
    TP_GRID_STAMP(7);
}

// ===========================================================================
// k_grid_reg: the same solve with the rows in REGISTERS instead of shared
// memory, for full blocks of uniform chunks (L = 2, 4, 5 or 8 rows). Each
// thread loads its two chunks straight from HBM / L2 (256-bit loads where
// aligned), reduces them in registers (leaf_reduce, as k_fast's Stage 1),
// merges them and runs the same thread / warp-root / grid trees; the merge
// saves go to shared memory (one slot per thread and level). After the top
// solve the tree is walked down numerically and every thread re-reads its
// chunks (L2-resident: they were read microseconds earlier), recomputes the
// up-sweep and back-substitutes in registers (as k_fast's Stage 3), storing x
// directly. Shared-memory traffic drops from 17 values per row (staging,
// kept sweep values, row forms) to none; the tail block (make_plan's last
// block, up to m + 1 rows) is staged in shared memory and swept from there.
// ===========================================================================
constexpr int kGregTail = 2 * 256 + 16;  // staged tail rows per array (m + 1 <= 257, x2 for chunk slack)

template <class T, int L>
__device__ __forceinline__ void upsweep_keep(const Chunk<T, L>& r, T (&rbeta)[L], T (&gam)[L], T (&del)[L]) {
    T beta = r.b[L - 2], gamma = r.c[L - 2], delta = r.d[L - 2];
    gam[L - 2] = gamma;
    del[L - 2] = delta;
#pragma unroll
    for (int i = L - 3; i >= 0; --i) {
        const T rb = rcp(beta);
        rbeta[i + 1] = rb;
        const T w = r.c[i] * rb;
        beta = r.b[i] - w * r.a[i + 1];
        gamma = -w * gamma;
        delta = r.d[i] - w * delta;
        gam[i] = gamma;
        del[i] = delta;
    }
}

template <class T, int L, int MODE>
__global__ void __launch_bounds__(kGridThreads, 1)
    k_grid_reg(SysPtrs<T> sys, GridGeom geo, T* __restrict__ x, T* pairs, unsigned* bar,
               unsigned long long* err, int level, const __grid_constant__ ShardLink link, int vec) {
    static_assert(L >= 2 && L <= 8, "register chunks of 2..8 rows");
    extern __shared__ __align__(16) unsigned char greg_smem[];
    SchurSave<T>* ssv = reinterpret_cast<SchurSave<T>*>(greg_smem);  // [6][threads]: tree levels 0..4, in-thread
    T* ta = reinterpret_cast<T*>(ssv + 6 * kGridThreads);            // tail block rows (CTA P-1 only)
    T* tb = ta + kGregTail;
    T* tcc = tb + kGregTail;
    T* td = tcc + kGregTail;
    __shared__ Eq2<T> wroot[kGridWarps];
    __shared__ SchurSave<T> wsv[kGridWarps - 1];
    __shared__ Eq2<T> troot[8];
    __shared__ SchurSave<T> tpath[8];
    __shared__ int tside[8];
    __shared__ T wx[2 * kGridWarps];
    __shared__ T cx[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x, P = geo.P;
    const int64_t n = geo.n, m = geo.m, K = geo.K;
    const int lg = geo.lg;
    const bool tr = geo.trace != 0 && tid == 0;
    pdl_begin();
    TP_GRID_STAMP(0);

    // ---- this CTA's rows: whole blocks [kb0, kb1) (as k_grid_solve) ----
    const int64_t kb0 = cta_block0(geo, b), kb1 = cta_block0(geo, b + 1);
    const int64_t r0 = kb0 * m;
    const int64_t r1 = (kb1 == K) ? n : kb1 * m;
    const int R = (int)(r1 - r0);
    const bool has_tail = (kb1 == K) && (n - (K - 1) * m != m);
    const int nfull = (int)((kb1 - kb0) - (has_tail ? 1 : 0));
    const int tlen = has_tail ? (int)(n - (K - 1) * m) : 0;
    const int g = 1 << lg;
    int lgt = 0;
    if (has_tail)
        while ((1 << (lgt + 1)) <= g && tlen >= 4 << lgt) ++lgt;
    const int C = nfull * g + (has_tail ? 1 << lgt : 0);
    const int NTh = (C + 1) / 2;
    const int mm = (int)m;
    const int tail0 = nfull * mm;  // CTA-local first row of the tail block
    const int tlo = tlen >> lgt, tex = tlen & ((1 << lgt) - 1);
    auto cstart = [&](int c) -> int {
        if (c >= C) return R;
        const int blk = c >> lg;
        if (blk < nfull) return c * L;  // full blocks: uniform chunks of L rows
        const int q = c - (nfull << lg);
        return tail0 + q * tlo + (q < tex ? q : tex);
    };
    if (has_tail) {  // stage the tail block (<= m + 1 rows) for its chunks' sweeps
        for (int i = tid; i < tlen; i += kGridThreads) {
            ta[i] = sys.sub[r0 + tail0 + i];
            tb[i] = sys.diag[r0 + tail0 + i];
            tcc[i] = sys.sup[r0 + tail0 + i];
            td[i] = sys.rhs[r0 + tail0 + i];
        }
    }
    if (tid < 8) tside[tid] = 0;
    __syncthreads();
    TP_GRID_STAMP(1);

    const bool active = tid < NTh;
    int la0 = 0, la = 2, lb0 = 0, lb = 0;
    if (active) {
        la0 = cstart(2 * tid);
        lb0 = cstart(2 * tid + 1);
        la = lb0 - la0;
        lb = (2 * tid + 1 < C) ? cstart(2 * tid + 2) - lb0 : 0;
    }

    // ---- leaves in registers: two chunks per thread, then their merge ----
    MinGuard<T> mg;
    RowGuard tg;  // tail chunks (shared-memory sweeps)
    bool flag = false;
    auto leaf = [&](int l0, int len) -> Eq2<T> {
        if (l0 < tail0 || !has_tail) {
            Chunk<T, L> r;
            const int64_t row0 = r0 + l0;
            if (vec) load_chunk<T, L, true>(sys, row0, true, r);
            else load_chunk<T, L, false>(sys, row0, true, r);
            return leaf_reduce<T, L, L>(r, row0, mg);
        }
        const int o = l0 - tail0;
        return leaf_smem<T, true>(ta + o, tb + o, tcc + o, td + o, len, r0 + l0, tg);
    };
    Eq2<T> cur = identity_eq<T>();
    if (active) {
        const Eq2<T> EA = leaf(la0, la);
        if (lb > 0) {
            const Eq2<T> EB = leaf(lb0, lb);
            SchurSave<T> s0;
            cur = merge_schur(EA, EB, flag, s0);
            ssv[5 * kGridThreads + tid] = s0;
        } else {
            cur = EA;
        }
    }
    TP_GRID_STAMP(2);

    // ---- thread tree (5 shuffle levels), saves to shared memory ----
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
        const int h = 1 << lv;
        const Eq2<T> oth = shfl_down_eq(cur, h);
        if ((lane & (2 * h - 1)) == 0 && tid + h < NTh) {
            SchurSave<T> sv;
            cur = merge_schur(cur, oth, flag, sv);
            ssv[lv * kGridThreads + tid] = sv;
        }
    }
    const int nwr = (NTh + 31) / 32;
    TP_GRID_STAMP(8);
    if (lane == 0 && warp < nwr) wroot[warp] = cur;
    __syncthreads();

    // ---- warp 0: the warp roots -> this CTA's pair, published ----
    if (warp == 0) {
        Eq2<T> wc = lane < nwr ? wroot[lane] : identity_eq<T>();
#pragma unroll
        for (int lv = 0, off = 0; lv < 4; off += kGridWarps >> (lv + 1), ++lv) {
            const int h = 1 << lv;
            const Eq2<T> oth = shfl_down_eq(wc, h);
            if ((lane & (2 * h - 1)) == 0 && lane + h < nwr) {
                SchurSave<T> sv;
                wc = merge_schur(wc, oth, flag, sv);
                wsv[off + (lane >> (lv + 1))] = sv;
            }
        }
        if (lane == 0) {
            store_cta_pair(pairs + 8 * (int64_t)b, wc);
            TP_GRID_STAMP(3);
            if ((geo.flags & kResetErr) && b == 0 && err != nullptr) *reinterpret_cast<volatile unsigned long long*>(err) = kNoError;
            __threadfence();
            atomicAdd(bar, 1u);
            long spins = 0;  // tight spin; departure on warp 15 (as k_grid_hyb)
            while (ld_acquire_gpu(bar) < (unsigned)P) {
                if (++spins > kGridSpinsTight) {
                    if (err != nullptr)
                        atomicMin(err, ((unsigned long long)kGridBarrierLevel << 48) | (unsigned long long)b);
                    break;
                }
            }
            TP_GRID_STAMP(9);
        }
    }
    __syncthreads();

    // ---- every CTA: the tree over the P CTA pairs, root, its own path (as k_grid_solve) ----
    bool tflag = false;
    {
        const int ntw = (P + 31) / 32;
        if (warp < ntw) {
            Eq2<T> tc = identity_eq<T>();
            if (tid < P) tc = load_cta_pair(pairs + 8 * (int64_t)tid);
#pragma unroll
            for (int lv = 0; lv < 5; ++lv) {
                const int h = 1 << lv;
                const Eq2<T> oth = shfl_down_eq(tc, h);
                if ((lane & (2 * h - 1)) == 0 && tid + h < P) {
                    SchurSave<T> sv;
                    tc = merge_schur(tc, oth, tflag, sv);
                    if ((tid >> (lv + 1)) == (b >> (lv + 1))) {
                        tpath[3 + lv] = sv;
                        tside[3 + lv] = ((b >> lv) & 1) ? 2 : 1;
                    }
                }
            }
            if (lane == 0) troot[warp] = tc;
        }
        if constexpr (MODE != kShard)
            if (tid == kGridThreads - 32) grid_depart(bar, P);  // warp 15: never a top-tree warp (P <= 256)
        __syncthreads();
        if (warp == 0) {
            Eq2<T> rc = lane < ntw ? troot[lane] : identity_eq<T>();
            const int bw = b >> 5;
#pragma unroll
            for (int lv = 0; lv < 3; ++lv) {
                const int h = 1 << lv;
                const Eq2<T> oth = shfl_down_eq(rc, h);
                if ((lane & (2 * h - 1)) == 0 && lane + h < ntw) {
                    SchurSave<T> sv;
                    rc = merge_schur(rc, oth, tflag, sv);
                    if ((lane >> (lv + 1)) == (bw >> (lv + 1))) {
                        tpath[2 - lv] = sv;
                        tside[2 - lv] = ((bw >> lv) & 1) ? 2 : 1;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                T xs = 0, xe = 0;
                if constexpr (MODE == kShard) {
                    T* root = pairs + 8 * 256;
                    if (b == 0) {
                        __shared__ double top_cm[2 * kMaxPeers], top_x[2 * kMaxPeers];
                        RowGuard top_bad;
                        int missing = -1;
                        if (!shard_exchange(link, rc, top_cm, top_x, xs, xe, top_bad, missing) && err != nullptr)
                            atomicMin(err, ((unsigned long long)kExchangeLevel << 48) | (unsigned long long)missing);
                        report_pivot(err, level + 1, top_bad.bad);
                        root[0] = xs;
                        root[1] = xe;
                        __threadfence();
                        atomicAdd(bar, 1u);
                    } else {
                        long spins = 0;
                        while (ld_acquire_gpu(bar) < (unsigned)P + 1u) {
                            if (++spins > 2 * kExchangeSpins) {
                                if (err != nullptr)
                                    atomicMin(err, ((unsigned long long)kGridBarrierLevel << 48) | (unsigned long long)b);
                                break;
                            }
                            __nanosleep(64);
                        }
                        xs = __ldcg(root);
                        xe = __ldcg(root + 1);
                    }
                    grid_depart(bar, P);
                } else {
                    RowGuard rg;
                    root_solve(rc, n - 1, rg, xs, xe);
                    tflag |= rg.bad != INT64_MAX;
                }
#pragma unroll 1
                for (int k = 0; k < 8; ++k) {
                    const int j = k < 3 ? k : 10 - k;  // warp-root levels 2, 1, 0, then warp levels 4..0
                    if (tside[j] == 0) continue;
                    T xt, xt1;
                    schur_down(tpath[j], xs, xe, xt, xt1);
                    if (tside[j] == 1) xe = xt;
                    else xs = xt1;
                }
                cx[0] = xs;
                cx[1] = xe;
            }
        }
        __syncthreads();
    }
    TP_GRID_STAMP(5);

    // ---- the CTA's tree top-down, numerically: warp roots, then every warp ----
    if (warp == 0) {
        T xs = lane == 0 ? cx[0] : T(0), xe = lane == 0 ? cx[1] : T(0);
#pragma unroll
        for (int lv = 3; lv >= 0; --lv) {
            const int h = 1 << lv;
            int off = 0;
            for (int j = 0; j < lv; ++j) off += kGridWarps >> (j + 1);
            const bool left = (lane & (2 * h - 1)) == 0 && lane + h < nwr;
            const bool right = (lane & (2 * h - 1)) == h && lane < nwr;
            T xt = 0, xt1 = 0;
            if (left) schur_down(wsv[off + (lane >> (lv + 1))], xs, xe, xt, xt1);
            const T r1 = __shfl_up_sync(0xffffffffu, xt1, h);
            const T re = __shfl_up_sync(0xffffffffu, xe, h);
            if (right) {
                xs = r1;
                xe = re;
            } else if (left) {
                xe = xt;
            }
        }
        if (lane < nwr) {
            wx[2 * lane] = xs;
            wx[2 * lane + 1] = xe;
        }
    }
    __syncthreads();
    bool nf = false;
    {
        T xs = 0, xe = 0;
        if (lane == 0 && warp < nwr) {
            xs = wx[2 * warp];
            xe = wx[2 * warp + 1];
        }
#pragma unroll
        for (int lv = 4; lv >= 0; --lv) {
            const int h = 1 << lv;
            const bool left = (lane & (2 * h - 1)) == 0 && tid + h < NTh;
            const bool right = (lane & (2 * h - 1)) == h && tid < NTh;
            T xt = 0, xt1 = 0;
            if (left) schur_down(ssv[lv * kGridThreads + tid], xs, xe, xt, xt1);
            const T r1 = __shfl_up_sync(0xffffffffu, xt1, h);
            const T re = __shfl_up_sync(0xffffffffu, xe, h);
            if (right) {
                xs = r1;
                xe = re;
            } else if (left) {
                xe = xt;
            }
        }
        TP_GRID_STAMP(6);
        // ---- Stage 3 of the chunks: re-read (L2), up-sweep, back_substitute, store ----
        auto expand = [&](int l0, int len, T cs, T ce) {
            if (l0 < tail0 || !has_tail) {
                Chunk<T, L> r;
                const int64_t row0 = r0 + l0;
                if (vec) load_chunk<T, L, true>(sys, row0, true, r);
                else load_chunk<T, L, false>(sys, row0, true, r);
                T rbeta[L], gam[L], del[L], xv[L];
                upsweep_keep<T, L>(r, rbeta, gam, del);
                leaf_expand<T, L, L>(r, rbeta, gam, del, cs, ce, xv);
                if (vec) store_rows<T, L, true>(x, row0, xv);
                else store_rows<T, L, false>(x, row0, xv);
                nf |= any_nonfinite(xv);
                return;
            }
            const int o = l0 - tail0;  // tail chunk: kept sweep values in shared memory
            T prev = cs;
            x[r0 + l0] = cs;
            for (int i = 1; i < len - 1; ++i) {
                prev = (td[o + i] - ta[o + i] * prev - tcc[o + i] * ce) * tb[o + i];
                x[r0 + l0 + i] = prev;
                nf |= !isfinite(prev);
            }
            x[r0 + l0 + len - 1] = ce;
            nf |= !isfinite(cs) || !isfinite(ce);
        };
        if (active) {
            if (lb > 0) {
                T xt, xt1;
                schur_down(ssv[5 * kGridThreads + tid], xs, xe, xt, xt1);
                expand(la0, la, xs, xt);
                expand(lb0, lb, xt1, xe);
            } else {
                expand(la0, la, xs, xe);
            }
        }
    }
    TP_GRID_STAMP(7);
    if (nf) report_nonfinite(err, r0);
    if (mg.tripped() || flag) report_pivot(err, level, r0 + la0);
    report_pivot(err, level, tg.bad);
    if (tflag) report_pivot(err, level, r0);
}

// ===========================================================================
// k_grid_hyb: rows loaded into registers (256-bit) and swept from there, as
// k_grid_reg; each interior row keeps p = delta/beta, q = a/beta, r =
// gamma/beta in the padded shared-memory layout of k_grid_solve, so Stage 3 is
// one FMA chain per chunk from shared memory instead of an L2 re-read; the
// merge saves stay in registers (as k_grid_solve). Shared-memory traffic: 6
// values per interior row (k_grid_solve: 17), no L2 re-read (k_grid_reg).
// ===========================================================================
template <class T, int L, int MODE>
__global__ void __launch_bounds__(kGridThreads, 1)
    k_grid_hyb(SysPtrs<T> sys, GridGeom geo, T* __restrict__ x, T* pairs, unsigned* bar,
               unsigned long long* err, int level, const __grid_constant__ ShardLink link, int vec) {
    static_assert(L >= 2 && L <= 8, "register chunks of 2..8 rows");
    extern __shared__ __align__(16) unsigned char ghyb_smem[];
    T* sa = reinterpret_cast<T*>(ghyb_smem);  // the CTA's rows, padded (as k_grid_solve)
    T* sb = sa + geo.S;
    T* sc = sb + geo.S;
    T* sd = sc + geo.S;
    const int qs = geo.qs;
    __shared__ Eq2<T> wroot[kGridWarps];
    __shared__ SchurSave<T> wsv[kGridWarps - 1];
    __shared__ Eq2<T> troot[8];
    __shared__ SchurSave<T> tpath[8];
    __shared__ int tside[8];
    __shared__ T wx[2 * kGridWarps];
    __shared__ T cx[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x, P = geo.P;
    const int64_t n = geo.n, m = geo.m, K = geo.K;
    const int lg = geo.lg;
    const bool tr = geo.trace != 0 && tid == 0;
    pdl_begin();
    TP_GRID_STAMP(0);

    // ---- this CTA's rows: whole blocks [kb0, kb1) (as k_grid_solve) ----
    const int64_t kb0 = cta_block0(geo, b), kb1 = cta_block0(geo, b + 1);
    const int64_t r0 = kb0 * m;
    const int64_t r1 = (kb1 == K) ? n : kb1 * m;
    const int R = (int)(r1 - r0);
    const bool has_tail = (kb1 == K) && (n - (K - 1) * m != m);
    const int nfull = (int)((kb1 - kb0) - (has_tail ? 1 : 0));
    const int tlen = has_tail ? (int)(n - (K - 1) * m) : 0;
    const int g = 1 << lg;
    int lgt = 0;
    if (has_tail)
        while ((1 << (lgt + 1)) <= g && tlen >= 4 << lgt) ++lgt;
    const int C = nfull * g + (has_tail ? 1 << lgt : 0);
    const int NTh = (C + 1) / 2;
    const int mm = (int)m;
    const int tail0 = nfull * mm;  // CTA-local first row of the tail block
    const int tlo = tlen >> lgt, tex = tlen & ((1 << lgt) - 1);
    auto cstart = [&](int c) -> int {
        if (c >= C) return R;
        const int blk = c >> lg;
        if (blk < nfull) return c * L;  // full blocks: uniform chunks of L rows
        const int q = c - (nfull << lg);
        return tail0 + q * tlo + (q < tex ? q : tex);
    };
    if (has_tail) {  // stage the tail block (<= m + 1 rows) for its chunks' shared-memory sweeps
        for (int i = tid; i < tlen; i += kGridThreads) {
            const int k = padx(tail0 + i, qs);
            sa[k] = sys.sub[r0 + tail0 + i];
            sb[k] = sys.diag[r0 + tail0 + i];
            sc[k] = sys.sup[r0 + tail0 + i];
            sd[k] = sys.rhs[r0 + tail0 + i];
        }
    }
    if (tid < 8) tside[tid] = 0;
    __syncthreads();
    TP_GRID_STAMP(1);

    const bool active = tid < NTh;
    int la0 = 0, la = 2, lb0 = 0, lb = 0;
    if (active) {
        la0 = cstart(2 * tid);
        lb0 = cstart(2 * tid + 1);
        la = lb0 - la0;
        lb = (2 * tid + 1 < C) ? cstart(2 * tid + 2) - lb0 : 0;
    }

    // ---- leaves in registers: two chunks per thread, then their merge ----
    MinGuard<T> mg;
    bool flag = false;
    // full chunks: rows loaded into registers (256-bit), copied to shared
    // memory for Stage 3, swept from the registers; tail chunks: swept from
    // shared memory (kept values in place)
    auto leaf = [&](int l0, int len) -> Eq2<T> {
        if (l0 < tail0 || !has_tail) {
            Chunk<T, L> r;
            const int64_t row0 = r0 + l0;
            if (vec) load_chunk<T, L, true>(sys, row0, true, r);
            else load_chunk<T, L, false>(sys, row0, true, r);
            // sweep with the up-sweep's values kept (rcp(beta_i), gamma_i,
            // delta_i); back_substitute (partition.hpp:163-170) of interior
            // row i is x_i = (delta_i - a_i x_{i-1} - gamma_i x_e) / beta_i =
            // p_i - q_i x_{i-1} - r_i x_e, so the interior rows keep
            // p = delta/beta, q = a/beta, r = gamma/beta (3 shared-memory
            // values per row, and one dependent FMA per row in Stage 3)
            T rbeta[L] = {}, gam[L] = {}, del[L] = {};
            const Eq2<T> e = leaf_reduce_keep<T, L, L>(r, row0, mg, rbeta, gam, del);
#pragma unroll
            for (int i = 1; i < L - 1; ++i) {
                const int k = padx(l0 + i, qs);
                sa[k] = r.a[i] * rbeta[i];
                sb[k] = del[i] * rbeta[i];
                sc[k] = gam[i] * rbeta[i];
            }
            return e;
        }
        Eq2<T> e;
        leaf_loop<T>(sa, sb, sc, sd, l0, len, qs, flag, e);
        return e;
    };
    Eq2<T> cur = identity_eq<T>();
    SchurSave<T> s0{};
    if (active) {
        const Eq2<T> EA = leaf(la0, la);
        if (lb > 0) {
            const Eq2<T> EB = leaf(lb0, lb);
            cur = merge_schur(EA, EB, flag, s0);
        } else {
            cur = EA;
        }
    }
    TP_GRID_STAMP(2);

    // ---- thread tree (5 shuffle levels), saves in registers ----
    SchurSave<T> sw[5] = {};  // read (unused) by the non-merging lanes going down
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
        const int h = 1 << lv;
        const Eq2<T> oth = shfl_down_eq(cur, h);
        if ((lane & (2 * h - 1)) == 0 && tid + h < NTh) cur = merge_schur(cur, oth, flag, sw[lv]);
    }
    const int nwr = (NTh + 31) / 32;
    TP_GRID_STAMP(8);
    if (lane == 0 && warp < nwr) wroot[warp] = cur;
    __syncthreads();

    // ---- warp 0: the warp roots -> this CTA's pair, published ----
    if (warp == 0) {
        Eq2<T> wc = lane < nwr ? wroot[lane] : identity_eq<T>();
#pragma unroll
        for (int lv = 0, off = 0; lv < 4; off += kGridWarps >> (lv + 1), ++lv) {
            const int h = 1 << lv;
            const Eq2<T> oth = shfl_down_eq(wc, h);
            if ((lane & (2 * h - 1)) == 0 && lane + h < nwr) {
                SchurSave<T> sv;
                wc = merge_schur(wc, oth, flag, sv);
                wsv[off + (lane >> (lv + 1))] = sv;
            }
        }
        if (lane == 0) {
            store_cta_pair(pairs + 8 * (int64_t)b, wc);
            TP_GRID_STAMP(3);
            if ((geo.flags & kResetErr) && b == 0 && err != nullptr) *reinterpret_cast<volatile unsigned long long*>(err) = kNoError;
            // tight spin (a __nanosleep between polls measured 0.4-0.5 us
            // slower at C2; a release-add with relaxed polls slower still)
            __threadfence();
            atomicAdd(bar, 1u);
            long spins = 0;
            while (ld_acquire_gpu(bar) < (unsigned)P) {
                if (++spins > kGridSpinsTight) {
                    if (err != nullptr)
                        atomicMin(err, ((unsigned long long)kGridBarrierLevel << 48) | (unsigned long long)b);
                    break;
                }
            }
            // no departure here: its atomic returns a value, and the wait for
            // it would hold the CTA's next __syncthreads (an idle warp departs
            // during the top tree instead)
            TP_GRID_STAMP(9);
        }
    }
    __syncthreads();

    // ---- every CTA: the tree over the P CTA pairs, root, its own path (as k_grid_solve) ----
    bool tflag = false;
    {
        const int ntw = (P + 31) / 32;
        if (warp < ntw) {
            const int ptid = pin_reg(tid), pb = pin_reg(b);
            Eq2<T> tc = identity_eq<T>();
            if (ptid < P) tc = load_cta_pair(pairs + 8 * (int64_t)ptid);
            if (tr && tc.b1 != T(-1.2345e-300)) TP_GRID_STAMP(10);
            // unrolled (0.15 us faster than one rolled copy of the level once
            // the pair loads stopped contending; a dry pass by an idle warp to
            // warm the instruction cache, through a non-inlined copy, measured
            // 0.7 us slower)
#pragma unroll
            for (int lv = 0; lv < 5; ++lv) {
                const int h = 1 << lv;
                const Eq2<T> oth = shfl_down_eq(tc, h);
                // every lane merges (straight-line code); the tree's lanes keep it
                SchurSave<T> sv;
                bool f = false;
                const Eq2<T> pm = merge_schur(tc, oth, f, sv);
                if ((ptid & (2 * h - 1)) == 0 && ptid + h < P) {
                    tc = pm;
                    tflag |= f;
                    if ((ptid >> (lv + 1)) == (pb >> (lv + 1))) {
                        tpath[3 + lv] = sv;
                        tside[3 + lv] = ((pb >> lv) & 1) ? 2 : 1;
                    }
                }
            }
            if (lane == 0) troot[warp] = tc;
            TP_GRID_STAMP(11);
        }
        if constexpr (MODE != kShard)
            if (tid == kGridThreads - 32) grid_depart(bar, P);  // warp 15: never a top-tree warp (P <= 256)
        __syncthreads();
        if (warp == 0) {
            Eq2<T> rc = lane < ntw ? troot[lane] : identity_eq<T>();
            const int bw = pin_reg(b >> 5), plane = pin_reg(lane);
#pragma unroll
            for (int lv = 0; lv < 3; ++lv) {
                const int h = 1 << lv;
                const Eq2<T> oth = shfl_down_eq(rc, h);
                SchurSave<T> sv;
                bool f = false;
                const Eq2<T> pm = merge_schur(rc, oth, f, sv);
                if ((plane & (2 * h - 1)) == 0 && plane + h < ntw) {
                    rc = pm;
                    tflag |= f;
                    if ((plane >> (lv + 1)) == (bw >> (lv + 1))) {
                        tpath[2 - lv] = sv;
                        tside[2 - lv] = ((bw >> lv) & 1) ? 2 : 1;
                    }
                }
            }
            __syncwarp();
            TP_GRID_STAMP(12);
            if (lane == 0) {
                T xs = 0, xe = 0;
                if constexpr (MODE == kShard) {
                    T* root = pairs + 8 * 256;
                    if (b == 0) {
                        __shared__ double top_cm[2 * kMaxPeers], top_x[2 * kMaxPeers];
                        RowGuard top_bad;
                        int missing = -1;
                        if (!shard_exchange(link, rc, top_cm, top_x, xs, xe, top_bad, missing) && err != nullptr)
                            atomicMin(err, ((unsigned long long)kExchangeLevel << 48) | (unsigned long long)missing);
                        report_pivot(err, level + 1, top_bad.bad);
                        root[0] = xs;
                        root[1] = xe;
                        __threadfence();
                        atomicAdd(bar, 1u);
                    } else {
                        long spins = 0;
                        while (ld_acquire_gpu(bar) < (unsigned)P + 1u) {
                            if (++spins > 2 * kExchangeSpins) {
                                if (err != nullptr)
                                    atomicMin(err, ((unsigned long long)kGridBarrierLevel << 48) | (unsigned long long)b);
                                break;
                            }
                            __nanosleep(64);
                        }
                        xs = __ldcg(root);
                        xe = __ldcg(root + 1);
                    }
                    grid_depart(bar, P);
                } else {
                    RowGuard rg;
                    root_solve(rc, n - 1, rg, xs, xe);
                    tflag |= rg.bad != INT64_MAX;
                }
#pragma unroll 1
                for (int k = 0; k < 8; ++k) {
                    const int j = k < 3 ? k : 10 - k;  // warp-root levels 2, 1, 0, then warp levels 4..0
                    if (tside[j] == 0) continue;
                    T xt, xt1;
                    schur_down(tpath[j], xs, xe, xt, xt1);
                    if (tside[j] == 1) xe = xt;
                    else xs = xt1;
                }
                cx[0] = xs;
                cx[1] = xe;
                TP_GRID_STAMP(13);
            }
        }
        __syncthreads();
    }
    TP_GRID_STAMP(5);

    // ---- the CTA's tree top-down, numerically: warp roots, then every warp ----
    if (warp == 0) {
        T xs = lane == 0 ? cx[0] : T(0), xe = lane == 0 ? cx[1] : T(0);
#pragma unroll
        for (int lv = 3; lv >= 0; --lv) {
            const int h = 1 << lv;
            int off = 0;
            for (int j = 0; j < lv; ++j) off += kGridWarps >> (j + 1);
            const bool left = (lane & (2 * h - 1)) == 0 && lane + h < nwr;
            const bool right = (lane & (2 * h - 1)) == h && lane < nwr;
            T xt, xt1;
            schur_down(wsv[left ? off + (lane >> (lv + 1)) : 0], xs, xe, xt, xt1);
            const T r1 = __shfl_up_sync(0xffffffffu, xt1, h);
            const T re = __shfl_up_sync(0xffffffffu, xe, h);
            if (right) {
                xs = r1;
                xe = re;
            } else if (left) {
                xe = xt;
            }
        }
        if (lane < nwr) {
            wx[2 * lane] = xs;
            wx[2 * lane + 1] = xe;
        }
        TP_GRID_STAMP(4);
    }
    __syncthreads();
    TP_GRID_STAMP(14);
    bool nf = false;
    {
        T xs = 0, xe = 0;
        if (lane == 0 && warp < nwr) {
            xs = wx[2 * warp];
            xe = wx[2 * warp + 1];
        }
#pragma unroll
        for (int lv = 4; lv >= 0; --lv) {
            const int h = 1 << lv;
            const bool left = (lane & (2 * h - 1)) == 0 && tid + h < NTh;
            const bool right = (lane & (2 * h - 1)) == h && tid < NTh;
            T xt, xt1;
            schur_down(sw[lv], xs, xe, xt, xt1);
            const T r1 = __shfl_up_sync(0xffffffffu, xt1, h);
            const T re = __shfl_up_sync(0xffffffffu, xe, h);
            if (right) {
                xs = r1;
                xe = re;
            } else if (left) {
                xe = xt;
            }
        }
        TP_GRID_STAMP(6);
        // ---- Stage 3 of the chunks: rows from shared memory, up-sweep, back_substitute, store ----
        auto expand = [&](int l0, int len, T cs, T ce) {
            if (l0 < tail0 || !has_tail) {
                const int64_t row0 = r0 + l0;
                T q[L], pv[L], rv[L], xv[L];
#pragma unroll
                for (int i = 1; i < L - 1; ++i) {
                    const int k = padx(l0 + i, qs);
                    q[i] = sa[k];
                    pv[i] = sb[k];
                    rv[i] = sc[k];
                }
                if (tr && q[1] != T(-1.2345e-300)) TP_GRID_STAMP(15);
                xv[0] = cs;
                T prev = cs;
#pragma unroll
                for (int i = 1; i < L - 1; ++i) {
                    prev = fma(-q[i], prev, fma(-rv[i], ce, pv[i]));
                    xv[i] = prev;
                }
                xv[L - 1] = ce;
                if (vec) store_rows<T, L, true>(x, row0, xv);
                else store_rows<T, L, false>(x, row0, xv);
                nf |= any_nonfinite(xv);
                return;
            }
            T prev = cs;  // tail chunk: kept sweep values in shared memory
            x[r0 + l0] = cs;
            for (int i = 1; i < len - 1; ++i) {
                const int k = padx(l0 + i, qs);
                prev = (sd[k] - sa[k] * prev - sc[k] * ce) * sb[k];
                x[r0 + l0 + i] = prev;
                nf |= !isfinite(prev);
            }
            x[r0 + l0 + len - 1] = ce;
            nf |= !isfinite(cs) || !isfinite(ce);
        };
        if (active) {
            // the two chunks through ONE copy of the expand code (its second
            // pass runs from a warm instruction cache)
            T xt = xe, xt1 = T(0);
            if (lb > 0) schur_down(s0, xs, xe, xt, xt1);
            const int nch = lb > 0 ? 2 : 1;
#pragma unroll 1
            for (int c = 0; c < nch; ++c) expand(c ? lb0 : la0, c ? lb : la, c ? xt1 : xs, c ? xe : xt);
        }
    }
    TP_GRID_STAMP(7);
    if (nf) report_nonfinite(err, r0);
    if (mg.tripped() || flag) report_pivot(err, level, r0 + la0);
    if (tflag) report_pivot(err, level, r0);
}

// ---------------------------------------------------------------- host side

static size_t grid_smem_bytes(int64_t S, size_t elem) { return (size_t)4 * S * elem; }

// Geometry for (n, m) on `sms` SMs, or false when the system does not fit.
template <class T>
static bool grid_geom(int64_t n, int64_t m, int sms, GridGeom& geo) {
    if (m < 2 || n < kGridMinRows) return false;
    const int64_t K = plan_blocks_dev(n, m);
    const int64_t me = m < n ? m : n;  // longest full block
    int P = sms;
    if (K < P) P = (int)K;
    if (P > 256) P = 256;
    const int64_t bpc = (K + P - 1) / P;  // blocks of the largest CTA
    const int64_t cmax = (int64_t)kGridThreads * kGridChunksPerThread;
    if (bpc > cmax) return false;
    int lg = 0;
    while (bpc * (2 << lg) <= cmax && me >= (4 << lg)) ++lg;
    const int64_t lmax = (me + 1 + (1 << lg) - 1) >> lg;  // longest chunk (a tail block has up to m+1 rows)
    if (lmax > kGridMaxChunk) return false;
    int qs = 5;
    while ((1 << qs) < lmax) ++qs;
    const int64_t rows = bpc * m + 1;  // rows of the largest CTA
    const int64_t S = ((rows + (rows >> qs) + 1 + 3) / 4) * 4;
    if (grid_smem_bytes(S, sizeof(T)) > kGridDynSmem) return false;
    static const int trace = [] { const char* v = getenv("TPB_GRID_TRACE"); return v ? atoi(v) : 0; }();
    geo = GridGeom{n, m, K, lg, P, (int)S, qs, trace, 0, K / P, (int)(K % P)};
    return true;
}

bool grid_fits(int64_t n, int64_t m, size_t elem, int sms) {
    GridGeom geo;
    return elem == 8 ? grid_geom<double>(n, m, sms, geo) : grid_geom<float>(n, m, sms, geo);
}

template <class T, int MODE>
using GridKernel = void (*)(SysPtrs<T>, GridGeom, T*, T*, unsigned*, unsigned long long*, int, const ShardLink);
template <class T, int MODE>
using GregKernel = void (*)(SysPtrs<T>, GridGeom, T*, T*, unsigned*, unsigned long long*, int, const ShardLink, int);

template <class T, int MODE>
static GridKernel<T, MODE> grid_kernel(int L) {
    return L == 8 ? k_grid_solve<T, 8, MODE> : L == 5 ? k_grid_solve<T, 5, MODE> : L == 4 ? k_grid_solve<T, 4, MODE>
           : L == 2 ? k_grid_solve<T, 2, MODE> : k_grid_solve<T, 0, MODE>;
}
template <class T, int MODE>
static GregKernel<T, MODE> greg_kernel(int L) {
    return L == 8 ? k_grid_reg<T, 8, MODE> : L == 5 ? k_grid_reg<T, 5, MODE> : L == 4 ? k_grid_reg<T, 4, MODE>
           : L == 2 ? k_grid_reg<T, 2, MODE> : nullptr;
}
template <class T, int MODE>
static GregKernel<T, MODE> ghyb_kernel(int L) {
    return L == 8 ? k_grid_hyb<T, 8, MODE> : L == 5 ? k_grid_hyb<T, 5, MODE> : L == 4 ? k_grid_hyb<T, 4, MODE>
           : L == 2 ? k_grid_hyb<T, 2, MODE> : nullptr;
}
static int g_ghyb = -1;  // hybrid variant (TPB_GRID_HYB=0 turns it off)
static size_t greg_smem_bytes(size_t elem) {
    return (size_t)6 * kGridThreads * 6 * elem + (size_t)4 * kGregTail * elem;
}
static int g_greg = -1;  // register variant (TPB_GRID_REG=0 turns it off)

template <class T>
cudaError_t launch_grid_solve(const SysPtrs<T>& sys, int64_t n, int64_t m, T* x, void* scratch,
                              unsigned long long* err, int level, int sms, cudaStream_t st, int mode,
                              const ShardLink* link, int flags) {
    GridGeom geo;
    if (!grid_geom<T>(n, m, sms, geo)) return cudaErrorInvalidValue;
    geo.flags = flags;
    // test hook of the host's level-path fallback (TPB_GRID_FORCE_FAIL=1)
    static const bool force_fail = [] { const char* v = getenv("TPB_GRID_FORCE_FAIL"); return v && atoi(v) != 0; }();
    if (force_fail) return cudaErrorCooperativeLaunchTooLarge;
    if (mode == kShard && (sizeof(T) != 8 || link == nullptr || link->nranks < 1 || link->nranks > kMaxPeers))
        return cudaErrorInvalidValue;  // the mailboxes carry FP64 pairs
    unsigned* bar = static_cast<unsigned*>(scratch);
    T* pairs = reinterpret_cast<T*>(static_cast<unsigned char*>(scratch) + 256);
    // chunk length as a compile-time constant when every full block splits
    // into equal chunks of 2, 4, 5 or 8 rows (unrolled register sweeps; 5:
    // the m = 10 / 20 / 40 levels of the kNN policies)
    const int64_t cl = geo.m >> geo.lg;
    const int L = ((cl << geo.lg) == geo.m && (cl == 2 || cl == 4 || cl == 5 || cl == 8)) ? (int)cl : 0;
    if (g_greg < 0) {
        const char* v = getenv("TPB_GRID_REG");
        g_greg = (v != nullptr && atoi(v) == 0) ? 0 : 1;
    }
    static bool attr_done[2] = {false, false};
    if (!attr_done[sizeof(T) == 8]) {
        for (int l : {8, 5, 4, 2, 0}) {
            cudaError_t e = cudaFuncSetAttribute(grid_kernel<T, kSolve>(l), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)kGridDynSmem);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(grid_kernel<T, kShard>(l), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kGridDynSmem);
            if (e == cudaSuccess && greg_kernel<T, kSolve>(l) != nullptr)
                e = cudaFuncSetAttribute(greg_kernel<T, kSolve>(l), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)greg_smem_bytes(sizeof(T)));
            if (e == cudaSuccess && greg_kernel<T, kShard>(l) != nullptr)
                e = cudaFuncSetAttribute(greg_kernel<T, kShard>(l), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)greg_smem_bytes(sizeof(T)));
            if (e == cudaSuccess && ghyb_kernel<T, kSolve>(l) != nullptr)
                e = cudaFuncSetAttribute(ghyb_kernel<T, kSolve>(l), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kGridDynSmem);
            if (e == cudaSuccess && ghyb_kernel<T, kShard>(l) != nullptr)
                e = cudaFuncSetAttribute(ghyb_kernel<T, kShard>(l), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kGridDynSmem);
            if (e != cudaSuccess) return e;
        }
        attr_done[sizeof(T) == 8] = true;
    }
    // the grid barrier needs every CTA resident: a cooperative launch
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)geo.P);
    cfg.blockDim = dim3(kGridThreads);
    cfg.dynamicSmemBytes = grid_smem_bytes(geo.S, sizeof(T));
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const ShardLink none{};
    const ShardLink& lk = (mode == kShard) ? *link : none;
    // rows in registers (k_grid_reg) where that measured faster: chunks of
    // 2, 4 or 8 rows (5-row chunks: 18.8 vs 15.8 us at 6e5 {20}) and <= ~5K
    // rows per SM (its L2 re-read of the rows costs more than the shared-
    // memory staging above that: 1e6 {32} 20.5 vs 20.0 us, 6e5 {32} 14.6 vs
    // 15.6 us, 1e5 {32} 10.9 vs 11.8 us, C3's level 2 17.9 vs 18.4 us;
    // tools/ab_grid_reg.sh)
    const int64_t rows_cta = ((geo.K + geo.P - 1) / geo.P) * geo.m;
    if (g_ghyb < 0) {
        const char* v = getenv("TPB_GRID_HYB");
        g_ghyb = (v != nullptr && atoi(v) == 0) ? 0 : 1;
    }
    // Which variant (in-graph kernel durations, tools/ab_grid_reg.sh and
    // ab_grid_hyb.sh): 4- and 8-row chunks: k_grid_hyb (C2 19.3 vs 20.0 us,
    // C3's level 2 16.8 vs 17.9 us, 6e5 {32} 14.3 vs 14.6 us); 2-row chunks at
    // <= 5K rows per SM: k_grid_reg (1e5 {32} 10.9 vs 11.3 / 11.8 us); 5-row
    // and uneven chunks: k_grid_solve (6e5 {20} 16.2 vs 18.0 us).
    if ((L == 8 || L == 4) && g_ghyb == 1) {  // rows into registers and shared memory (k_grid_hyb)
        auto a32 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; };
        const int vec = a32(sys.sub) && a32(sys.diag) && a32(sys.sup) && a32(sys.rhs) && a32(x) ? 1 : 0;
        if (mode == kShard) return cudaLaunchKernelEx(&cfg, ghyb_kernel<T, kShard>(L), sys, geo, x, pairs, bar, err, level, lk, vec);
        return cudaLaunchKernelEx(&cfg, ghyb_kernel<T, kSolve>(L), sys, geo, x, pairs, bar, err, level, lk, vec);
    }
    if (L == 2 && rows_cta <= 5000 && g_greg == 1) {
        auto a32 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; };
        const int vec = a32(sys.sub) && a32(sys.diag) && a32(sys.sup) && a32(sys.rhs) && a32(x) ? 1 : 0;
        cfg.dynamicSmemBytes = greg_smem_bytes(sizeof(T));
        if (mode == kShard) return cudaLaunchKernelEx(&cfg, greg_kernel<T, kShard>(L), sys, geo, x, pairs, bar, err, level, lk, vec);
        return cudaLaunchKernelEx(&cfg, greg_kernel<T, kSolve>(L), sys, geo, x, pairs, bar, err, level, lk, vec);
    }
    if (mode == kShard) return cudaLaunchKernelEx(&cfg, grid_kernel<T, kShard>(L), sys, geo, x, pairs, bar, err, level, lk);
    return cudaLaunchKernelEx(&cfg, grid_kernel<T, kSolve>(L), sys, geo, x, pairs, bar, err, level, lk);
}

template cudaError_t launch_grid_solve<double>(const SysPtrs<double>&, int64_t, int64_t, double*, void*,
                                               unsigned long long*, int, int, cudaStream_t, int, const ShardLink*,
                                               int);
template cudaError_t launch_grid_solve<float>(const SysPtrs<float>&, int64_t, int64_t, float*, void*,
                                              unsigned long long*, int, int, cudaStream_t, int, const ShardLink*,
                                              int);

}  // namespace tpb

// Phase timestamps of the last traced launch (TPB_GRID_TRACE=1): 8 per CTA.
extern "C" int tp_debug_grid_trace(unsigned long long* out, int count) {
    if (count > 2 * 256 * tpb::kGridTraceSlots) count = 2 * 256 * tpb::kGridTraceSlots;
    return (int)cudaMemcpyFromSymbol(out, tpb::g_grid_trace, (size_t)count * sizeof(unsigned long long));
}
