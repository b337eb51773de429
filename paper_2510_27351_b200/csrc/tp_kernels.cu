// sm_100a kernels of the B200 partition solver (FP64, HBM-bound).
//
// Kernel map (reference call stack partition.hpp:191-224):
//   k_fast<T,L,G,STAGE1> parallel_for(reduce_block) + assemble_interface   :203-205
//   k_fast<T,L,G,STAGE3> parallel_for(back_substitute + scatter)            :214-222
//   k_fast_rt<T,...>     the same for any m <= 256 (runtime chunk lengths)
//   k_generic<T,MODE>    the same for any block length (tail blocks, m > 256)
//   k_final_cl<T,MODE>   8-CTA cluster finishing solve replacing
//                        thomas_solve(iface) at the deepest level          :208-211
//                        (k_final: single-CTA version, systems < 64 rows);
//                        kShard = the fused multi-GPU exchange (tp_final.cuh)
//   k_gather_solve       sharded top level (NCCL transport): Thomas on 2P rows
//   k_generate           device-side counter-based generate_system analogue
//   k_residual           residual_inf (tridiagonal.hpp:74-87)
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

#include "tp_device.cuh"
#include "tp_kernels.h"
#include "tp_fast.cuh"

namespace tpb {

// Phase timestamps of the finishing solve (scratch builds with -DTPB_TRACE only).
#ifdef TPB_TRACE
__device__ unsigned long long g_trace[24];  // [0, 12) finishing solve, [12, 18) fused level
#define TP_TRACE_DECL long long tp_tr[12]
#define TP_TRACE(k) tp_tr[k] = clock64()
#define TP_TRACE_FLUSH \
    do { if (threadIdx.x == 0) for (int k_ = 0; k_ < 12; ++k_) g_trace[k_] = tp_tr[k_]; } while (0)
#define TP_LF_TRACE(k) do { if (threadIdx.x == 0 && blockIdx.x == 0) g_trace[12 + (k)] = clock64(); } while (0)
#else
#define TP_LF_TRACE(k) do { } while (0)
#define TP_TRACE_DECL
#define TP_TRACE(k) do { } while (0)
#define TP_TRACE_FLUSH do { } while (0)
#endif

}  // namespace tpb

#include "tp_generic.cuh"
#include "tp_final.cuh"
#include "tp_fold.cuh"
#include "tp_split.cuh"

namespace tpb {

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
// 0: off (default), 1: every solve-path launch, 2: launches of levels >= 1
// only. Mode 2 measured 2.5 us faster per C3 solve, but early-launched
// dependents hold SMs while they wait: ranks sharing one GPU (simulated fused
// ranks) then starve each other's exchange, so it stays opt-in.
static int g_pdl = 0;

template <typename... KArgs, typename... Args>
static cudaError_t launch_kc(int level, unsigned cluster, void (*kern)(KArgs...), unsigned grid, unsigned block,
                             size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (g_pdl == 1 || (g_pdl == 2 && level > 0)) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster > 0) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = cluster;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}
template <class... KArgs, class... Args>
static cudaError_t launch_k(int level, void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                            cudaStream_t st, Args... args) {
    return launch_kc(level, 0, kern, grid, block, smem, st, args...);
}

// Error-word reset at the head of every solve (a kernel rather than a memset
// node, so the first Stage-1 grid can be launched programmatically after it).
__global__ void k_reset(unsigned long long* err) {
    pdl_begin();
    if (threadIdx.x == 0) *err = kNoError;
}

cudaError_t launch_reset(unsigned long long* err, cudaStream_t st) {
    return launch_k(0, k_reset, 1, 32, 0, st, err);
}

// Launch shapes chosen by measurement (tools/microbench/level_shapes.cu and
// in-graph A/B runs on B200, N=1e8, m=64):
// Stage 1  128 threads, <=80 regs (6 CTAs/SM), one chunk per thread (full grid);
//          L = 8 chunks at <=96 regs (5 CTAs/SM): at 80 their leaf spilled
//          40-48 bytes per thread
// Stage 3  128 threads, <=128 regs (4 CTAs/SM), one chunk per thread (full
//          grid: 1.2% faster in the solve graph than a persistent grid-stride)
template <class T, int L, int G, int MODE, bool VEC>
struct FastCfg {
    static constexpr int kThreads = 128;
    static constexpr int kMinBlocks = (MODE == kStage1) ? (L == 8 ? 5 : 6) : 4;
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
        return launch_k(level, k_fast<T, L, G, kStage1, VEC, C::kThreads, C::kMinBlocks>, (unsigned)grid,
                        C::kThreads, 0, st, sys, nblocks, out, xi, x, err, level);
    } else {
        using C = FastCfg<T, L, G, kStage3, VEC>;
        int64_t grid = (nchunks + C::kThreads - 1) / C::kThreads;
        if (grid < 1) grid = 1;
        return launch_k(level, k_fast<T, L, G, kStage3, VEC, C::kThreads, C::kMinBlocks>, (unsigned)grid,
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


// Level 0 + level 1 Stage 1 in one kernel (tp_fold.cuh). Requires full
// level-0 blocks of a fixed shape, an even m1 whose blocks are exactly m1/2
// level-0 blocks (no level-1 tail) and G = 8 (16 level-0 blocks per pass).
// 5 CTAs/SM (96 registers): at 6 (80 registers) the pass loop spills and the
// kernel runs 492 vs 485 us (C3, in-graph)
static bool g_fold = true;

bool fold_fits(int64_t m0, int64_t K0, int64_t n1, int64_t m1, int64_t K1) {
    int L, G;
    if (!g_fold || !fast_shape(m0, &L, &G) || G != 8) return false;
    if (m1 < 4 || m1 % 2 != 0 || m1 > 64) return false;
    return n1 == 2 * K0 && K1 * m1 == n1 && K1 >= kFoldL1Blocks;
}

// level 2 folded as well: m2 == 32 makes level-2 block j exactly tile j
static bool g_fold2 = true;
static int g_fold_keep = 1;  // L2 evict_last on the deeper systems the fold writes (TPB_FOLD_KEEP)
bool fold2_fits(int64_t K1, int64_t n2, int64_t m2, int64_t K2) {
    return g_fold2 && m2 == 2 * kFoldL1Blocks && n2 == 2 * K1 && K2 == (K1 + kFoldL1Blocks - 1) / kFoldL1Blocks;
}

template <class T>
cudaError_t launch_fold(int64_t m0, bool vec, const SysPtrs<T>& sys, int64_t K0, const IfacePtrs<T>& out0,
                        int64_t m1, int64_t K1, const IfacePtrs<T>& out1, const IfacePtrs<T>* out2,
                        unsigned long long* err, int level, cudaStream_t st) {
    if (!fold_fits(m0, K0, 2 * K0, m1, K1)) return cudaErrorInvalidValue;
    const int64_t grid = (K1 + kFoldL1Blocks - 1) / kFoldL1Blocks;
    const size_t smem = (size_t)4 * kFoldL1Blocks * m1 * sizeof(T);
    const IfacePtrs<T> none{};
#define TPB_FOLD(MM, LL)                                                                               \
    if (m0 == MM) {                                                                                  \
        auto k = out2 != nullptr                                                                     \
                     ? (vec ? k_fast_s1fold<T, LL, 8, true, 128, 5, true> : k_fast_s1fold<T, LL, 8, false, 128, 5, true>) \
                     : (vec ? k_fast_s1fold<T, LL, 8, true, 128, 5> : k_fast_s1fold<T, LL, 8, false, 128, 5>); \
        return launch_k(level, k, (unsigned)grid, 128u, smem, st, sys, K0, out0, (int)m1, K1, out1,        \
                        out2 != nullptr ? *out2 : none, err, level, g_fold_keep);                    \
    }
    TPB_FOLD(40, 5)
    TPB_FOLD(64, 8)
#undef TPB_FOLD
    return cudaErrorInvalidValue;
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
            return launch_k(level, k_fast_rt<T, 8, GG, kStage1>, (unsigned)grid, 128, 0, st, sys, nblocks, m, out, xi, x, err, level); \
        return launch_k(level, k_fast_rt<T, 8, GG, kStage3>, (unsigned)grid, 128, 0, st, sys, nblocks, m, out, xi, x, err, level);
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
    return launch_k(level, k, (unsigned)grid, (unsigned)threads, smem, st, sys, row_base, blk_base, nblocks, blen, G,
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
        return launch_k(level, kc, kFinCS, kFinNT, 0, st, sys, n, gtot, out, xi, x, err, level,
                        link != nullptr ? *link : none);
    }
    const int G = final_G(n);
    const size_t smem = (size_t)(4 * n) * sizeof(T);
    auto k = mode == kStage1   ? k_final<T, kStage1>
             : mode == kStage3 ? k_final<T, kStage3>
             : mode == kShard  ? k_final<T, kShard>
                               : k_final<T, kSolve>;
    const ShardLink none{};
    return launch_k(level, k, 1, kFinalThreads2, smem, st, sys, n, G, out, xi, x, err, level,
                    link != nullptr ? *link : none);
}

// k_level_final_cl: odd block stride, >= m + 1 (the tail block has <= m + 1 rows)
static int level_final_stride(int64_t m) { return (int)((m + 1) % 2 == 1 ? m + 1 : m + 2); }
constexpr size_t kLfDynSmem = 176 * 1024;  // + 40 KB static (interface rows, solution)
static bool g_fuse_last = true;
// CTAs per cluster of the fused kernel: 16 (non-portable) when the GPU can
// co-schedule it, else 8; TPB_LF_CLUSTER=8 forces the portable shape
static int g_lf_cs = 8;

static int lf_cluster(int cs) { return cs == 8 ? 8 : g_lf_cs; }
static size_t level_final_smem(int64_t m, int64_t K, size_t elem, int c) {
    return (size_t)4 * (size_t)((K + c - 1) / c) * (size_t)level_final_stride(m) * elem;
}

bool level_final_fits(int64_t n, int64_t m, int64_t K, size_t elem, int cs) {
    // m <= 16: above that the one-thread-per-block sweeps of the fused kernel
    // lose to the level kernels' lane trees (C2, m = 32: 24.7 vs 22.6 us per solve).
    // The interface may exceed kFinalCap: each CTA solves <= 2 * kLfMaxBlocks of it.
    const int c = lf_cluster(cs);
    if (!g_fuse_last || !g_final_cluster || m < 4 || m > 16 || K < kFinClusterMin) return false;
    if ((K + c - 1) / c > kLfMaxBlocks) return false;
    if ((K - 1) * m >= n || n - (K - 1) * m > m + 1) return false;  // make_plan's shape
    return level_final_smem(m, K, elem, c) <= kLfDynSmem;
}

template <class T>
using LfKernel = void (*)(SysPtrs<T>, int64_t, int, int64_t, int, IfacePtrs<T>, T*, unsigned long long*, int,
                          ShardLink, int);

// kShard variants exist for FP64 only (the sharded C-ABI is FP64)
template <class T, int CS, int MODE>
static LfKernel<T> level_final_kernel(int64_t m) {
    if constexpr (MODE == kShard && !std::is_same<T, double>::value) {
        (void)m;
        return nullptr;
    } else {
        return m == 4 ? k_level_final_cl<T, 4, CS, MODE> : m == 8 ? k_level_final_cl<T, 8, CS, MODE>
               : m == 16 ? k_level_final_cl<T, 16, CS, MODE> : k_level_final_cl<T, 0, CS, MODE>;
    }
}

template <class T>
cudaError_t launch_level_final(const SysPtrs<T>& sys, int64_t n, int64_t m, int64_t K, const IfacePtrs<T>& iface,
                               T* x, unsigned long long* err, int level, cudaStream_t st, int mode,
                               const ShardLink* link, int cs, int flags) {
    if (!level_final_fits(n, m, K, sizeof(T), cs)) return cudaErrorInvalidValue;
    const int c = lf_cluster(cs);
    LfKernel<T> k = nullptr;
    if (mode == kShard) {
        if (link == nullptr || link->nranks < 1 || link->nranks > kMaxPeers) return cudaErrorInvalidValue;
        k = c == 16 ? level_final_kernel<T, 16, kShard>(m) : level_final_kernel<T, 8, kShard>(m);
    } else {
        k = c == 16 ? level_final_kernel<T, 16, kSolve>(m) : level_final_kernel<T, 8, kSolve>(m);
    }
    if (k == nullptr) return cudaErrorInvalidValue;
    const ShardLink none{};
    return launch_kc(level, (unsigned)c, k, (unsigned)c, kFinNT, level_final_smem(m, K, sizeof(T), c), st, sys, n,
                     (int)m, K, level_final_stride(m), iface, x, err, level, link != nullptr ? *link : none, flags);
}

template <class T, int CS, int MODE>
static cudaError_t set_level_final_attributes_m() {
    cudaError_t e = cudaSuccess;
    for (int64_t m : {4, 8, 16, 0}) {
        auto k = level_final_kernel<T, CS, MODE>(m);
        if (k == nullptr) continue;
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLfDynSmem);
        if (e == cudaSuccess && CS > 8) e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    return e;
}
template <class T, int CS>
static cudaError_t set_level_final_attributes() {
    cudaError_t e = set_level_final_attributes_m<T, CS, kSolve>();
    if (e == cudaSuccess) e = set_level_final_attributes_m<T, CS, kShard>();
    return e;
}

// 16 when a 16-CTA cluster of the fused kernel at full shared memory fits the GPU
static int probe_level_final_cluster() {
    if (set_level_final_attributes<double, 16>() != cudaSuccess ||
        set_level_final_attributes<float, 16>() != cudaSuccess) {
        cudaGetLastError();
        return 8;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(kFinNT);
    cfg.dynamicSmemBytes = kLfDynSmem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 16;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)k_level_final_cl<double, 16, 16, kSolve>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 8;
    }
    return nclusters >= 1 ? 16 : 8;
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
    if (e == cudaSuccess) e = set_level_final_attributes<T, 8>();
    return e;
}

cudaError_t init_kernel_attributes() {
    if (const char* v = getenv("TPB_PDL")) g_pdl = atoi(v);
    if (const char* v = getenv("TPB_FINAL_CLUSTER")) g_final_cluster = atoi(v) != 0;
    if (const char* v = getenv("TPB_FUSE_LAST")) g_fuse_last = atoi(v) != 0;
    if (const char* v = getenv("TPB_FOLD")) g_fold = atoi(v) != 0;
    if (const char* v = getenv("TPB_FOLD2")) g_fold2 = atoi(v) != 0;
    if (const char* v = getenv("TPB_FOLD_KEEP")) g_fold_keep = atoi(v);
    cudaError_t e = set_smem_attributes<double>();
    if (e == cudaSuccess) e = set_smem_attributes<float>();
    g_lf_cs = probe_level_final_cluster();
    if (const char* v = getenv("TPB_LF_CLUSTER")) if (atoi(v) == 8) g_lf_cs = 8;
    return e;
}

template <class T>
cudaError_t launch_split(int mode, const SysPtrs<T>& sys, int64_t row_base, int64_t nblocks, int64_t blen,
                         int64_t nsub, int64_t q_base, const IfacePtrs<T>& out, const T* xi, T* x,
                         unsigned long long* err, int level, cudaStream_t st) {
    if (nblocks < 1 || nsub < 1 || blen < 2 * nsub || (blen + nsub - 1) / nsub > kSplitRows)
        return cudaErrorInvalidValue;
    const int64_t grid = (nblocks * nsub + 127) / 128;
    if (mode == kStage1)
        return launch_k(level, k_split<T, kStage1>, (unsigned)grid, 128, 0, st, sys, row_base, nblocks, blen, nsub,
                        q_base, out, xi, x, err, level);
    return launch_k(level, k_split<T, kStage3>, (unsigned)grid, 128, 0, st, sys, row_base, nblocks, blen, nsub,
                    q_base, out, xi, x, err, level);
}

template <class T>
cudaError_t launch_ref_sweep(const SysPtrs<T>& sys, int64_t n, int64_t m, int64_t K, int64_t* first,
                             unsigned long long* jmin, T* eq8, T* ua, T* ubeta, T* ugamma, T* udelta,
                             cudaStream_t st) {
    int64_t grid = (K + 127) / 128;
    if (grid > 148 * 16) grid = 148 * 16;
    if (grid < 1) grid = 1;
    if (eq8 != nullptr)
        k_ref_sweep<T, true><<<(unsigned)grid, 128, 0, st>>>(sys, n, m, K, first, jmin, eq8, ua, ubeta, ugamma,
                                                             udelta);
    else
        k_ref_sweep<T, false><<<(unsigned)grid, 128, 0, st>>>(sys, n, m, K, first, jmin, nullptr, nullptr, nullptr,
                                                              nullptr, nullptr);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_ref_thomas(const SysPtrs<T>& sys, int64_t n, int64_t* out, cudaStream_t st) {
    k_ref_thomas<T><<<1, 32, 0, st>>>(sys, n, out);
    return cudaGetLastError();
}

template <class T>
cudaError_t launch_gather_solve(const T* eqs, int nranks, int rank, T* x2, T* scratch,
                                unsigned long long* err, int level, cudaStream_t st) {
    return launch_k(level, k_gather_solve<T>, 1, 32, 0, st, eqs, nranks, rank, x2, scratch, err, level);
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
    template cudaError_t launch_fold<T>(int64_t, bool, const SysPtrs<T>&, int64_t, const IfacePtrs<T>&, \
                                        int64_t, int64_t, const IfacePtrs<T>&, const IfacePtrs<T>*,        \
                                        unsigned long long*, int, cudaStream_t);                        \
    template cudaError_t launch_level_final<T>(const SysPtrs<T>&, int64_t, int64_t, int64_t,        \
                                               const IfacePtrs<T>&, T*, unsigned long long*, int,   \
                                               cudaStream_t, int, const ShardLink*, int, int);      \
    template cudaError_t launch_split<T>(int, const SysPtrs<T>&, int64_t, int64_t, int64_t, int64_t,   \
                                         int64_t, const IfacePtrs<T>&, const T*, T*,                \
                                         unsigned long long*, int, cudaStream_t);                   \
    template cudaError_t launch_ref_sweep<T>(const SysPtrs<T>&, int64_t, int64_t, int64_t, int64_t*,   \
                                             unsigned long long*, T*, T*, T*, T*, T*, cudaStream_t);  \
    template cudaError_t launch_ref_thomas<T>(const SysPtrs<T>&, int64_t, int64_t*, cudaStream_t);      \
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
