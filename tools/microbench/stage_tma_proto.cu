// Prototype: Stage 1 / Stage 3 of one level (m = 64: L = 8, G = 8) fed by a TMA
// (2D, 128B-swizzled) multi-stage shared-memory pipeline, versus the library's
// register-load k_fast. Same arithmetic -> outputs must be bit-identical.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "../../paper_2510_27351_b200/csrc/tp_fast.cuh"

using namespace tpb;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n }" ::"r"(sa(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(sa(dst)), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(sa(bar)) : "memory");
}

struct Maps { CUtensorMap a, b, c, d; };

template <int MODE, int NT, int S, int MINB>
__global__ void __launch_bounds__(NT + 32, MINB)
k_tma(const __grid_constant__ Maps tm, int64_t nblocks, IfacePtrs<double> out, const double* __restrict__ xi,
      double* __restrict__ x, unsigned long long* err, int level) {
    constexpr int L = 8, G = 8;
    constexpr bool KEEP = (MODE != kStage1);
    constexpr int TILE = NT * L;
    constexpr int ABYTES = TILE * 8;
    extern __shared__ uint8_t raw[];
    uint8_t* buf = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[S], empty[S];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nchunks = nblocks * G;
    const int64_t ntiles = (nchunks + NT - 1) / NT;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NT / 32); }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (warp == NT / 32) {  // producer
        if (lane == 0) {
            int k = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
                const int s = k % S;
                if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
                mbar_expect(&full[s], 4 * ABYTES);
                uint8_t* st = buf + (size_t)s * 4 * ABYTES;
                const int r16 = (int)(t * (TILE / 16));
                tma2d(st + 0 * ABYTES, &tm.a, 0, r16, &full[s]);
                tma2d(st + 1 * ABYTES, &tm.b, 0, r16, &full[s]);
                tma2d(st + 2 * ABYTES, &tm.c, 0, r16, &full[s]);
                tma2d(st + 3 * ABYTES, &tm.d, 0, r16, &full[s]);
            }
        }
        return;
    }
    const int c = lane % G;
    const int line = tid >> 1, half = tid & 1;
    int64_t bad = INT64_MAX;
    int k = 0;
    for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++k) {
        const int s = k % S;
        const int64_t t = tl * NT + tid;
        const bool active = t < nchunks;
        const int64_t row0 = t * L;
        const int64_t blk = t / G;
        double xs = 0, xe = 0;
        if constexpr (MODE != kStage1) {
            if (c == 0 && active) {
                const Pair<double> v = load_pair(xi + 2 * blk);
                xs = v.x;
                xe = v.y;
            }
        }
        LaneState<double, L, G, KEEP> st;
        mbar_wait(&full[s], (k / S) & 1);
        const uint8_t* sb = buf + (size_t)s * 4 * ABYTES;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int off = line * 128 + (((4 * half + q) ^ (line & 7)) << 4);
            const double2 va = *reinterpret_cast<const double2*>(sb + 0 * ABYTES + off);
            const double2 vb = *reinterpret_cast<const double2*>(sb + 1 * ABYTES + off);
            const double2 vc = *reinterpret_cast<const double2*>(sb + 2 * ABYTES + off);
            const double2 vd = *reinterpret_cast<const double2*>(sb + 3 * ABYTES + off);
            st.r.a[2 * q] = va.x; st.r.a[2 * q + 1] = va.y;
            st.r.b[2 * q] = vb.x; st.r.b[2 * q + 1] = vb.y;
            st.r.c[2 * q] = vc.x; st.r.c[2 * q + 1] = vc.y;
            st.r.d[2 * q] = vd.x; st.r.d[2 * q + 1] = vd.y;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (!active) {
#pragma unroll
            for (int i = 0; i < L; ++i) { st.r.a[i] = 0; st.r.b[i] = 1; st.r.c[i] = 0; st.r.d[i] = 0; }
        }
        lane_leaf<double, L, G, KEEP>(st, row0);
        lanes_tree<double, L, G, KEEP>(st, c, row0);
        if constexpr (MODE == kStage1) {
            if (active) {
                if (st.guard.tripped()) bad = row0 < bad ? row0 : bad;
                if (c == 0) store_block_eqs(out, blk, st.cur);
            }
        } else {
            double xv[L];
            lanes_tree_down<double, L, G>(st, c, xs, xe);
            leaf_expand<double, L, L>(st.r, st.rbeta, st.gam, st.del, xs, xe, xv);
            if (active) {
                if (st.guard.tripped()) bad = row0 < bad ? row0 : bad;
                store_rows<double, L, true>(x, row0, xv);
            }
        }
    }
    report_pivot(err, level, bad);
}

__global__ void gen(double* a, double* b, double* c, double* d, double* xi, int64_t n, int64_t nx) {
    for (int64_t i = blockIdx.x * 256L + threadIdx.x; i < n; i += gridDim.x * 256L) {
        uint64_t h = i * 0x9E3779B97F4A7C15ULL;
        h ^= h >> 31; h *= 0xbf58476d1ce4e5b9ULL; h ^= h >> 29;
        const double u = (double)(h >> 11) * 0x1.0p-53 * 2 - 1, v = (double)((h * 31) >> 11) * 0x1.0p-53 * 2 - 1;
        a[i] = u; c[i] = v; b[i] = 1.5 * (fabs(u) + fabs(v)) + 1; d[i] = u * v;
        if (i < nx) xi[i] = v;
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
CUtensorMap make(const double* p, int64_t rows, int tile) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {16, (cuuint64_t)(rows / 16)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {16, (cuuint32_t)(tile / 16)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return tm;
}

static double *A, *B, *Cc, *D, *XI, *X, *X2, *IF[4], *IF2[4];
static unsigned long long* ERR;
static const int64_t N = 100000000, NB = N / 64;

template <class F>
float timeit(F f, int reps = 7) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    return best;
}
bool same(const double* p, const double* q, int64_t n) {
    std::vector<double> h1(n), h2(n);
    cudaMemcpy(h1.data(), p, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), q, n * 8, cudaMemcpyDeviceToHost);
    return memcmp(h1.data(), h2.data(), n * 8) == 0;
}

template <int NT, int S, int MINB>
void run(int ctas_per_sm) {
    const int TILE = NT * 8;
    Maps m{make(A, N, TILE), make(B, N, TILE), make(Cc, N, TILE), make(D, N, TILE)};
    const size_t smem = (size_t)S * 4 * TILE * 8 + 1024;
    cudaFuncSetAttribute(k_tma<kStage1, NT, S, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_tma<kStage3, NT, S, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    IfacePtrs<double> o2{IF2[0], IF2[1], IF2[2], IF2[3]};
    const int grid = 148 * ctas_per_sm;
    float t1 = timeit([&] { k_tma<kStage1, NT, S, MINB><<<grid, NT + 32, smem>>>(m, NB, o2, nullptr, nullptr, ERR, 0); });
    float t3 = timeit([&] { k_tma<kStage3, NT, S, MINB><<<grid, NT + 32, smem>>>(m, NB, o2, XI, X2, ERR, 0); });
    cudaError_t e = cudaGetLastError();
    bool ok1 = true;
    for (int q = 0; q < 4; ++q) ok1 = ok1 && same(IF[q], IF2[q], 2 * NB);
    bool ok3 = same(X, X2, N);
    printf("TMA NT=%3d S=%d ctas/SM=%d smem=%6zu: S1 %.3f ms (%.0f GB/s) %s | S3 %.3f ms (%.0f GB/s) %s  %s\n", NT, S,
           ctas_per_sm, smem, t1, 32.0 * N / t1 / 1e6, ok1 ? "bit-identical" : "MISMATCH", t3, 40.0 * N / t3 / 1e6,
           ok3 ? "bit-identical" : "MISMATCH", cudaGetErrorString(e));
    cudaMemset(X2, 0, N * 8);
    for (int q = 0; q < 4; ++q) cudaMemset(IF2[q], 0, 2 * NB * 8);
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    cudaMalloc(&A, N * 8); cudaMalloc(&B, N * 8); cudaMalloc(&Cc, N * 8); cudaMalloc(&D, N * 8);
    cudaMalloc(&X, N * 8); cudaMalloc(&X2, N * 8); cudaMalloc(&XI, 2 * NB * 8); cudaMalloc(&ERR, 8);
    for (int i = 0; i < 4; ++i) { cudaMalloc(&IF[i], 2 * NB * 8); cudaMalloc(&IF2[i], 2 * NB * 8); }
    gen<<<1184, 256>>>(A, B, Cc, D, XI, N, 2 * NB);
    cudaDeviceSynchronize();
    SysPtrs<double> sys{A, B, Cc, D};
    IfacePtrs<double> o{IF[0], IF[1], IF[2], IF[3]};
    const int64_t nch = NB * 8;
    float r1 = timeit([&] { k_fast<double, 8, 8, kStage1, true, 128, 6><<<(unsigned)((nch + 127) / 128), 128>>>(sys, NB, o, nullptr, nullptr, ERR, 0); });
    float r3 = timeit([&] { k_fast<double, 8, 8, kStage3, true, 128, 4><<<592, 128>>>(sys, NB, o, XI, X, ERR, 0); });
    printf("k_fast (library)          : S1 %.3f ms (%.0f GB/s)              | S3 %.3f ms (%.0f GB/s)  %s\n", r1, 32.0 * N / r1 / 1e6,
           r3, 40.0 * N / r3 / 1e6, cudaGetErrorString(cudaGetLastError()));
    run<256, 3, 1>(1);
    run<512, 2, 1>(1);
    run<256, 2, 1>(1);
    run<128, 3, 2>(2);
    run<128, 2, 3>(3);
    run<384, 2, 1>(1);
    float r3b = timeit([&] { k_fast<double, 8, 8, kStage3, true, 128, 4><<<592, 128>>>(sys, NB, o, XI, X, ERR, 0); });
    printf("k_fast S3 again %.3f ms\n", r3b);
    return 0;
}
