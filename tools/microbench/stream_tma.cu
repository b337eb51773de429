// Stage-3-like streaming through a TMA (2D, 128B-swizzled) multi-stage smem pipeline:
// read 4 FP64 arrays, dependent DFMA chain of K ops per thread, write 1 array.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
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
__device__ __forceinline__ void st4(double* p, const double* v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
}
template <int NT, int S, int K>
__global__ void __launch_bounds__(NT + 32, 1) k_tma(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                                  const __grid_constant__ CUtensorMap tc, const __grid_constant__ CUtensorMap td,
                                                  double* x, long ntiles) {
    constexpr int TILE = NT * 8;               // rows per tile
    constexpr int ABYTES = TILE * 8;           // bytes per array per tile
    extern __shared__ uint8_t raw[];
    uint8_t* buf = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[S], empty[S];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) { for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NT / 32); } }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (warp == NT / 32) {  // producer warp
        if (lane == 0) {
            int k = 0;
            for (long t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
                const int s = k % S;
                if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
                mbar_expect(&full[s], 4 * ABYTES);
                uint8_t* st = buf + (size_t)s * 4 * ABYTES;
                const int row16 = (int)(t * (TILE / 16));
                tma2d(st + 0 * ABYTES, &ta, 0, row16, &full[s]);
                tma2d(st + 1 * ABYTES, &tb, 0, row16, &full[s]);
                tma2d(st + 2 * ABYTES, &tc, 0, row16, &full[s]);
                tma2d(st + 3 * ABYTES, &td, 0, row16, &full[s]);
            }
        }
        return;
    }
    int k = 0;
    const int line = tid >> 1, half = tid & 1;
    for (long t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % S;
        mbar_wait(&full[s], (k / S) & 1);
        const uint8_t* st = buf + (size_t)s * 4 * ABYTES;
        double v[4][8];
#pragma unroll
        for (int arr = 0; arr < 4; ++arr)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int phys = (4 * half + q) ^ (line & 7);
                const double2 d2 = *reinterpret_cast<const double2*>(st + arr * ABYTES + line * 128 + phys * 16);
                v[arr][2 * q] = d2.x; v[arr][2 * q + 1] = d2.y;
            }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        double sacc = v[0][0], m = v[1][1];
#pragma unroll 1
        for (int j = 0; j < K; ++j) sacc = fma(sacc, m, 1e-3);
        double o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = v[0][j] + v[1][j] + v[2][j] + v[3][j] + sacc;
        double* xp = x + (t * TILE + tid * 8);
        st4(xp, o); st4(xp + 4, o + 4);
    }
}
static PFN_cuTensorMapEncodeTiled_v12000 enc;
CUtensorMap make(double* p, long n, int tile) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {16, (cuuint64_t)(n / 16)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {16, (cuuint32_t)(tile / 16)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return tm;
}
static double *A, *B, *Cc, *D, *X; static const long N = 100000000;
template <int NT, int S, int K>
void run(int ctas_per_sm) {
    const int TILE = NT * 8;
    CUtensorMap ta = make(A, N, TILE), tb = make(B, N, TILE), tc = make(Cc, N, TILE), td = make(D, N, TILE);
    const size_t smem = (size_t)S * 4 * TILE * 8 + 1024;
    cudaFuncSetAttribute(k_tma<NT, S, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long ntiles = N / TILE;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        k_tma<NT, S, K><<<148 * ctas_per_sm, NT + 32, smem>>>(ta, tb, tc, td, X, ntiles);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    // check correctness of one tile
    double h[16]; cudaMemcpy(h, X + 12345 * 8, sizeof(h), cudaMemcpyDeviceToHost);
    printf("NT=%3d S=%d K=%4d ctas/SM=%d smem=%6zu: %.3f ms %.0f GB/s  %s x=%g\n", NT, S, K, ctas_per_sm, smem, best,
           40.0 * ntiles * TILE / best / 1e6, cudaGetErrorString(e), h[3]);
}
__global__ void init(double* p, long n, double v) { for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += gridDim.x * 256L) p[i] = v + (i % 7); }
int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    cudaMalloc(&A, N * 8); cudaMalloc(&B, N * 8); cudaMalloc(&Cc, N * 8); cudaMalloc(&D, N * 8); cudaMalloc(&X, N * 8);
    init<<<1184, 256>>>(A, N, 1); init<<<1184, 256>>>(B, N, 10); init<<<1184, 256>>>(Cc, N, 100); init<<<1184, 256>>>(D, N, 1000);
    cudaDeviceSynchronize();
    run<256, 3, 0>(1); run<256, 3, 200>(1); run<256, 3, 400>(1);
    run<128, 3, 0>(2); run<128, 3, 200>(2); run<128, 3, 400>(2);
    run<512, 1, 0>(1); run<256, 2, 200>(1); run<128, 4, 200>(1); run<128, 2, 200>(3);
    run<64, 4, 200>(4); run<64, 3, 200>(5);
    return 0;
}
