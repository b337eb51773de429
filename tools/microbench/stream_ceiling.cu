// Streaming ceilings on B200 for the partition solver's access patterns:
//   r4w1: read 4 arrays, write 1 (Stage 3 pattern), r4: read 4 arrays (Stage 1), copy: 1r1w
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void ld4(const double* p, double* v) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void st4(double* p, const double* v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
}
template <int MODE>  // 0: r4w1, 1: r4 (sum to one atomic), 2: copy
__global__ void __launch_bounds__(256) k(const double* a, const double* b, const double* c, const double* d, double* x, long n, double* sink) {
    double acc = 0;
    for (long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n; i += (long)gridDim.x * blockDim.x * 8) {
        double va[8], vb[8], vc[8], vd[8], o[8];
        ld4(a + i, va); ld4(a + i + 4, va + 4);
        if (MODE != 2) { ld4(b + i, vb); ld4(b + i + 4, vb + 4); ld4(c + i, vc); ld4(c + i + 4, vc + 4); ld4(d + i, vd); ld4(d + i + 4, vd + 4); }
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = MODE == 2 ? va[j] : va[j] + vb[j] + vc[j] + vd[j];
        if (MODE == 1) { for (int j = 0; j < 8; ++j) acc += o[j]; }
        else { st4(x + i, o); st4(x + i + 4, o + 4); }
    }
    if (MODE == 1 && acc == 12345.678) *sink = acc;
}
int main() {
    const long n = 100000000;
    double *a, *b, *c, *d, *x, *s;
    cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8); cudaMalloc(&c, n * 8); cudaMalloc(&d, n * 8); cudaMalloc(&x, n * 8); cudaMalloc(&s, 8);
    cudaMemset(a, 0, n * 8); cudaMemset(b, 0, n * 8); cudaMemset(c, 0, n * 8); cudaMemset(d, 0, n * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int grids[] = {148 * 2, 148 * 4, 148 * 8, (int)(n / 8 / 256)};
    const char* names[] = {"r4w1", "r4", "copy"};
    for (int mode = 0; mode < 3; ++mode) for (int g : grids) {
        float best = 1e9;
        for (int rep = 0; rep < 10; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<g, 256>>>(a, b, c, d, x, n, s);
            if (mode == 1) k<1><<<g, 256>>>(a, b, c, d, x, n, s);
            if (mode == 2) k<2><<<g, 256>>>(a, b, c, d, x, n, s);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        double bytes = mode == 0 ? 40.0 * n : mode == 1 ? 32.0 * n : 16.0 * n;
        printf("%-5s grid %7d: %.3f ms  %.0f GB/s\n", names[mode], g, best, bytes / best / 1e6);
    }
    return 0;
}
