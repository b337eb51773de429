// FP64 latency microbenchmark (dependent chains, one warp / many warps)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcpa(double x) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__global__ void k(double* out, long long* cyc, double s, int n) {
    double a = s + threadIdx.x, b = 1.0000001, c = 1e-9, r = s;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = fma(a, b, c); }
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) { a = a * b; }
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) { r = rcpa(r); }
    long long t3 = clock64();
    float f = (float)s;
    for (int i = 0; i < n; ++i) { f = fmaf(f, 1.0000001f, 1e-9f); }
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) { double e = fma(-a, r, 1.0); r = fma(r, fma(e, e, e), r); }
    long long t5 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + r + f;
    if (threadIdx.x == 0 && blockIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMallocManaged(&c, 64);
    const int n = 1024;
    int cfg[][2] = {{1, 32}, {1, 128}, {1, 512}, {148, 512}, {148 * 4, 512}};
    for (auto& g : cfg) {
        for (int rep = 0; rep < 2; ++rep) k<<<g[0], g[1]>>>(o, c, 1.5, n);
        cudaDeviceSynchronize();
        printf("grid %4d x %4d: DFMA %.1f  DMUL %.1f  MUFU.RCP64H %.1f  FFMA %.1f  newton(3 DFMA) %.1f cycles/op\n", g[0], g[1],
               c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n);
    }
    return 0;
}
