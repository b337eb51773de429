// FP64 issue throughput on one SM: independent DFMA / DMUL / MUFU.RCP64H
// streams (8 chains per thread), 512 threads per CTA, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/fp64_tput fp64_tput.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(512, 1) k(int iters, double* out, long long* cyc) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 1.0 + 1e-3 * (threadIdx.x + j);
    const double a = 0.999999, c = 1e-9;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) v[j] = fma(v[j], a, c);
            else if (OP == 1) v[j] = v[j] * a;
            else {
                double r;
                asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v[j]));
                v[j] = r;
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 512 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    const int iters = 4096;
    const char* names[3] = {"DFMA", "DMUL", "MUFU.RCP64H"};
    for (int op = 0; op < 3; ++op)
        for (int threads : {32, 128, 512}) {
            long long c = 0;
            for (int t = 0; t < 3; ++t) {
                if (op == 0) k<0><<<148, threads>>>(iters, out, cyc);
                if (op == 1) k<1><<<148, threads>>>(iters, out, cyc);
                if (op == 2) k<2><<<148, threads>>>(iters, out, cyc);
                cudaDeviceSynchronize();
                cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
            }
            const double warp_ops = (double)iters * 8 * (threads / 32);
            std::printf("%-12s %3d threads/SM: %.3f warp-instr per cycle per SM (%.1f lanes/cycle)\n", names[op],
                        threads, warp_ops / c, 32 * warp_ops / c);
        }
    return 0;
}
