// Launch-shape sweep of the level kernels at m = 64 (N = 1e8): (L, G) x threads x min-blocks.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_27351_b200/csrc/tp_fast.cuh"
using namespace tpb;
__global__ void gen(double* a, double* b, double* c, double* d, double* xi, int64_t n, int64_t nx) {
    for (int64_t i = blockIdx.x * 256L + threadIdx.x; i < n; i += gridDim.x * 256L) {
        uint64_t h = i * 0x9E3779B97F4A7C15ULL; h ^= h >> 31; h *= 0xbf58476d1ce4e5b9ULL; h ^= h >> 29;
        const double u = (double)(h >> 11) * 0x1.0p-53 * 2 - 1, v = (double)((h * 31) >> 11) * 0x1.0p-53 * 2 - 1;
        a[i] = u; c[i] = v; b[i] = 1.5 * (fabs(u) + fabs(v)) + 1; d[i] = u * v;
        if (i < nx) xi[i] = v;
    }
}
static double *A, *B, *Cc, *D, *XI, *X, *IF[4];
static unsigned long long* ERR;
static const int64_t N = 100000000, NB = N / 64;
template <class F> float timeit(F f, int reps = 7) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float best = 1e9;
    for (int r = 0; r < reps; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; }
    return best;
}
template <int L, int G, int NT, int MB1, int MB3>
void run() {
    SysPtrs<double> sys{A, B, Cc, D};
    IfacePtrs<double> o{IF[0], IF[1], IF[2], IF[3]};
    const int64_t nch = NB * G;
    int nb1, nb3;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb1, k_fast<double, L, G, kStage1, true, NT, MB1>, NT, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb3, k_fast<double, L, G, kStage3, true, NT, MB3>, NT, 0);
    float t1 = timeit([&] { k_fast<double, L, G, kStage1, true, NT, MB1><<<(unsigned)((nch + NT - 1) / NT), NT>>>(sys, NB, o, nullptr, nullptr, ERR, 0); });
    float t3p = timeit([&] { k_fast<double, L, G, kStage3, true, NT, MB3><<<148 * nb3, NT>>>(sys, NB, o, XI, X, ERR, 0); });
    float t3f = timeit([&] { k_fast<double, L, G, kStage3, true, NT, MB3><<<(unsigned)((nch + NT - 1) / NT), NT>>>(sys, NB, o, XI, X, ERR, 0); });
    printf("L=%d G=%2d NT=%3d | S1 minb %d occ %d: %.4f ms (%5.0f GB/s) | S3 minb %d occ %d: pers %.4f full %.4f ms (%5.0f GB/s)  %s\n",
           L, G, NT, MB1, nb1, t1, 33.0 * N / t1 / 1e6, MB3, nb3, t3p, t3f, 40.0 * N / (t3p < t3f ? t3p : t3f) / 1e6,
           cudaGetErrorString(cudaGetLastError()));
}
int main() {
    cudaMalloc(&A, N * 8); cudaMalloc(&B, N * 8); cudaMalloc(&Cc, N * 8); cudaMalloc(&D, N * 8);
    cudaMalloc(&X, N * 8); cudaMalloc(&XI, 2 * NB * 8); cudaMalloc(&ERR, 8);
    for (int i = 0; i < 4; ++i) cudaMalloc(&IF[i], 2 * NB * 8);
    gen<<<1184, 256>>>(A, B, Cc, D, XI, N, 2 * NB); cudaDeviceSynchronize();
    run<8, 8, 128, 6, 4>();   // library shape
    run<8, 8, 128, 6, 4>();
    run<8, 8, 256, 3, 2>();
    run<8, 8, 64, 12, 8>();
    run<8, 8, 128, 5, 3>();
    run<8, 8, 128, 7, 5>();
    run<8, 8, 128, 8, 4>();
    run<4, 16, 128, 8, 5>();
    run<4, 16, 128, 10, 6>();
    run<4, 16, 256, 4, 3>();
    run<16, 4, 128, 4, 2>();
    run<16, 4, 128, 3, 3>();
    return 0;
}
