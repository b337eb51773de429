// Stage-3-like streaming (read 4 arrays, FP64 dependent chain of K ops, write 1) with
// different load schemes: LDG to registers vs per-thread cp.async prefetch of the next tile.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void ld4(const double* p, double* v) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void st4(double* p, const double* v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
}
__device__ __forceinline__ void cpa16(void* s, const void* g) {
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int K>
__device__ __forceinline__ void work(double (&va)[8], double (&vb)[8], double (&vc)[8], double (&vd)[8], double* x, long i) {
    double s = va[0], t = vb[1];
#pragma unroll 1
    for (int j = 0; j < K; ++j) { s = fma(s, t, 1e-3); }
    double o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = va[j] + vb[j] + vc[j] + vd[j] + s;
    st4(x + i, o); st4(x + i + 4, o + 4);
}
// scheme 0: LDG, grid-stride over tiles of NT*8 rows (grid = full or persistent)
template <int K, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_ldg(const double* a, const double* b, const double* c, const double* d, double* x, long n) {
    for (long i = ((long)blockIdx.x * NT + threadIdx.x) * 8; i < n; i += (long)gridDim.x * NT * 8) {
        double va[8], vb[8], vc[8], vd[8];
        ld4(a + i, va); ld4(a + i + 4, va + 4); ld4(b + i, vb); ld4(b + i + 4, vb + 4);
        ld4(c + i, vc); ld4(c + i + 4, vc + 4); ld4(d + i, vd); ld4(d + i + 4, vd + 4);
        work<K>(va, vb, vc, vd, x, i);
    }
}
// scheme 1: per-thread cp.async of the next tile into a private 80 B-stride smem slot;
// tiles assigned grid-stride (BLOCKED=0) or T consecutive tiles per CTA (BLOCKED=1)
template <int K, int NT, int MINB, int BLOCKED>
__global__ void __launch_bounds__(NT, MINB) k_cpa(const double* a, const double* b, const double* c, const double* d, double* x, long n, int T) {
    __shared__ __align__(16) double sm[4][NT * 10];
    const long ntiles = n / (NT * 8);
    long tile, tstep, tend;
    if (BLOCKED) { tile = (long)blockIdx.x * T; tstep = 1; tend = tile + T < ntiles ? tile + T : ntiles; }
    else { tile = blockIdx.x; tstep = gridDim.x; tend = ntiles; }
    const int me = threadIdx.x * 10;
    auto issue = [&](long tl) {
        const long i = (tl * NT + threadIdx.x) * 8;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            cpa16(&sm[0][me + 2 * q], a + i + 2 * q); cpa16(&sm[1][me + 2 * q], b + i + 2 * q);
            cpa16(&sm[2][me + 2 * q], c + i + 2 * q); cpa16(&sm[3][me + 2 * q], d + i + 2 * q);
        }
        cpa_commit();
    };
    if (tile < tend) issue(tile);
    for (; tile < tend; tile += tstep) {
        cpa_wait0();
        double va[8], vb[8], vc[8], vd[8];
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
            double2 t0 = *reinterpret_cast<double2*>(&sm[0][me + q]); va[q] = t0.x; va[q + 1] = t0.y;
            double2 t1 = *reinterpret_cast<double2*>(&sm[1][me + q]); vb[q] = t1.x; vb[q + 1] = t1.y;
            double2 t2 = *reinterpret_cast<double2*>(&sm[2][me + q]); vc[q] = t2.x; vc[q + 1] = t2.y;
            double2 t3 = *reinterpret_cast<double2*>(&sm[3][me + q]); vd[q] = t3.x; vd[q + 1] = t3.y;
        }
        if (tile + tstep < tend) issue(tile + tstep);
        work<K>(va, vb, vc, vd, x, (tile * NT + threadIdx.x) * 8);
    }
}
float timeit(void (*f)(cudaStream_t), int reps = 6) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < reps; ++r) { cudaEventRecord(e0); f(0); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; }
    return best;
}
static double *A, *B, *Cc, *D, *X; static const long N = 100000000;
#define REPORT(tag, expr, kern)                                                                    \
    { int nb; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 128, 0);                       \
      float ms = timeit([](cudaStream_t) { expr; });                                                \
      printf("%-26s occ %d/SM: %.3f ms %.0f GB/s\n", tag, nb, ms, 40.0 * N / ms / 1e6); }
template <int K>
void sweep() {
    printf("--- K=%d dependent DFMA\n", K);
    REPORT("ldg full", (k_ldg<K, 128, 4><<<N / 1024, 128>>>(A, B, Cc, D, X, N)), (k_ldg<K, 128, 4>));
    REPORT("ldg persistent 4/SM", (k_ldg<K, 128, 4><<<592, 128>>>(A, B, Cc, D, X, N)), (k_ldg<K, 128, 4>));
    REPORT("cpa grid-stride 4/SM", (k_cpa<K, 128, 4, 0><<<592, 128>>>(A, B, Cc, D, X, N, 0)), (k_cpa<K, 128, 4, 0>));
    REPORT("cpa grid-stride 5/SM", (k_cpa<K, 128, 5, 0><<<740, 128>>>(A, B, Cc, D, X, N, 0)), (k_cpa<K, 128, 5, 0>));
    REPORT("cpa blocked T=4", (k_cpa<K, 128, 4, 1><<<N / 1024 / 4 + 1, 128>>>(A, B, Cc, D, X, N, 4)), (k_cpa<K, 128, 4, 1>));
    REPORT("cpa blocked T=16", (k_cpa<K, 128, 4, 1><<<N / 1024 / 16 + 1, 128>>>(A, B, Cc, D, X, N, 16)), (k_cpa<K, 128, 4, 1>));
    REPORT("cpa blocked T=165 (1 wave)", (k_cpa<K, 128, 4, 1><<<N / 1024 / 165 + 1, 128>>>(A, B, Cc, D, X, N, 165)), (k_cpa<K, 128, 4, 1>));
}
int main() {
    cudaMalloc(&A, N * 8); cudaMalloc(&B, N * 8); cudaMalloc(&Cc, N * 8); cudaMalloc(&D, N * 8); cudaMalloc(&X, N * 8);
    cudaMemset(A, 0, N * 8); cudaMemset(B, 0, N * 8); cudaMemset(Cc, 0, N * 8); cudaMemset(D, 0, N * 8);
    sweep<0>(); sweep<100>(); sweep<200>(); sweep<400>();
    return 0;
}
