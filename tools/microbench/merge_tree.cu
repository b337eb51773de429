// Cost of one level of the warp merge tree (up: shuffle 8 values + merge; down:
// top-down step), for the sweep-form merge (`merge`, 4 reciprocals) and the
// Schur-complement form (`merge_schur`, 1 reciprocal). Cycles per level from
// clock64 over R repetitions of a 5-level up + 5-level down tree, with 1 warp
// and 16 warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I../../paper_2510_27351_b200/csrc -o merge_tree merge_tree.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tp_device.cuh"

using namespace tpb;

template <int KIND>
__global__ void k_tree(int reps, double* out, long long* cyc) {
    const int lane = threadIdx.x & 31;
    Eq2<double> q{0.1 * lane, 3.0 + 0.01 * lane, -0.2, 0.5 + lane, 0.3, 2.5, -0.1 * lane, 0.7};
    double acc = 0;
    bool flag = false;
    RowGuard bad;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        Eq2<double> cur = q;
        cur.d1 += acc * 1e-30;
        SchurSave<double> ss[5];
        MergeSave<double> ms[5];
#pragma unroll
        for (int lv = 0; lv < 5; ++lv) {
            const int h = 1 << lv;
            const Eq2<double> oth = shfl_down_eq(cur, h);
            if ((lane & (2 * h - 1)) == 0) {
                if (KIND == 0) cur = merge(cur, oth, (long long)lane, bad, ms[lv]);
                else cur = merge_schur(cur, oth, flag, ss[lv]);
            }
        }
        double xs = 0, xe = 0;
        if (lane == 0) root_solve(cur, 31, bad, xs, xe);
#pragma unroll
        for (int lv = 4; lv >= 0; --lv) {
            const int h = 1 << lv;
            const bool left = (lane & (2 * h - 1)) == 0, right = (lane & (2 * h - 1)) == h;
            if (KIND == 0) {
                double xt = 0;
                if (left) xt = merge_xt(ms[lv], xs, xe);
                const double rxt = __shfl_up_sync(0xffffffffu, xt, h);
                const double rxe = __shfl_up_sync(0xffffffffu, xe, h);
                if (right) { xs = first_from_e1(cur, rxt, rxe); xe = rxe; }
                else if (left) xe = xt;
            } else {
                double xt = 0, xt1 = 0;
                if (left) schur_down(ss[lv], xs, xe, xt, xt1);
                const double r1 = __shfl_up_sync(0xffffffffu, xt1, h);
                const double rxe = __shfl_up_sync(0xffffffffu, xe, h);
                if (right) { xs = r1; xe = rxe; }
                else if (left) xe = xt;
            }
        }
        acc += xs + xe;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + (flag ? 1 : 0) + (bad.bad != INT64_MAX ? 1 : 0);
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    const int reps = 2000;
    for (int kind = 0; kind < 2; ++kind)
        for (int warps : {1, 16}) {
            long long c = 0;
            for (int t = 0; t < 3; ++t) {
                if (kind == 0) k_tree<0><<<148, 32 * warps>>>(reps, out, cyc);
                else k_tree<1><<<148, 32 * warps>>>(reps, out, cyc);
                cudaDeviceSynchronize();
                cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
            }
            std::printf("%-12s warps/SM %2d: %.1f cycles per tree (5 up + root + 5 down), %.1f per level\n",
                        kind == 0 ? "merge" : "merge_schur", warps, (double)c / reps, (double)c / reps / 10.0);
        }
    return 0;
}
