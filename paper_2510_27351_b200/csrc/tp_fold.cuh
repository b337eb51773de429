// Stage 1 of level 0 with level 1's Stage 1 folded in (k_fast_s1fold).
//
// When level 1's block size m1 is even, one level-1 block is exactly h = m1/2
// level-0 blocks' interface rows (assemble_interface order, partition.hpp:
// 139-149). A CTA here owns 16 level-1 blocks = 16 h level-0 blocks: it runs
// the k_fast Stage-1 pass over them h times (16 level-0 blocks per pass, G
// lanes each), keeps their E1/E2 rows in shared memory as well as writing
// them to HBM (Stage 3 of level 1 reads that system), then 16 threads sweep
// the 16 level-1 blocks from shared memory (leaf_smem, partition.hpp:90-124)
// and write level 2's system. The separate Stage-1 kernel of level 1 and its
// 100 MB re-read (C3) disappear; with m2 = 32 (C3, C4) level 2's Stage-1
// kernel and its tail branch as well (FOLD2).
#pragma once
#include "tp_fast.cuh"
#include "tp_generic.cuh"

namespace tpb {

constexpr int kFoldL1Blocks = 16;  // level-1 blocks per CTA

// Stores of the small deeper-level systems (C3: 20 MB + 1.25 MB) marked
// L2 evict_last so they survive the level-0 stream until their readers.
__device__ __forceinline__ uint64_t l2_keep_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void store_pair_keep(double* p, double x0, double x1, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(x0), "d"(x1), "l"(pol) : "memory");
}
__device__ __forceinline__ void store_pair_keep(float* p, float x0, float x1, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(x0), "f"(x1), "l"(pol) : "memory");
}
template <class T>
__device__ __forceinline__ void store_block_eqs_keep(const IfacePtrs<T>& out, int64_t blk, const Eq2<T>& q, bool keep) {
    if (!keep) {
        store_block_eqs(out, blk, q);
        return;
    }
    const uint64_t pol = l2_keep_policy();
    const int64_t o = 2 * blk;
    store_pair_keep(out.sub + o, q.a1, q.a2, pol);
    store_pair_keep(out.diag + o, q.b1, q.b2, pol);
    store_pair_keep(out.sup + o, q.g1, q.g2, pol);
    store_pair_keep(out.rhs + o, q.d1, q.d2, pol);
}

// FOLD2: level 2 has m2 = 32 = 2 x 16, so its block j IS this CTA's 16
// level-1 blocks' interface rows: the CTA also sweeps it (8 lanes x 4 rows in
// warp 0, the k_fast lane tree) and writes level 3's system; level 2's
// system is still written to HBM for its Stage 3.
template <class T, int L, int G, bool VEC, int THREADS, int MINB, bool FOLD2 = false>
__global__ void __launch_bounds__(THREADS, MINB)
    k_fast_s1fold(SysPtrs<T> sys, int64_t nblocks0, IfacePtrs<T> out0, int m1, int64_t nblocks1,
                  IfacePtrs<T> out1, IfacePtrs<T> out2, unsigned long long* err, int level, int keep) {
    static_assert(32 % G == 0, "G must divide the warp");
    constexpr int BP = THREADS / G;  // level-0 blocks per pass
    static_assert(BP == kFoldL1Blocks, "one pass = 16 level-0 blocks");
    extern __shared__ __align__(16) unsigned char fold_raw[];
    const int h = m1 / 2;                           // level-0 blocks per level-1 block
    const int rows1 = kFoldL1Blocks * m1;           // level-1 rows per CTA
    T* sa = reinterpret_cast<T*>(fold_raw);
    T* sb = sa + rows1;
    T* sc = sb + rows1;
    T* sd = sc + rows1;
    const int c = (threadIdx.x & 31) % G;
    const int64_t blk0_base = (int64_t)blockIdx.x * kFoldL1Blocks * h;
    __shared__ T s2[4][FOLD2 ? 2 * kFoldL1Blocks : 1];  // level-2 rows of this tile
    pdl_begin();

    for (int p = 0; p < h; ++p) {
        const int lb = p * BP + (int)threadIdx.x / G;  // level-0 block inside the tile
        const int64_t blk = blk0_base + lb;
        const bool active = blk < nblocks0;           // warp-uniform (BP blocks per pass, G | 32)
        const int64_t t = blk * G + c;
        const int64_t row0 = t * L;
        LaneState<T, L, G, false> s;
        load_chunk<T, L, VEC>(sys, row0, active, s.r);
        lane_leaf<T, L, G, false>(s, row0);
        lanes_tree<T, L, G, false>(s, c, row0);
        if (active) {
            if (s.guard.tripped()) report_pivot(err, level, row0);
            if (c == 0) {
                store_block_eqs(out0, blk, s.cur);
                const int r = 2 * lb;
                sa[r] = s.cur.a1; sa[r + 1] = s.cur.a2;
                sb[r] = s.cur.b1; sb[r + 1] = s.cur.b2;
                sc[r] = s.cur.g1; sc[r + 1] = s.cur.g2;
                sd[r] = s.cur.d1; sd[r + 1] = s.cur.d2;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < kFoldL1Blocks) {
        const int64_t j = (int64_t)blockIdx.x * kFoldL1Blocks + threadIdx.x;
        if (j < nblocks1) {
            const int o = (int)threadIdx.x * m1;
            RowGuard bad;
            Eq2<T> q;
            if (m1 == 10) {  // C3's level 1: both sweeps from registers (independent chains)
                Chunk<T, 10> r;
#pragma unroll
                for (int i = 0; i < 10; ++i) { r.a[i] = sa[o + i]; r.b[i] = sb[o + i]; r.c[i] = sc[o + i]; r.d[i] = sd[o + i]; }
                q = leaf_reduce<T, 10, 10>(r, j * m1, bad);
            } else {
                q = leaf_smem<T, false>(sa + o, sb + o, sc + o, sd + o, m1, j * m1, bad);
            }
            store_block_eqs_keep(out1, j, q, keep != 0);
            report_pivot(err, level + 1, bad.bad);
            if constexpr (FOLD2) {
                const int r = 2 * (int)threadIdx.x;
                s2[0][r] = q.a1; s2[0][r + 1] = q.a2;
                s2[1][r] = q.b1; s2[1][r + 1] = q.b2;
                s2[2][r] = q.g1; s2[2][r + 1] = q.g2;
                s2[3][r] = q.d1; s2[3][r + 1] = q.d2;
            }
        }
    }
    if constexpr (FOLD2) {
        __syncwarp();  // the 16 writers are lanes 0-15 of warp 0
        if (threadIdx.x < 32) {
            const int64_t j2 = blockIdx.x;
            const int64_t nb1 = nblocks1 - j2 * kFoldL1Blocks;  // level-1 blocks in this tile
            const int lane = (int)threadIdx.x;
            if (nb1 >= kFoldL1Blocks) {
                // full level-2 block: 32 rows, lanes 0-7 hold 4 rows each
                const bool act = lane < 8;
                const int64_t row0 = j2 * 32 + 4 * lane;
                LaneState<T, 4, 8, false> st;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    st.r.a[i] = act ? s2[0][4 * lane + i] : T(0);
                    st.r.b[i] = act ? s2[1][4 * lane + i] : T(1);
                    st.r.c[i] = act ? s2[2][4 * lane + i] : T(0);
                    st.r.d[i] = act ? s2[3][4 * lane + i] : T(0);
                }
                lane_leaf<T, 4, 8, false>(st, row0);
                lanes_tree<T, 4, 8, false>(st, lane & 7, row0);
                if (act) {
                    if (st.guard.tripped()) report_pivot(err, level + 2, row0);
                    if (lane == 0) store_block_eqs_keep(out2, j2, st.cur, keep != 0);
                }
            } else if (lane == 0) {
                // the level-2 tail block (2 nb1 rows, nb1 >= 1)
                RowGuard bad;
                const Eq2<T> q = leaf_smem<T, false>(s2[0], s2[1], s2[2], s2[3], (int)(2 * nb1), j2 * 32, bad);
                store_block_eqs_keep(out2, j2, q, keep != 0);
                report_pivot(err, level + 2, bad.bad);
            }
        }
    }
}

}  // namespace tpb
