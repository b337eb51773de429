// Internal launcher interface between the C-ABI layer and the sm_100a kernels.
// Every launcher is a template over the element type T (double or float) and
// is explicitly instantiated for both in tp_kernels.cu.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tpb {

constexpr int kStage1 = 0;  // reduce blocks -> next level's interface rows
constexpr int kStage3 = 1;  // expand blocks from the next level's solution
constexpr int kSolve = 2;   // whole system as one block: reduce, 2x2 root, expand
constexpr int kShard = 3;   // one shard of a multi-GPU solve: reduce, exchange the boundary
                            // pair with every peer over peer memory, top solve, expand
// Launch flag of a kernel that is a solve graph's only kernel: it resets the
// error word itself (CTA 0, before the first cluster / grid barrier, which
// every error report follows), so the graph needs no k_reset.
constexpr int kResetErr = 1;

constexpr int kFastThreads = 256;
constexpr int kGenericThreads = 256;
constexpr int kFinalThreads = 1024;   // k_generic CTA cap
constexpr int kFinalThreads2 = 512;   // k_final CTA
// Largest system the single-CTA finishing solve keeps in shared memory
// (32 B per FP64 row; 6144 rows = 192 KiB of the 227 KiB opt-in limit).
constexpr int64_t kFinalCap = 6144;
constexpr size_t kMaxDynSmem = 227 * 1024;
// Long-block path (k_split, tp_split.cuh): blocks longer than kSplitAbove rows
// are cut into chunks of <= kSplitRows rows by a split level.
constexpr int kSplitRows = 8;
constexpr int64_t kSplitAbove = 2048;
constexpr unsigned long long kNoError = ~0ULL;

template <class T>
struct SysPtrs {
    const T* sub;
    const T* diag;
    const T* sup;
    const T* rhs;
};
template <class T>
struct IfacePtrs {
    T* sub;
    T* diag;
    T* sup;
    T* rhs;
};

// Peer mailboxes of the fused multi-GPU solve (k_final<kShard>). Each rank owns
// one mailbox in its HBM, mapped into every peer (CUDA IPC over NVLink/NVSwitch).
// Entry (slot, p) = rank p's boundary pair {sub0, sub1, diag0, diag1, sup0,
// sup1, rhs0, rhs1} (FP64) + a 64-bit epoch flag, 128 B apart; the two slots
// alternate by epoch parity, so a rank one solve ahead never overwrites a pair
// a slower peer is still reading.
constexpr int kMaxPeers = 64;
constexpr int kMailboxEntryDoubles = 16;
constexpr int kExchangeLevel = 0x7FFF;  // err-word level of a peer-exchange timeout
// err-word level of a non-finite solution value (no pivot below the floor
// seen): the host then replays the reference's pivot order (diagnose_pivot)
constexpr int kNonFiniteLevel = 0x7FFE;
struct ShardLink {
    double* peers[kMaxPeers];   // every rank's mailbox, by rank (peers[rank] = own)
    double* own;                // this rank's mailbox
    unsigned long long* epoch;  // exchanges completed by this context
    int nranks;
    int rank;
};
inline size_t mailbox_bytes(int nranks) { return (size_t)2 * nranks * kMailboxEntryDoubles * sizeof(double); }

cudaError_t init_kernel_attributes();
cudaError_t launch_reset(unsigned long long* err, cudaStream_t st);
bool fast_shape(int64_t m, int* L, int* G);
int fast_rt_G(int64_t m);

template <class T>
cudaError_t launch_fast(int64_t m, bool vec, int mode, const SysPtrs<T>& sys, int64_t nblocks,
                        const IfacePtrs<T>& out, const T* xi, T* x, unsigned long long* err,
                        int level, cudaStream_t st);
template <class T>
cudaError_t launch_fast_rt(int64_t m, int mode, const SysPtrs<T>& sys, int64_t nblocks,
                           const IfacePtrs<T>& out, const T* xi, T* x, unsigned long long* err,
                           int level, int sms, cudaStream_t st);
size_t generic_smem_bytes(int threads, int G, int64_t blen, size_t elem);
template <class T>
cudaError_t launch_generic(int mode, int threads, int G, int grid, const SysPtrs<T>& sys,
                           int64_t row_base, int64_t blk_base, int64_t nblocks, int64_t blen,
                           const IfacePtrs<T>& out, const T* xi, T* x, unsigned long long* err,
                           int level, cudaStream_t st);
template <class T>
cudaError_t launch_final(int mode, const SysPtrs<T>& sys, int64_t n, const IfacePtrs<T>& out,
                         const T* xi, T* x, unsigned long long* err, int level, cudaStream_t st,
                         const ShardLink* link = nullptr);
// Level 0's Stage 1 with level 1's folded in (k_fast_s1fold, tp_fold.cuh).
// With out2 (fold2_fits: m2 == 32) level 2's Stage 1 is folded in as well.
bool fold_fits(int64_t m0, int64_t K0, int64_t n1, int64_t m1, int64_t K1);
bool fold2_fits(int64_t K1, int64_t n2, int64_t m2, int64_t K2);
template <class T>
cudaError_t launch_fold(int64_t m0, bool vec, const SysPtrs<T>& sys, int64_t K0, const IfacePtrs<T>& out0,
                        int64_t m1, int64_t K1, const IfacePtrs<T>& out1, const IfacePtrs<T>* out2,
                        unsigned long long* err, int level, cudaStream_t st);
// The deepest level fused with the finishing solve (k_level_final_cl):
// level_final_fits says whether a level of n rows in K blocks of m fits the
// cluster's shared memory; launch_level_final returns cudaErrorInvalidValue
// when it does not (the caller then runs the three-kernel form).
// mode kSolve (single system) or kShard (FP64: the shard's root pair goes
// through the peer exchange of `link`); cs = 8 forces the portable 8-CTA
// cluster (ranks sharing one GPU), 0 = the probed shape (16 where it fits).
bool level_final_fits(int64_t n, int64_t m, int64_t K, size_t elem, int cs = 0);
template <class T>
cudaError_t launch_level_final(const SysPtrs<T>& sys, int64_t n, int64_t m, int64_t K, const IfacePtrs<T>& iface,
                               T* x, unsigned long long* err, int level, cudaStream_t st, int mode = kSolve,
                               const ShardLink* link = nullptr, int cs = 0, int flags = 0);
// One split level (tp_split.cuh): nblocks blocks of blen rows starting at
// row_base, nsub chunks each, chunk pairs written from pair q_base on.
template <class T>
cudaError_t launch_split(int mode, const SysPtrs<T>& sys, int64_t row_base, int64_t nblocks, int64_t blen,
                         int64_t nsub, int64_t q_base, const IfacePtrs<T>& out, const T* xi, T* x,
                         unsigned long long* err, int level, cudaStream_t st);
// Reference-order sweeps (tp_split.cuh): reduce_block over make_plan(n, m)
// (first[j] = the block's failing pivot row or -1; jmin = atomicMin of the
// failing block indices; with eq8 != NULL the interface pairs and up-sweep
// vectors are stored) and thomas_solve's pivot scan.
template <class T>
cudaError_t launch_ref_sweep(const SysPtrs<T>& sys, int64_t n, int64_t m, int64_t K, int64_t* first,
                             unsigned long long* jmin, T* eq8, T* ua, T* ubeta, T* ugamma, T* udelta,
                             cudaStream_t st);
template <class T>
cudaError_t launch_ref_thomas(const SysPtrs<T>& sys, int64_t n, int64_t* out, cudaStream_t st);
// Whole-system solve on one co-resident grid (k_grid_solve, tp_grid.cu): a
// one-level policy whose rows fit the GPU's aggregate shared memory, one CTA
// per SM, one grid barrier. grid_fits says whether (n, m) fits; the launcher
// returns cudaErrorInvalidValue when it does not. scratch: kGridScratchBytes of device memory, zeroed once
// (the barrier counters reset themselves at the end of every launch).
constexpr int kGridBarrierLevel = 0x7FFD;  // err-word level of a grid-barrier timeout
constexpr int64_t kGridMaxChunk = 64;  // longest leaf chunk (rows)
constexpr int64_t kGridMinRows = 4;
constexpr size_t kGridDynSmem = 232448 - 6144;
constexpr size_t kGridScratchBytes = 256 + (8 * 256 + 8) * sizeof(double);  // counter, CTA pairs, root ends
inline int64_t plan_blocks_dev(int64_t n, int64_t m) {  // make_plan's block count, partition.hpp:30-49
    if (m >= n) return 1;
    int64_t leading = n / m;
    if (n % m <= 1) --leading;
    return leading + 1;
}
bool grid_fits(int64_t n, int64_t m, size_t elem, int sms);
template <class T>
cudaError_t launch_grid_solve(const SysPtrs<T>& sys, int64_t n, int64_t m, T* x, void* scratch,
                              unsigned long long* err, int level, int sms, cudaStream_t st, int mode = kSolve,
                              const ShardLink* link = nullptr, int flags = 0);
template <class T>
cudaError_t launch_gather_solve(const T* eqs, int nranks, int rank, T* x2, T* scratch,
                                unsigned long long* err, int level, cudaStream_t st);
template <class T>
cudaError_t launch_generate(int64_t n, int64_t row0, int64_t n_global, uint64_t seed, double delta,
                            T* sub, T* diag, T* sup, T* rhs, int sms, cudaStream_t st);
template <class T>
cudaError_t launch_residual(const SysPtrs<T>& sys, int64_t n, const T* x, unsigned long long* out,
                            int sms, cudaStream_t st);

}  // namespace tpb
