// C-ABI layer: context, level planner, CUDA-graph cache and the entry points
// declared in include/tridpart_b200.h (FP64 and FP32, as the reference's
// solve_partition<Real> template).
//
// The planner restates detail::solve_partition_level (partition.hpp:191-224):
//   level l with n_l < 4            -> finishing solve of that system      (:197)
//   else make_plan(n_l, sizes[l])   -> Stage 1, interface of 2*K_l rows    (:199-205)
//   l == depth                      -> finishing solve of the interface    (:208-211)
//   Stage 3 back up every level                                           (:213-222)
// The finishing solve runs on the device (single CTA, k_final); a final
// system larger than kFinalCap first gets extra device-internal partition
// levels (m = 32). Those do not change the policy, only how the
// thomas_solve(iface) of the reference is computed.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tridpart_b200.h"
#include "tp_kernels.h"
#include "tp_stage.h"

using tpb::IfacePtrs;
using tpb::SysPtrs;

namespace {

constexpr int64_t kInternalM = 32;
constexpr int64_t kFusedInternalM = 16;  // internal level absorbed by k_level_final_cl

void set_err(tp_error* err, tp_status code, const std::string& msg, int64_t row = -1, int32_t level = -1) {
    if (!err) return;
    err->code = code;
    err->row = row;
    err->level = level;
    std::snprintf(err->msg, sizeof(err->msg), "%s", msg.c_str());
}
void clear_err(tp_error* err) {
    if (!err) return;
    err->code = TP_OK;
    err->row = -1;
    err->level = -1;
    err->msg[0] = 0;
}

#define TP_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            set_err(err, TP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
            return TP_ERR_CUDA;                                                            \
        }                                                                                  \
    } while (0)

#define TP_NEED_CTX(ctx)                                          \
    do {                                                          \
        if (!(ctx)) {                                             \
            set_err(err, TP_ERR_INVALID_ARGUMENT, "ctx is NULL"); \
            return TP_ERR_INVALID_ARGUMENT;                       \
        }                                                         \
    } while (0)

// make_plan — partition.hpp:30-49 (block count only).
int64_t plan_blocks(int64_t n, int64_t m) {
    if (m >= n) return 1;
    int64_t leading = n / m;
    if (n % m <= 1) --leading;
    return leading + 1;
}

template <class T>
struct Level {
    int64_t n = 0;      // rows of this level's system
    int64_t m = 0;      // requested block size
    int64_t K = 0;      // blocks (make_plan)
    int64_t kfull = 0;  // blocks of exactly m rows
    int64_t tail = 0;   // length of the final block when != m (0 = none)
    bool internal = false;
    // long-block chain (tp_split.cuh): a split level cuts every block into
    // nsub (tail: nsub_tail) chunks and writes their E1/E2 pairs as a finer
    // system of out_rows rows; the level after it keeps the block boundaries
    bool split = false;
    int64_t nsub = 0, nsub_tail = 0;
    int64_t out_rows = 0;   // rows of the system this level writes (2K, or the finer system)
    int policy_level = -1;  // RecursionPolicy level this plan level belongs to (-1: device-internal)
    // bound pointers
    SysPtrs<T> in{};
    T* x_out = nullptr;    // solution of this level's system
    IfacePtrs<T> iface{};  // next level's system (out_rows rows)
    T* x_iface = nullptr;
};

template <class T>
struct Plan {
    std::vector<Level<T>> levels;
    int64_t n0 = 0, m0 = 0;  // the system and the policy's level-0 block size
    int32_t npol = 0;        // policy levels
    int64_t n_final = 0;
    SysPtrs<T> final_in{};
    T* final_x = nullptr;
    size_t ws_elems = 0;  // workspace, in elements of T
    int cs = 0;           // cluster shape of k_level_final_cl (0 = probed, 8 = portable)
};

inline size_t pad32(size_t v) { return (v + 31) & ~size_t(31); }

// A level whose blocks are too long for shared-memory staging becomes a chain
// of split levels ending in a level with the original block boundaries
// (tp_split.cuh): each split cuts every block into chunks of <= kSplitRows
// rows and hands the next level 2 rows per chunk.
inline bool needs_split(int64_t kfull, int64_t m, int64_t tail) {
    return (kfull > 0 && m > tpb::kSplitAbove) || tail > tpb::kSplitAbove + 1;
}

template <class T>
void push_chain(Plan<T>& p, Level<T> L, size_t& ws) {
    while (needs_split(L.kfull, L.m, L.tail)) {
        Level<T> S = L;
        S.split = true;
        S.nsub = L.kfull > 0 ? (L.m + tpb::kSplitRows - 1) / tpb::kSplitRows : 0;
        S.nsub_tail = L.tail > 0 ? (L.tail + tpb::kSplitRows - 1) / tpb::kSplitRows : 0;
        S.out_rows = 2 * (L.kfull * S.nsub + S.nsub_tail);
        ws += 5 * pad32((size_t)S.out_rows);
        p.levels.push_back(S);
        Level<T> M = L;
        M.n = S.out_rows;
        M.m = L.kfull > 0 ? 2 * S.nsub : 2 * S.nsub_tail;
        M.tail = 2 * S.nsub_tail;
        L = M;
    }
    L.out_rows = 2 * L.K;
    ws += 5 * pad32((size_t)L.out_rows);
    p.levels.push_back(L);
}

// fused = the plan is for solve_body, which runs the deepest level and the
// finishing solve as one kernel when that level fits k_level_final_cl: then
// the deepest interface may exceed kFinalCap (no device-internal level is
// added for it), and an oversized final system gets ONE fused internal level
// of m = 16 when that fits. The sharded paths keep n_final <= kFinalCap.
template <class T>
void build_plan(int64_t n, const int64_t* sizes, int32_t nsizes, Plan<T>& p, bool fused = false, int cs = 0) {
    p.levels.clear();
    p.cs = cs;
    p.n0 = n;
    p.m0 = nsizes > 0 ? sizes[0] : 0;
    p.npol = nsizes;
    int64_t cur = n;
    int lvl = 0;
    size_t ws = 0;
    while (nsizes > 0) {
        if (cur < 4) break;
        Level<T> L;
        L.n = cur;
        L.m = sizes[lvl];
        L.K = plan_blocks(cur, L.m);
        L.policy_level = lvl;
        const int64_t last_len = cur - (L.K - 1) * L.m;
        if (L.m >= cur) {
            L.kfull = (cur == L.m) ? 1 : 0;
            L.tail = (cur == L.m) ? 0 : cur;
        } else if (last_len == L.m) {
            L.kfull = L.K;
            L.tail = 0;
        } else {
            L.kfull = L.K - 1;
            L.tail = last_len;
        }
        push_chain(p, L, ws);
        cur = 2 * L.K;
        if (lvl == nsizes - 1) break;
        ++lvl;
    }
    // device-internal levels so the finishing solve fits one cluster
    const bool last_fused = fused && !p.levels.empty() && !p.levels.back().split &&
                            tpb::level_final_fits(p.levels.back().n, p.levels.back().m, p.levels.back().K, sizeof(T), cs);
    while (!last_fused && cur > tpb::kFinalCap) {
        Level<T> L;
        L.n = cur;
        L.m = kInternalM;
        if (fused && tpb::level_final_fits(cur, kFusedInternalM, plan_blocks(cur, kFusedInternalM), sizeof(T), cs))
            L.m = kFusedInternalM;
        L.K = plan_blocks(cur, L.m);
        const int64_t last_len = cur - (L.K - 1) * L.m;
        L.kfull = (last_len == L.m) ? L.K : L.K - 1;
        L.tail = (last_len == L.m) ? 0 : last_len;
        L.internal = true;
        L.out_rows = 2 * L.K;
        ws += 5 * pad32((size_t)(2 * L.K));
        p.levels.push_back(L);
        cur = 2 * L.K;
        if (L.m == kFusedInternalM) break;  // solved by k_level_final_cl
    }
    p.n_final = cur;
    p.ws_elems = ws;
}

template <class T>
void bind_plan(Plan<T>& p, const SysPtrs<T>& sys, T* x, void* ws) {
    SysPtrs<T> in = sys;
    T* xo = x;
    T* w = static_cast<T*>(ws);
    for (auto& L : p.levels) {
        L.in = in;
        L.x_out = xo;
        const size_t k2 = pad32((size_t)L.out_rows);
        L.iface.sub = w;
        L.iface.diag = w + k2;
        L.iface.sup = w + 2 * k2;
        L.iface.rhs = w + 3 * k2;
        L.x_iface = w + 4 * k2;
        w += 5 * k2;
        in = SysPtrs<T>{L.iface.sub, L.iface.diag, L.iface.sup, L.iface.rhs};
        xo = L.x_iface;
    }
    p.final_in = in;
    p.final_x = xo;
}

int generic_G(int64_t blen, int tmax) {
    int G = 1;
    while (G * 2 <= tmax && blen / (G * 2) >= 4) G *= 2;
    return G;
}

bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; }

}  // namespace

struct tp_obs_set;

struct tp_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t side = nullptr;  // tail-block branch
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t stream = nullptr;
    bool graphs = true;
    void* ws = nullptr;  // level workspace
    size_t ws_cap = 0;   // bytes
    unsigned long long* d_err = nullptr;
    unsigned long long* h_err = nullptr;
    unsigned long long* d_red = nullptr;  // residual / scratch words
    void* d_small = nullptr;              // shard scratch (x2 + gather scratch)
    void* d_grid = nullptr;               // k_grid_solve: barrier word + CTA pairs
    bool no_grid = false;                 // observer solves: keep the level path (interfaces in HBM)
    bool grid_on = true;                  // tp_ctx_set_grid / TPB_GRID
    int64_t grid_min = 80000;             // tp_ctx_set_grid / TPB_GRID_MIN
    // fused multi-GPU path (k_final<kShard>): own mailbox, peer links, epoch word
    void* mailbox = nullptr;
    int mailbox_ranks = 0;
    unsigned long long* d_epoch = nullptr;
    tpb::ShardLink link{};
    bool linked = false;
    bool link_shared = false;  // a peer's mailbox lives on this context's GPU
    int64_t link_gen = 0;
    std::vector<void*> ipc_opened;
    bool prepare_only = false;  // capture + instantiate the graph, do not launch
    tpb::Stager stager;         // pinned staging of pageable host buffers
    void* dsys = nullptr;                 // host-path staging (5 arrays)
    size_t dsys_cap = 0;                  // bytes
    int64_t last_launches = 0;
    std::string last_names;  // the last solve's kernels (Runner::names)
    // The last solve whose zero pivot tp_check_device_error / the synchronous
    // calls may have to locate in the reference's order (diagnose_pivot).
    struct LastSolve {
        int kind = 0;  // 0 none / not diagnosable, 1 solve_partition, 2 thomas_solve
        bool f32 = false;
        int64_t n = 0;
        std::vector<int64_t> sizes;
        const void* in[4] = {nullptr, nullptr, nullptr, nullptr};
        void* x = nullptr;
    } last;
    struct GraphEntry {
        std::vector<int64_t> key;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        std::string names;
        uint64_t stamp = 0;
    };
    std::vector<GraphEntry> gcache;
    uint64_t clock = 0;
};

namespace {


using KernelHook = void (*)(void* user, const char* name);

// k_grid_solve takes the rest of the solve from the shallowest plan level whose
// system fits the grid's shared memory (k = 0: the whole solve, e.g. config 2;
// k >= 1: the levels below Stage 1 of levels 0..k-1), for systems of
// >= ctx->grid_min rows (tp_ctx_set_grid; env TPB_GRID, TPB_GRID_MIN at context
// creation). Below ~8e4 rows the level path is faster: measured in-graph spans,
// tools/ab_grid_span.sh. Returns the plan level, or -1.
template <class T>
int grid_level(const tp_ctx* ctx, const Plan<T>& p) {
    if (!ctx->grid_on || ctx->no_grid) return -1;
    for (size_t k = 0; k < p.levels.size(); ++k) {
        const Level<T>& L = p.levels[k];
        if (L.n < ctx->grid_min || L.n < 4) return -1;  // deeper levels are smaller still
        // (a split level carries its level's original n and m: the grid takes
        // the original blocks, long ones as many chunks)
        if (tpb::grid_fits(L.n, L.m, sizeof(T), ctx->sms)) return (int)k;
    }
    return -1;
}

template <class T>
struct Runner {
    tp_ctx* ctx;
    cudaStream_t st;
    KernelHook hook = nullptr;
    void* hook_user = nullptr;
    int64_t launches = 0;
    cudaError_t status = cudaSuccess;

    std::string names;  // "what:Llevel" of every kernel, comma-separated (tp_ctx_last_kernels)
    void after(const char* what, int level) {
        ++launches;
        char name[32];
        std::snprintf(name, sizeof(name), "%s:L%d", what, level);
        if (!names.empty()) names += ',';
        names += name;
        if (hook) hook(hook_user, name);
    }
    void check(cudaError_t e) {
        if (e != cudaSuccess && status == cudaSuccess) status = e;
    }

    void main_part(const Level<T>& L, int level, int mode) {
        const bool s1 = (mode == tpb::kStage1);
        int fl, fg;
        if (L.split) {
            check(tpb::launch_split<T>(mode, L.in, 0, L.kfull, L.m, L.nsub, 0, L.iface, L.x_iface, L.x_out,
                                       ctx->d_err, level, st));
            after(s1 ? "stage1s" : "stage3s", level);
        } else if (tpb::fast_shape(L.m, &fl, &fg)) {
            const bool vec = aligned32(L.in.sub) && aligned32(L.in.diag) && aligned32(L.in.sup) &&
                             aligned32(L.in.rhs) && (s1 || aligned32(L.x_out));
            check(tpb::launch_fast<T>(L.m, vec, mode, L.in, L.kfull, L.iface, L.x_iface, L.x_out,
                                      ctx->d_err, level, st));
            after(s1 ? "stage1" : "stage3", level);
        } else if (tpb::fast_rt_G(L.m) > 0) {
            check(tpb::launch_fast_rt<T>(L.m, mode, L.in, L.kfull, L.iface, L.x_iface, L.x_out,
                                         ctx->d_err, level, ctx->sms, st));
            after(s1 ? "stage1r" : "stage3r", level);
        } else {
            const int NT = tpb::kGenericThreads;
            const int G = generic_G(L.m, NT);
            const int64_t bpc = NT / G;
            int64_t grid = (L.kfull + bpc - 1) / bpc;
            grid = std::min<int64_t>(grid, (int64_t)ctx->sms * 8);
            check(tpb::launch_generic<T>(mode, NT, G, (int)grid, L.in, 0, 0, L.kfull, L.m, L.iface,
                                         L.x_iface, L.x_out, ctx->d_err, level, st));
            after(s1 ? "stage1g" : "stage3g", level);
        }
    }
    void tail_part(const Level<T>& L, int level, int mode, cudaStream_t s) {
        if (L.split) {
            check(tpb::launch_split<T>(mode, L.in, L.kfull * L.m, 1, L.tail, L.nsub_tail, L.kfull * L.nsub, L.iface,
                                       L.x_iface, L.x_out, ctx->d_err, level, s));
            after(mode == tpb::kStage1 ? "stage1st" : "stage3st", level);
            return;
        }
        // short Stage-3 tails on one lane (no tree, no cross-lane barriers):
        // 4.8 -> 3.9 us for the 8-row tail on the critical path of C3 level 3;
        // Stage-1 tails run beside their main kernel and keep the 2-lane form
        const int G = (mode == tpb::kStage3 && L.tail <= 16) ? 1 : generic_G(L.tail, tpb::kGenericThreads);
        const int NT = std::max(32, G);
        check(tpb::launch_generic<T>(mode, NT, G, 1, L.in, L.kfull * L.m, L.kfull, 1, L.tail, L.iface,
                                     L.x_iface, L.x_out, ctx->d_err, level, s));
        after(mode == tpb::kStage1 ? "stage1t" : "stage3t", level);
    }

    // One level of Stage 1 or Stage 3. The tail block (make_plan's last block
    // when its length != m) is independent of the full blocks, so it runs on a
    // forked stream (a parallel branch of the captured graph) and joins before
    // the next dependent kernel. The instrumented path keeps them serial.
    void stage(const Level<T>& L, int level, int mode) {
        const bool fork = L.kfull > 0 && L.tail > 0 && hook == nullptr;
        if (fork) {
            check(cudaEventRecord(ctx->ev_fork, st));
            check(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            tail_part(L, level, mode, ctx->side);
            check(cudaEventRecord(ctx->ev_join, ctx->side));
            main_part(L, level, mode);
            check(cudaStreamWaitEvent(st, ctx->ev_join, 0));
            return;
        }
        if (L.kfull > 0) main_part(L, level, mode);
        if (L.tail > 0) tail_part(L, level, mode, st);
    }

    void final_solve(const Plan<T>& p) {
        check(tpb::launch_final<T>(tpb::kSolve, p.final_in, p.n_final, IfacePtrs<T>{}, nullptr, p.final_x,
                                   ctx->d_err, (int)p.levels.size(), st));
        after("final", (int)p.levels.size());
    }

    // The plan level the grid solve takes in this mode, or -1. Sharded (FP64):
    // not when a peer shares this GPU (every rank's grid kernel needs all SMs
    // while it waits for the others' pairs).
    int grid_level_for(const Plan<T>& p, int mode) const {
        if (mode == tpb::kSolve) return grid_level(ctx, p);
        if (mode == tpb::kShard && sizeof(T) == 8 && !ctx->link_shared) return grid_level(ctx, p);
        return -1;
    }

    // Whole solve: reset the error word, Stage 1 down, finish, Stage 3 up —
    // or, for a one-level policy that fits the grid's shared memory, the one
    // co-resident kernel k_grid_solve (tp_grid.cu).
    // When the whole solve is one kernel (the grid solve from level 0, or the
    // fused deepest level of a one-level plan) that kernel resets the error
    // word itself and the graph has no k_reset node.
    bool single_kernel(const Plan<T>& p, int mode) const {
        const int gk = grid_level_for(p, mode);
        if (gk >= 0) return gk == 0;
        const size_t nl = p.levels.size();
        return nl == 1 && !p.levels[0].split &&
               tpb::level_final_fits(p.levels[0].n, p.levels[0].m, p.levels[0].K, sizeof(T), p.cs);
    }
    void solve(const Plan<T>& p) {
        if (single_kernel(p, tpb::kSolve)) {
            solve_body(p, tpb::kSolve, tpb::kResetErr);
            return;
        }
        check(tpb::launch_reset(ctx->d_err, st));
        ++launches;  // k_reset: counted, not timed by the profile hook
        solve_body(p, tpb::kSolve);
    }
    // Stage 1 of levels [0, top): level 1's (and level 2's) folded into level
    // 0's kernel (k_fast_s1fold) where the shapes allow, the rest per level.
    void stage1_down(const Plan<T>& p, size_t top) {
        size_t l = 0;
        if (top >= 2) {  // level 1's Stage 1 folded into level 0's (k_fast_s1fold)
            const Level<T>& A = p.levels[0];
            const Level<T>& B = p.levels[1];
            if (!A.split && !B.split && A.tail == 0 && A.kfull == A.K && B.tail == 0 &&
                tpb::fold_fits(A.m, A.K, B.n, B.m, B.K)) {
                const bool vec = aligned32(A.in.sub) && aligned32(A.in.diag) && aligned32(A.in.sup) &&
                                 aligned32(A.in.rhs);
                // level 2 too when its blocks are the fold CTAs' tiles (m2 = 32)
                const bool f2 = top >= 3 && !p.levels[2].split && tpb::fold2_fits(B.K, p.levels[2].n, p.levels[2].m, p.levels[2].K);
                check(tpb::launch_fold<T>(A.m, vec, A.in, A.K, A.iface, B.m, B.K, B.iface,
                                          f2 ? &p.levels[2].iface : nullptr, ctx->d_err, 0, st));
                after(f2 ? "stage1_fold2" : "stage1_fold", 0);
                l = f2 ? 3 : 2;
            }
        }
        for (; l < top; ++l) stage(p.levels[l], (int)l, tpb::kStage1);
    }

    // The deepest level and the finishing solve run as one cluster kernel when
    // that level fits the cluster's shared memory (k_level_final_cl); its
    // interface is still written out (for the observer), never read back.
    // mode kShard (sharded plan, fused = true): the same graph with the peer
    // exchange at the root of the deepest level (k_level_final_cl<kShard>) or
    // of the finishing solve (k_final<kShard>).
    // flags = kResetErr: the plan is one kernel, which resets the error word.
    void solve_body(const Plan<T>& p, int mode = tpb::kSolve, int flags = 0) {
        const int gk = grid_level_for(p, mode);
        if (gk >= 0) {  // Stage 1 down to level gk, the grid solve from there, Stage 3 up
            stage1_down(p, (size_t)gk);
            const Level<T>& G = p.levels[(size_t)gk];
            check(tpb::launch_grid_solve<T>(G.in, G.n, G.m, G.x_out, ctx->d_grid, ctx->d_err, gk, ctx->sms, st, mode,
                                            mode == tpb::kShard ? &ctx->link : nullptr, flags));
            after(mode == tpb::kShard ? "grid_exchange" : "grid_solve", gk);
            for (int l = gk; l-- > 0;) stage(p.levels[(size_t)l], l, tpb::kStage3);
            return;
        }
        const size_t nl = p.levels.size();
        const bool fuse = nl > 0 && !p.levels.back().split &&
                          tpb::level_final_fits(p.levels.back().n, p.levels.back().m, p.levels.back().K, sizeof(T),
                                                p.cs);
        const size_t top = fuse ? nl - 1 : nl;
        stage1_down(p, top);
        if (fuse) {
            const Level<T>& L = p.levels.back();
            check(tpb::launch_level_final<T>(L.in, L.n, L.m, L.K, L.iface, L.x_out, ctx->d_err, (int)top, st, mode,
                                             mode == tpb::kShard ? &ctx->link : nullptr, p.cs, top == 0 ? flags : 0));
            after(mode == tpb::kShard ? "level_exchange" : "level_final", (int)top);
        } else if (mode == tpb::kShard) {
            check(tpb::launch_final<T>(tpb::kShard, p.final_in, p.n_final, IfacePtrs<T>{}, nullptr, p.final_x,
                                       ctx->d_err, (int)p.levels.size(), st, &ctx->link));
            after("shard_exchange", (int)p.levels.size());
        } else {
            final_solve(p);
        }
        for (size_t l = top; l-- > 0;) stage(p.levels[l], (int)l, tpb::kStage3);
    }

    // Sharded halves.
    void shard_reduce(const Plan<T>& p, T* eq8) {
        check(tpb::launch_reset(ctx->d_err, st));
        ++launches;  // k_reset: counted, not timed by the profile hook
        stage1_down(p, p.levels.size());
        IfacePtrs<T> o{eq8, eq8 + 2, eq8 + 4, eq8 + 6};
        check(tpb::launch_final<T>(tpb::kStage1, p.final_in, p.n_final, o, nullptr, nullptr, ctx->d_err,
                                   (int)p.levels.size(), st));
        after("shard_reduce", (int)p.levels.size());
    }
    // Fused multi-GPU solve of one shard: the single-GPU graph (folded Stage 1,
    // the deepest level fused with the finishing solve, Stage 3 up) with the
    // peer exchange and the top solve at the root of the deepest level.
    void shard_solve(const Plan<T>& p) {
        if (single_kernel(p, tpb::kShard)) {
            solve_body(p, tpb::kShard, tpb::kResetErr);
            return;
        }
        check(tpb::launch_reset(ctx->d_err, st));
        ++launches;  // k_reset: counted, not timed by the profile hook
        solve_body(p, tpb::kShard);
    }
    void shard_finish(const Plan<T>& p, const T* eq_all, int nranks, int rank) {
        T* x2 = static_cast<T*>(ctx->d_small);
        T* scratch = x2 + 32;
        check(tpb::launch_gather_solve<T>(eq_all, nranks, rank, x2, scratch, ctx->d_err,
                                          (int)p.levels.size() + 1, st));
        after("gather_solve", (int)p.levels.size() + 1);
        check(tpb::launch_final<T>(tpb::kStage3, p.final_in, p.n_final, IfacePtrs<T>{}, x2, p.final_x,
                                   ctx->d_err, (int)p.levels.size(), st));
        after("shard_expand", (int)p.levels.size());
        for (size_t l = p.levels.size(); l-- > 0;) stage(p.levels[l], (int)l, tpb::kStage3);
    }
};

tp_status validate_policy(int64_t n, const int64_t* sizes, int32_t nsizes, tp_error* err) {
    // RecursionPolicy::valid — partition.hpp:181-186, checked first (:239)
    if (nsizes < 1 || sizes == nullptr) {
        set_err(err, TP_ERR_INVALID_SIZE, "invalid recursion policy");
        return TP_ERR_INVALID_SIZE;
    }
    for (int i = 0; i < nsizes; ++i)
        if (sizes[i] < 2) {
            set_err(err, TP_ERR_INVALID_SIZE, "invalid recursion policy");
            return TP_ERR_INVALID_SIZE;
        }
    if (n <= 0) {  // :240
        set_err(err, TP_ERR_INVALID_SIZE, "empty system");
        return TP_ERR_INVALID_SIZE;
    }
    return TP_OK;
}

tp_status validate(const void* a, const void* b, const void* c, const void* d, int64_t n,
                   const int64_t* sizes, int32_t nsizes, const void* x, tp_error* err) {
    tp_status s = validate_policy(n, sizes, nsizes, err);
    if (s != TP_OK) return s;
    if (!a || !b || !c || !d || !x) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null array pointer");
        return TP_ERR_INVALID_ARGUMENT;
    }
    return TP_OK;
}

void drop_graphs(tp_ctx* ctx) {
    for (auto& g : ctx->gcache) cudaGraphExecDestroy(g.exec);
    ctx->gcache.clear();
}

tp_status ensure_ws(tp_ctx* ctx, size_t bytes, tp_error* err) {
    if (bytes <= ctx->ws_cap) return TP_OK;
    drop_graphs(ctx);  // growing the workspace invalidates every captured graph
    if (ctx->ws) cudaFree(ctx->ws);
    ctx->ws = nullptr;
    ctx->ws_cap = 0;
    const size_t want = bytes + bytes / 8 + 8192;
    TP_CUDA(cudaMalloc(&ctx->ws, want));
    ctx->ws_cap = want;
    return TP_OK;
}

// host-path staging: five arrays of n elements (sub, diag, super, rhs, x)
template <class T>
tp_status ensure_dsys(tp_ctx* ctx, int64_t n, T** arrays, tp_error* err) {
    const size_t rows = pad32((size_t)n);
    const size_t bytes = 5 * rows * sizeof(T);
    if (bytes > ctx->dsys_cap) {
        drop_graphs(ctx);
        if (ctx->dsys) cudaFree(ctx->dsys);
        ctx->dsys = nullptr;
        ctx->dsys_cap = 0;
        TP_CUDA(cudaMalloc(&ctx->dsys, bytes));
        ctx->dsys_cap = bytes;
    }
    T* base = static_cast<T*>(ctx->dsys);
    for (int i = 0; i < 5; ++i) arrays[i] = base + i * rows;
    return TP_OK;
}

template <class T>
tp_status diagnose_pivot(tp_ctx* ctx, int64_t dev_row, int32_t dev_level, tp_error* err);

tp_status decode_device_error(tp_ctx* ctx, tp_error* err) {
    const unsigned long long code = *ctx->h_err;
    if (code == tpb::kNoError) return TP_OK;
    const int32_t level = (int32_t)(code >> 48);
    const int64_t row = (int64_t)(code & 0xFFFFFFFFFFFFULL);
    if (level == tpb::kGridBarrierLevel) {
        set_err(err, TP_ERR_CUDA, "grid solve: CTA " + std::to_string(row) + " timed out at the grid barrier", row, -1);
        return TP_ERR_CUDA;
    }
    if (level == tpb::kExchangeLevel) {
        set_err(err, TP_ERR_NCCL, "peer exchange timed out waiting for rank " + std::to_string(row), row, -1);
        return TP_ERR_NCCL;
    }
    // a pivot below the floor, or (kNonFiniteLevel) a non-finite solution
    // value: locate the reference's zero pivot, if its order meets one
    if (ctx->last.kind != 0)
        return ctx->last.f32 ? diagnose_pivot<float>(ctx, row, level, err)
                             : diagnose_pivot<double>(ctx, row, level, err);
    if (level == tpb::kNonFiniteLevel) return TP_OK;  // the reference throws nothing either
    set_err(err, TP_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(row), row, level);
    return TP_ERR_ZERO_PIVOT;
}

// Runs `fn(runner)` directly or through a cached CUDA graph keyed by `key`.
template <class T, class Fn>
tp_status run_maybe_graph(tp_ctx* ctx, cudaStream_t st, const std::vector<int64_t>& key, Fn&& fn,
                          tp_error* err) {
    if (!ctx->graphs) {
        Runner<T> r{ctx, st};
        fn(r);
        ctx->last_launches = r.launches;
        ctx->last_names = r.names;
        if (r.status != cudaSuccess) {
            set_err(err, TP_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(r.status));
            return TP_ERR_CUDA;
        }
        return TP_OK;
    }
    for (auto& g : ctx->gcache) {
        if (g.key == key) {
            g.stamp = ++ctx->clock;
            if (!ctx->prepare_only) TP_CUDA(cudaGraphLaunch(g.exec, st));
            ctx->last_launches = g.launches;
            ctx->last_names = g.names;
            return TP_OK;
        }
    }
    cudaStream_t cap = st;
    bool own_cap = false;
    if (st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread) {
        // the legacy stream cannot be captured: capture on a private stream
        TP_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        own_cap = true;
    }
    static const bool dbg = getenv("TPB_DEBUG_GRAPH") != nullptr;
    auto now_ms = [] { return std::chrono::duration<double, std::milli>(
                           std::chrono::steady_clock::now().time_since_epoch()).count(); };
    const double t0 = dbg ? now_ms() : 0;
    TP_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    Runner<T> r{ctx, cap};
    fn(r);
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(cap, &graph);
    const double t1 = dbg ? now_ms() : 0;
    if (r.status != cudaSuccess || ce != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        if (own_cap) cudaStreamDestroy(cap);
        set_err(err, TP_ERR_CUDA,
                std::string("graph capture: ") +
                    cudaGetErrorString(r.status != cudaSuccess ? r.status : ce));
        return TP_ERR_CUDA;
    }
    if (own_cap) cudaStreamDestroy(cap);
    cudaGraphExec_t exec = nullptr;
    cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    const double t2 = dbg ? now_ms() : 0;
    if (ie != cudaSuccess) {
        set_err(err, TP_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
        return TP_ERR_CUDA;
    }
    if (ctx->gcache.size() >= 16) {
        auto it = std::min_element(ctx->gcache.begin(), ctx->gcache.end(),
                                   [](const auto& x, const auto& y) { return x.stamp < y.stamp; });
        cudaGraphExecDestroy(it->exec);
        ctx->gcache.erase(it);
    }
    tp_ctx::GraphEntry ge;
    ge.key = key;
    ge.exec = exec;
    ge.launches = r.launches;
    ge.names = r.names;
    ge.stamp = ++ctx->clock;
    ctx->gcache.push_back(ge);
    ctx->last_launches = r.launches;
    ctx->last_names = r.names;
    if (!ctx->prepare_only) TP_CUDA(cudaGraphLaunch(exec, st));
    if (dbg)
        std::fprintf(stderr, "[tpb graph] capture %.3f ms, instantiate %.3f ms, launch %.3f ms (%lld kernels)\n",
                     t1 - t0, t2 - t1, now_ms() - t2, (long long)r.launches);
    return TP_OK;
}

// A solve graph with the grid solve whose capture or launch fails (the
// cooperative launch cannot make every CTA resident: fewer SMs available than
// the device reports, e.g. under MPS limits) is retried once on the level
// path, and the context keeps the level path from then on.
template <class T, class Fn>
tp_status run_with_grid_fallback(tp_ctx* ctx, cudaStream_t st, std::vector<int64_t> key, const Plan<T>& p, Fn&& fn,
                                 tp_error* err) {
    const bool grid = grid_level(ctx, p) >= 0;
    tp_status s = run_maybe_graph<T>(ctx, st, key, fn, err);
    if (s != TP_ERR_CUDA || !grid) return s;
    cudaGetLastError();  // clear the launch error
    ctx->grid_on = false;
    drop_graphs(ctx);
    key.push_back(-2);  // a distinct graph-cache entry for the level-path graph
    clear_err(err);
    return run_maybe_graph<T>(ctx, st, key, fn, err);
}

template <class T>
std::vector<int64_t> make_key(int64_t tag, int64_t n, const int64_t* sizes, int32_t nsizes,
                              std::initializer_list<const void*> ptrs, int64_t extra = 0) {
    std::vector<int64_t> k;
    k.push_back(tag * 16 + (int64_t)sizeof(T));
    k.push_back(n);
    k.push_back(extra);
    for (int i = 0; i < nsizes; ++i) k.push_back(sizes[i]);
    k.push_back(-1);
    for (const void* p : ptrs) k.push_back((int64_t) reinterpret_cast<uintptr_t>(p));
    return k;
}

cudaStream_t pick_stream(tp_ctx* ctx, void* s) {
    return s ? static_cast<cudaStream_t>(s) : ctx->stream;
}

// ------------------------------------------------------------ implementations
template <class T>
tp_status solve_dev(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs, int64_t n,
                    const int64_t* sizes, int32_t nsizes, T* x, void* stream, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    tp_status s = validate(sub, diag, super, rhs, n, sizes, nsizes, x, err);
    if (s != TP_OK) return s;
    TP_CUDA(cudaSetDevice(ctx->device));
    Plan<T> p;
    build_plan(n, sizes, nsizes, p, true);
    s = ensure_ws(ctx, p.ws_elems * sizeof(T), err);
    if (s != TP_OK) return s;
    bind_plan(p, SysPtrs<T>{sub, diag, super, rhs}, x, ctx->ws);
    const cudaStream_t st = pick_stream(ctx, stream);
    ctx->last.kind = 1;
    ctx->last.f32 = sizeof(T) == 4;
    ctx->last.n = n;
    ctx->last.sizes.assign(sizes, sizes + nsizes);
    ctx->last.in[0] = sub;
    ctx->last.in[1] = diag;
    ctx->last.in[2] = super;
    ctx->last.in[3] = rhs;
    ctx->last.x = x;
    auto key = make_key<T>(1, n, sizes, nsizes, {sub, diag, super, rhs, x, ctx->ws}, ctx->no_grid ? 1 : 0);
    return run_with_grid_fallback<T>(ctx, st, key, p, [&](Runner<T>& r) { r.solve(p); }, err);
}

// A solve reported a zero pivot (the device error word; dev_row / dev_level
// are the device's own, in plan-level numbering). Locate it as the reference
// would: replay detail::solve_partition_level's checks in ITS order with ITS
// arithmetic (k_ref_sweep / k_ref_thomas, tp_split.cuh) — level by level,
// block by block, up-sweep then down-sweep — on the level systems this solve
// left in HBM (level 0 = the input, level l = the interface the device
// assembled from level l-1). The first failing check gives ZeroPivotError's
// row and the level whose system it indexes (0 = input; depth+1 = the
// interface thomas_solve finishes). The reference's back_substitute pivots
// are its up-sweep pivots, so Stage 3 never fails first. When no
// reference-order check fails: a device pivot below the floor (the chunked
// elimination met one the sequential sweeps do not) keeps the device's own
// report; mere non-finite values return TP_OK, as the reference would.
template <class T>
tp_status diagnose_pivot(tp_ctx* ctx, int64_t dev_row, int32_t dev_level, tp_error* err) {
    const auto& ls = ctx->last;
    Plan<T> p;
    const int32_t npol = ls.kind == 1 ? (int32_t)ls.sizes.size() : 0;
    build_plan(ls.n, ls.sizes.data(), npol, p, true);
    bind_plan(p, SysPtrs<T>{(const T*)ls.in[0], (const T*)ls.in[1], (const T*)ls.in[2], (const T*)ls.in[3]},
              (T*)ls.x, ctx->ws);
    const cudaStream_t st = ctx->own;
    if (grid_level(ctx, p) >= 0) {
        // k_grid_solve keeps its levels' interfaces on chip: assemble them now
        // (the same Stage-1 kernels and arithmetic as the level path)
        Runner<T> r{ctx, st};
        r.stage1_down(p, p.levels.size());
        TP_CUDA(r.status);
        TP_CUDA(cudaStreamSynchronize(st));
    }
    int64_t kmax = 1;
    for (const auto& L : p.levels) kmax = std::max(kmax, L.K);
    void* scratch = nullptr;
    TP_CUDA(cudaMalloc(&scratch, (size_t)(kmax + 2) * sizeof(int64_t)));
    int64_t* first = static_cast<int64_t*>(scratch);
    unsigned long long* word = reinterpret_cast<unsigned long long*>(first + kmax);
    auto fail = [&](int64_t row, int32_t level) {
        cudaFree(scratch);
        set_err(err, TP_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(row), row, level);
        return TP_ERR_ZERO_PIVOT;
    };
    auto thomas_row = [&](const SysPtrs<T>& sys, int64_t n, int64_t* row) -> cudaError_t {
        cudaError_t e = tpb::launch_ref_thomas<T>(sys, n, first, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(row, first, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        return e;
    };
    SysPtrs<T> cur{(const T*)ls.in[0], (const T*)ls.in[1], (const T*)ls.in[2], (const T*)ls.in[3]};
    int64_t cn = ls.n;
    bool finished = false;  // a level below 4 rows ended the recursion (partition.hpp:197)
    cudaError_t e = cudaSuccess;
    int32_t l = 0;
    for (; l < npol && e == cudaSuccess; ++l) {
        int64_t row = -1;
        if (cn < 4) {
            e = thomas_row(cur, cn, &row);
            if (e == cudaSuccess && row >= 0) return fail(row, l);
            finished = true;
            break;
        }
        const int64_t m = ls.sizes[(size_t)l];
        const int64_t K = plan_blocks(cn, m);
        unsigned long long jmin = ~0ULL;
        e = cudaMemsetAsync(word, 0xFF, sizeof(unsigned long long), st);
        if (e == cudaSuccess)
            e = tpb::launch_ref_sweep<T>(cur, cn, m, K, first, word, nullptr, nullptr, nullptr, nullptr, nullptr, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&jmin, word, sizeof(jmin), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e == cudaSuccess && jmin != ~0ULL) {
            e = cudaMemcpy(&row, first + jmin, sizeof(int64_t), cudaMemcpyDeviceToHost);
            if (e == cudaSuccess) return fail(row, l);
        }
        // the interface this policy level assembled: the next system
        const Level<T>* lv = nullptr;
        for (const auto& L : p.levels)
            if (L.policy_level == l && !L.split) lv = &L;
        if (lv == nullptr) break;
        cur = SysPtrs<T>{lv->iface.sub, lv->iface.diag, lv->iface.sup, lv->iface.rhs};
        cn = 2 * K;
    }
    if (e == cudaSuccess && !finished) {  // thomas_solve(iface) of the deepest level (:208-211), or of the input
        int64_t row = -1;
        e = thomas_row(cur, cn, &row);
        if (e == cudaSuccess && row >= 0) return fail(row, npol);
    }
    cudaFree(scratch);
    if (e != cudaSuccess) {
        set_err(err, TP_ERR_CUDA, std::string("zero-pivot diagnosis: ") + cudaGetErrorString(e));
        return TP_ERR_CUDA;
    }
    // no reference-order check fails. Only non-finite values (a singular
    // system whose pivots stayed above the floor in both orders): the
    // reference returns its x without an exception, so does this call.
    if (dev_level == tpb::kNonFiniteLevel) return TP_OK;
    // A device pivot below the floor: keep the device's report (a result
    // computed through it is not returned), on the policy level its plan
    // level belongs to
    int32_t level = npol;
    if (dev_level >= 0 && (size_t)dev_level < p.levels.size() && p.levels[(size_t)dev_level].policy_level >= 0)
        level = p.levels[(size_t)dev_level].policy_level;
    set_err(err, TP_ERR_ZERO_PIVOT,
            "zero pivot at row " + std::to_string(dev_row) + " (device elimination order)", dev_row, level);
    return TP_ERR_ZERO_PIVOT;
}

// H2D of the four arrays into the context's staging buffers, `body(device
// arrays)` on the context stream, D2H of x, synchronise, decode zero pivots.
// With `async`, everything is enqueued on `st` and the call returns at once
// (host buffers should be pinned); zero pivots then surface through
// tp_check_device_error after the caller synchronises.
template <class T, class Body>
tp_status host_roundtrip(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs,
                         int64_t n, T* x, Body&& body, tp_error* err, cudaStream_t stream = nullptr,
                         bool async = false) {
    T* d[5];
    tp_status s = ensure_dsys<T>(ctx, n, d, err);
    if (s != TP_OK) return s;
    const cudaStream_t st = stream ? stream : ctx->stream;
    const size_t bytes = (size_t)n * sizeof(T);
    // pinned buffers: direct DMA; pageable ones (synchronous calls): staged
    // through the context's pinned chunks by host threads (tp_stage.h)
    const T* in[4] = {sub, diag, super, rhs};
    for (int i = 0; i < 4; ++i) {
        if (async || tpb::is_pinned_host(in[i]))
            TP_CUDA(cudaMemcpyAsync(d[i], in[i], bytes, cudaMemcpyHostToDevice, st));
        else
            TP_CUDA(ctx->stager.h2d(d[i], in[i], bytes, st));
    }
    s = body(d, st);
    if (s != TP_OK) return s;
    if (async || tpb::is_pinned_host(x))
        TP_CUDA(cudaMemcpyAsync(x, d[4], bytes, cudaMemcpyDeviceToHost, st));
    else
        TP_CUDA(ctx->stager.d2h(x, d[4], bytes, st));
    if (async) return TP_OK;
    TP_CUDA(cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    TP_CUDA(cudaStreamSynchronize(st));
    return decode_device_error(ctx, err);
}

// Host buffers, asynchronous on `stream`: H2D, the device solve and D2H are
// enqueued and the call returns. Two contexts on two streams let the D2H of
// one solve overlap the H2D of the next (PCIe is full duplex).
template <class T>
tp_status solve_host_async(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs,
                           int64_t n, const int64_t* sizes, int32_t nsizes, T* x, void* stream,
                           tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    tp_status s = validate(sub, diag, super, rhs, n, sizes, nsizes, x, err);
    if (s != TP_OK) return s;
    TP_CUDA(cudaSetDevice(ctx->device));
    const cudaStream_t st = pick_stream(ctx, stream);
    return host_roundtrip<T>(ctx, sub, diag, super, rhs, n, x,
                             [&](T** d, cudaStream_t s2) {
                                 return solve_dev<T>(ctx, d[0], d[1], d[2], d[3], n, sizes, nsizes,
                                                     d[4], s2, err);
                             },
                             err, st, true);
}

template <class T>
tp_status solve_host(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs, int64_t n,
                     const int64_t* sizes, int32_t nsizes, T* x, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    tp_status s = validate(sub, diag, super, rhs, n, sizes, nsizes, x, err);
    if (s != TP_OK) return s;
    TP_CUDA(cudaSetDevice(ctx->device));
    return host_roundtrip<T>(ctx, sub, diag, super, rhs, n, x,
                             [&](T** d, cudaStream_t st) {
                                 return solve_dev<T>(ctx, d[0], d[1], d[2], d[3], n, sizes, nsizes,
                                                     d[4], st, err);
                             },
                             err);
}

template <class T>
tp_status solve_observe(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs,
                        int64_t n, const int64_t* sizes, int32_t nsizes, T* x,
                        void (*emit)(int64_t, int64_t, const T*, const T*, const T*, const T*, void*),
                        void* user, tp_error* err) {
    // the observer reads every level's interface back: keep the level path
    ctx->no_grid = emit != nullptr;
    tp_status s = solve_host<T>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, err);
    ctx->no_grid = false;
    if (emit == nullptr || (s != TP_OK && s != TP_ERR_ZERO_PIVOT)) return s;
    // the reference calls the observer after each level's assembly
    // (partition.hpp:205-206): a zero pivot in level l's Stage 1 (or in the
    // finishing thomas_solve, l = depth + 1) comes after levels 0 .. l-1
    const int32_t upto = s == TP_OK ? nsizes : (err ? err->level : 0);
    const tp_error saved = err ? *err : tp_error{};
    T* d[5];
    tp_status s2 = ensure_dsys<T>(ctx, n, d, err);  // same buffers the solve used
    if (s2 != TP_OK) return s2;
    Plan<T> p;
    build_plan(n, sizes, nsizes, p, true);
    bind_plan(p, SysPtrs<T>{d[0], d[1], d[2], d[3]}, d[4], ctx->ws);
    std::vector<T> h;
    for (size_t l = 0; l < p.levels.size(); ++l) {
        const Level<T>& L = p.levels[l];
        if (L.internal) break;  // device-internal levels are not part of the policy
        if (L.split || L.policy_level >= upto) continue;
        const int64_t n2 = 2 * L.K;
        h.resize((size_t)(4 * n2));
        TP_CUDA(cudaMemcpy(h.data(), L.iface.sub, n2 * sizeof(T), cudaMemcpyDeviceToHost));
        TP_CUDA(cudaMemcpy(h.data() + n2, L.iface.diag, n2 * sizeof(T), cudaMemcpyDeviceToHost));
        TP_CUDA(cudaMemcpy(h.data() + 2 * n2, L.iface.sup, n2 * sizeof(T), cudaMemcpyDeviceToHost));
        TP_CUDA(cudaMemcpy(h.data() + 3 * n2, L.iface.rhs, n2 * sizeof(T), cudaMemcpyDeviceToHost));
        emit((int64_t)L.policy_level, n2, h.data(), h.data() + n2, h.data() + 2 * n2, h.data() + 3 * n2, user);
    }
    if (err) *err = saved;
    return s;
}

// thomas_solve: no policy levels, only device-internal ones (large n) + finish.
template <class T>
tp_status thomas_host(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs, int64_t n,
                      T* x, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    if (n <= 0) {
        set_err(err, TP_ERR_INVALID_SIZE, "empty system");
        return TP_ERR_INVALID_SIZE;
    }
    if (!sub || !diag || !super || !rhs || !x) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null array pointer");
        return TP_ERR_INVALID_ARGUMENT;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    return host_roundtrip<T>(
        ctx, sub, diag, super, rhs, n, x,
        [&](T** d, cudaStream_t st) -> tp_status {
            Plan<T> p;
            build_plan(n, nullptr, 0, p, true);
            tp_status s2 = ensure_ws(ctx, p.ws_elems * sizeof(T), err);
            if (s2 != TP_OK) return s2;
            bind_plan(p, SysPtrs<T>{d[0], d[1], d[2], d[3]}, d[4], ctx->ws);
            ctx->last.kind = 2;
            ctx->last.f32 = sizeof(T) == 4;
            ctx->last.n = n;
            ctx->last.sizes.clear();
            for (int i = 0; i < 4; ++i) ctx->last.in[i] = d[i];
            ctx->last.x = d[4];
            auto key = make_key<T>(2, n, nullptr, 0, {d[0], d[1], d[2], d[3], d[4], ctx->ws});
            return run_with_grid_fallback<T>(ctx, st, key, p, [&](Runner<T>& r) { r.solve(p); }, err);
        },
        err);
}

template <class T>
tp_status residual_dev(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs, int64_t n,
                       const T* x, double* out, void* stream, tp_error* err) {
    clear_err(err);
    if (!ctx || !out || !sub || !diag || !super || !rhs || !x) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    // on the caller's stream (NULL = the context's): ordered after the solve
    // or generator that produced x on that stream
    const cudaStream_t st = pick_stream(ctx, stream);
    TP_CUDA(cudaMemsetAsync(ctx->d_red, 0, 2 * sizeof(unsigned long long), st));
    TP_CUDA(tpb::launch_residual<T>(SysPtrs<T>{sub, diag, super, rhs}, n, x, ctx->d_red, ctx->sms, st));
    unsigned long long h[2];
    TP_CUDA(cudaMemcpyAsync(h, ctx->d_red, sizeof(h), cudaMemcpyDeviceToHost, st));
    TP_CUDA(cudaStreamSynchronize(st));
    double num, den;
    std::memcpy(&num, &h[0], sizeof(double));
    std::memcpy(&den, &h[1], sizeof(double));
    if (den < 1.0) den = 1.0;
    *out = num / den;
    return TP_OK;
}

template <class T>
tp_status shard_reduce(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs,
                       int64_t n_local, const int64_t* sizes, int32_t nsizes, T* eq8_dev, void* stream,
                       tp_error* err) {
    clear_err(err);
    if (!ctx || !eq8_dev) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    tp_status s = validate(sub, diag, super, rhs, n_local, sizes, nsizes, eq8_dev, err);
    if (s != TP_OK) return s;
    if (n_local < 2) {
        set_err(err, TP_ERR_INVALID_SIZE, "a shard needs at least 2 rows");
        return TP_ERR_INVALID_SIZE;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    Plan<T> p;
    build_plan(n_local, sizes, nsizes, p);
    s = ensure_ws(ctx, p.ws_elems * sizeof(T), err);
    if (s != TP_OK) return s;
    bind_plan(p, SysPtrs<T>{sub, diag, super, rhs}, (T*)nullptr, ctx->ws);
    const cudaStream_t st = pick_stream(ctx, stream);
    ctx->last.kind = 0;
    auto key = make_key<T>(3, n_local, sizes, nsizes, {sub, diag, super, rhs, eq8_dev, ctx->ws});
    return run_maybe_graph<T>(ctx, st, key, [&](Runner<T>& r) { r.shard_reduce(p, eq8_dev); }, err);
}

template <class T>
tp_status shard_finish(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs,
                       int64_t n_local, const int64_t* sizes, int32_t nsizes, const T* eq_all_dev,
                       int32_t nranks, int32_t rank, T* x_dev, void* stream, tp_error* err) {
    clear_err(err);
    if (!ctx || !eq_all_dev) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    // d_small holds 32 + 4*nranks elements of scratch (4096 bytes)
    if (nranks < 1 || nranks > 120 || rank < 0 || rank >= nranks) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "bad rank / nranks (1..120 ranks)");
        return TP_ERR_INVALID_ARGUMENT;
    }
    tp_status s = validate(sub, diag, super, rhs, n_local, sizes, nsizes, x_dev, err);
    if (s != TP_OK) return s;
    if (n_local < 2) {
        set_err(err, TP_ERR_INVALID_SIZE, "a shard needs at least 2 rows");
        return TP_ERR_INVALID_SIZE;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    Plan<T> p;
    build_plan(n_local, sizes, nsizes, p);
    s = ensure_ws(ctx, p.ws_elems * sizeof(T), err);
    if (s != TP_OK) return s;
    bind_plan(p, SysPtrs<T>{sub, diag, super, rhs}, x_dev, ctx->ws);
    const cudaStream_t st = pick_stream(ctx, stream);
    ctx->last.kind = 0;
    auto key = make_key<T>(4, n_local, sizes, nsizes,
                           {sub, diag, super, rhs, eq_all_dev, x_dev, ctx->ws},
                           ((int64_t)nranks << 32) | rank);
    return run_maybe_graph<T>(ctx, st, key,
                              [&](Runner<T>& r) { r.shard_finish(p, eq_all_dev, nranks, rank); }, err);
}

template <class T>
tp_status shard_solve(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs, int64_t n_local,
                      const int64_t* sizes, int32_t nsizes, T* x_dev, void* stream, tp_error* err) {
    clear_err(err);
    if (!ctx) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    if (!ctx->linked) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "no peer links: call tp_shard_attach first");
        return TP_ERR_INVALID_ARGUMENT;
    }
    tp_status s = validate(sub, diag, super, rhs, n_local, sizes, nsizes, x_dev, err);
    if (s != TP_OK) return s;
    if (n_local < 2) {
        set_err(err, TP_ERR_INVALID_SIZE, "a shard needs at least 2 rows");
        return TP_ERR_INVALID_SIZE;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    Plan<T> p;
    build_plan(n_local, sizes, nsizes, p, /*fused=*/true, ctx->link_shared ? 8 : 0);
    s = ensure_ws(ctx, p.ws_elems * sizeof(T), err);
    if (s != TP_OK) return s;
    bind_plan(p, SysPtrs<T>{sub, diag, super, rhs}, x_dev, ctx->ws);
    const cudaStream_t st = pick_stream(ctx, stream);
    ctx->last.kind = 0;
    auto key = make_key<T>(5, n_local, sizes, nsizes, {sub, diag, super, rhs, x_dev, ctx->ws},
                           ctx->link_gen * 2 + (ctx->link_shared ? 1 : 0));
    return run_maybe_graph<T>(ctx, st, key, [&](Runner<T>& r) { r.shard_solve(p); }, err);
}

template <class T>
tp_status generate_dev(tp_ctx* ctx, int64_t n, int64_t row0, int64_t n_global, uint64_t seed, double delta,
                       T* sub, T* diag, T* super, T* rhs, void* stream, tp_error* err) {
    clear_err(err);
    if (!ctx || !sub || !diag || !super || !rhs) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    if (n_global < 2 || n < 0 || row0 < 0 || row0 + n > n_global) {  // bench.hpp:69
        set_err(err, TP_ERR_INVALID_SIZE, "system size must be >= 2");
        return TP_ERR_INVALID_SIZE;
    }
    if (!(delta > 1.0)) {  // bench.hpp:70
        set_err(err, TP_ERR_INVALID_SIZE, "dominance factor must be > 1");
        return TP_ERR_INVALID_SIZE;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    TP_CUDA(tpb::launch_generate<T>(n, row0, n_global, seed, delta, sub, diag, super, rhs, ctx->sms,
                                    pick_stream(ctx, stream)));
    return TP_OK;
}

// reduce_block(sys, Block{start, end}) — partition.hpp:77-126, on the device
// with the reference's own arithmetic (k_ref_sweep<STORE>): the interface
// pair and the up-sweep vectors of ReducedBlock (indexed by offset from
// start; the entry at len-1 is left 0, as the reference never writes it).
template <class T>
tp_status reduce_block_host(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs, int64_t n,
                            int64_t start, int64_t end, T* eq8, T* a, T* beta, T* gamma, T* delta,
                            tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    if (!sub || !diag || !super || !rhs || !eq8) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    if (start < 0 || end > n || end - start < 2) {  // partition.hpp:79
        set_err(err, TP_ERR_INVALID_SIZE, "block length must be >= 2");
        return TP_ERR_INVALID_SIZE;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    const int64_t len = end - start;
    T* d[5];
    tp_status s = ensure_dsys<T>(ctx, 2 * len + 8, d, err);  // 5 arrays of >= 2 len + 8 rows
    if (s != TP_OK) return s;
    const cudaStream_t st = ctx->stream;
    const T* in[4] = {sub, diag, super, rhs};
    for (int i = 0; i < 4; ++i)
        TP_CUDA(cudaMemcpyAsync(d[i], in[i] + start, (size_t)len * sizeof(T), cudaMemcpyHostToDevice, st));
    // outputs: d[4] = eq8 (8) + first (1 int64); up-sweep vectors in the
    // second halves of d[0..3]
    T* ov[4] = {d[0] + len, d[1] + len, d[2] + len, d[3] + len};
    for (int i = 0; i < 4; ++i) TP_CUDA(cudaMemsetAsync(ov[i], 0, (size_t)len * sizeof(T), st));
    int64_t* first = reinterpret_cast<int64_t*>(d[4] + 8);
    TP_CUDA(tpb::launch_ref_sweep<T>(SysPtrs<T>{d[0], d[1], d[2], d[3]}, len, len, 1, first, nullptr, d[4], ov[0],
                                     ov[1], ov[2], ov[3], st));
    int64_t bad = -1;
    TP_CUDA(cudaMemcpyAsync(&bad, first, sizeof(bad), cudaMemcpyDeviceToHost, st));
    TP_CUDA(cudaMemcpyAsync(eq8, d[4], 8 * sizeof(T), cudaMemcpyDeviceToHost, st));
    T* outs[4] = {a, beta, gamma, delta};
    for (int i = 0; i < 4; ++i)
        if (outs[i]) TP_CUDA(cudaMemcpyAsync(outs[i], ov[i], (size_t)len * sizeof(T), cudaMemcpyDeviceToHost, st));
    TP_CUDA(cudaStreamSynchronize(st));
    if (bad >= 0) {
        set_err(err, TP_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(start + bad), start + bad, 0);
        return TP_ERR_ZERO_PIVOT;
    }
    return TP_OK;
}

struct ProfileState {
    cudaStream_t st;
    std::vector<cudaEvent_t> evs;
    std::vector<std::string> names;
};

void profile_hook(void* user, const char* name) {
    auto* ps = static_cast<ProfileState*>(user);
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, ps->st);
    ps->evs.push_back(e);
    ps->names.push_back(name);
}

}  // namespace

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

int32_t tp_abi_version(void) { return TP_ABI_VERSION; }

tp_status tp_ctx_create(int32_t device, tp_ctx** out, tp_error* err) {
    clear_err(err);
    if (!out) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "out is NULL");
        return TP_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    int ndev = 0;
    TP_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "device index out of range");
        return TP_ERR_INVALID_ARGUMENT;
    }
    TP_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    TP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0) {
        set_err(err, TP_ERR_CUDA,
                "tridpart_b200 is built for sm_100a (B200); found sm_" + std::to_string(prop.major) +
                    std::to_string(prop.minor));
        return TP_ERR_CUDA;
    }
    TP_CUDA(tpb::init_kernel_attributes());
    tp_ctx* c = new tp_ctx();
    c->device = device;
    c->sms = prop.multiProcessorCount;
    cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_err, 64);
    if (e == cudaSuccess) e = cudaMemset(c->d_err, 0xFF, 64);  // kNoError
    if (e == cudaSuccess) e = cudaMalloc(&c->d_red, 64);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_small, 4096);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_grid, tpb::kGridScratchBytes);
    if (e == cudaSuccess) e = cudaMemset(c->d_grid, 0, tpb::kGridScratchBytes);
    if (const char* v = getenv("TPB_GRID")) c->grid_on = atoi(v) != 0;
    if (const char* v = getenv("TPB_GRID_MIN")) c->grid_min = std::max<int64_t>(4, atoll(v));
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_err, 64);
    if (e != cudaSuccess) {
        set_err(err, TP_ERR_CUDA, std::string("context allocation: ") + cudaGetErrorString(e));
        tp_ctx_destroy(c);
        return TP_ERR_CUDA;
    }
    c->stream = c->own;
    *out = c;
    return TP_OK;
}

void tp_ctx_destroy(tp_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (auto& g : ctx->gcache) cudaGraphExecDestroy(g.exec);
    if (ctx->ws) cudaFree(ctx->ws);
    if (ctx->dsys) cudaFree(ctx->dsys);
    if (ctx->d_err) cudaFree(ctx->d_err);
    if (ctx->d_red) cudaFree(ctx->d_red);
    if (ctx->d_small) cudaFree(ctx->d_small);
    if (ctx->d_grid) cudaFree(ctx->d_grid);
    for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
    if (ctx->mailbox) cudaFree(ctx->mailbox);
    if (ctx->d_epoch) cudaFree(ctx->d_epoch);
    if (ctx->h_err) cudaFreeHost(ctx->h_err);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    delete ctx;
}

tp_status tp_ctx_set_stream(tp_ctx* ctx, void* stream, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
    return TP_OK;
}

tp_status tp_ctx_set_graphs(tp_ctx* ctx, int32_t enabled, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    ctx->graphs = enabled != 0;
    return TP_OK;
}

tp_status tp_ctx_set_grid(tp_ctx* ctx, int32_t enabled, int64_t min_rows, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    if (min_rows < 4) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "min_rows must be >= 4");
        return TP_ERR_INVALID_ARGUMENT;
    }
    if ((enabled != 0) != ctx->grid_on || min_rows != ctx->grid_min) drop_graphs(ctx);
    ctx->grid_on = enabled != 0;
    ctx->grid_min = min_rows;
    return TP_OK;
}

int64_t tp_ctx_last_launch_count(const tp_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

int64_t tp_ctx_last_kernels(const tp_ctx* ctx, char* buf, int64_t cap) {
    if (!ctx) return 0;
    const int64_t len = (int64_t)ctx->last_names.size();
    if (buf && cap > 0) {
        const int64_t k = len < cap - 1 ? len : cap - 1;
        std::memcpy(buf, ctx->last_names.data(), (size_t)k);
        buf[k] = '\0';
    }
    return len;
}

tp_status tp_check_device_error(tp_ctx* ctx, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    TP_CUDA(cudaMemcpy(ctx->h_err, ctx->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return decode_device_error(ctx, err);
}

// ---- solve_partition ------------------------------------------------------
tp_status tp_solve_partition_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                     const double* super, const double* rhs, int64_t n,
                                     const int64_t* sizes, int32_t nsizes, double* x, void* stream,
                                     tp_error* err) {
    return solve_dev<double>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, stream, err);
}
tp_status tp_solve_partition_f32_dev(tp_ctx* ctx, const float* sub, const float* diag,
                                     const float* super, const float* rhs, int64_t n,
                                     const int64_t* sizes, int32_t nsizes, float* x, void* stream,
                                     tp_error* err) {
    return solve_dev<float>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, stream, err);
}
tp_status tp_solve_partition_f64(tp_ctx* ctx, const double* sub, const double* diag,
                                 const double* super, const double* rhs, int64_t n,
                                 const int64_t* sizes, int32_t nsizes, double* x, tp_error* err) {
    return solve_host<double>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, err);
}
tp_status tp_solve_partition_f32(tp_ctx* ctx, const float* sub, const float* diag,
                                 const float* super, const float* rhs, int64_t n,
                                 const int64_t* sizes, int32_t nsizes, float* x, tp_error* err) {
    return solve_host<float>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, err);
}
tp_status tp_solve_partition_f64_async(tp_ctx* ctx, const double* sub, const double* diag,
                                       const double* super, const double* rhs, int64_t n,
                                       const int64_t* sizes, int32_t nsizes, double* x, void* stream,
                                       tp_error* err) {
    return solve_host_async<double>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, stream, err);
}
tp_status tp_solve_partition_f32_async(tp_ctx* ctx, const float* sub, const float* diag,
                                       const float* super, const float* rhs, int64_t n,
                                       const int64_t* sizes, int32_t nsizes, float* x, void* stream,
                                       tp_error* err) {
    return solve_host_async<float>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, stream, err);
}
tp_status tp_solve_partition_observe_f64(tp_ctx* ctx, const double* sub, const double* diag,
                                         const double* super, const double* rhs, int64_t n,
                                         const int64_t* sizes, int32_t nsizes, double* x,
                                         tp_interface_cb cb, void* user, tp_error* err) {
    return solve_observe<double>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, cb, user, err);
}
tp_status tp_solve_partition_observe_f32(tp_ctx* ctx, const float* sub, const float* diag,
                                         const float* super, const float* rhs, int64_t n,
                                         const int64_t* sizes, int32_t nsizes, float* x,
                                         tp_interface_cb_f32 cb, void* user, tp_error* err) {
    return solve_observe<float>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, cb, user, err);
}

// ---- thomas_solve / residual_inf ------------------------------------------
tp_status tp_thomas_solve_f64(tp_ctx* ctx, const double* sub, const double* diag,
                              const double* super, const double* rhs, int64_t n, double* x,
                              tp_error* err) {
    return thomas_host<double>(ctx, sub, diag, super, rhs, n, x, err);
}
tp_status tp_thomas_solve_f32(tp_ctx* ctx, const float* sub, const float* diag, const float* super,
                              const float* rhs, int64_t n, float* x, tp_error* err) {
    return thomas_host<float>(ctx, sub, diag, super, rhs, n, x, err);
}
tp_status tp_residual_inf_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                  const double* super, const double* rhs, int64_t n,
                                  const double* x, double* out, void* stream, tp_error* err) {
    return residual_dev<double>(ctx, sub, diag, super, rhs, n, x, out, stream, err);
}
tp_status tp_residual_inf_f32_dev(tp_ctx* ctx, const float* sub, const float* diag,
                                  const float* super, const float* rhs, int64_t n, const float* x,
                                  double* out, void* stream, tp_error* err) {
    return residual_dev<float>(ctx, sub, diag, super, rhs, n, x, out, stream, err);
}

// ---- reduce_block ---------------------------------------------------------
tp_status tp_reduce_block_f64(tp_ctx* ctx, const double* sub, const double* diag, const double* super,
                              const double* rhs, int64_t n, int64_t start, int64_t end, double* eq8,
                              double* a, double* beta, double* gamma, double* delta, tp_error* err) {
    return reduce_block_host<double>(ctx, sub, diag, super, rhs, n, start, end, eq8, a, beta, gamma, delta, err);
}
tp_status tp_reduce_block_f32(tp_ctx* ctx, const float* sub, const float* diag, const float* super,
                              const float* rhs, int64_t n, int64_t start, int64_t end, float* eq8, float* a,
                              float* beta, float* gamma, float* delta, tp_error* err) {
    return reduce_block_host<float>(ctx, sub, diag, super, rhs, n, start, end, eq8, a, beta, gamma, delta, err);
}

// ---- sharded --------------------------------------------------------------
tp_status tp_shard_reduce_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                  const double* super, const double* rhs, int64_t n_local,
                                  const int64_t* sizes, int32_t nsizes, double* eq8_dev,
                                  void* stream, tp_error* err) {
    return shard_reduce<double>(ctx, sub, diag, super, rhs, n_local, sizes, nsizes, eq8_dev, stream, err);
}
tp_status tp_shard_finish_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                  const double* super, const double* rhs, int64_t n_local,
                                  const int64_t* sizes, int32_t nsizes, const double* eq_all_dev,
                                  int32_t nranks, int32_t rank, double* x_dev, void* stream,
                                  tp_error* err) {
    return shard_finish<double>(ctx, sub, diag, super, rhs, n_local, sizes, nsizes, eq_all_dev, nranks,
                                rank, x_dev, stream, err);
}

tp_status tp_shard_solve_f64_dev(tp_ctx* ctx, const double* sub, const double* diag, const double* super,
                                 const double* rhs, int64_t n_local, const int64_t* sizes, int32_t nsizes,
                                 double* x_dev, void* stream, tp_error* err) {
    return shard_solve<double>(ctx, sub, diag, super, rhs, n_local, sizes, nsizes, x_dev, stream, err);
}

tp_status tp_shard_prepare_f64_dev(tp_ctx* ctx, const double* sub, const double* diag, const double* super,
                                   const double* rhs, int64_t n_local, const int64_t* sizes, int32_t nsizes,
                                   double* x_dev, void* stream, tp_error* err) {
    if (!ctx) return shard_solve<double>(ctx, sub, diag, super, rhs, n_local, sizes, nsizes, x_dev, stream, err);
    if (!ctx->graphs) {
        clear_err(err);
        return TP_OK;  // nothing to prepare without graphs
    }
    ctx->prepare_only = true;
    const tp_status s = shard_solve<double>(ctx, sub, diag, super, rhs, n_local, sizes, nsizes, x_dev, stream, err);
    ctx->prepare_only = false;
    return s;
}

tp_status tp_shard_mailbox(tp_ctx* ctx, int32_t nranks, void** mailbox, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    if (!mailbox || nranks < 1 || nranks > tpb::kMaxPeers) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "mailbox: bad arguments (1..64 ranks)");
        return TP_ERR_INVALID_ARGUMENT;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    if (ctx->mailbox && ctx->mailbox_ranks != nranks) {
        TP_CUDA(cudaDeviceSynchronize());
        TP_CUDA(cudaFree(ctx->mailbox));
        ctx->mailbox = nullptr;
        ctx->linked = false;
    }
    if (!ctx->mailbox) {
        // its own allocation, so a CUDA IPC handle of it maps exactly the mailbox
        TP_CUDA(cudaMalloc(&ctx->mailbox, tpb::mailbox_bytes(nranks)));
        TP_CUDA(cudaMemset(ctx->mailbox, 0, tpb::mailbox_bytes(nranks)));
        ctx->mailbox_ranks = nranks;
    }
    if (!ctx->d_epoch) {
        TP_CUDA(cudaMalloc(&ctx->d_epoch, 256));
        TP_CUDA(cudaMemset(ctx->d_epoch, 0, 256));
    }
    *mailbox = ctx->mailbox;
    return TP_OK;
}

tp_status tp_ipc_get_handle(tp_ctx* ctx, void* dev_ptr, uint8_t* handle64, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    if (!dev_ptr || !handle64) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    cudaIpcMemHandle_t h;
    TP_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, 64);
    return TP_OK;
}

tp_status tp_ipc_open_handle(tp_ctx* ctx, const uint8_t* handle64, void** dev_ptr, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    if (!dev_ptr || !handle64) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    TP_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->ipc_opened.push_back(*dev_ptr);
    return TP_OK;
}

tp_status tp_shard_attach(tp_ctx* ctx, int32_t nranks, int32_t rank, void* const* mailboxes, tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    if (!mailboxes || nranks < 1 || nranks > tpb::kMaxPeers || rank < 0 || rank >= nranks) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "attach: bad rank / nranks (1..64 ranks)");
        return TP_ERR_INVALID_ARGUMENT;
    }
    if (!ctx->mailbox || ctx->mailbox_ranks != nranks || mailboxes[rank] != ctx->mailbox) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "attach: mailboxes[rank] must be this context's tp_shard_mailbox");
        return TP_ERR_INVALID_ARGUMENT;
    }
    for (int p = 0; p < nranks; ++p)
        if (!mailboxes[p]) {
            set_err(err, TP_ERR_INVALID_ARGUMENT, "attach: null peer mailbox");
            return TP_ERR_INVALID_ARGUMENT;
        }
    TP_CUDA(cudaSetDevice(ctx->device));
    TP_CUDA(cudaDeviceSynchronize());
    TP_CUDA(cudaMemset(ctx->mailbox, 0, tpb::mailbox_bytes(nranks)));
    TP_CUDA(cudaMemset(ctx->d_epoch, 0, 256));
    TP_CUDA(cudaDeviceSynchronize());
    tpb::ShardLink lk{};
    for (int p = 0; p < nranks; ++p) lk.peers[p] = static_cast<double*>(mailboxes[p]);
    lk.own = static_cast<double*>(ctx->mailbox);
    lk.epoch = ctx->d_epoch;
    lk.nranks = nranks;
    lk.rank = rank;
    ctx->link = lk;
    // peers on this very GPU (simulated ranks, TPB_SHARE_GPU): every rank's
    // exchange kernel spins on one device, so they take the portable 8-CTA
    // cluster shape (more of them co-resident, SMs left for the others' levels)
    ctx->link_shared = false;
    for (int p = 0; p < nranks; ++p) {
        if (p == rank) continue;
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, mailboxes[p]) != cudaSuccess) {
            cudaGetLastError();
            ctx->link_shared = true;  // unknown: the conservative shape
        } else if (pa.device == ctx->device) {
            ctx->link_shared = true;
        }
    }
    ctx->linked = true;
    ++ctx->link_gen;  // graphs captured with the previous links stay keyed to them
    return TP_OK;
}

// ---- synthetic inputs -----------------------------------------------------
tp_status tp_generate_system_f64_dev(tp_ctx* ctx, int64_t n, int64_t row0, int64_t n_global,
                                     uint64_t seed, double delta, double* sub, double* diag,
                                     double* super, double* rhs, void* stream, tp_error* err) {
    return generate_dev<double>(ctx, n, row0, n_global, seed, delta, sub, diag, super, rhs, stream, err);
}
tp_status tp_generate_system_f32_dev(tp_ctx* ctx, int64_t n, int64_t row0, int64_t n_global,
                                     uint64_t seed, double delta, float* sub, float* diag,
                                     float* super, float* rhs, void* stream, tp_error* err) {
    return generate_dev<float>(ctx, n, row0, n_global, seed, delta, sub, diag, super, rhs, stream, err);
}

// ---- plans ----------------------------------------------------------------
tp_status tp_make_plan(int64_t n, int64_t m, int64_t* bounds, int64_t* nblocks, tp_error* err) {
    clear_err(err);
    if (n < 2) {
        set_err(err, TP_ERR_INVALID_SIZE, "system size must be >= 2");
        return TP_ERR_INVALID_SIZE;
    }
    if (m < 2) {
        set_err(err, TP_ERR_INVALID_SIZE, "sub-system size must be >= 2");
        return TP_ERR_INVALID_SIZE;
    }
    const int64_t K = plan_blocks(n, m);
    if (nblocks) *nblocks = K;
    if (bounds) {
        for (int64_t j = 0; j < K; ++j) bounds[j] = j * m;
        bounds[K] = n;
    }
    return TP_OK;
}

tp_status tp_plan_levels(int64_t n, const int64_t* sizes, int32_t nsizes, int64_t* level_n,
                         int64_t* level_m, int32_t* nlevels, int32_t max_levels, int64_t* n_final,
                         tp_error* err) {
    clear_err(err);
    tp_status s = validate_policy(n, sizes, nsizes, err);
    if (s != TP_OK) return s;
    Plan<double> p;
    build_plan(n, sizes, nsizes, p, true);
    if ((int32_t)p.levels.size() > max_levels) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "max_levels too small");
        return TP_ERR_INVALID_ARGUMENT;
    }
    for (size_t l = 0; l < p.levels.size(); ++l) {
        if (level_n) level_n[l] = p.levels[l].n;
        if (level_m) level_m[l] = (p.levels[l].internal || p.levels[l].split) ? -p.levels[l].m : p.levels[l].m;
    }
    if (nlevels) *nlevels = (int32_t)p.levels.size();
    if (n_final) *n_final = p.n_final;
    return TP_OK;
}

// ---- instrumented solve ---------------------------------------------------
tp_status tp_solve_profile_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                   const double* super, const double* rhs, int64_t n,
                                   const int64_t* sizes, int32_t nsizes, double* x, float* kernel_ms,
                                   char* names, int32_t max_kernels, int32_t* nkernels,
                                   tp_error* err) {
    clear_err(err);
    TP_NEED_CTX(ctx);
    tp_status s = validate(sub, diag, super, rhs, n, sizes, nsizes, x, err);
    if (s != TP_OK) return s;
    TP_CUDA(cudaSetDevice(ctx->device));
    Plan<double> p;
    build_plan(n, sizes, nsizes, p, true);
    s = ensure_ws(ctx, p.ws_elems * sizeof(double), err);
    if (s != TP_OK) return s;
    bind_plan(p, SysPtrs<double>{sub, diag, super, rhs}, x, ctx->ws);
    const cudaStream_t st = ctx->stream;
    ProfileState ps{st, {}, {}};
    cudaEvent_t e0;
    TP_CUDA(cudaEventCreate(&e0));
    TP_CUDA(cudaMemsetAsync(ctx->d_err, 0xFF, sizeof(unsigned long long), st));
    TP_CUDA(cudaEventRecord(e0, st));
    Runner<double> r{ctx, st};
    r.hook = profile_hook;
    r.hook_user = &ps;
    r.solve_body(p);
    ctx->last_launches = r.launches;
    TP_CUDA(cudaStreamSynchronize(st));
    const int32_t cnt = (int32_t)std::min<size_t>(ps.evs.size(), (size_t)max_kernels);
    cudaEvent_t prev = e0;
    for (int32_t i = 0; i < cnt; ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, prev, ps.evs[i]);
        if (kernel_ms) kernel_ms[i] = ms;
        if (names) std::snprintf(names + 32 * i, 32, "%s", ps.names[i].c_str());
        prev = ps.evs[i];
    }
    if (nkernels) *nkernels = cnt;
    for (auto e : ps.evs) cudaEventDestroy(e);
    cudaEventDestroy(e0);
    if (r.status != cudaSuccess) {
        set_err(err, TP_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(r.status));
        return TP_ERR_CUDA;
    }
    return TP_OK;
}

}  // extern "C"
