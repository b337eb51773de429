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
    // bound pointers
    SysPtrs<T> in{};
    T* x_out = nullptr;    // solution of this level's system
    IfacePtrs<T> iface{};  // next level's system (2K rows)
    T* x_iface = nullptr;
};

template <class T>
struct Plan {
    std::vector<Level<T>> levels;
    int64_t n_final = 0;
    SysPtrs<T> final_in{};
    T* final_x = nullptr;
    size_t ws_elems = 0;  // workspace, in elements of T
};

inline size_t pad32(size_t v) { return (v + 31) & ~size_t(31); }

// fused = the plan is for solve_body, which runs the deepest level and the
// finishing solve as one kernel when that level fits k_level_final_cl: then
// the deepest interface may exceed kFinalCap (no device-internal level is
// added for it), and an oversized final system gets ONE fused internal level
// of m = 16 when that fits. The sharded paths keep n_final <= kFinalCap.
template <class T>
void build_plan(int64_t n, const int64_t* sizes, int32_t nsizes, Plan<T>& p, bool fused = false) {
    p.levels.clear();
    int64_t cur = n;
    int lvl = 0;
    size_t ws = 0;
    while (nsizes > 0) {
        if (cur < 4) break;
        Level<T> L;
        L.n = cur;
        L.m = sizes[lvl];
        L.K = plan_blocks(cur, L.m);
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
        ws += 5 * pad32((size_t)(2 * L.K));
        p.levels.push_back(L);
        cur = 2 * L.K;
        if (lvl == nsizes - 1) break;
        ++lvl;
    }
    // device-internal levels so the finishing solve fits one cluster
    const bool last_fused = fused && !p.levels.empty() &&
                            tpb::level_final_fits(p.levels.back().n, p.levels.back().m, p.levels.back().K, sizeof(T));
    while (!last_fused && cur > tpb::kFinalCap) {
        Level<T> L;
        L.n = cur;
        L.m = kInternalM;
        if (fused && tpb::level_final_fits(cur, kFusedInternalM, plan_blocks(cur, kFusedInternalM), sizeof(T)))
            L.m = kFusedInternalM;
        L.K = plan_blocks(cur, L.m);
        const int64_t last_len = cur - (L.K - 1) * L.m;
        L.kfull = (last_len == L.m) ? L.K : L.K - 1;
        L.tail = (last_len == L.m) ? 0 : last_len;
        L.internal = true;
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
        const size_t k2 = pad32((size_t)(2 * L.K));
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
    // fused multi-GPU path (k_final<kShard>): own mailbox, peer links, epoch word
    void* mailbox = nullptr;
    int mailbox_ranks = 0;
    unsigned long long* d_epoch = nullptr;
    tpb::ShardLink link{};
    bool linked = false;
    int64_t link_gen = 0;
    std::vector<void*> ipc_opened;
    bool prepare_only = false;  // capture + instantiate the graph, do not launch
    tpb::Stager stager;         // pinned staging of pageable host buffers
    void* dsys = nullptr;                 // host-path staging (5 arrays)
    size_t dsys_cap = 0;                  // bytes
    int64_t last_launches = 0;
    struct GraphEntry {
        std::vector<int64_t> key;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        uint64_t stamp = 0;
    };
    std::vector<GraphEntry> gcache;
    uint64_t clock = 0;
};

namespace {


using KernelHook = void (*)(void* user, const char* name);

template <class T>
struct Runner {
    tp_ctx* ctx;
    cudaStream_t st;
    KernelHook hook = nullptr;
    void* hook_user = nullptr;
    int64_t launches = 0;
    cudaError_t status = cudaSuccess;

    void after(const char* what, int level) {
        ++launches;
        if (hook) {
            char name[32];
            std::snprintf(name, sizeof(name), "%s:L%d", what, level);
            hook(hook_user, name);
        }
    }
    void check(cudaError_t e) {
        if (e != cudaSuccess && status == cudaSuccess) status = e;
    }

    void main_part(const Level<T>& L, int level, int mode) {
        const bool s1 = (mode == tpb::kStage1);
        int fl, fg;
        if (tpb::fast_shape(L.m, &fl, &fg)) {
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

    // Whole solve: reset the error word, Stage 1 down, finish, Stage 3 up.
    void solve(const Plan<T>& p) {
        check(tpb::launch_reset(ctx->d_err, st));
        solve_body(p);
    }
    // The deepest level and the finishing solve run as one cluster kernel when
    // that level fits the cluster's shared memory (k_level_final_cl); its
    // interface is still written out (for the observer), never read back.
    void solve_body(const Plan<T>& p) {
        const size_t nl = p.levels.size();
        const bool fuse = nl > 0 && tpb::level_final_fits(p.levels.back().n, p.levels.back().m,
                                                          p.levels.back().K, sizeof(T));
        const size_t top = fuse ? nl - 1 : nl;
        size_t l = 0;
        if (top >= 2) {  // level 1's Stage 1 folded into level 0's (k_fast_s1fold)
            const Level<T>& A = p.levels[0];
            const Level<T>& B = p.levels[1];
            if (A.tail == 0 && A.kfull == A.K && B.tail == 0 && tpb::fold_fits(A.m, A.K, B.n, B.m, B.K)) {
                const bool vec = aligned32(A.in.sub) && aligned32(A.in.diag) && aligned32(A.in.sup) &&
                                 aligned32(A.in.rhs);
                // level 2 too when its blocks are the fold CTAs' tiles (m2 = 32)
                const bool f2 = top >= 3 && tpb::fold2_fits(B.K, p.levels[2].n, p.levels[2].m, p.levels[2].K);
                check(tpb::launch_fold<T>(A.m, vec, A.in, A.K, A.iface, B.m, B.K, B.iface,
                                          f2 ? &p.levels[2].iface : nullptr, ctx->d_err, 0, st));
                after(f2 ? "stage1_fold2" : "stage1_fold", 0);
                l = f2 ? 3 : 2;
            }
        }
        for (; l < top; ++l) stage(p.levels[l], (int)l, tpb::kStage1);
        if (fuse) {
            const Level<T>& L = p.levels.back();
            check(tpb::launch_level_final<T>(L.in, L.n, L.m, L.K, L.iface, L.x_out, ctx->d_err, (int)top, st));
            after("level_final", (int)top);
        } else {
            final_solve(p);
        }
        for (size_t l = top; l-- > 0;) stage(p.levels[l], (int)l, tpb::kStage3);
    }

    // Sharded halves.
    void shard_reduce(const Plan<T>& p, T* eq8) {
        check(tpb::launch_reset(ctx->d_err, st));
        for (size_t l = 0; l < p.levels.size(); ++l) stage(p.levels[l], (int)l, tpb::kStage1);
        IfacePtrs<T> o{eq8, eq8 + 2, eq8 + 4, eq8 + 6};
        check(tpb::launch_final<T>(tpb::kStage1, p.final_in, p.n_final, o, nullptr, nullptr, ctx->d_err,
                                   (int)p.levels.size(), st));
        after("shard_reduce", (int)p.levels.size());
    }
    // Fused multi-GPU solve of one shard: every local level, the peer exchange
    // and top solve inside the finishing kernel, every local Stage 3.
    void shard_solve(const Plan<T>& p) {
        check(tpb::launch_reset(ctx->d_err, st));
        for (size_t l = 0; l < p.levels.size(); ++l) stage(p.levels[l], (int)l, tpb::kStage1);
        check(tpb::launch_final<T>(tpb::kShard, p.final_in, p.n_final, IfacePtrs<T>{}, nullptr, p.final_x,
                                   ctx->d_err, (int)p.levels.size(), st, &ctx->link));
        after("shard_exchange", (int)p.levels.size());
        for (size_t l = p.levels.size(); l-- > 0;) stage(p.levels[l], (int)l, tpb::kStage3);
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

tp_status decode_device_error(tp_ctx* ctx, tp_error* err) {
    const unsigned long long code = *ctx->h_err;
    if (code == tpb::kNoError) return TP_OK;
    const int32_t level = (int32_t)(code >> 48);
    const int64_t row = (int64_t)(code & 0xFFFFFFFFFFFFULL);
    if (level == tpb::kExchangeLevel) {
        set_err(err, TP_ERR_NCCL, "peer exchange timed out waiting for rank " + std::to_string(row), row, -1);
        return TP_ERR_NCCL;
    }
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
    ge.stamp = ++ctx->clock;
    ctx->gcache.push_back(ge);
    ctx->last_launches = r.launches;
    if (!ctx->prepare_only) TP_CUDA(cudaGraphLaunch(exec, st));
    if (dbg)
        std::fprintf(stderr, "[tpb graph] capture %.3f ms, instantiate %.3f ms, launch %.3f ms (%lld kernels)\n",
                     t1 - t0, t2 - t1, now_ms() - t2, (long long)r.launches);
    return TP_OK;
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
    auto key = make_key<T>(1, n, sizes, nsizes, {sub, diag, super, rhs, x, ctx->ws});
    return run_maybe_graph<T>(ctx, st, key, [&](Runner<T>& r) { r.solve(p); }, err);
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
    tp_status s = solve_host<T>(ctx, sub, diag, super, rhs, n, sizes, nsizes, x, err);
    if (s != TP_OK || emit == nullptr) return s;
    T* d[5];
    s = ensure_dsys<T>(ctx, n, d, err);  // same buffers the solve used
    if (s != TP_OK) return s;
    Plan<T> p;
    build_plan(n, sizes, nsizes, p, true);
    bind_plan(p, SysPtrs<T>{d[0], d[1], d[2], d[3]}, d[4], ctx->ws);
    std::vector<T> h;
    for (size_t l = 0; l < p.levels.size(); ++l) {
        const Level<T>& L = p.levels[l];
        if (L.internal) break;  // device-internal levels are not part of the policy
        const int64_t n2 = 2 * L.K;
        h.resize((size_t)(4 * n2));
        TP_CUDA(cudaMemcpy(h.data(), L.iface.sub, n2 * sizeof(T), cudaMemcpyDeviceToHost));
        TP_CUDA(cudaMemcpy(h.data() + n2, L.iface.diag, n2 * sizeof(T), cudaMemcpyDeviceToHost));
        TP_CUDA(cudaMemcpy(h.data() + 2 * n2, L.iface.sup, n2 * sizeof(T), cudaMemcpyDeviceToHost));
        TP_CUDA(cudaMemcpy(h.data() + 3 * n2, L.iface.rhs, n2 * sizeof(T), cudaMemcpyDeviceToHost));
        emit((int64_t)l, n2, h.data(), h.data() + n2, h.data() + 2 * n2, h.data() + 3 * n2, user);
    }
    return TP_OK;
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
            auto key = make_key<T>(2, n, nullptr, 0, {d[0], d[1], d[2], d[3], d[4], ctx->ws});
            return run_maybe_graph<T>(ctx, st, key, [&](Runner<T>& r) { r.solve(p); }, err);
        },
        err);
}

template <class T>
tp_status residual_dev(tp_ctx* ctx, const T* sub, const T* diag, const T* super, const T* rhs, int64_t n,
                       const T* x, double* out, tp_error* err) {
    clear_err(err);
    if (!ctx || !out || !sub || !diag || !super || !rhs || !x) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    TP_CUDA(cudaSetDevice(ctx->device));
    const cudaStream_t st = ctx->stream;
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
    build_plan(n_local, sizes, nsizes, p);
    s = ensure_ws(ctx, p.ws_elems * sizeof(T), err);
    if (s != TP_OK) return s;
    bind_plan(p, SysPtrs<T>{sub, diag, super, rhs}, x_dev, ctx->ws);
    const cudaStream_t st = pick_stream(ctx, stream);
    auto key = make_key<T>(5, n_local, sizes, nsizes, {sub, diag, super, rhs, x_dev, ctx->ws}, ctx->link_gen);
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
    if (e == cudaSuccess) e = cudaMalloc(&c->d_red, 64);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_small, 4096);
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

int64_t tp_ctx_last_launch_count(const tp_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

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
                                  const double* x, double* out, tp_error* err) {
    return residual_dev<double>(ctx, sub, diag, super, rhs, n, x, out, err);
}
tp_status tp_residual_inf_f32_dev(tp_ctx* ctx, const float* sub, const float* diag,
                                  const float* super, const float* rhs, int64_t n, const float* x,
                                  double* out, tp_error* err) {
    return residual_dev<float>(ctx, sub, diag, super, rhs, n, x, out, err);
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
        if (level_m) level_m[l] = p.levels[l].internal ? -p.levels[l].m : p.levels[l].m;
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
