/*
 * tridpart_b200.h — C-ABI of the B200-native (sm_100a) partition solver.
 *
 * Drop-in boundary for the reference `tridpart` header-only C++20 library
 * (/root/reference/proj/include/tridpart). The reference has no C ABI of its
 * own; each entry point below names the reference function whose contract it
 * replaces (file:line, paths relative to /root/reference/proj/). Plain
 * pointers and sizes only — no C++ or torch types. The C++ shim
 * include/tridpart_b200.hpp rebuilds the reference's `tridpart::` API
 * (same names, same exception types) on top of these calls.
 *
 * Conventions
 *   - System arrays are the reference's SoA layout (tridiagonal.hpp:22-28):
 *     row i reads sub[i]*x[i-1] + diag[i]*x[i] + super[i]*x[i+1] = rhs[i].
 *     sub[0] and super[n-1] are never used numerically (as in the reference).
 *   - `sizes[0..nsizes)` is RecursionPolicy::sizes (partition.hpp:176-187):
 *     nsizes == 1 is the non-recursive method, nsizes == R+1 recursive depth R.
 *   - Every call returns a tp_status; on failure `err` (may be NULL) carries
 *     the code, the zero-pivot row and level, and a message.
 *   - A tp_ctx owns one CUDA device, a stream, a workspace and CUDA-graph
 *     caches. It is not thread-safe: use one context per host thread
 *     (the reference is reentrant, partition.hpp has no shared state).
 */
#ifndef TRIDPART_B200_H
#define TRIDPART_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TP_ABI_VERSION 2

/* Error classes of include/tridpart/errors.hpp:7-96. */
typedef enum tp_status {
    TP_OK = 0,
    TP_ERR_ZERO_PIVOT = 1,          /* ZeroPivotError(row)          errors.hpp:16-24 */
    TP_ERR_INVALID_SIZE = 2,        /* InvalidSizeError             errors.hpp:26-29 */
    TP_ERR_DEPTH_OUT_OF_RANGE = 3,  /* DepthOutOfRangeError         errors.hpp:31-34 */
    TP_ERR_EMPTY_TRAINING_SET = 4,  /* EmptyTrainingSetError        errors.hpp:38-41 */
    TP_ERR_K_TOO_LARGE = 5,         /* KTooLargeError               errors.hpp:43-46 */
    TP_ERR_MALFORMED_HEADER = 6,    /* MalformedHeaderError         errors.hpp:70-73 */
    TP_ERR_BAD_NUMBER = 7,          /* BadNumberError(line)         errors.hpp:75-84 */
    TP_ERR_IO = 8,                  /* Error("cannot open ...")     io.hpp:80-84     */
    TP_ERR_CUDA = 9,                /* device / runtime failure (no reference analogue) */
    TP_ERR_INVALID_ARGUMENT = 10,   /* NULL pointer, bad rank, ... */
    TP_ERR_NCCL = 11                /* collective path: peer exchange timed out, ... */
} tp_status;

typedef struct tp_error {
    int32_t code;   /* tp_status */
    int32_t level;  /* partition level of a zero pivot (0 = the input system) */
    int64_t row;    /* ZeroPivotError::row() (row index within that level's system, in the
                       reference's sweep order); BadNumberError: the line */
    char msg[256];
} tp_error;

typedef struct tp_ctx tp_ctx;

/* ---------------------------------------------------------------- context */
int32_t tp_abi_version(void);
tp_status tp_ctx_create(int32_t device, tp_ctx** out, tp_error* err);
void tp_ctx_destroy(tp_ctx* ctx);
/* Stream used by the synchronous host-pointer calls (cudaStream_t; NULL = ctx-owned). */
tp_status tp_ctx_set_stream(tp_ctx* ctx, void* stream, tp_error* err);
/* Disable/enable CUDA-graph capture of the device solve (default enabled). */
tp_status tp_ctx_set_graphs(tp_ctx* ctx, int32_t enabled, tp_error* err);
/* One-kernel grid solve (k_grid_solve) of one-level policies that fit the
 * GPU's shared memory: enabled (default 1; env TPB_GRID) for n >= min_rows
 * (default 80000, env TPB_GRID_MIN; below it the level path is faster). */
tp_status tp_ctx_set_grid(tp_ctx* ctx, int32_t enabled, int64_t min_rows, tp_error* err);
/* Number of kernels the last solve on this context launched (0 if none). */
int64_t tp_ctx_last_launch_count(const tp_ctx* ctx);
/* Names ("kernel:Llevel", comma-separated) of the kernels of the last solve on
 * this context, NUL-terminated into buf (cap bytes); returns the full length.
 * Diagnostic: which fused / folded kernels a plan took. */
int64_t tp_ctx_last_kernels(const tp_ctx* ctx, char* buf, int64_t cap);

/* ---------------------------------------------------- the partition solve */
/* solve_partition(sys, policy) — partition.hpp:244-248 (validation :235-242).
 * Host pointers, synchronous; x receives n doubles. */
tp_status tp_solve_partition_f64(tp_ctx* ctx, const double* sub, const double* diag,
                                 const double* super, const double* rhs, int64_t n,
                                 const int64_t* sizes, int32_t nsizes, double* x, tp_error* err);

/* Same contract on DEVICE pointers, asynchronous on `stream` (cudaStream_t,
 * NULL = ctx stream). Zero pivots are detected on the device: call
 * tp_check_device_error after synchronising the stream. */
tp_status tp_solve_partition_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                     const double* super, const double* rhs, int64_t n,
                                     const int64_t* sizes, int32_t nsizes, double* x, void* stream,
                                     tp_error* err);
/* Zero pivots (host and device calls): err->row / err->level are the ones
 * ZeroPivotError carries in the reference — the first failing pivot of its
 * sequential order (levels 0..depth, blocks in order, up-sweep then
 * down-sweep; then thomas_solve of the deepest interface), found by replaying
 * the reference's arithmetic on the device over the level systems of the
 * failed solve. tp_check_device_error needs the last solve's buffers alive. */
tp_status tp_check_device_error(tp_ctx* ctx, tp_error* err);

/* Host pointers, asynchronous on `stream` (NULL = ctx stream): the H2D copies,
 * the device solve and the D2H copy are enqueued and the call returns. Host
 * buffers should be pinned. Solves on two contexts / two streams overlap one
 * solve's D2H with the next one's H2D (full-duplex PCIe). After synchronising
 * the stream, tp_check_device_error reports zero pivots. */
tp_status tp_solve_partition_f64_async(tp_ctx* ctx, const double* sub, const double* diag,
                                       const double* super, const double* rhs, int64_t n,
                                       const int64_t* sizes, int32_t nsizes, double* x, void* stream,
                                       tp_error* err);

/* Observer overload solve_partition(sys, policy, on_interface) — partition.hpp:235-242,
 * hook at :206. Host pointers; after the solve, `cb` receives each level's
 * assembled interface system (host copies, valid during the call), level 0 first.
 * On a zero pivot at level l (err->level) the levels the reference completed
 * before it (0 .. l-1) are delivered, then the error is returned. */
typedef void (*tp_interface_cb)(int64_t level, int64_t n, const double* sub, const double* diag,
                                const double* super, const double* rhs, void* user);
tp_status tp_solve_partition_observe_f64(tp_ctx* ctx, const double* sub, const double* diag,
                                         const double* super, const double* rhs, int64_t n,
                                         const int64_t* sizes, int32_t nsizes, double* x,
                                         tp_interface_cb cb, void* user, tp_error* err);

/* FP32: solve_partition<float> / thomas_solve<float> (the reference templates
 * on Real, partition.hpp:61-77; test_partition.cpp:206-223). Same contracts. */
typedef void (*tp_interface_cb_f32)(int64_t level, int64_t n, const float* sub, const float* diag,
                                    const float* super, const float* rhs, void* user);
tp_status tp_solve_partition_f32(tp_ctx* ctx, const float* sub, const float* diag,
                                 const float* super, const float* rhs, int64_t n,
                                 const int64_t* sizes, int32_t nsizes, float* x, tp_error* err);
tp_status tp_solve_partition_f32_dev(tp_ctx* ctx, const float* sub, const float* diag,
                                     const float* super, const float* rhs, int64_t n,
                                     const int64_t* sizes, int32_t nsizes, float* x, void* stream,
                                     tp_error* err);
tp_status tp_solve_partition_f32_async(tp_ctx* ctx, const float* sub, const float* diag,
                                       const float* super, const float* rhs, int64_t n,
                                       const int64_t* sizes, int32_t nsizes, float* x, void* stream,
                                       tp_error* err);
tp_status tp_solve_partition_observe_f32(tp_ctx* ctx, const float* sub, const float* diag,
                                         const float* super, const float* rhs, int64_t n,
                                         const int64_t* sizes, int32_t nsizes, float* x,
                                         tp_interface_cb_f32 cb, void* user, tp_error* err);
tp_status tp_thomas_solve_f32(tp_ctx* ctx, const float* sub, const float* diag, const float* super,
                              const float* rhs, int64_t n, float* x, tp_error* err);
tp_status tp_residual_inf_f32_dev(tp_ctx* ctx, const float* sub, const float* diag,
                                  const float* super, const float* rhs, int64_t n, const float* x,
                                  double* out, void* stream, tp_error* err);
tp_status tp_reduce_block_f32(tp_ctx* ctx, const float* sub, const float* diag, const float* super,
                              const float* rhs, int64_t n, int64_t start, int64_t end, float* eq8, float* a,
                              float* beta, float* gamma, float* delta, tp_error* err);

/* thomas_solve(sys) — tridiagonal.hpp:52-72. Same solution, computed by the
 * device finishing solver (exact parallel elimination, not a sequential sweep). */
tp_status tp_thomas_solve_f64(tp_ctx* ctx, const double* sub, const double* diag,
                              const double* super, const double* rhs, int64_t n, double* x,
                              tp_error* err);

/* residual_inf(sys, x) — tridiagonal.hpp:74-87, on device pointers; runs on
 * `stream` (NULL = ctx stream, so ordered after work the caller queued there)
 * and returns when the value is on the host. */
tp_status tp_residual_inf_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                  const double* super, const double* rhs, int64_t n,
                                  const double* x, double* out, void* stream, tp_error* err);

/* reduce_block(sys, Block{start, end}) — partition.hpp:77-126. Host pointers to
 * the whole system (n rows); computed on the device with the reference's own
 * sequential arithmetic. eq8 = alpha1 beta1 gamma1 delta1 alpha2 beta2 gamma2
 * delta2; a / beta / gamma / delta (each end-start values, may be NULL) = the
 * ReducedBlock up-sweep vectors by offset from start (entry end-start-1 = 0).
 * ZeroPivotError row = the system row; block length < 2 -> INVALID_SIZE. */
tp_status tp_reduce_block_f64(tp_ctx* ctx, const double* sub, const double* diag, const double* super,
                              const double* rhs, int64_t n, int64_t start, int64_t end, double* eq8,
                              double* a, double* beta, double* gamma, double* delta, tp_error* err);

/* ------------------------------------------------ sharded (multi-GPU) solve
 * Contiguous shard [row0, row0+n_local) of a global system, one rank per GPU.
 * 1) tp_shard_reduce: all local levels + reduction of the shard to its two
 *    boundary equations, written to eq8_dev as {sub[2], diag[2], super[2], rhs[2]}
 *    (the assemble_interface rows of partition.hpp:139-149 for the shard).
 * 2) the caller all-gathers the 8 doubles of every rank (rank order).
 * 3) tp_shard_finish: solves the 2P-row top system redundantly and expands the
 *    local levels (Stage 3) into x_dev. Same ctx, pointers and sizes as step 1. */
tp_status tp_shard_reduce_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                  const double* super, const double* rhs, int64_t n_local,
                                  const int64_t* sizes, int32_t nsizes, double* eq8_dev,
                                  void* stream, tp_error* err);
tp_status tp_shard_finish_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                  const double* super, const double* rhs, int64_t n_local,
                                  const int64_t* sizes, int32_t nsizes, const double* eq_all_dev,
                                  int32_t nranks, int32_t rank, double* x_dev, void* stream,
                                  tp_error* err);

/* Fused multi-GPU solve (the collective inside the kernel, no NCCL call):
 * every rank allocates a mailbox (tp_shard_mailbox), exports it with
 * tp_ipc_get_handle, opens every peer's with tp_ipc_open_handle (CUDA IPC:
 * peer memory over NVLink/NVSwitch; same-process peers pass raw pointers),
 * then calls tp_shard_attach with all P mailboxes in rank order and a barrier
 * across ranks. tp_shard_solve_f64_dev then runs the whole shard solve as one
 * captured graph: Stage 1 levels -> a single-CTA kernel that reduces the shard
 * to its boundary pair, stores it into every peer's mailbox, waits for all P
 * pairs (bounded spin; timeout -> TP_ERR_NCCL), solves the 2P-row top system
 * (Thomas) and expands -> Stage 3 levels. All ranks must call it the same
 * number of times (the epoch flags pair the calls). */
/* A call with a different nranks frees and reallocates the mailbox: export,
 * open and attach again on every rank. */
tp_status tp_shard_mailbox(tp_ctx* ctx, int32_t nranks, void** mailbox, tp_error* err);
tp_status tp_ipc_get_handle(tp_ctx* ctx, void* dev_ptr, uint8_t* handle64, tp_error* err);
tp_status tp_ipc_open_handle(tp_ctx* ctx, const uint8_t* handle64, void** dev_ptr, tp_error* err);
tp_status tp_shard_attach(tp_ctx* ctx, int32_t nranks, int32_t rank, void* const* mailboxes,
                          tp_error* err);
tp_status tp_shard_solve_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                 const double* super, const double* rhs, int64_t n_local,
                                 const int64_t* sizes, int32_t nsizes, double* x_dev, void* stream,
                                 tp_error* err);
/* Same arguments: capture and instantiate the solve's graph without launching
 * it (graph instantiation can wait for the device to go idle, so ranks that
 * share one GPU prepare every graph before any rank's exchange is in flight). */
tp_status tp_shard_prepare_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                   const double* super, const double* rhs, int64_t n_local,
                                   const int64_t* sizes, int32_t nsizes, double* x_dev, void* stream,
                                   tp_error* err);

/* --------------------------------------------------- synthetic inputs */
/* generate_system(n, seed, delta) — bench.hpp:68-93, BIT-IDENTICAL to the
 * reference: std::mt19937_64(seed), libstdc++ uniform_real_distribution<double>
 * (-1, 1) and bernoulli_distribution(0.5), drawn sub, super, rhs, flip per row.
 * Host code, host arrays of n doubles. n < 2 or delta <= 1 -> INVALID_SIZE. */
tp_status tp_generate_system_f64(int64_t n, uint64_t seed, double delta, double* sub, double* diag,
                                 double* super, double* rhs, tp_error* err);

/* Device analogue of generate_system(n, seed, delta) — bench.hpp:68-93: same
 * distributions, counter-based (rows [row0, row0+n) of an n_global system),
 * not bit-identical to std::mt19937_64. */
tp_status tp_generate_system_f64_dev(tp_ctx* ctx, int64_t n, int64_t row0, int64_t n_global,
                                     uint64_t seed, double delta, double* sub, double* diag,
                                     double* super, double* rhs, void* stream, tp_error* err);
tp_status tp_generate_system_f32_dev(tp_ctx* ctx, int64_t n, int64_t row0, int64_t n_global,
                                     uint64_t seed, double delta, float* sub, float* diag,
                                     float* super, float* rhs, void* stream, tp_error* err);

/* ------------------------------------------------------- plan / profile */
/* make_plan(n, m) — partition.hpp:30-49. bounds (optional) gets K+1 entries. */
tp_status tp_make_plan(int64_t n, int64_t m, int64_t* bounds, int64_t* nblocks, tp_error* err);

/* Level structure the device solve will execute: per level its size and m
 * (negative m = device-internal level); n_final is the size of the system
 * handed to the finishing solver. When the deepest level runs fused with the
 * finishing solve (k_level_final_cl; needs m <= 16 and a CUDA context, whose
 * creation fixes the cluster shape) n_final may exceed 6144. */
tp_status tp_plan_levels(int64_t n, const int64_t* sizes, int32_t nsizes, int64_t* level_n,
                         int64_t* level_m, int32_t* nlevels, int32_t max_levels, int64_t* n_final,
                         tp_error* err);

/* Instrumented device solve: per-kernel durations (ms) measured with CUDA
 * events on the launch stream; names receive "<stage>:L<level>" labels. */
tp_status tp_solve_profile_f64_dev(tp_ctx* ctx, const double* sub, const double* diag,
                                   const double* super, const double* rhs, int64_t n,
                                   const int64_t* sizes, int32_t nsizes, double* x,
                                   float* kernel_ms, char* names /* [max_kernels][32] */,
                                   int32_t max_kernels, int32_t* nkernels, tp_error* err);

/* Diagnostic: max ulp distance between the solver's reciprocal (MUFU.RCP64H +
 * one cubic Newton step) and the correctly rounded 1/x over n random x. */
int tp_diag_rcp_ulp(int64_t n, uint64_t seed, uint64_t* max_ulp);

/* Diagnostic: %globaltimer phase stamps (8 per CTA: start, staged, leaves,
 * pair published, barrier passed, top tree done, expanded, stored) of the last
 * k_grid_solve launched with TPB_GRID_TRACE=1. Returns a cudaError_t. */
int tp_debug_grid_trace(unsigned long long* out, int count);

/* ------------------------------------------------------ kNN predictors */
/* predict(model, n) — knn.hpp:57-77 (feature_of :38): k-NN on log10(N);
 * distance ties -> smaller N, vote ties -> smaller label. Host code. */
tp_status tp_predict(const int64_t* pairs_n, const int32_t* pairs_label, int64_t npairs, int32_t k,
                     int64_t n, int32_t* label, tp_error* err);
/* fit_knn(train, k) — knn.hpp:40-55: validates k and sorts pairs by n (stable). */
tp_status tp_fit_knn(int64_t* pairs_n, int32_t* pairs_label, int64_t npairs, int32_t k,
                     tp_error* err);
/* recursion_sizes(n, depth, size_model) — policy.hpp:25-45 (kMaxRecursionDepth=4). */
tp_status tp_recursion_sizes(int64_t n, int32_t depth, const int64_t* pairs_n,
                             const int32_t* pairs_label, int64_t npairs, int32_t k,
                             int64_t* sizes /* >= 5 */, int32_t* nsizes, tp_error* err);
/* The bundled models: which = 0 -> fit_knn(Table I FP64 corrected, k=1),
 * which = 1 -> fit_depth_model(Table II) (test_policy.cpp:14-21),
 * which = 2 -> fit_knn(Table IV FP32 corrected, k=1). */
tp_status tp_default_model(int32_t which, int64_t* pairs_n, int32_t* pairs_label, int64_t cap,
                           int64_t* npairs, int32_t* k, tp_error* err);

/* read_observations(path) — io.hpp:80-138. Folds rows by (N, precision,
 * device); the is_opt row carries the label (m, or opt_R for depth rows). */
typedef struct tp_observation {
    int64_t n;
    int32_t label;
    int32_t corrected;      /* valid when has_corrected */
    int32_t has_corrected;
    int32_t depth_label;
    int32_t streams;
    int32_t ntimes;
    char precision[16];
    char device[48];
} tp_observation;
typedef struct tp_obs_set tp_obs_set;
tp_status tp_obs_read(const char* path, tp_obs_set** out, int64_t* count, tp_error* err);
tp_status tp_obs_get(const tp_obs_set* set, int64_t i, tp_observation* out, int32_t* cand,
                     double* times_ms /* ntimes each, may be NULL */, tp_error* err);
void tp_obs_free(tp_obs_set* set);

#ifdef __cplusplus
}
#endif

#endif /* TRIDPART_B200_H */
