/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference `tridpart` CPU algorithm for the FP64
 * partition solve and the kNN policy predictors. It is the parity CHECKER:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product path
 * (paper_2510_27351_b200/) never links or calls it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/). Operation order follows the
 * reference exactly and the file is compiled with -ffp-contract=off, so on the
 * same toolchain results are bit-identical to the reference's own headers
 * (pinned by tests/test_oracle.py against oracle/_ref).
 *
 * Error convention: functions returning int64_t return -1 on success, or the
 * row index of a zero pivot (ZeroPivotError(row), include/tridpart/errors.hpp:16-24),
 * or -2 for InvalidSizeError (errors.hpp:26-29).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK (-1)
#define ORC_INVALID_SIZE (-2)
#define ORC_DEPTH_OUT_OF_RANGE (-3)

/* kPivotFloor<double> = 1e-30 — include/tridpart/tridiagonal.hpp:15-16 */
static const double kPivotFloor = 1e-30;

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (the C++ standard's parameters) + libstdc++ distributions  */
/* as used by generate_system — include/tridpart/bench.hpp:68-93.            */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_mt64;

static void mt64_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(orc_mt64* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* libstdc++ std::generate_canonical<double, 53>(mt19937_64): one draw,
 * sum = double(x), ret = sum / 2^64, clamped below 1. */
static double canonical(orc_mt64* g) {
    double sum = (double)mt64_next(g);
    double ret = sum / 18446744073709551616.0;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}

/* std::uniform_real_distribution<double>(-1, 1): canonical * (b - a) + a */
static double unit(orc_mt64* g) { return canonical(g) * 2.0 + -1.0; }

/* std::bernoulli_distribution(0.5): canonical < p * (max - min) */
static int flip(orc_mt64* g) { return canonical(g) < 0.5 * 1.0; }

/* generate_system(n, seed, delta) — include/tridpart/bench.hpp:68-93.
 * Draw order per row: sub (skipped at i=0), super (skipped at n-1), rhs, flip. */
int64_t orc_generate_system(int64_t n, uint64_t seed, double delta, double* sub, double* diag,
                            double* sup, double* rhs) {
    if (n < 2) return ORC_INVALID_SIZE;
    if (!(delta > 1.0)) return ORC_INVALID_SIZE;
    orc_mt64 g;
    mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) {
        sub[i] = (i == 0) ? 0.0 : unit(&g);
        sup[i] = (i + 1 == n) ? 0.0 : unit(&g);
        diag[i] = delta * (fabs(sub[i]) + fabs(sup[i])) + 1.0;
        rhs[i] = unit(&g);
        if (flip(&g)) {
            sub[i] = -sub[i];
            diag[i] = -diag[i];
            sup[i] = -sup[i];
            rhs[i] = -rhs[i];
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Sequential kernels — include/tridpart/tridiagonal.hpp                     */
/* ------------------------------------------------------------------------ */

/* thomas_solve — tridiagonal.hpp:52-72. Returns ORC_OK or the zero-pivot row. */
int64_t orc_thomas_solve(int64_t n, const double* sub, const double* diag, const double* sup,
                         const double* rhs, double* x) {
    if (n <= 0) return ORC_INVALID_SIZE;
    double* c_mod = (double*)malloc((size_t)n * sizeof(double));
    double pivot = diag[0];
    if (fabs(pivot) < kPivotFloor) { free(c_mod); return 0; }
    c_mod[0] = sup[0] / pivot;
    x[0] = rhs[0] / pivot;
    for (int64_t i = 1; i < n; ++i) {
        pivot = diag[i] - sub[i] * c_mod[i - 1];
        if (fabs(pivot) < kPivotFloor) { free(c_mod); return i; }
        c_mod[i] = sup[i] / pivot;
        x[i] = (rhs[i] - sub[i] * x[i - 1]) / pivot;
    }
    for (int64_t i = n - 1; i-- > 0;) x[i] -= c_mod[i] * x[i + 1];
    free(c_mod);
    return ORC_OK;
}

/* residual_inf — tridiagonal.hpp:74-87: ||Ax - d||_inf / max(1, ||d||_inf) */
double orc_residual_inf(int64_t n, const double* sub, const double* diag, const double* sup,
                        const double* rhs, const double* x) {
    double num = 0, den = 1;
    for (int64_t i = 0; i < n; ++i) {
        double ax = diag[i] * x[i];
        if (i > 0) ax += sub[i] * x[i - 1];
        if (i + 1 < n) ax += sup[i] * x[i + 1];
        double r = fabs(ax - rhs[i]);
        if (r > num) num = r;
        double d = fabs(rhs[i]);
        if (d > den) den = d;
    }
    return num / den;
}

/* ------------------------------------------------------------------------ */
/* Partition method — include/tridpart/partition.hpp                         */
/* ------------------------------------------------------------------------ */

/* make_plan — partition.hpp:30-49. Writes block starts (K+1 entries, the last
 * equal to n) when `bounds` is non-NULL; returns K or ORC_INVALID_SIZE. */
int64_t orc_make_plan(int64_t n, int64_t m, int64_t* bounds) {
    if (n < 2) return ORC_INVALID_SIZE;
    if (m < 2) return ORC_INVALID_SIZE;
    if (m >= n) {
        if (bounds) { bounds[0] = 0; bounds[1] = n; }
        return 1;
    }
    int64_t leading = n / m;
    if (n % m <= 1) --leading;
    if (bounds) {
        int64_t pos = 0;
        for (int64_t b = 0; b < leading; ++b, pos += m) bounds[b] = pos;
        bounds[leading] = pos;
        bounds[leading + 1] = n;
    }
    return leading + 1;
}

/* ReducedBlock — partition.hpp:61-71. The up-sweep vectors are stored in a
 * caller-owned slab (4 * len doubles) so the recursion frees them per level. */
typedef struct {
    int64_t start, end;
    double alpha1, beta1, gamma1, delta1;
    double alpha2, beta2, gamma2, delta2;
    double *a, *beta, *gamma, *delta;
} orc_reduced;

/* reduce_block — partition.hpp:77-126 (up-sweep :90-108, down-sweep :110-124). */
static int64_t reduce_block(const double* sub, const double* diag, const double* sup,
                            const double* rhs, int64_t start, int64_t end, orc_reduced* out) {
    const int64_t s = start, e = end - 1, len = end - start;
    if (len < 2) return ORC_INVALID_SIZE;
    out->start = start;
    out->end = end;
#define OFF(i) ((i) - s)
    out->a[OFF(e - 1)] = sub[e - 1];
    out->beta[OFF(e - 1)] = diag[e - 1];
    out->gamma[OFF(e - 1)] = sup[e - 1];
    out->delta[OFF(e - 1)] = rhs[e - 1];
    for (int64_t i = e - 1; i-- > s;) {
        const double piv = out->beta[OFF(i + 1)];
        if (fabs(piv) < kPivotFloor) return i + 1;
        const double w = sup[i] / piv;
        out->a[OFF(i)] = sub[i];
        out->beta[OFF(i)] = diag[i] - w * sub[i + 1];
        out->gamma[OFF(i)] = -w * out->gamma[OFF(i + 1)];
        out->delta[OFF(i)] = rhs[i] - w * out->delta[OFF(i + 1)];
    }
    out->alpha1 = sub[s];
    out->beta1 = out->beta[0];
    out->gamma1 = out->gamma[0];
    out->delta1 = out->delta[0];

    double phi = sub[s + 1];
    double beta_p = diag[s + 1];
    double delta_p = rhs[s + 1];
    for (int64_t i = s + 2; i <= e; ++i) {
        if (fabs(beta_p) < kPivotFloor) return i - 1;
        const double w = sub[i] / beta_p;
        phi = -w * phi;
        beta_p = diag[i] - w * sup[i - 1];
        delta_p = rhs[i] - w * delta_p;
    }
    out->alpha2 = phi;
    out->beta2 = beta_p;
    out->gamma2 = sup[e];
    out->delta2 = delta_p;
#undef OFF
    return ORC_OK;
}

/* back_substitute — partition.hpp:156-172; writes len-2 interior values. */
static int64_t back_substitute(const orc_reduced* blk, double x_s, double x_e, double* interior) {
    const int64_t len = blk->end - blk->start;
    if (len <= 2) return ORC_OK;
    double prev = x_s;
    for (int64_t off = 1; off + 1 < len; ++off) {
        if (fabs(blk->beta[off]) < kPivotFloor) return blk->start + off;
        const double xi = (blk->delta[off] - blk->a[off] * prev - blk->gamma[off] * x_e) / blk->beta[off];
        interior[off - 1] = xi;
        prev = xi;
    }
    return ORC_OK;
}

/* Observer hook: on_interface(iface, level) — partition.hpp:206 */
typedef void (*orc_observer)(int64_t level, int64_t n, const double* sub, const double* diag,
                             const double* sup, const double* rhs, void* user);

/* detail::solve_partition_level — partition.hpp:191-224. The reference's two
 * parallel_for loops (:203, :214) are sequential loops here: per-index slot
 * writes make the result schedule-independent (parallel.hpp:9-10). */
static int64_t solve_level(int64_t n, const double* sub, const double* diag, const double* sup,
                           const double* rhs, const int64_t* sizes, int64_t nlevels, int64_t level,
                           double* x, orc_observer obs, void* user, int64_t* err_level) {
    if (n < 4) {
        int64_t r = orc_thomas_solve(n, sub, diag, sup, rhs, x);
        if (r != ORC_OK) *err_level = level;
        return r;
    }
    const int64_t m = sizes[level];
    const int64_t k = orc_make_plan(n, m, NULL);
    if (k < 0) return k;
    int64_t* bounds = (int64_t*)malloc((size_t)(k + 1) * sizeof(int64_t));
    orc_make_plan(n, m, bounds);

    orc_reduced* red = (orc_reduced*)calloc((size_t)k, sizeof(orc_reduced));
    double* slab = (double*)malloc((size_t)n * 4 * sizeof(double));
    int64_t status = ORC_OK;
    for (int64_t j = 0; j < k && status == ORC_OK; ++j) {
        const int64_t s = bounds[j];
        red[j].a = slab + s;
        red[j].beta = slab + n + s;
        red[j].gamma = slab + 2 * n + s;
        red[j].delta = slab + 3 * n + s;
        status = reduce_block(sub, diag, sup, rhs, bounds[j], bounds[j + 1], &red[j]);
    }
    double* iface = NULL;
    double* ix = NULL;
    if (status == ORC_OK) {
        /* assemble_interface — partition.hpp:131-151 */
        const int64_t n2 = 2 * k;
        iface = (double*)malloc((size_t)n2 * 4 * sizeof(double));
        double *isub = iface, *idiag = iface + n2, *isup = iface + 2 * n2, *irhs = iface + 3 * n2;
        for (int64_t j = 0; j < k; ++j) {
            isub[2 * j] = red[j].alpha1;
            idiag[2 * j] = red[j].beta1;
            isup[2 * j] = red[j].gamma1;
            irhs[2 * j] = red[j].delta1;
            isub[2 * j + 1] = red[j].alpha2;
            idiag[2 * j + 1] = red[j].beta2;
            isup[2 * j + 1] = red[j].gamma2;
            irhs[2 * j + 1] = red[j].delta2;
        }
        if (obs) obs(level, n2, isub, idiag, isup, irhs, user);
        ix = (double*)malloc((size_t)n2 * sizeof(double));
        if (level < nlevels - 1) {
            status = solve_level(n2, isub, idiag, isup, irhs, sizes, nlevels, level + 1, ix, obs,
                                 user, err_level);
        } else {
            status = orc_thomas_solve(n2, isub, idiag, isup, irhs, ix);
            if (status != ORC_OK) *err_level = level + 1;
        }
        for (int64_t j = 0; j < k && status == ORC_OK; ++j) {
            const double x_s = ix[2 * j], x_e = ix[2 * j + 1];
            x[red[j].start] = x_s;
            x[red[j].end - 1] = x_e;
            status = back_substitute(&red[j], x_s, x_e, x + red[j].start + 1);
            if (status != ORC_OK) *err_level = level;
        }
    } else {
        *err_level = level;
    }
    free(ix);
    free(iface);
    free(slab);
    free(red);
    free(bounds);
    return status;
}

/* solve_partition — partition.hpp:235-248 (policy.valid() :181-186). */
int64_t orc_solve_partition(int64_t n, const double* sub, const double* diag, const double* sup,
                            const double* rhs, const int64_t* sizes, int64_t nlevels, double* x,
                            orc_observer obs, void* user, int64_t* err_level) {
    int64_t dummy = 0;
    if (!err_level) err_level = &dummy;
    if (nlevels < 1) return ORC_INVALID_SIZE;
    for (int64_t l = 0; l < nlevels; ++l)
        if (sizes[l] < 2) return ORC_INVALID_SIZE;
    if (n == 0) return ORC_INVALID_SIZE;
    return solve_level(n, sub, diag, sup, rhs, sizes, nlevels, 0, x, obs, user, err_level);
}

/* Stage-1 diagnostic: reduce_block on one block, output 8 interface scalars
 * (alpha1, beta1, gamma1, delta1, alpha2, beta2, gamma2, delta2). */
int64_t orc_reduce_block(const double* sub, const double* diag, const double* sup,
                         const double* rhs, int64_t start, int64_t end, double* eq8) {
    const int64_t len = end - start;
    if (len < 2) return ORC_INVALID_SIZE;
    double* slab = (double*)malloc((size_t)len * 4 * sizeof(double));
    orc_reduced r;
    r.a = slab; r.beta = slab + len; r.gamma = slab + 2 * len; r.delta = slab + 3 * len;
    int64_t st = reduce_block(sub, diag, sup, rhs, start, end, &r);
    if (st == ORC_OK) {
        eq8[0] = r.alpha1; eq8[1] = r.beta1; eq8[2] = r.gamma1; eq8[3] = r.delta1;
        eq8[4] = r.alpha2; eq8[5] = r.beta2; eq8[6] = r.gamma2; eq8[7] = r.delta2;
    }
    free(slab);
    return st;
}

/* ------------------------------------------------------------------------ */
/* kNN predictors — include/tridpart/knn.hpp:38,57-77; policy.hpp:11-45      */
/* ------------------------------------------------------------------------ */

typedef struct {
    double dist;
    int64_t n;
    int label;
} orc_ranked;

static int ranked_cmp(const void* pa, const void* pb) {
    const orc_ranked* a = (const orc_ranked*)pa;
    const orc_ranked* b = (const orc_ranked*)pb;
    /* std::tuple<double, int64, int> operator< : lexicographic */
    if (a->dist < b->dist) return -1;
    if (b->dist < a->dist) return 1;
    if (a->n < b->n) return -1;
    if (b->n < a->n) return 1;
    if (a->label < b->label) return -1;
    if (b->label < a->label) return 1;
    return 0;
}

/* feature_of — knn.hpp:38 */
static double feature_of(int64_t n) { return log10((double)n); }

/* predict — knn.hpp:57-77. pairs_n / pairs_label: the fitted model's pairs
 * (fit_knn, knn.hpp:40-55). Votes: std::map ascending + strict '>' means the
 * smallest label wins a count tie. */
int orc_predict(const int64_t* pairs_n, const int* pairs_label, int64_t npairs, int k, int64_t n) {
    const double q = feature_of(n);
    orc_ranked* r = (orc_ranked*)malloc((size_t)npairs * sizeof(orc_ranked));
    for (int64_t i = 0; i < npairs; ++i) {
        r[i].dist = fabs(feature_of(pairs_n[i]) - q);
        r[i].n = pairs_n[i];
        r[i].label = pairs_label[i];
    }
    qsort(r, (size_t)npairs, sizeof(orc_ranked), ranked_cmp);
    /* first k labels; mode with ties -> smallest label */
    int best_label = 0, best_count = -1;
    int* labs = (int*)malloc((size_t)k * sizeof(int));
    for (int i = 0; i < k; ++i) labs[i] = r[i].label;
    /* iterate distinct labels ascending, as std::map does */
    for (;;) {
        int have = 0, cur = 0;
        for (int i = 0; i < k; ++i) {
            if (labs[i] == -2147483647 - 1) continue;
            if (!have || labs[i] < cur) { cur = labs[i]; have = 1; }
        }
        if (!have) break;
        int count = 0;
        for (int i = 0; i < k; ++i)
            if (labs[i] == cur) { ++count; labs[i] = -2147483647 - 1; }
        if (count > best_count) { best_label = cur; best_count = count; }
    }
    free(labs);
    free(r);
    return best_label;
}

/* recursion_sizes — policy.hpp:25-45 (kMaxRecursionDepth = 4, :11).
 * Writes depth+1 sizes; returns depth+1 or ORC_DEPTH_OUT_OF_RANGE. */
int64_t orc_recursion_sizes(int64_t n, int depth, const int64_t* pairs_n, const int* pairs_label,
                            int64_t npairs, int k, int64_t* sizes) {
    if (depth < 0 || depth > 4) return ORC_DEPTH_OUT_OF_RANGE;
    int64_t level_n = n;
    for (int level = 0; level <= depth; ++level) {
        int64_t m;
        if (level == 1 && depth >= 2) m = 10;
        else m = orc_predict(pairs_n, pairs_label, npairs, k, level_n);
        sizes[level] = m;
        if (level == depth) break;
        const int64_t kb = orc_make_plan(level_n, m, NULL);
        if (kb < 0) return kb;
        level_n = 2 * kb;
    }
    return depth + 1;
}
