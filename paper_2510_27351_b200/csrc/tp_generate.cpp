// generate_system(n, seed, delta) — bench.hpp:68-93, bit-identical to the
// reference: the same standard-library engine and distributions (libstdc++
// std::mt19937_64, uniform_real_distribution<double>(-1, 1),
// bernoulli_distribution(0.5)) consumed in the same order per row — sub (not
// row 0), super (not row n-1), rhs, then the whole-row sign flip. Host code;
// built with -ffp-contract=off so diag = delta*(|a|+|c|)+1 rounds as the
// reference's x86-64 build does (no FMA).
#include <cmath>
#include <cstdio>
#include <random>

#include "../../include/tridpart_b200.h"

extern "C" tp_status tp_generate_system_f64(int64_t n, uint64_t seed, double delta, double* sub, double* diag,
                                            double* super, double* rhs, tp_error* err) {
    auto fail = [&](tp_status code, const char* msg) {
        if (err) {
            err->code = code;
            err->row = -1;
            err->level = -1;
            std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
        }
        return code;
    };
    if (err) {
        err->code = TP_OK;
        err->row = -1;
        err->level = -1;
        err->msg[0] = 0;
    }
    if (n < 2) return fail(TP_ERR_INVALID_SIZE, "system size must be >= 2");
    if (!(delta > 1.0)) return fail(TP_ERR_INVALID_SIZE, "dominance factor must be > 1");
    if (!sub || !diag || !super || !rhs) return fail(TP_ERR_INVALID_ARGUMENT, "null array pointer");
    std::mt19937_64 engine(seed);
    std::uniform_real_distribution<double> unit(-1.0, 1.0);
    std::bernoulli_distribution coin(0.5);
    for (int64_t i = 0; i < n; ++i) {
        const double a = i > 0 ? unit(engine) : 0.0;
        const double c = i + 1 < n ? unit(engine) : 0.0;
        const double b = delta * (std::abs(a) + std::abs(c)) + 1.0;
        const double d = unit(engine);
        const bool neg = coin(engine);
        sub[i] = neg ? -a : a;
        diag[i] = neg ? -b : b;
        super[i] = neg ? -c : c;
        rhs[i] = neg ? -d : d;
    }
    return TP_OK;
}
