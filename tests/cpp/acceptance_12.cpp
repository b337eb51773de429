// Acceptance criteria 1 and 2 of the reference (proj/tests/acceptance.cpp:72-123)
// run against the B200 solver through the drop-in headers (TEST INFRASTRUCTURE).
// Same case lists as the reference: std::mt19937_64(20240601) draws 200
// systems (n in [10, 100000], depth 0..4, m from {2,4,7,8,16,20,32,40,64}) and
// std::mt19937_64(7) draws 1000 (n in [10, 2009], depth 0..2, m in [2, 16]);
// generate_system is bit-identical, so these are the reference's systems.
//   criterion 1: rel_inf_diff(solve_partition, thomas_solve) <= 1e-10 on all
//                200, in < 120 s (acceptance.cpp:72-100)
//   criterion 2: every interface the observer sees is diagonally dominant to
//                1e-12 slack (acceptance.cpp:102-123)
// Exit status 0 when both pass.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "tridpart/bench.hpp"
#include "tridpart/partition.hpp"
#include "tridpart/tridiagonal.hpp"

using namespace tridpart;

namespace {

// tests/oracles.hpp:46-53
double rel_inf_diff(const std::vector<double>& a, const std::vector<double>& b) {
    double diff = 0, scale = 1;
    for (std::size_t i = 0; i < a.size(); ++i) {
        diff = std::max(diff, std::fabs(a[i] - b[i]));
        scale = std::max(scale, std::fabs(b[i]));
    }
    return diff / scale;
}

bool criterion1() {
    const auto t0 = std::chrono::steady_clock::now();
    std::mt19937_64 rng(20240601);
    const std::vector<std::size_t> choices = {2, 4, 7, 8, 16, 20, 32, 40, 64};
    double worst = 0;
    std::string where;
    int done = 0;
    for (int t = 0; t < 200; ++t) {
        const std::size_t n = 10 + rng() % (100000 - 10 + 1);
        const int depth = int(rng() % 5);
        RecursionPolicy policy;
        for (int l = 0; l <= depth; ++l) policy.sizes.push_back(choices[rng() % choices.size()]);
        const auto sys = generate_system(n, rng());
        const auto ref = thomas_solve(sys);
        const auto x = solve_partition(sys, policy);
        const double d = rel_inf_diff(x, ref);
        if (!(d <= worst)) {
            worst = d;
            where = "n=" + std::to_string(n);
        }
        ++done;
        if (!(d <= 1e-10)) break;
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool ok = done == 200 && worst <= 1e-10 && secs < 120.0;
    std::printf("%s  criterion 1: partition/Thomas equivalence over 200 random systems  "
                "[worst rel_inf_diff %.3e at %s, %.2f s]\n",
                ok ? "PASS" : "FAIL", worst, where.c_str(), secs);
    return ok;
}

bool criterion2() {
    std::mt19937_64 rng(7);
    bool ok = true;
    std::string detail;
    long levels = 0;
    for (int t = 0; t < 1000 && ok; ++t) {
        const std::size_t n = 10 + rng() % 2000;
        const int depth = int(rng() % 3);
        RecursionPolicy policy;
        for (int l = 0; l <= depth; ++l) policy.sizes.push_back(2 + rng() % 15);
        const auto sys = generate_system(n, rng());
        solve_partition(sys, policy, [&](const Tridiagonal& f, std::size_t) {
            ++levels;
            for (std::size_t i = 0; i < f.size(); ++i)
                if (!(std::fabs(f.diag[i]) >= std::fabs(f.sub[i]) + std::fabs(f.super[i]) - 1e-12)) {
                    ok = false;
                    detail = "n=" + std::to_string(n) + " row " + std::to_string(i);
                }
        });
    }
    std::printf("%s  criterion 2: interface systems preserve diagonal dominance (1000 systems, %ld levels)%s%s\n",
                ok ? "PASS" : "FAIL", levels, detail.empty() ? "" : "  ", detail.c_str());
    return ok;
}

}  // namespace

int main() {
    const bool a = criterion1();
    const bool b = criterion2();
    return (a && b) ? 0 : 1;
}
