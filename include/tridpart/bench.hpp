// bench.hpp — drop-in for the solver-facing half of /root/reference/proj/include/tridpart/bench.hpp:
//   kBenchResidualTol / Clock / SteadyClock / TraceClock   bench.hpp:22-63
//   generate_system                                        bench.hpp:68-93 — bit-identical: the
//       library's tp_generate_system_f64 runs std::mt19937_64(seed) with libstdc++'s
//       uniform_real_distribution<double>(-1, 1) and bernoulli_distribution(0.5), drawing
//       sub, super, rhs, flip per row in the reference's order
//   TimingStats / time_solve                               bench.hpp:95-127 (the B200 solve
//       under the same residual gate and median statistic)
// The m / R sweeps (sweep_m / sweep_r) are driven from Python (paper_2510_27351_b200/sweep.py).
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <functional>
#include <string>
#include <utility>
#include <vector>

#include "errors.hpp"
#include "observations.hpp"
#include "partition.hpp"
#include "policy.hpp"
#include "tridiagonal.hpp"

namespace tridpart {

inline constexpr double kBenchResidualTol = 1e-8;

class Clock {
public:
    virtual ~Clock() = default;
    virtual double time_ms(const std::function<void()>& work) = 0;
    virtual std::string name() const = 0;
};

class SteadyClock final : public Clock {
public:
    double time_ms(const std::function<void()>& work) override {
        const auto t0 = std::chrono::steady_clock::now();
        work();
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    std::string name() const override { return "steady"; }
};

// Replays a scripted trace (the workload still runs, so the gate stays in force).
class TraceClock final : public Clock {
public:
    explicit TraceClock(std::vector<double> trace_ms) : trace_(std::move(trace_ms)) {
        if (trace_.empty()) throw InvalidSizeError("empty clock trace");
    }
    double time_ms(const std::function<void()>& work) override {
        work();
        return trace_[next_++ % trace_.size()];
    }
    std::string name() const override { return "trace"; }

private:
    std::vector<double> trace_;
    std::size_t next_ = 0;
};

inline Tridiagonal generate_system(std::size_t n, std::uint64_t seed, double delta = 1.5) {
    Tridiagonal s;
    if (n >= 2) {
        s.sub.resize(n);
        s.diag.resize(n);
        s.super.resize(n);
        s.rhs.resize(n);
    }
    tp_error e{};
    b200::throw_on(tp_generate_system_f64((int64_t)n, seed, delta, s.sub.data(), s.diag.data(), s.super.data(),
                                          s.rhs.data(), &e),
                   e);
    return s;
}

struct TimingStats {
    double median_ms = 0;
    double min_ms = 0;
    double max_ms = 0;
    int runs = 0;
};

// 1 warm-up + `runs` timed solves, each gated on residual_inf <= kBenchResidualTol.
inline TimingStats time_solve(const Tridiagonal& sys, const RecursionPolicy& policy, int runs, Clock& clock) {
    if (runs < 1) throw InvalidSizeError("runs must be >= 1");
    auto gated = [&] {
        const auto x = solve_partition(sys, policy);
        const double res = residual_inf(sys, x);
        if (!(res <= kBenchResidualTol)) throw SolveFailedError("residual " + std::to_string(res) + " above gate");
    };
    gated();
    std::vector<double> t((std::size_t)runs);
    for (auto& v : t) v = clock.time_ms(gated);
    std::sort(t.begin(), t.end());
    TimingStats st;
    st.runs = runs;
    st.min_ms = t.front();
    st.max_ms = t.back();
    const std::size_t h = (std::size_t)runs / 2;
    st.median_ms = (runs % 2) ? t[h] : 0.5 * (t[h - 1] + t[h]);
    return st;
}

}  // namespace tridpart
