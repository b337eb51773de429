// Minimal Catch2-compatible test harness (TEST INFRASTRUCTURE): just enough of
// the Catch2 v3 surface the reference's unit tests use — TEST_CASE, flat
// SECTIONs (one section per run of its test case, as Catch2 does), CHECK /
// REQUIRE (variadic, so braced initialisers with commas work), CHECK_FALSE,
// CHECK_THROWS_AS / REQUIRE_THROWS_AS, CHECK_NOTHROW, CHECK_THAT with
// Catch::Matchers::WithinAbs / WithinRel, INFO and FAIL — so the reference's
// tests/test_{partition,tridiagonal,policy}.cpp compile unmodified against the
// drop-in headers (include/tridpart/*.hpp). The amalgamated Catch2 is not in
// this image. main() is in catch_main.cpp.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace tpcatch {

struct Abort {};  // a failed REQUIRE ends the current run of the test case

struct Registry {
    struct Case {
        std::string name;
        std::function<void()> fn;
    };
    std::vector<Case> cases;
    int section_target = 0;  // the section this run executes
    int section_seen = 0;    // sections met so far in this run
    int checks = 0, failures = 0;
    bool case_failed = false;
    std::string info;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

struct Register {
    Register(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    auto& r = Registry::get();
    ++r.checks;
    if (ok) return;
    ++r.failures;
    r.case_failed = true;
    std::printf("  FAILED %s:%d: %s%s%s\n", file, line, expr, r.info.empty() ? "" : "  [", r.info.c_str());
    if (!r.info.empty()) std::printf("]\n");
    if (fatal) throw Abort{};
}

struct Section {
    bool run;
    explicit Section(const char*) {
        auto& r = Registry::get();
        run = (r.section_seen++ == r.section_target);
    }
    explicit operator bool() const { return run; }
};

template <class M, class V>
bool match(const M& m, const V& v) {
    return m.match(v);
}

}  // namespace tpcatch

namespace Catch::Matchers {
struct WithinAbs {
    double target, margin;
    WithinAbs(double t, double m) : target(t), margin(m) {}
    bool match(double v) const { return std::fabs(v - target) <= margin; }
};
struct WithinRel {
    double target, eps;
    WithinRel(double t, double e) : target(t), eps(e) {}
    bool match(double v) const {
        return std::fabs(v - target) <= eps * std::fmax(std::fabs(v), std::fabs(target));
    }
};
}  // namespace Catch::Matchers

#define TPCATCH_CAT2(a, b) a##b
#define TPCATCH_CAT(a, b) TPCATCH_CAT2(a, b)
#define TPCATCH_CASE(fn, name)                                 \
    static void fn();                                         \
    static tpcatch::Register TPCATCH_CAT(fn, _reg)(name, &fn); \
    static void fn()
#define TEST_CASE(name, ...) TPCATCH_CASE(TPCATCH_CAT(tpcatch_case_, __LINE__), name)
#define SECTION(name, ...) if (tpcatch::Section TPCATCH_CAT(tpcatch_sec_, __LINE__){name})

#define CHECK(...) tpcatch::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) tpcatch::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) tpcatch::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) tpcatch::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define TPCATCH_THROWS_AS(expr, type, fatal)                                   \
    do {                                                                       \
        bool tpc_ok = false;                                                   \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (const type&) {                                                \
            tpc_ok = true;                                                     \
        } catch (...) {                                                        \
        }                                                                      \
        tpcatch::report(tpc_ok, #expr " throws " #type, __FILE__, __LINE__, fatal); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) TPCATCH_THROWS_AS(expr, __VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) TPCATCH_THROWS_AS(expr, __VA_ARGS__, true)
#define CHECK_NOTHROW(...)                                                              \
    do {                                                                                \
        bool tpc_ok = true;                                                             \
        try {                                                                           \
            (void)(__VA_ARGS__);                                                        \
        } catch (...) {                                                                 \
            tpc_ok = false;                                                             \
        }                                                                               \
        tpcatch::report(tpc_ok, #__VA_ARGS__ " does not throw", __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THAT(arg, ...) \
    tpcatch::report(tpcatch::match(__VA_ARGS__, (arg)), #arg " matches " #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE_THAT(arg, ...) \
    tpcatch::report(tpcatch::match(__VA_ARGS__, (arg)), #arg " matches " #__VA_ARGS__, __FILE__, __LINE__, true)
#define INFO(...) (tpcatch::Registry::get().info = std::string() + (__VA_ARGS__))
#define FAIL(...) tpcatch::report(false, "FAIL: " #__VA_ARGS__, __FILE__, __LINE__, true)
