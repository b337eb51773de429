// Runner of the Catch2-compatible shim (TEST INFRASTRUCTURE): every test case
// runs once per SECTION it contains (once if it has none); prints one line per
// case and a summary; exit status 1 on any failure.
#include <cstdio>
#include <exception>

#include "catch_amalgamated.hpp"

int main() {
    auto& r = tpcatch::Registry::get();
    int failed_cases = 0;
    for (const auto& c : r.cases) {
        bool failed = false;
        int runs = 0;
        for (int target = 0;; ++target) {
            r.section_target = target;
            r.section_seen = 0;
            r.case_failed = false;
            r.info.clear();
            try {
                c.fn();
            } catch (const tpcatch::Abort&) {
            } catch (const std::exception& e) {
                std::printf("  FAILED: unexpected exception: %s\n", e.what());
                ++r.failures;
                r.case_failed = true;
            }
            failed = failed || r.case_failed;
            ++runs;
            if (target + 1 >= r.section_seen) break;  // every section has had its run
        }
        std::printf("%s  %s (%d run%s)\n", failed ? "FAIL" : "PASS", c.name.c_str(), runs, runs == 1 ? "" : "s");
        failed_cases += failed ? 1 : 0;
    }
    std::printf("%zu test cases, %d failed; %d checks, %d failed\n", r.cases.size(), failed_cases, r.checks,
                r.failures);
    if (failed_cases == 0) std::printf("All tests passed\n");
    return failed_cases == 0 ? 0 : 1;
}
