// tridpart_b200.hpp — the whole drop-in C++20 API in one include: the
// shadows of the reference's headers under include/tridpart/ (same names,
// signatures, value semantics and exception types as
// /root/reference/proj/include/tridpart/*.hpp) on top of the C-ABI
// (tridpart_b200.h), plus the bundled models. A reference caller either keeps
// its #include "tridpart/partition.hpp" lines and swaps -I<reference>/proj/include
// for -I<repo>/include, or includes this file; both link -ltridpart_b200.
//   tridiagonal.hpp  TridiagonalSystem / thomas_solve / residual_inf
//   partition.hpp    make_plan / ReducedBlock / reduce_block / assemble_interface /
//                    back_substitute / RecursionPolicy / solve_partition (both overloads)
//   knn.hpp          TrainingPair / HeuristicModel / feature_of / fit_knn / predict / accuracy
//   policy.hpp       kMaxRecursionDepth / fit_depth_model / recursion_sizes
//   observations.hpp Observation / ObservationSet (with_corrected_labels, ...)
//   io.hpp           read_observations
//   bench.hpp        generate_system (bit-identical) / Clock / time_solve
//   errors.hpp       the Error hierarchy (+ DeviceError)
#pragma once

#include <map>

#include "tridpart/bench.hpp"
#include "tridpart/errors.hpp"
#include "tridpart/io.hpp"
#include "tridpart/knn.hpp"
#include "tridpart/observations.hpp"
#include "tridpart/partition.hpp"
#include "tridpart/policy.hpp"
#include "tridpart/tridiagonal.hpp"

namespace tridpart {

namespace b200 {
inline HeuristicModel bundled(int which) {
    tp_error e{};
    int64_t cnt = 0;
    int32_t k = 1;
    throw_on(tp_default_model(which, nullptr, nullptr, 0, &cnt, &k, &e), e);
    std::vector<int64_t> n((std::size_t)cnt);
    std::vector<int32_t> l((std::size_t)cnt);
    throw_on(tp_default_model(which, n.data(), l.data(), cnt, &cnt, &k, &e), e);
    HeuristicModel m;
    m.k = k;
    for (int64_t i = 0; i < cnt; ++i) m.pairs.push_back({n[(std::size_t)i], l[(std::size_t)i]});
    std::map<int, int> seen;
    for (auto v : l) seen[v] = 1;
    for (auto& [v, _] : seen) m.labels.push_back(v);
    return m;
}
}  // namespace b200

// The models the reference's tests fit, bundled in the library (no CSV needed):
// fit_knn(read_observations(table1_fp64.csv).with_corrected_labels(), 1) and
// fit_depth_model(read_observations(table2_recursion.csv)) (test_policy.cpp:14-21);
// default_fp32_size_model: Table IV (FP32) with corrected labels.
inline HeuristicModel default_size_model() { return b200::bundled(0); }
inline HeuristicModel default_fp32_size_model() { return b200::bundled(2); }
inline HeuristicModel default_depth_model() { return b200::bundled(1); }

}  // namespace tridpart
