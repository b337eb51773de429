// policy.hpp — drop-in for /root/reference/proj/include/tridpart/policy.hpp:
//   kMaxRecursionDepth   policy.hpp:11
//   fit_depth_model      policy.hpp:14-16
//   recursion_sizes      policy.hpp:25-45 (tp_recursion_sizes: m0 = predict(N), m1 = 10 when
//                        R >= 2, deeper levels predicted on N_{l+1} = 2 K_l)
#pragma once

#include <cstdint>
#include <vector>

#include "errors.hpp"
#include "knn.hpp"
#include "partition.hpp"

namespace tridpart {

inline constexpr int kMaxRecursionDepth = 4;

inline HeuristicModel fit_depth_model(const ObservationSet& data, int k = 1) { return fit_knn(data, k); }

inline RecursionPolicy recursion_sizes(std::int64_t n, int depth, const HeuristicModel& size_model) {
    std::vector<int64_t> pn;
    std::vector<int32_t> pl;
    for (const auto& p : size_model.pairs) {
        pn.push_back(p.n);
        pl.push_back(p.label);
    }
    int64_t sizes[kMaxRecursionDepth + 1];
    int32_t cnt = 0;
    tp_error e{};
    b200::throw_on(tp_recursion_sizes(n, depth, pn.data(), pl.data(), (int64_t)pn.size(), size_model.k, sizes,
                                      &cnt, &e),
                   e);
    RecursionPolicy p;
    for (int32_t i = 0; i < cnt; ++i) p.sizes.push_back((std::size_t)sizes[i]);
    return p;
}

}  // namespace tridpart
