// knn.hpp — drop-in for the predictor half of /root/reference/proj/include/tridpart/knn.hpp:
//   TrainingPair / HeuristicModel   knn.hpp:18-36
//   feature_of                      knn.hpp:38
//   fit_knn(ObservationSet, k)      knn.hpp:40-55  (validation + ordering in the library, tp_fit_knn)
//   predict                         knn.hpp:57-77  (host C++ in the library, tp_predict: bit-exact
//                                                   log10 distances, ties -> smaller N, vote ties ->
//                                                   smaller label)
//   accuracy                        knn.hpp:126-133
// The offline model-selection tools (split / grid_search_k / evaluate /
// alignment_report) are out of the solver path and not shadowed.
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "errors.hpp"
#include "observations.hpp"

namespace tridpart {

struct TrainingPair {
    std::int64_t n = 0;
    int label = 0;
    bool operator==(const TrainingPair&) const = default;
};

struct HeuristicModel {
    std::vector<TrainingPair> pairs;  // sorted by n
    int k = 1;
    std::string transform = "log10_n";
    std::vector<int> labels;  // label domain, ascending
    std::map<std::string, std::string> metadata;
    bool operator==(const HeuristicModel&) const = default;
};

inline double feature_of(std::int64_t n) { return std::log10(static_cast<double>(n)); }

inline HeuristicModel fit_knn(const ObservationSet& train, int k) {
    std::vector<int64_t> pn;
    std::vector<int32_t> pl;
    for (const auto& r : train.rows) {
        pn.push_back(r.n);
        pl.push_back(r.label);
    }
    tp_error e{};
    b200::throw_on(tp_fit_knn(pn.data(), pl.data(), (int64_t)pn.size(), k, &e), e);
    HeuristicModel m;
    m.k = k;
    for (std::size_t i = 0; i < pn.size(); ++i) m.pairs.push_back({pn[i], pl[i]});
    m.labels = train.unique_labels();
    m.metadata["device"] = train.rows.front().device;
    m.metadata["precision"] = train.rows.front().precision;
    return m;
}

inline int predict(const HeuristicModel& model, std::int64_t n) {
    std::vector<int64_t> pn;
    std::vector<int32_t> pl;
    for (const auto& p : model.pairs) {
        pn.push_back(p.n);
        pl.push_back(p.label);
    }
    int32_t out = 0;
    tp_error e{};
    b200::throw_on(tp_predict(pn.data(), pl.data(), (int64_t)pn.size(), model.k, n, &out, &e), e);
    return out;
}

inline double accuracy(const HeuristicModel& model, const ObservationSet& test) {
    if (test.empty()) throw InvalidSizeError("empty test set");
    std::size_t hits = 0;
    for (const auto& r : test.rows) hits += predict(model, r.n) == r.label ? 1 : 0;
    return static_cast<double>(hits) / static_cast<double>(test.size());
}

}  // namespace tridpart
