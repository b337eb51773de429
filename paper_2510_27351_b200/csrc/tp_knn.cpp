// Host-side policy predictors and the observation reader (C++, no device code).
//
// These stay on the host on purpose: the reference predicts with host double
// math (std::log10, knn.hpp:38) and a (distance, N, label) ordering
// (knn.hpp:57-77); evaluating the same expression with the same libm on the
// host is what makes m and R bit-exact. Compiled without -ffast-math.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <optional>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/tridpart_b200.h"
#include "tp_models_data.h"

namespace {

void set_err(tp_error* err, tp_status code, const std::string& msg) {
    if (!err) return;
    err->code = code;
    err->row = -1;
    err->level = -1;
    std::snprintf(err->msg, sizeof(err->msg), "%s", msg.c_str());
}
void clear_err(tp_error* err) {
    if (!err) return;
    err->code = TP_OK;
    err->row = -1;
    err->level = -1;
    err->msg[0] = 0;
}

// feature_of — knn.hpp:38
inline double log_size(int64_t n) { return std::log10(static_cast<double>(n)); }

struct Neighbour {
    double dist;
    int64_t n;
    int32_t label;
};
inline bool closer(const Neighbour& x, const Neighbour& y) {
    if (x.dist != y.dist) return x.dist < y.dist;
    if (x.n != y.n) return x.n < y.n;
    return x.label < y.label;
}

int32_t knn_vote(const int64_t* pn, const int32_t* pl, int64_t np, int32_t k, int64_t n) {
    const double q = log_size(n);
    std::vector<Neighbour> nb((size_t)np);
    for (int64_t i = 0; i < np; ++i) nb[(size_t)i] = {std::fabs(log_size(pn[i]) - q), pn[i], pl[i]};
    // only the k nearest matter: a partial sort on the full key is equivalent
    // to the reference's full sort of the (distance, n, label) tuples
    std::partial_sort(nb.begin(), nb.begin() + k, nb.end(), closer);
    std::vector<int32_t> labels((size_t)k);
    for (int32_t i = 0; i < k; ++i) labels[(size_t)i] = nb[(size_t)i].label;
    std::sort(labels.begin(), labels.end());
    // mode; on a count tie the smallest label (first in ascending order) wins
    int32_t best = labels[0], best_count = 0;
    for (size_t i = 0; i < labels.size();) {
        size_t j = i;
        while (j < labels.size() && labels[j] == labels[i]) ++j;
        if ((int32_t)(j - i) > best_count) {
            best = labels[i];
            best_count = (int32_t)(j - i);
        }
        i = j;
    }
    return best;
}

int64_t blocks_of(int64_t n, int64_t m) {  // make_plan block count, partition.hpp:30-49
    if (m >= n) return 1;
    int64_t leading = n / m;
    if (n % m <= 1) --leading;
    return leading + 1;
}

}  // namespace

struct tp_obs_set {
    struct Row {
        tp_observation o;
        std::vector<int32_t> cand;
        std::vector<double> times;
    };
    std::vector<Row> rows;
};

extern "C" {

tp_status tp_predict(const int64_t* pairs_n, const int32_t* pairs_label, int64_t npairs, int32_t k,
                     int64_t n, int32_t* label, tp_error* err) {
    clear_err(err);
    if (!pairs_n || !pairs_label || !label) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    if (npairs < 1) {
        set_err(err, TP_ERR_EMPTY_TRAINING_SET, "training set is empty");
        return TP_ERR_EMPTY_TRAINING_SET;
    }
    if (k < 1 || k > npairs) {
        set_err(err, TP_ERR_K_TOO_LARGE, "k must be in [1, |train|]");
        return TP_ERR_K_TOO_LARGE;
    }
    *label = knn_vote(pairs_n, pairs_label, npairs, k, n);
    return TP_OK;
}

tp_status tp_fit_knn(int64_t* pairs_n, int32_t* pairs_label, int64_t npairs, int32_t k,
                     tp_error* err) {
    clear_err(err);
    if (npairs < 1) {
        set_err(err, TP_ERR_EMPTY_TRAINING_SET, "training set is empty");
        return TP_ERR_EMPTY_TRAINING_SET;
    }
    if (k < 1 || k > npairs) {
        set_err(err, TP_ERR_K_TOO_LARGE, "k must be in [1, |train|]");
        return TP_ERR_K_TOO_LARGE;
    }
    if (!pairs_n || !pairs_label) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    std::vector<std::pair<int64_t, int32_t>> v((size_t)npairs);
    for (int64_t i = 0; i < npairs; ++i) v[(size_t)i] = {pairs_n[i], pairs_label[i]};
    std::stable_sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    for (int64_t i = 0; i < npairs; ++i) {
        pairs_n[i] = v[(size_t)i].first;
        pairs_label[i] = v[(size_t)i].second;
    }
    return TP_OK;
}

tp_status tp_recursion_sizes(int64_t n, int32_t depth, const int64_t* pairs_n,
                             const int32_t* pairs_label, int64_t npairs, int32_t k, int64_t* sizes,
                             int32_t* nsizes, tp_error* err) {
    clear_err(err);
    if (depth < 0 || depth > 4) {  // kMaxRecursionDepth, policy.hpp:11,27-28
        set_err(err, TP_ERR_DEPTH_OUT_OF_RANGE, "recursion depth must be in [0, 4]");
        return TP_ERR_DEPTH_OUT_OF_RANGE;
    }
    if (!sizes || !nsizes) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    int64_t level_n = n;
    for (int32_t level = 0; level <= depth; ++level) {
        int64_t m;
        if (level == 1 && depth >= 2) {
            m = 10;  // "fix m1 to 10" (policy.hpp:34-35)
        } else {
            int32_t lab = 0;
            tp_status s = tp_predict(pairs_n, pairs_label, npairs, k, level_n, &lab, err);
            if (s != TP_OK) return s;
            m = lab;
        }
        sizes[level] = m;
        if (level == depth) break;
        if (level_n < 2 || m < 2) {  // make_plan's own checks (partition.hpp:31-32)
            set_err(err, TP_ERR_INVALID_SIZE,
                    level_n < 2 ? "system size must be >= 2" : "sub-system size must be >= 2");
            return TP_ERR_INVALID_SIZE;
        }
        level_n = 2 * blocks_of(level_n, m);
    }
    *nsizes = depth + 1;
    return TP_OK;
}

tp_status tp_default_model(int32_t which, int64_t* pairs_n, int32_t* pairs_label, int64_t cap,
                           int64_t* npairs, int32_t* k, tp_error* err) {
    clear_err(err);
    const int64_t* src_n;
    const int32_t* src_l;
    int64_t cnt;
    if (which == 0) {
        src_n = tpb_models::kSizeN;
        src_l = tpb_models::kSizeLabel;
        cnt = tpb_models::kSizeCount;
    } else if (which == 1) {
        src_n = tpb_models::kDepthN;
        src_l = tpb_models::kDepthLabel;
        cnt = tpb_models::kDepthCount;
    } else if (which == 2) {
        src_n = tpb_models::kSize32N;
        src_l = tpb_models::kSize32Label;
        cnt = tpb_models::kSize32Count;
    } else {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "which must be 0 (fp64 size), 1 (depth) or 2 (fp32 size)");
        return TP_ERR_INVALID_ARGUMENT;
    }
    if (npairs) *npairs = cnt;
    if (k) *k = 1;
    if (pairs_n && pairs_label) {
        if (cap < cnt) {
            set_err(err, TP_ERR_INVALID_ARGUMENT, "capacity too small");
            return TP_ERR_INVALID_ARGUMENT;
        }
        for (int64_t i = 0; i < cnt; ++i) {
            pairs_n[i] = src_n[i];
            pairs_label[i] = src_l[i];
        }
    }
    return TP_OK;
}

// read_observations — io.hpp:80-138 (header :21-22, field parsing :44-66).
tp_status tp_obs_read(const char* path, tp_obs_set** out, int64_t* count, tp_error* err) {
    clear_err(err);
    if (!path || !out) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "null argument");
        return TP_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    std::ifstream in(path);
    if (!in) {
        set_err(err, TP_ERR_IO, std::string("cannot open ") + path);
        return TP_ERR_IO;
    }
    static const char* kHeader = "N,precision,device,streams,m,time_ms,is_opt,corrected_m,opt_R";
    std::string line;
    if (!std::getline(in, line)) {
        set_err(err, TP_ERR_MALFORMED_HEADER, std::string("empty file: ") + path);
        return TP_ERR_MALFORMED_HEADER;
    }
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line != kHeader) {
        set_err(err, TP_ERR_MALFORMED_HEADER, std::string("unexpected header in ") + path);
        return TP_ERR_MALFORMED_HEADER;
    }
    auto fields_of = [](const std::string& l) {
        std::vector<std::string> f(1);
        for (char ch : l) {
            if (ch == ',') f.emplace_back();
            else if (ch != '\r') f.back().push_back(ch);
        }
        return f;
    };
    auto bad = [&](size_t ln, const std::string& what) {
        set_err(err, TP_ERR_BAD_NUMBER, "line " + std::to_string(ln) + ": bad number: " + what);
        if (err) err->row = (int64_t)ln;
        return TP_ERR_BAD_NUMBER;
    };
    auto parse_i64 = [](const std::string& s, int64_t& v) {
        if (s.empty()) return false;
        size_t i = 0;
        bool neg = false;
        if (s[0] == '-') { neg = true; i = 1; }
        if (i >= s.size()) return false;
        int64_t acc = 0;
        for (; i < s.size(); ++i) {
            if (s[i] < '0' || s[i] > '9') return false;
            acc = acc * 10 + (s[i] - '0');
        }
        v = neg ? -acc : acc;
        return true;
    };
    auto parse_f64 = [](const std::string& s, double& v) {
        if (s.find_first_not_of("0123456789.eE+-") != std::string::npos || s.empty()) return false;
        char* end = nullptr;
        v = std::strtod(s.c_str(), &end);
        return end == s.c_str() + s.size();
    };

    using Key = std::tuple<int64_t, std::string, std::string>;
    std::map<Key, tp_obs_set::Row> grouped;
    std::map<Key, std::map<int32_t, double>> times;
    size_t ln = 1;
    while (std::getline(in, line)) {
        ++ln;
        if (line.empty() || line == "\r") continue;
        const auto f = fields_of(line);
        if (f.size() != 9) {
            set_err(err, TP_ERR_BAD_NUMBER,
                    "line " + std::to_string(ln) + ": bad number: expected 9 fields, got " +
                        std::to_string(f.size()));
            if (err) err->row = (int64_t)ln;
            return TP_ERR_BAD_NUMBER;
        }
        int64_t n;
        if (!parse_i64(f[0], n)) return bad(ln, "'" + f[0] + "'");
        const Key key{n, f[1], f[2]};
        auto& row = grouped[key];
        row.o.n = n;
        std::snprintf(row.o.precision, sizeof(row.o.precision), "%s", f[1].c_str());
        std::snprintf(row.o.device, sizeof(row.o.device), "%s", f[2].c_str());
        int64_t streams;
        if (!parse_i64(f[3], streams)) return bad(ln, "'" + f[3] + "'");
        row.o.streams = (int32_t)streams;
        std::optional<int64_t> m;
        if (!f[4].empty()) {
            int64_t mv;
            if (!parse_i64(f[4], mv)) return bad(ln, "'" + f[4] + "'");
            m = mv;
        }
        if (!f[5].empty() && m) {
            double t;
            if (!parse_f64(f[5], t)) return bad(ln, "'" + f[5] + "'");
            times[key][(int32_t)*m] = t;
        }
        int64_t is_opt;
        if (!parse_i64(f[6], is_opt)) return bad(ln, "'" + f[6] + "'");
        if (is_opt != 0) {
            if (!f[8].empty() && !m) {
                int64_t r;
                if (!parse_i64(f[8], r)) return bad(ln, "'" + f[8] + "'");
                row.o.label = (int32_t)r;
                row.o.depth_label = 1;
            } else if (m) {
                row.o.label = (int32_t)*m;
            } else {
                set_err(err, TP_ERR_BAD_NUMBER,
                        "line " + std::to_string(ln) + ": bad number: optimum row carries neither m nor opt_R");
                if (err) err->row = (int64_t)ln;
                return TP_ERR_BAD_NUMBER;
            }
            if (!f[7].empty()) {
                int64_t cv;
                if (!parse_i64(f[7], cv)) return bad(ln, "'" + f[7] + "'");
                row.o.corrected = (int32_t)cv;
                row.o.has_corrected = 1;
            }
        }
    }
    auto* set = new tp_obs_set();
    for (auto& [key, row] : grouped) {
        auto& tm = times[key];
        row.o.ntimes = (int32_t)tm.size();
        for (auto& [c, t] : tm) {
            row.cand.push_back(c);
            row.times.push_back(t);
        }
        set->rows.push_back(row);
    }
    *out = set;
    if (count) *count = (int64_t)set->rows.size();
    return TP_OK;
}

tp_status tp_obs_get(const tp_obs_set* set, int64_t i, tp_observation* out, int32_t* cand,
                     double* times_ms, tp_error* err) {
    clear_err(err);
    if (!set || !out || i < 0 || i >= (int64_t)set->rows.size()) {
        set_err(err, TP_ERR_INVALID_ARGUMENT, "bad observation index");
        return TP_ERR_INVALID_ARGUMENT;
    }
    const auto& r = set->rows[(size_t)i];
    *out = r.o;
    if (cand)
        for (size_t j = 0; j < r.cand.size(); ++j) cand[j] = r.cand[j];
    if (times_ms)
        for (size_t j = 0; j < r.times.size(); ++j) times_ms[j] = r.times[j];
    return TP_OK;
}

void tp_obs_free(tp_obs_set* set) { delete set; }

}  // extern "C"
