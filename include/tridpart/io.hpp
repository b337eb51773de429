// io.hpp — drop-in for the reader half of /root/reference/proj/include/tridpart/io.hpp:
//   kObservationsHeader / kModelFormatVersion   io.hpp:21-24
//   read_observations                           io.hpp:80-138 (the library's C++ reader,
//                                               tp_obs_read: rows folded by (N, precision,
//                                               device), label from the is_opt row, same errors)
// Model JSON persistence lives in the Python layer (tridpart.save_model / load_model).
#pragma once

#include <filesystem>
#include <string>
#include <vector>

#include "errors.hpp"
#include "observations.hpp"

namespace tridpart {

inline constexpr const char* kObservationsHeader =
    "N,precision,device,streams,m,time_ms,is_opt,corrected_m,opt_R";
inline constexpr int kModelFormatVersion = 1;

inline ObservationSet read_observations(const std::filesystem::path& path) {
    tp_obs_set* h = nullptr;
    int64_t cnt = 0;
    tp_error e{};
    b200::throw_on(tp_obs_read(path.string().c_str(), &h, &cnt, &e), e);
    ObservationSet out;
    try {
        for (int64_t i = 0; i < cnt; ++i) {
            tp_observation o{};
            b200::throw_on(tp_obs_get(h, i, &o, nullptr, nullptr, &e), e);
            std::vector<int32_t> cand((std::size_t)(o.ntimes > 0 ? o.ntimes : 1));
            std::vector<double> ms(cand.size());
            b200::throw_on(tp_obs_get(h, i, &o, cand.data(), ms.data(), &e), e);
            Observation r;
            r.n = o.n;
            r.label = o.label;
            if (o.has_corrected) r.corrected = o.corrected;
            for (int32_t t = 0; t < o.ntimes; ++t) r.times[cand[(std::size_t)t]] = ms[(std::size_t)t];
            r.precision = o.precision;
            r.device = o.device;
            r.streams = o.streams;
            r.depth_label = o.depth_label != 0;
            out.rows.push_back(std::move(r));
        }
    } catch (...) {
        tp_obs_free(h);
        throw;
    }
    tp_obs_free(h);
    return out;
}

}  // namespace tridpart
