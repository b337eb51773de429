// Peer exchange of the fused multi-GPU solve, shared by the finishing kernels
// (tp_final.cuh) and the grid solve (tp_grid.cu).
#pragma once
#include "tp_device.cuh"

namespace tpb {

// ---------------------------------------------------------------------------
// Peer exchange of the fused multi-GPU solve (k_final<kShard>, one thread).
// Publish this shard's boundary pair into every rank's mailbox, release the
// epoch flag (system scope), wait for all P flags in our own mailbox (acquire,
// bounded), then assemble the 2P-row top system (assemble_interface order,
// partition.hpp:139-149) and solve it with Thomas (tridiagonal.hpp:52-72).
// Returns this shard's (x_s, x_e); false on a peer timeout.
// ---------------------------------------------------------------------------
constexpr long kExchangeSpins = 1L << 24;  // x >= 64 ns back-off: ~1-2 s before giving up

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

template <class T>
__device__ bool shard_exchange(const ShardLink& lk, const Eq2<T>& q, double* cm, double* xx, T& xs, T& xe,
                               RowGuard& top_bad, int& missing) {
    const unsigned long long e = *lk.epoch + 1;
    const int P = lk.nranks;
    const size_t slot = (size_t)(e & 1);
    const double v[8] = {(double)q.a1, (double)q.a2, (double)q.b1, (double)q.b2,
                         (double)q.g1, (double)q.g2, (double)q.d1, (double)q.d2};
    for (int p = 0; p < P; ++p) {
        double* dst = lk.peers[p] + (slot * P + lk.rank) * kMailboxEntryDoubles;
#pragma unroll
        for (int k = 0; k < 8; ++k) dst[k] = v[k];
    }
    __threadfence_system();
    for (int p = 0; p < P; ++p)
        st_release_sys(reinterpret_cast<unsigned long long*>(
                           lk.peers[p] + (slot * P + lk.rank) * kMailboxEntryDoubles + 8), e);
    for (int p = 0; p < P; ++p) {
        const unsigned long long* f = reinterpret_cast<const unsigned long long*>(
            lk.own + (slot * P + p) * kMailboxEntryDoubles + 8);
        long spins = 0;
        while (ld_acquire_sys(f) != e) {
            if (++spins > kExchangeSpins) {
                missing = p;
                *lk.epoch = e;  // stay paired with the peers' next exchange
                return false;
            }
            __nanosleep(64);
        }
    }
    const int n = 2 * P;
    for (int i = 0; i < n; ++i) {
        const double* e8 = lk.own + (slot * P + (i >> 1)) * kMailboxEntryDoubles;
        const int k = i & 1;
        const double sub = ld_relaxed_sys(e8 + 0 + k), dg = ld_relaxed_sys(e8 + 2 + k);
        const double sp = ld_relaxed_sys(e8 + 4 + k), rh = ld_relaxed_sys(e8 + 6 + k);
        if (i == 0) {
            top_bad.see(dg, 0);
            cm[0] = sp / dg;
            xx[0] = rh / dg;
        } else {
            const double piv = dg - sub * cm[i - 1];
            top_bad.see(piv, i);
            cm[i] = sp / piv;
            xx[i] = (rh - sub * xx[i - 1]) / piv;
        }
    }
    for (int i = n - 2; i >= 0; --i) xx[i] -= cm[i] * xx[i + 1];
    xs = (T)xx[2 * lk.rank];
    xe = (T)xx[2 * lk.rank + 1];
    *lk.epoch = e;
    return true;
}

}  // namespace tpb
