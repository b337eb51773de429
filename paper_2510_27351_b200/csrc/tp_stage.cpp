// Pinned two-buffer staging of pageable host transfers (see tp_stage.h).
#include "tp_stage.h"

#include <algorithm>
#include <cstring>

namespace tpb {

HostPool::HostPool(int nthreads) {
    for (int i = 1; i < nthreads; ++i) workers_.emplace_back([this, i] { loop(i); });
}

HostPool::~HostPool() {
    {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
}

void HostPool::loop(int id) {
    long seen = 0;
    for (;;) {
        const std::function<void(int)>* job;
        int parts;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || generation_ != seen; });
            if (stop_) return;
            seen = generation_;
            job = job_;
            parts = parts_;
        }
        for (int p = id; p < parts; p += size()) (*job)(p);
        {
            std::lock_guard<std::mutex> g(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
}

HostPool& HostPool::shared() {
    static HostPool pool((int)std::max(1u, std::min(std::thread::hardware_concurrency(), 16u)));
    return pool;
}

void HostPool::run(int parts, const std::function<void(int)>& fn) {
    if (workers_.empty() || parts <= 1) {
        for (int p = 0; p < parts; ++p) fn(p);
        return;
    }
    std::lock_guard<std::mutex> turn(run_mu_);
    {
        std::lock_guard<std::mutex> g(mu_);
        job_ = &fn;
        parts_ = parts;
        pending_ = (int)workers_.size();
        ++generation_;
    }
    cv_.notify_all();
    for (int p = 0; p < parts; p += size()) fn(p);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
}

bool is_pinned_host(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // unregistered pointers can set a sticky-free error on old drivers
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

Stager::~Stager() {
    for (int i = 0; i < 2; ++i) {
        if (buf_[i]) cudaFreeHost(buf_[i]);
        if (ev_[i]) cudaEventDestroy(ev_[i]);
    }
}

cudaError_t Stager::ensure() {
    if (buf_[0]) return cudaSuccess;
    for (int i = 0; i < 2; ++i) {
        cudaError_t e = cudaMallocHost(&buf_[i], kChunk);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

void Stager::parallel_copy(void* dst, const void* src, size_t bytes) {
    HostPool& pool = HostPool::shared();
    const int parts = pool.size() * 2;
    const size_t per = ((bytes + parts - 1) / parts + 4095) & ~size_t(4095);
    pool.run(parts, [&](int p) {
        const size_t lo = std::min(bytes, (size_t)p * per), hi = std::min(bytes, lo + per);
        if (hi > lo) std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
    });
}

cudaError_t Stager::h2d(void* dst_dev, const void* src_host, size_t bytes, cudaStream_t st) {
    cudaError_t e = ensure();
    if (e != cudaSuccess) return e;
    char* d = static_cast<char*>(dst_dev);
    const char* s = static_cast<const char*>(src_host);
    for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
        const int b = (int)(i & 1);
        const size_t len = std::min(kChunk, bytes - off);
        e = cudaEventSynchronize(ev_[b]);  // the DMA that last read this buffer is done
        if (e != cudaSuccess) return e;
        parallel_copy(buf_[b], s + off, len);
        e = cudaMemcpyAsync(d + off, buf_[b], len, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev_[b], st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t Stager::d2h(void* dst_host, const void* src_dev, size_t bytes, cudaStream_t st) {
    cudaError_t e = ensure();
    if (e != cudaSuccess) return e;
    char* d = static_cast<char*>(dst_host);
    const char* s = static_cast<const char*>(src_dev);
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t i) {
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        cudaError_t r = cudaMemcpyAsync(buf_[i & 1], s + off, len, cudaMemcpyDeviceToHost, st);
        return r == cudaSuccess ? cudaEventRecord(ev_[i & 1], st) : r;
    };
    if (nch > 0 && (e = issue(0)) != cudaSuccess) return e;
    for (size_t i = 0; i < nch; ++i) {
        // chunk i+1 lands in the other buffer while the threads drain chunk i
        if (i + 1 < nch && (e = issue(i + 1)) != cudaSuccess) return e;
        if ((e = cudaEventSynchronize(ev_[i & 1])) != cudaSuccess) return e;
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        parallel_copy(d + off, buf_[i & 1], len);
    }
    return cudaSuccess;
}

}  // namespace tpb
