// Host staging for PAGEABLE host buffers (the reference's std::vector callers).
//
// cudaMemcpy from/to pageable memory goes through the driver's small bounce
// buffers at ~10-13 GB/s, plus first-touch page faults on a fresh output vector
// (measured: 480 ms per N=1e8 host solve from pageable numpy arrays against
// 73 ms from pinned ones). Here the copy is a two-buffer pipeline through
// pinned chunks owned by the context: host threads (a small pool) copy chunk
// i+1 between the user's pages and pinned memory while the DMA engine moves
// chunk i over PCIe. Pinned user buffers skip all of this (direct DMA).
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace tpb {

// Fixed pool of worker threads running one parallel_for at a time.
class HostPool {
public:
    explicit HostPool(int nthreads);
    ~HostPool();
    HostPool(const HostPool&) = delete;
    HostPool& operator=(const HostPool&) = delete;
    int size() const { return (int)workers_.size() + 1; }
    // fn(part) for part in [0, parts), the caller runs part 0; calls from
    // several host threads take turns (one job at a time)
    void run(int parts, const std::function<void(int)>& fn);
    // the process-wide pool every context's Stager shares
    static HostPool& shared();

private:
    void loop(int id);
    std::vector<std::thread> workers_;
    std::mutex run_mu_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* job_ = nullptr;
    int parts_ = 0;
    long generation_ = 0;
    int pending_ = 0;
    bool stop_ = false;
};

class Stager {
public:
    Stager() = default;
    ~Stager();
    Stager(const Stager&) = delete;
    Stager& operator=(const Stager&) = delete;
    // host (pageable) -> device, enqueued on `st`; returns when every chunk
    // has been handed to the DMA engine (the last one may still be in flight)
    cudaError_t h2d(void* dst_dev, const void* src_host, size_t bytes, cudaStream_t st);
    // device -> host (pageable), synchronous with respect to `st`
    cudaError_t d2h(void* dst_host, const void* src_dev, size_t bytes, cudaStream_t st);

private:
    cudaError_t ensure();
    void parallel_copy(void* dst, const void* src, size_t bytes);
    static constexpr size_t kChunk = size_t(64) << 20;
    void* buf_[2] = {nullptr, nullptr};
    cudaEvent_t ev_[2] = {nullptr, nullptr};
};

// true when `p` is page-locked (cudaMallocHost / cudaHostRegister) memory
bool is_pinned_host(const void* p);

}  // namespace tpb
