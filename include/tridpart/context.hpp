// context.hpp — the per-thread device context behind the drop-in headers.
// A tp_ctx (C-ABI, tridpart_b200.h) is not thread-safe; the reference is
// reentrant (partition.hpp keeps no shared state), so every host thread gets
// its own context on device 0, created on first use.
#pragma once

#include "errors.hpp"

namespace tridpart::b200 {

class Context {
public:
    explicit Context(int device = 0) {
        tp_error e{};
        throw_on(tp_ctx_create(device, &ctx_, &e), e);
    }
    ~Context() { tp_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    tp_ctx* get() const noexcept { return ctx_; }

private:
    tp_ctx* ctx_ = nullptr;
};

inline Context& thread_context() {
    thread_local Context ctx(0);
    return ctx;
}

}  // namespace tridpart::b200
