#pragma once
// rivulet (B200 build) -- device contexts.
// Drop-in for /root/reference/proj/include/rivulet/context.hpp:75-123.  The
// reference runs a context's FIFO on a host agent thread; here a context IS a
// CUDA stream (plus reduction scratch), so FIFO order, wait_for and
// query_idle are the hardware's, and nothing ever blocks the host except the
// explicit synchronize()/drain_all() and the globally-blocking forms.

#include "rivulet/common.hpp"

#include <memory>
#include <string>

struct rvk_ctx_s;
struct CUstream_st;

namespace rivulet {

enum class StreamType { DefaultBlocking, GloballyBlocking };
const char* to_string(StreamType type);

namespace detail {
struct ContextImpl;
}

class Context {
public:
    explicit Context(StreamType type = StreamType::DefaultBlocking, std::string name = "");

    ObjectId           id() const;
    StreamType         stream_type() const;
    const std::string& name() const;

    // Future work here starts after everything enqueued on `waitee` so far
    // (cudaStreamWaitEvent).  Does not block.  Self-wait is a no-op.
    void wait_for(const Context& waitee) const;
    bool query_idle() const;  // never blocks
    void synchronize() const; // blocks (counted host sync)

    CUstream_st* cuda_stream() const;
    rvk_ctx_s*   handle() const;

    const std::shared_ptr<detail::ContextImpl>& impl() const { return impl_; }

private:
    std::shared_ptr<detail::ContextImpl> impl_;
};

// Block until every live context is idle.
void drain_all();

namespace detail {
// Shared globally-blocking context behind the synchronous API forms.
const Context& global_sync_context();
} // namespace detail

} // namespace rivulet
