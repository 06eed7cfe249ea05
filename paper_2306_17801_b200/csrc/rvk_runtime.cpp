// rvk_runtime.cpp -- contexts, errors, memory and host-sync accounting.
//
// rvk_ctx is the B200 replacement of rivulet::Context (context.hpp:75-114):
// the reference runs each context's FIFO on a host agent thread
// (context.cpp:151-232); here a context IS a CUDA stream, so FIFO order,
// wait_for (cudaStreamWaitEvent) and query_idle (cudaStreamQuery) are the
// hardware's.  Every host-blocking call is counted like the reference's
// trace::host_sync events (trace.hpp:40-41).
#include <cstdlib>
#include "rvk_common.cuh"
#include "rvk_context.hpp"

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

namespace rvk {

namespace {
thread_local char     g_err[512] = "";
std::atomic<uint64_t> g_host_syncs{0};
constexpr int         kMaxDevices = 64;
std::atomic<int>      g_sm_count[kMaxDevices]; // 0 = not queried yet
} // namespace

rvk_status set_error(rvk_status s, const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

rvk_status cuda_error(cudaError_t e, const char* what)
{
    return set_error(e == cudaErrorMemoryAllocation ? RVK_ERR_ALLOC : RVK_ERR_CUDA, "%s: %s (%s)",
                     what, cudaGetErrorString(e), cudaGetErrorName(e));
}

void note_host_sync() { g_host_syncs.fetch_add(1, std::memory_order_relaxed); }

int current_device()
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    return dev;
}

int sm_count()
{
    const int dev = current_device() & (kMaxDevices - 1);
    int       n   = g_sm_count[dev].load(std::memory_order_relaxed);
    if (n > 0) return n;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        n = 148;
    g_sm_count[dev].store(n, std::memory_order_relaxed);
    return n;
}

} // namespace rvk

using namespace rvk;

extern "C" {

const char* rvk_last_error(void) { return g_err; }
#ifndef RVK_BUILD_ID
#define RVK_BUILD_ID "unknown"
#endif
const char* rvk_build_id(void) { return RVK_BUILD_ID; }
int         rvk_abi_version(void) { return RVK_ABI_VERSION; }

int rvk_device_info(int* sms, char* name, int name_len)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return RVK_ERR_CUDA;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return RVK_ERR_CUDA;
    if (sms) *sms = prop.multiProcessorCount;
    if (name && name_len > 0) {
        std::strncpy(name, prop.name, (size_t)name_len - 1);
        name[name_len - 1] = 0;
    }
    return RVK_OK;
}

int rvk_device_count(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

rvk_status rvk_set_device(int device)
{
    RVK_CUDA(cudaSetDevice(device));
    return RVK_OK;
}

uint64_t rvk_host_sync_count(void) { return g_host_syncs.load(); }
void     rvk_host_sync_reset(void) { g_host_syncs.store(0); }

rvk_status rvk_ctx_create(void* cuda_stream, rvk_ctx* out)
{
    if (!out) return set_error(RVK_ERR_INVALID, "ctx_create: null out");
    *out   = nullptr;
    static std::atomic<uint64_t> next_id{0};
    auto c = new rvk_ctx_s();
    c->id  = ++next_id;
    if (cuda_stream) {
        c->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete c;
            return cuda_error(e, "cudaStreamCreateWithFlags");
        }
        c->owns_stream = true;
    }
    const size_t pbytes = sizeof(double) * (size_t)kMaxReduceBlocks * 4;
    cudaError_t  e      = cudaMalloc(&c->scratch.partials, pbytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->scratch.tickets, 16 * sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemset(c->scratch.tickets, 0, 16 * sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->wait_event, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaDeviceSynchronize(); // memset complete before first use
    if (e != cudaSuccess) {
        rvk_ctx_destroy(c);
        return cuda_error(e, "rvk_ctx_create");
    }
    *out = c;
    return RVK_OK;
}

rvk_status rvk_ctx_destroy(rvk_ctx c)
{
    if (!c) return RVK_OK;
    // a destroyed context first drains its queue.
    if (c->stream) cudaStreamSynchronize(c->stream);
    cudaFree(c->scratch.partials);
    cudaFree(c->scratch.tickets);
    if (c->wait_event) cudaEventDestroy(c->wait_event);
    if (c->owns_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return RVK_OK;
}

void* rvk_ctx_stream(rvk_ctx c) { return c ? static_cast<void*>(c->stream) : nullptr; }
uint64_t rvk_ctx_id(rvk_ctx c) { return c ? c->id : 0; }

rvk_status rvk_ctx_set_name(rvk_ctx c, const char* name)
{
    if (!c) return set_error(RVK_ERR_INVALID, "null context");
    std::snprintf(c->name, sizeof c->name, "%s", name ? name : "");
    return RVK_OK;
}

rvk_status rvk_ctx_synchronize(rvk_ctx c)
{
    if (!c) return set_error(RVK_ERR_INVALID, "null context");
    {
        trace::HostSyncScope hs_("rvk_ctx_synchronize", c->id);
        RVK_CUDA(cudaStreamSynchronize(c->stream));
    }
    return RVK_OK;
}

rvk_status rvk_ctx_query_idle(rvk_ctx c, int* idle)
{
    if (!c || !idle) return set_error(RVK_ERR_INVALID, "null argument");
    cudaError_t e = cudaStreamQuery(c->stream);
    if (e == cudaSuccess) *idle = 1;
    else if (e == cudaErrorNotReady) {
        (void)cudaGetLastError();
        *idle = 0;
    } else return cuda_error(e, "cudaStreamQuery");
    return RVK_OK;
}

rvk_status rvk_ctx_wait_for(rvk_ctx waiter, rvk_ctx waitee)
{
    if (!waiter || !waitee) return set_error(RVK_ERR_INVALID, "null context");
    if (waiter == waitee || waiter->stream == waitee->stream) return RVK_OK; // no-op
    RVK_CUDA(cudaEventRecord(waitee->wait_event, waitee->stream));
    RVK_CUDA(cudaStreamWaitEvent(waiter->stream, waitee->wait_event, 0));
    trace::wait_edge(waiter->id, waitee->id, "wait_for ctx");
    return RVK_OK;
}

rvk_status rvk_malloc(void** dev, size_t bytes)
{
    if (!dev) return set_error(RVK_ERR_INVALID, "null out");
    *dev = nullptr;
    if (bytes == 0) return RVK_OK;
    RVK_CUDA(cudaMalloc(dev, bytes));
    return RVK_OK;
}

rvk_status rvk_free(void* dev)
{
    if (dev) RVK_CUDA(cudaFree(dev));
    return RVK_OK;
}

// Stream-ordered allocation: the allocation is usable by work enqueued on ctx
// after this call; the release happens once the work enqueued before
// rvk_free_async has run -- the reference's "resource lifetime extends past
// handle destruction until the stream is idle" (managed_state.hpp:13-15)
// without a host wait.
rvk_status rvk_malloc_async(rvk_ctx ctx, void** dev, size_t bytes)
{
    if (!ctx || !dev) return set_error(RVK_ERR_INVALID, "null argument");
    *dev = nullptr;
    if (bytes == 0) return RVK_OK;
    RVK_CUDA(cudaMallocAsync(dev, bytes, ctx->stream));
    return RVK_OK;
}

rvk_status rvk_free_async(rvk_ctx ctx, void* dev)
{
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    if (dev) RVK_CUDA(cudaFreeAsync(dev, ctx->stream));
    return RVK_OK;
}

rvk_status rvk_host_alloc(void** host, size_t bytes)
{
    if (!host) return set_error(RVK_ERR_INVALID, "null out");
    *host = nullptr;
    if (bytes == 0) return RVK_OK;
    RVK_CUDA(cudaMallocHost(host, bytes));
    return RVK_OK;
}

rvk_status rvk_host_free(void* host)
{
    if (host) RVK_CUDA(cudaFreeHost(host));
    return RVK_OK;
}

rvk_status rvk_memcpy_h2d(rvk_ctx c, void* dst, const void* src, size_t bytes)
{
    if (!c) return set_error(RVK_ERR_INVALID, "null context");
    if (bytes) RVK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    return RVK_OK;
}

rvk_status rvk_memcpy_d2h(rvk_ctx c, void* dst, const void* src, size_t bytes)
{
    if (!c) return set_error(RVK_ERR_INVALID, "null context");
    if (bytes) RVK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    return RVK_OK;
}

rvk_status rvk_memcpy_d2d(rvk_ctx c, void* dst, const void* src, size_t bytes)
{
    if (!c) return set_error(RVK_ERR_INVALID, "null context");
    if (bytes) RVK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
    return RVK_OK;
}

rvk_status rvk_scalar_read(rvk_ctx c, const double* s_dev, double* out_host)
{
    if (!c || !s_dev || !out_host) return set_error(RVK_ERR_INVALID, "null argument");
    RVK_CUDA(cudaMemcpyAsync(out_host, s_dev, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    {
        trace::HostSyncScope hs_("rvk_scalar_read");
        RVK_CUDA(cudaStreamSynchronize(c->stream));
    }
    return RVK_OK;
}

} // extern "C"
