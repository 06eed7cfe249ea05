// core.cpp -- contexts, dependency tracking, launches, storage, counters.
#include "internal.hpp"
#include "rvk_context.hpp"

#include <memory>
#include <mutex>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>

namespace rivulet {

ObjectId next_object_id()
{
    static std::atomic<ObjectId> counter{kUnknownId};
    return ++counter;
}

namespace detail {

void throw_status(rvk_status st, const char* what)
{
    std::string msg = std::string(what) + ": " + rvk_last_error();
    if (st == RVK_ERR_BREAKDOWN) throw BreakdownError(msg, -1);
    throw Error(msg);
}

void check_cuda(cudaError_t e, const char* what)
{
    if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- event pool ------------------------------------------------------------------
namespace {
std::mutex               g_ev_mu;
std::vector<cudaEvent_t> g_ev_free;
} // namespace

Ev::~Ev()
{
    if (!e) return;
    std::lock_guard lk(g_ev_mu);
    g_ev_free.push_back(e);
}

EvPtr make_event()
{
    auto ev = std::make_shared<Ev>();
    {
        std::lock_guard lk(g_ev_mu);
        if (!g_ev_free.empty()) {
            ev->e = g_ev_free.back();
            g_ev_free.pop_back();
        }
    }
    if (!ev->e) check_cuda(cudaEventCreateWithFlags(&ev->e, cudaEventDisableTiming), "cudaEventCreate");
    return ev;
}

// ---- context registry --------------------------------------------------------------
namespace {
std::mutex                              g_ctx_mu;
std::vector<std::weak_ptr<ContextImpl>> g_contexts;
} // namespace

ContextImpl::~ContextImpl()
{
    if (h) rvk_ctx_destroy(h); // drains first
}

// One per device (the calling thread's current device): a process may drive
// several GPUs, e.g. one host thread per device.
const Context& global_sync_context()
{
    static std::mutex                              m;
    static std::unique_ptr<Context>                per_dev[64];
    int                                            dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(m);
    auto&                       c = per_dev[dev & 63];
    if (!c) c = std::make_unique<Context>(StreamType::GloballyBlocking, "global_sync");
    return *c;
}

// ---- tracker -------------------------------------------------------------------
Tracker& Tracker::get()
{
    static Tracker t;
    return t;
}

void Tracker::begin(const Context& ctx, ObjectId id, Mode mode)
{
    std::lock_guard lk(mu_);
    auto it = recs_.find(id);
    if (it == recs_.end()) return;
    DepRecord& r = it->second;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(ctx.cuda_stream());
    auto wait = [&](const Access& a) {
        if (a.ctx == ctx.id() || !a.ev) return; // FIFO on the same stream covers it
        check_cuda(cudaStreamWaitEvent(s, a.ev->e, 0), "cudaStreamWaitEvent");
        rvk::trace::wait_edge(ctx.id(), a.ctx, "wait_for ctx");
        ++edges_;
    };
    if (r.last_write) wait(*r.last_write);
    if (mode != Mode::Read)
        for (const auto& a : r.readers) wait(a);
}

void Tracker::end(const Context& ctx, ObjectId id, Mode mode, const EvPtr& ev)
{
    std::lock_guard lk(mu_);
    DepRecord& r = recs_[id];
    if (mode == Mode::Read) {
        for (auto& a : r.readers)
            if (a.ctx == ctx.id()) {
                a.ev = ev;
                return;
            }
        r.readers.push_back(Access{ev, ctx.id()});
    } else {
        r.last_write = Access{ev, ctx.id()};
        r.readers.clear();
    }
}

bool Tracker::await_host(ObjectId id, Mode mode)
{
    std::vector<EvPtr> evs;
    {
        std::lock_guard lk(mu_);
        auto it = recs_.find(id);
        if (it == recs_.end()) return false;
        if (it->second.last_write) evs.push_back(it->second.last_write->ev);
        if (mode != Mode::Read)
            for (auto& a : it->second.readers) evs.push_back(a.ev);
    }
    std::vector<EvPtr> busy;
    for (auto& e : evs) {
        if (!e) continue;
        if (cudaEventQuery(e->e) == cudaErrorNotReady) busy.push_back(e);
        else (void)cudaGetLastError();
    }
    if (busy.empty()) return false;
    rvk::trace::HostSyncScope hs("await_host", 0, true); // counted + traced
    for (auto& e : busy) check_cuda(cudaEventSynchronize(e->e), "cudaEventSynchronize");
    return true;
}

void Tracker::release_on(ObjectId id, cudaStream_t stream)
{
    std::lock_guard lk(mu_);
    auto it = recs_.find(id);
    if (it == recs_.end()) return;
    if (it->second.last_write && it->second.last_write->ev)
        cudaStreamWaitEvent(stream, it->second.last_write->ev->e, 0);
    for (auto& a : it->second.readers)
        if (a.ev) cudaStreamWaitEvent(stream, a.ev->e, 0);
    recs_.erase(it);
}

void Tracker::reset()
{
    std::lock_guard lk(mu_);
    edges_ = 0;
}

// ---- launches ----------------------------------------------------------------------
Launch::Launch(const Context& ctx, std::string label) : ctx_(ctx), label_(std::move(label)) {}

Launch& Launch::access(ObjectId id, Mode mode)
{
    for (auto& [eid, m] : acc_)
        if (eid == id) {
            if (m != mode) m = Mode::ReadWrite; // merged intent (launch.cpp:15-27)
            return *this;
        }
    acc_.emplace_back(id, mode);
    return *this;
}

void Launch::begin()
{
    if (ctx_.stream_type() == StreamType::GloballyBlocking) drain_all();
    auto& t = Tracker::get();
    for (auto& [id, m] : acc_) t.begin(ctx_, id, m);
    task_ = std::make_unique<rvk::trace::TaskScope>(
        reinterpret_cast<cudaStream_t>(ctx_.cuda_stream()), label_.c_str(), ctx_.id(), ctx_.name().c_str());
}

EvPtr Launch::end()
{
    task_.reset(); // the task ends after its kernel(s)
    auto         ev = make_event();
    cudaStream_t s  = reinterpret_cast<cudaStream_t>(ctx_.cuda_stream());
    check_cuda(cudaEventRecord(ev->e, s), "cudaEventRecord");
    auto& t = Tracker::get();
    for (auto it = acc_.rbegin(); it != acc_.rend(); ++it) t.end(ctx_, it->first, it->second, ev);
    if (ctx_.stream_type() == StreamType::GloballyBlocking) ctx_.synchronize();
    return ev;
}

// ---- storage ----------------------------------------------------------------------
namespace {
// The allocation stream of a device (created on first use, with that device
// current).  Storage lives on the device that was current when it was
// allocated; its release goes to the same device's stream.
cudaStream_t mem_stream(int dev)
{
    static std::mutex   m;
    static cudaStream_t per_dev[64] = {};
    std::lock_guard<std::mutex> lk(m);
    cudaStream_t& s = per_dev[dev & 63];
    if (!s) {
        int prev = 0;
        check_cuda(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
        const cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        if (prev != dev) cudaSetDevice(prev);
        check_cuda(e, "cudaStreamCreate");
    }
    return s;
}
int current_device()
{
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    return dev;
}
} // namespace

void* device_alloc(std::size_t bytes)
{
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    const cudaStream_t s = mem_stream(current_device());
    check_cuda(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
    // allocation is setup, not data: make it usable from any stream now
    check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize(alloc)");
    return p;
}

void device_release(void* p, ObjectId id)
{
    // Deferred release (managed_state.hpp:13-15): the free is
    // stream-ordered after every outstanding access, the host never waits.
    // The owning device's stream (the handle may die on another thread).
    int                   dev = current_device();
    cudaPointerAttributes a{};
    if (p && cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeDevice)
        dev = a.device;
    else
        cudaGetLastError();
    const cudaStream_t s    = mem_stream(dev);
    const int          prev = current_device();
    if (prev != dev) cudaSetDevice(dev); // events and the free on the owning device
    Tracker::get().release_on(id, s);
    if (p) cudaFreeAsync(p, s);
    if (prev != dev) cudaSetDevice(prev);
}

void check_no_write_view(const VecState& v, const char* api)
{
    if (v.write_views > 0)
        throw Error(std::string(api) + ": vector '" + v.name +
                    "' has an open host write view (restore() it first)");
}

ManagedState::ManagedState(std::size_t n_, std::string name_)
    : id(next_object_id()), name(std::move(name_)), n(n_), host(n_, 0.0)
{
    dev = static_cast<double*>(device_alloc(n * sizeof(double)));
}

ManagedState::~ManagedState() { device_release(dev, id); }

VecState::VecState(std::size_t n_, std::string name_)
    : id(next_object_id()), name(std::move(name_)), n(n_)
{
    dev = static_cast<double*>(device_alloc(n * sizeof(double)));
}

VecState::~VecState() { device_release(dev, id); }

MatState::MatState(std::string name_) : id(next_object_id()), name(std::move(name_)) {}

MatState::~MatState()
{
    plans.reset();
    // the three arrays live on one device: release them there (device_release
    // finds it from the pointer); the tracker entry of the matrix goes with
    // the first non-null array
    bool released = false;
    for (void* p : {static_cast<void*>(off), static_cast<void*>(cols), static_cast<void*>(vals)})
        if (p) {
            device_release(p, released ? kUnknownId : id);
            released = true;
        }
    if (!released) Tracker::get().release_on(id, mem_stream(current_device()));
}

} // namespace detail

// ---- Context ---------------------------------------------------------------------------
const char* to_string(StreamType t)
{
    return t == StreamType::DefaultBlocking ? "default_blocking" : "globally_blocking";
}

Context::Context(StreamType type, std::string name) : impl_(std::make_shared<detail::ContextImpl>())
{
    impl_->id   = next_object_id();
    impl_->type = type;
    impl_->name = std::move(name);
    detail::check(rvk_ctx_create(nullptr, &impl_->h), "Context");
    impl_->h->id = impl_->id; // one id in the trace for the C++ and C views
    detail::check(rvk_ctx_set_name(impl_->h, impl_->name.c_str()), "Context");
    std::lock_guard lk(detail::g_ctx_mu);
    detail::g_contexts.push_back(impl_);
}

ObjectId           Context::id() const { return impl_->id; }
StreamType         Context::stream_type() const { return impl_->type; }
const std::string& Context::name() const { return impl_->name; }
rvk_ctx_s*         Context::handle() const { return impl_->h; }
CUstream_st*       Context::cuda_stream() const
{
    return static_cast<CUstream_st*>(rvk_ctx_stream(impl_->h));
}

void Context::wait_for(const Context& waitee) const
{
    if (waitee.id() == id()) return;
    detail::check(rvk_ctx_wait_for(impl_->h, waitee.impl_->h), "Context::wait_for");
}

bool Context::query_idle() const
{
    int idle = 0;
    detail::check(rvk_ctx_query_idle(impl_->h, &idle), "Context::query_idle");
    return idle != 0;
}

void Context::synchronize() const { detail::check(rvk_ctx_synchronize(impl_->h), "Context::synchronize"); }

void drain_all()
{
    std::vector<std::shared_ptr<detail::ContextImpl>> live;
    {
        std::lock_guard lk(detail::g_ctx_mu);
        auto& v = detail::g_contexts;
        v.erase(std::remove_if(v.begin(), v.end(), [](auto& w) { return w.expired(); }), v.end());
        for (auto& w : v)
            if (auto s = w.lock()) live.push_back(std::move(s));
    }
    for (auto& c : live) {
        int idle = 0;
        if (rvk_ctx_query_idle(c->h, &idle) == RVK_OK && idle) continue;
        detail::check(rvk_ctx_synchronize(c->h), "drain_all");
    }
}

// ---- runtime counters ------------------------------------------------------------------
namespace runtime {
namespace {
std::mutex g_mu;
Census     g_census;
CopyCounts g_copies;
} // namespace

const char* to_string(KernelKind k)
{
    static const char* names[] = {"matmult", "dot",  "norm", "axpy",    "aypx",
                                  "waxpy",   "scale", "copy", "expr_eval", "pc_apply"};
    const int i = static_cast<int>(k);
    return i >= 0 && i < static_cast<int>(KernelKind::kCount) ? names[i] : "?";
}

std::uint64_t Census::total_flops() const
{
    std::uint64_t t = 0;
    for (auto f : flops) t += f;
    return t;
}
std::uint64_t Census::reductions() const { return kernels_of(KernelKind::Dot) + kernels_of(KernelKind::Norm); }
Census        Census::operator-(const Census& r) const
{
    Census d;
    for (int i = 0; i < static_cast<int>(KernelKind::kCount); ++i) {
        d.kernels[i] = kernels[i] - r.kernels[i];
        d.flops[i]   = flops[i] - r.flops[i];
    }
    return d;
}

Census census()
{
    std::lock_guard lk(g_mu);
    return g_census;
}

void log_kernel(KernelKind k, std::uint64_t flops, std::uint64_t count)
{
    std::lock_guard lk(g_mu);
    g_census.kernels[static_cast<int>(k)] += count;
    g_census.flops[static_cast<int>(k)] += flops;
}

CopyCounts copy_counts()
{
    std::lock_guard lk(g_mu);
    return g_copies;
}
void log_h2d(std::uint64_t bytes)
{
    std::lock_guard lk(g_mu);
    ++g_copies.h2d;
    g_copies.h2d_bytes += bytes;
}
void log_d2h(std::uint64_t bytes)
{
    std::lock_guard lk(g_mu);
    ++g_copies.d2h;
    g_copies.d2h_bytes += bytes;
}

std::uint64_t host_syncs() { return rvk_host_sync_count(); }

std::string to_json()
{
    const Census     c = census();
    const CopyCounts k = copy_counts();
    std::string      j = "{\"census\":{";
    for (int i = 0; i < static_cast<int>(KernelKind::kCount); ++i) {
        j += (i ? ",\"" : "\"") + std::string(to_string(static_cast<KernelKind>(i))) +
             "\":{\"kernels\":" + std::to_string(c.kernels[i]) +
             ",\"flops\":" + std::to_string(c.flops[i]) + "}";
    }
    j += "},\"total_flops\":" + std::to_string(c.total_flops());
    j += ",\"reductions\":" + std::to_string(c.reductions());
    j += ",\"copies\":{\"h2d\":" + std::to_string(k.h2d) + ",\"d2h\":" + std::to_string(k.d2h) +
         ",\"h2d_bytes\":" + std::to_string(k.h2d_bytes) +
         ",\"d2h_bytes\":" + std::to_string(k.d2h_bytes) + "}";
    j += ",\"host_syncs\":" + std::to_string(host_syncs());
    j += ",\"dependency_edges\":" + std::to_string(detail::Tracker::get().edges()) + "}";
    return j;
}

void write_json(const std::string& path)
{
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw Error("runtime: cannot open '" + path + "' for writing");
    const std::string j = to_json() + "\n";
    const bool        ok = std::fwrite(j.data(), 1, j.size(), f) == j.size();
    if (std::fclose(f) != 0 || !ok) throw Error("runtime: cannot write '" + path + "'");
}

void reset_all()
{
    {
        std::lock_guard lk(g_mu);
        g_census = Census{};
        g_copies = CopyCounts{};
    }
    rvk_host_sync_reset();
    detail::Tracker::get().reset();
}

} // namespace runtime
} // namespace rivulet
