// rvk_trace.cpp -- event store, device-timed tasks, JSONL / Chrome export.
// See rvk_trace.hpp; the reference's store is trace.cpp:11-104 (a vector of
// events under a mutex, gated by an atomic flag).
#include "rvk_trace.hpp"

#include "rvk.h"

#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <map>
#include <mutex>

namespace rvk {
void       note_host_sync(); // rvk_runtime.cpp
rvk_status set_error(rvk_status s, const char* fmt, ...);
}

namespace rvk::trace {

namespace {

struct DeviceTask {
    Event       ev;
    bool        closed = false; // end event recorded
    int         device = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
};

struct DeviceBase {
    cudaEvent_t  ev = nullptr;
    std::int64_t host_ns = 0;
};

std::atomic<bool>          g_on{false};
std::atomic<std::uint64_t> g_seq{0};
std::mutex                 g_mu;
std::vector<Event>         g_events;  // host-timed (and resolved device) events
std::map<std::uint64_t, DeviceTask> g_pending; // by enqueue_seq: device-timed tasks not yet resolved
std::map<int, DeviceBase>  g_base;    // per device: GPU time origin on the host clock
// Open TaskScopes on this thread: only the outermost records an event (a
// C++-API launch that calls an ABI entry point, a solve's internal vector
// ops); the NVTX ranges nest.
thread_local int           t_depth = 0;

// Caller holds g_mu.  A timing event recorded on an idle private stream and
// waited for: its GPU timestamp is "now" on the host clock (to within the
// wait's wake-up latency).
bool ensure_base(int dev)
{
    if (g_base.count(dev)) return true;
    DeviceBase   b;
    cudaStream_t s = nullptr;
    if (cudaEventCreate(&b.ev) != cudaSuccess) return false;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
        cudaEventDestroy(b.ev);
        return false;
    }
    cudaEventRecord(b.ev, s);
    cudaEventSynchronize(b.ev);
    b.host_ns = now_ns();
    cudaStreamDestroy(s);
    g_base[dev] = b;
    return true;
}

// Caller holds g_mu.
void resolve_pending()
{
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto it = g_pending.begin(); it != g_pending.end();) {
        DeviceTask& t = it->second;
        if (!t.closed) { // its scope is still open on another thread
            ++it;
            continue;
        }
        cudaSetDevice(t.device);
        const DeviceBase& b = g_base[t.device];
        float             m0 = 0.f, m1 = 0.f;
        if (cudaEventSynchronize(t.e1) == cudaSuccess &&
            cudaEventElapsedTime(&m0, b.ev, t.e0) == cudaSuccess &&
            cudaEventElapsedTime(&m1, b.ev, t.e1) == cudaSuccess) {
            t.ev.t_start_ns = b.host_ns + (std::int64_t)((double)m0 * 1e6);
            t.ev.t_end_ns   = b.host_ns + (std::int64_t)((double)m1 * 1e6);
            t.ev.device     = true;
        } else {
            (void)cudaGetLastError(); // keep the host enqueue times
        }
        cudaEventDestroy(t.e0);
        cudaEventDestroy(t.e1);
        g_events.push_back(std::move(t.ev));
        it = g_pending.erase(it);
    }
    cudaSetDevice(cur);
}

void json_str(std::FILE* f, const std::string& s)
{
    std::fputc('"', f);
    for (unsigned char c : s) {
        if (c == '"' || c == '\\') std::fprintf(f, "\\%c", c);
        else if (c < 0x20) std::fprintf(f, "\\u%04x", c);
        else std::fputc(c, f);
    }
    std::fputc('"', f);
}

} // namespace

const char* kind_name(int kind)
{
    switch (kind) {
    case Task: return "task";
    case Wait: return "wait";
    case HostSync: return "host_sync";
    case Marker: return "marker";
    }
    return "?";
}

bool enabled() { return g_on.load(std::memory_order_relaxed); }

void set_enabled(bool on)
{
    if (on) {
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard lk(g_mu);
        ensure_base(dev);
    }
    g_on.store(on, std::memory_order_relaxed);
}

void clear()
{
    std::lock_guard lk(g_mu);
    for (auto it = g_pending.begin(); it != g_pending.end();) {
        if (!it->second.closed) { // still open: its scope finishes it
            ++it;
            continue;
        }
        cudaEventDestroy(it->second.e0);
        cudaEventDestroy(it->second.e1);
        it = g_pending.erase(it);
    }
    g_events.clear();
}

std::int64_t now_ns()
{
    return std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

void record(Event ev)
{
    if (!enabled()) return;
    std::lock_guard lk(g_mu);
    g_events.push_back(std::move(ev));
}

void marker(const std::string& label)
{
    nvtxMarkA(label.c_str());
    if (!enabled()) return;
    Event ev;
    ev.label      = label;
    ev.kind       = Marker;
    ev.t_start_ns = ev.t_end_ns = now_ns();
    record(std::move(ev));
}

std::vector<Event> snapshot()
{
    std::lock_guard lk(g_mu);
    resolve_pending();
    return g_events;
}

bool write_jsonl(const std::string& path)
{
    const auto ev = snapshot();
    std::FILE* f  = std::fopen(path.c_str(), "w");
    if (!f) return false;
    for (const auto& e : ev) {
        std::fprintf(f, "{\"task\":%llu,\"enqueue_seq\":%llu,\"ctx\":%llu,\"ctx_name\":",
                     (unsigned long long)e.task_id, (unsigned long long)e.enqueue_seq,
                     (unsigned long long)e.ctx_id);
        json_str(f, e.ctx_name);
        std::fputs(",\"label\":", f);
        json_str(f, e.label);
        std::fprintf(f, ",\"kind\":\"%s\",\"blocked\":%s,\"device_timed\":%s,\"start\":%lld,\"end\":%lld}\n",
                     kind_name(e.kind), e.blocked ? "true" : "false", e.device ? "true" : "false",
                     (long long)e.t_start_ns, (long long)e.t_end_ns);
    }
    return std::fclose(f) == 0;
}

bool write_chrome(const std::string& path)
{
    const auto ev = snapshot();
    std::FILE* f  = std::fopen(path.c_str(), "w");
    if (!f) return false;
    std::int64_t t0 = 0;
    for (const auto& e : ev)
        if (t0 == 0 || e.t_start_ns < t0) t0 = e.t_start_ns;
    std::map<std::uint64_t, std::string> rows; // tid -> name
    std::fputs("{\"displayTimeUnit\":\"ns\",\"traceEvents\":[\n", f);
    bool first = true;
    for (const auto& e : ev) {
        const bool          host = e.kind == HostSync || e.kind == Marker;
        const std::uint64_t tid  = host ? 0 : e.ctx_id + 1;
        // a context's row is named from any of its events that carries the name
        if (!rows.count(tid) || (!host && !e.ctx_name.empty() && rows[tid].find('(') == std::string::npos))
            rows[tid] = host ? std::string("host")
                             : "ctx " + std::to_string(e.ctx_id) +
                                   (e.ctx_name.empty() ? "" : " (" + e.ctx_name + ")");
        std::fputs(first ? "" : ",\n", f);
        first = false;
        std::fputs("{\"name\":", f);
        json_str(f, e.label);
        const double ts = (double)(e.t_start_ns - t0) * 1e-3;
        const double du = (double)(e.t_end_ns - e.t_start_ns) * 1e-3;
        if (e.kind == Marker || e.kind == Wait)
            std::fprintf(f, ",\"cat\":\"%s\",\"ph\":\"i\",\"s\":\"t\",\"ts\":%.3f,\"pid\":0,\"tid\":%llu}",
                         kind_name(e.kind), ts, (unsigned long long)tid);
        else
            std::fprintf(f,
                         ",\"cat\":\"%s\",\"ph\":\"X\",\"ts\":%.3f,\"dur\":%.3f,\"pid\":0,\"tid\":%llu,"
                         "\"args\":{\"task\":%llu,\"seq\":%llu,\"blocked\":%s,\"device_timed\":%s}}",
                         kind_name(e.kind), ts, du, (unsigned long long)tid,
                         (unsigned long long)e.task_id, (unsigned long long)e.enqueue_seq,
                         e.blocked ? "true" : "false", e.device ? "true" : "false");
    }
    for (const auto& [tid, name] : rows) {
        std::fprintf(f, "%s{\"name\":\"thread_name\",\"ph\":\"M\",\"pid\":0,\"tid\":%llu,\"args\":{\"name\":",
                     first ? "" : ",\n", (unsigned long long)tid);
        first = false;
        json_str(f, name);
        std::fputs("}}", f);
    }
    std::fputs("\n]}\n", f);
    return std::fclose(f) == 0;
}

TaskScope::TaskScope(cudaStream_t s, const char* label, std::uint64_t ctx_id, const char* ctx_name)
    : s_(s)
{
    nvtxRangePushA(label);
    if (t_depth++ > 0 || !enabled()) return;
    on_              = true;
    ev_.kind         = Task;
    ev_.label        = label;
    ev_.ctx_id       = ctx_id;
    ev_.ctx_name     = ctx_name ? ctx_name : "";
    ev_.enqueue_seq  = ++g_seq;
    ev_.task_id      = ev_.enqueue_seq;
    ev_.t_start_ns   = now_ns();
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s_, &cs) != cudaSuccess) {
        (void)cudaGetLastError();
        return;
    }
    if (cs != cudaStreamCaptureStatusNone) return; // graph capture: host times only
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard lk(g_mu);
    if (!ensure_base(dev)) return;
    DeviceTask t;
    t.device = dev;
    if (cudaEventCreate(&t.e0) != cudaSuccess || cudaEventCreate(&t.e1) != cudaSuccess ||
        cudaEventRecord(t.e0, s_) != cudaSuccess) {
        (void)cudaGetLastError();
        if (t.e0) cudaEventDestroy(t.e0);
        if (t.e1) cudaEventDestroy(t.e1);
        return;
    }
    slot_            = (std::int64_t)ev_.enqueue_seq;
    g_pending[ev_.enqueue_seq] = t;
}

TaskScope::~TaskScope()
{
    nvtxRangePop();
    --t_depth;
    if (!on_) return;
    ev_.t_end_ns = now_ns();
    std::lock_guard lk(g_mu);
    auto it = slot_ >= 0 ? g_pending.find((std::uint64_t)slot_) : g_pending.end();
    if (it != g_pending.end()) {
        DeviceTask& t = it->second;
        if (cudaEventRecord(t.e1, s_) == cudaSuccess) {
            t.ev     = std::move(ev_);
            t.closed = true;
            return;
        }
        (void)cudaGetLastError();
        cudaEventDestroy(t.e0);
        cudaEventDestroy(t.e1);
        g_pending.erase(it);
    }
    g_events.push_back(std::move(ev_));
}

HostSyncScope::HostSyncScope(const char* api, std::uint64_t ctx_id, bool blocked)
    : api_(api), ctx_(ctx_id), blocked_(blocked), t0_(0)
{
    rvk::note_host_sync();
    nvtxRangePushA(api);
    if (enabled()) t0_ = now_ns();
}

HostSyncScope::~HostSyncScope()
{
    nvtxRangePop();
    if (!enabled() || t0_ == 0) return;
    Event ev;
    ev.kind       = HostSync;
    ev.label      = api_;
    ev.ctx_id     = ctx_;
    ev.blocked    = blocked_;
    ev.t_start_ns = t0_;
    ev.t_end_ns   = now_ns();
    record(std::move(ev));
}

void wait_edge(std::uint64_t waiter_ctx, std::uint64_t waitee, const char* what)
{
    if (!enabled()) return;
    Event ev;
    ev.kind       = Wait;
    ev.ctx_id     = waiter_ctx;
    ev.label      = std::string(what) + " " + std::to_string(waitee);
    ev.t_start_ns = ev.t_end_ns = now_ns();
    record(std::move(ev));
}

} // namespace rvk::trace

extern "C" {

void rvk_trace_enable(int on) { rvk::trace::set_enabled(on != 0); }
int  rvk_trace_enabled(void) { return rvk::trace::enabled() ? 1 : 0; }
void rvk_trace_clear(void) { rvk::trace::clear(); }
void rvk_trace_marker(const char* label) { rvk::trace::marker(label ? label : ""); }

size_t rvk_trace_count(void) { return rvk::trace::snapshot().size(); }

rvk_status rvk_trace_write_jsonl(const char* path)
{
    if (!path) return rvk::set_error(RVK_ERR_INVALID, "trace_write_jsonl: null path");
    if (!rvk::trace::write_jsonl(path))
        return rvk::set_error(RVK_ERR_INVALID, "trace: cannot write '%s'", path);
    return RVK_OK;
}

rvk_status rvk_trace_write_chrome(const char* path)
{
    if (!path) return rvk::set_error(RVK_ERR_INVALID, "trace_write_chrome: null path");
    if (!rvk::trace::write_chrome(path))
        return rvk::set_error(RVK_ERR_INVALID, "trace: cannot write '%s'", path);
    return RVK_OK;
}

} // extern "C"
