// rvk_trace.hpp -- Task / Wait / HostSync / Marker events and NVTX ranges.
//
// The reference records a TraceEvent per task its agent thread executes
// (context.cpp:216-227), per host wait (managed.cpp:74-84,
// deptrack.cpp:286-288) and per user marker, with steady-clock ns
// timestamps, gated by trace::enabled() and exported as JSONL
// (trace.hpp:11-46, trace.cpp:48-104).  Here a task is device work: while
// tracing is on, each traced enqueue brackets its stream with two timing
// events whose GPU times are mapped onto the host steady clock when the trace
// is read (snapshot() waits for the recorded work -- a debugging read, not
// counted as a library host sync).  Inside a stream capture no events are
// recorded (a replayed graph would re-use them); the task is logged with its
// host enqueue time instead.  Every traced scope is also an NVTX range
// (nvtx3, header-only), so ncu --nvtx / Nsight timelines show the solve,
// its phases and the host waits by name whether or not tracing is on.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace rvk::trace {

enum Kind : int { Task = 0, Wait = 1, HostSync = 2, Marker = 3 };
const char* kind_name(int kind);

struct Event {
    std::uint64_t task_id     = 0; // global id of the task (0 for host events)
    std::uint64_t enqueue_seq = 0; // global enqueue order (0 for host events)
    std::uint64_t ctx_id      = 0;
    std::string   ctx_name;
    std::string   label;
    int           kind    = Task;
    bool          blocked = false; // HostSync: whether the wait actually blocked
    bool          device  = false; // Task: times are the GPU's (else host enqueue)
    std::int64_t  t_start_ns = 0;
    std::int64_t  t_end_ns   = 0;
};

bool         enabled();
void         set_enabled(bool on);
void         clear();
std::int64_t now_ns();
void         record(Event ev);
void         marker(const std::string& label);
// Resolves the device timings of every recorded task (waits for them).
std::vector<Event> snapshot();
bool               write_jsonl(const std::string& path);
// Chrome trace-event JSON (chrome://tracing, Perfetto): one row per context,
// one for host syncs.
bool write_chrome(const std::string& path);

// RAII: NVTX range + (tracing on, stream not capturing) a device-timed task.
class TaskScope {
public:
    TaskScope(cudaStream_t s, const char* label, std::uint64_t ctx_id = 0,
              const char* ctx_name = nullptr);
    ~TaskScope();
    TaskScope(const TaskScope&)            = delete;
    TaskScope& operator=(const TaskScope&) = delete;

private:
    cudaStream_t  s_;
    std::int64_t  slot_ = -1; // key of the pending device task (its enqueue_seq)
    Event         ev_;
    bool          on_ = false;
};

// RAII around a blocking host wait: counts it (rvk_host_sync_count) and,
// when tracing, records a HostSync event with its duration.
class HostSyncScope {
public:
    explicit HostSyncScope(const char* api, std::uint64_t ctx_id = 0, bool blocked = true);
    ~HostSyncScope();
    void set_blocked(bool b) { blocked_ = b; }
    HostSyncScope(const HostSyncScope&)            = delete;
    HostSyncScope& operator=(const HostSyncScope&) = delete;

private:
    const char*   api_;
    std::uint64_t ctx_;
    bool          blocked_;
    std::int64_t  t0_;
};

// A cross-stream ordering edge (cudaStreamWaitEvent): a zero-duration Wait
// event on the waiting context.
void wait_edge(std::uint64_t waiter_ctx, std::uint64_t waitee, const char* what);

} // namespace rvk::trace
