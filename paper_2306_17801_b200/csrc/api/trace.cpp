// trace.cpp -- rivulet::trace (trace.hpp:11-46 of the reference) over the
// library's event store (csrc/rvk_trace.cpp).
#include "rivulet/trace.hpp"

#include "rvk_trace.hpp"

namespace rivulet::trace {

namespace {
TraceEvent from_rvk(const rvk::trace::Event& e)
{
    TraceEvent t;
    t.task_id      = e.task_id;
    t.enqueue_seq  = e.enqueue_seq;
    t.context_id   = e.ctx_id;
    t.context_name = e.ctx_name;
    t.label        = e.label;
    t.kind         = static_cast<EventKind>(e.kind);
    t.blocked      = e.blocked;
    t.device_timed = e.device;
    t.t_start_ns   = e.t_start_ns;
    t.t_end_ns     = e.t_end_ns;
    return t;
}
} // namespace

const char* to_string(EventKind kind) { return rvk::trace::kind_name(static_cast<int>(kind)); }

void set_enabled(bool on) { rvk::trace::set_enabled(on); }
bool enabled() { return rvk::trace::enabled(); }
void clear() { rvk::trace::clear(); }

std::int64_t now_ns() { return rvk::trace::now_ns(); }

void record(TraceEvent ev)
{
    rvk::trace::Event e;
    e.task_id     = ev.task_id;
    e.enqueue_seq = ev.enqueue_seq;
    e.ctx_id      = ev.context_id;
    e.ctx_name    = std::move(ev.context_name);
    e.label       = std::move(ev.label);
    e.kind        = static_cast<int>(ev.kind);
    e.blocked     = ev.blocked;
    e.device      = ev.device_timed;
    e.t_start_ns  = ev.t_start_ns;
    e.t_end_ns    = ev.t_end_ns;
    rvk::trace::record(std::move(e));
}

void marker(const std::string& label) { rvk::trace::marker(label); }

void host_sync(const std::string& api, ObjectId context_id, bool blocked, std::int64_t t_start_ns,
               std::int64_t t_end_ns)
{
    TraceEvent ev;
    ev.context_id = context_id;
    ev.label      = api;
    ev.kind       = EventKind::HostSync;
    ev.blocked    = blocked;
    ev.t_start_ns = t_start_ns;
    ev.t_end_ns   = t_end_ns;
    record(std::move(ev));
}

std::vector<TraceEvent> snapshot()
{
    std::vector<TraceEvent> out;
    for (const auto& e : rvk::trace::snapshot()) out.push_back(from_rvk(e));
    return out;
}

void write_jsonl(const std::string& path)
{
    if (!rvk::trace::write_jsonl(path)) throw Error("trace: cannot open '" + path + "' for writing");
}

void write_chrome(const std::string& path)
{
    if (!rvk::trace::write_chrome(path)) throw Error("trace: cannot open '" + path + "' for writing");
}

} // namespace rivulet::trace
