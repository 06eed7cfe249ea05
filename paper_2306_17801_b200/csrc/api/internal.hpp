// internal.hpp -- shared internals of the rivulet C++ API (B200 build).
//
// The reference implements ordering with host agent threads, epochs and a
// dependency tracker (deptrack.cpp:184-290, launch.cpp:29-37).  Here the
// same RAW/WAR/WAW rules (no edge between two reads) are
// applied to CUDA streams: every launch records one pooled cudaEvent on its
// context's stream; a later launch from another context that conflicts with
// an object's last writer (or, for writes, its readers) gets a
// cudaStreamWaitEvent edge.  Nothing blocks the host except the explicit
// host accessors, each counted as a host sync.
#pragma once

#include "rivulet/common.hpp"
#include "rivulet/context.hpp"
#include "rivulet/csr.hpp"
#include "rivulet/managed.hpp"
#include "rivulet/runtime.hpp"
#include "rivulet/vector.hpp"
#include "rvk.h"
#include "rvk_trace.hpp"

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <unordered_map>
#include <vector>

namespace rvk {
void note_host_sync(); // rvk_runtime.cpp: the library-wide host-sync counter
}

namespace rivulet::detail {

[[noreturn]] void throw_status(rvk_status st, const char* what);
inline void       check(rvk_status st, const char* what)
{
    if (st != RVK_OK) throw_status(st, what);
}
void check_cuda(cudaError_t e, const char* what);

// ---- pooled CUDA events ------------------------------------------------------
struct Ev {
    cudaEvent_t e = nullptr;
    ~Ev();
};
using EvPtr = std::shared_ptr<Ev>;
EvPtr make_event();

// ---- contexts ------------------------------------------------------------------
struct ContextImpl {
    rvk_ctx     h = nullptr;
    ObjectId    id = 0;
    StreamType  type = StreamType::DefaultBlocking;
    std::string name;
    ~ContextImpl();
};

// ---- dependency tracking ---------------------------------------------------------
enum class Mode { Read, Write, ReadWrite };

struct Access {
    EvPtr    ev;
    ObjectId ctx = 0;
};

struct DepRecord {
    std::optional<Access> last_write;
    std::vector<Access>   readers; // since last_write, at most one per context
};

class Tracker {
public:
    static Tracker& get();
    // Install the cross-context waits `mode` on `id` requires (deptrack.cpp:184-225).
    void begin(const Context& ctx, ObjectId id, Mode mode);
    // Publish the launch's completion event (deptrack.cpp:227-269).
    void end(const Context& ctx, ObjectId id, Mode mode, const EvPtr& ev);
    // Host access: wait for conflicting device work (deptrack.cpp:271-290).
    // Returns true if it had to block (counted as one host sync).
    bool await_host(ObjectId id, Mode mode);
    // Make `stream` wait for every outstanding access of `id`, then forget it.
    void release_on(ObjectId id, cudaStream_t stream);
    std::uint64_t edges() const { return edges_; }
    void          reset();

private:
    std::mutex                              mu_;
    std::unordered_map<ObjectId, DepRecord> recs_;
    std::uint64_t                           edges_ = 0;
};

// One kernel launch bracketed with its operand marks (launch.hpp:17-43).  For a
// globally-blocking context begin() first drains every context and end()
// synchronises, so the call completes before returning (context.hpp:15-19).
class Launch {
public:
    Launch(const Context& ctx, std::string label);
    Launch& read(ObjectId id) { return access(id, Mode::Read); }
    Launch& write(ObjectId id) { return access(id, Mode::Write); }
    Launch& read_write(ObjectId id) { return access(id, Mode::ReadWrite); }
    Launch& access(ObjectId id, Mode mode);
    void    begin();
    EvPtr   end();
    const Context& ctx() const { return ctx_; }

private:
    Context                                 ctx_;
    std::string                             label_;
    std::vector<std::pair<ObjectId, Mode>>  acc_;
    std::unique_ptr<rvk::trace::TaskScope>  task_; // begin() .. end(): NVTX range + trace Task
};

// ---- storage ---------------------------------------------------------------------
void* device_alloc(std::size_t bytes);                      // stream-ordered pool, ready on return
void  device_release(void* p, ObjectId id);                 // after id's outstanding accesses

struct ManagedState {
    ObjectId            id;
    std::string         name;
    std::size_t         n;
    double*             dev = nullptr;
    EvPtr               pending;          // last write still in flight
    ObjectId            pending_ctx = 0;
    std::vector<double> host;             // cached host value (valid if host_valid)
    bool                host_valid = false;
    ManagedState(std::size_t n, std::string name);
    ~ManagedState();
    void mark_written(const EvPtr& ev, ObjectId ctx)
    {
        pending     = ev;
        pending_ctx = ctx;
        host_valid  = false;
    }
};

struct VecState {
    ObjectId            id;
    std::string         name;
    std::size_t         n;
    double*             dev = nullptr;
    std::vector<double> host;
    bool                host_valid  = false;
    int                 read_views  = 0;
    int                 write_views = 0;
    std::mutex          view_mutex;
    VecState(std::size_t n, std::string name);
    ~VecState();
};

struct CgPlanCache; // solvers.cpp

struct MatState {
    ObjectId                  id;
    std::string               name;
    std::size_t               n_rows = 0, n_cols = 0, nnz = 0;
    std::int64_t*             off  = nullptr;
    std::int32_t*             cols = nullptr;
    double*                   vals = nullptr;
    std::int64_t              max_row_len = 0;
    // lazily materialised host copies
    std::mutex                host_mutex;
    bool                      host_loaded = false;
    std::vector<std::int64_t> h_off;
    std::vector<std::int32_t> h_cols;
    std::vector<double>       h_vals;
    std::shared_ptr<CgPlanCache> plans;
    MatState(std::string name);
    ~MatState();
    rvk_csr view() const
    {
        return rvk_csr{(int64_t)n_rows, (int64_t)n_cols, (int64_t)nnz, off, cols, vals};
    }
};

// Device work on a vector with an open host write view is a usage error here.
void check_no_write_view(const VecState& v, const char* api);
// A device kernel wrote the vector: the host mirror is stale.
inline void device_wrote(VecState& v) { v.host_valid = false; }

// Internal scalar-expression runner (rvk_expr.cu).
struct ExprStep {
    std::uint8_t  kind; // 0 leaf, 1 const, 2 unary, 3 binary
    std::uint8_t  op;
    std::int16_t  a, b;
    std::uint32_t len;
    double        value;
    const double* leaf;
};
constexpr int kMaxExprSteps = 96;
struct ExprProgramDev {
    int      n_steps;
    ExprStep steps[kMaxExprSteps];
};
rvk_status expr_run(cudaStream_t s, const ExprProgramDev& prog, double* out, std::size_t len);

// Records which iteration first produced a non-finite ratio / zero divisor.
rvk_status breakdown_check(cudaStream_t s, const double* num, const double* den, int iteration,
                           int* flag);

} // namespace rivulet::detail
