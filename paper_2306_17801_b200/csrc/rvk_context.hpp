// rvk_context.hpp -- internal definition of rvk_ctx (stream + reduction scratch).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "rvk.h"

namespace rvk {

// Upper bound on blocks of any reduction launched through a context.
constexpr int kMaxReduceBlocks = 148 * 16;
constexpr int kReduceThreads   = 256;

struct Scratch {
    double*       partials;  // kMaxReduceBlocks * 4 doubles
    unsigned int* tickets;   // 16 grid tickets, kept at 0 between launches
};

} // namespace rvk

struct rvk_ctx_s {
    cudaStream_t  stream      = nullptr;
    bool          owns_stream = false;
    rvk::Scratch  scratch{};
    cudaEvent_t   wait_event  = nullptr; // reused by rvk_ctx_wait_for
    uint64_t      id          = 0;       // process-unique (trace rows)
    char          name[48]    = "";      // rvk_ctx_set_name (trace rows)
};

namespace rvk {
// Number of reduction blocks for n elements (fixed for a given n and GPU, so
// reductions are deterministic).
int reduce_grid(int64_t n);
} // namespace rvk
