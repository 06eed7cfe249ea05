#pragma once
// rivulet (B200 build) -- census, copy and host-sync counters.
// Mirrors /root/reference/proj/include/rivulet/runtime.hpp:49-121 (delay
// injection is out of scope: it simulates the launch latency a real GPU has).

#include "rivulet/common.hpp"

#include <array>
#include <cstdint>
#include <string>

namespace rivulet::runtime {

struct CopyCounts {
    std::uint64_t h2d = 0, d2h = 0, h2d_bytes = 0, d2h_bytes = 0;
};
CopyCounts copy_counts();
void       log_h2d(std::uint64_t bytes);
void       log_d2h(std::uint64_t bytes);

enum class KernelKind : int { MatMult = 0, Dot, Norm, Axpy, Aypx, Waxpy, Scale, Copy, ExprEval, PcApply, kCount };
const char* to_string(KernelKind kind);

struct Census {
    std::array<std::uint64_t, static_cast<int>(KernelKind::kCount)> kernels{};
    std::array<std::uint64_t, static_cast<int>(KernelKind::kCount)> flops{};
    std::uint64_t kernels_of(KernelKind k) const { return kernels[static_cast<int>(k)]; }
    std::uint64_t flops_of(KernelKind k) const { return flops[static_cast<int>(k)]; }
    std::uint64_t total_flops() const;
    std::uint64_t reductions() const; // Dot + Norm kernels
    Census operator-(const Census& rhs) const;
};
Census census();
// Counted at issue time on the calling thread (exact per-iteration tallies
// while the kernels are still in flight).  kernel_count 0 attributes flops
// fused into another kernel.
void log_kernel(KernelKind kind, std::uint64_t flops, std::uint64_t kernel_count = 1);

// Host synchronisations performed by the library (trace::host_sync analogue).
std::uint64_t host_syncs();

// The counters above as one JSON object: {"census": {kind: {kernels, flops}},
// "total_flops", "reductions", "copies": {h2d, d2h, h2d_bytes, d2h_bytes},
// "host_syncs", "dependency_edges"} (the metrics export; the event timeline
// is rivulet::trace).
std::string to_json();
void        write_json(const std::string& path);

void reset_all();

} // namespace rivulet::runtime
