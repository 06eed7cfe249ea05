// rvk_common.cuh -- shared device helpers for the sm_100a Jacobi-CG kernels.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>

#include "rvk.h"
#include "rvk_trace.hpp"

namespace rvk {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// IEEE mul-then-add with no contraction.  The reference's kernels are
// compiled without -march (no FMA; kernels_avx2.cpp:9-13), so every product is
// rounded before it is summed.  __dmul_rn/__dadd_rn are never fused by nvcc.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
// y + a*x   (axpy:  kernels_scalar.cpp:27  y[i] += a * x[i])
__device__ __forceinline__ double axpy1(double a, double x, double y) { return add(y, mul(a, x)); }
// x + b*y   (aypx:  kernels_scalar.cpp:33  y[i] = x[i] + b * y[i])
__device__ __forceinline__ double aypx1(double b, double x, double y) { return add(x, mul(b, y)); }

// ---------------------------------------------------------------------------
// ScalarArg evaluated inside the consuming kernel (linalg.hpp:17-38).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double eval_scalar(const rvk_scalar& s)
{
    switch (s.kind) {
    case RVK_SCALAR_CONST: return s.c;
    case RVK_SCALAR_PTR: return *s.p0;
    case RVK_SCALAR_NEG_PTR: return -(*s.p0);
    case RVK_SCALAR_DIV_PTR_PTR: return (*s.p0) / (*s.p1);
    case RVK_SCALAR_SQRT_PTR: return sqrt(*s.p0);
    case RVK_SCALAR_RECIP_PTR: return 1.0 / (*s.p0);
    }
    return 0.0;
}

// ---------------------------------------------------------------------------
// Deterministic reductions: warp shuffle tree, then a fixed-order tree over
// the warps of the block.  Each block writes its partial; the last block to
// finish (atomic ticket) folds the partials in index order and runs the
// scalar "tail".  No floating-point atomics anywhere, so for a fixed grid the
// result is bit-reproducible (SPEC.md:604 fingerprint requirement).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Sum `v` over the first `nthreads` threads (multiple of 32, <= 1024) of the
// block.  `smem` needs nthreads/32 doubles per value.  Result valid in the
// thread with (threadIdx.x - first) == 0.  `bar` is a named barrier id so
// warp-specialised kernels can reduce over the consumer warps only.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem, int tid, int nthreads,
                                          int bar)
{
    const int lane = tid & 31, warp = tid >> 5, nw = nthreads >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) smem[j * 32 + warp] = v[j];
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nthreads) : "memory");
    if (warp == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            double t = lane < nw ? smem[j * 32 + lane] : 0.0;
            v[j]     = warp_sum(t);
        }
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nthreads) : "memory");
}

// Grid-level ticket: returns true in exactly one block (the last to arrive)
// after every block has published its partials.  Call from ALL threads of
// the participating thread group; `flag` is a shared int.  SYS: the block's
// earlier stores include stores to PEER GPUs' memory -- fence at system
// scope so the last block's release covers them.
template <bool SYS = false>
__device__ __forceinline__ bool last_block(unsigned int* ticket, int tid, int* flag, int nthreads,
                                           int bar)
{
    if (tid == 0) {
        if constexpr (SYS) __threadfence_system();
        else __threadfence();
        const unsigned int t = atomicAdd(ticket, 1u);
        *flag                = (t == gridDim.x - 1);
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nthreads) : "memory");
    const bool last = *flag != 0;
    if (last) __threadfence();
    return last;
}

// Fold `count` partials (stride NV, index-ordered) into v[] inside the last
// block: thread t sums partials t, t+n, t+2n, ... sequentially, then a block
// tree.  Deterministic.
template <int NV>
__device__ __forceinline__ void fold_partials(const double* partials, int count, double (&v)[NV],
                                              double* smem, int tid, int nthreads, int bar)
{
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = 0.0;
    for (int i = tid; i < count; i += nthreads) {
#pragma unroll
        for (int j = 0; j < NV; ++j) v[j] += __ldcg(partials + (size_t)i * NV + j);
    }
    block_sum<NV>(v, smem, tid, nthreads, bar);
}

// ---------------------------------------------------------------------------
// mbarrier / bulk-copy (TMA) helpers (sm_90+ PTX, used on sm_100a).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// L2 eviction policy for streamed-once operands (CSR values/indices): keeps
// the reused x-gather window resident in L2 instead.
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ... default priority (an explicit policy for bulk copies that must not be
// demoted, e.g. operands other CTAs gather again soon).
__device__ __forceinline__ uint64_t policy_evict_normal()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ... and for data several CTAs will re-read soon (the x-windows).
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 1-D bulk copy global -> shared, completion signalled on `bar` (tx bytes).
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// Bulk L2 prefetch (no destination): src 16-B aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Streaming global loads (read-once data).
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }

} // namespace rvk

// Host-side error plumbing shared by the .cu/.cpp translation units.
namespace rvk {
rvk_status set_error(rvk_status s, const char* fmt, ...);
rvk_status cuda_error(cudaError_t e, const char* what);
void       note_host_sync();
// SM count of the CURRENT device (cached per device: one process may drive
// several GPUs, e.g. one host thread per device)
int        sm_count();
// Per-device one-time setup (function attributes are per device): true when
// bit `device` of `mask` is not set yet; device_mark_done sets it.
int        current_device();
inline bool device_first_use(std::atomic<uint64_t>& mask)
{
    return !(mask.load(std::memory_order_acquire) & (1ull << (current_device() & 63)));
}
inline void device_mark_done(std::atomic<uint64_t>& mask)
{
    mask.fetch_or(1ull << (current_device() & 63), std::memory_order_acq_rel);
}
// kern<<<grid, block, smem, s>>>(args...) with the arguments converted to
// the kernel's parameter types; returns the launch error (not cleared).
template <class... KArgs, class... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args)
{
    kern<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
    return cudaPeekAtLastError();
}
} // namespace rvk

// Device task of an ABI entry point: NVTX range + trace Task event (rvk_trace.hpp).
#define RVK_TRACE_TASK(ctx, label) ::rvk::trace::TaskScope rvk_task_((ctx)->stream, (label), (ctx)->id, (ctx)->name)

#define RVK_CUDA(call)                                                   \
    do {                                                                 \
        cudaError_t e_ = (call);                                         \
        if (e_ != cudaSuccess) return ::rvk::cuda_error(e_, #call);      \
    } while (0)

#define RVK_CHECK_LAUNCH(what)                                           \
    do {                                                                 \
        cudaError_t e_ = cudaGetLastError();                             \
        if (e_ != cudaSuccess) return ::rvk::cuda_error(e_, what);       \
    } while (0)
