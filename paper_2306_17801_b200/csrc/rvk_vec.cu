// rvk_vec.cu -- Vec kernels behind linalg.hpp:48-66 (VecDot/VecNorm/VecAXPY/
// VecAYPX/VecWAXPY/VecScale/VecPointwiseMult/VecCopy/VecSet) on sm_100a.
//
// All are HBM-bound streaming kernels: 128-bit (double2) coalesced loads and
// stores, grid sized as a multiple of the SM count, grid-stride loops.
// Reductions write their result to DEVICE memory through a last-block tail
// (no host round trip: the paper's scalar problem) and are
// deterministic for a fixed n.
#include "rvk_common.cuh"
#include "rvk_context.hpp"
#include "rvk_internal.hpp"

#include <cmath>

namespace rvk {

namespace {

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int elementwise_grid(int64_t n_vec)
{
    const int64_t want = (n_vec + kReduceThreads - 1) / kReduceThreads;
    const int64_t cap  = (int64_t)sm_count() * 16;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

// ---- reductions -------------------------------------------------------------
// OP 0: dot(x,y) -> out0                     (kernels_scalar.cpp:11-17)
// OP 1: nrm2(x)  -> out0 = sqrt(x.x)         (kernels_scalar.cpp:19-22)
// OP 2: dot2     -> out0 = z.z, out1 = z.r   (fused CG pair)
template <int OP>
__global__ void __launch_bounds__(kReduceThreads)
    k_reduce(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
             double* out0, double* out1, Scratch scratch, bool vec, const int* guard)
{
    if (guard && *guard) return; // device-side early exit (CG converged / broke down)
    constexpr int NV = OP == 2 ? 2 : 1;
    __shared__ double smem[NV * 32];
    __shared__ int    flag;
    double acc[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) acc[j] = 0.0;

    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0     = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (vec) {
        const int64_t n2 = n >> 1;
        const double2* x2 = reinterpret_cast<const double2*>(x);
        const double2* y2 = reinterpret_cast<const double2*>(y);
        for (int64_t i = t0; i < n2; i += stride) {
            const double2 a = ld_stream(x2 + i);
            if (OP == 1) {
                acc[0] = add(acc[0], mul(a.x, a.x));
                acc[0] = add(acc[0], mul(a.y, a.y));
            } else {
                const double2 b = ld_stream(y2 + i);
                if (OP == 0) {
                    acc[0] = add(acc[0], mul(a.x, b.x));
                    acc[0] = add(acc[0], mul(a.y, b.y));
                } else {
                    acc[0] = add(acc[0], mul(a.x, a.x));
                    acc[0] = add(acc[0], mul(a.y, a.y));
                    acc[NV - 1] = add(acc[NV - 1], mul(a.x, b.x));
                    acc[NV - 1] = add(acc[NV - 1], mul(a.y, b.y));
                }
            }
        }
        if ((n & 1) && t0 == 0) {
            const double a = x[n - 1];
            if (OP == 1) acc[0] = add(acc[0], mul(a, a));
            else if (OP == 0) acc[0] = add(acc[0], mul(a, y[n - 1]));
            else {
                acc[0]      = add(acc[0], mul(a, a));
                acc[NV - 1] = add(acc[NV - 1], mul(a, y[n - 1]));
            }
        }
    } else {
        for (int64_t i = t0; i < n; i += stride) {
            const double a = x[i];
            if (OP == 1) acc[0] = add(acc[0], mul(a, a));
            else if (OP == 0) acc[0] = add(acc[0], mul(a, y[i]));
            else {
                acc[0]      = add(acc[0], mul(a, a));
                acc[NV - 1] = add(acc[NV - 1], mul(a, y[i]));
            }
        }
    }
    const int tid = threadIdx.x;
    block_sum<NV>(acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) scratch.partials[(size_t)blockIdx.x * NV + j] = acc[j];
    }
    if (!last_block(scratch.tickets, tid, &flag, blockDim.x, 1)) return;
    fold_partials<NV>(scratch.partials, gridDim.x, acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        if (OP == 0) *out0 = acc[0];
        else if (OP == 1) *out0 = sqrt(acc[0]);
        else {
            *out0 = acc[0];
            *out1 = acc[1];
        }
        *scratch.tickets = 0u; // re-arm for the next launch on this stream
    }
}

// ---- elementwise --------------------------------------------------------------

template <int OP>
__device__ __forceinline__ double ew1(double s, double x, double y)
{
    if (OP == EW_AXPY) return axpy1(s, x, y);  // y + s*x          kernels_scalar.cpp:27
    if (OP == EW_AYPX) return aypx1(s, x, y);  // x + s*y          :33
    if (OP == EW_WAXPY) return add(mul(s, x), y); // s*x + y       :39
    if (OP == EW_SCALE) return mul(y, s);      // y *= s           :44
    if (OP == EW_PMULT) return mul(x, y);      // a[i]*b[i]        :50
    return s;                                  // set
}

// out[i] = f(s, x[i], y[i]); x or y may be unused (nullptr) depending on OP.
template <int OP>
__global__ void __launch_bounds__(kReduceThreads)
    k_elementwise(int64_t n, rvk_scalar sa, const double* x,
                  const double* y, double* out, bool vec, const int* guard)
{
    if (guard && *guard) return;
    const double  s      = (OP == EW_PMULT) ? 0.0 : eval_scalar(sa);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0     = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool    needx  = OP == EW_AXPY || OP == EW_AYPX || OP == EW_WAXPY || OP == EW_PMULT;
    const bool    needy  = OP != EW_SET;
    if (vec) {
        const int64_t n2 = n >> 1;
        for (int64_t i = t0; i < n2; i += stride) {
            double2 a = make_double2(0, 0), b = make_double2(0, 0);
            if (needx) a = ld_stream(reinterpret_cast<const double2*>(x) + i);
            if (needy) b = ld_stream(reinterpret_cast<const double2*>(y) + i);
            double2 o;
            o.x = ew1<OP>(s, a.x, b.x);
            o.y = ew1<OP>(s, a.y, b.y);
            st_stream(reinterpret_cast<double2*>(out) + i, o);
        }
        if ((n & 1) && t0 == 0) {
            const double a = needx ? x[n - 1] : 0.0, b = needy ? y[n - 1] : 0.0;
            out[n - 1] = ew1<OP>(s, a, b);
        }
    } else {
        for (int64_t i = t0; i < n; i += stride) {
            const double a = needx ? x[i] : 0.0, b = needy ? y[i] : 0.0;
            out[i] = ew1<OP>(s, a, b);
        }
    }
}

__global__ void k_scalar_eval(rvk_scalar s, double* out) { *out = eval_scalar(s); }

template <int OP>
rvk_status launch_reduce(cudaStream_t stream, Scratch scratch, int64_t n, const double* x,
                         const double* y, double* o0, double* o1, const int* guard)
{
    if (n < 0) return set_error(RVK_ERR_INVALID, "negative length");
    if (!o0 || (OP == 2 && !o1)) return set_error(RVK_ERR_INVALID, "null output scalar");
    if (n > 0 && (!x || (OP != 1 && !y))) return set_error(RVK_ERR_INVALID, "null vector");
    const bool vec = aligned16(x) && (OP == 1 || aligned16(y));
    const int  g   = reduce_grid(vec ? (n + 1) / 2 : n);
    k_reduce<OP><<<g, kReduceThreads, 0, stream>>>(n, x, y, o0, o1, scratch, vec, guard);
    RVK_CHECK_LAUNCH("k_reduce");
    return RVK_OK;
}

template <int OP>
rvk_status launch_ew(cudaStream_t stream, int64_t n, rvk_scalar s, const double* x,
                     const double* y, double* out, const int* guard)
{
    if (n < 0) return set_error(RVK_ERR_INVALID, "negative length");
    if (n == 0) return RVK_OK;
    if (!out) return set_error(RVK_ERR_INVALID, "null output vector");
    if (s.kind < RVK_SCALAR_CONST || s.kind > RVK_SCALAR_RECIP_PTR)
        return set_error(RVK_ERR_INVALID, "bad scalar kind %d", s.kind);
    if (s.kind != RVK_SCALAR_CONST && !s.p0) return set_error(RVK_ERR_INVALID, "null scalar ptr");
    if (s.kind == RVK_SCALAR_DIV_PTR_PTR && !s.p1)
        return set_error(RVK_ERR_INVALID, "null scalar divisor ptr");
    const bool vec = aligned16(out) && (!x || aligned16(x)) && (!y || aligned16(y));
    const int  g   = elementwise_grid(vec ? (n + 1) / 2 : n);
    k_elementwise<OP><<<g, kReduceThreads, 0, stream>>>(n, s, x, y, out, vec, guard);
    RVK_CHECK_LAUNCH("k_elementwise");
    return RVK_OK;
}

} // namespace

rvk_scalar const_scalar(double c) { return rvk_scalar{RVK_SCALAR_CONST, c, nullptr, nullptr}; }

rvk_status vec_reduce(cudaStream_t st, Scratch sc, int op, int64_t n, const double* x,
                      const double* y, double* o0, double* o1, const int* guard)
{
    switch (op) {
    case RED_DOT: return launch_reduce<0>(st, sc, n, x, y, o0, o1, guard);
    case RED_NRM2: return launch_reduce<1>(st, sc, n, x, y, o0, o1, guard);
    case RED_DOT2: return launch_reduce<2>(st, sc, n, x, y, o0, o1, guard);
    }
    return set_error(RVK_ERR_INVALID, "bad reduction op");
}

rvk_status vec_ew(cudaStream_t st, int op, int64_t n, rvk_scalar s, const double* x,
                  const double* y, double* out, const int* guard)
{
    switch (op) {
    case EW_AXPY: return launch_ew<EW_AXPY>(st, n, s, x, y, out, guard);
    case EW_AYPX: return launch_ew<EW_AYPX>(st, n, s, x, y, out, guard);
    case EW_WAXPY: return launch_ew<EW_WAXPY>(st, n, s, x, y, out, guard);
    case EW_SCALE: return launch_ew<EW_SCALE>(st, n, s, x, y, out, guard);
    case EW_PMULT: return launch_ew<EW_PMULT>(st, n, s, x, y, out, guard);
    case EW_SET: return launch_ew<EW_SET>(st, n, s, x, y, out, guard);
    }
    return set_error(RVK_ERR_INVALID, "bad elementwise op");
}

int reduce_grid(int64_t n)
{
    // >= 4 elements per thread, at most 8 blocks per SM, always a fixed
    // function of n (determinism).
    const int64_t per  = (int64_t)kReduceThreads * 4;
    int64_t       want = (n + per - 1) / per;
    const int64_t cap  = (int64_t)sm_count() * 8;
    if (cap > kMaxReduceBlocks) return kMaxReduceBlocks;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

} // namespace rvk

using namespace rvk;

extern "C" {

rvk_status rvk_dot(rvk_ctx ctx, int64_t n, const double* x, const double* y, double* out_dev)
{
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    RVK_TRACE_TASK(ctx, "rvk_dot");
    return launch_reduce<0>(ctx->stream, ctx->scratch, n, x, y, out_dev, nullptr, nullptr);
}

rvk_status rvk_nrm2(rvk_ctx ctx, int64_t n, const double* x, double* out_dev)
{
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    RVK_TRACE_TASK(ctx, "rvk_nrm2");
    return launch_reduce<1>(ctx->stream, ctx->scratch, n, x, nullptr, out_dev, nullptr, nullptr);
}

rvk_status rvk_dot2(rvk_ctx ctx, int64_t n, const double* z, const double* r, double* zz_dev,
                    double* zr_dev)
{
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    RVK_TRACE_TASK(ctx, "rvk_dot2");
    return launch_reduce<2>(ctx->stream, ctx->scratch, n, z, r, zz_dev, zr_dev, nullptr);
}

rvk_status rvk_axpy(rvk_ctx ctx, int64_t n, rvk_scalar a, const double* x, double* y)
{
    if (n > 0 && (!x || !y)) return set_error(RVK_ERR_INVALID, "axpy: null vector");
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    RVK_TRACE_TASK(ctx, "rvk_axpy");
    return launch_ew<EW_AXPY>(ctx->stream, n, a, x, y, y, nullptr);
}

rvk_status rvk_aypx(rvk_ctx ctx, int64_t n, rvk_scalar b, const double* x, double* y)
{
    if (n > 0 && (!x || !y)) return set_error(RVK_ERR_INVALID, "aypx: null vector");
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    RVK_TRACE_TASK(ctx, "rvk_aypx");
    return launch_ew<EW_AYPX>(ctx->stream, n, b, x, y, y, nullptr);
}

rvk_status rvk_waxpy(rvk_ctx ctx, int64_t n, rvk_scalar a, const double* x, const double* y,
                     double* w)
{
    if (n > 0 && (!x || !y)) return set_error(RVK_ERR_INVALID, "waxpy: null vector");
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    RVK_TRACE_TASK(ctx, "rvk_waxpy");
    return launch_ew<EW_WAXPY>(ctx->stream, n, a, x, y, w, nullptr);
}

rvk_status rvk_scale(rvk_ctx ctx, int64_t n, rvk_scalar a, double* x)
{
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    RVK_TRACE_TASK(ctx, "rvk_scale");
    return launch_ew<EW_SCALE>(ctx->stream, n, a, nullptr, x, x, nullptr);
}

rvk_status rvk_pointwise_mult(rvk_ctx ctx, int64_t n, const double* a, const double* b,
                              double* out)
{
    if (n > 0 && (!a || !b)) return set_error(RVK_ERR_INVALID, "pointwise_mult: null vector");
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    RVK_TRACE_TASK(ctx, "rvk_pointwise_mult");
    return launch_ew<EW_PMULT>(ctx->stream, n, const_scalar(0.0), a, b, out, nullptr);
}

rvk_status rvk_set(rvk_ctx ctx, int64_t n, double value, double* x)
{
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    RVK_TRACE_TASK(ctx, "rvk_set");
    return launch_ew<EW_SET>(ctx->stream, n, const_scalar(value), nullptr, nullptr, x, nullptr);
}

rvk_status rvk_copy(rvk_ctx ctx, int64_t n, const double* src, double* dst)
{
    if (!ctx) return set_error(RVK_ERR_INVALID, "null context");
    if (n < 0) return set_error(RVK_ERR_INVALID, "negative length");
    if (n == 0 || src == dst) return RVK_OK;
    RVK_TRACE_TASK(ctx, "rvk_copy");
    RVK_CUDA(cudaMemcpyAsync(dst, src, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    return RVK_OK;
}

rvk_status rvk_scalar_eval(rvk_ctx ctx, rvk_scalar s, double* out_dev)
{
    if (!ctx || !out_dev) return set_error(RVK_ERR_INVALID, "scalar_eval: null argument");
    if (s.kind < RVK_SCALAR_CONST || s.kind > RVK_SCALAR_RECIP_PTR)
        return set_error(RVK_ERR_INVALID, "bad scalar kind %d", s.kind);
    if (s.kind != RVK_SCALAR_CONST && !s.p0) return set_error(RVK_ERR_INVALID, "null scalar ptr");
    if (s.kind == RVK_SCALAR_DIV_PTR_PTR && !s.p1)
        return set_error(RVK_ERR_INVALID, "null scalar divisor ptr");
    RVK_TRACE_TASK(ctx, "rvk_scalar_eval");
    k_scalar_eval<<<1, 1, 0, ctx->stream>>>(s, out_dev);
    RVK_CHECK_LAUNCH("k_scalar_eval");
    return RVK_OK;
}

} // extern "C"
