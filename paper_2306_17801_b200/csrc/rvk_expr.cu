// rvk_expr.cu -- device side of Eval()/execute() (expr.cpp:314-386 restated
// for the GPU): one thread per target element walks the folded, CSE'd step
// program; leaves are read in place from device memory.  IEEE +,-,*,/,sqrt
// round exactly like the host interpreter; sin/cos/exp use CUDA's libdevice
// (<= 2 ulp from glibc).  Also the CG breakdown monitor used by the
// API-level (listing) solver.
#include "api/internal.hpp"
#include "rvk_common.cuh"

namespace rivulet::detail {

namespace {

__device__ double un(std::uint8_t op, double a)
{
    switch (op) {
    case 0: return -a;
    case 1: return fabs(a);
    case 2: return sqrt(a);
    case 3: return sin(a);
    case 4: return cos(a);
    case 5: return exp(a);
    }
    return a;
}

__device__ double bin(std::uint8_t op, double a, double b)
{
    switch (op) {
    case 0: return __dadd_rn(a, b);
    case 1: return __dsub_rn(a, b);
    case 2: return __dmul_rn(a, b);
    case 3: return a / b;
    case 4: return fmin(a, b);
    case 5: return fmax(a, b);
    }
    return a;
}

__global__ void k_expr(ExprProgramDev prog, double* out, std::size_t len)
{
    const std::size_t i = (std::size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    double slot[kMaxExprSteps];
    for (int s = 0; s < prog.n_steps; ++s) {
        const ExprStep& st = prog.steps[s];
        double          v  = 0.0;
        switch (st.kind) {
        case 0: v = st.leaf[st.len == 1 ? 0 : i]; break;
        case 1: v = st.value; break;
        case 2: v = un(st.op, slot[st.a]); break;
        case 3: v = bin(st.op, slot[st.a], slot[st.b]); break;
        }
        slot[s] = v;
    }
    out[i] = slot[prog.n_steps - 1];
}

// flag (int): INT_MAX while healthy; the smallest iteration whose ratio
// num/den hits a zero divisor or a non-finite value is recorded.
// atomicMin: checks issued from different contexts may land in any order.
__global__ void k_breakdown(const double* num, const double* den, int iteration, int* flag)
{
    const double d = *den, q = *num / d;
    if (d == 0.0 || !isfinite(q)) atomicMin(flag, iteration);
}

} // namespace

rvk_status expr_run(cudaStream_t s, const ExprProgramDev& prog, double* out, std::size_t len)
{
    if (len == 0) return RVK_OK;
    const int threads = 128;
    k_expr<<<(unsigned)((len + threads - 1) / threads), threads, 0, s>>>(prog, out, len);
    RVK_CHECK_LAUNCH("k_expr");
    return RVK_OK;
}

rvk_status breakdown_check(cudaStream_t s, const double* num, const double* den, int iteration,
                           int* flag)
{
    k_breakdown<<<1, 1, 0, s>>>(num, den, iteration, flag);
    RVK_CHECK_LAUNCH("k_breakdown");
    return RVK_OK;
}

} // namespace rivulet::detail
