// rvk_cg_small.cu -- the whole Jacobi-CG solve as ONE persistent cooperative
// kernel, for grids whose working set sits in L2 (the SURVEY.md 8d latency
// sweep, 64^2 ... 1024^2).  There, a 20-iteration solve is bounded by
// per-launch latency (41 launches even inside a CUDA graph), not by HBM; the
// paper's scalar problem at its purest.
//
// Phases are separated by grid-wide barriers (cooperative launch, all blocks
// co-resident); every block folds the per-block partials itself in block
// order, so each block derives identical scalars (alpha, beta, dp) and takes
// identical exit decisions -- no atomics on floating point, no host.
// Element arithmetic is the reference's (mul-then-add, same operand order);
// vectors written inside the kernel are re-read through L2 (__ldcg), never
// through the non-coherent read-only path.
#include "rvk_cg.cuh"
#include "rvk_common.cuh"
#include "rvk_context.hpp"
#include "rvk_internal.hpp"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace rvk {

namespace {

constexpr int kPThreads = 256;

// Fold slot `j` of every block's partials in block order; result broadcast
// to the whole block (identical in every block).
__device__ __forceinline__ double fold_slot(const double* partials, int j, double* sh)
{
    const int tid = threadIdx.x;
    if (tid < 32) {
        double v = 0.0;
        for (int blk = tid; blk < (int)gridDim.x; blk += 32) v += __ldcg(partials + blk * 4 + j);
        v = warp_sum(v);
        if (tid == 0) *sh = v;
    }
    __syncthreads();
    const double out = *sh;
    __syncthreads();
    return out;
}

template <bool JACOBI>
__global__ void __launch_bounds__(kPThreads) k_cg_persistent(PersistArgs a)
{
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[64];
    __shared__ double bcast;
    const int     tid    = threadIdx.x;
    const bool    lead   = blockIdx.x == 0 && tid == 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0     = (int64_t)blockIdx.x * blockDim.x + tid;

    // ---- setup: r = b, x = 0, z = B r; z.z, z.r ----------------------------
    double acc[2] = {0.0, 0.0};
    for (int64_t i = t0; i < a.n; i += stride) {
        const double bi = a.b[i];
        const double zi = JACOBI ? mul(a.dinv[i], bi) : bi;
        a.r[i] = bi;
        a.z[i] = zi;
        a.x[i] = 0.0;
        acc[0] = add(acc[0], mul(zi, zi));
        acc[1] = add(acc[1], mul(zi, bi));
    }
    block_sum<2>(acc, red, tid, blockDim.x, 1);
    if (tid == 0) {
        a.partials[blockIdx.x * 4 + 0] = acc[0];
        a.partials[blockIdx.x * 4 + 1] = acc[1];
    }
    grid.sync();
    double zz = fold_slot(a.partials, 0, &bcast), beta = fold_slot(a.partials, 1, &bcast);
    const double dp0 = sqrt(zz);
    if (lead) {
        a.hist[0]             = dp0;
        a.st->dp0             = dp0;
        a.st->dp              = dp0;
        a.st->beta            = beta;
        a.st->iterations      = 0;
        a.st->breakdown_iter  = -1;
        a.st->state           = RVK_CG_RUNNING;
        a.st->done            = 0;
    }
    if (cg_converged(dp0, dp0, a.rtol, a.atol)) {
        if (lead) {
            a.st->state = RVK_CG_CONVERGED;
            a.st->done  = 1;
        }
        return;
    }
    double betaold = 0.0;

    for (int it = 0; it < a.max_it; ++it) {
        // ---- K1: p = z + b p_old (on the fly), w = A p, p.w ----------------
        double bb = 0.0;
        if (it > 0) {
            if (betaold == 0.0) {
                if (lead) {
                    a.st->state          = RVK_CG_BREAKDOWN;
                    a.st->breakdown_iter = it;
                    a.st->done           = 1;
                }
                return;
            }
            bb = beta / betaold;
        }
        const double* po = (it & 1) ? a.p1 : a.p0;
        double*       pn = (it & 1) ? a.p0 : a.p1;
        auto src = [&](int64_t j) {
            const double zj = __ldcg(a.z + j);
            return it == 0 ? zj : aypx1(bb, zj, __ldcg(po + j));
        };
        double pw = 0.0;
        for (int64_t i = t0; i < a.n; i += stride) {
            const int64_t kb = __ldg(a.off + i), ke = __ldg(a.off + i + 1);
            double        sum = 0.0;
            for (int64_t k = kb; k < ke; k += 8) {
                int32_t c[8];
                double  v[8];
                bool    ok[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    ok[u]            = k + u < ke;
                    const int64_t ks = ok[u] ? k + u : ke - 1;
                    c[u]             = __ldg(a.cols + ks);
                    v[u]             = __ldg(a.vals + ks);
                }
                double xv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) xv[u] = src(c[u]);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double t = add(sum, mul(v[u], xv[u]));
                    sum            = ok[u] ? t : sum;
                }
            }
            const double p = src(i);
            pn[i]          = p;
            a.w[i]         = sum;
            pw             = add(pw, mul(p, sum));
        }
        double v1[1] = {pw};
        block_sum<1>(v1, red, tid, blockDim.x, 1);
        if (tid == 0) a.partials[blockIdx.x * 4 + 2] = v1[0];
        grid.sync();
        const double pAp = fold_slot(a.partials, 2, &bcast);
        const double al  = beta / pAp;
        if (pAp == 0.0 || !isfinite(al)) {
            if (lead) {
                a.st->state          = RVK_CG_BREAKDOWN;
                a.st->breakdown_iter = it;
                a.st->done           = 1;
                a.st->pAp            = pAp;
            }
            return;
        }
        betaold = beta;
        // ---- K2: x += a p, r += (-a) w, z = B r; z.z, z.r ---------------
        const double na = -al;
        acc[0] = acc[1] = 0.0;
        for (int64_t i = t0; i < a.n; i += stride) {
            a.x[i]          = axpy1(al, __ldcg(pn + i), a.x[i]);
            const double ri = axpy1(na, __ldcg(a.w + i), a.r[i]);
            const double zi = JACOBI ? mul(a.dinv[i], ri) : ri;
            a.r[i]          = ri;
            a.z[i]          = zi;
            acc[0]          = add(acc[0], mul(zi, zi));
            acc[1]          = add(acc[1], mul(zi, ri));
        }
        block_sum<2>(acc, red, tid, blockDim.x, 1);
        if (tid == 0) {
            a.partials[blockIdx.x * 4 + 0] = acc[0];
            a.partials[blockIdx.x * 4 + 1] = acc[1];
        }
        grid.sync();
        zz              = fold_slot(a.partials, 0, &bcast);
        const double zr = fold_slot(a.partials, 1, &bcast);
        const double dp = sqrt(zz);
        if (lead) {
            a.hist[it + 1]  = dp;
            a.st->dp        = dp;
            a.st->alpha     = al;
            a.st->pAp       = pAp;
            a.st->betaold   = betaold;
            a.st->iterations = it + 1;
        }
        if (cg_converged(dp, dp0, a.rtol, a.atol)) {
            if (lead) {
                a.st->state = RVK_CG_CONVERGED;
                a.st->done  = 1;
            }
            return;
        }
        beta = zr;
        if (lead) a.st->beta = beta;
    }
}

} // namespace

int persistent_grid(int64_t n)
{
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_persistent<true>, kPThreads, 0) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    const int64_t cap  = (int64_t)sm_count() * std::min(per_sm, 2);
    const int64_t want = (n + kPThreads * 4 - 1) / (kPThreads * 4); // >= 4 rows per thread
    return (int)std::max<int64_t>(1, std::min(cap, want));
}

rvk_status launch_persistent(cudaStream_t s, const PersistArgs& args, bool jacobi, int grid)
{
    void* kargs[] = {const_cast<PersistArgs*>(&args)};
    const void* fn = jacobi ? (const void*)k_cg_persistent<true> : (const void*)k_cg_persistent<false>;
    RVK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kPThreads), kargs, 0, s));
    return RVK_OK;
}

} // namespace rvk
