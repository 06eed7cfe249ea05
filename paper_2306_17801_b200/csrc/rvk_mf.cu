// rvk_mf.cu -- matrix-free K1 for the constant-coefficient stencils
// (the reference's SPEC.md:556 lists matrix-free as a
// non-goal of the *artifact*, the paper's JAX comparison uses it,
// PAPER.md:378-382).
//
// Same CG semantics as the CSR K1 (CgSpmvOp init/row/tail: p = z + b p_old
// on the fly, w = A p, p.w, alpha tail), but the operator is applied from the
// grid geometry: row i = (x, y, z) visits its in-grid neighbours in the
// (dz, dy, dx) ascending order rvk_build_laplacian writes them, multiplying
// by the centre weight or -1 with the same rounding -- so w is bit-identical
// to the CSR path while the 12 B/nnz + 8 B/row of CSR traffic disappear.
// Per iteration HBM bytes drop from 12 nnz + 8 (n+1) + 96 n to 88 n (K2 reads
// no dinv: the Jacobi diagonal is the constant centre weight).
#include "rvk_cg.cuh"
#include "rvk_common.cuh"
#include "rvk_context.hpp"
#include "rvk_internal.hpp"
#include "rvk_spmv.cuh"

namespace rvk {

namespace {

constexpr int kMfThreads = 256;

// Unsigned 32-bit division by a run-time constant via multiply-high (the
// coordinates of a row without the 64-bit division subroutine).
struct FastDiv {
    uint32_t d, mul, shift;
    static FastDiv make(uint32_t d)
    {
        FastDiv f{d, 0, 0};
        while ((1ull << f.shift) < d) ++f.shift;
        f.mul = (uint32_t)(((1ull << 32) * ((1ull << f.shift) - d)) / d + 1);
        return f;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const
    {
        return (uint32_t)(((uint64_t)__umulhi(n, mul) + n) >> shift);
    }
};

template <class F>
__device__ __forceinline__ F shfl_fetch_up(const F& v)
{
    F o = v;
    o.z = __shfl_up_sync(0xffffffffu, v.z, 1);
    o.p = __shfl_up_sync(0xffffffffu, v.p, 1);
    return o;
}
template <class F>
__device__ __forceinline__ F shfl_fetch_down(const F& v)
{
    F o = v;
    o.z = __shfl_down_sync(0xffffffffu, v.z, 1);
    o.p = __shfl_down_sync(0xffffffffu, v.p, 1);
    return o;
}

// One row per thread; consecutive lanes own consecutive rows, so the x-1 /
// x+1 neighbours of a grid line come from the neighbouring lanes by shuffle
// (warp-edge lanes load them) and each (dy, dz) line costs one coalesced load
// per vector.  All loads are issued before any product is formed.
template <bool FIRST, int DIM, bool BOX>
__global__ void __launch_bounds__(kMfThreads, 2)
    k_mf_cg(StencilGeom g, FastDiv fdx, FastDiv fdy, CgSpmvOp<FIRST> op_in, TailArgs tail,
            int64_t lead_lo, int64_t lead_hi)
{
    using F = typename CgSpmvOp<FIRST>::Fetch;
    CgSpmvOp<FIRST> op = op_in;
    if (!op.init()) return; // device-side early exit (converged / breakdown)
    __shared__ double red[32];
    __shared__ int    flag;
    constexpr int     ZR = DIM == 3 ? 1 : 0;
    constexpr int     NL = (2 * ZR + 1) * 3; // (dz, dy) lines
    const int32_t     nx = (int32_t)g.nx, ny = (int32_t)g.ny, nz = (int32_t)g.nz;
    const int32_t     nxy    = (int32_t)(g.nx * g.ny);
    const int64_t     ntiles = (g.n + kMfThreads - 1) / kMfThreads;
    const int         lane   = threadIdx.x & 31;
    double            acc    = 0.0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        if (threadIdx.x == 0) {
            // first-touch columns of this block's next tile (highest band)
            const int64_t tn = t + gridDim.x;
            if (tn < ntiles) {
                int64_t lo = max(tn * kMfThreads + lead_lo, (int64_t)0) & ~int64_t(1);
                int64_t hi = min(tn * kMfThreads + kMfThreads + lead_hi, g.n) & ~int64_t(1);
                if (hi > lo) {
                    bulk_prefetch_l2(op.z + lo, (uint32_t)(hi - lo) * 8);
                    if (!FIRST) bulk_prefetch_l2(op.p_old + lo, (uint32_t)(hi - lo) * 8);
                }
            }
        }
        const int64_t irow = t * kMfThreads + threadIdx.x;
        const bool    live = irow < g.n;
        const int32_t i    = (int32_t)(live ? irow : g.n - 1); // dead lanes still shuffle
        const uint32_t q   = fdx.div((uint32_t)i);
        const int32_t  xc  = i - (int32_t)q * nx;
        const int32_t  zc  = (int32_t)fdy.div(q);
        const int32_t  yc  = (int32_t)q - zc * ny;
        const bool     xl = xc > 0, xr = xc < nx - 1;
        // ---- phase 1: every load of the row ------------------------------------
        F    ctr[NL], eL[NL], eR[NL];
        bool lin[NL];
#pragma unroll
        for (int L = 0; L < NL; ++L) {
            const int  dz = L / 3 - ZR, dy = L % 3 - 1;
            const bool used = BOX || dz == 0 || dy == 0; // star: no diagonal lines
            const bool xs   = BOX || (dz == 0 && dy == 0); // line uses x +- 1
            lin[L]          = used && yc + dy >= 0 && yc + dy < ny && zc + dz >= 0 && zc + dz < nz;
            const int32_t jl = lin[L] ? i + dy * nx + dz * nxy : i;
            ctr[L]           = op.fetch(jl);
            if (xs) {
                eL[L] = op.fetch(lane == 0 && xl ? jl - 1 : jl);
                eR[L] = op.fetch(lane == 31 && xr ? jl + 1 : jl);
            }
        }
        // ---- phase 2: x-neighbours from the neighbouring lanes ---------------------
        F lft[NL], rgt[NL];
#pragma unroll
        for (int L = 0; L < NL; ++L) {
            const int  dz = L / 3 - ZR, dy = L % 3 - 1;
            const bool xs = BOX || (dz == 0 && dy == 0);
            if (xs) {
                const F u = shfl_fetch_up(ctr[L]), d = shfl_fetch_down(ctr[L]);
                lft[L]    = lane == 0 ? eL[L] : u;
                rgt[L]    = lane == 31 ? eR[L] : d;
            }
        }
        // ---- phase 3: products in ascending column order (dz, dy, dx) ---------
        double sum = 0.0;
#pragma unroll
        for (int L = 0; L < NL; ++L) {
            const int  dz = L / 3 - ZR, dy = L % 3 - 1;
            const bool xs = BOX || (dz == 0 && dy == 0);
            const bool c  = dz == 0 && dy == 0;
            if (xs) {
                const double tl = add(sum, mul(-1.0, op.value(lft[L])));
                sum             = lin[L] && xl ? tl : sum;
            }
            const double tc = add(sum, mul(c ? g.centre : -1.0, op.value(ctr[L])));
            sum             = lin[L] ? tc : sum;
            if (xs) {
                const double tr = add(sum, mul(-1.0, op.value(rgt[L])));
                sum             = lin[L] && xr ? tr : sum;
            }
        }
        if (live) acc = op.row(irow, sum, acc, ctr[NL / 2]);
    }
    double v[1] = {acc};
    block_sum<1>(v, red, threadIdx.x, kMfThreads, 1);
    if (threadIdx.x == 0) tail.partials[blockIdx.x] = v[0];
    if (!last_block(tail.ticket, threadIdx.x, &flag, kMfThreads, 1)) return;
    fold_partials<1>(tail.partials, gridDim.x, v, red, threadIdx.x, kMfThreads, 1);
    if (threadIdx.x == 0) {
        op.tail(v[0]);
        *tail.ticket = 0u;
    }
}

template <bool FIRST>
rvk_status launch_first(cudaStream_t s, const StencilGeom& g, const CgSpmvOp<FIRST>& op,
                        TailArgs ta, int grid)
{
    // leading edge: the dz = +1 plane (3D) or dy = +1 line (2D), +-1 row/column
    const int64_t far = g.dim == 3 ? g.nx * g.ny : g.nx;
    const int64_t lo = far - (g.dim == 3 ? g.nx : 0) - 1, hi = far + (g.dim == 3 ? g.nx : 0) + 1;
    const FastDiv fx = FastDiv::make((uint32_t)g.nx), fy = FastDiv::make((uint32_t)g.ny);
    if (g.dim == 3 && g.box) k_mf_cg<FIRST, 3, true><<<grid, kMfThreads, 0, s>>>(g, fx, fy, op, ta, lo, hi);
    else if (g.dim == 3) k_mf_cg<FIRST, 3, false><<<grid, kMfThreads, 0, s>>>(g, fx, fy, op, ta, lo, hi);
    else if (g.box) k_mf_cg<FIRST, 2, true><<<grid, kMfThreads, 0, s>>>(g, fx, fy, op, ta, lo, hi);
    else k_mf_cg<FIRST, 2, false><<<grid, kMfThreads, 0, s>>>(g, fx, fy, op, ta, lo, hi);
    RVK_CHECK_LAUNCH("k_mf_cg");
    return RVK_OK;
}

} // namespace

int mf_grid(const StencilGeom& g)
{
    int per_sm = 0;
    cudaError_t e;
    if (g.dim == 3 && g.box) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_cg<false, 3, true>, kMfThreads, 0);
    else if (g.dim == 3) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_cg<false, 3, false>, kMfThreads, 0);
    else if (g.box) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_cg<false, 2, true>, kMfThreads, 0);
    else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_cg<false, 2, false>, kMfThreads, 0);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    const int64_t tiles = (g.n + kMfThreads - 1) / kMfThreads;
    return (int)std::min<int64_t>(tiles, (int64_t)sm_count() * per_sm);
}

rvk_status launch_mf_k1(cudaStream_t s, const StencilGeom& g, bool first, const double* z,
                        const double* p_old, double* p_new, double* w, CgState* st, int64_t n,
                        int it, double* partials, unsigned int* ticket, int grid)
{
    const TailArgs ta{partials, ticket};
    if (first) return launch_first(s, g, CgSpmvOp<true>{z, p_old, p_new, w, st, n, it, 0.0}, ta, grid);
    return launch_first(s, g, CgSpmvOp<false>{z, p_old, p_new, w, st, n, it, 0.0}, ta, grid);
}

} // namespace rvk
