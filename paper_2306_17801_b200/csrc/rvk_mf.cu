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
//
// Two kernels:
//  * k_mf_tma (default when the grid allows a TMA tensor map: even nx): 2.5D
//    marching.  A block owns a TX x TY tile of the (x, y) plane (2D: a TX
//    segment of x) and marches through a chunk of planes (2D: rows).  Each
//    plane's (TX+4) x (TY+2) box of z and p_old (the halo included; x starts
//    at x0-2 because TMA needs a 16-B aligned innermost start) arrives by
//    ONE cp.async.bulk.tensor per vector into a kTmaStages-deep ring; OOB
//    coordinates are zero-filled by the TMA unit, so the grid boundary needs
//    no branches: p = z + b p_old is formed ONCE per element into a 4-plane
//    ring (p(OOB) = +0), and every row adds its neighbours in ascending
//    column order -- an out-of-grid neighbour contributes (-1) * (+0) = -0,
//    and sum + (-0) == sum exactly, so w is bit-identical to the CSR path,
//    which skips it.  Each z / p_old element is fetched once (plus the halo,
//    served by L2 from the neighbouring tiles): no index division, no
//    redundant gathers.
//  * k_mf_cg: one row per thread with fast-divmod coordinates and warp
//    shuffles for the x-neighbours (any geometry; the fallback).
#include "rvk_cg.cuh"
#include "rvk_common.cuh"

#include <cuda.h> // CUtensorMap + enums; cuTensorMapEncodeTiled is resolved at run time

#include <mutex>
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
template <class OpT, int DIM, bool BOX>
__global__ void __launch_bounds__(kMfThreads, 2)
    k_mf_cg(StencilGeom g, FastDiv fdx, FastDiv fdy, OpT op_in, TailArgs tail,
            int64_t lead_lo, int64_t lead_hi)
{
    constexpr bool FIRST = OpT::kFirst;
    using F              = typename OpT::Fetch;
    OpT op               = op_in;
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

// ---------------------------------------------------------------------------
// TMA 2.5D marching kernel
// ---------------------------------------------------------------------------
struct MfTmaGeom {
    int32_t nx, ny, nm;       // plane extent (2D: nx, 1) and marching extent (3D nz, 2D ny)
    int32_t tiles_x, tiles_y; // plane tiles
    int32_t chunk;            // planes per block
    double  centre;
};

// Tile of the plane per block (TX x TY rows), RY rows per thread along y,
// ring depth.  27-point: each thread sweeps 2 y-rows so every loaded p value
// of a (plane, line) serves the up-to-3 rows it neighbours -- 12 shared-memory
// loads per plane for 2 rows instead of 18 (the 1-row kernel is bound by its
// 27 LDS per row).
template <int DIM, bool BOX>
struct MfShape {
    static constexpr int TX = 128, TY = 1, RY = 1, STAGES = 6; // 2D
};
template <>
struct MfShape<3, false> {
    static constexpr int TX = 32, TY = 8, RY = 1, STAGES = 6;
};
template <>
struct MfShape<3, true> {
    static constexpr int TX = 32, TY = 16, RY = 2, STAGES = 2;
};
template <int DIM, bool BOX>
constexpr int mf_threads()
{
    return MfShape<DIM, BOX>::TX * (MfShape<DIM, BOX>::TY / MfShape<DIM, BOX>::RY);
}
// dynamic shared memory of k_mf_tma: STAGES x 2 boxes + 4 p planes (box pitch BP)
template <int DIM, bool BOX>
constexpr size_t mf_smem_bytes()
{
    using S          = MfShape<DIM, BOX>;
    constexpr int be = (S::TX + 4) * (DIM == 3 ? S::TY + 2 : 1);
    constexpr int bp = (be + 15) & ~15;
    return sizeof(double) * (size_t)bp * (2 * S::STAGES + 4);
}

template <int DIM>
__device__ __forceinline__ void tma_plane(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                          int32_t m, uint64_t* bar)
{
    if constexpr (DIM == 3)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
                     "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(m), "r"(smem_u32(bar))
                     : "memory");
    else
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
                     "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(m), "r"(smem_u32(bar))
                     : "memory");
    (void)y;
}

template <class OpT, int DIM, bool BOX>
__global__ void __launch_bounds__(mf_threads<DIM, BOX>())
    k_mf_tma(const __grid_constant__ CUtensorMap tz, const __grid_constant__ CUtensorMap tp,
             MfTmaGeom g, OpT op_in, TailArgs tail)
{
    using S                    = MfShape<DIM, BOX>;
    constexpr int TX = S::TX, TY = S::TY, RY = S::RY, NT = mf_threads<DIM, BOX>();
    constexpr int kTmaStages   = S::STAGES;
    // box: x0-2 .. x0+TX+1 (the innermost TMA start coordinate must be 16-B
    // aligned -- x0-1 traps with an illegal instruction on B200, measured),
    // y0-1 .. y0+TY (3D), one plane
    constexpr int BW = TX + 4, BH = DIM == 3 ? TY + 2 : 1, BE = BW * BH;
    constexpr int BP   = (BE + 15) & ~15; // box pitch: every TMA destination 128-B aligned
    constexpr bool FIRST = OpT::kFirst;
    constexpr int NSRC = FIRST ? 1 : 2;
    // dynamic shared memory (> 48 KB for the 27-point tile): [z | p_old] box
    // ring, then the 4-plane p ring
    extern __shared__ __align__(128) unsigned char mf_smem[];
    auto stage = reinterpret_cast<double(*)[2][BP]>(mf_smem);
    auto pr    = reinterpret_cast<double(*)[BP]>(mf_smem + sizeof(double) * kTmaStages * 2 * BP);
    __shared__ __align__(8) uint64_t full[kTmaStages];
    __shared__ double                red[32];
    __shared__ int                   flag;

    OpT op = op_in;
    if (!op.init()) return; // device-side early exit (converged / breakdown)
    const int     tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
    const int32_t tiles = g.tiles_x * g.tiles_y;
    const int32_t tile = (int32_t)blockIdx.x % tiles, ch = (int32_t)blockIdx.x / tiles;
    const int32_t x0 = (tile % g.tiles_x) * TX, y0 = (tile / g.tiles_x) * TY;
    const int32_t m0 = ch * g.chunk, m1 = min(m0 + g.chunk, g.nm);
    const int     nsteps = (m1 - m0) + 2; // planes m0-1 .. m1 (p of both neighbours)
    if (tid == 0) {
        for (int k = 0; k < kTmaStages; ++k) mbar_init(&full[k], 1);
        fence_mbar_init();
    }
    __syncthreads();
    // the tensor maps must be addressed in parameter space (a lambda capture
    // would copy them to local memory, where TMA cannot read a descriptor)
    const CUtensorMap* mz = &tz;
    const CUtensorMap* mp = &tp;
#define RVK_MF_ISSUE(j)                                                                            \
    do {                                                                                           \
        const int k_ = (j) % kTmaStages;                                                           \
        mbar_arrive_expect_tx(&full[k_], NSRC * BE * 8);                                           \
        tma_plane<DIM>(&stage[k_][0][0], mz, x0 - 2, y0 - 1, m0 - 1 + (j), &full[k_]);             \
        if (!FIRST) tma_plane<DIM>(&stage[k_][1][0], mp, x0 - 2, y0 - 1, m0 - 1 + (j), &full[k_]); \
    } while (0)
    if (tid == 0)
        for (int j = 0; j < min(kTmaStages, nsteps); ++j) RVK_MF_ISSUE(j);
    // this thread's rows: (x, y0 + ty*RY + r), r < RY; box index of row r: c + r*BW
    const int     c  = (DIM == 3 ? (ty * RY + 1) * BW : 0) + tx + 2;
    const int32_t x = x0 + tx, y = y0 + ty * RY;
    double        acc = 0.0;
    for (int j = 0; j < nsteps; ++j) {
        const int k = j % kTmaStages;
        mbar_wait(&full[k], (j / kTmaStages) & 1);
        double* P = pr[j & 3];
        for (int e = tid; e < BE; e += NT) {
            const double zv = op.zval(stage[k][0][e]); // ZV: the box holds r, z = d r
            P[e]            = FIRST ? zv : aypx1(op.b, zv, stage[k][1][e]);
        }
        __syncthreads(); // ring slot j complete; stage k consumed by every thread
        if (tid == 0 && j + kTmaStages < nsteps) RVK_MF_ISSUE(j + kTmaStages);
        if (j < 2) continue;
        // rows (x, y+r, m) with m = m0 + j - 2: planes m-1, m, m+1 = ring j-2, j-1, j
        const double* Pl[3] = {pr[(j - 2) & 3], pr[(j - 1) & 3], pr[j & 3]};
        double        sum[RY];
#pragma unroll
        for (int r = 0; r < RY; ++r) sum[r] = 0.0;
        auto term = [&](int r, double coef, double v) { sum[r] = add(sum[r], mul(coef, v)); };
        if constexpr (BOX) {
            // (dz, line, dx) ascending; a line yy feeds every row r with
            // dy = yy - r in [-1, 1] -- per row the terms stay in ascending
            // column order (dz, dy, dx), exactly the CSR's
#pragma unroll
            for (int dz = 0; dz < 3; ++dz)
#pragma unroll
                for (int yy = (DIM == 3 ? -1 : 0); yy <= (DIM == 3 ? RY : 0); ++yy)
#pragma unroll
                    for (int dx = -1; dx <= 1; ++dx) {
                        const double v = Pl[dz][c + yy * BW + dx];
#pragma unroll
                        for (int r = 0; r < RY; ++r) {
                            const int dy = yy - r;
                            if (DIM == 3 && (dy < -1 || dy > 1)) continue;
                            term(r, dz == 1 && dy == 0 && dx == 0 ? g.centre : -1.0, v);
                        }
                    }
        } else {
            term(0, -1.0, Pl[0][c]);
            if (DIM == 3) term(0, -1.0, Pl[1][c - BW]);
            term(0, -1.0, Pl[1][c - 1]);
            term(0, g.centre, Pl[1][c]);
            term(0, -1.0, Pl[1][c + 1]);
            if (DIM == 3) term(0, -1.0, Pl[1][c + BW]);
            term(0, -1.0, Pl[2][c]);
        }
#pragma unroll
        for (int r = 0; r < RY; ++r)
            if (x < g.nx && y + r < g.ny) {
                const int64_t i = ((int64_t)(m0 + j - 2) * g.ny + y + r) * g.nx + x;
                const double  p = Pl[1][c + r * BW];
                op.p_new[i]     = p;
                op.w[i]         = sum[r];
                acc             = add(acc, mul(p, sum[r]));
            }
    }
#undef RVK_MF_ISSUE
    double v[1] = {acc};
    block_sum<1>(v, red, tid, NT, 1);
    if (tid == 0) tail.partials[blockIdx.x] = v[0];
    if (!last_block(tail.ticket, tid, &flag, NT, 1)) return;
    fold_partials<1>(tail.partials, gridDim.x, v, red, tid, NT, 1);
    if (tid == 0) {
        op.tail(v[0]);
        *tail.ticket = 0u;
    }
}

template <class OpT>
rvk_status launch_first(cudaStream_t s, const StencilGeom& g, const OpT& op,
                        TailArgs ta, int grid)
{
    // leading edge: the dz = +1 plane (3D) or dy = +1 line (2D), +-1 row/column
    const int64_t far = g.dim == 3 ? g.nx * g.ny : g.nx;
    const int64_t lo = far - (g.dim == 3 ? g.nx : 0) - 1, hi = far + (g.dim == 3 ? g.nx : 0) + 1;
    const FastDiv fx = FastDiv::make((uint32_t)g.nx), fy = FastDiv::make((uint32_t)g.ny);
    if (g.dim == 3 && g.box) launch_k(k_mf_cg<OpT, 3, true>, grid, kMfThreads, 0, s, g, fx, fy, op, ta, lo, hi);
    else if (g.dim == 3) launch_k(k_mf_cg<OpT, 3, false>, grid, kMfThreads, 0, s, g, fx, fy, op, ta, lo, hi);
    else if (g.box) launch_k(k_mf_cg<OpT, 2, true>, grid, kMfThreads, 0, s, g, fx, fy, op, ta, lo, hi);
    else launch_k(k_mf_cg<OpT, 2, false>, grid, kMfThreads, 0, s, g, fx, fy, op, ta, lo, hi);
    RVK_CHECK_LAUNCH("k_mf_cg");
    return RVK_OK;
}

} // namespace

// ---- TMA plan state -----------------------------------------------------------
struct MfTma {
    CUtensorMap   z, r, pm[kMaxXq]; // pm[k]: p buffer k
    MfTmaGeom     g{};
    const double* p_ptr[kMaxXq] = {};
    int           np       = 2;
    int           grid   = 0;
    int           dim    = 3;
    bool          box    = false;
};

namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled()
{
    static EncodeTiledFn  fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void*                           f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(f);
    });
    return fn;
}

// Box (TX+4) x (TY+2) x 1 (2D: (TX+4) x 1) over the grid viewed as
// [march][y][x]; OOB coordinates read as zero (FLOAT_OOB_FILL_NONE).
bool encode_plane_map(CUtensorMap* m, const double* base, const StencilGeom& g, int bw, int bh)
{
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    cuuint64_t dims[3], strides[2];
    cuuint32_t box[3], es[3] = {1, 1, 1};
    cuuint32_t rank;
    if (g.dim == 3) {
        rank    = 3;
        dims[0] = (cuuint64_t)g.nx;
        dims[1] = (cuuint64_t)g.ny;
        dims[2] = (cuuint64_t)g.nz;
        strides[0] = (cuuint64_t)g.nx * 8;
        strides[1] = (cuuint64_t)g.nx * g.ny * 8;
        box[0] = (cuuint32_t)bw;
        box[1] = (cuuint32_t)bh;
        box[2] = 1;
    } else {
        rank    = 2;
        dims[0] = (cuuint64_t)g.nx;
        dims[1] = (cuuint64_t)g.ny;
        strides[0] = (cuuint64_t)g.nx * 8;
        box[0] = (cuuint32_t)bw;
        box[1] = 1;
    }
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dims, strides, box,
               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int DIM, bool BOX>
void mf_configure()
{
    // per device (function attributes are per device; plan creation, before
    // any graph capture)
    static std::atomic<uint64_t> configured{0};
    if (!device_first_use(configured)) return;
    const int sm = (int)mf_smem_bytes<DIM, BOX>();
    cudaFuncSetAttribute(k_mf_tma<CgSpmvOp<true, false>, DIM, BOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_mf_tma<CgSpmvOp<false, false>, DIM, BOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_mf_tma<CgSpmvOp<true, true>, DIM, BOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_mf_tma<CgSpmvOp<false, true>, DIM, BOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    device_mark_done(configured);
}

template <int DIM, bool BOX>
int tma_blocks_per_sm()
{
    mf_configure<DIM, BOX>();
    int per_sm = 0;
    constexpr int nt = mf_threads<DIM, BOX>();
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_tma<CgSpmvOp<false, true>, DIM, BOX>, nt,
                                                      mf_smem_bytes<DIM, BOX>()) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    return per_sm;
}
} // namespace

MfTma* mf_tma_create(const StencilGeom& g, const double* z, double* const* p, int np,
                     const double* r)
{
    // TMA needs 16-B global strides (nx even) and 32-bit coordinates
    if (g.nx % 2 || g.nx > (1 << 30) || g.ny > (1 << 30) || g.nz > (1 << 30)) return nullptr;
    auto* t = new MfTma();
    t->dim  = g.dim;
    t->box  = g.box != 0;
    const int TX = g.dim == 3 ? (g.box ? MfShape<3, true>::TX : MfShape<3, false>::TX) : MfShape<2, false>::TX;
    const int TY = g.dim == 3 ? (g.box ? MfShape<3, true>::TY : MfShape<3, false>::TY) : MfShape<2, false>::TY;
    const int bw = TX + 4, bh = g.dim == 3 ? TY + 2 : 1; // see k_mf_tma: 16-B aligned x start
    bool ok = encode_plane_map(&t->z, z, g, bw, bh) && encode_plane_map(&t->r, r, g, bw, bh);
    for (int k = 0; k < np && ok; ++k) ok = encode_plane_map(&t->pm[k], p[k], g, bw, bh);
    if (!ok) {
        delete t;
        return nullptr;
    }
    t->np = np;
    for (int k = 0; k < np; ++k) t->p_ptr[k] = p[k];
    MfTmaGeom& G = t->g;
    G.nx      = (int32_t)g.nx;
    G.ny      = g.dim == 3 ? (int32_t)g.ny : 1;
    G.nm      = g.dim == 3 ? (int32_t)g.nz : (int32_t)g.ny;
    G.tiles_x = (int32_t)((g.nx + TX - 1) / TX);
    G.tiles_y = g.dim == 3 ? (int32_t)((g.ny + TY - 1) / TY) : 1;
    G.centre  = g.centre;
    // chunks of planes: a few waves of resident blocks, >= 16 planes each
    // (every chunk re-reads 2 halo planes), grid within the reduction scratch
    int per_sm = 1;
    if (g.dim == 3) per_sm = g.box ? tma_blocks_per_sm<3, true>() : tma_blocks_per_sm<3, false>();
    else per_sm = g.box ? tma_blocks_per_sm<2, true>() : tma_blocks_per_sm<2, false>();
    const int64_t tiles  = (int64_t)G.tiles_x * G.tiles_y;
    // ~4 waves of resident blocks (measured: 7-point 256^3 K1 125 / 110 / 107 /
    // 101 / 101 us at 1 / 2 / 3 / 4 / 8 waves)
    const int64_t waves  = 4;
    const int64_t want   = waves * sm_count() * per_sm;
    int64_t       chunks = std::max<int64_t>(1, (want + tiles - 1) / tiles);
    chunks               = std::min<int64_t>(chunks, std::max<int64_t>(1, G.nm / 16));
    while (chunks > 1 && tiles * chunks > kMaxReduceBlocks) --chunks;
    if (tiles * chunks > kMaxReduceBlocks) { // too many plane tiles for one launch's scratch
        delete t;
        return nullptr;
    }
    G.chunk = (int32_t)((G.nm + chunks - 1) / chunks);
    t->grid = (int)(tiles * ((G.nm + G.chunk - 1) / G.chunk));
    return t;
}

void mf_tma_destroy(MfTma* t) { delete t; }

int mf_grid(const StencilGeom& g)
{
    int per_sm = 0;
    cudaError_t e;
    if (g.dim == 3 && g.box) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_cg<CgSpmvOp<false, true>, 3, true>, kMfThreads, 0);
    else if (g.dim == 3) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_cg<CgSpmvOp<false, true>, 3, false>, kMfThreads, 0);
    else if (g.box) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_cg<CgSpmvOp<false, true>, 2, true>, kMfThreads, 0);
    else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mf_cg<CgSpmvOp<false, true>, 2, false>, kMfThreads, 0);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    const int64_t tiles = (g.n + kMfThreads - 1) / kMfThreads;
    return (int)std::min<int64_t>(tiles, (int64_t)sm_count() * per_sm);
}

namespace {
template <class OpT>
rvk_status launch_tma(cudaStream_t s, const MfTma& t, const OpT& op, TailArgs ta)
{
    int kp = 0; // the map of p_old among the rotating buffers
    for (int k = 0; k < t.np; ++k)
        if (op.p_old == t.p_ptr[k]) kp = k;
    const CUtensorMap& tp = t.pm[kp];
#define RVK_MF_LAUNCH(D, B)                                                                        \
    launch_k(k_mf_tma<OpT, D, B>, t.grid, mf_threads<D, B>(), mf_smem_bytes<D, B>(), s,            \
               OpT::kZv ? t.r : t.z, tp, t.g, op, ta)
    if (t.dim == 3 && t.box) RVK_MF_LAUNCH(3, true);
    else if (t.dim == 3) RVK_MF_LAUNCH(3, false);
    else if (t.box) RVK_MF_LAUNCH(2, true);
    else RVK_MF_LAUNCH(2, false);
#undef RVK_MF_LAUNCH
    RVK_CHECK_LAUNCH("k_mf_tma");
    return RVK_OK;
}
} // namespace

rvk_status launch_mf_k1(cudaStream_t s, const StencilGeom& g, bool first, const double* z,
                        const double* p_old, double* p_new, double* w, CgState* st, int64_t n,
                        int it, double* partials, unsigned int* ticket, int grid, const MfTma* tma,
                        bool zv, double zs)
{
    const TailArgs ta{partials, ticket};
    if (tma) {
        if (zv) {
            if (first) return launch_tma(s, *tma, CgSpmvOp<true, true>{z, p_old, p_new, w, st, n, it, 0.0, zs}, ta);
            return launch_tma(s, *tma, CgSpmvOp<false, true>{z, p_old, p_new, w, st, n, it, 0.0, zs}, ta);
        }
        if (first) return launch_tma(s, *tma, CgSpmvOp<true>{z, p_old, p_new, w, st, n, it, 0.0}, ta);
        return launch_tma(s, *tma, CgSpmvOp<false>{z, p_old, p_new, w, st, n, it, 0.0}, ta);
    }
    if (zv) {
        if (first) return launch_first(s, g, CgSpmvOp<true, true>{z, p_old, p_new, w, st, n, it, 0.0, zs}, ta, grid);
        return launch_first(s, g, CgSpmvOp<false, true>{z, p_old, p_new, w, st, n, it, 0.0, zs}, ta, grid);
    }
    if (first) return launch_first(s, g, CgSpmvOp<true>{z, p_old, p_new, w, st, n, it, 0.0}, ta, grid);
    return launch_first(s, g, CgSpmvOp<false>{z, p_old, p_new, w, st, n, it, 0.0}, ta, grid);
}

} // namespace rvk
