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
#include <cstdlib>

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
        // all of a lane's loads first (grid <= 2 x 148 blocks: <= 10 per
        // lane), then the adds in ascending block order
        constexpr int kPer = (2 * 148 + 31) / 32;
        double        pv[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int blk = tid + 32 * q;
            pv[q]         = blk < (int)gridDim.x ? __ldcg(partials + blk * 4 + j) : 0.0;
        }
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < kPer; ++q)
            if (tid + 32 * q < (int)gridDim.x) v += pv[q];
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


// ---------------------------------------------------------------------------
// Thread-block-cluster solve for the smallest grids (n <= 16 x 1024 rows):
// ONE cluster of C = ceil(n / 1024) CTAs (<= 16, non-portable size), one row
// per thread.  The gathered vectors z and p (ping-pong) live in the CTAs'
// shared memory and neighbours read them through distributed shared memory
// (DSMEM); r, w, x, dinv and the row's CSR entries (<= 9) stay in registers
// for the whole solve.  Two cluster barriers per iteration (after p.w and
// after z.z / z.r), each preceded by every CTA storing its block partial into
// a slot of EVERY CTA, so each CTA folds the C partials in rank order and all
// derive identical scalars and exit decisions.  Element arithmetic as
// k_cg_persistent (the reference's mul-then-add order).  Replaces 41 launches
// (or 60 grid barriers) by one launch and 40 cluster barriers.
constexpr int kCRows   = 1024; // rows per CTA = threads per CTA
constexpr int kCMaxCta = 16;
constexpr int kCMaxNnz = 9;

template <bool JACOBI, int NZ> // NZ: longest row (5, 7 or 9), sizes the register arrays
__global__ void __launch_bounds__(kCRows, 1) k_cg_cluster(PersistArgs a)
{
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double zs[kCRows], pb[2][kCRows];
    __shared__ double slot_a[kCMaxCta], slot_b[kCMaxCta][2];
    __shared__ double red[64];
    const int     C    = (int)cl.num_blocks();
    const int     q    = (int)cl.block_rank();
    const int     tid  = threadIdx.x;
    const int64_t i    = (int64_t)q * kCRows + tid;
    const bool    own  = i < a.n;
    const bool    lead = q == 0 && tid == 0;

    // the row's entries: value + generic (DSMEM) address of z[col] in its CTA;
    // p_old / p_new sit at fixed offsets from it (same layout in every CTA)
    const double* zp[NZ];
    double        va[NZ];
    int           cnt = 0;
    if (own) {
        const int64_t kb = a.off[i], ke = a.off[i + 1];
        cnt              = (int)(ke - kb);
#pragma unroll
        for (int k = 0; k < NZ; ++k) {
            if (k < cnt) {
                const int32_t c = a.cols[kb + k];
                va[k]           = a.vals[kb + k];
                zp[k]           = cl.map_shared_rank(&zs[c & (kCRows - 1)], c / kCRows);
            } else {
                va[k] = 0.0;
                zp[k] = &zs[0];
            }
        }
    }
    const ptrdiff_t to_p0 = &pb[0][0] - &zs[0], to_p1 = &pb[1][0] - &zs[0];

    // every CTA of the cluster is running before anyone touches DSMEM
    cl.sync();
    // publish this CTA's block partial(s) into every CTA's slots, then barrier
    auto publish = [&](double* slots, int stride_d, const double* v, int nv) {
        if (tid == 0)
            for (int t = 0; t < C; ++t) {
                double* dst = cl.map_shared_rank(slots, t);
                for (int j = 0; j < nv; ++j) dst[q * stride_d + j] = v[j];
            }
        cl.sync();
    };
    auto fold = [&](const double* slots, int stride_d, int j) {
        double v = 0.0;
        for (int t = 0; t < C; ++t) v = add(v, slots[t * stride_d + j]);
        return v;
    };

    // ---- setup: r = b, x = 0, z = B r; z.z, z.r ------------------------------
    const double d  = (own && JACOBI) ? a.dinv[i] : 1.0;
    double       r  = own ? a.b[i] : 0.0;
    double       z  = JACOBI ? mul(d, r) : r;
    double       x  = 0.0;
    double       pv = 0.0; // this row's current p
    zs[tid]         = z;
    double acc[2]   = {own ? mul(z, z) : 0.0, own ? mul(z, r) : 0.0};
    block_sum<2>(acc, red, tid, kCRows, 1);
    publish(&slot_b[0][0], 2, acc, 2);
    double       beta = fold(&slot_b[0][0], 2, 1);
    const double dp0  = sqrt(fold(&slot_b[0][0], 2, 0));
    int          state = RVK_CG_RUNNING, iters = 0, bk = -1;
    double       alpha = 0.0, pAp = 0.0, betaold = 0.0, dp = dp0;
    if (cg_converged(dp0, dp0, a.rtol, a.atol)) state = RVK_CG_CONVERGED;

    for (int it = 0; it < a.max_it && state == RVK_CG_RUNNING; ++it) {
        // ---- w = A p with p = z + b p_old formed per gathered entry ----------
        double bb = 0.0;
        if (it > 0) {
            if (betaold == 0.0) {
                state = RVK_CG_BREAKDOWN;
                bk    = it;
                break;
            }
            bb = beta / betaold;
        }
        const int       po = it & 1, pn = po ^ 1;
        const ptrdiff_t tp = po ? to_p1 : to_p0;
        double          w  = 0.0;
        if (own) {
            double g[NZ];
#pragma unroll
            for (int k = 0; k < NZ; ++k) {
                if (k < cnt) {
                    const double zj = zp[k][0];
                    g[k]            = it == 0 ? zj : aypx1(bb, zj, zp[k][tp]);
                }
            }
#pragma unroll
            for (int k = 0; k < NZ; ++k)
                if (k < cnt) w = add(w, mul(va[k], g[k]));
            pv          = it == 0 ? zs[tid] : aypx1(bb, zs[tid], pb[po][tid]);
            pb[pn][tid] = pv;
        }
        double v1[1] = {own ? mul(pv, w) : 0.0};
        block_sum<1>(v1, red, tid, kCRows, 1);
        publish(slot_a, 1, v1, 1);
        pAp             = fold(slot_a, 1, 0);
        const double al = beta / pAp;
        if (pAp == 0.0 || !isfinite(al)) {
            state = RVK_CG_BREAKDOWN;
            bk    = it;
            break;
        }
        alpha   = al;
        betaold = beta;
        // ---- x += a p, r += (-a) w, z = B r; z.z, z.r ------------------------
        x        = axpy1(al, pv, x);
        r        = axpy1(-al, w, r);
        z        = JACOBI ? mul(d, r) : r;
        zs[tid]  = z;
        acc[0]   = own ? mul(z, z) : 0.0;
        acc[1]   = own ? mul(z, r) : 0.0;
        block_sum<2>(acc, red, tid, kCRows, 1);
        publish(&slot_b[0][0], 2, acc, 2);
        dp    = sqrt(fold(&slot_b[0][0], 2, 0));
        iters = it + 1;
        if (lead) a.hist[it + 1] = dp;
        if (cg_converged(dp, dp0, a.rtol, a.atol)) state = RVK_CG_CONVERGED;
        beta = fold(&slot_b[0][0], 2, 1);
    }
    if (own) {
        a.x[i] = x;
        a.r[i] = r;
        a.z[i] = z;
    }
    if (lead) {
        a.hist[0]            = dp0;
        a.st->dp0            = dp0;
        a.st->dp             = dp;
        a.st->alpha          = alpha;
        a.st->pAp            = pAp;
        a.st->beta           = beta;
        a.st->betaold        = betaold;
        a.st->iterations     = iters;
        a.st->breakdown_iter = bk;
        a.st->state          = state;
        a.st->done           = 1;
    }
    cl.sync(); // no CTA leaves while a neighbour may still address its shared memory
}


// ---------------------------------------------------------------------------
// Grid solve for mid-size L2-resident grids (16 K < n <= ~450 K rows): the
// whole solve in ONE cooperative launch of <= 148 CTAs x 1024 threads, R
// rows per thread.  Each CTA keeps its rows' CSR in shared memory (ELL
// layout, loaded once), and x, r, z, p and the Jacobi diagonal of its rows in
// registers for the whole solve; only the gathered operands z and p travel
// through global memory (L2).  Two grid barriers per iteration, each fused
// with its reduction: a CTA stores its block partial, releases a monotonic
// arrival counter and spins on it; then EVERY CTA folds the G partials in
// the same fixed order (lane l sums blocks l, l+32, ... ascending, then a
// shuffle tree), so all CTAs derive bit-identical scalars and exit together.
// Element arithmetic is the reference's (mul-then-add, same operand order),
// p is formed per gathered entry as in the fused K1.  Replaces the 41
// launches of the fused graph, whose ~5 us per launch floor bounds 256^2 -
// 512^2 solves.
#ifndef RVK_GRID_THREADS
#define RVK_GRID_THREADS 512 // measured: 256^2 0.128 (1024 threads) -> 0.115 ms
#endif
constexpr int kGThreads = RVK_GRID_THREADS;
constexpr int kGMaxR    = 3 * 1024 / kGThreads; // rows per thread (capacity 148 x 3072 rows)
constexpr int kGMaxCta  = 148;
constexpr int kG2MaxRpc = 8192; // k_cg_grid_l2: x, r, p in shared memory (8 K rows: 200 KB)

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Block-sum v, publish, grid barrier #`index`, fold every CTA's partials.
template <int NV>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], double* partials, unsigned* bar,
                                            unsigned target, double* red, double* out_sh)
{
    const int tid = threadIdx.x;
    block_sum<NV>(v, red, tid, kGThreads, 1);
    if (tid == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) partials[blockIdx.x * 4 + j] = v[j];
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_u32(bar) < target) {
        }
    }
    __syncthreads();
    if (tid < 32) {
        // every lane issues all its loads (<= 5 blocks x NV) before the first
        // add: one L2 round trip instead of one per block; the adds keep the
        // ascending block order
        constexpr int kPer = (kGMaxCta + 31) / 32;
        double        pv[kPer][NV];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int blk = tid + 32 * q;
#pragma unroll
            for (int j = 0; j < NV; ++j)
                pv[q][j] = blk < (int)gridDim.x ? __ldcg(partials + blk * 4 + j) : 0.0;
        }
        double f[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) f[j] = 0.0;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            if (tid + 32 * q < (int)gridDim.x) {
#pragma unroll
                for (int j = 0; j < NV; ++j) f[j] = add(f[j], pv[q][j]);
            }
        }
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            f[j] = warp_sum(f[j]);
            if (tid == 0) out_sh[j] = f[j];
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = out_sh[j];
    __syncthreads(); // out_sh reusable
}

// No JACOBI template parameter: a plan without a preconditioner stores
// dinv = 1.0 and z = 1.0 * r is r exactly.
template <int NZ, int R>
__global__ void __launch_bounds__(kGThreads, 1)
    k_cg_grid(PersistArgs a, unsigned* bar, int rpc)
{
    extern __shared__ __align__(16) unsigned char gsm[];
    double*  ev   = reinterpret_cast<double*>(gsm);                   // [rpc][NZ] values
    int32_t* ec   = reinterpret_cast<int32_t*>(ev + (size_t)rpc * NZ); // [rpc][NZ] columns
    uint8_t* ecnt = reinterpret_cast<uint8_t*>(ec + (size_t)rpc * NZ); // [rpc] row lengths
    __shared__ double red[128], out_sh[4];
    const int     tid  = threadIdx.x;
    const bool    lead = blockIdx.x == 0 && tid == 0;
    const int64_t r0   = (int64_t)blockIdx.x * rpc;
    unsigned      nbar = 0; // barriers passed
    const unsigned G   = gridDim.x;

    // this CTA's rows into shared memory (ELL, row order kept)
    for (int j = tid; j < rpc; j += kGThreads) {
        const int64_t i = r0 + j;
        int           c = 0;
        if (i < a.n) {
            const int64_t kb = a.off[i], ke = a.off[i + 1];
            c                = (int)(ke - kb);
            for (int k = 0; k < c; ++k) {
                ev[(size_t)j * NZ + k] = a.vals[kb + k];
                ec[(size_t)j * NZ + k] = a.cols[kb + k];
            }
        }
        ecnt[j] = (uint8_t)c;
    }

    // ---- setup: r = b, x = 0, z = B r; z.z, z.r ------------------------------
    double x[R], r[R], z[R], pv[R], d[R];
    bool   own[R];
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int     j = tid + m * kGThreads;
        const int64_t i = r0 + j;
        own[m]          = j < rpc && i < a.n;
        d[m]            = own[m] ? a.dinv[i] : 1.0;
        r[m]            = own[m] ? a.b[i] : 0.0;
        z[m]            = mul(d[m], r[m]);
        x[m]            = 0.0;
        pv[m]           = 0.0;
        if (own[m]) {
            a.z[i] = z[m];
            acc[0] = add(acc[0], mul(z[m], z[m]));
            acc[1] = add(acc[1], mul(z[m], r[m]));
        }
    }
    grid_reduce<2>(acc, a.partials, bar, ++nbar * G, red, out_sh); // (also publishes the smem CSR)
    double       beta = acc[1];
    const double dp0  = sqrt(acc[0]);
    int          state = RVK_CG_RUNNING, iters = 0, bk = -1;
    double       alpha = 0.0, pAp = 0.0, betaold = 0.0, dp = dp0;
    if (cg_converged(dp0, dp0, a.rtol, a.atol)) state = RVK_CG_CONVERGED;

    for (int it = 0; it < a.max_it && state == RVK_CG_RUNNING; ++it) {
        // ---- w = A p, p = z + b p_old formed per gathered entry ---------------
        double bb = 0.0;
        if (it > 0) {
            if (betaold == 0.0) {
                state = RVK_CG_BREAKDOWN;
                bk    = it;
                break;
            }
            bb = beta / betaold;
        }
        const double* po = (it & 1) ? a.p1 : a.p0;
        double*       pn = (it & 1) ? a.p0 : a.p1;
        double        w[R];
        double        pw = 0.0;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            w[m] = 0.0;
            if (!own[m]) continue;
            const int j   = tid + m * kGThreads;
            const int cnt = ecnt[j];
            double    zj[NZ], pj[NZ];
#pragma unroll
            for (int k = 0; k < NZ; ++k) {
                const int32_t c = k < cnt ? ec[(size_t)j * NZ + k] : 0;
                zj[k]           = __ldcg(a.z + c);
                pj[k]           = it == 0 ? 0.0 : __ldcg(po + c);
            }
#pragma unroll
            for (int k = 0; k < NZ; ++k)
                if (k < cnt)
                    w[m] = add(w[m], mul(ev[(size_t)j * NZ + k], it == 0 ? zj[k] : aypx1(bb, zj[k], pj[k])));
            pv[m] = it == 0 ? z[m] : aypx1(bb, z[m], pv[m]);
            pn[r0 + j] = pv[m];
            pw = add(pw, mul(pv[m], w[m]));
        }
        double v1[1] = {pw};
        grid_reduce<1>(v1, a.partials, bar, ++nbar * G, red, out_sh);
        pAp             = v1[0];
        const double al = beta / pAp;
        if (pAp == 0.0 || !isfinite(al)) {
            state = RVK_CG_BREAKDOWN;
            bk    = it;
            break;
        }
        alpha   = al;
        betaold = beta;
        // ---- x += a p, r += (-a) w, z = B r; z.z, z.r ------------------------
        acc[0] = acc[1] = 0.0;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            if (!own[m]) continue;
            x[m] = axpy1(al, pv[m], x[m]);
            r[m] = axpy1(-al, w[m], r[m]);
            z[m] = mul(d[m], r[m]);
            a.z[r0 + tid + m * kGThreads] = z[m];
            acc[0] = add(acc[0], mul(z[m], z[m]));
            acc[1] = add(acc[1], mul(z[m], r[m]));
        }
        grid_reduce<2>(acc, a.partials, bar, ++nbar * G, red, out_sh);
        dp    = sqrt(acc[0]);
        iters = it + 1;
        if (lead) a.hist[it + 1] = dp;
        if (cg_converged(dp, dp0, a.rtol, a.atol)) state = RVK_CG_CONVERGED;
        beta = acc[1];
    }
#pragma unroll
    for (int m = 0; m < R; ++m)
        if (own[m]) {
            const int64_t i = r0 + tid + m * kGThreads;
            a.x[i]          = x[m];
            a.r[i]          = r[m];
        }
    if (lead) {
        a.hist[0]            = dp0;
        a.st->dp0            = dp0;
        a.st->dp             = dp;
        a.st->alpha          = alpha;
        a.st->pAp            = pAp;
        a.st->beta           = beta;
        a.st->betaold        = betaold;
        a.st->iterations     = iters;
        a.st->breakdown_iter = bk;
        a.st->state          = state;
        a.st->done           = 1;
    }
}

// Plan-time ELL copy for the L2 grid solve: k-major (entry k of row i at
// k * n + i, so a warp's 32 rows read 32 consecutive words per k), row
// lengths in bytes.  Entries past a row's length are never read.
__global__ void k_ell_build(int64_t n, const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                            const double* __restrict__ vals, int nz, double* ev, int32_t* ec, uint8_t* en)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kb = off[i];
        const int     c  = (int)(off[i + 1] - kb);
        for (int k = 0; k < c; ++k) {
            ev[k * n + i] = vals[kb + k];
            ec[k * n + i] = cols[kb + k];
        }
        en[i] = (uint8_t)c;
    }
}

// The grid solve past the shared-memory ELL's reach (3 K .. 8 K rows per CTA:
// 1024^2 5-point = 7104).  The matrix comes from the plan's k-major ELL copy
// in global memory (63 MB at 1024^2 5-point: with z and the two p's, 88 MB,
// L2-resident across iterations); x, r and p of the CTA's rows live in
// shared memory, w in registers (R rows per thread).  Same barriers, same
// fold order and element arithmetic as k_cg_grid; the own row's z is formed
// from r (z = d r, the value K2 stores) instead of being kept.
template <int NZ, int R>
__global__ void __launch_bounds__(kGThreads, 1)
    k_cg_grid_l2(PersistArgs a, unsigned* bar, int rpc, const double* __restrict__ ev,
                 const int32_t* __restrict__ ec, const uint8_t* __restrict__ en)
{
    extern __shared__ __align__(16) unsigned char gsm[];
    double*  xs  = reinterpret_cast<double*>(gsm);
    double*  rs  = xs + rpc;
    double*  ps  = rs + rpc;
    uint8_t* cs  = reinterpret_cast<uint8_t*>(ps + rpc);
    __shared__ double red[128], out_sh[4];
    const int      tid  = threadIdx.x;
    const bool     lead = blockIdx.x == 0 && tid == 0;
    const int64_t  n    = a.n;
    const int64_t  r0   = (int64_t)blockIdx.x * rpc;
    const int      nown = (int)(n - r0 < rpc ? n - r0 : rpc); // rows of this CTA
    unsigned       nbar = 0;
    const unsigned G    = gridDim.x;

    // ---- setup: r = b, x = 0, z = B r; z.z, z.r ------------------------------
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int j = tid + m * kGThreads;
        if (j >= nown) continue;
        const int64_t i  = r0 + j;
        const double  ri = a.b[i];
        const double  zi = mul(a.dinv[i], ri);
        xs[j] = 0.0;
        rs[j] = ri;
        ps[j] = 0.0;
        cs[j] = en[i];
        a.z[i] = zi;
        acc[0] = add(acc[0], mul(zi, zi));
        acc[1] = add(acc[1], mul(zi, ri));
    }
    grid_reduce<2>(acc, a.partials, bar, ++nbar * G, red, out_sh);
    double       beta = acc[1];
    const double dp0  = sqrt(acc[0]);
    int          state = RVK_CG_RUNNING, iters = 0, bk = -1;
    double       alpha = 0.0, pAp = 0.0, betaold = 0.0, dp = dp0;
    if (cg_converged(dp0, dp0, a.rtol, a.atol)) state = RVK_CG_CONVERGED;

    for (int it = 0; it < a.max_it && state == RVK_CG_RUNNING; ++it) {
        double bb = 0.0;
        if (it > 0) {
            if (betaold == 0.0) {
                state = RVK_CG_BREAKDOWN;
                bk    = it;
                break;
            }
            bb = beta / betaold;
        }
        const double* po = (it & 1) ? a.p1 : a.p0;
        double*       pn = (it & 1) ? a.p0 : a.p1;
        double w[R];
        double pw = 0.0;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            w[m]        = 0.0;
            const int j = tid + m * kGThreads;
            if (j >= nown) continue;
            const int64_t i   = r0 + j;
            const int     cnt = cs[j];
            int32_t       c[NZ];
            double        v[NZ], zj[NZ], pj[NZ];
#pragma unroll
            for (int k = 0; k < NZ; ++k) {
                c[k] = k < cnt ? __ldg(ec + k * n + i) : 0;
                v[k] = k < cnt ? __ldg(ev + k * n + i) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < NZ; ++k) {
                zj[k] = __ldcg(a.z + c[k]);
                pj[k] = it == 0 ? 0.0 : __ldcg(po + c[k]);
            }
#pragma unroll
            for (int k = 0; k < NZ; ++k)
                if (k < cnt) w[m] = add(w[m], mul(v[k], it == 0 ? zj[k] : aypx1(bb, zj[k], pj[k])));
            const double zi = mul(__ldg(a.dinv + i), rs[j]);
            const double pv = it == 0 ? zi : aypx1(bb, zi, ps[j]);
            ps[j] = pv;
            pn[i] = pv;
            pw    = add(pw, mul(pv, w[m]));
        }
        double v1[1] = {pw};
        grid_reduce<1>(v1, a.partials, bar, ++nbar * G, red, out_sh);
        pAp             = v1[0];
        const double al = beta / pAp;
        if (pAp == 0.0 || !isfinite(al)) {
            state = RVK_CG_BREAKDOWN;
            bk    = it;
            break;
        }
        alpha   = al;
        betaold = beta;
        // ---- x += a p, r += (-a) w, z = B r; z.z, z.r ------------------------
        acc[0] = acc[1] = 0.0;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int j = tid + m * kGThreads;
            if (j >= nown) continue;
            const int64_t i  = r0 + j;
            xs[j]            = axpy1(al, ps[j], xs[j]);
            const double ri  = axpy1(-al, w[m], rs[j]);
            const double zi  = mul(__ldg(a.dinv + i), ri);
            rs[j]            = ri;
            a.z[i]           = zi;
            acc[0]           = add(acc[0], mul(zi, zi));
            acc[1]           = add(acc[1], mul(zi, ri));
        }
        grid_reduce<2>(acc, a.partials, bar, ++nbar * G, red, out_sh);
        dp    = sqrt(acc[0]);
        iters = it + 1;
        if (lead) a.hist[it + 1] = dp;
        if (cg_converged(dp, dp0, a.rtol, a.atol)) state = RVK_CG_CONVERGED;
        beta = acc[1];
    }
    for (int j = tid; j < nown; j += kGThreads) {
        a.x[r0 + j] = xs[j];
        a.r[r0 + j] = rs[j];
    }
    if (lead) {
        a.hist[0]            = dp0;
        a.st->dp0            = dp0;
        a.st->dp             = dp;
        a.st->alpha          = alpha;
        a.st->pAp            = pAp;
        a.st->beta           = beta;
        a.st->betaold        = betaold;
        a.st->iterations     = iters;
        a.st->breakdown_iter = bk;
        a.st->state          = state;
        a.st->done           = 1;
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

// Cluster size for the DSMEM solve, 0 when the system does not qualify
// (n > 16 x 1024 rows, rows longer than kCMaxNnz, or no co-resident cluster).
int cluster_ctas(int64_t n, int64_t max_row_len)
{
    if (n < 1 || max_row_len > kCMaxNnz || n > (int64_t)kCMaxCta * kCRows) return 0;
    const int C = (int)((n + kCRows - 1) / kCRows);
    for (auto fn : {k_cg_cluster<true, 5>, k_cg_cluster<false, 5>, k_cg_cluster<true, 7>,
                    k_cg_cluster<false, 7>, k_cg_cluster<true, 9>, k_cg_cluster<false, 9>})
        if (C > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id               = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim            = dim3(C);
    cfg.blockDim           = dim3(kCRows);
    cfg.attrs              = at;
    cfg.numAttrs           = 1;
    int nc                 = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k_cg_cluster<true, 9>, &cfg) != cudaSuccess || nc < 1) {
        cudaGetLastError();
        return 0;
    }
    return C;
}

rvk_status launch_cluster(cudaStream_t s, const PersistArgs& args, bool jacobi, int C, int nz)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id               = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim            = dim3(C);
    cfg.blockDim           = dim3(kCRows);
    cfg.stream             = s;
    cfg.attrs              = at;
    cfg.numAttrs           = 1;
    auto go = [&](auto fn) { return cudaLaunchKernelEx(&cfg, fn, args); };
    if (nz <= 5) RVK_CUDA(jacobi ? go(k_cg_cluster<true, 5>) : go(k_cg_cluster<false, 5>));
    else if (nz <= 7) RVK_CUDA(jacobi ? go(k_cg_cluster<true, 7>) : go(k_cg_cluster<false, 7>));
    else RVK_CUDA(jacobi ? go(k_cg_cluster<true, 9>) : go(k_cg_cluster<false, 9>));
    return RVK_OK;
}

rvk_status launch_persistent(cudaStream_t s, const PersistArgs& args, bool jacobi, int grid)
{
    void* kargs[] = {const_cast<PersistArgs*>(&args)};
    const void* fn = jacobi ? (const void*)k_cg_persistent<true> : (const void*)k_cg_persistent<false>;
    RVK_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kPThreads), kargs, 0, s));
    return RVK_OK;
}

} // namespace rvk

namespace rvk {

// Grid-solve geometry: rows per CTA (32-aligned) and CTAs, or 0 when the
// system does not qualify (rows > 9 entries or more than 148 x 8 K rows).
// *l2 = 1: the rows' ELL does not fit the shared memory (more than 3 K rows
// per CTA, or the ELL bytes), so the solve reads the plan's global ELL copy
// (k_cg_grid_l2, x / r / p in shared memory).
int grid_solve_rows(int64_t n, int64_t max_row_len, int* ctas, int* l2)
{
    if (n < 1 || max_row_len > kCMaxNnz) return 0;
    const int     nz  = max_row_len <= 5 ? 5 : (max_row_len <= 7 ? 7 : 9);
    const int64_t rpc = ((n + kGMaxCta - 1) / kGMaxCta + 31) / 32 * 32;
    if (rpc > kG2MaxRpc) return 0;
    const size_t smem = (size_t)rpc * nz * 12 + rpc;
    *l2               = (rpc > (int64_t)kGMaxR * kGThreads || smem > 220 * 1024) ? 1 : 0;
    *ctas             = (int)((n + rpc - 1) / rpc);
    return (int)rpc;
}

rvk_status build_grid_ell(cudaStream_t s, int64_t n, const int64_t* off, const int32_t* cols,
                          const double* vals, int max_row_len, double* ev, int32_t* ec, uint8_t* en)
{
    const int nz = max_row_len <= 5 ? 5 : (max_row_len <= 7 ? 7 : 9);
    k_ell_build<<<(int)std::min<int64_t>((n + 255) / 256, 4 * 148 * 8), 256, 0, s>>>(n, off, cols, vals, nz, ev,
                                                                                     ec, en);
    RVK_CHECK_LAUNCH("k_ell_build");
    return RVK_OK;
}

rvk_status launch_grid_solve(cudaStream_t s, const PersistArgs& args, unsigned* bar, bool jacobi,
                             int rpc, int ctas, int max_row_len, const GridEll* ell)
{
    (void)jacobi; // the plan's dinv is 1.0 without a preconditioner
    const int    nz   = max_row_len <= 5 ? 5 : (max_row_len <= 7 ? 7 : 9);
    const int    R    = (rpc + kGThreads - 1) / kGThreads;
    RVK_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), s));
    if (ell) {
        const size_t smem    = (size_t)rpc * 24 + rpc;
        void*        kargs[] = {const_cast<PersistArgs*>(&args), &bar, &rpc, const_cast<double**>(&ell->v),
                                const_cast<int32_t**>(&ell->c), const_cast<uint8_t**>(&ell->n)};
        auto go = [&](auto fn) -> rvk_status {
            RVK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            RVK_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3(ctas), dim3(kGThreads), kargs, smem, s));
            return RVK_OK;
        };
        const int Ri = R <= 8 ? 8 : (R <= 12 ? 12 : 16);
#define RVK_GRID2_CASE(NZ, RR)                                                        \
        if (nz == NZ && Ri == RR) return go(k_cg_grid_l2<NZ, RR>);
        RVK_GRID2_CASE(5, 8) RVK_GRID2_CASE(5, 12) RVK_GRID2_CASE(5, 16)
        RVK_GRID2_CASE(7, 8) RVK_GRID2_CASE(7, 12) RVK_GRID2_CASE(7, 16)
        RVK_GRID2_CASE(9, 8) RVK_GRID2_CASE(9, 12) RVK_GRID2_CASE(9, 16)
#undef RVK_GRID2_CASE
        return set_error(RVK_ERR_INVALID, "grid solve (L2): unsupported geometry (R %d, nz %d)", R, nz);
    }
    const size_t smem = (size_t)rpc * nz * 12 + rpc;
    void* kargs[] = {const_cast<PersistArgs*>(&args), &bar, &rpc};
    auto go = [&](auto fn) -> rvk_status {
        // > 48 KB dynamic shared memory: per device and instantiation (idempotent)
        RVK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        RVK_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3(ctas), dim3(kGThreads), kargs, smem, s));
        return RVK_OK;
    };
#define RVK_GRID_CASE(NZ, RR)                                                      \
    if (nz == NZ && R == RR) return go(k_cg_grid<NZ, RR>);
#define RVK_GRID_NZ(NZ) RVK_GRID_CASE(NZ, 1) RVK_GRID_CASE(NZ, 2) RVK_GRID_CASE(NZ, 3) \
    if constexpr (kGMaxR > 3) { RVK_GRID_CASE(NZ, 4) RVK_GRID_CASE(NZ, 5) RVK_GRID_CASE(NZ, 6) }
    RVK_GRID_NZ(5) RVK_GRID_NZ(7) RVK_GRID_NZ(9)
#undef RVK_GRID_NZ
#undef RVK_GRID_CASE
    return set_error(RVK_ERR_INVALID, "grid solve: unsupported geometry (R %d, nz %d)", R, nz);
}

} // namespace rvk
