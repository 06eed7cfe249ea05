// rvk_cg.cu -- Jacobi-preconditioned CG on sm_100a with zero host syncs per
// iteration.
//
// Reference path: cg_solve running the PETSc
// KSPCG loop of PAPER.md:104-150:
//   setup:  r = b, z = B r, dp = ||z|| -> hist[0], beta = z.r
//   iter i: b = beta/betaold (i>=1); p = z + b p (i==0: p = z); w = A p
//           a = beta/(p.w); betaold = beta; x += a p; r += (-a) w; z = B r
//           dp = ||z|| -> hist[i+1]; converged?; beta = z.r
//
// FUSED mode (default) -- per iteration two kernels, all scalars on device:
//   K1 = k_spmv_tma<CgSpmvOp>: p_new = z + b p_old evaluated on the fly for
//        every gathered column (b = beta/betaold read from device memory),
//        w = A p_new, p.w partials; last block: alpha = beta/pAp, breakdown
//        check, betaold = beta.  p ping-pongs between two buffers because
//        neighbouring tiles still gather p_old while p_new is written.
//   K2 = k_cg_update: x += a p; r += (-a) w; z = dinv .* r; z.z and z.r
//        partials; last block: dp = sqrt(z.z) -> hist, convergence, beta.
//   K0 = k_cg_setup once per solve (r = b, x = 0, z = B r, dp0, beta).
// Every per-element result uses the reference's rounding sequence, so p, w,
// x, r, z differ from the CPU oracle only through the reduction order of the
// three scalars (tolerance 1e-10, BASELINE.json north_star).
//
// UNFUSED mode issues the reference's one-kernel-per-op sequence
// through the same Vec/SpMV kernels with device-scalar arguments; it exists
// for the fusion A/B and as the literal drop-in for the listing.
//
// Early exit (converged / breakdown) is decided on device: the tails set a
// `done` flag and every later kernel of the solve returns immediately, so
// the whole solve is one CUDA graph replayed with no host involvement.
#include "rvk_common.cuh"
#include "rvk_context.hpp"
#include "rvk_spmv_march.cuh"
#include "rvk_internal.hpp"
#include "rvk_cg.cuh"
#include "rvk_spmv.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace rvk {

// K1 of iteration 0 with the setup folded in (fold_setup: FUSED CSR plans
// on the unrolled graph / stream path, 16-B aligned b; any Jacobi diagonal --
// constant (d) or a per-row vector gathered beside b (VECD) -- and any x
// group: without the whole-solve group the caller zeroes x with a memset):
// z_j = d b_j formed per gathered column, p = z, w = A p; the row owner
// writes p, w and r = b; sums p.w, z.z and z.b; the tail does the setup's
// scalars (hist[0], dp0, beta, the convergence test) and then K1's (alpha).
// A one-thread reset (k_cg_reset) runs before it.  Element values are the
// setup's and K1's (z = d b, p = z); only the reduction order of z.z / z.b
// differs (another fixed tree), so hist[0] and beta_0 may differ in the last
// ulp from the WHILE-graph / unfused / persistent paths of the same plan.
template <bool VECD> // VECD: per-row Jacobi diagonal (gathered beside b)
struct CgFirstBOp {
    static constexpr bool kHasTail = true;
    static constexpr int  kSums    = 3;
    const double* __restrict__ b;
    const double* __restrict__ dinv;
    double* __restrict__ p_new;
    double* __restrict__ w;
    double* __restrict__ r;
    CgState* st;
    double*  hist;
    double   d; // the constant diagonal (1.0 without a preconditioner: 1 * b == b exactly)
    double   rtol, atol;

    __device__ __forceinline__ bool init() { return true; }
    struct Fetch {
        double b, dv;
    };
    __device__ __forceinline__ int           num_src() const { return VECD ? 2 : 1; }
    __device__ __forceinline__ const double* src_ptr(int k) const { return k == 0 ? b : dinv; }
    __device__ __forceinline__ Fetch         fetch(int32_t j) const
    {
        return Fetch{__ldg(b + j), VECD ? __ldg(dinv + j) : 0.0};
    }
    __device__ __forceinline__ double  value(const Fetch& f) const { return mul(VECD ? f.dv : d, f.b); }
    __device__ __forceinline__ int64_t own_col(int64_t i) const { return i; }
    __device__ __forceinline__ SumVec<3> row(int64_t i, double sum, SumVec<3> acc, const Fetch& o) const
    {
        const double z = value(o);
        p_new[i]       = z;
        w[i]           = sum;
        r[i]           = o.b;
        acc.v[0]       = add(acc.v[0], mul(z, sum));
        acc.v[1]       = add(acc.v[1], mul(z, z));
        acc.v[2]       = add(acc.v[2], mul(z, o.b));
        return acc;
    }
    __device__ __forceinline__ void tail(const double (&v)[3]) const
    {
        const double dp0 = sqrt(v[1]);
        hist[0]          = dp0;
        st->dp0          = dp0;
        st->dp           = dp0;
        st->beta         = v[2];
        if (cg_converged(dp0, dp0, rtol, atol)) {
            st->state = RVK_CG_CONVERGED;
            st->done  = 1;
            return;
        }
        const double pAp = v[0];
        const double a   = st->beta / pAp;
        st->pAp          = pAp;
        if (pAp == 0.0 || !isfinite(a)) {
            st->state          = RVK_CG_BREAKDOWN;
            st->breakdown_iter = 0;
            st->done           = 1;
        } else {
            st->alpha   = a;
            st->betaold = st->beta;
        }
    }
};

// CgState, kUpdThreads, cg_converged, resident_grid: rvk_cg.cuh

// State reset of a solve whose setup is folded into K1(0) (CgFirstBOp).
__global__ void k_cg_reset(CgState* st)
{
    st->x_pending      = 0;
    st->betaold        = 0.0;
    st->alpha          = 0.0;
    st->pAp            = 0.0;
    st->iterations     = 0;
    st->breakdown_iter = -1;
    st->state          = RVK_CG_RUNNING;
    st->done           = 0;
}

// ---------------------------------------------------------------------------
// K0: setup.  r = b; x = 0; z = B r; partials z.z, z.r.
// ---------------------------------------------------------------------------
template <bool VEC, int PC> // PC: 0 none, 1 dinv vector, 2 constant dinv (matrix-free stencil)
__global__ void __launch_bounds__(kUpdThreads)
    k_cg_setup(int64_t n, const double* __restrict__ b, const double* __restrict__ dinv,
               double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
               CgState* st, double* hist, double rtol, double atol, double* partials,
               unsigned int* ticket, double dconst, int zw, int xw)
{
    __shared__ double smem[64];
    __shared__ int    flag;
    double            acc[2] = {0.0, 0.0};
    const int64_t     stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t     t0     = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (VEC) {
        const int64_t n2 = n >> 1;
        for (int64_t i = t0; i < n2; i += stride) {
            const double2 bi = ld_stream(reinterpret_cast<const double2*>(b) + i);
            double2       zi = bi;
            if (PC != 0) {
                const double2 d = PC == 1 ? ld_stream(reinterpret_cast<const double2*>(dinv) + i)
                                          : make_double2(dconst, dconst);
                zi.x = mul(d.x, bi.x);
                zi.y = mul(d.y, bi.y);
            }
            reinterpret_cast<double2*>(r)[i] = bi;
            if (zw) reinterpret_cast<double2*>(z)[i] = zi; // zw = 0: z stays virtual (d r)
            if (xw) st_stream(reinterpret_cast<double2*>(x) + i, make_double2(0.0, 0.0));
            acc[0] = add(acc[0], mul(zi.x, zi.x));
            acc[0] = add(acc[0], mul(zi.y, zi.y));
            acc[1] = add(acc[1], mul(zi.x, bi.x));
            acc[1] = add(acc[1], mul(zi.y, bi.y));
        }
    }
    for (int64_t i = (VEC ? (n & ~int64_t(1)) : 0) + t0; i < n; i += stride) {
        const double bi = b[i];
        const double zi = PC == 0 ? bi : mul(PC == 1 ? dinv[i] : dconst, bi);
        r[i] = bi;
        if (zw) z[i] = zi;
        if (xw) x[i] = 0.0; // xw = 0: the whole-solve x pass starts from 0.0 itself
        acc[0] = add(acc[0], mul(zi, zi));
        acc[1] = add(acc[1], mul(zi, bi));
    }
    const int tid = threadIdx.x;
    block_sum<2>(acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        partials[2 * blockIdx.x]     = acc[0];
        partials[2 * blockIdx.x + 1] = acc[1];
    }
    if (!last_block(ticket, tid, &flag, blockDim.x, 1)) return;
    fold_partials<2>(partials, gridDim.x, acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        const double dp0 = sqrt(acc[0]);
        hist[0]            = dp0;
        st->dp0            = dp0;
        st->dp             = dp0;
        st->beta           = acc[1];
        st->x_pending      = 0;
        st->betaold        = 0.0;
        st->alpha          = 0.0;
        st->pAp            = 0.0;
        st->iterations     = 0;
        st->breakdown_iter = -1;
        const bool conv    = cg_converged(dp0, dp0, rtol, atol);
        st->state          = conv ? RVK_CG_CONVERGED : RVK_CG_RUNNING;
        st->done           = conv ? 1 : 0;
        *ticket            = 0u;
    }
}


// ---------------------------------------------------------------------------
// K2: x += a p; r += (-a) w; z = B r; partials z.z, z.r; tail dp/hist/beta.
// ---------------------------------------------------------------------------
// Shared K2 tail: block sums -> last block -> dp into hist, convergence,
// beta = z.r, the WHILE condition.  Call from all threads of the block.
template <bool COND>
__device__ __forceinline__ void cg_update_tail(double (&acc)[2], double* smem, int* flag, CgState* st,
                                               double* hist, int it, double rtol, double atol,
                                               double* partials, unsigned int* ticket, int max_it,
                                               cudaGraphConditionalHandle cond, int use_cond)
{
    const int tid = threadIdx.x;
    block_sum<2>(acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        partials[2 * blockIdx.x]     = acc[0];
        partials[2 * blockIdx.x + 1] = acc[1];
    }
    if (!last_block(ticket, tid, flag, blockDim.x, 1)) return;
    fold_partials<2>(partials, gridDim.x, acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        const double dp = sqrt(acc[0]);
        hist[it + 1]    = dp;
        st->dp          = dp;
        st->iterations  = it + 1;
        bool more = it + 1 < max_it;
        if (cg_converged(dp, st->dp0, rtol, atol)) {
            st->state = RVK_CG_CONVERGED;
            st->done  = 1;
            more      = false;
        } else {
            st->beta = acc[1];
            if (!more) st->done = 1; // ran max_it: later kernels of a WHILE body no-op
        }
        if constexpr (COND) {
            if (use_cond) cudaGraphSetConditional(cond, more ? 1u : 0u);
        }
        *ticket = 0u;
    }
}

// COND: this instantiation may set the WHILE node's condition.  Kept a
// template parameter so the plain-graph/stream variant contains no
// cudaGraphSetConditional (ncu refuses to profile kernels that can set one).
// x update per GROUP of Q iterations (plan: Q = 1, 2 or 4).  NP < 0: DEFER
// -- x untouched, this iteration's a recorded in pend_a[slot]; NP >= 0:
// x = (((x + a_0 p_0) + a_1 p_1) + ...) + a p with the NP pending updates
// first -- the same roundings in the same order as one update per iteration,
// so x is bit-identical while per group of Q iterations Q-1 x read/writes
// and the p re-reads of the plain update disappear.  The pending p's are the
// plan's rotating p buffers (still intact: iteration j writes p[(j+1) % Q]).
// k_cg_xfix applies updates an early exit left pending.
template <bool VEC, int PC, bool COND = false, int NP = 0> // PC: 0 none, 1 dinv vector, 2 constant dinv
__global__ void __launch_bounds__(kUpdThreads)
    k_cg_update(int64_t n, const double* __restrict__ p, const double* __restrict__ w,
                const double* __restrict__ dinv, double* __restrict__ x, double* __restrict__ r,
                double* __restrict__ z, CgState* st, double* hist, int it, double rtol,
                double atol, double* partials, unsigned int* ticket, double dconst, int max_it,
                cudaGraphConditionalHandle cond, int use_cond, const double* __restrict__ pp0,
                const double* __restrict__ pp1, const double* __restrict__ pp2, int slot, int zw)
{
    static_assert(VEC || NP == 0, "grouped x updates use the vector path");
    static_assert(NP >= -1 && NP <= 3, "at most 3 pending updates");
    // In the device WHILE loop (use_cond) `it` comes from the device state and
    // this kernel decides whether the loop body runs again.
    if (st->done) {
        if constexpr (COND)
            if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
        return;
    }
    if (it < 0) it = st->iterations;
    __shared__ double smem[64];
    __shared__ int    flag;
    const double      a      = st->alpha;
    const double      na     = -a;
    double            pa[3]  = {0.0, 0.0, 0.0}; // pending a's, iteration order
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (k < NP) pa[k] = st->pend_a[k];
    double            acc[2] = {0.0, 0.0};
    const int64_t     stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t     t0     = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // pend_a[slot] is written only by a DEFER launch, read only by later
        // flushes: no kernel both reads and writes the same slot
        if (NP < 0) {
            st->pend_a[slot] = a;
            st->x_pending    = slot + 1;
            if (slot == 0) st->pend_it = it;
        } else if (NP > 0) {
            st->x_pending = 0;
        }
    }
    if (VEC) {
        // two double2 per thread per trip, every load issued before any use
        const int64_t  n2 = n >> 1;
        const double2* p2 = reinterpret_cast<const double2*>(p);
        const double2* q2[3] = {reinterpret_cast<const double2*>(pp0), reinterpret_cast<const double2*>(pp1),
                                reinterpret_cast<const double2*>(pp2)};
        const double2* w2 = reinterpret_cast<const double2*>(w);
        const double2* d2 = reinterpret_cast<const double2*>(dinv);
        double2*       x2 = reinterpret_cast<double2*>(x);
        double2*       r2 = reinterpret_cast<double2*>(r);
        double2*       z2 = reinterpret_cast<double2*>(z);
        struct In {
            double2 p, q[3], w, x, r, d;
        };
        auto load = [&](int64_t i) {
            In v;
            if (NP >= 0) {
                v.p = ld_stream(p2 + i);
                v.x = ld_stream(x2 + i);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (k < NP) v.q[k] = ld_stream(q2[k] + i);
            v.w = ld_stream(w2 + i);
            v.r = ld_stream(r2 + i);
            v.d = PC == 1 ? ld_stream(d2 + i) : make_double2(dconst, dconst);
            return v;
        };
        auto step = [&](In v, int64_t i) {
            if (NP >= 0) {
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    if (k < NP) {
                        v.x.x = axpy1(pa[k], v.q[k].x, v.x.x);
                        v.x.y = axpy1(pa[k], v.q[k].y, v.x.y);
                    }
                v.x.x = axpy1(a, v.p.x, v.x.x);
                v.x.y = axpy1(a, v.p.y, v.x.y);
                st_stream(x2 + i, v.x);
            }
            double2 ri = v.r;
            ri.x       = axpy1(na, v.w.x, ri.x);
            ri.y       = axpy1(na, v.w.y, ri.y);
            double2 zi = ri;
            if (PC != 0) {
                zi.x = mul(v.d.x, ri.x);
                zi.y = mul(v.d.y, ri.y);
            }
            if (!(zw & 2)) r2[i] = ri;
            if (zw & 1) z2[i] = zi; // bit 0 clear: z stays virtual (K1 forms d r); bit 1: last K2, r and z dead
            acc[0] = add(acc[0], mul(zi.x, zi.x));
            acc[0] = add(acc[0], mul(zi.y, zi.y));
            acc[1] = add(acc[1], mul(zi.x, ri.x));
            acc[1] = add(acc[1], mul(zi.y, ri.y));
        };
        int64_t i = t0;
        for (; i + stride < n2; i += 2 * stride) {
            const In va = load(i), vb = load(i + stride);
            step(va, i);
            step(vb, i + stride);
        }
        if (i < n2) step(load(i), i);
    }
    for (int64_t i = (VEC ? (n & ~int64_t(1)) : 0) + t0; i < n; i += stride) {
        if (NP >= 0) {
            double xi = x[i];
            if (NP >= 1) xi = axpy1(pa[0], pp0[i], xi);
            if (NP >= 2) xi = axpy1(pa[1], pp1[i], xi);
            if (NP >= 3) xi = axpy1(pa[2], pp2[i], xi);
            x[i] = axpy1(a, p[i], xi);
        }
        const double ri = axpy1(na, w[i], r[i]);
        const double zi = PC == 0 ? ri : mul(PC == 1 ? dinv[i] : dconst, ri);
        if (!(zw & 2)) r[i] = ri;
        if (zw & 1) z[i]    = zi;
        acc[0]          = add(acc[0], mul(zi, zi));
        acc[1]          = add(acc[1], mul(zi, ri));
    }
    cg_update_tail<COND>(acc, smem, &flag, st, hist, it, rtol, atol, partials, ticket, max_it, cond,
                         use_cond);
}

// ---------------------------------------------------------------------------
// Unfused-mode scalar tails (one thread each): the Eval() steps of the
// listing plus state bookkeeping.
// ---------------------------------------------------------------------------
__global__ void k_unfused_tail0(CgState* st, double* hist, const double* dp, double rtol,
                                double atol)
{
    const double dp0   = *dp;
    hist[0]            = dp0;
    st->dp0            = dp0;
    st->dp             = dp0;
    st->betaold        = 0.0;
    st->iterations     = 0;
    st->breakdown_iter = -1;
    const bool conv    = cg_converged(dp0, dp0, rtol, atol);
    st->state          = conv ? RVK_CG_CONVERGED : RVK_CG_RUNNING;
    st->done           = conv ? 1 : 0;
}

__global__ void k_unfused_pre(CgState* st, int it) // b = beta/betaold guard
{
    if (st->done) return;
    if (st->betaold == 0.0) {
        st->state          = RVK_CG_BREAKDOWN;
        st->breakdown_iter = it;
        st->done           = 1;
    }
}

__global__ void k_unfused_alpha(CgState* st, int it) // a = beta/a; betaold = beta
{
    if (st->done) return;
    const double pAp = st->pAp;
    const double a   = st->beta / pAp;
    if (pAp == 0.0 || !isfinite(a)) {
        st->state          = RVK_CG_BREAKDOWN;
        st->breakdown_iter = it;
        st->done           = 1;
    } else {
        st->alpha   = a;
        st->betaold = st->beta;
    }
}

__global__ void k_unfused_hist(CgState* st, double* hist, int it, double rtol, double atol)
{
    if (st->done) return;
    hist[it + 1]   = st->dp;
    st->iterations = it + 1;
    if (cg_converged(st->dp, st->dp0, rtol, atol)) {
        st->state = RVK_CG_CONVERGED;
        st->done  = 1;
    }
}

// guarded copy p = z (iteration 0 of the unfused sequence)
__global__ void k_guarded_copy(int64_t n, const double* __restrict__ src, double* __restrict__ dst,
                               const int* guard)
{
    if (*guard) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = src[i];
}


// diag / dinv (csr.hpp:76-77): zero where absent; dinv = 1/diag.
// col_off: column of row r's diagonal is r + col_off (0, or a shard's lo halo).
template <bool INV>
__global__ void k_diagonal(int64_t n, const int64_t* __restrict__ off,
                           const int32_t* __restrict__ cols, const double* __restrict__ vals,
                           double* __restrict__ out, int64_t col_off)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
        double d = 0.0;
        for (int64_t k = off[r]; k < off[r + 1]; ++k)
            if (cols[k] == r + col_off) d = vals[k];
        out[r] = INV ? 1.0 / d : d;
    }
}

// Structural checks + max row length (csr.hpp:46-53).  err bits:
// 1 off[0]!=0, 2 decreasing offsets, 4 off[n]!=nnz, 8 col out of range,
// 16 columns not strictly increasing.
__global__ void k_validate(int64_t n, int64_t n_cols, int64_t nnz, const int64_t* __restrict__ off,
                           const int32_t* __restrict__ cols, unsigned int* err,
                           unsigned long long* maxlen)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned int  e      = 0;
    unsigned long long ml = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
        const int64_t a = off[r], b = off[r + 1];
        if (r == 0 && a != 0) e |= 1u;
        if (b < a) { e |= 2u; continue; }
        if (r == n - 1 && b != nnz) e |= 4u;
        if (a < 0 || b > nnz) { e |= 4u; continue; }
        if ((unsigned long long)(b - a) > ml) ml = (unsigned long long)(b - a);
        int64_t prev = -1;
        for (int64_t k = a; k < b; ++k) {
            const int64_t c = cols[k];
            if (c < 0 || c >= n_cols) e |= 8u;
            if (c <= prev) e |= 16u;
            prev = c;
        }
    }
    if (e) atomicOr(err, e);
    if (ml) atomicMax(maxlen, ml);
}

int update_grid(int64_t n)
{
    const int64_t want = (n / 2 + kUpdThreads - 1) / kUpdThreads;
    const int64_t cap  = (int64_t)sm_count() * 4;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- stencil structure (plan time) -------------------------------------------
// AUTO: fixed-iteration solves up to this many rows (past the grid solves)
// would run as the fused persistent kernel (k_cg_fp).  0: measured slower
// than (or level with) the fused graph almost everywhere -- 5-point 1024^2
// 0.695 vs 0.588 ms, 9-point 1024^2 0.699 vs 0.696, 7-point 100^3 0.606 vs
// 0.635, 128^3 1.24 vs 1.15, 9-point 2048^2 2.92 vs 2.35 --
// so it is opt-in (RVK_OPT_FPERSIST) and the explicit PERSISTENT mode's
// kernel past the grid solves
constexpr int64_t            kFpAutoRows = 0;
constexpr int                kDiagTable = 128;
constexpr unsigned long long kDiagEmpty = ~0ull;

__global__ void k_diagonals(int64_t n, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ cols, unsigned long long* table,
                            int* overflow)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
        for (int64_t k = off[r]; k < off[r + 1]; ++k) {
            // sign bit flipped so no diagonal (d = -1 included) aliases the empty marker
            const unsigned long long key =
                (unsigned long long)((long long)cols[k] - (long long)r) ^ (1ull << 63);
            // lanes that found the same diagonal insert once (warp dedupe)
            const unsigned peers  = __match_any_sync(__activemask(), key);
            const int      leader = __ffs(peers) - 1;
            if ((int)(threadIdx.x & 31) != leader) continue;
            unsigned h = (unsigned)((key * 0x9E3779B97F4A7C15ull) >> 57) & (kDiagTable - 1);
            bool     done = false;
            for (int probe = 0; probe < kDiagTable && !done; ++probe, h = (h + 1) & (kDiagTable - 1)) {
                const unsigned long long v = *((volatile unsigned long long*)&table[h]);
                if (v == key) done = true;
                else if (v == kDiagEmpty) {
                    const unsigned long long old = atomicCAS(&table[h], kDiagEmpty, key);
                    done = (old == kDiagEmpty || old == key);
                }
            }
            if (!done) atomicExch(overflow, 1);
        }
    }
}

rvk_status csr_bands(cudaStream_t s, const rvk_csr& A, SpmvBands* out)
{
    *out = SpmvBands{};
    if (A.n_rows == 0 || A.nnz == 0) return RVK_OK;
    unsigned long long* table = nullptr;
    RVK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&table), kDiagTable * 8 + 16, s));
    int* overflow = reinterpret_cast<int*>(table + kDiagTable);
    RVK_CUDA(cudaMemsetAsync(table, 0xff, kDiagTable * 8, s));
    RVK_CUDA(cudaMemsetAsync(overflow, 0, 4, s));
    const int g = (int)std::min<int64_t>((A.n_rows + 255) / 256, (int64_t)sm_count() * 8);
    k_diagonals<<<g, 256, 0, s>>>(A.n_rows, A.row_offsets, A.col_indices, table, overflow);
    RVK_CHECK_LAUNCH("k_diagonals");
    std::vector<unsigned long long> h(kDiagTable + 2);
    RVK_CUDA(cudaMemcpyAsync(h.data(), table, kDiagTable * 8 + 16, cudaMemcpyDeviceToHost, s));
    RVK_CUDA(cudaFreeAsync(table, s));
    {
        trace::HostSyncScope hs_("cg_plan.diagonal_scan");
        RVK_CUDA(cudaStreamSynchronize(s));
    }
    if (reinterpret_cast<int*>(&h[kDiagTable])[0]) return RVK_OK; // > 128 diagonals: general CSR
    std::vector<int64_t> d;
    for (int i = 0; i < kDiagTable; ++i)
        if (h[i] != kDiagEmpty) d.push_back((int64_t)(long long)(h[i] ^ (1ull << 63)));
    std::sort(d.begin(), d.end());
    // the highest band: diagonals closer than kGap belong to it
    constexpr int64_t kGap = 64, kMaxBand = 4096;
    if (d.empty()) return RVK_OK;
    int64_t lo = d.back();
    for (size_t i = d.size() - 1; i > 0 && lo - d[i - 1] <= kGap; --i) lo = d[i - 1];
    if (d.back() - lo <= kMaxBand) {
        out->has_lead = true;
        out->lead_lo  = lo;
        out->lead_hi  = d.back();
    }
    // plane stride (3D stencils): split the positive diagonals at their
    // largest gap; the upper cluster is the +plane band, Q its middle
    // diagonal, which must be mirrored by -Q and exceed twice the widths of
    // the in-plane and plane bands (the plane-marching K1's cache geometry)
    std::vector<int64_t> pos;
    for (int64_t v : d)
        if (v > 0) pos.push_back(v);
    if (pos.size() >= 2) {
        size_t  cut = 0;
        int64_t gap = pos[0];
        for (size_t i = 1; i < pos.size(); ++i)
            if (pos[i] - pos[i - 1] > gap) {
                gap = pos[i] - pos[i - 1];
                cut = i;
            }
        if (cut > 0) {
            const int64_t q    = pos[cut + (pos.size() - cut) / 2];
            const int64_t band = std::max(q - pos[cut], pos.back() - q);
            const int64_t w    = pos[cut - 1];
            if (std::binary_search(d.begin(), d.end(), -q) && q % 32 == 0 && q > 2 * (w + band) &&
                pos[cut] - w > w + band)
                out->plane_q = q;
        }
    }
    return RVK_OK;
}

bool make_spmv_march(const rvk_csr& A, int64_t max_row_len, int64_t Q, int grid, SpmvArgs* a,
                     SpmvMarch* M)
{
    if (Q <= 0 || Q % 32 != 0 || Q / 32 < grid || A.n_rows < 3 * Q) return false;
    // the fewest ranges per CTA (passes: a smaller cache) that leave a TMA
    // ring of >= 3 stages; else the fewest with 2
    bool found = false;
    for (int passes = 1; passes <= 16 && Q / 32 >= (int64_t)grid * passes; ++passes) {
        SpmvMarch m;
        m.Q      = Q;
        m.K      = (A.n_rows + Q - 1) / Q;
        m.grid   = grid;
        m.passes = passes;
        m.Lmax   = (int)(((Q / 32 + (int64_t)grid * passes - 1) / ((int64_t)grid * passes)) * 32);
        const int64_t budget =
            (int64_t)kSpmvMarchSmem - (int64_t)kSpmvHeaderBytes - (int64_t)3 * m.Lmax * 8;
        if (budget <= 0) continue;
        // the stage also holds the tile's +plane z / p_old (16 B per row)
        SpmvArgs s{};
        for (int64_t b = budget; b > 0; b -= 4096) {
            s = make_spmv_args(A, max_row_len, nullptr, b);
            const int64_t sb = s.stage_bytes + (int64_t)s.R * 16;
            if (s.stages >= 2 && (int64_t)s.stages * sb <= budget) break;
        }
        m.stage_bytes = s.stage_bytes + s.R * 16;
        if (s.stages < 2 || (int64_t)s.stages * m.stage_bytes > budget) continue;
        if (!found) {
            *a    = s;
            *M    = m;
            found = true;
        }
        if (s.stages >= 3) {
            *a = s;
            *M = m;
            return true;
        }
    }
    return found;
}

rvk_status diag_inverse(cudaStream_t s, const rvk_csr& A, int64_t col_off, double* dinv)
{
    if (A.n_rows == 0) return RVK_OK;
    k_diagonal<true><<<update_grid(2 * A.n_rows), kUpdThreads, 0, s>>>(
        A.n_rows, A.row_offsets, A.col_indices, A.values, dinv, col_off);
    RVK_CHECK_LAUNCH("k_diagonal");
    return RVK_OK;
}

// Is v[0..n) one bit pattern?  (plan time; one counted sync)
__global__ void k_const_check(int64_t n, const unsigned long long* __restrict__ v, int* differs)
{
    const unsigned long long v0 = v[0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (v[i] != v0) {
            *differs = 1;
            return;
        }
}

rvk_status vector_is_constant(cudaStream_t s, int64_t n, const double* v, bool* is_const,
                              double* value)
{
    int* d = nullptr;
    RVK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(int), s));
    RVK_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
    k_const_check<<<update_grid(n), kUpdThreads, 0, s>>>(n, reinterpret_cast<const unsigned long long*>(v), d);
    RVK_CHECK_LAUNCH("k_const_check");
    int h = 1;
    RVK_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
    RVK_CUDA(cudaMemcpyAsync(value, v, sizeof(double), cudaMemcpyDeviceToHost, s));
    RVK_CUDA(cudaFreeAsync(d, s));
    {
        trace::HostSyncScope hs_("cg_plan.const_diag_check");
        RVK_CUDA(cudaStreamSynchronize(s));
    }
    *is_const = h == 0;
    return RVK_OK;
}

} // namespace rvk

using namespace rvk;

struct rvk_cg_plan_s {
    rvk_ctx       ctx = nullptr;
    rvk_csr       A{};
    rvk_cg_config cfg{};
    SpmvArgs      sa{};
    bool          march = false;            // K1 (it >= 1) is k_spmv_march (RVK_PLAN_MARCH)
    SpmvArgs      sa_m{};                   // ... its ring geometry
    SpmvMarch     mg{};                     // ... and plane ranges
    int           spmv_grid = 0, upd_grid = 0, setup_grid = 0, persist_grid = 0;
    int           xfix_grid = 0;             // k_cg_xfix: its own resident wave (46 registers)
    int           mode = RVK_CG_MODE_FUSED; // resolved (AUTO -> FUSED | PERSISTENT)
    int           cluster = 0;              // PERSISTENT: CTAs of the one-cluster DSMEM solve (0: grid barriers)
    int           grid_rpc = 0, grid_ctas = 0; // PERSISTENT: the one-launch grid solve (k_cg_grid), rows per CTA
    unsigned*     gbar = nullptr;            // ... its arrival counter
    bool          grid_l2 = false;           // ... past the shared-memory ELL: k_cg_grid_l2 over ell
    bool          fp      = false;           // PERSISTENT: the fused persistent solve (k_cg_fp)
    GridEll       ell{};
    void*         ell_buf = nullptr;
    int           maxlen  = 0;              // longest row
    bool          k2_last = false;          // enqueue_fused: the K2 being launched is the solve's last
    bool          stencil = false;          // matrix-free operator (rvk_cg_plan_create_stencil)
    StencilGeom   geom{};
    double        dconst = 0.0;             // constant dinv (stencil, or a detected constant diagonal)
    bool          const_diag = false;       // CSR plan: every dinv[i] bit-identical -> scalar
    bool          zv         = false;       // fused solve keeps z virtual (z = d r)
    int           mf_grid = 0;
    MfTma*        mf_tma  = nullptr;         // TMA 2.5D matrix-free kernel state (or null)
    double*       dinv = nullptr;
    double*       r = nullptr;
    double*       z = nullptr;
    double*       p[kMaxXq] = {}; // rotating: iteration j writes p[(j+1) % npb]
    int           npb  = 2; // p buffers: max(2, xq)
    int           xq   = 4; // x updated once per group of xq iterations (1 = every one;
                            // max_it = the whole solve, one x pass at the end)
    double*       w    = nullptr;
    double*       hist = nullptr;
    CgState*      st   = nullptr;
    double*       partials = nullptr;     // plan-owned reduction scratch
    unsigned int* tickets  = nullptr;
    double*       tmp      = nullptr;     // unfused: dp scratch
    double*       b_buf    = nullptr;     // host e2e staging
    double*       x_buf    = nullptr;
    // rvk_cg_solve_host_many: second staging pair, copy streams, per-RHS results
    double*       b_buf2   = nullptr;
    double*       x_buf2   = nullptr;
    cudaStream_t  s_in = nullptr, s_out = nullptr;
    cudaEvent_t   ev_many[8] = {};        // b_ready[2], solved[2], x_free[2], b_free[2]
    double*       hist_all = nullptr;     // [cap_many][max_it + 1]
    CgState*      st_all   = nullptr;     // [cap_many]
    int           cap_many = 0;
    // graph cache: two slots, so alternating (b, x) pairs (the pipelined
    // many-RHS solve) replay without re-capturing
    struct GraphSlot {
        cudaGraphExec_t exec = nullptr;
        const double*   b    = nullptr;
        double*         x    = nullptr;
        bool            prof = false;
        int             kind = 0; // 1 unrolled, 2 device WHILE loop
        int             launches = 0;
    };
    GraphSlot gs[2];
    int       g_victim = 0;
    // profiling
    bool                     profiling = false;
    std::vector<cudaEvent_t> ev;          // 4 per iteration: K1 begin/end, K2 begin/end
    int                      launches  = 0;
};

namespace {

// Launch K0 / K2 for the preconditioner mode: 0 none, 1 dinv vector (CSR),
// 2 constant dinv (matrix-free stencil: the diagonal is the centre weight).
template <bool V>
rvk_status launch_setup(rvk_cg_plan P, int pcm, const double* b, double* x, bool xw = true)
{
    cudaStream_t s = P->ctx->stream;
    auto go = [&](auto kern) {
        launch_k(kern, P->setup_grid, kUpdThreads, 0, s, P->A.n_rows, b, P->dinv, x, P->r, P->z,
                   P->st, P->hist, P->cfg.rtol, P->cfg.atol, P->partials, P->tickets, P->dconst,
                   P->zv ? 0 : 1, xw ? 1 : 0);
    };
    if (pcm == 0) go(k_cg_setup<V, 0>);
    else if (pcm == 1) go(k_cg_setup<V, 1>);
    else go(k_cg_setup<V, 2>);
    RVK_CHECK_LAUNCH("k_cg_setup");
    return RVK_OK;
}

// x-update mode of one K2 launch (k_cg_update NP): np = 0 plain, -1 defer
// into pend_a[slot], 1..3 flush those pending updates (pp: their p buffers).
struct XUpd {
    int           np   = 0;
    int           slot = 0;
    const double* pp[3] = {nullptr, nullptr, nullptr};
};

// K2 store mask: bit 0 store z (clear: z virtual), bit 1 the last K2 of a
// fixed-iteration solve -- its r and z are never read again in this solve, so
// neither is stored (16 n bytes per solve).  The next solve starts from b: its
// setup (k_cg_setup, or K1(0) folded) writes r, and z is either formed on the
// fly (virtual / folded) or written before any read.  rvk_cg_plan_vector(R / Z)
// after a solve is therefore only meaningful with RVK_OPT_KEEP_WORK.
int k2_store(rvk_cg_plan P) { return P->k2_last ? 2 : (P->zv ? 0 : 1); }

template <int PC, bool COND, int NP>
void launch_update_k(rvk_cg_plan P, const double* p_new, double* x, int it,
                     cudaGraphConditionalHandle cond, int use_cond, const XUpd& u)
{
    launch_k(k_cg_update<true, PC, COND, NP>, P->upd_grid, kUpdThreads, 0, P->ctx->stream,
               P->A.n_rows, p_new, P->w, P->dinv, x, P->r, P->z, P->st, P->hist, it, P->cfg.rtol,
               P->cfg.atol, P->partials, P->tickets, P->dconst, P->cfg.max_it, cond, use_cond,
               u.pp[0], u.pp[1], u.pp[2], u.slot, k2_store(P));
}

template <int PC, bool COND>
void launch_update_xm(rvk_cg_plan P, const double* p_new, double* x, int it,
                      cudaGraphConditionalHandle cond, int use_cond, const XUpd& u)
{
    switch (u.np) {
    case -1: launch_update_k<PC, COND, -1>(P, p_new, x, it, cond, use_cond, u); break;
    case 1: launch_update_k<PC, COND, 1>(P, p_new, x, it, cond, use_cond, u); break;
    case 2: launch_update_k<PC, COND, 2>(P, p_new, x, it, cond, use_cond, u); break;
    case 3: launch_update_k<PC, COND, 3>(P, p_new, x, it, cond, use_cond, u); break;
    default: launch_update_k<PC, COND, 0>(P, p_new, x, it, cond, use_cond, u);
    }
}

template <bool V>
rvk_status launch_update(rvk_cg_plan P, int pcm, const double* p_new, double* x, int it,
                         cudaGraphConditionalHandle cond = 0, int use_cond = 0, XUpd u = {})
{
    cudaStream_t s = P->ctx->stream;
    if (V && u.np != 0) {
        if (use_cond) {
            if (pcm == 0) launch_update_xm<0, true>(P, p_new, x, it, cond, use_cond, u);
            else if (pcm == 1) launch_update_xm<1, true>(P, p_new, x, it, cond, use_cond, u);
            else launch_update_xm<2, true>(P, p_new, x, it, cond, use_cond, u);
        } else {
            if (pcm == 0) launch_update_xm<0, false>(P, p_new, x, it, cond, use_cond, u);
            else if (pcm == 1) launch_update_xm<1, false>(P, p_new, x, it, cond, use_cond, u);
            else launch_update_xm<2, false>(P, p_new, x, it, cond, use_cond, u);
        }
        RVK_CHECK_LAUNCH("k_cg_update");
        return RVK_OK;
    }
    auto go = [&](auto kern) {
        launch_k(kern, P->upd_grid, kUpdThreads, 0, s, P->A.n_rows, p_new, P->w, P->dinv, x,
                   P->r, P->z, P->st, P->hist, it, P->cfg.rtol, P->cfg.atol, P->partials,
                   P->tickets, P->dconst, P->cfg.max_it, cond, use_cond, (const double*)nullptr,
                   (const double*)nullptr, (const double*)nullptr, 0, k2_store(P));
    };
    if (use_cond) {
        if (pcm == 0) go(k_cg_update<V, 0, true>);
        else if (pcm == 1) go(k_cg_update<V, 1, true>);
        else go(k_cg_update<V, 2, true>);
    } else {
        if (pcm == 0) go(k_cg_update<V, 0>);
        else if (pcm == 1) go(k_cg_update<V, 1>);
        else go(k_cg_update<V, 2>);
    }
    RVK_CHECK_LAUNCH("k_cg_update");
    return RVK_OK;
}

rvk_status launch_xfix(rvk_cg_plan P, double* x, int npb, bool xzero = false)
{
    XBufs pb{};
    for (int k = 0; k < npb; ++k) pb.p[k] = P->p[k];
    // 4 p streams in flight per thread (measured 7-point 256^3, 20 p's:
    // 2 / 4 / 8 per batch = 500 / 475 / 492 us)
    launch_k(k_cg_xfix<4>, P->xfix_grid, kUpdThreads, 0, P->ctx->stream, P->A.n_rows, x, pb, npb,
               (const CgState*)P->st, xzero ? 1 : 0);
    RVK_CHECK_LAUNCH("k_cg_xfix");
    return RVK_OK;
}

// x-update group of a FUSED plan.  Default: the whole solve when it fits
// (5 <= max_it <= kMaxXq, max_it p buffers in free HBM): every
// K2 defers and k_cg_xfix applies the max_it updates in one pass at the end
// -- 16 n + 8 n max_it bytes per solve instead of 24 n per iteration.  Else
// groups of 4 (the WHILE-loop graph always uses groups of <= 4: its p ring is
// static).  Measured on B200, 7-point 256^3: pairs 9.25 -> groups of 4 8.58
// -> whole solve 8.46 ms.
void set_x_group(rvk_cg_plan P)
{
    const int mi = P->cfg.max_it;
    int       q  = (P->cfg.opts & RVK_OPT_X_EACH) ? 1 : 4;
    if (mi >= 5 && mi <= kMaxXq && !(P->cfg.opts & (RVK_OPT_X_EACH | RVK_OPT_X_GROUP4))) {
        const size_t vb = (size_t)P->A.n_rows * sizeof(double) + 32;
        size_t       fr = 0, tot = 0;
        const bool   fits = cudaMemGetInfo(&fr, &tot) == cudaSuccess &&
                          fr > (size_t)(mi - 2) * vb + 8 * vb + (size_t(2) << 30);
        if (fits) q = mi;
    }
    if (P->mode != RVK_CG_MODE_FUSED) q = 1;
    P->xq  = q;
    P->npb = q > 2 ? q : 2;
}

// Group and p-ring size of the device WHILE-loop graph (body = one ring turn)
int while_group(rvk_cg_plan P) { return P->xq < 4 ? P->xq : 4; }
int while_ring(rvk_cg_plan P) { return while_group(P) > 2 ? while_group(P) : 2; }

// Grouped x updates on this solve? (vector path, max_it >= 2, group > 1)
bool x_defer(rvk_cg_plan P, bool vec) { return vec && P->cfg.max_it >= 2 && P->xq > 1; }

// Setup folded into K1(0) (CgFirstBOp): fixed-iteration FUSED CSR solves on
// the unrolled graph / stream path.  b is gathered (and L2-bulk-prefetched)
// by the SpMV, so it must be 16-B aligned; the WHILE graph and matrix-free
// plans keep k_cg_setup.  b == nullptr: the plan-level answer (flags).
bool fold_setup(rvk_cg_plan P, const double* b)
{
    return P->mode == RVK_CG_MODE_FUSED && !P->stencil && P->cfg.use_graph != 2 &&
           !(P->cfg.opts & RVK_OPT_NO_FOLD) && (b == nullptr || aligned16(b));
}

// The x-update mode of iteration `it` (for a WHILE body any index with the
// right residue mod npb): defer inside a group, flush at its end or at the
// solve's last iteration.
// A group longer than 4 (the whole solve) is flushed by k_cg_xfix only.
XUpd x_mode(rvk_cg_plan P, bool defer, int it, bool last, int q, int npb)
{
    XUpd u;
    if (!defer) return u;
    const int c = it % q;
    if ((c == q - 1 || last) && q <= 4) {
        u.np = c;
        for (int k = 0; k < c; ++k) u.pp[k] = P->p[(it - c + k + 1) % npb];
    } else {
        u.np   = -1;
        u.slot = c;
    }
    return u;
}

// K1 of one iteration: it >= 0 static index, it == -1 read from the device
// (WHILE body); `first` selects the p = z variant of iteration 0.
rvk_status launch_k1(rvk_cg_plan P, int it, bool first, const double* p_old, double* p_new)
{
    cudaStream_t   s = P->ctx->stream;
    const int64_t  n = P->A.n_rows;
    const TailArgs ta{P->partials + 2 * kMaxReduceBlocks, P->tickets + 1};
    // virtual z: gather r and form z = d r (d = the constant diagonal, 1 w/o PC)
    const double zs = P->cfg.pc == RVK_PC_JACOBI ? P->dconst : 1.0;
    if (P->stencil)
        return launch_mf_k1(s, P->geom, first, P->zv ? P->r : P->z, p_old, p_new, P->w, P->st, n,
                            it, ta.partials, ta.ticket, P->mf_grid, P->mf_tma, P->zv, zs);
    if (P->zv) {
        if (first) {
            CgSpmvOp<true, true> op{P->r, p_old, p_new, P->w, P->st, n, it, 0.0, zs};
            return launch_spmv(s, P->sa, op, ta, P->spmv_grid);
        }
        CgSpmvOp<false, true> op{P->r, p_old, p_new, P->w, P->st, n, it, 0.0, zs};
        if (P->march) return launch_spmv_march(s, P->sa_m, P->mg, op, ta);
        return launch_spmv(s, P->sa, op, ta, P->spmv_grid);
    }
    if (first) {
        CgSpmvOp<true> op{P->z, p_old, p_new, P->w, P->st, n, it, 0.0};
        return launch_spmv(s, P->sa, op, ta, P->spmv_grid);
    }
    CgSpmvOp<false> op{P->z, p_old, p_new, P->w, P->st, n, it, 0.0};
    if (P->march) return launch_spmv_march(s, P->sa_m, P->mg, op, ta);
    return launch_spmv(s, P->sa, op, ta, P->spmv_grid);
}

// Virtual z for the fused solve (z = d r never stored): constant diagonal or
// no preconditioner, FUSED mode, classic K2.  Measured (B200, 20-iteration
// solves): K2 131 -> 107 us everywhere, but the extra d * r per gathered
// nonzero costs the 7-nonzero-batch SpMV more than that (7-point 256^3 K1
// 316 -> 347 us, solve 8.83 -> 8.95 ms; 5-point likewise), while the 9-batch
// kernels absorb it (27-point 21.02 -> 20.50 ms, 9-point 10.01 -> 9.47 ms)
// and the matrix-free operator gains (4.60 -> 4.10 ms).  So: matrix-free and
// 9-batch CSR plans (RVK_OPT_Z_STORED / RVK_OPT_Z_VIRTUAL override).
bool virtual_z(rvk_cg_plan P)
{
    const int o = P->cfg.opts;
    if (o & RVK_OPT_Z_STORED) return false;
    const bool ok = P->mode == RVK_CG_MODE_FUSED && (P->cfg.pc == RVK_PC_NONE || P->const_diag || P->stencil);
    return ok && (P->stencil || P->sa.unroll == 9 || (o & RVK_OPT_Z_VIRTUAL));
}

// the convergence loop entirely on the device.  Graph =
// [K0, K1(0), K2(0)] -> WHILE(cond) { K1, K2, K1, K2 } where K2's last block
// sets the condition (not converged, no breakdown, iterations < max_it); the
// body holds two iterations so the p ping-pong is static.  No kernel launches
// after convergence, no host involvement.
rvk_status build_while_graph(rvk_cg_plan P, const double* b, double* x, cudaGraphExec_t* out)
{
    cudaStream_t s   = P->ctx->stream;
    const int    pcm = P->cfg.pc != RVK_PC_JACOBI ? 0 : ((P->stencil || P->const_diag) ? 2 : 1);
    const bool   vec = aligned16(b) && aligned16(x) && aligned16(P->dinv);
    cudaGraph_t  g = nullptr, pro = nullptr, tmp = nullptr;
    RVK_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    RVK_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    auto fail = [&](rvk_status rc) {
        if (pro) cudaGraphDestroy(pro);
        cudaGraphDestroy(g);
        return rc;
    };
    // prologue
    RVK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    rvk_status rc = vec ? launch_setup<true>(P, pcm, b, x) : launch_setup<false>(P, pcm, b, x);
    if (rc == RVK_OK) rc = launch_k1(P, 0, true, P->p[0], P->p[1]);
    const bool defer = x_defer(P, vec);
    const int wq = while_group(P), wr = while_ring(P);
    if (rc == RVK_OK)
        rc = vec ? launch_update<true>(P, pcm, P->p[1], x, 0, h, 1,
                                       x_mode(P, defer, 0, P->cfg.max_it == 1, wq, wr))
                 : launch_update<false>(P, pcm, P->p[1], x, 0, h, 1);
    cudaError_t e = cudaStreamEndCapture(s, &pro);
    if (rc != RVK_OK) return fail(rc);
    if (e != cudaSuccess) return fail(cuda_error(e, "capture (while prologue)"));
    cudaGraphNode_t npro, nwhile;
    if ((e = cudaGraphAddChildGraphNode(&npro, g, nullptr, 0, pro)) != cudaSuccess)
        return fail(cuda_error(e, "cudaGraphAddChildGraphNode"));
    cudaGraphNodeParams prm = {};
    prm.type               = cudaGraphNodeTypeConditional;
    prm.conditional.handle = h;
    prm.conditional.type   = cudaGraphCondTypeWhile;
    prm.conditional.size   = 1;
    if ((e = cudaGraphAddNode(&nwhile, g, &npro, 1, &prm)) != cudaSuccess)
        return fail(cuda_error(e, "cudaGraphAddNode(WHILE)"));
    cudaGraph_t body = prm.conditional.phGraph_out[0];
    // body: odd iteration (p_old = p[1]) then even iteration (p_old = p[0])
    if ((e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        return fail(cuda_error(e, "cudaStreamBeginCaptureToGraph"));
    // body: npb iterations (residues 1, 2, ..., 0 mod npb), so every p buffer
    // index is static; a group ending mid-body is flushed by the epilogue
    for (int j = 1; j <= wr && rc == RVK_OK; ++j) {
        const int c = j % wr;
        rc = launch_k1(P, -1, false, P->p[c], P->p[(c + 1) % wr]);
        if (rc == RVK_OK)
            rc = vec ? launch_update<true>(P, pcm, P->p[(c + 1) % wr], x, -1, h, 1,
                                           x_mode(P, defer, c, false, wq, wr))
                     : launch_update<false>(P, pcm, P->p[(c + 1) % wr], x, -1, h, 1);
    }
    e = cudaStreamEndCapture(s, &tmp);
    if (rc != RVK_OK) return fail(rc);
    if (e != cudaSuccess) return fail(cuda_error(e, "capture (while body)"));
    if (defer) { // epilogue after the loop: apply an update left pending
        cudaGraph_t epi = nullptr;
        RVK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        rc = launch_xfix(P, x, wr);
        e  = cudaStreamEndCapture(s, &epi);
        if (rc != RVK_OK) return fail(rc);
        if (e != cudaSuccess) return fail(cuda_error(e, "capture (while epilogue)"));
        cudaGraphNode_t nepi;
        e = cudaGraphAddChildGraphNode(&nepi, g, &nwhile, 1, epi);
        cudaGraphDestroy(epi);
        if (e != cudaSuccess) return fail(cuda_error(e, "cudaGraphAddChildGraphNode (epilogue)"));
    }
    e = cudaGraphInstantiate(out, g, 0);
    fail(RVK_OK);
    if (e != cudaSuccess) return cuda_error(e, "cudaGraphInstantiate (while)");
    return RVK_OK;
}

rvk_status enqueue_fused(rvk_cg_plan P, const double* b, double* x)
{
    const int64_t n    = P->A.n_rows;
    cudaStream_t  s    = P->ctx->stream;
    const int     pcm  = P->cfg.pc != RVK_PC_JACOBI ? 0 : ((P->stencil || P->const_diag) ? 2 : 1);
    const bool    vec  = aligned16(b) && aligned16(x) && aligned16(P->dinv);
    const TailArgs ta{P->partials + 2 * kMaxReduceBlocks, P->tickets + 1};
    const bool     defer = x_defer(P, vec);
    P->launches = 0;
    auto rec = [&](int k) -> rvk_status {
        if (P->profiling)
            RVK_CUDA(cudaEventRecordWithFlags(P->ev[k], s, cudaEventRecordExternal));
        return RVK_OK;
    };
    // whole-solve x group: x is written once, by the final pass, which starts
    // from 0.0 itself -- the setup skips its x = 0 store (16 n bytes per solve)
    const bool     xz = defer && P->xq > 4;
    // setup folded into K1(0) (CSR, aligned b; any x group / diagonal)
    const bool     fold = fold_setup(P, b);
    rvk_status     rc   = RVK_OK;
    if (fold) {
        // x = 0 only where a K2 reads x (no whole-solve group)
        if (!xz) RVK_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
        k_cg_reset<<<1, 1, 0, s>>>(P->st);
        RVK_CHECK_LAUNCH("k_cg_reset");
    } else {
        rc = vec ? launch_setup<true>(P, pcm, b, x, !xz) : launch_setup<false>(P, pcm, b, x);
    }
    if (rc != RVK_OK) return rc;
    ++P->launches;
    for (int it = 0; it < P->cfg.max_it; ++it) {
        const double* p_old = P->p[it % P->npb];
        double*       p_new = P->p[(it + 1) % P->npb];
        if ((rc = rec(4 * it + 0)) != RVK_OK) return rc;
        if (fold && it == 0) {
            const double d = pcm == 2 ? P->dconst : 1.0;
            if (pcm == 1) {
                CgFirstBOp<true> op{b, P->dinv, p_new, P->w, P->r, P->st, P->hist, d, P->cfg.rtol, P->cfg.atol};
                rc = launch_spmv(s, P->sa, op, ta, P->spmv_grid);
            } else {
                CgFirstBOp<false> op{b, P->dinv, p_new, P->w, P->r, P->st, P->hist, d, P->cfg.rtol, P->cfg.atol};
                rc = launch_spmv(s, P->sa, op, ta, P->spmv_grid);
            }
        } else {
            rc = launch_k1(P, it, it == 0, p_old, p_new);
        }
        if (rc != RVK_OK) return rc;
        ++P->launches;
        if ((rc = rec(4 * it + 1)) != RVK_OK || (rc = rec(4 * it + 2)) != RVK_OK) return rc;
        // grouped x: defer inside a group, flush at its end (or the last iteration)
        P->k2_last = it + 1 == P->cfg.max_it && !(P->cfg.opts & RVK_OPT_KEEP_WORK);
        rc = vec ? launch_update<true>(P, pcm, p_new, x, it, 0, 0,
                                       x_mode(P, defer, it, it + 1 == P->cfg.max_it, P->xq, P->npb))
                 : launch_update<false>(P, pcm, p_new, x, it);
        P->k2_last = false;
        if (rc != RVK_OK) return rc;
        ++P->launches;
        if ((rc = rec(4 * it + 3)) != RVK_OK) return rc;
    }
    if (defer) { // the whole-solve group, or an early exit mid-group, leaves x pending
        if ((rc = launch_xfix(P, x, P->npb, xz)) != RVK_OK) return rc;
        ++P->launches;
    }
    return RVK_OK;
}

#define RVK_TRY(x)                                                                             \
    do {                                                                                       \
        rvk_status rc_ = (x);                                                                  \
        if (rc_ != RVK_OK) return rc_;                                                         \
    } while (0)

// The reference's op-per-kernel sequence, every scalar a
// device pointer: identical arithmetic to the fused path.
rvk_status enqueue_unfused(rvk_cg_plan P, const double* b, double* x)
{
    const int64_t n   = P->A.n_rows;
    cudaStream_t  s   = P->ctx->stream;
    const bool    jac = P->cfg.pc == RVK_PC_JACOBI;
    Scratch       sc{P->partials, P->tickets};
    CgState*      st  = P->st;
    const int*    g   = &st->done;
    double*       dp  = P->tmp;
    auto ptr = [](const double* p) { return rvk_scalar{RVK_SCALAR_PTR, 0.0, p, nullptr}; };
    P->launches = 0;

    RVK_CUDA(cudaMemcpyAsync(P->r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    RVK_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
    if (jac) RVK_TRY(vec_ew(s, EW_PMULT, n, const_scalar(0), P->dinv, P->r, P->z, nullptr));
    else RVK_CUDA(cudaMemcpyAsync(P->z, P->r, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    RVK_TRY(vec_reduce(s, sc, RED_NRM2, n, P->z, nullptr, dp, nullptr, nullptr));
    RVK_TRY(vec_reduce(s, sc, RED_DOT, n, P->z, P->r, &st->beta, nullptr, nullptr));
    k_unfused_tail0<<<1, 1, 0, s>>>(st, P->hist, dp, P->cfg.rtol, P->cfg.atol);
    RVK_CHECK_LAUNCH("k_unfused_tail0");
    P->launches += 5;

    double*        p  = P->p[0];
    const SpmvArgs& sa = P->sa;
    for (int it = 0; it < P->cfg.max_it; ++it) {
        if (it == 0) {
            k_guarded_copy<<<update_grid(n), kUpdThreads, 0, s>>>(n, P->z, p, g);
            RVK_CHECK_LAUNCH("k_guarded_copy");
        } else {
            k_unfused_pre<<<1, 1, 0, s>>>(st, it);
            RVK_CHECK_LAUNCH("k_unfused_pre");
            const rvk_scalar bb{RVK_SCALAR_DIV_PTR_PTR, 0.0, &st->beta, &st->betaold};
            RVK_TRY(vec_ew(s, EW_AYPX, n, bb, P->z, p, p, g));             // p = z + b p
            ++P->launches;
        }
        if (P->profiling) RVK_CUDA(cudaEventRecordWithFlags(P->ev[4 * it + 0], s, cudaEventRecordExternal));
        SpmvGuardedOp op;
        op.x     = p;
        op.y     = P->w;
        op.guard = g;
        RVK_TRY(launch_spmv(s, sa, op, TailArgs{nullptr, nullptr}, P->spmv_grid)); // w = A p
        if (P->profiling) {
            RVK_CUDA(cudaEventRecordWithFlags(P->ev[4 * it + 1], s, cudaEventRecordExternal));
            RVK_CUDA(cudaEventRecordWithFlags(P->ev[4 * it + 2], s, cudaEventRecordExternal));
        }
        RVK_TRY(vec_reduce(s, sc, RED_DOT, n, p, P->w, &st->pAp, nullptr, g));       // a = p.w
        k_unfused_alpha<<<1, 1, 0, s>>>(st, it);                                    // a = beta/a
        RVK_CHECK_LAUNCH("k_unfused_alpha");
        RVK_TRY(vec_ew(s, EW_AXPY, n, ptr(&st->alpha), p, x, x, g));                // x += a p
        const rvk_scalar na{RVK_SCALAR_NEG_PTR, 0.0, &st->alpha, nullptr};
        RVK_TRY(vec_ew(s, EW_AXPY, n, na, P->w, P->r, P->r, g));                    // r += -a w
        if (jac) RVK_TRY(vec_ew(s, EW_PMULT, n, const_scalar(0), P->dinv, P->r, P->z, g));
        else k_guarded_copy<<<update_grid(n), kUpdThreads, 0, s>>>(n, P->r, P->z, g);
        RVK_TRY(vec_reduce(s, sc, RED_NRM2, n, P->z, nullptr, &st->dp, nullptr, g)); // dp = ||z||
        k_unfused_hist<<<1, 1, 0, s>>>(st, P->hist, it, P->cfg.rtol, P->cfg.atol);
        RVK_CHECK_LAUNCH("k_unfused_hist");
        RVK_TRY(vec_reduce(s, sc, RED_DOT, n, P->z, P->r, &st->beta, nullptr, g));  // beta = z.r
        if (P->profiling) RVK_CUDA(cudaEventRecordWithFlags(P->ev[4 * it + 3], s, cudaEventRecordExternal));
        P->launches += 10;
    }
    return RVK_OK;
}

rvk_status enqueue_persistent(rvk_cg_plan P, const double* b, double* x)
{
    PersistArgs a{P->A.n_rows, P->A.row_offsets, P->A.col_indices, P->A.values, b, P->dinv, x, P->r,
                  P->z, P->p[0], P->p[1], P->w, P->hist, P->st, P->partials, P->cfg.max_it,
                  P->cfg.rtol, P->cfg.atol};
    P->launches = 1;
    if (P->fp) {
        const FpArgs f{P->A.n_rows, b, P->dinv, P->dconst, P->const_diag ? 0 : 1, x, P->r, P->z, P->p[0],
                       P->p[1], P->w, P->hist, P->st, P->partials, P->gbar, P->cfg.max_it, P->cfg.rtol,
                       P->cfg.atol};
        return launch_fp(P->ctx->stream, P->sa, f);
    }
    if (P->cluster)
        return launch_cluster(P->ctx->stream, a, P->cfg.pc == RVK_PC_JACOBI, P->cluster, P->maxlen);
    if (P->grid_rpc)
        return launch_grid_solve(P->ctx->stream, a, P->gbar, P->cfg.pc == RVK_PC_JACOBI, P->grid_rpc,
                                 P->grid_ctas, P->maxlen, P->grid_l2 ? &P->ell : nullptr);
    return launch_persistent(P->ctx->stream, a, P->cfg.pc == RVK_PC_JACOBI, P->persist_grid);
}

// Baseline that exposes the scalar problem: every dot/norm
// result is copied to the host and the stream synchronised (3 per
// iteration, like PETSc main's VecDot/VecNorm), and scalars travel back to
// the kernels as host constants.  Same kernels and arithmetic otherwise.
rvk_status solve_hostsync(rvk_cg_plan P, const double* b, double* x)
{
    const int64_t n   = P->A.n_rows;
    cudaStream_t  s   = P->ctx->stream;
    const bool    jac = P->cfg.pc == RVK_PC_JACOBI;
    Scratch       sc{P->partials, P->tickets};
    double*       d   = P->tmp; // device scalar slot
    auto          read = [&](double* out) -> rvk_status {
        RVK_CUDA(cudaMemcpyAsync(out, d, sizeof(double), cudaMemcpyDeviceToHost, s));
        {
            trace::HostSyncScope hs_("cg_hostsync.read_scalar");
            RVK_CUDA(cudaStreamSynchronize(s));
        }
        return RVK_OK;
    };
    std::vector<double> hist(P->cfg.max_it + 1, 0.0);
    CgState             st{};
    st.breakdown_iter = -1;
    P->launches       = 0;
    RVK_CUDA(cudaMemcpyAsync(P->r, b, n * 8, cudaMemcpyDeviceToDevice, s));
    RVK_CUDA(cudaMemsetAsync(x, 0, n * 8, s));
    if (jac) RVK_TRY(vec_ew(s, EW_PMULT, n, const_scalar(0), P->dinv, P->r, P->z, nullptr));
    else RVK_CUDA(cudaMemcpyAsync(P->z, P->r, n * 8, cudaMemcpyDeviceToDevice, s));
    double dp0 = 0, beta = 0, betaold = 0, pAp = 0, dp = 0;
    RVK_TRY(vec_reduce(s, sc, RED_NRM2, n, P->z, nullptr, d, nullptr, nullptr));
    RVK_TRY(read(&dp0));
    hist[0] = dp = dp0;
    auto conv = [&](double v) { return v <= std::fmax(P->cfg.rtol * dp0, P->cfg.atol); };
    st.state = conv(dp0) ? RVK_CG_CONVERGED : RVK_CG_RUNNING;
    if (st.state == RVK_CG_RUNNING) {
        RVK_TRY(vec_reduce(s, sc, RED_DOT, n, P->z, P->r, d, nullptr, nullptr));
        RVK_TRY(read(&beta));
    }
    double* p = P->p[0];
    for (int it = 0; it < P->cfg.max_it && st.state == RVK_CG_RUNNING; ++it) {
        if (it == 0) {
            RVK_CUDA(cudaMemcpyAsync(p, P->z, n * 8, cudaMemcpyDeviceToDevice, s));
        } else {
            if (betaold == 0.0) {
                st.state          = RVK_CG_BREAKDOWN;
                st.breakdown_iter = it;
                break;
            }
            RVK_TRY(vec_ew(s, EW_AYPX, n, const_scalar(beta / betaold), P->z, p, p, nullptr));
        }
        SpmvPlainOp op;
        op.x = p;
        op.y = P->w;
        RVK_TRY(launch_spmv(s, P->sa, op, TailArgs{nullptr, nullptr}, P->spmv_grid));
        RVK_TRY(vec_reduce(s, sc, RED_DOT, n, p, P->w, d, nullptr, nullptr));
        RVK_TRY(read(&pAp));
        const double a = beta / pAp;
        if (pAp == 0.0 || !std::isfinite(a)) {
            st.state          = RVK_CG_BREAKDOWN;
            st.breakdown_iter = it;
            break;
        }
        betaold = beta;
        RVK_TRY(vec_ew(s, EW_AXPY, n, const_scalar(a), p, x, x, nullptr));
        RVK_TRY(vec_ew(s, EW_AXPY, n, const_scalar(-a), P->w, P->r, P->r, nullptr));
        if (jac) RVK_TRY(vec_ew(s, EW_PMULT, n, const_scalar(0), P->dinv, P->r, P->z, nullptr));
        else RVK_CUDA(cudaMemcpyAsync(P->z, P->r, n * 8, cudaMemcpyDeviceToDevice, s));
        RVK_TRY(vec_reduce(s, sc, RED_NRM2, n, P->z, nullptr, d, nullptr, nullptr));
        RVK_TRY(read(&dp));
        hist[it + 1]  = dp;
        st.iterations = it + 1;
        if (conv(dp)) {
            st.state = RVK_CG_CONVERGED;
            break;
        }
        RVK_TRY(vec_reduce(s, sc, RED_DOT, n, P->z, P->r, d, nullptr, nullptr));
        RVK_TRY(read(&beta));
        P->launches += 9;
    }
    st.done = st.state != RVK_CG_RUNNING;
    st.dp0  = dp0;
    st.dp   = dp;
    RVK_CUDA(cudaMemcpyAsync(P->hist, hist.data(), hist.size() * 8, cudaMemcpyHostToDevice, s));
    RVK_CUDA(cudaMemcpyAsync(P->st, &st, sizeof st, cudaMemcpyHostToDevice, s));
    RVK_CUDA(cudaStreamSynchronize(s)); // host buffers above are stack-local
    return RVK_OK;
}

rvk_status enqueue_solve(rvk_cg_plan P, const double* b, double* x)
{
    switch (P->mode) {
    case RVK_CG_MODE_UNFUSED: return enqueue_unfused(P, b, x);
    case RVK_CG_MODE_PERSISTENT: return enqueue_persistent(P, b, x);
    default: return enqueue_fused(P, b, x);
    }
}

rvk_status destroy_graph(rvk_cg_plan P)
{
    for (auto& g : P->gs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g = rvk_cg_plan_s::GraphSlot{};
    }
    return RVK_OK;
}

} // namespace

extern "C" {

rvk_status rvk_csr_validate(rvk_ctx ctx, const rvk_csr* A, int64_t* max_row_len)
{
    if (!ctx || !A) return set_error(RVK_ERR_INVALID, "csr_validate: null argument");
    if (A->n_rows < 0 || A->n_cols < 0 || A->nnz < 0)
        return set_error(RVK_ERR_INVALID, "csr_validate: negative size");
    if (A->n_cols > INT32_MAX) return set_error(RVK_ERR_INVALID, "n_cols exceeds int32 indices");
    if (A->n_rows > 0 && !A->row_offsets) return set_error(RVK_ERR_INVALID, "null row_offsets");
    if (A->nnz > 0 && (!A->col_indices || !A->values))
        return set_error(RVK_ERR_INVALID, "null col_indices/values");
    unsigned int*       err = nullptr;
    unsigned long long* ml  = nullptr;
    RVK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&err), 16, ctx->stream));
    ml = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(err) + 8);
    RVK_CUDA(cudaMemsetAsync(err, 0, 16, ctx->stream));
    if (A->n_rows > 0) {
        const int g = (int)std::min<int64_t>((A->n_rows + 255) / 256, (int64_t)sm_count() * 8);
        k_validate<<<g, 256, 0, ctx->stream>>>(A->n_rows, A->n_cols, A->nnz, A->row_offsets,
                                               A->col_indices, err, ml);
        RVK_CHECK_LAUNCH("k_validate");
    }
    unsigned long long host[2] = {0, 0};
    RVK_CUDA(cudaMemcpyAsync(host, err, 16, cudaMemcpyDeviceToHost, ctx->stream));
    RVK_CUDA(cudaFreeAsync(err, ctx->stream));
    {
        trace::HostSyncScope hs_("csr_validate");
        RVK_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    const unsigned int e = (unsigned int)host[0];
    if (max_row_len) *max_row_len = (int64_t)host[1];
    if (A->n_rows == 0 && A->nnz != 0) return set_error(RVK_ERR_INVALID, "CsrMatrix: nnz != 0 with no rows");
    if (e & 1u) return set_error(RVK_ERR_INVALID, "CsrMatrix: row_offsets[0] != 0");
    if (e & 2u) return set_error(RVK_ERR_INVALID, "CsrMatrix: row_offsets decreasing");
    if (e & 4u) return set_error(RVK_ERR_INVALID, "CsrMatrix: row_offsets[n_rows] != nnz");
    if (e & 8u) return set_error(RVK_ERR_INVALID, "CsrMatrix: column index out of range");
    if (e & 16u)
        return set_error(RVK_ERR_INVALID, "CsrMatrix: columns not strictly increasing in a row");
    return RVK_OK;
}

rvk_status rvk_csr_spmv(rvk_ctx ctx, const rvk_csr* A, const double* x, double* y)
{
    if (!ctx || !A) return set_error(RVK_ERR_INVALID, "csr_spmv: null argument");
    if (A->n_rows == 0) return RVK_OK;
    if (!x || !y) return set_error(RVK_ERR_INVALID, "csr_spmv: null vector");
    RVK_TRACE_TASK(ctx, "rvk_csr_spmv");
    if (A->nnz == 0) return rvk_set(ctx, A->n_rows, 0.0, y); // every row empty: y = 0
    // Tile height from the mean row length (no host sync on this path);
    // tiles that overflow a stage fall back to direct global reads.
    const int64_t avg = (A->nnz + A->n_rows - 1) / A->n_rows;
    SpmvPlainOp   op;
    op.x = x;
    op.y = y;
    return launch_spmv(ctx->stream, make_spmv_args(*A, avg + avg / 4 + 1), op,
                       TailArgs{nullptr, nullptr}, sm_count());
}

rvk_status rvk_csr_diagonal(rvk_ctx ctx, const rvk_csr* A, double* diag)
{
    if (!ctx || !A || (A->n_rows > 0 && !diag)) return set_error(RVK_ERR_INVALID, "null argument");
    if (A->n_rows == 0) return RVK_OK;
    RVK_TRACE_TASK(ctx, "rvk_csr_diagonal");
    k_diagonal<false><<<update_grid(2 * A->n_rows), kUpdThreads, 0, ctx->stream>>>(
        A->n_rows, A->row_offsets, A->col_indices, A->values, diag, 0);
    RVK_CHECK_LAUNCH("k_diagonal");
    return RVK_OK;
}

rvk_status rvk_csr_diagonal_inverse(rvk_ctx ctx, const rvk_csr* A, double* dinv)
{
    if (!ctx || !A || (A->n_rows > 0 && !dinv)) return set_error(RVK_ERR_INVALID, "null argument");
    if (A->n_rows == 0) return RVK_OK;
    RVK_TRACE_TASK(ctx, "rvk_csr_diagonal_inverse");
    k_diagonal<true><<<update_grid(2 * A->n_rows), kUpdThreads, 0, ctx->stream>>>(
        A->n_rows, A->row_offsets, A->col_indices, A->values, dinv, 0);
    RVK_CHECK_LAUNCH("k_diagonal");
    return RVK_OK;
}

rvk_status rvk_cg_plan_create(rvk_ctx ctx, const rvk_csr* A, rvk_cg_config cfg, rvk_cg_plan* out)
{
    if (!ctx || !A || !out) return set_error(RVK_ERR_INVALID, "cg_plan_create: null argument");
    *out = nullptr;
    RVK_TRACE_TASK(ctx, "cg.plan_create");
    if (A->n_rows != A->n_cols) return set_error(RVK_ERR_DIM, "cg_solve: matrix is not square");
    if (A->n_rows < 1) return set_error(RVK_ERR_DIM, "cg_solve: empty system");
    if (cfg.max_it < 1) return set_error(RVK_ERR_INVALID, "cg_solve: max_it must be >= 1");
    if (cfg.pc != RVK_PC_NONE && cfg.pc != RVK_PC_JACOBI)
        return set_error(RVK_ERR_INVALID, "cg_solve: unknown preconditioner %d", cfg.pc);
    if (cfg.mode < RVK_CG_MODE_FUSED || cfg.mode > RVK_CG_MODE_HOSTSYNC)
        return set_error(RVK_ERR_INVALID, "cg_solve: unknown mode %d", cfg.mode);
    int64_t maxlen = 0;
    RVK_TRY(rvk_csr_validate(ctx, A, &maxlen));

    auto P       = new rvk_cg_plan_s();
    P->ctx       = ctx;
    P->A         = *A;
    P->cfg       = cfg;
    // leading-edge L2 prefetch band (stencil-like matrices)
    SpmvBands bands;
    if (csr_bands(ctx->stream, *A, &bands) != RVK_OK) bands = SpmvBands{};
    P->sa            = make_spmv_args(*A, maxlen, &bands);
    P->sa.small_rows = (cfg.opts & RVK_OPT_SMALL_K1) ? 512 * 1024 : 0;
    {
        // the matrix keeps normal L2 priority when it and the five vectors
        // one iteration touches fit in 100 MB of the 126 MB L2 (re-read from
        // L2 by every K1).  Measured, fused 5-point: 512^2 (47 MB) 0.336 ->
        // 0.317 ms per solve; 1024^2 (111 MB, not kept) 0.618 ms either way,
        // 0.685 ms if kept (L2 thrash).
        const int64_t ws = A->nnz * 12 + (A->n_rows + 1) * 8 + A->n_rows * 40;
        P->sa.csr_keep   = ws <= (int64_t)100 * 1024 * 1024 ? 1 : 0;
    }
    P->spmv_grid = sm_count();
    // plane-marching K1 (opt-in): DRAM reads at the algorithmic minimum for
    // large 3D planes, but measured slower than the row-order kernel on B200
    // (768^3: 12.4-13.9 vs 10.3 ms per K1, profiles/r02/march_768.md), so
    // only RVK_OPT_MARCH selects it
    if ((cfg.opts & RVK_OPT_MARCH) && bands.plane_q > 0)
        P->march = make_spmv_march(*A, maxlen, bands.plane_q, P->spmv_grid, &P->sa_m, &P->mg);
    // one resident wave each (the vectorised loops take 2 elements per thread)
    P->upd_grid   = resident_grid(k_cg_update<true, 1>, kUpdThreads, (A->n_rows + 1) / 2);
    P->xfix_grid  = resident_grid(k_cg_xfix<4>, kUpdThreads, (A->n_rows + 1) / 2);
    P->setup_grid = resident_grid(k_cg_setup<true, 1>, kUpdThreads, (A->n_rows + 1) / 2);
    P->persist_grid = persistent_grid(A->n_rows);
    P->mode         = cfg.mode;
    P->maxlen = (int)std::min<int64_t>(maxlen, 1 << 30);
    if (cfg.mode == RVK_CG_MODE_AUTO || cfg.mode == RVK_CG_MODE_PERSISTENT) {
        P->cluster = (cfg.opts & RVK_OPT_NO_CLUSTER) ? 0 : cluster_ctas(A->n_rows, maxlen);
        // the grid solve from 8 K rows up (measured: 128^2 grid 0.109 vs
        // cluster 0.119 ms, 64^2 cluster 0.096 vs grid 0.111 ms)
        if ((!P->cluster || P->cluster > 8) && !(cfg.opts & RVK_OPT_NO_GRID)) {
            int l2      = 0;
            P->grid_rpc = grid_solve_rows(A->n_rows, maxlen, &P->grid_ctas, &l2);
            if (l2 && (cfg.opts & RVK_OPT_NO_GRID_L2)) P->grid_rpc = 0;
            // AUTO takes the L2 grid solve up to 4 K rows per CTA (8 rows per
            // thread): measured 5-point 768^2 0.315 vs fused 0.421 ms; at
            // 1024^2 (7 K rows per CTA, 97 MB of ELL + vectors, L2 hit 70%)
            // 0.700 vs fused 0.589 ms -- explicit PERSISTENT still runs it
            if (l2 && cfg.mode == RVK_CG_MODE_AUTO && P->grid_rpc > 4096) P->grid_rpc = 0;
            P->grid_l2 = P->grid_rpc && l2;
            if (P->grid_rpc) P->cluster = 0;
        }
    }
    if ((cfg.mode == RVK_CG_MODE_AUTO || cfg.mode == RVK_CG_MODE_PERSISTENT) && !P->cluster && !P->grid_rpc &&
        fp_eligible(P->sa) && !(cfg.opts & RVK_OPT_NO_FPERSIST)) {
        // the fused persistent solve (k_cg_fp): explicit PERSISTENT always;
        // AUTO for fixed-iteration solves up to kFpAutoRows (launch / tail
        // latency bound there) or when RVK_OPT_FPERSIST asks
        const bool fixed = cfg.rtol == 0.0 && cfg.atol == 0.0 && cfg.use_graph != 2;
        P->fp = cfg.mode == RVK_CG_MODE_PERSISTENT ||
                (fixed && (A->n_rows <= kFpAutoRows || (cfg.opts & RVK_OPT_FPERSIST)));
    }
    if (cfg.mode == RVK_CG_MODE_AUTO) {
        // up to 16 K rows: the one-cluster DSMEM solve (one launch, cluster
        // barriers); up to ~450 K rows the one-launch grid solve (grid
        // barriers, CSR in shared memory; ~606 K over a global ELL copy);
        // fixed-iteration solves up to kFpAutoRows the fused persistent
        // solve; above, the HBM-streaming fused graph
        P->mode = (P->cluster || P->grid_rpc || P->fp) ? RVK_CG_MODE_PERSISTENT : RVK_CG_MODE_FUSED;
        // and up to 512 K rows the plain-block K1 (k_spmv_small: 256^2 5-point
        // solve 0.229 -> 0.211 ms; explicit FUSED keeps the TMA kernel unless
        // RVK_OPT_SMALL_K1 asks)
        P->sa.small_rows = 512 * 1024;
    }
    const size_t vb = (size_t)A->n_rows * sizeof(double);
    cudaError_t  e  = cudaSuccess;
    auto alloc = [&](void** p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(p, bytes);
    };
    // every vector a K1 may gather (dinv, r with a virtual z, z, p) padded by
    // 4 doubles
    alloc(reinterpret_cast<void**>(&P->dinv), vb + 32);
    alloc(reinterpret_cast<void**>(&P->r), vb + 32);
    alloc(reinterpret_cast<void**>(&P->z), vb + 32);
    alloc(reinterpret_cast<void**>(&P->p[0]), vb + 32);
    alloc(reinterpret_cast<void**>(&P->p[1]), vb + 32);
    set_x_group(P);
    for (int k = 2; k < P->npb; ++k) alloc(reinterpret_cast<void**>(&P->p[k]), vb + 32);
    alloc(reinterpret_cast<void**>(&P->w), vb);
    alloc(reinterpret_cast<void**>(&P->hist), sizeof(double) * (cfg.max_it + 1));
    alloc(reinterpret_cast<void**>(&P->st), sizeof(CgState));
    alloc(reinterpret_cast<void**>(&P->partials), sizeof(double) * 4 * kMaxReduceBlocks);
    alloc(reinterpret_cast<void**>(&P->tickets), 16 * sizeof(unsigned int));
    alloc(reinterpret_cast<void**>(&P->tmp), 16 * sizeof(double));
    alloc(reinterpret_cast<void**>(&P->gbar), 16 * sizeof(unsigned));
    size_t ell_c_at = 0, ell_n_at = 0;
    if (P->grid_l2) {
        // k-major ELL of the matrix for k_cg_grid_l2 (values, columns, lengths)
        const size_t nz = P->maxlen <= 5 ? 5 : (P->maxlen <= 7 ? 7 : 9);
        ell_c_at        = (nz * vb + 255) / 256 * 256;
        ell_n_at        = ell_c_at + (nz * (size_t)A->n_rows * 4 + 255) / 256 * 256;
        alloc(&P->ell_buf, ell_n_at + (size_t)A->n_rows);
    }
    if (e != cudaSuccess) {
        rvk_cg_plan_destroy(P);
        return cuda_error(e, "rvk_cg_plan_create: allocation");
    }
    cudaStream_t s = ctx->stream;
    if (P->grid_l2) {
        unsigned char* base = static_cast<unsigned char*>(P->ell_buf);
        P->ell.v            = reinterpret_cast<double*>(base);
        P->ell.c            = reinterpret_cast<int32_t*>(base + ell_c_at);
        P->ell.n            = base + ell_n_at;
        const rvk_status bs = build_grid_ell(s, A->n_rows, A->row_offsets, A->col_indices, A->values, P->maxlen,
                                             P->ell.v, P->ell.c, P->ell.n);
        if (bs != RVK_OK) {
            rvk_cg_plan_destroy(P);
            return bs;
        }
    }
    e              = cudaMemsetAsync(P->tickets, 0, 16 * sizeof(unsigned int), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->p[0], 0, vb, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->p[1], 0, vb, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->st, 0, sizeof(CgState), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->hist, 0, sizeof(double) * (cfg.max_it + 1), s);
    if (e != cudaSuccess) {
        rvk_cg_plan_destroy(P);
        return cuda_error(e, "rvk_cg_plan_create: init");
    }
    rvk_status rc = RVK_OK;
    if (cfg.pc == RVK_PC_JACOBI) rc = rvk_csr_diagonal_inverse(ctx, A, P->dinv);
    else rc = rvk_set(ctx, A->n_rows, 1.0, P->dinv);
    // Constant-coefficient operators with Dirichlet truncation have ONE
    // diagonal value, so dinv is a constant vector: the fused K0/K2 then
    // multiply by the scalar (bit-identical z = dinv[i] * r[i]) and skip the
    // 8n-byte dinv stream per iteration (RVK_OPT_DINV_VECTOR disables).  Measured
    // on B200 (7-point 256^3): with the per-iteration x update it was a wash
    // (K2 -12 us, K1 +11 us); with the pairwise x update K2 151 -> 137 us,
    // K1 unchanged, solve 9.31 -> 9.00 ms.
    if (rc == RVK_OK && cfg.pc == RVK_PC_JACOBI && !(cfg.opts & RVK_OPT_DINV_VECTOR))
        rc = vector_is_constant(s, A->n_rows, P->dinv, &P->const_diag, &P->dconst);
    if (rc == RVK_OK) P->zv = virtual_z(P); // after the constant-diagonal check
    if (rc != RVK_OK) {
        rvk_cg_plan_destroy(P);
        return rc;
    }
    *out = P;
    return RVK_OK;
}

int rvk_cg_plan_flags(rvk_cg_plan P)
{
    if (!P) return -1;
    return (P->const_diag ? RVK_PLAN_CONST_DIAG : 0) | (P->stencil ? RVK_PLAN_MATRIX_FREE : 0) |
           (P->mf_tma ? RVK_PLAN_MF_TMA : 0) |
           ((P->mode == RVK_CG_MODE_FUSED && x_defer(P, true)) ? RVK_PLAN_X_DEFER : 0) |
           ((P->mode == RVK_CG_MODE_FUSED && x_defer(P, true) && P->xq == 4) ? RVK_PLAN_X_GROUP4 : 0) |
           ((P->mode == RVK_CG_MODE_FUSED && x_defer(P, true) && P->xq > 4) ? RVK_PLAN_X_SOLVE : 0) |
           ((P->mode == RVK_CG_MODE_PERSISTENT && P->cluster) ? RVK_PLAN_CLUSTER : 0) |
           ((P->mode == RVK_CG_MODE_PERSISTENT && P->grid_rpc) ? RVK_PLAN_GRID : 0) |
           ((P->mode == RVK_CG_MODE_PERSISTENT && P->grid_rpc && P->grid_l2) ? RVK_PLAN_GRID_L2 : 0) |
           ((P->mode == RVK_CG_MODE_PERSISTENT && P->fp) ? RVK_PLAN_FPERSIST : 0) |
           (fold_setup(P, nullptr) ? RVK_PLAN_FOLD_SETUP : 0) |
           (P->zv ? RVK_PLAN_Z_VIRTUAL : 0) |
           ((P->march && !P->stencil && P->mode != RVK_CG_MODE_PERSISTENT) ? RVK_PLAN_MARCH : 0);
}

const double* rvk_cg_plan_vector(rvk_cg_plan P, int which)
{
    if (!P) return nullptr;
    switch (which) {
    case RVK_VEC_R: return P->r;
    case RVK_VEC_Z: return P->z;
    case RVK_VEC_P0: return P->p[0];
    case RVK_VEC_P1: return P->p[1];
    case RVK_VEC_W: return P->w;
    }
    return nullptr;
}

rvk_status rvk_cg_plan_create_stencil(rvk_ctx ctx, int dim, int points, int64_t nx, int64_t ny,
                                      int64_t nz, rvk_cg_config cfg, rvk_cg_plan* out)
{
    if (!ctx || !out) return set_error(RVK_ERR_INVALID, "cg_plan_create_stencil: null argument");
    RVK_TRACE_TASK(ctx, "cg.plan_create_stencil");
    *out = nullptr;
    if (dim == 2) nz = 1;
    int64_t n = 0, nnz = 0;
    RVK_TRY(rvk_laplacian_size(dim, points, nx, ny, nz, &n, &nnz));
    if (cfg.max_it < 1) return set_error(RVK_ERR_INVALID, "cg_solve: max_it must be >= 1");
    if (cfg.pc != RVK_PC_NONE && cfg.pc != RVK_PC_JACOBI)
        return set_error(RVK_ERR_INVALID, "cg_solve: unknown preconditioner %d", cfg.pc);
    if (cfg.mode != RVK_CG_MODE_FUSED && cfg.mode != RVK_CG_MODE_AUTO)
        return set_error(RVK_ERR_UNSUPPORTED, "matrix-free stencil plans run the FUSED mode only");
    auto P        = new rvk_cg_plan_s();
    P->ctx        = ctx;
    P->A          = rvk_csr{n, n, nnz, nullptr, nullptr, nullptr};
    P->cfg        = cfg;
    P->mode       = RVK_CG_MODE_FUSED;
    P->stencil    = true;
    P->geom       = StencilGeom{nx, ny, nz, n, dim, (points == 9 || points == 27) ? 1 : 0,
                          (double)(points - 1)};
    P->dconst     = 1.0 / (double)(points - 1); // == 1/diag, as the CSR path's dinv
    P->mf_grid    = mf_grid(P->geom);
    P->spmv_grid  = sm_count();
    P->upd_grid   = resident_grid(k_cg_update<true, 2>, kUpdThreads, (n + 1) / 2);
    P->xfix_grid  = resident_grid(k_cg_xfix<4>, kUpdThreads, (n + 1) / 2);
    P->setup_grid = resident_grid(k_cg_setup<true, 2>, kUpdThreads, (n + 1) / 2);
    const size_t vb = (size_t)n * sizeof(double);
    cudaError_t  e  = cudaSuccess;
    auto alloc = [&](void** q, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(q, bytes);
    };
    alloc(reinterpret_cast<void**>(&P->dinv), 64); // unused: the diagonal is constant
    alloc(reinterpret_cast<void**>(&P->r), vb + 32);
    alloc(reinterpret_cast<void**>(&P->z), vb + 32);
    alloc(reinterpret_cast<void**>(&P->p[0]), vb + 32);
    alloc(reinterpret_cast<void**>(&P->p[1]), vb + 32);
    set_x_group(P);
    for (int k = 2; k < P->npb; ++k) alloc(reinterpret_cast<void**>(&P->p[k]), vb + 32);
    alloc(reinterpret_cast<void**>(&P->w), vb);
    alloc(reinterpret_cast<void**>(&P->hist), sizeof(double) * (cfg.max_it + 1));
    alloc(reinterpret_cast<void**>(&P->st), sizeof(CgState));
    alloc(reinterpret_cast<void**>(&P->partials), sizeof(double) * 4 * kMaxReduceBlocks);
    alloc(reinterpret_cast<void**>(&P->tickets), 16 * sizeof(unsigned int));
    alloc(reinterpret_cast<void**>(&P->tmp), 16 * sizeof(double));
    cudaStream_t s = ctx->stream;
    if (e == cudaSuccess) e = cudaMemsetAsync(P->tickets, 0, 16 * sizeof(unsigned int), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->p[0], 0, vb, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->p[1], 0, vb, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->st, 0, sizeof(CgState), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->hist, 0, sizeof(double) * (cfg.max_it + 1), s);
    if (e != cudaSuccess) {
        rvk_cg_plan_destroy(P);
        return cuda_error(e, "rvk_cg_plan_create_stencil");
    }
    P->mf_tma = (cfg.opts & RVK_OPT_MF_SIMPLE) ? nullptr : mf_tma_create(P->geom, P->z, P->p, P->npb, P->r);
    P->zv     = virtual_z(P);
    *out = P;
    return RVK_OK;
}

rvk_status rvk_cg_plan_destroy(rvk_cg_plan P)
{
    if (!P) return RVK_OK;
    if (P->ctx) cudaStreamSynchronize(P->ctx->stream);
    destroy_graph(P);
    mf_tma_destroy(P->mf_tma);
    for (auto ev : P->ev) cudaEventDestroy(ev);
    for (auto ev : P->ev_many)
        if (ev) cudaEventDestroy(ev);
    if (P->s_in) cudaStreamDestroy(P->s_in);
    if (P->s_out) cudaStreamDestroy(P->s_out);
    void* bufs[] = {P->dinv, P->r, P->z, P->w, P->hist, P->st,
                    P->partials, P->tickets, P->tmp, P->b_buf, P->x_buf, P->b_buf2,
                    P->x_buf2, P->hist_all, P->st_all, P->gbar, P->ell_buf};
    for (void* b : bufs)
        if (b) cudaFree(b);
    for (double* b : P->p)
        if (b) cudaFree(b);
    delete P;
    return RVK_OK;
}

rvk_status rvk_cg_set_profiling(rvk_cg_plan P, int on)
{
    if (!P) return set_error(RVK_ERR_INVALID, "null plan");
    P->profiling = on != 0;
    if (P->profiling && P->ev.empty()) {
        P->ev.resize(4 * (size_t)P->cfg.max_it);
        for (auto& ev : P->ev) RVK_CUDA(cudaEventCreate(&ev));
    }
    return RVK_OK;
}

rvk_status rvk_cg_solve_dev(rvk_cg_plan P, const double* b, double* x)
{
    if (!P) return set_error(RVK_ERR_INVALID, "null plan");
    if (!b || !x) return set_error(RVK_ERR_INVALID, "cg_solve: null vector");
    if (b == x) return set_error(RVK_ERR_INVALID, "cg_solve: b and x must not alias");
    RVK_TRACE_TASK(P->ctx, "cg.solve");
    cudaStream_t s = P->ctx->stream;
    if (P->mode == RVK_CG_MODE_HOSTSYNC) return solve_hostsync(P, b, x);
    // one cooperative launch needs no graph
    if (!P->cfg.use_graph || P->mode == RVK_CG_MODE_PERSISTENT) return enqueue_solve(P, b, x);
    const int kind = (P->cfg.use_graph == 2 && P->mode == RVK_CG_MODE_FUSED) ? 2 : 1;
    for (auto& g : P->gs)
        if (g.exec && g.b == b && g.x == x && g.kind == kind && (kind == 2 || g.prof == P->profiling)) {
            P->launches = g.launches;
            RVK_CUDA(cudaGraphLaunch(g.exec, s));
            return RVK_OK;
        }
    auto& slot = P->gs[P->g_victim];
    P->g_victim ^= 1;
    if (slot.exec) cudaGraphExecDestroy(slot.exec);
    slot = rvk_cg_plan_s::GraphSlot{};
    if (kind == 2) { // device WHILE loop
        RVK_TRY(build_while_graph(P, b, x, &slot.exec));
        P->launches = -1; // data-dependent: 3 + 4 per body pass
    } else {
        cudaGraph_t g = nullptr;
        // Thread-local capture mode: ANY synchronous CUDA call this thread
        // makes while the solve is being enqueued invalidates the capture --
        // a structural proof that the solve performs zero host
        // synchronisations.  (Thread-local, not global: a global capture is
        // invalidated by other host threads' allocations, which breaks one
        // process driving several GPUs from several threads.)
        RVK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        rvk_status rc = enqueue_solve(P, b, x);
        cudaError_t e = cudaStreamEndCapture(s, &g);
        if (rc != RVK_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) return cuda_error(e, "cudaStreamEndCapture (solve not capturable)");
        e = cudaGraphInstantiate(&slot.exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            slot.exec = nullptr;
            return cuda_error(e, "cudaGraphInstantiate");
        }
    }
    slot.b        = b;
    slot.x        = x;
    slot.prof     = P->profiling;
    slot.kind     = kind;
    slot.launches = P->launches;
    RVK_CUDA(cudaGraphLaunch(slot.exec, s));
    return RVK_OK;
}

const double* rvk_cg_history_dev(rvk_cg_plan P) { return P ? P->hist : nullptr; }

int rvk_cg_plan_mode(rvk_cg_plan P) { return P ? P->mode : -1; }

rvk_status rvk_cg_result(rvk_cg_plan P, double* hist_host, rvk_cg_info* info)
{
    if (!P) return set_error(RVK_ERR_INVALID, "null plan");
    CgState      h{};
    cudaStream_t s = P->ctx->stream;
    RVK_CUDA(cudaMemcpyAsync(&h, P->st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
    if (hist_host)
        RVK_CUDA(cudaMemcpyAsync(hist_host, P->hist, sizeof(double) * (P->cfg.max_it + 1),
                                 cudaMemcpyDeviceToHost, s));
    {
        trace::HostSyncScope hs_("rvk_cg_result");
        RVK_CUDA(cudaStreamSynchronize(s));
    }
    if (info) {
        info->state          = h.state;
        info->iterations     = h.iterations;
        info->breakdown_iter = h.breakdown_iter;
    }
    if (h.state == RVK_CG_BREAKDOWN)
        return set_error(RVK_ERR_BREAKDOWN, "cg_solve: breakdown at iteration %d",
                         h.breakdown_iter);
    return RVK_OK;
}

rvk_status rvk_cg_solve_host(rvk_cg_plan P, const double* b_host, double* x_host,
                             double* hist_host, rvk_cg_info* info)
{
    if (!P || !b_host || !x_host) return set_error(RVK_ERR_INVALID, "null argument");
    RVK_TRACE_TASK(P->ctx, "cg.solve_host");
    const size_t vb = (size_t)P->A.n_rows * sizeof(double);
    if (!P->b_buf) RVK_CUDA(cudaMalloc(&P->b_buf, vb));
    if (!P->x_buf) RVK_CUDA(cudaMalloc(&P->x_buf, vb));
    cudaStream_t s = P->ctx->stream;
    RVK_CUDA(cudaMemcpyAsync(P->b_buf, b_host, vb, cudaMemcpyHostToDevice, s));
    RVK_TRY(rvk_cg_solve_dev(P, P->b_buf, P->x_buf));
    RVK_CUDA(cudaMemcpyAsync(x_host, P->x_buf, vb, cudaMemcpyDeviceToHost, s));
    return rvk_cg_result(P, hist_host, info);
}

// Many right-hand sides from host memory, pipelined (PETSc KSPMatSolve-like
// usage: a stream of independent solves with the same operator).  Two device
// staging pairs and two copy streams: the H2D of b[k+1] and the D2H of x[k-1]
// run on the copy engines while solve k runs on the plan's stream, so with
// PINNED host buffers a step costs max(H2D, solve, D2H) instead of their sum.
// Every step's copies still happen (nothing is cached); per-RHS histories and
// states are kept on the device and read back once at the end (one sync).
rvk_status rvk_cg_solve_host_many(rvk_cg_plan P, int nrhs, const double* const* b_host,
                                  double* const* x_host, double* hist_host, rvk_cg_info* infos)
{
    if (!P || nrhs < 0 || (nrhs && (!b_host || !x_host)))
        return set_error(RVK_ERR_INVALID, "null argument");
    if (nrhs == 0) return RVK_OK;
    RVK_TRACE_TASK(P->ctx, "cg.solve_host_many");
    const size_t vb = (size_t)P->A.n_rows * sizeof(double);
    const int    H  = P->cfg.max_it + 1;
    cudaStream_t s  = P->ctx->stream;
    if (!P->b_buf) RVK_CUDA(cudaMalloc(&P->b_buf, vb));
    if (!P->x_buf) RVK_CUDA(cudaMalloc(&P->x_buf, vb));
    if (!P->b_buf2) RVK_CUDA(cudaMalloc(&P->b_buf2, vb));
    if (!P->x_buf2) RVK_CUDA(cudaMalloc(&P->x_buf2, vb));
    if (!P->s_in) RVK_CUDA(cudaStreamCreateWithFlags(&P->s_in, cudaStreamNonBlocking));
    if (!P->s_out) RVK_CUDA(cudaStreamCreateWithFlags(&P->s_out, cudaStreamNonBlocking));
    for (auto& ev : P->ev_many)
        if (!ev) RVK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (P->cap_many < nrhs) {
        RVK_CUDA(cudaStreamSynchronize(s));
        if (P->hist_all) cudaFree(P->hist_all);
        if (P->st_all) cudaFree(P->st_all);
        P->hist_all = nullptr;
        P->st_all   = nullptr;
        P->cap_many = 0;
        RVK_CUDA(cudaMalloc(&P->hist_all, (size_t)nrhs * H * sizeof(double)));
        RVK_CUDA(cudaMalloc(&P->st_all, (size_t)nrhs * sizeof(CgState)));
        P->cap_many = nrhs;
    }
    double*      bd[2] = {P->b_buf, P->b_buf2};
    double*      xd[2] = {P->x_buf, P->x_buf2};
    cudaEvent_t* b_ready = P->ev_many, *solved = P->ev_many + 2, *x_free = P->ev_many + 4,
               * b_free = P->ev_many + 6;
    // order the pipeline after everything already queued on the plan's stream
    RVK_CUDA(cudaEventRecord(solved[0], s));
    RVK_CUDA(cudaStreamWaitEvent(P->s_in, solved[0], 0));
    RVK_CUDA(cudaStreamWaitEvent(P->s_out, solved[0], 0));
    for (int k = 0; k < nrhs; ++k) {
        const int j = k & 1;
        if (k >= 2) RVK_CUDA(cudaStreamWaitEvent(P->s_in, b_free[j], 0)); // solve k-2 read bd[j]
        RVK_CUDA(cudaMemcpyAsync(bd[j], b_host[k], vb, cudaMemcpyHostToDevice, P->s_in));
        RVK_CUDA(cudaEventRecord(b_ready[j], P->s_in));
        RVK_CUDA(cudaStreamWaitEvent(s, b_ready[j], 0));
        if (k >= 2) RVK_CUDA(cudaStreamWaitEvent(s, x_free[j], 0));       // x[k-2] left xd[j]
        RVK_TRY(rvk_cg_solve_dev(P, bd[j], xd[j]));
        RVK_CUDA(cudaEventRecord(b_free[j], s));
        RVK_CUDA(cudaMemcpyAsync(P->hist_all + (size_t)k * H, P->hist, H * sizeof(double),
                                 cudaMemcpyDeviceToDevice, s));
        RVK_CUDA(cudaMemcpyAsync(P->st_all + k, P->st, sizeof(CgState), cudaMemcpyDeviceToDevice, s));
        RVK_CUDA(cudaEventRecord(solved[j], s));
        RVK_CUDA(cudaStreamWaitEvent(P->s_out, solved[j], 0));
        RVK_CUDA(cudaMemcpyAsync(x_host[k], xd[j], vb, cudaMemcpyDeviceToHost, P->s_out));
        RVK_CUDA(cudaEventRecord(x_free[j], P->s_out));
    }
    // the plan's stream owns completion: later work (and the sync below) sees x on the host
    RVK_CUDA(cudaStreamWaitEvent(s, x_free[(nrhs - 1) & 1], 0));
    if (nrhs >= 2) RVK_CUDA(cudaStreamWaitEvent(s, x_free[nrhs & 1], 0));
    std::vector<CgState> st(nrhs);
    if (hist_host)
        RVK_CUDA(cudaMemcpyAsync(hist_host, P->hist_all, (size_t)nrhs * H * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
    RVK_CUDA(cudaMemcpyAsync(st.data(), P->st_all, nrhs * sizeof(CgState), cudaMemcpyDeviceToHost, s));
    {
        trace::HostSyncScope hs_("rvk_cg_solve_host_many");
        RVK_CUDA(cudaStreamSynchronize(s));
    }
    int broke = -1;
    for (int k = 0; k < nrhs; ++k) {
        if (infos) {
            infos[k].state          = st[k].state;
            infos[k].iterations     = st[k].iterations;
            infos[k].breakdown_iter = st[k].breakdown_iter;
        }
        if (st[k].state == RVK_CG_BREAKDOWN && broke < 0) broke = k;
    }
    if (broke >= 0)
        return set_error(RVK_ERR_BREAKDOWN, "cg_solve: right-hand side %d broke down at iteration %d",
                         broke, st[broke].breakdown_iter);
    return RVK_OK;
}

rvk_status rvk_cg_kernel_times(rvk_cg_plan P, float* spmv_ms, float* update_ms, int* launches)
{
    if (!P) return set_error(RVK_ERR_INVALID, "null plan");
    if (launches) *launches = P->launches;
    if (!P->profiling || P->ev.empty()) return set_error(RVK_ERR_INVALID, "profiling is off");
    float a = 0.f, b = 0.f;
    for (int it = 0; it < P->cfg.max_it; ++it) {
        float t1 = 0.f, t2 = 0.f;
        RVK_CUDA(cudaEventElapsedTime(&t1, P->ev[4 * it + 0], P->ev[4 * it + 1]));
        RVK_CUDA(cudaEventElapsedTime(&t2, P->ev[4 * it + 2], P->ev[4 * it + 3]));
        a += t1;
        b += t2;
    }
    if (spmv_ms) *spmv_ms = a;
    if (update_ms) *update_ms = b;
    return RVK_OK;
}

} // extern "C"
