// rvk_tfqmr.cu -- left-Jacobi TFQMR on sm_100a (SPEC.md
// :467-475; "two matrix-vector products and roughly twice
// the number of vector inner products").
//
// Same recurrence and operation order as oracle/rvk_oracle.c:ro_tfqmr_solve
// (PETSc KSPSolve_TFQMR order); the scalar recurrence (a, psi, cm, tau, eta,
// cf, b) is device-resident, so the solve is stream-ordered with ZERO host
// syncs and captured as one CUDA graph.  A device `done` flag (convergence /
// breakdown) turns every later kernel of the solve into a no-op.  Elementwise
// results are bit-identical to the oracle's; the three reductions per
// iteration use tree order (SPEC's TFQMR tolerance is 1e-8).
//
// FUSED (default): three kernels per outer iteration.
//   KA  SpMV over t = u + q formed on the fly from gathered u, v (q = u - a v):
//       q, r -= a B A t written by the row owner; ||r||^2 and (r, rp) fused;
//       the tail runs both half steps' scalars, the convergence tests and b.
//   KM  elementwise: d, x for the half steps that ran; u, q, p for the next
//       iteration (skipped in the last one).
//   KB  SpMV over p: v = B A p and (v, rp); the tail forms a for the next
//       iteration (not launched after the last one).
// Per iteration HBM bytes: 2 CSR passes + 22 n doubles (KA 7, KM 11, KB 4).
// UNFUSED: the reference's op-per-kernel sequence over the Vec/SpMV kernels.
#include "rvk_cg.cuh"
#include "rvk_common.cuh"
#include "rvk_context.hpp"
#include "rvk_internal.hpp"
#include "rvk_spmv.cuh"

#include <cmath>
#include <cstdlib>
#include <vector>

namespace rvk {

struct TfqState {
    double rhoold, rho, s, a, b, dp, dpold, tau, etaold, psiold, eta, psi, cf, dp0;
    double cf0, eta0, cf1, eta1; // fused: the two half steps of the current iteration
    int    done, state, iterations, breakdown_iter, nhist;
    int    done_it, halves;      // fused: iteration that finished, half steps it ran
};

namespace {

__device__ __forceinline__ bool tfq_conv(double v, double dp0, double rtol, double atol)
{
    return v <= fmax(rtol * dp0, atol);
}

// after dp = ||R0|| and rho = (R0, RP): hist[0], initial scalars
__global__ void k_tfq_init(TfqState* st, double* hist, double rtol, double atol)
{
    const double dp    = st->dp;
    hist[0]            = dp;
    st->dp0            = dp;
    st->nhist          = 1;
    st->iterations     = 0;
    st->breakdown_iter = -1;
    st->etaold         = 0.0;
    st->psiold         = 0.0;
    st->tau            = dp;
    st->dpold          = dp;
    st->rhoold         = st->rho;
    const bool conv    = tfq_conv(dp, dp, rtol, atol);
    st->state          = conv ? RVK_CG_CONVERGED : RVK_CG_RUNNING;
    st->done           = conv ? 1 : 0;
}

// a = rho_old / s with s = (V, RP); serious breakdown when s == 0
__global__ void k_tfq_alpha(TfqState* st, int it)
{
    if (st->done) return;
    if (st->s == 0.0) {
        st->state          = RVK_CG_BREAKDOWN;
        st->breakdown_iter = it;
        st->done           = 1;
        return;
    }
    st->a = st->rhoold / st->s;
}

// half step m, before the D / X updates: w, psi, cm, tau, eta, cf
__global__ void k_tfq_half(TfqState* st, int m)
{
    if (st->done) return;
    const double w   = m == 0 ? sqrt(__dmul_rn(st->dp, st->dpold)) : st->dp;
    const double psi = w / st->tau;
    const double cm  = 1.0 / sqrt(__dadd_rn(1.0, __dmul_rn(psi, psi)));
    st->tau          = __dmul_rn(__dmul_rn(st->tau, psi), cm);
    st->eta          = __dmul_rn(__dmul_rn(cm, cm), st->a);
    st->cf           = __dmul_rn(__dmul_rn(st->psiold, st->psiold), st->etaold) / st->a;
    st->psi          = psi;
}

// after X += eta D: quasi-residual estimate, convergence, shift eta/psi
__global__ void k_tfq_post(TfqState* st, double* hist, int m, int it, double rtol, double atol)
{
    if (st->done) return;
    const double dpest = __dmul_rn(sqrt(2.0 * it + m + 2.0), st->tau); // ||r_k|| <= sqrt(k+1) tau
    hist[st->nhist++]  = dpest;
    if (tfq_conv(dpest, st->dp0, rtol, atol)) {
        st->state      = RVK_CG_CONVERGED;
        st->iterations = it + 1;
        st->done       = 1;
        return;
    }
    st->etaold = st->eta;
    st->psiold = st->psi;
}

// b = rho / rho_old (rho = (R, RP)); breakdown when rho_old == 0
__global__ void k_tfq_beta(TfqState* st, int it)
{
    if (st->done) return;
    st->iterations = it + 1;
    if (st->rhoold == 0.0) {
        st->state          = RVK_CG_BREAKDOWN;
        st->breakdown_iter = it;
        st->done           = 1;
        return;
    }
    st->b = st->rho / st->rhoold;
}

__global__ void k_tfq_shift(TfqState* st)
{
    if (st->done) return;
    st->rhoold = st->rho;
    st->dpold  = st->dp;
}

__global__ void k_tfq_copy(int64_t n, const double* __restrict__ src, double* __restrict__ dst,
                           const int* guard)
{
    if (guard && *guard) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

// ===========================================================================
// FUSED path
// ===========================================================================
constexpr int kTfqThreads = 256;

// scalar recurrence of one half step (the oracle's loop body), shared by the
// fused tail; returns true when the bound converged
__device__ __forceinline__ bool tfq_half_step(TfqState* st, double* hist, int m, int it, double rtol,
                                              double atol, double& cf, double& eta)
{
    const double w   = m == 0 ? sqrt(__dmul_rn(st->dp, st->dpold)) : st->dp;
    const double psi = w / st->tau;
    const double cm  = 1.0 / sqrt(__dadd_rn(1.0, __dmul_rn(psi, psi)));
    st->tau          = __dmul_rn(__dmul_rn(st->tau, psi), cm);
    eta              = __dmul_rn(__dmul_rn(cm, cm), st->a);
    cf               = __dmul_rn(__dmul_rn(st->psiold, st->psiold), st->etaold) / st->a;
    const double dpest = __dmul_rn(sqrt(2.0 * it + m + 2.0), st->tau);
    hist[st->nhist++]  = dpest;
    if (tfq_conv(dpest, st->dp0, rtol, atol)) return true;
    st->etaold = eta;
    st->psiold = psi;
    return false;
}

// done_it: the iteration whose KM still has to apply `halves` half steps
// (-1: nothing pending)
__device__ __forceinline__ void tfq_finish(TfqState* st, int state, int it, int done_it, int halves)
{
    st->state   = state;
    st->done    = 1;
    st->done_it = done_it;
    st->halves  = halves;
    if (state == RVK_CG_BREAKDOWN) st->breakdown_iter = it;
}

// K0: r = B b; rp = u = p = r; d = x = 0; ||r||^2 (= (r, rp)); initial scalars.
// PC: 0 no preconditioner, 1 dinv vector, 2 constant diagonal dc (every
// dinv[i] the same bit pattern: the scalar gives bit-identical products and
// the dinv stream disappears from K0, KA and KB)
template <bool VEC, int PC>
__global__ void __launch_bounds__(kTfqThreads)
    k_tfq_setup(int64_t n, const double* __restrict__ b, const double* __restrict__ dinv, double dc,
                double* __restrict__ R, double* __restrict__ RP, double* __restrict__ U,
                double* __restrict__ P, double* __restrict__ D, double* __restrict__ X, TfqState* st,
                double* hist, double rtol, double atol, double* partials, unsigned int* ticket)
{
    __shared__ double smem[32];
    __shared__ int    flag;
    double            acc[1] = {0.0};
    const int64_t     stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t     t0     = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (VEC) {
        for (int64_t i = t0; i < (n >> 1); i += stride) {
            const double2 bi = ld_stream(reinterpret_cast<const double2*>(b) + i);
            double2       r  = bi;
            if (PC) {
                const double2 d = PC == 1 ? ld_stream(reinterpret_cast<const double2*>(dinv) + i)
                                          : make_double2(dc, dc);
                r.x             = mul(d.x, bi.x);
                r.y             = mul(d.y, bi.y);
            }
            reinterpret_cast<double2*>(R)[i]  = r;
            reinterpret_cast<double2*>(RP)[i] = r;
            reinterpret_cast<double2*>(U)[i]  = r;
            reinterpret_cast<double2*>(P)[i]  = r;
            reinterpret_cast<double2*>(D)[i]  = make_double2(0.0, 0.0);
            st_stream(reinterpret_cast<double2*>(X) + i, make_double2(0.0, 0.0));
            acc[0] = add(acc[0], mul(r.x, r.x));
            acc[0] = add(acc[0], mul(r.y, r.y));
        }
    }
    for (int64_t i = (VEC ? (n & ~int64_t(1)) : 0) + t0; i < n; i += stride) {
        const double r = PC ? mul(PC == 1 ? dinv[i] : dc, b[i]) : b[i];
        R[i] = RP[i] = U[i] = P[i] = r;
        D[i] = X[i] = 0.0;
        acc[0]      = add(acc[0], mul(r, r));
    }
    const int tid = threadIdx.x;
    block_sum<1>(acc, smem, tid, blockDim.x, 1);
    if (tid == 0) partials[blockIdx.x] = acc[0];
    if (!last_block(ticket, tid, &flag, blockDim.x, 1)) return;
    fold_partials<1>(partials, gridDim.x, acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        const double dp    = sqrt(acc[0]);
        hist[0]            = dp;
        st->dp = st->dp0 = st->tau = st->dpold = dp;
        st->rho = st->rhoold = acc[0]; // (r, rp) with rp = r: the same products
        st->etaold = st->psiold = 0.0;
        st->nhist          = 1;
        st->iterations     = 0;
        st->breakdown_iter = -1;
        st->done_it        = -1;
        st->halves         = 0;
        const bool conv    = tfq_conv(dp, dp, rtol, atol);
        st->state          = conv ? RVK_CG_CONVERGED : RVK_CG_RUNNING;
        st->done           = conv ? 1 : 0;
        *ticket            = 0u;
    }
}

// KA op: t = u + (u - a v) on the fly, q and r written by the row owner,
// sums ||r||^2 and (r, rp); tail = the iteration's scalar recurrence.
template <int PC>
struct TfqAOp {
    static constexpr bool kHasTail = true;
    static constexpr bool kNoSmall = true; // TFQMR plans never take the small-system K1
    static constexpr int  kSums    = 2;
    const double* __restrict__ u;
    const double* __restrict__ v;
    const double* __restrict__ rp;
    const double* __restrict__ dinv;
    double* __restrict__ q;
    double* __restrict__ r;
    TfqState* st;
    double*   hist;
    double    rtol, atol;
    int       it;
    double    na; // -a, set by init()
    double    dc; // PC 2: the constant diagonal

    __device__ __forceinline__ bool init()
    {
        if (st->done) return false;
        na = -st->a;
        return true;
    }
    struct Fetch {
        double u, v;
    };
    __device__ __forceinline__ int           num_src() const { return 2; }
    __device__ __forceinline__ const double* src_ptr(int k) const { return k == 0 ? u : v; }
    __device__ __forceinline__ Fetch         fetch(int32_t j) const
    {
        return Fetch{__ldg(u + j), __ldg(v + j)};
    }
    // t = 1 u + q, q = (-a) v + u  (VecWAXPY twice, kernels_scalar.cpp:36-40)
    __device__ __forceinline__ double value(const Fetch& f) const
    {
        return add(f.u, add(mul(na, f.v), f.u));
    }
    __device__ __forceinline__ int64_t own_col(int64_t i) const { return i; }
    struct Own {
        double u, v, r, rp, d;
    };
    __device__ __forceinline__ Own own(int64_t i) const
    {
        return Own{__ldg(u + i), __ldg(v + i), r[i], __ldg(rp + i),
                   PC == 1 ? __ldg(dinv + i) : (PC == 2 ? dc : 1.0)};
    }
    __device__ __forceinline__ SumVec<2> row(int64_t i, double sum, SumVec<2> acc, const Own& o) const
    {
        q[i]            = add(mul(na, o.v), o.u);
        const double bt = PC ? mul(o.d, sum) : sum;   // B A t
        const double ri = add(o.r, mul(na, bt));      // r += (-a) B A t
        r[i]            = ri;
        acc.v[0]        = add(acc.v[0], mul(ri, ri));
        acc.v[1]        = add(acc.v[1], mul(ri, o.rp));
        return acc;
    }
    __device__ __forceinline__ void tail(const double (&v)[2]) const
    {
        st->dp  = sqrt(v[0]);
        st->rho = v[1];
        if (tfq_half_step(st, hist, 0, it, rtol, atol, st->cf0, st->eta0)) {
            st->iterations = it + 1;
            tfq_finish(st, RVK_CG_CONVERGED, it, it, 1);
            return;
        }
        if (tfq_half_step(st, hist, 1, it, rtol, atol, st->cf1, st->eta1)) {
            st->iterations = it + 1;
            tfq_finish(st, RVK_CG_CONVERGED, it, it, 2);
            return;
        }
        st->iterations = it + 1;
        if (st->rhoold == 0.0) {
            tfq_finish(st, RVK_CG_BREAKDOWN, it, it, 2);
            return;
        }
        st->b = st->rho / st->rhoold;
    }
};

// KB op: v = B A p, (v, rp); tail: rho_old = rho, dp_old = dp, a = rho_old / s.
// `it` = the iteration the new a belongs to (0 for the setup launch).
template <int PC>
struct TfqBOp {
    static constexpr bool kHasTail = true;
    static constexpr bool kNoSmall = true;
    const double* __restrict__ p;
    const double* __restrict__ rp;
    const double* __restrict__ dinv;
    double* __restrict__ v;
    TfqState* st;
    int       it;
    double    dc; // PC 2: the constant diagonal

    __device__ __forceinline__ bool init() { return st->done == 0; }
    struct Fetch {
        double p;
    };
    __device__ __forceinline__ int           num_src() const { return 1; }
    __device__ __forceinline__ const double* src_ptr(int) const { return p; }
    __device__ __forceinline__ Fetch         fetch(int32_t j) const { return Fetch{__ldg(p + j)}; }
    __device__ __forceinline__ double  value(const Fetch& f) const { return f.p; }
    __device__ __forceinline__ int64_t own_col(int64_t i) const { return i; }
    struct Own {
        double rp, d;
    };
    __device__ __forceinline__ Own own(int64_t i) const
    {
        return Own{__ldg(rp + i), PC == 1 ? __ldg(dinv + i) : (PC == 2 ? dc : 1.0)};
    }
    __device__ __forceinline__ double row(int64_t i, double sum, double acc, const Own& o) const
    {
        const double vi = PC ? mul(o.d, sum) : sum;
        v[i]            = vi;
        return add(acc, mul(vi, o.rp));
    }
    __device__ __forceinline__ void tail(double s) const
    {
        st->rhoold = st->rho;
        st->dpold  = st->dp;
        st->s      = s;
        if (s == 0.0) {
            tfq_finish(st, RVK_CG_BREAKDOWN, it, -1, 0);
            return;
        }
        st->a = st->rhoold / s;
    }
};

// KM: the half steps' d / x updates that ran in iteration `it`, then (unless
// the solve finished or this is the last iteration) u, q, p for the next one.
template <bool VEC>
__global__ void __launch_bounds__(kTfqThreads)
    k_tfq_merge(int64_t n, double* __restrict__ U, double* __restrict__ Q, const double* __restrict__ R,
                double* __restrict__ P, double* __restrict__ D, double* __restrict__ X,
                const TfqState* st, int it, int last)
{
    const int done = st->done;
    if (done && st->done_it != it) return;
    const int    halves = done ? st->halves : 2;
    const bool   upd    = !done && !last;
    const double cf0 = st->cf0, eta0 = st->eta0, cf1 = st->cf1, eta1 = st->eta1, b = st->b;
    auto one = [&](double& u, double& q, double r, double& p, double& d, double& x) {
        d = add(u, mul(cf0, d)); // VecAYPX(D, cf, U)
        x = add(x, mul(eta0, d)); // VecAXPY(X, eta, D)
        if (halves == 2) {
            d = add(q, mul(cf1, d));
            x = add(x, mul(eta1, d));
        }
        if (upd) {
            u = add(mul(b, q), r); // VecWAXPY(U, b, Q, R)
            q = add(q, mul(b, p)); // VecAXPY(Q, b, P)
            p = add(mul(b, q), u); // VecWAXPY(P, b, Q, U)
        }
    };
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0     = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (VEC) {
        for (int64_t i = t0; i < (n >> 1); i += stride) {
            double2       u = reinterpret_cast<double2*>(U)[i], q = reinterpret_cast<double2*>(Q)[i];
            const double2 r = upd ? ld_stream(reinterpret_cast<const double2*>(R) + i) : make_double2(0, 0);
            double2       p = upd ? reinterpret_cast<double2*>(P)[i] : make_double2(0, 0);
            double2       d = reinterpret_cast<double2*>(D)[i], x = reinterpret_cast<double2*>(X)[i];
            one(u.x, q.x, r.x, p.x, d.x, x.x);
            one(u.y, q.y, r.y, p.y, d.y, x.y);
            reinterpret_cast<double2*>(D)[i] = d;
            reinterpret_cast<double2*>(X)[i] = x;
            if (upd) {
                reinterpret_cast<double2*>(U)[i] = u;
                reinterpret_cast<double2*>(Q)[i] = q;
                reinterpret_cast<double2*>(P)[i] = p;
            }
        }
    }
    for (int64_t i = (VEC ? (n & ~int64_t(1)) : 0) + t0; i < n; i += stride) {
        double u = U[i], q = Q[i], p = upd ? P[i] : 0.0, d = D[i], x = X[i];
        one(u, q, upd ? R[i] : 0.0, p, d, x);
        D[i] = d;
        X[i] = x;
        if (upd) {
            U[i] = u;
            Q[i] = q;
            P[i] = p;
        }
    }
}

} // namespace

// Distinct op type: k_spmv_tma<TfqSpmvOp> is this file's own instantiation
// (no template kernel shared across non-rdc translation units).
struct TfqSpmvOp : SpmvGuardedOp {};

} // namespace rvk

using namespace rvk;

struct rvk_tfqmr_plan_s {
    rvk_ctx       ctx = nullptr;
    rvk_csr       A{};
    rvk_cg_config cfg{};
    SpmvArgs      sa{};
    double *R = nullptr, *RP = nullptr, *U = nullptr, *P = nullptr, *V = nullptr, *D = nullptr;
    double *Q = nullptr, *T = nullptr, *AUQ = nullptr, *T1 = nullptr, *dinv = nullptr;
    double*         hist = nullptr;
    TfqState*       st = nullptr;
    double*         partials = nullptr;
    unsigned int*   tickets = nullptr;
    cudaGraphExec_t graph = nullptr;
    const double*   g_b = nullptr;
    double*         g_x = nullptr;
    bool            fused    = true;
    int             upd_grid = 1; // resident grid of the streaming kernels (K0, KM)
    bool            const_diag = false; // fused: dinv is one value, dconst
    double          dconst     = 0.0;
};

namespace {

#define RVK_TRY(x)                                                                             \
    do {                                                                                       \
        rvk_status rc_ = (x);                                                                  \
        if (rc_ != RVK_OK) return rc_;                                                         \
    } while (0)

rvk_scalar sptr(const double* p, int kind = RVK_SCALAR_PTR)
{
    return rvk_scalar{kind, 0.0, p, nullptr};
}

int copy_grid(int64_t n)
{
    const int64_t want = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * 8));
}

// out = B A v: T1 = A v, out = dinv .* T1 (no PC: the SpMV writes `out`)
rvk_status apply_BA(rvk_tfqmr_plan P, const double* v, double* out, const int* g)
{
    cudaStream_t  s   = P->ctx->stream;
    const bool    jac = P->cfg.pc == RVK_PC_JACOBI;
    TfqSpmvOp     op;
    op.x     = v;
    op.y     = jac ? P->T1 : out;
    op.guard = g;
    RVK_TRY(launch_spmv(s, P->sa, op, TailArgs{nullptr, nullptr}, sm_count()));
    if (jac) RVK_TRY(vec_ew(s, EW_PMULT, P->A.n_rows, const_scalar(0), P->dinv, P->T1, out, g));
    return RVK_OK;
}

template <int PC>
rvk_status enqueue_fused_t(rvk_tfqmr_plan P, const double* b, double* x)
{
    const int64_t  n    = P->A.n_rows;
    cudaStream_t   s    = P->ctx->stream;
    TfqState*      st   = P->st;
    const double   rtol = P->cfg.rtol, atol = P->cfg.atol;
    const bool     vec  = ((reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(x)) & 15) == 0;
    const int      sg   = sm_count();
    // partial / ticket slots: K0 + KM-free, KA (2 sums), KB (1 sum) -- each
    // kernel re-arms its own ticket, consecutive kernels use different slots
    const TailArgs ta{P->partials, P->tickets + 1};
    const TailArgs tb{P->partials + 2 * kMaxReduceBlocks, P->tickets + 2};
    if (vec)
        k_tfq_setup<true, PC><<<P->upd_grid, kTfqThreads, 0, s>>>(
            n, b, P->dinv, P->dconst, P->R, P->RP, P->U, P->P, P->D, x, st, P->hist, rtol, atol, P->partials,
            P->tickets);
    else
        k_tfq_setup<false, PC><<<P->upd_grid, kTfqThreads, 0, s>>>(
            n, b, P->dinv, P->dconst, P->R, P->RP, P->U, P->P, P->D, x, st, P->hist, rtol, atol, P->partials,
            P->tickets);
    RVK_CHECK_LAUNCH("k_tfq_setup");
    RVK_TRY(launch_spmv(s, P->sa, TfqBOp<PC>{P->P, P->RP, P->dinv, P->V, st, 0, P->dconst}, tb, sg));
    for (int it = 0; it < P->cfg.max_it; ++it) {
        const bool last = it + 1 == P->cfg.max_it;
        TfqAOp<PC> a{P->U, P->V, P->RP, P->dinv, P->Q, P->R, st, P->hist, rtol, atol, it, 0.0, P->dconst};
        RVK_TRY(launch_spmv(s, P->sa, a, ta, sg));
        if (vec)
            k_tfq_merge<true><<<P->upd_grid, kTfqThreads, 0, s>>>(n, P->U, P->Q, P->R, P->P, P->D, x,
                                                                  st, it, last);
        else
            k_tfq_merge<false><<<P->upd_grid, kTfqThreads, 0, s>>>(n, P->U, P->Q, P->R, P->P, P->D,
                                                                   x, st, it, last);
        RVK_CHECK_LAUNCH("k_tfq_merge");
        if (!last)
            RVK_TRY(launch_spmv(s, P->sa, TfqBOp<PC>{P->P, P->RP, P->dinv, P->V, st, it + 1, P->dconst}, tb, sg));
    }
    return RVK_OK;
}

rvk_status enqueue_tfqmr(rvk_tfqmr_plan P, const double* b, double* x)
{
    if (P->fused)
        return P->cfg.pc != RVK_PC_JACOBI ? enqueue_fused_t<0>(P, b, x)
               : P->const_diag            ? enqueue_fused_t<2>(P, b, x)
                                          : enqueue_fused_t<1>(P, b, x);
    const int64_t n   = P->A.n_rows;
    cudaStream_t  s   = P->ctx->stream;
    const bool    jac = P->cfg.pc == RVK_PC_JACOBI;
    Scratch       sc{P->partials, P->tickets};
    TfqState*     st  = P->st;
    const int*    g   = &st->done;
    const double  rtol = P->cfg.rtol, atol = P->cfg.atol;
    const int     cg  = copy_grid(n);

    // setup: x = 0, R = B b, dp = ||R||, RP = R, rho = (R, RP), U = P = R, V = B A P, D = 0
    RVK_CUDA(cudaMemsetAsync(x, 0, n * 8, s));
    if (jac) RVK_TRY(vec_ew(s, EW_PMULT, n, const_scalar(0), P->dinv, b, P->R, nullptr));
    else RVK_CUDA(cudaMemcpyAsync(P->R, b, n * 8, cudaMemcpyDeviceToDevice, s));
    RVK_TRY(vec_reduce(s, sc, RED_NRM2, n, P->R, nullptr, &st->dp, nullptr, nullptr));
    RVK_CUDA(cudaMemcpyAsync(P->RP, P->R, n * 8, cudaMemcpyDeviceToDevice, s));
    RVK_TRY(vec_reduce(s, sc, RED_DOT, n, P->R, P->RP, &st->rho, nullptr, nullptr));
    k_tfq_init<<<1, 1, 0, s>>>(st, P->hist, rtol, atol);
    RVK_CHECK_LAUNCH("k_tfq_init");
    k_tfq_copy<<<cg, 256, 0, s>>>(n, P->R, P->U, g);
    k_tfq_copy<<<cg, 256, 0, s>>>(n, P->R, P->P, g);
    RVK_TRY(apply_BA(P, P->P, P->V, g));
    RVK_CUDA(cudaMemsetAsync(P->D, 0, n * 8, s));

    for (int it = 0; it < P->cfg.max_it; ++it) {
        RVK_TRY(vec_reduce(s, sc, RED_DOT, n, P->V, P->RP, &st->s, nullptr, g));        // s = (v, rp)
        k_tfq_alpha<<<1, 1, 0, s>>>(st, it);                                              // a = rho/s
        RVK_TRY(vec_ew(s, EW_WAXPY, n, sptr(&st->a, RVK_SCALAR_NEG_PTR), P->V, P->U, P->Q, g)); // q = u - a v
        RVK_TRY(vec_ew(s, EW_WAXPY, n, const_scalar(1.0), P->U, P->Q, P->T, g));          // t = u + q
        RVK_TRY(apply_BA(P, P->T, P->AUQ, g));                                            // B A t
        RVK_TRY(vec_ew(s, EW_AXPY, n, sptr(&st->a, RVK_SCALAR_NEG_PTR), P->AUQ, P->R, P->R, g)); // r -= a BAt
        RVK_TRY(vec_reduce(s, sc, RED_NRM2, n, P->R, nullptr, &st->dp, nullptr, g));      // dp = ||r||
        for (int m = 0; m < 2; ++m) {
            k_tfq_half<<<1, 1, 0, s>>>(st, m);
            RVK_TRY(vec_ew(s, EW_AYPX, n, sptr(&st->cf), m == 0 ? P->U : P->Q, P->D, P->D, g)); // d = (u|q) + cf d
            RVK_TRY(vec_ew(s, EW_AXPY, n, sptr(&st->eta), P->D, x, x, g));                      // x += eta d
            k_tfq_post<<<1, 1, 0, s>>>(st, P->hist, m, it, rtol, atol);
        }
        RVK_TRY(vec_reduce(s, sc, RED_DOT, n, P->R, P->RP, &st->rho, nullptr, g));      // rho = (r, rp)
        k_tfq_beta<<<1, 1, 0, s>>>(st, it);                                               // b = rho/rho_old
        RVK_TRY(vec_ew(s, EW_WAXPY, n, sptr(&st->b), P->Q, P->R, P->U, g));             // u = r + b q
        RVK_TRY(vec_ew(s, EW_AXPY, n, sptr(&st->b), P->P, P->Q, P->Q, g));              // q += b p
        RVK_TRY(vec_ew(s, EW_WAXPY, n, sptr(&st->b), P->Q, P->U, P->P, g));             // p = u + b q
        RVK_TRY(apply_BA(P, P->P, P->V, g));                                              // v = B A p
        k_tfq_shift<<<1, 1, 0, s>>>(st);
        RVK_CHECK_LAUNCH("tfqmr iteration");
    }
    return RVK_OK;
}

} // namespace

extern "C" {

rvk_status rvk_tfqmr_plan_create(rvk_ctx ctx, const rvk_csr* A, rvk_cg_config cfg,
                                 rvk_tfqmr_plan* out)
{
    if (!ctx || !A || !out) return set_error(RVK_ERR_INVALID, "tfqmr_plan_create: null argument");
    RVK_TRACE_TASK(ctx, "tfqmr.plan_create");
    *out = nullptr;
    if (A->n_rows != A->n_cols) return set_error(RVK_ERR_DIM, "tfqmr_solve: matrix is not square");
    if (A->n_rows < 1) return set_error(RVK_ERR_DIM, "tfqmr_solve: empty system");
    if (cfg.max_it < 1) return set_error(RVK_ERR_INVALID, "tfqmr_solve: max_it must be >= 1");
    if (cfg.pc != RVK_PC_NONE && cfg.pc != RVK_PC_JACOBI)
        return set_error(RVK_ERR_INVALID, "tfqmr_solve: unknown preconditioner %d", cfg.pc);
    if (cfg.mode != RVK_CG_MODE_FUSED && cfg.mode != RVK_CG_MODE_AUTO && cfg.mode != RVK_CG_MODE_UNFUSED)
        return set_error(RVK_ERR_UNSUPPORTED, "tfqmr_solve: mode %d (FUSED, UNFUSED or AUTO)", cfg.mode);
    int64_t maxlen = 0;
    RVK_TRY(rvk_csr_validate(ctx, A, &maxlen));
    auto P = new rvk_tfqmr_plan_s();
    P->ctx = ctx;
    P->A   = *A;
    P->cfg = cfg;
    SpmvBands bands; // leading-edge L2 prefetch
    if (csr_bands(ctx->stream, *A, &bands) != RVK_OK) bands = SpmvBands{};
    P->fused    = cfg.mode != RVK_CG_MODE_UNFUSED;
    P->sa       = make_spmv_args(*A, maxlen, &bands);
    P->upd_grid = resident_grid(k_tfq_merge<true>, kTfqThreads, (A->n_rows + 1) / 2);
    const size_t vb = (size_t)A->n_rows * 8;
    cudaError_t  e  = cudaSuccess;
    auto alloc = [&](double** p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
    };
    for (double** v : {&P->R, &P->RP, &P->U, &P->P, &P->V, &P->D, &P->Q, &P->dinv})
        alloc(v, vb + 32);
    if (!P->fused)
        for (double** v : {&P->T, &P->AUQ, &P->T1}) alloc(v, vb + 32);
    alloc(&P->hist, 8 * (2 * (size_t)cfg.max_it + 1));
    alloc(&P->partials, 8 * 4 * (size_t)kMaxReduceBlocks);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&P->st), sizeof(TfqState));
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&P->tickets), 64);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->tickets, 0, 64, ctx->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(P->st, 0, sizeof(TfqState), ctx->stream);
    if (e != cudaSuccess) {
        rvk_tfqmr_plan_destroy(P);
        return cuda_error(e, "rvk_tfqmr_plan_create");
    }
    rvk_status rc = cfg.pc == RVK_PC_JACOBI ? rvk_csr_diagonal_inverse(ctx, A, P->dinv) : RVK_OK;
    // constant-coefficient operators: one diagonal value -> a scalar in the
    // fused kernels (as the CG plans; RVK_OPT_DINV_VECTOR disables)
    if (rc == RVK_OK && P->fused && cfg.pc == RVK_PC_JACOBI && !(cfg.opts & RVK_OPT_DINV_VECTOR))
        rc = vector_is_constant(ctx->stream, A->n_rows, P->dinv, &P->const_diag, &P->dconst);
    if (rc != RVK_OK) {
        rvk_tfqmr_plan_destroy(P);
        return rc;
    }
    *out = P;
    return RVK_OK;
}

rvk_status rvk_tfqmr_plan_destroy(rvk_tfqmr_plan P)
{
    if (!P) return RVK_OK;
    if (P->ctx) cudaStreamSynchronize(P->ctx->stream);
    if (P->graph) cudaGraphExecDestroy(P->graph);
    void* bufs[] = {P->R, P->RP, P->U, P->P, P->V, P->D, P->Q, P->T, P->AUQ, P->T1, P->dinv,
                    P->hist, P->st, P->partials, P->tickets};
    for (void* q : bufs)
        if (q) cudaFree(q);
    delete P;
    return RVK_OK;
}

rvk_status rvk_tfqmr_solve_dev(rvk_tfqmr_plan P, const double* b, double* x)
{
    if (!P || !b || !x) return set_error(RVK_ERR_INVALID, "tfqmr_solve: null argument");
    if (b == x) return set_error(RVK_ERR_INVALID, "tfqmr_solve: b and x must not alias");
    RVK_TRACE_TASK(P->ctx, "tfqmr.solve");
    cudaStream_t s = P->ctx->stream;
    if (!P->cfg.use_graph) return enqueue_tfqmr(P, b, x);
    if (!P->graph || P->g_b != b || P->g_x != x) {
        if (P->graph) cudaGraphExecDestroy(P->graph);
        P->graph      = nullptr;
        cudaGraph_t g = nullptr;
        RVK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal)); // proves 0 host syncs
        rvk_status  rc = enqueue_tfqmr(P, b, x);
        cudaError_t e  = cudaStreamEndCapture(s, &g);
        if (rc != RVK_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) return cuda_error(e, "cudaStreamEndCapture (tfqmr)");
        e = cudaGraphInstantiate(&P->graph, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return cuda_error(e, "cudaGraphInstantiate (tfqmr)");
        P->g_b = b;
        P->g_x = x;
    }
    RVK_CUDA(cudaGraphLaunch(P->graph, s));
    return RVK_OK;
}

int rvk_tfqmr_plan_flags(rvk_tfqmr_plan P)
{
    if (!P) return -1;
    return P->const_diag ? RVK_PLAN_CONST_DIAG : 0;
}

rvk_status rvk_tfqmr_result(rvk_tfqmr_plan P, double* hist_host, int* n_hist, rvk_cg_info* info)
{
    if (!P) return set_error(RVK_ERR_INVALID, "null plan");
    TfqState     h{};
    cudaStream_t s = P->ctx->stream;
    RVK_CUDA(cudaMemcpyAsync(&h, P->st, sizeof h, cudaMemcpyDeviceToHost, s));
    if (hist_host)
        RVK_CUDA(cudaMemcpyAsync(hist_host, P->hist, 8 * (2 * (size_t)P->cfg.max_it + 1),
                                 cudaMemcpyDeviceToHost, s));
    {
        trace::HostSyncScope hs_("rvk_tfqmr_result");
        RVK_CUDA(cudaStreamSynchronize(s));
    }
    if (n_hist) *n_hist = h.nhist;
    if (info) {
        info->state          = h.state;
        info->iterations     = h.iterations;
        info->breakdown_iter = h.breakdown_iter;
    }
    if (h.state == RVK_CG_BREAKDOWN)
        return set_error(RVK_ERR_BREAKDOWN, "tfqmr_solve: breakdown at iteration %d", h.breakdown_iter);
    return RVK_OK;
}

} // extern "C"
