// solvers.cpp -- cg_solve / pc_jacobi_apply / build_laplacian.
//
// Three execution modes over the same arithmetic:
//  * Fused (default, the B200 path): librvk's CG plan -- 2 fused kernels per
//    iteration, device-side scalar tails and exit flags, the whole solve one
//    CUDA graph (rvk_cg.cu).  Plans are cached per matrix (KSPSetUp reuse).
//  * Async: the PAPER.md:104-150 listing through the linalg API on three
//    contexts (dctx_a/b/c as SPEC.md:497 assigns them).  The listing's two
//    synchronous calls (VecAYPX(P, b.front(), Z) and the context-less
//    MatMult) are issued asynchronously on dctx_a instead, which is what
//    keeps the loop free of host syncs on a GPU.
//  * SyncBaseline: the same listing on the globally-blocking context.
#include "internal.hpp"
#include "rivulet/expr.hpp"
#include "rivulet/linalg.hpp"
#include "rivulet/solvers.hpp"
#include "rivulet/stencil.hpp"

#include <climits>
#include <cmath>
#include <map>
#include <tuple>

namespace rivulet {

using detail::Launch;
using runtime::KernelKind;

namespace detail {

struct CgPlanCache {
    Context ctx{StreamType::DefaultBlocking, "cg_fused"};
    std::map<std::tuple<int, int, double, double>, rvk_cg_plan> plans;
    std::map<std::tuple<int, int, double, double>, rvk_tfqmr_plan> tfqmr;
    ~CgPlanCache()
    {
        for (auto& [k, p] : plans) rvk_cg_plan_destroy(p);
        for (auto& [k, p] : tfqmr) rvk_tfqmr_plan_destroy(p);
    }
};

} // namespace detail

namespace {

void log_iteration_census(std::size_t n, std::size_t nnz, int it)
{
    runtime::log_kernel(KernelKind::MatMult, 2 * nnz);
    runtime::log_kernel(KernelKind::Dot, 4 * n, 2);
    runtime::log_kernel(KernelKind::Norm, 2 * n);
    runtime::log_kernel(KernelKind::Axpy, 4 * n, 2);
    if (it == 0) runtime::log_kernel(KernelKind::Copy, 0);
    else runtime::log_kernel(KernelKind::Aypx, 2 * n);
    runtime::log_kernel(KernelKind::PcApply, 0);
    runtime::log_kernel(KernelKind::ExprEval, it == 0 ? 1 : 2, it == 0 ? 1 : 2); // a (+ b)
    runtime::log_kernel(KernelKind::ExprEval, 1, 0);                            // -a, fused
}

FlopLog make_floplog(const runtime::Census& d, const runtime::CopyCounts& c0)
{
    FlopLog f;
    f.matmult     = d.flops_of(KernelKind::MatMult);
    f.dot         = d.flops_of(KernelKind::Dot);
    f.norm        = d.flops_of(KernelKind::Norm);
    f.axpy        = d.flops_of(KernelKind::Axpy) + d.flops_of(KernelKind::Waxpy);
    f.aypx        = d.flops_of(KernelKind::Aypx);
    f.scalar_expr = d.flops_of(KernelKind::ExprEval);
    f.total_flops = f.matmult + f.dot + f.norm + f.axpy + f.aypx + f.scalar_expr;
    const auto c  = runtime::copy_counts();
    f.h2d         = c.h2d - c0.h2d;
    f.d2h         = c.d2h - c0.d2h;
    return f;
}

SolveResult cg_fused(const CsrMatrix& A, const DenseVector& b, DenseVector& x, const SolverConfig& cfg)
{
    if (cfg.convergence_callback)
        throw Error("cg_solve: convergence_callback needs SolverMode::Async or SyncBaseline "
                    "(the fused solve is a single device graph; use rtol/atol)");
    auto& ms = *A.state();
    if (!ms.plans) ms.plans = std::make_shared<detail::CgPlanCache>();
    auto&      cache = *ms.plans;
    const auto key   = std::make_tuple(cfg.max_it, cfg.pc == PcType::Jacobi ? 1 : 0, cfg.rtol, cfg.atol);
    auto       it    = cache.plans.find(key);
    if (it == cache.plans.end()) {
        // AUTO: the one-cluster DSMEM solve for small systems (<= 16 K rows of
        // <= 9 entries, one launch), else the fused 2-kernel graph
        rvk_cg_config c{cfg.max_it, cfg.pc == PcType::Jacobi ? RVK_PC_JACOBI : RVK_PC_NONE,
                        cfg.rtol, cfg.atol, RVK_CG_MODE_AUTO, 1, 0};
        rvk_cg_plan   p = nullptr;
        const rvk_csr v = ms.view();
        detail::check(rvk_cg_plan_create(cache.ctx.handle(), &v, c, &p), "cg_solve(setup)");
        it = cache.plans.emplace(key, p).first;
    }
    rvk_cg_plan plan = it->second;
    const auto  c0   = runtime::census();
    const auto  cc0  = runtime::copy_counts();
    Launch      L(cache.ctx, "cg_solve(fused)");
    L.read(A.id()).read(b.id()).write(x.id());
    L.begin();
    detail::check(rvk_cg_solve_dev(plan, b.device_data(), x.device_data()), "cg_solve");
    L.end();
    detail::device_wrote(*x.state());

    std::vector<double> hist(cfg.max_it + 1);
    rvk_cg_info         info{};
    const rvk_status    st = rvk_cg_result(plan, hist.data(), &info);
    runtime::log_d2h(hist.size() * sizeof(double));
    // census of the logical operations the fused kernels performed (setup:
    // r = b, z = B r, ||z||, z.r; then per iteration), matching the listing
    runtime::log_kernel(KernelKind::Copy, 0, 2);
    runtime::log_kernel(KernelKind::PcApply, 0);
    runtime::log_kernel(KernelKind::Norm, 2 * A.rows());
    runtime::log_kernel(KernelKind::Dot, 2 * A.rows());
    for (int i = 0; i < info.iterations; ++i) log_iteration_census(A.rows(), A.nnz(), i);
    if (st == RVK_ERR_BREAKDOWN)
        throw BreakdownError("cg_solve: breakdown at iteration " + std::to_string(info.breakdown_iter),
                             info.breakdown_iter);
    detail::check(st, "cg_solve");
    SolveResult r;
    r.iterations = info.iterations;
    r.converged  = info.state == RVK_CG_CONVERGED;
    r.history.assign(hist.begin(), hist.begin() + info.iterations + 1);
    r.flops = make_floplog(runtime::census() - c0, cc0);
    return r;
}

// Copy a device scalar into slot k of a device history array (stream-ordered).
void record_history(const Context& ctx, const Managed& dp, DenseVector& hist, int k)
{
    Launch L(ctx, "history");
    L.read(dp.id()).read_write(hist.id());
    L.begin();
    detail::check(rvk_memcpy_d2d(ctx.handle(), hist.device_data() + k, dp.device_data(), sizeof(double)),
                  "history");
    L.end();
    detail::device_wrote(*hist.state());
}

void monitor(const Context& ctx, const Managed& num, const Managed& den, int it, int* flag)
{
    Launch L(ctx, "breakdown_monitor");
    L.read(num.id()).read(den.id());
    L.begin();
    detail::check(detail::breakdown_check(reinterpret_cast<cudaStream_t>(ctx.cuda_stream()),
                                          num.device_data(), den.device_data(), it, flag),
                  "breakdown monitor");
    L.end();
}

SolveResult cg_listing(const CsrMatrix& A, const DenseVector& b, DenseVector& x, const SolverConfig& cfg)
{
    const bool    sync = cfg.mode == SolverMode::SyncBaseline;
    const Context a    = sync ? detail::global_sync_context() : Context(StreamType::DefaultBlocking, "dctx_a");
    const Context bctx = sync ? detail::global_sync_context() : Context(StreamType::DefaultBlocking, "dctx_b");
    const Context c    = sync ? detail::global_sync_context() : Context(StreamType::DefaultBlocking, "dctx_c");
    const std::size_t n = A.rows();
    const auto        c0  = runtime::census();
    const auto        cc0 = runtime::copy_counts();

    DenseVector R(n, "R"), Z(n, "Z"), P(n, "P"), W(n, "W"), Dinv(n, "Dinv"), hist(cfg.max_it + 1, "hist");
    Managed     beta(0.0, "beta"), betaold(0.0, "betaold"), alpha(0.0, "a"), bb(0.0, "b"), dp(0.0, "dp"),
        pAp(0.0, "pAp");
    int* flag = static_cast<int*>(detail::device_alloc(sizeof(int)));
    {
        const int big = INT_MAX;
        detail::check_cuda(cudaMemcpy(flag, &big, sizeof(int), cudaMemcpyHostToDevice), "flag");
    }

    vec_set_async(x, 0.0, a, "x0");
    vec_copy_async(b, R, a, "r0");
    if (cfg.pc == PcType::Jacobi) {
        Launch L(a, "pc_setup");
        L.read(A.id()).write(Dinv.id());
        L.begin();
        const rvk_csr v = A.state()->view();
        detail::check(rvk_csr_diagonal_inverse(a.handle(), &v, Dinv.device_data()), "pc_setup");
        L.end();
        detail::device_wrote(*Dinv.state());
        pc_jacobi_apply(Dinv, R, Z, a);
    } else {
        vec_copy_async(R, Z, a, "z=r");
    }
    vec_norm_async(Z, NormType::Norm2, dp, a, "dp0");
    record_history(a, dp, hist, 0);
    std::function<bool(Managed&, int)> cb = cfg.convergence_callback;
    double                             dp0 = -1.0;
    if (!cb && (cfg.rtol > 0.0 || cfg.atol > 0.0)) {
        // the reference's convergence test reads dp on the host (one sync per iteration)
        cb = [&](Managed& d, int) {
            const double v = d.front();
            if (dp0 < 0) dp0 = v;
            return v <= std::fmax(cfg.rtol * dp0, cfg.atol);
        };
    }
    int  its  = 0;
    // the default rtol/atol test also checks the initial residual; a user
    // callback is only consulted inside the loop, as in the listing
    bool conv = (cb && !cfg.convergence_callback) ? cb(dp, -1) : false;
    if (!conv) vec_dot_async(Z, R, beta, bctx, "beta");
    for (int i = 0; i < cfg.max_it && !conv; ++i) {
        if (i == 0) {
            vec_copy_async(Z, P, a, "p=z");
        } else {
            monitor(a, beta, betaold, i, flag);
            bb = Eval(beta / betaold, a);        // b <- beta/betaold
            vec_aypx_async(P, bb, Z, a, "aypx"); // p <- z + b p           (:122)
        }
        mat_mult(A, P, W, a, "matmult");         // w <- A p               (:125)
        vec_dot_async(P, W, pAp, bctx, "pAp");   // a <- p'w               (:127)
        monitor(c, beta, pAp, i, flag);
        alpha   = Eval(beta / pAp, c);           // a <- beta / a          (:129)
        betaold = Eval(beta, a);                 // betaold <- beta        (:132)
        vec_axpy_async(x, alpha, P, bctx, "x+=ap");  // (:136)
        vec_axpy_async(R, -alpha, W, c, "r-=aw");    // (:137)
        if (cfg.pc == PcType::Jacobi) pc_jacobi_apply(Dinv, R, Z, a); // (:140)
        else vec_copy_async(R, Z, a, "z=r");
        vec_norm_async(Z, NormType::Norm2, dp, a, "dp");             // (:141)
        record_history(a, dp, hist, i + 1);
        its = i + 1;
        if (cb && cb(dp, i)) {                   // user callback        (:143-144)
            conv = true;
            break;
        }
        vec_dot_async(Z, R, beta, bctx, "beta"); // beta <- z'r            (:145)
    }
    // results: one host read of the history (and the breakdown flag)
    std::vector<double> h;
    {
        auto view = hist.array_read();
        h.assign(view.span().begin(), view.span().begin() + its + 1);
    }
    int bd = INT_MAX;
    detail::check_cuda(cudaMemcpy(&bd, flag, sizeof(int), cudaMemcpyDeviceToHost), "flag");
    detail::device_release(flag, 0);
    if (!sync) {
        a.synchronize();
        bctx.synchronize();
        c.synchronize();
    }
    if (bd != INT_MAX)
        throw BreakdownError("cg_solve: breakdown at iteration " + std::to_string(bd), bd);
    SolveResult r;
    r.iterations = its;
    r.converged  = conv;
    r.history    = std::move(h);
    r.flops      = make_floplog(runtime::census() - c0, cc0);
    return r;
}

} // namespace

SolveResult cg_solve(const CsrMatrix& A, const DenseVector& b, DenseVector& x, const SolverConfig& cfg)
{
    if (cfg.method != SolverMethod::CG) throw Error("cg_solve: method must be CG");
    if (A.rows() != A.cols()) throw Error("cg_solve: matrix is not square");
    if (b.size() != A.rows() || x.size() != A.cols()) throw Error("cg_solve: dimension mismatch");
    if (cfg.max_it < 1) throw Error("cg_solve: max_it must be >= 1");
    if (cfg.mode == SolverMode::Fused) return cg_fused(A, b, x, cfg);
    return cg_listing(A, b, x, cfg);
}

// Left-Jacobi TFQMR through librvk's TFQMR plan (rvk_tfqmr.cu): PETSc
// KSPSolve_TFQMR order, all scalars device-resident, the solve one CUDA graph.
// SolverMode is not consulted (there is no op-per-call listing for TFQMR in
// the paper); the history is ||B r0|| followed by one residual bound per half
// step (2 per outer iteration).
SolveResult tfqmr_solve(const CsrMatrix& A, const DenseVector& b, DenseVector& x, const SolverConfig& cfg)
{
    if (cfg.max_it < 1) throw Error("tfqmr_solve: max_it must be >= 1");
    if (A.rows() != A.cols()) throw Error("tfqmr_solve: matrix is not square");
    if (b.size() != A.rows() || x.size() != A.rows()) throw Error("tfqmr_solve: dimension mismatch");
    if (cfg.convergence_callback)
        throw Error("tfqmr_solve: convergence_callback is not supported (the solve is one device graph; "
                    "use rtol/atol)");
    auto& ms = *A.state();
    if (!ms.plans) ms.plans = std::make_shared<detail::CgPlanCache>();
    auto&      cache = *ms.plans;
    const auto key   = std::make_tuple(cfg.max_it, cfg.pc == PcType::Jacobi ? 1 : 0, cfg.rtol, cfg.atol);
    auto       it    = cache.tfqmr.find(key);
    if (it == cache.tfqmr.end()) {
        rvk_cg_config  c{cfg.max_it, cfg.pc == PcType::Jacobi ? RVK_PC_JACOBI : RVK_PC_NONE,
                         cfg.rtol, cfg.atol, RVK_CG_MODE_FUSED, 1, 0};
        rvk_tfqmr_plan p = nullptr;
        const rvk_csr  v = ms.view();
        detail::check(rvk_tfqmr_plan_create(cache.ctx.handle(), &v, c, &p), "tfqmr_solve(setup)");
        it = cache.tfqmr.emplace(key, p).first;
    }
    rvk_tfqmr_plan plan = it->second;
    const auto     c0   = runtime::census();
    const auto     cc0  = runtime::copy_counts();
    Launch         L(cache.ctx, "tfqmr_solve");
    L.read(A.id()).read(b.id()).write(x.id());
    L.begin();
    detail::check(rvk_tfqmr_solve_dev(plan, b.device_data(), x.device_data()), "tfqmr_solve");
    L.end();
    detail::device_wrote(*x.state());

    std::vector<double> hist(2 * (std::size_t)cfg.max_it + 1);
    rvk_cg_info         info{};
    int                 nh = 0;
    const rvk_status    st = rvk_tfqmr_result(plan, hist.data(), &nh, &info);
    runtime::log_d2h(hist.size() * sizeof(double));
    // census: setup (B b, ||r||, (r, rp), v = B A p), then per outer iteration
    // 2 matmults, 3 reductions, 7 vector updates (+2 on the continuing path)
    const std::size_t n = A.rows(), nnz = A.nnz();
    runtime::log_kernel(KernelKind::PcApply, 0);
    runtime::log_kernel(KernelKind::Norm, 2 * n);
    runtime::log_kernel(KernelKind::Dot, 2 * n);
    runtime::log_kernel(KernelKind::Copy, 0, 3);
    runtime::log_kernel(KernelKind::MatMult, 2 * nnz);
    runtime::log_kernel(KernelKind::PcApply, 0);
    for (int i = 0; i < info.iterations; ++i) {
        const bool last_conv = info.state == RVK_CG_CONVERGED && i + 1 == info.iterations;
        runtime::log_kernel(KernelKind::Dot, 2 * n);
        runtime::log_kernel(KernelKind::Waxpy, 4 * n, 2);
        runtime::log_kernel(KernelKind::MatMult, 2 * nnz);
        runtime::log_kernel(KernelKind::PcApply, 0);
        runtime::log_kernel(KernelKind::Axpy, 2 * n);
        runtime::log_kernel(KernelKind::Norm, 2 * n);
        runtime::log_kernel(KernelKind::ExprEval, 2, 2); // a, -a
        runtime::log_kernel(KernelKind::Aypx, 4 * n, 2);
        runtime::log_kernel(KernelKind::Axpy, 4 * n, 2);
        runtime::log_kernel(KernelKind::ExprEval, 28, 2); // psi, cm, tau, eta, cf, bound
        if (last_conv) continue;
        runtime::log_kernel(KernelKind::Dot, 2 * n);
        runtime::log_kernel(KernelKind::ExprEval, 1, 1); // b
        runtime::log_kernel(KernelKind::Waxpy, 4 * n, 2);
        runtime::log_kernel(KernelKind::Axpy, 2 * n);
        runtime::log_kernel(KernelKind::MatMult, 2 * nnz);
        runtime::log_kernel(KernelKind::PcApply, 0);
    }
    if (st == RVK_ERR_BREAKDOWN)
        throw BreakdownError("tfqmr_solve: breakdown at iteration " + std::to_string(info.breakdown_iter),
                             info.breakdown_iter);
    detail::check(st, "tfqmr_solve");
    SolveResult r;
    r.iterations = info.iterations;
    r.converged  = info.state == RVK_CG_CONVERGED;
    r.history.assign(hist.begin(), hist.begin() + nh);
    r.flops = make_floplog(runtime::census() - c0, cc0);
    return r;
}

void pc_jacobi_apply(const DenseVector& diag_inv, const DenseVector& r, DenseVector& z, const Context& ctx)
{
    vec_pointwise_mult_async(diag_inv, r, z, ctx, "pc_jacobi");
}

// ---- stencils ------------------------------------------------------------------------------
StencilCoefficients stencil_coefficients(int dim, int points)
{
    if (!((dim == 2 && (points == 5 || points == 9)) || (dim == 3 && (points == 7 || points == 27))))
        throw Error("stencil_coefficients: invalid (dim, points)");
    return StencilCoefficients{static_cast<double>(points - 1), -1.0};
}

CsrMatrix build_laplacian(const StencilSpec& spec)
{
    if ((int)spec.grid.size() != spec.dim) throw Error("build_laplacian: grid must have dim entries");
    const std::int64_t nx = spec.grid[0], ny = spec.grid[1], nz = spec.dim == 3 ? spec.grid[2] : 1;
    std::int64_t       n = 0, nnz = 0;
    if (rvk_laplacian_size(spec.dim, spec.points, nx, ny, nz, &n, &nnz) != RVK_OK)
        throw Error(std::string("build_laplacian: ") + rvk_last_error());
    auto s    = std::make_shared<detail::MatState>("laplacian");
    s->n_rows = s->n_cols = (std::size_t)n;
    s->nnz                = (std::size_t)nnz;
    s->max_row_len        = spec.points;
    s->off  = static_cast<std::int64_t*>(detail::device_alloc((n + 1) * sizeof(std::int64_t)));
    s->cols = static_cast<std::int32_t*>(detail::device_alloc(nnz * sizeof(std::int32_t)));
    s->vals = static_cast<double*>(detail::device_alloc(nnz * sizeof(double)));
    CsrMatrix      A(s);
    const Context& g = detail::global_sync_context();
    Launch         L(g, "build_laplacian");
    L.write(A.id());
    L.begin();
    detail::check(rvk_build_laplacian(g.handle(), spec.dim, spec.points, nx, ny, nz, s->off, s->cols,
                                      s->vals),
                  "build_laplacian");
    L.end();
    return A;
}

} // namespace rivulet
