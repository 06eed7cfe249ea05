// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" face over the reference's own arithmetic kernels, compiled from
// /root/reference/proj/src/kernels_{scalar,avx2,dispatch}.cpp + common.cpp
// (unmodified, read in place) into oracle/_ref/librivulet_ref.so by
// oracle/Makefile.  Used to (1) pin the C restatement in rvk_oracle.c
// bit-for-bit, (2) generate the golden vectors in tests/golden/, and (3) time
// the reference CPU solver in bench.py's cpu_baseline / --impl reference arm.
//
// The CG loop itself is not in the reference tree (solvers.cpp is absent);
// ref_cg_solve restates it exactly like rvk_oracle.c:ro_cg_solve but calls
// rivulet::kernels::{scalar,avx2} for every vector/matrix operation, which is
// what the reference's linalg layer does (one kernel per op).
#include "rivulet/kernels/kernels.hpp"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>

namespace rk = rivulet::kernels;

namespace {

struct Ops {
    double (*dot)(std::span<const double>, std::span<const double>);
    double (*nrm2)(std::span<const double>);
    void (*axpy)(double, std::span<const double>, std::span<double>);
    void (*aypx)(double, std::span<const double>, std::span<double>);
    void (*waxpy)(double, std::span<const double>, std::span<const double>, std::span<double>);
    void (*pointwise_mult)(std::span<const double>, std::span<const double>, std::span<double>);
    void (*csr_spmv)(std::span<const std::int64_t>, std::span<const std::int32_t>,
                     std::span<const double>, std::span<const double>, std::span<double>);
};

// backend 0: scalar (the documented reference order, kernels_scalar.cpp:8-9);
// backend 1: AVX2; backend 2: the reference's own dispatch (auto / env).
Ops ops_for(int backend)
{
    if (backend == 0)
        return {rk::scalar::dot, rk::scalar::nrm2, rk::scalar::axpy, rk::scalar::aypx, rk::scalar::waxpy,
                rk::scalar::pointwise_mult, rk::scalar::csr_spmv};
#if RIVULET_X86_64
    if (backend == 1)
        return {rk::avx2::dot, rk::avx2::nrm2, rk::avx2::axpy, rk::avx2::aypx, rk::avx2::waxpy,
                rk::avx2::pointwise_mult, rk::avx2::csr_spmv};
#endif
    return {rk::dot, rk::nrm2, rk::axpy, rk::aypx, rk::waxpy, rk::pointwise_mult, rk::csr_spmv};
}

template <typename T>
std::span<T> sp(T* p, std::int64_t n) { return {p, static_cast<std::size_t>(n)}; }
template <typename T>
std::span<const T> csp(const T* p, std::int64_t n) { return {p, static_cast<std::size_t>(n)}; }

} // namespace

extern "C" {

int ref_avx2_supported() { return rk::avx2_supported() ? 1 : 0; }

double ref_dot(int backend, std::int64_t n, const double* x, const double* y)
{
    return ops_for(backend).dot(csp(x, n), csp(y, n));
}
double ref_nrm2(int backend, std::int64_t n, const double* x)
{
    return ops_for(backend).nrm2(csp(x, n));
}
void ref_axpy(int backend, std::int64_t n, double a, const double* x, double* y)
{
    ops_for(backend).axpy(a, csp(x, n), sp(y, n));
}
void ref_aypx(int backend, std::int64_t n, double b, const double* x, double* y)
{
    ops_for(backend).aypx(b, csp(x, n), sp(y, n));
}
void ref_waxpy(std::int64_t n, double a, const double* x, const double* y, double* w)
{
    rk::scalar::waxpy(a, csp(x, n), csp(y, n), sp(w, n));
}
void ref_scale(std::int64_t n, double a, double* x) { rk::scalar::scale(a, sp(x, n)); }
void ref_pointwise_mult(int backend, std::int64_t n, const double* a, const double* b, double* o)
{
    ops_for(backend).pointwise_mult(csp(a, n), csp(b, n), sp(o, n));
}
void ref_csr_spmv(int backend, std::int64_t n_rows, std::int64_t nnz, const std::int64_t* off,
                  const std::int32_t* cols, const double* vals, std::int64_t n_cols,
                  const double* x, double* y)
{
    ops_for(backend).csr_spmv(csp(off, n_rows + 1), csp(cols, nnz), csp(vals, nnz),
                              csp(x, n_cols), sp(y, n_rows));
}

// Same contract as ro_cg_solve (rvk_oracle.h); pc: 0 none, 1 Jacobi.
// out3 = {status, iterations, breakdown_iter}.
void ref_cg_solve(int backend, std::int64_t n, std::int64_t nnz, const std::int64_t* off,
                  const std::int32_t* cols, const double* vals, const double* b, double* x,
                  double* hist, int max_it, int pc, double rtol, double atol, double* work,
                  int* out3)
{
    const Ops o = ops_for(backend);
    double* r    = work;
    double* z    = work + n;
    double* p    = work + 2 * n;
    double* w    = work + 3 * n;
    double* dinv = work + 4 * n;
    const auto bytes = static_cast<std::size_t>(n) * sizeof(double);
    out3[0] = 0; out3[1] = 0; out3[2] = -1;

    std::memset(x, 0, bytes);
    std::memset(p, 0, bytes);
    std::memcpy(r, b, bytes);
    if (pc == 1) {
        for (std::int64_t row = 0; row < n; ++row) {
            double d = 0.0;
            for (auto k = off[row]; k < off[row + 1]; ++k)
                if (cols[k] == row) d = vals[k];
            dinv[row] = 1.0 / d;
        }
        o.pointwise_mult(csp(dinv, n), csp(r, n), sp(z, n));
    } else {
        std::memcpy(z, r, bytes);
    }
    double dp = o.nrm2(csp(z, n));
    hist[0]   = dp;
    const double dp0 = dp;
    auto conv = [&](double v) { return v <= std::fmax(rtol * dp0, atol); };
    if (conv(dp)) { out3[0] = 1; return; }
    double beta = o.dot(csp(z, n), csp(r, n)), betaold = 0.0;
    for (int i = 0; i < max_it; ++i) {
        if (i == 0) {
            std::memcpy(p, z, bytes);
        } else {
            if (betaold == 0.0) { out3[0] = 2; out3[2] = i; return; }
            o.aypx(beta / betaold, csp(z, n), sp(p, n));
        }
        o.csr_spmv(csp(off, n + 1), csp(cols, nnz), csp(vals, nnz), csp(p, n), sp(w, n));
        const double pAp = o.dot(csp(p, n), csp(w, n));
        const double a   = beta / pAp;
        if (pAp == 0.0 || !std::isfinite(a)) { out3[0] = 2; out3[2] = i; return; }
        betaold = beta;
        o.axpy(a, csp(p, n), sp(x, n));
        o.axpy(-a, csp(w, n), sp(r, n));
        if (pc == 1) o.pointwise_mult(csp(dinv, n), csp(r, n), sp(z, n));
        else std::memcpy(z, r, bytes);
        dp          = o.nrm2(csp(z, n));
        hist[i + 1] = dp;
        out3[1]     = i + 1;
        if (conv(dp)) { out3[0] = 1; return; }
        beta = o.dot(csp(z, n), csp(r, n));
    }
}

// Left-Jacobi TFQMR (Freund's single-loop formulation, two
// half-iterations per outer iteration) in PETSc KSPSolve_TFQMR operation
// order -- the same loop as rvk_oracle.c:ro_tfqmr_solve, every vector and
// matrix operation through the reference's own kernels (the reference ships
// no TFQMR source: solvers.cpp is absent).  B = D^-1 applied on the left:
// each operator application is T1 = A v, out = dinv .* T1.  hist: ||B r0||
// then the residual bound sqrt(2i+m+2) tau of every half step.
// out4 = {status, iterations, breakdown_iter, n_hist}.
void ref_tfqmr_solve(int backend, std::int64_t n, std::int64_t nnz, const std::int64_t* off,
                     const std::int32_t* cols, const double* vals, const double* b, double* x,
                     double* hist, int max_it, int pc, double rtol, double atol, double* work,
                     int* out4)
{
    const Ops o = ops_for(backend);
    double *R = work, *RP = work + n, *U = work + 2 * n, *P = work + 3 * n, *V = work + 4 * n;
    double *D = work + 5 * n, *Q = work + 6 * n, *T = work + 7 * n, *AUQ = work + 8 * n;
    double *T1 = work + 9 * n, *dinv = work + 10 * n;
    const auto bytes = static_cast<std::size_t>(n) * sizeof(double);
    int        nh    = 0;
    out4[0] = 0; out4[1] = 0; out4[2] = -1; out4[3] = 0;
    auto apply_BA = [&](const double* v, double* out) {
        o.csr_spmv(csp(off, n + 1), csp(cols, nnz), csp(vals, nnz), csp(v, n), sp(T1, n));
        if (pc == 1) o.pointwise_mult(csp(dinv, n), csp(T1, n), sp(out, n));
        else std::memcpy(out, T1, bytes);
    };
    std::memset(x, 0, bytes);
    if (pc == 1) {
        for (std::int64_t row = 0; row < n; ++row) {
            double d = 0.0;
            for (auto k = off[row]; k < off[row + 1]; ++k)
                if (cols[k] == row) d = vals[k];
            dinv[row] = 1.0 / d;
        }
        o.pointwise_mult(csp(dinv, n), csp(b, n), sp(R, n)); // R = B (b - A x0), x0 = 0
    } else {
        std::memcpy(R, b, bytes);
    }
    double dp = o.nrm2(csp(R, n));
    hist[nh++] = dp;
    const double dp0 = dp;
    auto conv = [&](double v) { return v <= std::fmax(rtol * dp0, atol); };
    if (conv(dp)) { out4[0] = 1; out4[3] = nh; return; }
    std::memcpy(RP, R, bytes);
    double etaold = 0.0, psiold = 0.0, tau = dp, dpold = dp;
    double rhoold = o.dot(csp(R, n), csp(RP, n));
    std::memcpy(U, R, bytes);
    std::memcpy(P, R, bytes);
    apply_BA(P, V);
    std::memset(D, 0, bytes);
    for (int i = 0; i < max_it; ++i) {
        const double s = o.dot(csp(V, n), csp(RP, n));
        if (s == 0.0) { out4[0] = 2; out4[2] = i; out4[3] = nh; return; }
        const double a = rhoold / s;
        o.waxpy(-a, csp(V, n), csp(U, n), sp(Q, n));  // q = u - a v
        o.waxpy(1.0, csp(U, n), csp(Q, n), sp(T, n)); // t = u + q
        apply_BA(T, AUQ);
        o.axpy(-a, csp(AUQ, n), sp(R, n));            // r = r - a B A (u + q)
        dp = o.nrm2(csp(R, n));
        for (int m = 0; m < 2; ++m) {
            const double w   = m == 0 ? std::sqrt(dp * dpold) : dp;
            const double psi = w / tau;
            const double cm  = 1.0 / std::sqrt(1.0 + psi * psi);
            tau              = tau * psi * cm;
            const double eta = cm * cm * a;
            const double cf  = psiold * psiold * etaold / a;
            o.aypx(cf, csp(m == 0 ? U : Q, n), sp(D, n)); // d = (u|q) + cf d
            o.axpy(eta, csp(D, n), sp(x, n));             // x = x + eta d
            const double dpest = std::sqrt(2.0 * i + m + 2.0) * tau;
            hist[nh++]         = dpest;
            if (conv(dpest)) { out4[0] = 1; out4[1] = i + 1; out4[3] = nh; return; }
            etaold = eta;
            psiold = psi;
        }
        out4[1] = i + 1;
        const double rho = o.dot(csp(R, n), csp(RP, n));
        if (rhoold == 0.0) { out4[0] = 2; out4[2] = i; out4[3] = nh; return; }
        const double bb = rho / rhoold;
        o.waxpy(bb, csp(Q, n), csp(R, n), sp(U, n)); // u = r + b q
        o.axpy(bb, csp(P, n), sp(Q, n));             // q = q + b p
        o.waxpy(bb, csp(Q, n), csp(U, n), sp(P, n)); // p = u + b q
        apply_BA(P, V);
        rhoold = rho;
        dpold  = dp;
    }
    out4[3] = nh;
}

} // extern "C"
