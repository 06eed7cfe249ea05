/*
 * rvk_oracle.c -- TEST INFRASTRUCTURE ONLY (see rvk_oracle.h).
 *
 * Plain-C restatement of the reference's Jacobi-CG path.  Build flags must
 * keep IEEE mul-then-add semantics: -O2 -ffp-contract=off and no -march
 * (SURVEY.md 7.3 "FMA pitfalls"), matching proj/CMakeLists.txt's Release
 * flags, which carry no -march either.
 */
#include "rvk_oracle.h"

#include <math.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* kernels_scalar.cpp:11-17 -- single left-to-right chain.                   */
double ro_dot(int64_t n, const double* x, const double* y)
{
    double sum = 0.0;
    for (int64_t i = 0; i < n; ++i) sum += x[i] * y[i];
    return sum;
}

/* kernels_scalar.cpp:19-22 */
double ro_nrm2(int64_t n, const double* x) { return sqrt(ro_dot(n, x, x)); }

/* kernels_scalar.cpp:24-28: y += a*x */
void ro_axpy(int64_t n, double a, const double* x, double* y)
{
    for (int64_t i = 0; i < n; ++i) y[i] += a * x[i];
}

/* kernels_scalar.cpp:30-34: y = x + b*y */
void ro_aypx(int64_t n, double b, const double* x, double* y)
{
    for (int64_t i = 0; i < n; ++i) y[i] = x[i] + b * y[i];
}

/* kernels_scalar.cpp:36-40: w = a*x + y */
void ro_waxpy(int64_t n, double a, const double* x, const double* y, double* w)
{
    for (int64_t i = 0; i < n; ++i) w[i] = a * x[i] + y[i];
}

/* kernels_scalar.cpp:42-45 */
void ro_scale(int64_t n, double a, double* x)
{
    for (int64_t i = 0; i < n; ++i) x[i] *= a;
}

/* kernels_scalar.cpp:47-51 */
void ro_pointwise_mult(int64_t n, const double* a, const double* b, double* out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = a[i] * b[i];
}

/* kernels_scalar.cpp:53-63: per-row sequential sum starting from 0.0. */
void ro_csr_spmv(int64_t n_rows, const int64_t* off, const int32_t* cols,
                 const double* vals, const double* x, double* y)
{
    for (int64_t row = 0; row < n_rows; ++row) {
        double sum = 0.0;
        for (int64_t k = off[row]; k < off[row + 1]; ++k) sum += vals[k] * x[cols[k]];
        y[row] = sum;
    }
}

/* ------------------------------------------------------------------------ */
/* Stencils.
 *  - lexicographic ordering, x fastest: i = x + nx*(y + ny*z)
 *  - Dirichlet by truncation: out-of-grid neighbours are simply omitted (:529)
 *  - 5-pt (4,-1) and 7-pt (6,-1); 9-pt and 27-pt use
 *    centre = points-1 and -1 for every neighbour (SPEC leaves
 *    the weights open, :537, :550, :558)
 *  - columns strictly increasing within a row (csr.hpp:51-53): the
 *    (dz, dy, dx) loop nest below walks neighbours in ascending column order. */

int ro_stencil_valid(int dim, int points, int64_t nx, int64_t ny, int64_t nz)
{
    if (dim == 2) {
        if (points != 5 && points != 9) return 0;
        return nx >= 2 && ny >= 2;
    }
    if (dim == 3) {
        if (points != 7 && points != 27) return 0;
        return nx >= 2 && ny >= 2 && nz >= 2;
    }
    return 0;
}

int64_t ro_laplacian_rows(int dim, int64_t nx, int64_t ny, int64_t nz)
{
    return dim == 2 ? nx * ny : nx * ny * nz;
}

static int in_stencil(int points, int dx, int dy, int dz)
{
    if (points == 5 || points == 7) return (dx != 0) + (dy != 0) + (dz != 0) <= 1;
    return 1; /* 9 / 27: full box */
}

int64_t ro_laplacian_nnz(int dim, int points, int64_t nx, int64_t ny, int64_t nz)
{
    if (!ro_stencil_valid(dim, points, nx, ny, nz)) return -1;
    if (dim == 2) {
        if (points == 5) return 5 * nx * ny - 2 * nx - 2 * ny;
        return (3 * nx - 2) * (3 * ny - 2);
    }
    if (points == 7) return 7 * nx * ny * nz - 2 * (nx * ny + ny * nz + nx * nz);
    return (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2);
}

int64_t ro_build_laplacian(int dim, int points, int64_t nx, int64_t ny, int64_t nz,
                           int64_t* off, int32_t* cols, double* vals)
{
    if (!ro_stencil_valid(dim, points, nx, ny, nz)) return -1;
    if (dim == 2) nz = 1;
    const int    zr     = dim == 3 ? 1 : 0;
    const double centre = (double)(points - 1);
    int64_t      k      = 0;
    int64_t      row    = 0;
    off[0]              = 0;
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x, ++row) {
                for (int dz = -zr; dz <= zr; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (!in_stencil(points, dx, dy, dz)) continue;
                            const int64_t xx = x + dx, yy = y + dy, zz = z + dz;
                            if (xx < 0 || xx >= nx || yy < 0 || yy >= ny || zz < 0 || zz >= nz)
                                continue;
                            cols[k] = (int32_t)(xx + nx * (yy + ny * zz));
                            vals[k] = (dx == 0 && dy == 0 && dz == 0) ? centre : -1.0;
                            ++k;
                        }
                off[row + 1] = k;
            }
    return k;
}

/* csr.hpp:76-77: diagonal entries, zero where absent. */
void ro_csr_diagonal(int64_t n_rows, const int64_t* off, const int32_t* cols,
                     const double* vals, double* diag)
{
    for (int64_t r = 0; r < n_rows; ++r) {
        double d = 0.0;
        for (int64_t k = off[r]; k < off[r + 1]; ++k)
            if (cols[k] == r) d = vals[k];
        diag[r] = d;
    }
}

/* ------------------------------------------------------------------------ */
uint64_t ro_splitmix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void ro_rhs(uint64_t seed, int64_t n, double* b)
{
    const double scale = 1.0 / 4503599627370496.0; /* 2^-52 */
    for (int64_t i = 0; i < n; ++i)
        b[i] = (double)(ro_splitmix64(seed + (uint64_t)i) >> 11) * scale - 1.0;
}

/* ------------------------------------------------------------------------ */
/* Jacobi-PCG.
 *   setup:  r = b, z = B r, dp = ||z|| -> hist[0], beta = z.r
 *   iter i: b = beta/betaold (i>=1); p = z + b p (i==0: p = z)
 *           w = A p; pAp = p.w; a = beta/pAp; betaold = beta
 *           x += a p; r += (-a) w; z = B r; dp = ||z|| -> hist[i+1]
 *           converged?; beta = z.r
 * Breakdown (common.hpp:33-43): betaold == 0 at i >= 1, or
 * pAp == 0, or a non-finite alpha/beta ratio.                               */
static int converged(double dp, double dp0, const ro_cg_config* cfg)
{
    const double tol = fmax(cfg->rtol * dp0, cfg->atol);
    return dp <= tol;
}

ro_cg_result ro_cg_solve(int64_t n, const int64_t* off, const int32_t* cols,
                         const double* vals, const double* b, double* x,
                         double* hist, ro_cg_config cfg, double* work)
{
    ro_cg_result res = {RO_OK, 0, -1};
    double*      r    = work;
    double*      z    = work + n;
    double*      p    = work + 2 * n;
    double*      w    = work + 3 * n;
    double*      dinv = work + 4 * n;

    memset(x, 0, (size_t)n * sizeof(double));
    memset(p, 0, (size_t)n * sizeof(double));
    memcpy(r, b, (size_t)n * sizeof(double));
    if (cfg.pc == RO_PC_JACOBI) {
        ro_csr_diagonal(n, off, cols, vals, dinv);
        for (int64_t i = 0; i < n; ++i) dinv[i] = 1.0 / dinv[i];
        ro_pointwise_mult(n, dinv, r, z);
    } else {
        memcpy(z, r, (size_t)n * sizeof(double));
    }
    double dp = ro_nrm2(n, z);
    hist[0]   = dp;
    const double dp0 = dp;
    if (converged(dp, dp0, &cfg)) {
        res.status = RO_CONVERGED;
        return res;
    }
    double beta = ro_dot(n, z, r), betaold = 0.0;

    for (int i = 0; i < cfg.max_it; ++i) {
        if (i == 0) {
            memcpy(p, z, (size_t)n * sizeof(double));
        } else {
            if (betaold == 0.0) {
                res.status = RO_BREAKDOWN;
                res.breakdown_iter = i;
                return res;
            }
            const double bb = beta / betaold;
            ro_aypx(n, bb, z, p);
        }
        ro_csr_spmv(n, off, cols, vals, p, w);
        const double pAp = ro_dot(n, p, w);
        const double a   = beta / pAp;
        if (pAp == 0.0 || !isfinite(a)) {
            res.status = RO_BREAKDOWN;
            res.breakdown_iter = i;
            return res;
        }
        betaold = beta;
        ro_axpy(n, a, p, x);
        ro_axpy(n, -a, w, r);
        if (cfg.pc == RO_PC_JACOBI) ro_pointwise_mult(n, dinv, r, z);
        else memcpy(z, r, (size_t)n * sizeof(double));
        dp          = ro_nrm2(n, z);
        hist[i + 1] = dp;
        res.iterations = i + 1;
        if (converged(dp, dp0, &cfg)) {
            res.status = RO_CONVERGED;
            return res;
        }
        beta = ro_dot(n, z, r);
    }
    return res;
}

/* ------------------------------------------------------------------------ */
/* TFQMR (see rvk_oracle.h).  B = Jacobi applied on the left: every operator
 * application is T1 = A v, out = dinv .* T1. */
static void apply_BA(int64_t n, const int64_t* off, const int32_t* cols, const double* vals,
                     const double* dinv, int pc, const double* v, double* t1, double* out)
{
    ro_csr_spmv(n, off, cols, vals, v, t1);
    if (pc == RO_PC_JACOBI) ro_pointwise_mult(n, dinv, t1, out);
    else memcpy(out, t1, (size_t)n * sizeof(double));
}

ro_cg_result ro_tfqmr_solve(int64_t n, const int64_t* off, const int32_t* cols,
                            const double* vals, const double* b, double* x,
                            double* hist, ro_cg_config cfg, double* work, int* n_hist)
{
    ro_cg_result res = {RO_OK, 0, -1};
    double *R = work, *RP = work + n, *U = work + 2 * n, *P = work + 3 * n, *V = work + 4 * n;
    double *D = work + 5 * n, *Q = work + 6 * n, *T = work + 7 * n, *AUQ = work + 8 * n;
    double *T1 = work + 9 * n, *dinv = work + 10 * n;
    const size_t bytes = (size_t)n * sizeof(double);
    *n_hist = 0;

    memset(x, 0, bytes);
    if (cfg.pc == RO_PC_JACOBI) {
        ro_csr_diagonal(n, off, cols, vals, dinv);
        for (int64_t i = 0; i < n; ++i) dinv[i] = 1.0 / dinv[i];
        ro_pointwise_mult(n, dinv, b, R); /* R = B (b - A x0), x0 = 0 */
    } else {
        memcpy(R, b, bytes);
    }
    double dp = ro_nrm2(n, R);
    hist[(*n_hist)++] = dp;
    const double dp0 = dp;
    if (converged(dp, dp0, &cfg)) {
        res.status = RO_CONVERGED;
        return res;
    }
    memcpy(RP, R, bytes);
    double etaold = 0.0, psiold = 0.0, tau = dp, dpold = dp;
    double rhoold = ro_dot(n, R, RP);
    memcpy(U, R, bytes);
    memcpy(P, R, bytes);
    apply_BA(n, off, cols, vals, dinv, cfg.pc, P, T1, V);
    memset(D, 0, bytes);

    for (int i = 0; i < cfg.max_it; ++i) {
        const double s = ro_dot(n, V, RP);
        if (s == 0.0) {
            res.status = RO_BREAKDOWN;
            res.breakdown_iter = i;
            return res;
        }
        const double a = rhoold / s;
        ro_waxpy(n, -a, V, U, Q);  /* q = u - a v       */
        ro_waxpy(n, 1.0, U, Q, T); /* t = u + q         */
        apply_BA(n, off, cols, vals, dinv, cfg.pc, T, T1, AUQ);
        ro_axpy(n, -a, AUQ, R);    /* r = r - a B A (u + q) */
        dp = ro_nrm2(n, R);
        for (int m = 0; m < 2; ++m) {
            const double w   = m == 0 ? sqrt(dp * dpold) : dp;
            const double psi = w / tau;
            const double cm  = 1.0 / sqrt(1.0 + psi * psi);
            tau              = tau * psi * cm;
            const double eta = cm * cm * a;
            const double cf  = psiold * psiold * etaold / a;
            ro_aypx(n, cf, m == 0 ? U : Q, D); /* d = (u|q) + cf d */
            ro_axpy(n, eta, D, x);             /* x = x + eta d    */
            /* residual bound ||r_k|| <= sqrt(k+1) tau_k, k = 2i+m+1 half steps */
            const double dpest = sqrt(2.0 * i + m + 2.0) * tau;
            hist[(*n_hist)++]  = dpest;
            if (converged(dpest, dp0, &cfg)) {
                res.status     = RO_CONVERGED;
                res.iterations = i + 1;
                return res;
            }
            etaold = eta;
            psiold = psi;
        }
        res.iterations = i + 1;
        const double rho = ro_dot(n, R, RP);
        if (rhoold == 0.0) {
            res.status = RO_BREAKDOWN;
            res.breakdown_iter = i;
            return res;
        }
        const double bb = rho / rhoold;
        ro_waxpy(n, bb, Q, R, U); /* u = r + b q        */
        ro_axpy(n, bb, P, Q);     /* q = q + b p        */
        ro_waxpy(n, bb, Q, U, P); /* p = u + b q        */
        apply_BA(n, off, cols, vals, dinv, cfg.pc, P, T1, V);
        rhoold = rho;
        dpold  = dp;
    }
    return res;
}
