/*
 * rvk_oracle_mt.c -- TEST INFRASTRUCTURE ONLY (see rvk_oracle.h).
 *
 * The restatement at the sizes a single host thread cannot finish in test
 * time (the BASELINE.json 768^3 config: n = 4.5e8, nnz = 3.2e9):
 *
 *  - ro_build_laplacian_rows: rows [r0, r1) of ro_build_laplacian's CSR,
 *    the same loop nest started at row r0, offsets local to
 *    the slab (off[0] = 0).  Bit-identical to the corresponding slice of the
 *    full build (tests/test_oracle.py), so a device CSR can be checked slab
 *    by slab without 41.6 GB on the host.
 *  - ro_stencil_spmv_mt: y = A x for the same Laplacian without storing it.
 *    Each row is summed from 0.0 over its neighbours in ascending column
 *    order with the same coefficients (centre points-1, neighbours -1), i.e.
 *    exactly ro_csr_spmv (kernels_scalar.cpp:53-63) on ro_build_laplacian's
 *    CSR: bit-identical (tests/test_oracle.py pins it on every stencil).
 *  - ro_cg_solve_stencil_mt: ro_cg_solve's loop (same op
 *    order, every element rounded as in kernels_scalar.cpp) over that SpMV,
 *    host threads across rows (pthreads).  Elementwise results are bit-identical per element;
 *    the three reductions per iteration are summed in kChunks fixed chunks
 *    (each a left-to-right chain) whose partials are then added in chunk
 *    order -- deterministic and independent of the thread count, but not the
 *    reference's single chain, so the history agrees with ro_cg_solve to
 *    rounding (pinned at <= 1e-13 relative on grids the serial oracle runs).
 *
 * Built -O2 -ffp-contract=off -pthread (no -march), like rvk_oracle.c.
 */
#include "rvk_oracle.h"

#include <math.h>
#include <pthread.h>
#include <string.h>
#include <unistd.h>

enum { kChunks = 4096, kMaxThreads = 64 };

/* ---- static parallel for over [0, count): thread t gets one contiguous
 * range; fn(ctx, begin, end) ------------------------------------------------ */
typedef void (*range_fn)(void* ctx, int64_t begin, int64_t end);
typedef struct {
    range_fn fn;
    void*    ctx;
    int64_t  begin, end;
} par_job;

static void* par_run(void* a)
{
    par_job* j = (par_job*)a;
    j->fn(j->ctx, j->begin, j->end);
    return NULL;
}

static int n_threads(void)
{
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    if (c < 1) c = 1;
    return c > kMaxThreads ? kMaxThreads : (int)c;
}

static void par_for(int64_t count, range_fn fn, void* ctx, int64_t serial_below)
{
    int T = n_threads();
    if (count < serial_below || T == 1) {
        fn(ctx, 0, count);
        return;
    }
    if (T > count) T = (int)count;
    pthread_t th[kMaxThreads];
    par_job   jobs[kMaxThreads];
    int       started[kMaxThreads];
    for (int t = 0; t < T; ++t) {
        jobs[t].fn    = fn;
        jobs[t].ctx   = ctx;
        jobs[t].begin = count * t / T;
        jobs[t].end   = count * (t + 1) / T;
        started[t]    = t > 0 && pthread_create(&th[t], NULL, par_run, &jobs[t]) == 0;
    }
    for (int t = 0; t < T; ++t)
        if (!started[t]) fn(ctx, jobs[t].begin, jobs[t].end); /* thread 0 (or a failed create) */
    for (int t = 1; t < T; ++t)
        if (started[t]) pthread_join(th[t], NULL);
}

static int in_stencil_mt(int points, int dx, int dy, int dz)
{
    if (points == 5 || points == 7) return (dx != 0) + (dy != 0) + (dz != 0) <= 1;
    return 1;
}

int64_t ro_build_laplacian_rows(int dim, int points, int64_t nx, int64_t ny, int64_t nz,
                                int64_t r0, int64_t r1, int64_t* off, int32_t* cols,
                                double* vals)
{
    if (!ro_stencil_valid(dim, points, nx, ny, nz)) return -1;
    if (dim == 2) nz = 1;
    const int64_t n = nx * ny * nz;
    if (r0 < 0 || r1 > n || r1 < r0) return -1;
    const int    zr     = dim == 3 ? 1 : 0;
    const double centre = (double)(points - 1);
    int64_t      k      = 0;
    off[0]              = 0;
    for (int64_t row = r0; row < r1; ++row) {
        const int64_t x = row % nx, y = (row / nx) % ny, z = row / (nx * ny);
        for (int dz = -zr; dz <= zr; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if (!in_stencil_mt(points, dx, dy, dz)) continue;
                    const int64_t xx = x + dx, yy = y + dy, zz = z + dz;
                    if (xx < 0 || xx >= nx || yy < 0 || yy >= ny || zz < 0 || zz >= nz) continue;
                    cols[k] = (int32_t)(xx + nx * (yy + ny * zz));
                    vals[k] = (dx == 0 && dy == 0 && dz == 0) ? centre : -1.0;
                    ++k;
                }
        off[row - r0 + 1] = k;
    }
    return k;
}

/* one row of the stencil product, ascending column order, from 0.0 */
static inline double stencil_row(int zr, int points, double centre, int64_t nx, int64_t ny,
                                 int64_t nz, int64_t x, int64_t y, int64_t z, int64_t row,
                                 const double* v)
{
    double sum = 0.0;
    for (int dz = -zr; dz <= zr; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                if (!in_stencil_mt(points, dx, dy, dz)) continue;
                const int64_t xx = x + dx, yy = y + dy, zz = z + dz;
                if (xx < 0 || xx >= nx || yy < 0 || yy >= ny || zz < 0 || zz >= nz) continue;
                const double a = (dx == 0 && dy == 0 && dz == 0) ? centre : -1.0;
                sum += a * v[row + dx + nx * (dy + ny * (int64_t)dz)];
            }
    return sum;
}

typedef struct {
    int           zr, points;
    double        centre;
    int64_t       nx, ny, nz;
    const double* x;
    double*       y;
} spmv_ctx;

static void spmv_lines(void* c, int64_t l0, int64_t l1)
{
    const spmv_ctx* S = (const spmv_ctx*)c;
    for (int64_t line = l0; line < l1; ++line) {
        const int64_t yy = line % S->ny, zz = line / S->ny;
        for (int64_t xx = 0; xx < S->nx; ++xx) {
            const int64_t row = xx + S->nx * line;
            S->y[row] = stencil_row(S->zr, S->points, S->centre, S->nx, S->ny, S->nz, xx, yy, zz, row, S->x);
        }
    }
}

void ro_stencil_spmv_mt(int dim, int points, int64_t nx, int64_t ny, int64_t nz, const double* x,
                        double* y)
{
    if (dim == 2) nz = 1;
    spmv_ctx S = {dim == 3 ? 1 : 0, points, (double)(points - 1), nx, ny, nz, x, y};
    par_for(ny * nz, spmv_lines, &S, 2);
}

/* sum_i x_i y_i in kChunks fixed chunks, partials added in chunk order */
typedef struct {
    int64_t       n, cs;
    const double *x, *y;
    double*       part;
} dot_ctx;

static void dot_chunks(void* c, int64_t c0, int64_t c1)
{
    const dot_ctx* D = (const dot_ctx*)c;
    for (int64_t k = c0; k < c1; ++k) {
        const int64_t a = k * D->cs, b = a + D->cs < D->n ? a + D->cs : D->n;
        double        s = 0.0;
        for (int64_t i = a; i < b; ++i) s += D->x[i] * D->y[i];
        D->part[k] = s;
    }
}

static double dot_chunked(int64_t n, const double* x, const double* y)
{
    double  part[kChunks];
    dot_ctx D = {n, (n + kChunks - 1) / kChunks, x, y, part};
    if (n < 65536) {
        dot_chunks(&D, 0, kChunks);
    } else {
        /* par_for splits chunk indices; count >= 65536 is needed to fan out */
        int T = n_threads();
        pthread_t th[kMaxThreads];
        par_job   jobs[kMaxThreads];
        int       started[kMaxThreads];
        for (int t = 0; t < T; ++t) {
            jobs[t] = (par_job){dot_chunks, &D, (int64_t)kChunks * t / T, (int64_t)kChunks * (t + 1) / T};
            started[t] = t > 0 && pthread_create(&th[t], NULL, par_run, &jobs[t]) == 0;
        }
        for (int t = 0; t < T; ++t)
            if (!started[t]) dot_chunks(&D, jobs[t].begin, jobs[t].end);
        for (int t = 1; t < T; ++t)
            if (started[t]) pthread_join(th[t], NULL);
    }
    double s = 0.0;
    for (int c = 0; c < kChunks; ++c) s += part[c];
    return s;
}

/* the elementwise steps of one CG phase */
typedef struct {
    int           step, jac;
    double        d, a, na, bb;
    const double* b;
    double *      x, *r, *z, *p, *w;
} ew_ctx;

static void ew_range(void* c, int64_t i0, int64_t i1)
{
    const ew_ctx* E = (const ew_ctx*)c;
    switch (E->step) {
    case 0: /* setup: x = 0, r = b, z = B r (pointwise_mult(dinv, r)) */
        for (int64_t i = i0; i < i1; ++i) {
            E->x[i] = 0.0;
            E->r[i] = E->b[i];
            E->z[i] = E->jac ? E->d * E->r[i] : E->r[i];
        }
        break;
    case 1: /* p = z (iteration 0) */
        for (int64_t i = i0; i < i1; ++i) E->p[i] = E->z[i];
        break;
    case 2: /* aypx: p = z + bb p */
        for (int64_t i = i0; i < i1; ++i) E->p[i] = E->z[i] + E->bb * E->p[i];
        break;
    case 3: /* axpy x += a p; axpy r += (-a) w; z = B r */
        for (int64_t i = i0; i < i1; ++i) {
            E->x[i] += E->a * E->p[i];
            E->r[i] += E->na * E->w[i];
            E->z[i] = E->jac ? E->d * E->r[i] : E->r[i];
        }
        break;
    }
}

ro_cg_result ro_cg_solve_stencil_mt(int dim, int points, int64_t nx, int64_t ny, int64_t nz,
                                    const double* b, double* x, double* hist, ro_cg_config cfg,
                                    double* work)
{
    ro_cg_result  res = {RO_OK, 0, -1};
    const int64_t n   = dim == 2 ? nx * ny : nx * ny * nz;
    double*       r   = work;
    double*       z   = work + n;
    double*       p   = work + 2 * n;
    double*       w   = work + 3 * n;
    /* dinv = 1 / diag: every row of the Laplacian holds the centre weight */
    const double  d   = 1.0 / (double)(points - 1);
    const int     jac = cfg.pc == RO_PC_JACOBI;
    ew_ctx        E   = {0, jac, d, 0.0, 0.0, 0.0, b, x, r, z, p, w};
    par_for(n, ew_range, &E, 65536);
    double dp = sqrt(dot_chunked(n, z, z));
    hist[0]   = dp;
    const double dp0 = dp;
    if (dp <= fmax(cfg.rtol * dp0, cfg.atol)) {
        res.status = RO_CONVERGED;
        return res;
    }
    double beta = dot_chunked(n, z, r), betaold = 0.0;
    for (int it = 0; it < cfg.max_it; ++it) {
        if (it == 0) {
            E.step = 1;
            par_for(n, ew_range, &E, 65536);
        } else {
            if (betaold == 0.0) {
                res.status         = RO_BREAKDOWN;
                res.breakdown_iter = it;
                return res;
            }
            E.step = 2;
            E.bb   = beta / betaold;
            par_for(n, ew_range, &E, 65536);
        }
        ro_stencil_spmv_mt(dim, points, nx, ny, nz, p, w);
        const double pAp = dot_chunked(n, p, w);
        const double a   = beta / pAp;
        if (pAp == 0.0 || !isfinite(a)) {
            res.status         = RO_BREAKDOWN;
            res.breakdown_iter = it;
            return res;
        }
        betaold = beta;
        E.step  = 3;
        E.a     = a;
        E.na    = -a;
        par_for(n, ew_range, &E, 65536);
        dp          = sqrt(dot_chunked(n, z, z));
        hist[it + 1] = dp;
        res.iterations = it + 1;
        if (dp <= fmax(cfg.rtol * dp0, cfg.atol)) {
            res.status = RO_CONVERGED;
            return res;
        }
        beta = dot_chunked(n, z, r);
    }
    return res;
}
