/*
 * rvk.h -- C ABI of the B200-native Jacobi-CG path (librvk.so).
 *
 * This is the drop-in boundary between the reference's C++ Vec/Mat/KSP-style
 * API (include/rivulet/ headers here, mirroring /root/reference/proj/include/
 * rivulet/linalg.hpp:48-78) and hand-written sm_100a kernels.  Plain C types
 * only: pointers, sizes, an opaque context handle.  No torch types.
 *
 * Conventions
 *  - Every entry point returns an rvk_status (0 = RVK_OK).  On failure the
 *    thread-local message is available from rvk_last_error().
 *  - Pointers named *_dev are device pointers owned by the caller; *_host are
 *    host pointers (pinned or pageable).
 *  - Every compute entry point is ASYNCHRONOUS and stream-ordered on the
 *    rvk_ctx's CUDA stream: it never blocks the host.  The only host
 *    synchronisations are the explicitly named ones (rvk_ctx_synchronize,
 *    rvk_scalar_read, rvk_cg_result, rvk_cg_solve_host, rvk_*_plan_create);
 *    each is counted in rvk_host_sync_count(), mirroring trace::host_sync
 *    (reference trace.hpp:40-41, managed.cpp:74-84).
 *  - Reductions write their result to DEVICE memory (the paper's fix for the
 *    "scalar problem"), in a fixed order, so results are
 *    bit-reproducible run to run.
 *  - Elementwise ops and SpMV compute every element with IEEE mul-then-add
 *    (no FMA), in the reference's operand order, so they are bit-identical to
 *    rivulet::kernels::scalar (kernels_scalar.cpp:24-63).
 */
#ifndef RVK_H
#define RVK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RVK_ABI_VERSION 2

typedef enum {
    RVK_OK             = 0,
    RVK_ERR_INVALID    = 1, /* bad argument / invalid spec                     */
    RVK_ERR_DIM        = 2, /* dimension mismatch    */
    RVK_ERR_CUDA       = 3, /* CUDA runtime error                              */
    RVK_ERR_ALLOC      = 4, /* device / pinned allocation failed               */
    RVK_ERR_BREAKDOWN  = 5, /* Krylov breakdown (common.hpp:33-43)             */
    RVK_ERR_COMM       = 6, /* NCCL / communicator error                       */
    RVK_ERR_UNSUPPORTED = 7
} rvk_status;

/* Thread-local description of the last failure on this thread. */
const char* rvk_last_error(void);
int         rvk_abi_version(void);
/* sha256 (16 hex digits) of the library's sources: profiles record it, so a
 * bench run can tell whether committed ncu numbers came from this code. */
const char* rvk_build_id(void);
/* Number of SMs / name of the calling thread's current device (setup helper). */
int         rvk_device_info(int* sm_count, char* name, int name_len);
/* Device selection for the calling thread (cudaGetDeviceCount /
 * cudaSetDevice): contexts, vectors and plans created afterwards on this
 * thread live on that device.  One process may drive several GPUs (e.g. one
 * host thread per device); kernel attributes and per-device caches are kept
 * per device. */
int         rvk_device_count(void);
rvk_status  rvk_set_device(int device);

/* ---- context: a CUDA stream + reduction scratch (PetscDeviceContext) -----
 * Replaces rivulet::Context's agent-thread queue (context.hpp:75-114;
 * context.cpp:151-232).  A ctx created with cuda_stream == NULL owns a new
 * non-blocking stream; otherwise it wraps the caller's stream. */
typedef struct rvk_ctx_s* rvk_ctx;
rvk_status rvk_ctx_create(void* cuda_stream, rvk_ctx* out);
rvk_status rvk_ctx_destroy(rvk_ctx ctx);                 /* drains first */
void*      rvk_ctx_stream(rvk_ctx ctx);                  /* the cudaStream_t          */
rvk_status rvk_ctx_synchronize(rvk_ctx ctx);             /* context.hpp:96-99; counted */
rvk_status rvk_ctx_query_idle(rvk_ctx ctx, int* idle);   /* context.hpp:92; no block   */
/* wait_for (context.hpp:88-90): future work on `waiter` starts after all
 * work enqueued on `waitee` so far.  Self-wait is a no-op. */
rvk_status rvk_ctx_wait_for(rvk_ctx waiter, rvk_ctx waitee);
/* Process-unique id and a display name (context.hpp:80-86 id()/name()): the
 * trace's context rows. */
uint64_t   rvk_ctx_id(rvk_ctx ctx);
rvk_status rvk_ctx_set_name(rvk_ctx ctx, const char* name);

/* ---- host-sync accounting (trace.hpp:40-41 HostSync events) ------------- */
uint64_t rvk_host_sync_count(void);
void     rvk_host_sync_reset(void);

/* ---- tracing (trace.hpp:11-46, trace.cpp:48-104) ------------------------
 * Task events: every solve / vector op / SpMV / assembly enqueued through
 * this ABI and every C++-API kernel launch, timed ON THE DEVICE (two timing
 * events on the context's stream, mapped onto the host steady clock when the
 * trace is read; inside a stream capture the host enqueue time is logged
 * instead).  HostSync events: every counted host wait, with its duration.
 * Wait events: cross-context ordering edges.  Marker: user annotations.
 * Every task and host wait is also an NVTX range (names as in the trace).
 * Reading the trace (count / write) waits for the traced device work; it is
 * not counted as a host sync.  Off by default; recording costs nothing then
 * beyond the NVTX push/pop. */
void       rvk_trace_enable(int on);        /* trace::set_enabled */
int        rvk_trace_enabled(void);
void       rvk_trace_clear(void);
void       rvk_trace_marker(const char* label);
size_t     rvk_trace_count(void);           /* events recorded so far */
/* One JSON object per line, the reference's keys (trace.cpp:90-100):
 * task, enqueue_seq, ctx, ctx_name, label, kind, blocked, start, end (ns),
 * plus device_timed. */
rvk_status rvk_trace_write_jsonl(const char* path);
/* Chrome trace-event JSON (chrome://tracing / Perfetto timeline). */
rvk_status rvk_trace_write_chrome(const char* path);

/* ---- device memory (plumbing) -------------------------------------------- */
rvk_status rvk_malloc(void** dev, size_t bytes);
rvk_status rvk_free(void* dev);
/* stream-ordered (cudaMallocAsync pool): valid for work enqueued on ctx after
 * the call; freed after the work enqueued before rvk_free_async -- the
 * deferred release of managed_state.hpp:13-15 / dual_buffer.cpp:9-17 */
rvk_status rvk_malloc_async(rvk_ctx ctx, void** dev, size_t bytes);
rvk_status rvk_free_async(rvk_ctx ctx, void* dev);
rvk_status rvk_host_alloc(void** host, size_t bytes);    /* pinned */
rvk_status rvk_host_free(void* host);
rvk_status rvk_memcpy_h2d(rvk_ctx ctx, void* dst_dev, const void* src_host, size_t bytes);
rvk_status rvk_memcpy_d2h(rvk_ctx ctx, void* dst_host, const void* src_dev, size_t bytes);
rvk_status rvk_memcpy_d2d(rvk_ctx ctx, void* dst_dev, const void* src_dev, size_t bytes);

/* ---- scalar arguments: detail::ScalarArg (linalg.hpp:17-38) --------------
 * A constant, a device scalar, its negation, or a ratio of two device
 * scalars: exactly the expression shapes the CG listing passes to a
 * consuming kernel.  Evaluated inside the kernel;
 * the value never visits the host. */
typedef enum {
    RVK_SCALAR_CONST       = 0, /* c                                   */
    RVK_SCALAR_PTR         = 1, /* *p0                                 */
    RVK_SCALAR_NEG_PTR     = 2, /* -(*p0)                              */
    RVK_SCALAR_DIV_PTR_PTR = 3, /* (*p0) / (*p1)                       */
    RVK_SCALAR_SQRT_PTR    = 4, /* sqrt(*p0)                           */
    RVK_SCALAR_RECIP_PTR   = 5  /* 1.0 / (*p0)  (normalize) */
} rvk_scalar_kind;

typedef struct {
    int           kind;
    double        c;
    const double* p0;
    const double* p1;
} rvk_scalar;

/* out_dev = value of `s` (Eval(expr, ctx).execute(out), expr.cpp:314-386,
 * restricted to the scalar shapes above). */
rvk_status rvk_scalar_eval(rvk_ctx ctx, rvk_scalar s, double* out_dev);
/* Host read of a device scalar: Managed::front() (managed.cpp:86-91).
 * Synchronises the context; counted as one host sync. */
rvk_status rvk_scalar_read(rvk_ctx ctx, const double* s_dev, double* out_host);

/* ---- Vec kernels (linalg.hpp:48-66; kernels.hpp:38-48) ------------------ */
rvk_status rvk_dot(rvk_ctx ctx, int64_t n, const double* x, const double* y, double* out_dev);
rvk_status rvk_nrm2(rvk_ctx ctx, int64_t n, const double* x, double* out_dev);
/* fused pair: zz = z.z, zr = z.r in one pass */
rvk_status rvk_dot2(rvk_ctx ctx, int64_t n, const double* z, const double* r,
                    double* zz_dev, double* zr_dev);
rvk_status rvk_axpy(rvk_ctx ctx, int64_t n, rvk_scalar a, const double* x, double* y);  /* y += a*x   */
rvk_status rvk_aypx(rvk_ctx ctx, int64_t n, rvk_scalar b, const double* x, double* y);  /* y = x + b*y */
rvk_status rvk_waxpy(rvk_ctx ctx, int64_t n, rvk_scalar a, const double* x, const double* y,
                     double* w);                                                      /* w = a*x + y */
rvk_status rvk_scale(rvk_ctx ctx, int64_t n, rvk_scalar a, double* x);                  /* x *= a     */
rvk_status rvk_pointwise_mult(rvk_ctx ctx, int64_t n, const double* a, const double* b,
                              double* out);                                           /* out = a.*b */
rvk_status rvk_copy(rvk_ctx ctx, int64_t n, const double* src, double* dst);
rvk_status rvk_set(rvk_ctx ctx, int64_t n, double value, double* x);

/* ---- Mat: CSR (csr.hpp:19-85) -------------------------------------------
 * int64 row offsets, int32 column indices, double values, all on device.
 * Columns strictly increasing within a row (csr.hpp:51-53). */
typedef struct {
    int64_t        n_rows;
    int64_t        n_cols;
    int64_t        nnz;
    const int64_t* row_offsets;
    const int32_t* col_indices;
    const double*  values;
} rvk_csr;

/* y = A x (mat_mult, linalg.hpp:68-69; kernels_scalar.cpp:53-63): per-row
 * left-to-right sum from 0.0, mul-then-add => bit-identical to the reference. */
rvk_status rvk_csr_spmv(rvk_ctx ctx, const rvk_csr* A, const double* x, double* y);
/* diag = diagonal() (csr.hpp:76-77; zero where absent); dinv = 1/diag. */
rvk_status rvk_csr_diagonal(rvk_ctx ctx, const rvk_csr* A, double* diag);
rvk_status rvk_csr_diagonal_inverse(rvk_ctx ctx, const rvk_csr* A, double* dinv);
/* Structural validation (csr.hpp:46-53 contract).  Synchronises (setup).
 * Also returns the maximum row length. */
rvk_status rvk_csr_validate(rvk_ctx ctx, const rvk_csr* A, int64_t* max_row_len);

/* ---- stencil assembly on device --- */
rvk_status rvk_laplacian_size(int dim, int points, int64_t nx, int64_t ny, int64_t nz,
                              int64_t* n_rows, int64_t* nnz);
/* Fills caller-allocated device arrays off[n+1], cols[nnz], vals[nnz];
 * bit-identical to the CPU builder (lexicographic, x fastest, ascending
 * columns, Dirichlet by truncation, centre = points-1, neighbours -1). */
rvk_status rvk_build_laplacian(rvk_ctx ctx, int dim, int points, int64_t nx, int64_t ny,
                               int64_t nz, int64_t* off_dev, int32_t* cols_dev,
                               double* vals_dev);
/* Synthetic RHS b_i = (splitmix64(seed+i)>>11)*2^-52 - 1. */
rvk_status rvk_fill_rhs(rvk_ctx ctx, uint64_t seed, int64_t n, double* b_dev);

/* ---- KSP: Jacobi-preconditioned CG --- */
typedef enum { RVK_PC_NONE = 0, RVK_PC_JACOBI = 1 } rvk_pc;
typedef enum {
    RVK_CG_MODE_FUSED      = 0, /* 2 fused kernels per iteration, device tails (default) */
    RVK_CG_MODE_UNFUSED    = 1, /* the reference's op-per-kernel sequence               */
    RVK_CG_MODE_PERSISTENT = 2, /* whole solve in ONE cooperative kernel (L2-sized grids) */
    RVK_CG_MODE_AUTO       = 3, /* PERSISTENT when the working set fits L2, else FUSED   */
    RVK_CG_MODE_HOSTSYNC   = 4  /* baseline: every dot/norm read back to the host (3 syncs
                                   per iteration, PETSc main_gpu behaviour) */
} rvk_cg_mode;
typedef enum {
    RVK_CG_RUNNING    = 0,
    RVK_CG_CONVERGED  = 1,
    RVK_CG_BREAKDOWN  = 2,
    RVK_CG_COMM_ERROR = 3 /* row-sharded PEER backend: a peer never arrived (bounded wait) */
} rvk_cg_state;

typedef struct {
    int    max_it;    /* SPEC.md:444 default 20                                  */
    int    pc;        /* rvk_pc                                                  */
    double rtol;      /* converged if dp <= max(rtol*dp0, atol); 0,0 => only 0   */
    double atol;
    int    mode;      /* rvk_cg_mode                                             */
    int    use_graph; /* 1: the whole solve as one CUDA graph (max_it iterations
                         unrolled, replayed); 2: graph with a device-side WHILE
                         node -- no launches after convergence (FUSED only);
                         0: plain stream launches                             */
    int    opts;      /* RVK_OPT_* bits, 0 = the plan's own choices (below)  */
} rvk_cg_config;

/* Plan variant overrides (rvk_cg_config.opts).  The plan picks the fastest
 * measured variant by itself; these select the others explicitly (parity
 * tests exercise every variant; none changes a result bit except where
 * noted).  Read once at plan creation -- nothing is read from the
 * environment.
 *   RVK_OPT_KEEP_WORK    the last K2 of a fixed-iteration fused solve still
 *                        stores r and z, so rvk_cg_plan_vector(R / Z) is the
 *                        final residual (otherwise both are undefined after a
 *                        fused solve: dead stores are skipped)
 *   RVK_OPT_DINV_VECTOR  keep streaming the Jacobi diagonal even when it is one
 *                        constant (no RVK_PLAN_CONST_DIAG folding)
 *   RVK_OPT_Z_STORED     never use the virtual z (z = d r formed in the SpMV)
 *   RVK_OPT_Z_VIRTUAL    use the virtual z wherever it is legal (default: only
 *                        where it measured faster -- 9-batch CSR, matrix-free)
 *   RVK_OPT_NO_CLUSTER   PERSISTENT mode: grid-barrier kernel instead of the
 *                        one-cluster DSMEM solve
 *   RVK_OPT_SMALL_K1     FUSED mode: plain-block SpMV (k_spmv_small) for
 *                        systems up to 512 K rows (AUTO picks it itself)
 *   RVK_OPT_MF_SIMPLE    matrix-free plans: the one-row-per-thread stencil
 *                        kernel instead of the TMA 2.5D march
 *   RVK_OPT_NO_FOLD      fixed-iteration fused CSR solves keep the separate
 *                        setup kernel (no RVK_PLAN_FOLD_SETUP)
 *   RVK_OPT_X_GROUP4     fused solve: x updated per group of 4 iterations
 *                        instead of once per solve (RVK_PLAN_X_SOLVE)
 *   RVK_OPT_X_EACH       fused solve: x updated in every iteration's K2
 *   RVK_OPT_MARCH        CSR plans with a plane structure: the plane-marching
 *                        K1 (RVK_PLAN_MARCH; opt-in)
 *   RVK_OPT_NO_GRID      PERSISTENT mode: no one-launch grid solve for mid-size
 *                        systems (the generic grid-barrier kernel instead)
 *   RVK_OPT_NO_GRID_L2   no grid solve over the global ELL copy (RVK_PLAN_GRID_L2):
 *                        AUTO runs those systems as the fused graph
 *   RVK_OPT_FPERSIST     AUTO: the fused persistent solve (RVK_PLAN_FPERSIST) for
 *                        fixed-iteration solves past the grid solves (opt-in:
 *                        measured level with / slower than the fused graph)
 *   RVK_OPT_NO_FPERSIST  never the fused persistent solve                      */
#define RVK_OPT_KEEP_WORK   1
#define RVK_OPT_DINV_VECTOR 2
#define RVK_OPT_Z_STORED    4
#define RVK_OPT_Z_VIRTUAL   8
#define RVK_OPT_NO_CLUSTER  16
#define RVK_OPT_SMALL_K1    32
#define RVK_OPT_MF_SIMPLE   64
#define RVK_OPT_NO_FOLD     128
#define RVK_OPT_X_GROUP4    256
#define RVK_OPT_X_EACH      512
#define RVK_OPT_MARCH       1024
#define RVK_OPT_NO_GRID     4096
#define RVK_OPT_NO_GRID_L2  8192
#define RVK_OPT_FPERSIST    16384
#define RVK_OPT_NO_FPERSIST 32768

typedef struct {
    int state;          /* rvk_cg_state: RUNNING here means "ran max_it"     */
    int iterations;     /* completed iterations: hist[0..iterations] valid   */
    int breakdown_iter; /* iteration index of breakdown, -1 if none          */
} rvk_cg_info;

typedef struct rvk_cg_plan_s* rvk_cg_plan;

/* KSPSetUp analogue: validates A (one sync), computes dinv on device, sizes
 * the SpMV tiles, allocates the work vectors r, z, p0, p1, w. */
rvk_status rvk_cg_plan_create(rvk_ctx ctx, const rvk_csr* A_dev, rvk_cg_config cfg,
                              rvk_cg_plan* out);
/* Matrix-free variant (PETSc MatShell analogue): the
 * same constant-coefficient stencil rvk_build_laplacian assembles, applied
 * on the fly -- no CSR bytes, constant Jacobi diagonal.  Element arithmetic
 * and neighbour order are those of the assembled CSR (bit-identical w).
 * FUSED / AUTO mode only. */
rvk_status rvk_cg_plan_create_stencil(rvk_ctx ctx, int dim, int points, int64_t nx, int64_t ny,
                                      int64_t nz, rvk_cg_config cfg, rvk_cg_plan* out);
rvk_status rvk_cg_plan_destroy(rvk_cg_plan plan);
/* Enqueue one full solve (x0 = 0, r0 = b; max_it iterations or device-side
 * convergence/breakdown exit).  ZERO host synchronisations. */
rvk_status rvk_cg_solve_dev(rvk_cg_plan plan, const double* b_dev, double* x_dev);
/* Device pointer to the residual history hist[0..max_it] (||z_k||_2). */
const double* rvk_cg_history_dev(rvk_cg_plan plan);
/* Synchronise and read hist (max_it+1 doubles, may be NULL) and info;
 * returns RVK_ERR_BREAKDOWN if the solve broke down.  One counted sync. */
rvk_status rvk_cg_result(rvk_cg_plan plan, double* hist_host, rvk_cg_info* info);
/* End-to-end: copy b from host, solve, copy x and hist back, one sync. */
rvk_status rvk_cg_solve_host(rvk_cg_plan plan, const double* b_host, double* x_host,
                             double* hist_host, rvk_cg_info* info);
/* Many right-hand sides from host memory (KSPMatSolve-like stream of solves
 * with one operator): x_host[k] = A^-1 b_host[k].  H2D of the next b and
 * D2H of the previous x overlap the current solve on copy streams (double-
 * buffered staging; pinned host buffers required for overlap).  hist_host:
 * nrhs*(max_it+1) doubles (may be NULL); infos: nrhs entries (may be NULL).
 * One host sync at the end; RVK_ERR_BREAKDOWN if any right-hand side broke
 * down (infos tell which). */
rvk_status rvk_cg_solve_host_many(rvk_cg_plan plan, int nrhs, const double* const* b_host,
                                  double* const* x_host, double* hist_host, rvk_cg_info* infos);
/* Plan structure the solve exploits (bitmask):
 *   RVK_PLAN_CONST_DIAG   every diagonal entry is the same bit pattern (constant-
 *                         coefficient stencils): Jacobi uses the scalar, no dinv
 *                         stream (RVK_OPT_DINV_VECTOR disables)
 *   RVK_PLAN_MATRIX_FREE  rvk_cg_plan_create_stencil operator                       */
#define RVK_PLAN_CONST_DIAG  1
#define RVK_PLAN_MATRIX_FREE 2
#define RVK_PLAN_MF_TMA      4  /* matrix-free K1 is the TMA 2.5D marching kernel (RVK_OPT_MF_SIMPLE: not) */
#define RVK_PLAN_X_DEFER    16  /* fused solve applies x += a p for a GROUP of iterations in one
                                   pass (16-B aligned b / x; bit-identical x)                  */
#define RVK_PLAN_X_GROUP4   64  /* ... groups of 4 iterations (max_it > 32, p ring does not fit,
                                   or the device WHILE loop)                                   */
#define RVK_PLAN_FOLD_SETUP 512 /* fixed-iteration fused CSR solve (use_graph 0/1, 16-B aligned b):
                                   the setup runs inside K1(0) (z = d b per gathered column;
                                   RVK_OPT_NO_FOLD disables)                                   */
#define RVK_PLAN_CLUSTER    256 /* PERSISTENT / AUTO plan runs the one-cluster DSMEM solve (<= 16 K rows,
                                   rows <= 9 entries; RVK_OPT_NO_CLUSTER disables)              */
#define RVK_PLAN_X_SOLVE    128 /* ... one group = the whole fixed-iteration solve: x is written
                                   once, at the end (5 <= max_it <= 32, p buffers fit)          */
#define RVK_PLAN_MARCH      1024 /* fused CSR K1 (iterations >= 1) is the plane-marching SpMV:
                                    each SM owns an in-plane row range and walks it through
                                    the planes, the formed gathered operand of planes k-1,
                                    k, k+1 cached in shared memory (RVK_OPT_MARCH)       */
#define RVK_PLAN_GRID       2048 /* PERSISTENT / AUTO plan runs the one-launch grid solve (16 K < n <=
                                    ~450 K rows, rows <= 9 entries): CSR in shared memory, row
                                    vectors in registers, 2 grid barriers per iteration
                                    (RVK_OPT_NO_GRID disables)                                  */
#define RVK_PLAN_GRID_L2    4096 /* ... for 3 K - 8 K rows per CTA (up to 148 x 8 K rows; 1024^2):
                                    the matrix from a plan-owned k-major ELL copy in global
                                    memory (L2-resident), x / r / p in shared memory
                                    (RVK_OPT_NO_GRID_L2 disables)                               */
#define RVK_PLAN_FPERSIST   8192 /* PERSISTENT / AUTO plan runs the fused persistent solve: each
                                    iteration's SpMV (the TMA ring of the fused K1, kept
                                    across iterations) and update phases in ONE cooperative
                                    launch, grid barriers fused with the reductions (explicit
                                    PERSISTENT past the grid solves, or RVK_OPT_FPERSIST for
                                    fixed-iteration AUTO solves; rows <= 9 entries)             */
#define RVK_PLAN_Z_VIRTUAL  32  /* fused solve never stores z = d r (constant diagonal / no PC):
                                   the SpMV gathers r and forms d r (bit-identical;
                                   RVK_OPT_Z_STORED / RVK_OPT_Z_VIRTUAL override)               */
int        rvk_cg_plan_flags(rvk_cg_plan plan);
/* Test hook (the reference's "exposed for equivalence tests" spirit,
 * kernels.hpp:50-76): device pointer of a plan work vector after a solve.
 * p0 / p1 are the first two buffers of the plan's p ring (iteration k writes
 * p[(k+1) % ring]).  R and Z hold the final residual only when the plan was
 * created with RVK_OPT_KEEP_WORK (a fixed-iteration fused solve skips the
 * last, dead r / z stores); Z is also unused under RVK_PLAN_Z_VIRTUAL. */
enum { RVK_VEC_R = 0, RVK_VEC_Z = 1, RVK_VEC_P0 = 2, RVK_VEC_P1 = 3, RVK_VEC_W = 4 };
const double* rvk_cg_plan_vector(rvk_cg_plan plan, int which);
/* The mode the plan runs (AUTO resolved to FUSED or PERSISTENT). */
int        rvk_cg_plan_mode(rvk_cg_plan plan);
/* Per-kernel event timing of the last solve's dominant kernels (bench): */
rvk_status rvk_cg_set_profiling(rvk_cg_plan plan, int on);
rvk_status rvk_cg_kernel_times(rvk_cg_plan plan, float* spmv_ms, float* update_ms,
                               int* launches);

/* ---- KSP: left-Jacobi TFQMR --------
 * Freund's transpose-free QMR in PETSc KSPSolve_TFQMR operation order
 * (oracle/rvk_oracle.c:ro_tfqmr_solve): two B*A products and three
 * reductions per outer iteration, all scalars device-resident, zero host
 * syncs.  cfg.mode is ignored; cfg.use_graph 1 captures the whole solve as
 * one CUDA graph.  hist holds 2*max_it+1 doubles: ||B r0|| then the
 * residual bound sqrt(2i+m+2)*tau after half step m of outer iteration i. */
typedef struct rvk_tfqmr_plan_s* rvk_tfqmr_plan;
rvk_status rvk_tfqmr_plan_create(rvk_ctx ctx, const rvk_csr* A_dev, rvk_cg_config cfg,
                                 rvk_tfqmr_plan* out);
rvk_status rvk_tfqmr_plan_destroy(rvk_tfqmr_plan plan);
rvk_status rvk_tfqmr_solve_dev(rvk_tfqmr_plan plan, const double* b_dev, double* x_dev);
/* Synchronise; hist_host (2*max_it+1 doubles, may be NULL), *n_hist = valid
 * entries, info.iterations = outer iterations.  RVK_ERR_BREAKDOWN on
 * (v, rp) == 0 or rho_old == 0. */
rvk_status rvk_tfqmr_result(rvk_tfqmr_plan plan, double* hist_host, int* n_hist,
                            rvk_cg_info* info);
/* RVK_PLAN_CONST_DIAG when the fused kernels use the constant Jacobi
 * diagonal as a scalar (bit-identical; no dinv stream); -1 on a null plan. */
int        rvk_tfqmr_plan_flags(rvk_tfqmr_plan plan);

/* ---- row sharding across GPUs -----------------------------
 * The global grid is split into contiguous slabs of planes; shard `rank`
 * owns n_own rows and keeps one halo plane (halo_lo / halo_hi rows, 0 at the
 * outer boundary) on each interior side of the gathered vectors.  Its local
 * CSR has n_own rows and halo_lo + n_own + halo_hi columns. */
typedef struct rvk_comm_s*     rvk_comm;
typedef struct rvk_dcg_plan_s* rvk_dcg_plan;
typedef struct {
    int64_t n_own, halo_lo, halo_hi;
    int     rank, nranks;
} rvk_shard;

/* Rows [row_begin, row_end) of the stencil operator, offsets rebased to 0,
 * columns shifted by -col_shift (device arrays, caller-allocated). */
rvk_status rvk_laplacian_rows_nnz(int dim, int points, int64_t nx, int64_t ny, int64_t nz,
                                  int64_t row_begin, int64_t row_end, int64_t* nnz);
rvk_status rvk_build_laplacian_rows(rvk_ctx ctx, int dim, int points, int64_t nx, int64_t ny,
                                    int64_t nz, int64_t row_begin, int64_t row_end,
                                    int64_t col_shift, int64_t* off_dev, int32_t* cols_dev,
                                    double* vals_dev);
/* NCCL communicator (libnccl.so.2 resolved at run time).  The 128-byte
 * unique id is produced on rank 0 and broadcast by the caller. */
rvk_status rvk_comm_unique_id(void* id_out, int id_bytes);
rvk_status rvk_comm_init(const void* id, int nranks, int rank, rvk_comm* out);
rvk_status rvk_comm_destroy(rvk_comm comm);
/* The communicator's size and this process's rank as NCCL reports them
 * (ncclCommCount / ncclCommUserRank). */
rvk_status rvk_comm_size(rvk_comm comm, int* nranks, int* rank);
/* comm != NULL: NCCL backend.  comm == NULL with nranks > 1: either a
 * LOOPBACK shard (all shards on one device, sharing `shared_gather`,
 * 4*nranks doubles, solved by rvk_dcg_loopback_solve) or, with
 * shared_gather == NULL, a PEER shard (rvk_dcg_attach_peers below). */
rvk_status rvk_dcg_plan_create(rvk_ctx ctx, const rvk_csr* A_local, rvk_shard shard,
                               rvk_cg_config cfg, rvk_comm comm, double* shared_gather,
                               rvk_dcg_plan* out);
rvk_status rvk_dcg_plan_destroy(rvk_dcg_plan plan);
/* One shard per process: halo exchange (ncclSend/Recv) + partial-sum
 * allgather, or the PEER kernels, all stream-ordered -- zero host syncs.
 * cfg.use_graph != 0: the solve is captured once per (b, x) into a CUDA
 * graph (thread-local capture mode: any synchronous call made by the
 * enqueuing thread invalidates the capture) and replayed.  rvk_dcg_result also reports a
 * pending NCCL asynchronous communicator error (RVK_ERR_COMM). */
rvk_status rvk_dcg_solve_dev(rvk_dcg_plan plan, const double* b_own, double* x_own);
rvk_status rvk_dcg_loopback_solve(rvk_dcg_plan* plans, int nplans, const double* const* b_own,
                                  double* const* x_own);
rvk_status rvk_dcg_result(rvk_dcg_plan plan, double* hist_host, rvk_cg_info* info);
int        rvk_dcg_plan_flags(rvk_dcg_plan plan); /* RVK_PLAN_* bits (CONST_DIAG, X_DEFER, X_SOLVE) */

/* PEER backend (NVLink P2P; the fused compute+communication path).  Each
 * plan owns one device window [z | p0 | p1 | flags | gather slots]; once
 * every rank's window is mapped (own window as is, peers' via the cudaIpc
 * helpers below) and attached, rvk_dcg_solve_dev runs 2 kernels per
 * iteration that push the halo planes of z and p straight into the
 * neighbours' windows while computing them, broadcast the dot partials and
 * synchronise on per-rank arrival flags (bounded wait; RVK_ERR_COMM from
 * rvk_dcg_result if a peer never arrives).  Create the plan with comm = NULL
 * and shared_gather = NULL.  All ranks must attach before any rank solves,
 * and stay alive until every rank finished its last solve (barrier, then
 * destroy).  With every window on ONE device (windows of plans in one
 * process) the same kernels run as a PEER loopback (rvk_dcg_loopback_solve). */
rvk_status rvk_dcg_window(rvk_dcg_plan plan, void** base_dev, size_t* bytes);
rvk_status rvk_dcg_attach_peers(rvk_dcg_plan plan, void* const* windows, const rvk_shard* shards);
/* cudaIpc plumbing for the windows (64-byte handles). */
rvk_status rvk_ipc_get_handle(const void* dev_base, void* handle_out, int handle_bytes);
rvk_status rvk_ipc_open_handle(const void* handle, void** dev_ptr);
rvk_status rvk_ipc_close_handle(void* dev_ptr);

#ifdef __cplusplus
}
#endif
#endif
