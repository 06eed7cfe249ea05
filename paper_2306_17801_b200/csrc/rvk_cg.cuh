// rvk_cg.cuh -- pieces shared by the single-GPU (rvk_cg.cu) and the
// row-sharded (rvk_dcg.cu) Jacobi-CG.
#pragma once

#include "rvk_common.cuh"

namespace rvk {

// Device-resident solver scalars (the reference's Managed a, b, beta,
// betaold, dp of PAPER.md:108-109) plus the exit state.
// Most x updates one fused solve may defer (p buffers a plan may rotate).
constexpr int kMaxXq = 32;

struct CgState {
    double beta, betaold, alpha, pAp, dp0, dp;
    int    done, state, iterations, breakdown_iter;
    int    comm_error; // row-sharded PEER backend: a flag wait timed out
    unsigned int seq;  // row-sharded PEER backend: solves started on this plan
    double pend_alpha; // row-sharded CG: x += pend_alpha * p_{pend_it} not yet applied
    int    x_pending, pend_it; // pending x updates (count) and the first one's iteration
    double pend_a[kMaxXq]; // fused CG: a of the x updates deferred within the current group
};

constexpr int kUpdThreads = 256;

__device__ __forceinline__ bool cg_converged(double dp, double dp0, double rtol, double atol)
{
    return dp <= fmax(rtol * dp0, atol);
}

// Largest grid that is fully resident (one wave): blocks/SM from the
// occupancy calculator times the SM count.  Grid-stride kernels launched with
// more blocks than this run a second, equally long wave.
template <class K>
int resident_grid(K kernel, int threads, int64_t n_items)
{
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    const int64_t want = (n_items + threads - 1) / threads;
    const int64_t cap  = (int64_t)sm_count() * per_sm;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

// ---------------------------------------------------------------------------
// K1 op: p_new = z + b p_old on the fly; w = A p_new; tail alpha.
// ZV ("virtual z"): the Jacobi diagonal is one value d (or there is no
// preconditioner, d = 1), so z is never stored -- `z` points at r and every
// gathered z_j = d * r_j is formed here, the same single rounding K2 would
// have stored (bit-identical), saving the 8 n-byte z write per iteration.
// ---------------------------------------------------------------------------
template <bool FIRST, bool ZV = false>
struct CgSpmvOp {
    static constexpr bool kHasTail = true;
    static constexpr bool kFirst   = FIRST;
    static constexpr bool kZv      = ZV;
    const double* __restrict__ z; // ZV: r
    const double* __restrict__ p_old;
    double* __restrict__ p_new;
    double* __restrict__ w;
    CgState* st;
    int64_t  n;
    int      it;
    double   b;       // set by init()
    double   zs = 1.0; // ZV: the constant Jacobi diagonal d
    __device__ __forceinline__ double zval(double raw) const { return ZV ? mul(zs, raw) : raw; }

    __device__ __forceinline__ bool init()
    {
        if (st->done) return false;
        if (it < 0) it = st->iterations; // device WHILE loop: the iteration index lives on device
        if (!FIRST) {
            const double bo = st->betaold;
            if (bo == 0.0) { // breakdown in beta/betaold
                if (blockIdx.x == 0 && threadIdx.x == 0) {
                    st->state          = RVK_CG_BREAKDOWN;
                    st->breakdown_iter = it;
                    st->done           = 1;
                }
                return false;
            }
            b = st->beta / bo;
        }
        return true;
    }
    struct Fetch {
        double z, p;
    };
    __device__ __forceinline__ int           num_src() const { return FIRST ? 1 : 2; }
    __device__ __forceinline__ const double* src_ptr(int k) const { return k == 0 ? z : p_old; }
    __device__ __forceinline__ Fetch         fetch(int32_t j) const
    {
        return Fetch{__ldg(z + j), FIRST ? 0.0 : __ldg(p_old + j)};
    }
    __device__ __forceinline__ double value(const Fetch& f) const
    {
        return FIRST ? zval(f.z) : aypx1(b, zval(f.z), f.p); // z + b*p  (kernels_scalar.cpp:33)
    }
    __device__ __forceinline__ int64_t own_col(int64_t i) const { return i; }
    // p_new[i] = z[i] + b p_old[i] from the row's own (gathered) operands
    __device__ __forceinline__ double row(int64_t i, double sum, double acc, const Fetch& o) const
    {
        const double p = value(o);
        p_new[i]       = p;
        w[i]           = sum;
        return add(acc, mul(p, sum));
    }
    // k_spmv_march: a cached (already formed) gathered value rides in a Fetch
    static __device__ __forceinline__ Fetch  from_formed(double p) { return Fetch{p, 0.0}; }
    static __device__ __forceinline__ Fetch  raw(double z, double p) { return Fetch{z, p}; }
    static __device__ __forceinline__ double formed(const Fetch& f) { return f.z; }
    // the same epilogue with p_new[i] already formed (k_spmv_march's cache)
    __device__ __forceinline__ double row_p(int64_t i, double sum, double acc, double p) const
    {
        p_new[i] = p;
        w[i]     = sum;
        return add(acc, mul(p, sum));
    }
    __device__ __forceinline__ void tail(double pAp) const
    {
        const double a = st->beta / pAp;
        st->pAp        = pAp;
        if (pAp == 0.0 || !isfinite(a)) {
            st->state          = RVK_CG_BREAKDOWN;
            st->breakdown_iter = it;
            st->done           = 1;
        } else {
            st->alpha   = a;
            st->betaold = st->beta;
        }
    }
};

// Constant-coefficient stencil geometry for the matrix-free operator
// (rvk_mf.cu): the same operator rvk_build_laplacian assembles, applied
// without storing it (PETSc MatShell analogue).
struct StencilGeom {
    int64_t nx, ny, nz, n;
    int     dim, box; // box: 9/27-point, else 5/7-point
    double  centre;   // points - 1; every neighbour is -1
};
// K1 on the stencil: p = z + b p_old on the fly, w = A p, p.w; same
// CgSpmvOp semantics (init/tail) as the CSR kernel.  Bit-identical w to the
// CSR path: the neighbours are visited in ascending column order with the
// same coefficients.
// The TMA 2.5D variant's plan state (tensor maps of z, p0, p1); null when the
// geometry does not allow it (odd nx) or the plan asks RVK_OPT_MF_SIMPLE.
struct MfTma;
MfTma*     mf_tma_create(const StencilGeom& g, const double* z, double* const* p, int np,
                         const double* r); // p: the plan's np (2..4) rotating p buffers
void       mf_tma_destroy(MfTma* t);
rvk_status launch_mf_k1(cudaStream_t s, const StencilGeom& g, bool first, const double* z,
                        const double* p_old, double* p_new, double* w, CgState* st, int64_t n,
                        int it, double* partials, unsigned int* ticket, int grid,
                        const MfTma* tma, bool zv = false, double zs = 1.0);
int        mf_grid(const StencilGeom& g);

// Arguments of the single-kernel persistent solve (rvk_cg_small.cu).
struct PersistArgs {
    int64_t        n;
    const int64_t* off;
    const int32_t* cols;
    const double*  vals;
    const double*  b;
    const double*  dinv;
    double*        x;
    double*        r;
    double*        z;
    double*        p0;
    double*        p1;
    double*        w;
    double*        hist;
    CgState*       st;
    double*        partials; // 4 doubles per block
    int            max_it;
    double         rtol, atol;
};
int        persistent_grid(int64_t n);
rvk_status launch_persistent(cudaStream_t s, const PersistArgs& args, bool jacobi, int grid);
// one-cluster DSMEM solve (rvk_cg_small.cu): cluster size or 0 (not eligible)
int        cluster_ctas(int64_t n, int64_t max_row_len);
rvk_status launch_cluster(cudaStream_t s, const PersistArgs& args, bool jacobi, int ctas, int max_row_len);
// one-launch grid solve for mid-size grids (rvk_cg_small.cu): rows per CTA or
// 0 (not eligible); bar = a plan-owned arrival counter (zeroed per launch)
// (*l2 = 1: the rows' ELL exceeds the shared memory -> k_cg_grid_l2 over
// a plan-owned k-major ELL copy built by build_grid_ell, passed as ell)
struct GridEll {
    double*  v = nullptr; // [nz][n] values
    int32_t* c = nullptr; // [nz][n] columns
    uint8_t* n = nullptr; // [n] row lengths
};
int        grid_solve_rows(int64_t n, int64_t max_row_len, int* ctas, int* l2);
rvk_status build_grid_ell(cudaStream_t s, int64_t n, const int64_t* off, const int32_t* cols,
                          const double* vals, int max_row_len, double* ev, int32_t* ec, uint8_t* en);
rvk_status launch_grid_solve(cudaStream_t s, const PersistArgs& args, unsigned* bar, bool jacobi,
                             int rpc, int ctas, int max_row_len, const GridEll* ell);

// Fused persistent solve (rvk_cg_fp.cu): K1 / K2 phases of every iteration in
// one cooperative launch that keeps the TMA SpMV ring across iterations.
struct FpArgs {
    int64_t       n;
    const double* b;
    const double* dinv;
    double        dconst; // the constant Jacobi diagonal when dvec == 0
    int           dvec;
    double*       x;
    double*       r;
    double*       z;
    double*       p0;
    double*       p1;
    double*       w;
    double*       hist;
    CgState*      st;
    double*       partials; // 4 doubles per block
    unsigned*     bar;      // arrival counter (zeroed per launch)
    int           max_it;
    double        rtol, atol;
};
struct SpmvArgs;
bool       fp_eligible(const SpmvArgs& a);
rvk_status launch_fp(cudaStream_t s, const SpmvArgs& a, const FpArgs& f);

// After the last iteration (or an early exit): apply the updates DEFER K2s
// left pending, in iteration order: x = ((x + a_0 p_0) + a_1 p_1) + ... .
// pb: the q rotating p buffers; iteration j wrote pb[(j + 1) % q].  With the
// whole-solve group (q = max_it) this is the solve's only x pass: it streams
// the max_it p's once (4 per trip, all loads issued before the adds).  No-op
// (one flag read per block) when nothing is pending.
struct XBufs {
    const double* p[kMaxXq];
};

// (A template so rvk_cg.cu and rvk_dcg.cu share one definition; the
// row-sharded plan passes its buffers' owned slices.)
template <int V = 0>
__global__ void __launch_bounds__(kUpdThreads)
    k_cg_xfix(int64_t n, double* __restrict__ x, XBufs pb, int q, const CgState* __restrict__ st,
              int xzero)
{
    // xzero: x was not initialised (the whole-solve group): start every
    // element from 0.0 -- the same adds as from a stored 0.0 -- and write x
    // even when no update is pending (a solve converged at the setup)
    const int cnt = st->x_pending;
    if (cnt <= 0 && !xzero) return;
    __shared__ const double* sp[kMaxXq];
    __shared__ double        sa[kMaxXq];
    if (threadIdx.x < cnt) {
        sp[threadIdx.x] = pb.p[(st->pend_it + threadIdx.x + 1) % q];
        sa[threadIdx.x] = st->pend_a[threadIdx.x];
    }
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0     = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uintptr_t     al     = reinterpret_cast<uintptr_t>(x);
    for (int k = 0; k < cnt; ++k) al |= reinterpret_cast<uintptr_t>(sp[k]);
    if (al & 15) { // a shard's owned slice may start mid-16-B: scalar sweep
        for (int64_t i = t0; i < n; i += stride) {
            double xi = xzero ? 0.0 : x[i];
            for (int k = 0; k < cnt; ++k) xi = axpy1(sa[k], sp[k][i], xi);
            x[i] = xi;
        }
        return;
    }
    const int64_t n2 = n >> 1;
    double2*      x2 = reinterpret_cast<double2*>(x);
    for (int64_t i = t0; i < n2; i += stride) {
        double2 xi = xzero ? make_double2(0.0, 0.0) : ld_stream(x2 + i);
        int     k  = 0;
        constexpr int B = V > 0 ? V : 4; // p streams in flight per thread
        for (; k + B <= cnt; k += B) {
            double2 v[B];
#pragma unroll
            for (int u = 0; u < B; ++u) v[u] = ld_stream(reinterpret_cast<const double2*>(sp[k + u]) + i);
#pragma unroll
            for (int u = 0; u < B; ++u) {
                xi.x = axpy1(sa[k + u], v[u].x, xi.x);
                xi.y = axpy1(sa[k + u], v[u].y, xi.y);
            }
        }
        for (; k < cnt; ++k) {
            const double2 v = ld_stream(reinterpret_cast<const double2*>(sp[k]) + i);
            xi.x            = axpy1(sa[k], v.x, xi.x);
            xi.y            = axpy1(sa[k], v.y, xi.y);
        }
        st_stream(x2 + i, xi);
    }
    if ((n & 1) && t0 == 0) {
        double xi = xzero ? 0.0 : x[n - 1];
        for (int k = 0; k < cnt; ++k) xi = axpy1(sa[k], sp[k][n - 1], xi);
        x[n - 1] = xi;
    }
}

} // namespace rvk
