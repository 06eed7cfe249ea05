// rvk_dcg.cu -- row-sharded Jacobi-CG across GPUs.
//
// The global grid is cut into contiguous slabs of planes (z for 3D, y for
// 2D); shard r owns rows [r_lo, r_hi) and stores z and p with one halo plane
// on each interior side: [lo halo | owned | hi halo].  Its local CSR (built
// on the device by rvk_build_laplacian_rows) indexes columns in that extended
// space, so the TMA SpMV mainloop runs unchanged.
//
// Per iteration (same arithmetic as rvk_cg.cu, element for element):
//   halo exchange of z (and p_old) with the two neighbours
//   K1: p = z + b p_old on the fly, w = A p, local p.w  -> gather slot [rank]
//   allgather of the partials; every rank folds the P partials in rank
//   order (bit-identical scalars on every rank, independent of the backend)
//   K2: alpha = beta/pAp, x += a p, r -= a w, z = B r, local z.z, z.r -> slot
//   allgather
// The scalar bookkeeping the single-GPU path does in its last-block tails
// moves to the *next* kernel's prologue (each block folds the gathered
// partials itself; block 0 publishes state/hist), because the reduction is
// only complete after the collective.  Every scalar stays on the device.
//
// Backends: NCCL (one process per GPU; ncclSend/Recv for halos, ncclAllGather
// for the partials, all stream-ordered on the solve stream, no host sync), or
// LOOPBACK (all P shards on one device in one process: halos are D2D copies
// and the partials land in one shared gather buffer) -- the loopback path
// exercises the partition, halo indexing and the distributed kernels on a
// single GPU.
#include "rvk_cg.cuh"
#include "rvk_common.cuh"
#include "rvk_context.hpp"
#include "rvk_internal.hpp"
#include "rvk_spmv.cuh"

#include <nccl.h>

#include <dlfcn.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

namespace rvk {

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (the library does not link libnccl; when torch
// is loaded its libnccl.so.2 is already mapped and dlopen returns it).
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
    bool ok = false;
};

NcclApi& nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            return fn != nullptr;
        };
        api.ok = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
                 sym(api.CommDestroy, "ncclCommDestroy") && sym(api.Send, "ncclSend") &&
                 sym(api.Recv, "ncclRecv") && sym(api.AllGather, "ncclAllGather") &&
                 sym(api.GroupStart, "ncclGroupStart") && sym(api.GroupEnd, "ncclGroupEnd") &&
                 sym(api.GetErrorString, "ncclGetErrorString");
    });
    return api;
}

rvk_status nccl_error(ncclResult_t r, const char* what)
{
    return set_error(RVK_ERR_COMM, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
}

#define RVK_NCCL(call)                                                    \
    do {                                                                  \
        ncclResult_t r_ = (call);                                         \
        if (r_ != ncclSuccess) return nccl_error(r_, #call);              \
    } while (0)

constexpr int kMaxRanks = 64;

// Fold the P gathered partials (stride 4 doubles per rank) in rank order.
__device__ __forceinline__ void fold_gather(const double* g, int nranks, int j0, int nv, double* out)
{
    for (int v = 0; v < nv; ++v) out[v] = 0.0;
    for (int r = 0; r < nranks; ++r)
        for (int v = 0; v < nv; ++v) out[v] += g[r * 4 + j0 + v];
}

} // namespace

// ---------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------
namespace {

// K0: r = b, x = 0, z = B b on the owned rows; partial z.z, z.r -> gather[rank][0..1]
template <bool JACOBI>
__global__ void __launch_bounds__(kUpdThreads)
    k_dcg_setup(int64_t n, const double* __restrict__ b, const double* __restrict__ dinv,
                double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                double* gather, int rank, double* partials, unsigned int* ticket)
{
    __shared__ double smem[64];
    __shared__ int    flag;
    double            acc[2] = {0.0, 0.0};
    const int64_t     stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double bi = b[i];
        const double zi = JACOBI ? mul(dinv[i], bi) : bi;
        r[i] = bi;
        z[i] = zi;
        x[i] = 0.0;
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
        gather[rank * 4 + 0] = acc[0];
        gather[rank * 4 + 1] = acc[1];
        *ticket              = 0u;
    }
}

// Shared prologue of K1(it): fold z.z / z.r of the previous step, publish
// dp -> hist[it], convergence; beta_it.  Identical decision in every block.
struct DcgScalars {
    CgState* st;
    double*  hist;
    double*  beta;   // beta[it] = z_it . r_it  (history avoids in-kernel RAW races)
    const double* gather;
    int      nranks;
    double   rtol, atol;
};

template <bool FIRST>
struct DcgSpmvOp {
    static constexpr bool kHasTail = true;
    const double* __restrict__ z;     // extended (halo) layout
    const double* __restrict__ p_old; // extended
    double* __restrict__ p_new;       // extended
    double* __restrict__ w;           // owned
    DcgScalars sc;
    int64_t    own_off;               // = halo_lo
    double*    gather_out;            // &gather[rank*4 + 2]
    int        it;
    double     b;

    __device__ __forceinline__ bool init()
    {
        CgState* st = sc.st;
        if (st->done) return false;
        double v[2];
        fold_gather(sc.gather, sc.nranks, 0, 2, v); // z.z, z.r of z_it
        const double dp    = sqrt(v[0]);
        const bool   lead  = blockIdx.x == 0 && threadIdx.x == 0;
        const double dp0   = FIRST ? dp : st->dp0;
        if (lead) {
            sc.hist[it] = dp;
            sc.beta[it] = v[1];
            if (FIRST) {
                st->dp0 = dp;
                st->breakdown_iter = -1;
                st->state = RVK_CG_RUNNING;
            }
            st->dp         = dp;
            st->iterations = it;
        }
        if (cg_converged(dp, dp0, sc.rtol, sc.atol)) {
            if (lead) {
                st->state = RVK_CG_CONVERGED;
                st->done  = 1;
            }
            return false;
        }
        if (!FIRST) {
            const double bo = sc.beta[it - 1];
            if (bo == 0.0) {
                if (lead) {
                    st->state          = RVK_CG_BREAKDOWN;
                    st->breakdown_iter = it;
                    st->done           = 1;
                }
                return false;
            }
            b = v[1] / bo;
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
    __device__ __forceinline__ Fetch fetch_smem(const double* s0, const double* s1, int i) const
    {
        return Fetch{s0[i], FIRST ? 0.0 : s1[i]};
    }
    __device__ __forceinline__ double value(const Fetch& f) const
    {
        return FIRST ? f.z : aypx1(b, f.z, f.p);
    }
    __device__ __forceinline__ int64_t own_col(int64_t i) const { return i + own_off; }
    __device__ __forceinline__ double row(int64_t i, double sum, double acc, const Fetch& o) const
    {
        const double p     = value(o);
        p_new[i + own_off] = p;
        w[i]               = sum;
        return add(acc, mul(p, sum));
    }
    __device__ __forceinline__ void tail(double pAp_local) const { *gather_out = pAp_local; }
};

// K2(it): fold p.w; alpha = beta_it / pAp; updates; partial z.z, z.r.
template <bool JACOBI>
__global__ void __launch_bounds__(kUpdThreads)
    k_dcg_update(int64_t n, const double* __restrict__ p, const double* __restrict__ w,
                 const double* __restrict__ dinv, double* __restrict__ x, double* __restrict__ r,
                 double* __restrict__ z, DcgScalars sc, int it, int rank, double* gather_out,
                 double* partials, unsigned int* ticket)
{
    CgState* st = sc.st;
    if (st->done) return;
    double pv[1];
    fold_gather(sc.gather, sc.nranks, 2, 1, pv);
    const double pAp = pv[0];
    const double a   = sc.beta[it] / pAp;
    if (pAp == 0.0 || !isfinite(a)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->state          = RVK_CG_BREAKDOWN;
            st->breakdown_iter = it;
            st->done           = 1;
        }
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->pAp   = pAp;
        st->alpha = a;
    }
    __shared__ double smem[64];
    __shared__ int    flag;
    const double      na     = -a;
    double            acc[2] = {0.0, 0.0};
    const int64_t     stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        x[i]            = axpy1(a, p[i], x[i]);
        const double ri = axpy1(na, w[i], r[i]);
        const double zi = JACOBI ? mul(dinv[i], ri) : ri;
        r[i]            = ri;
        z[i]            = zi;
        acc[0]          = add(acc[0], mul(zi, zi));
        acc[1]          = add(acc[1], mul(zi, ri));
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
        gather_out[0] = acc[0];
        gather_out[1] = acc[1];
        *ticket       = 0u;
    }
    (void)rank;
}

// After the last iteration: publish hist[max_it] (the K1 prologue that would
// normally do it does not run).
__global__ void k_dcg_finish(DcgScalars sc, int it)
{
    CgState* st = sc.st;
    if (st->done) return;
    double v[2];
    fold_gather(sc.gather, sc.nranks, 0, 2, v);
    const double dp = sqrt(v[0]);
    sc.hist[it]     = dp;
    sc.beta[it]     = v[1];
    st->dp          = dp;
    st->iterations  = it;
    if (cg_converged(dp, st->dp0, sc.rtol, sc.atol)) {
        st->state = RVK_CG_CONVERGED;
        st->done  = 1;
    }
}

__global__ void k_dcg_reset(CgState* st)
{
    st->done = 0;
    st->state = RVK_CG_RUNNING;
    st->iterations = 0;
    st->breakdown_iter = -1;
}

} // namespace
} // namespace rvk

using namespace rvk;

struct rvk_comm_s {
    ncclComm_t comm   = nullptr;
    int        nranks = 1, rank = 0;
};

struct rvk_dcg_plan_s {
    rvk_ctx       ctx = nullptr;
    rvk_comm      comm = nullptr; // null: loopback group member
    rvk_csr       A{};
    rvk_shard     sh{};
    rvk_cg_config cfg{};
    SpmvArgs      sa{};
    int           upd_grid = 0;
    int64_t       n_ext = 0;
    double *dinv = nullptr, *r = nullptr, *z = nullptr, *p[2] = {nullptr, nullptr}, *w = nullptr;
    double *hist = nullptr, *beta = nullptr, *gather = nullptr, *partials = nullptr;
    bool          owns_gather = true;
    CgState*      st = nullptr;
    unsigned int* tickets = nullptr;
};

namespace {

rvk_status alloc_plan_buffers(rvk_dcg_plan P)
{
    const int64_t n = P->sh.n_own;
    P->n_ext        = P->sh.halo_lo + n + P->sh.halo_hi;
    cudaError_t e   = cudaSuccess;
    auto        alloc = [&](void** p, size_t b) {
        if (e == cudaSuccess) e = cudaMalloc(p, b);
        if (e == cudaSuccess) e = cudaMemsetAsync(*p, 0, b, P->ctx->stream);
    };
    alloc((void**)&P->dinv, n * 8);
    alloc((void**)&P->r, n * 8);
    alloc((void**)&P->w, n * 8);
    alloc((void**)&P->z, P->n_ext * 8 + 32); // padded: x-windows round up
    alloc((void**)&P->p[0], P->n_ext * 8 + 32);
    alloc((void**)&P->p[1], P->n_ext * 8 + 32);
    alloc((void**)&P->hist, (P->cfg.max_it + 1) * 8);
    alloc((void**)&P->beta, (P->cfg.max_it + 1) * 8);
    alloc((void**)&P->st, sizeof(CgState));
    alloc((void**)&P->partials, 4 * kMaxReduceBlocks * 8);
    alloc((void**)&P->tickets, 16 * 4);
    if (P->owns_gather) alloc((void**)&P->gather, 4 * kMaxRanks * 8);
    if (e != cudaSuccess) return cuda_error(e, "rvk_dcg_plan_create: allocation");
    return RVK_OK;
}

DcgScalars scalars(rvk_dcg_plan P)
{
    return DcgScalars{P->st, P->hist, P->beta, P->gather, P->sh.nranks, P->cfg.rtol, P->cfg.atol};
}

int64_t plane(const rvk_dcg_plan P) { return P->sh.halo_lo ? P->sh.halo_lo : P->sh.halo_hi; }

// ---- per-phase enqueue (one shard) -----------------------------------------
rvk_status phase_setup(rvk_dcg_plan P, const double* b, double* x)
{
    cudaStream_t s = P->ctx->stream;
    k_dcg_reset<<<1, 1, 0, s>>>(P->st);
    const int g = P->upd_grid;
    double*   z_own = P->z + P->sh.halo_lo;
    if (P->cfg.pc == RVK_PC_JACOBI)
        k_dcg_setup<true><<<g, kUpdThreads, 0, s>>>(P->sh.n_own, b, P->dinv, x, P->r, z_own, P->gather,
                                                    P->sh.rank, P->partials, P->tickets);
    else
        k_dcg_setup<false><<<g, kUpdThreads, 0, s>>>(P->sh.n_own, b, P->dinv, x, P->r, z_own, P->gather,
                                                     P->sh.rank, P->partials, P->tickets);
    RVK_CHECK_LAUNCH("k_dcg_setup");
    return RVK_OK;
}

rvk_status phase_k1(rvk_dcg_plan P, int it)
{
    cudaStream_t   s  = P->ctx->stream;
    const double*  po = P->p[it & 1];
    double*        pn = P->p[(it + 1) & 1];
    const TailArgs ta{P->partials + 2 * kMaxReduceBlocks, P->tickets + 1};
    double*        go = P->gather + P->sh.rank * 4 + 2;
    if (it == 0) {
        DcgSpmvOp<true> op{P->z, po, pn, P->w, scalars(P), P->sh.halo_lo, go, it, 0.0};
        return launch_spmv(s, P->sa, op, ta, sm_count());
    }
    DcgSpmvOp<false> op{P->z, po, pn, P->w, scalars(P), P->sh.halo_lo, go, it, 0.0};
    return launch_spmv(s, P->sa, op, ta, sm_count());
}

rvk_status phase_k2(rvk_dcg_plan P, int it, double* x)
{
    cudaStream_t  s  = P->ctx->stream;
    const double* pn = P->p[(it + 1) & 1] + P->sh.halo_lo;
    double*       z  = P->z + P->sh.halo_lo;
    double*       go = P->gather + P->sh.rank * 4;
    if (P->cfg.pc == RVK_PC_JACOBI)
        k_dcg_update<true><<<P->upd_grid, kUpdThreads, 0, s>>>(P->sh.n_own, pn, P->w, P->dinv, x, P->r, z,
                                                               scalars(P), it, P->sh.rank, go,
                                                               P->partials, P->tickets);
    else
        k_dcg_update<false><<<P->upd_grid, kUpdThreads, 0, s>>>(P->sh.n_own, pn, P->w, P->dinv, x, P->r, z,
                                                                scalars(P), it, P->sh.rank, go,
                                                                P->partials, P->tickets);
    RVK_CHECK_LAUNCH("k_dcg_update");
    return RVK_OK;
}

rvk_status phase_finish(rvk_dcg_plan P)
{
    k_dcg_finish<<<1, 1, 0, P->ctx->stream>>>(scalars(P), P->cfg.max_it);
    RVK_CHECK_LAUNCH("k_dcg_finish");
    return RVK_OK;
}

// ---- NCCL collectives (one shard per process) --------------------------------
rvk_status nccl_allgather(rvk_dcg_plan P)
{
    double* mine = P->gather + P->sh.rank * 4;
    RVK_NCCL(nccl().AllGather(mine, P->gather, 4, ncclDouble, P->comm->comm, P->ctx->stream));
    return RVK_OK;
}

rvk_status nccl_halo(rvk_dcg_plan P, bool with_p, int it)
{
    const int64_t pl   = plane(P);
    const int     rank = P->sh.rank, np = P->sh.nranks;
    if (np == 1) return RVK_OK;
    double*     vecs[2] = {P->z, P->p[it & 1]};
    const int   nv      = with_p ? 2 : 1;
    auto&       api     = nccl();
    cudaStream_t s      = P->ctx->stream;
    RVK_NCCL(api.GroupStart());
    for (int v = 0; v < nv; ++v) {
        double* base = vecs[v];
        double* own  = base + P->sh.halo_lo;
        if (rank > 0) {
            RVK_NCCL(api.Send(own, pl, ncclDouble, rank - 1, P->comm->comm, s));
            RVK_NCCL(api.Recv(base, pl, ncclDouble, rank - 1, P->comm->comm, s));
        }
        if (rank < np - 1) {
            RVK_NCCL(api.Send(own + P->sh.n_own - pl, pl, ncclDouble, rank + 1, P->comm->comm, s));
            RVK_NCCL(api.Recv(own + P->sh.n_own, pl, ncclDouble, rank + 1, P->comm->comm, s));
        }
    }
    RVK_NCCL(api.GroupEnd());
    return RVK_OK;
}

// ---- loopback (all shards on one device) -------------------------------------
rvk_status loop_halo(rvk_dcg_plan* Ps, int np, bool with_p, int it)
{
    for (int r = 0; r < np; ++r) {
        rvk_dcg_plan P  = Ps[r];
        cudaStream_t s  = P->ctx->stream;
        const int64_t pl = plane(P);
        for (int v = 0; v < (with_p ? 2 : 1); ++v) {
            auto vec = [&](rvk_dcg_plan Q) { return v == 0 ? Q->z : Q->p[it & 1]; };
            if (r > 0) { // my lo halo <- last owned plane of r-1
                rvk_dcg_plan L = Ps[r - 1];
                RVK_CUDA(cudaMemcpyAsync(vec(P), vec(L) + L->sh.halo_lo + L->sh.n_own - pl, pl * 8,
                                         cudaMemcpyDeviceToDevice, s));
            }
            if (r < np - 1) { // my hi halo <- first owned plane of r+1
                rvk_dcg_plan U = Ps[r + 1];
                RVK_CUDA(cudaMemcpyAsync(vec(P) + P->sh.halo_lo + P->sh.n_own, vec(U) + U->sh.halo_lo,
                                         pl * 8, cudaMemcpyDeviceToDevice, s));
            }
        }
    }
    return RVK_OK;
}

#define RVK_TRY(x)                                                                             \
    do {                                                                                       \
        rvk_status rc_ = (x);                                                                  \
        if (rc_ != RVK_OK) return rc_;                                                         \
    } while (0)

} // namespace

extern "C" {

rvk_status rvk_comm_unique_id(void* id_out, int id_bytes)
{
    if (!id_out || id_bytes < (int)sizeof(ncclUniqueId))
        return set_error(RVK_ERR_INVALID, "comm_unique_id: need %d bytes", (int)sizeof(ncclUniqueId));
    if (!nccl().ok) return set_error(RVK_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    RVK_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof id);
    return RVK_OK;
}

rvk_status rvk_comm_init(const void* id, int nranks, int rank, rvk_comm* out)
{
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks || nranks > kMaxRanks)
        return set_error(RVK_ERR_INVALID, "comm_init: bad arguments");
    if (!nccl().ok) return set_error(RVK_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
    auto c    = new rvk_comm_s();
    c->nranks = nranks;
    c->rank   = rank;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_error(r, "ncclCommInitRank");
    }
    *out = c;
    return RVK_OK;
}

rvk_status rvk_comm_destroy(rvk_comm c)
{
    if (!c) return RVK_OK;
    if (c->comm) nccl().CommDestroy(c->comm);
    delete c;
    return RVK_OK;
}

rvk_status rvk_dcg_plan_create(rvk_ctx ctx, const rvk_csr* A, rvk_shard sh, rvk_cg_config cfg,
                               rvk_comm comm, double* shared_gather, rvk_dcg_plan* out)
{
    if (!ctx || !A || !out) return set_error(RVK_ERR_INVALID, "dcg_plan_create: null argument");
    *out = nullptr;
    if (sh.nranks < 1 || sh.nranks > kMaxRanks || sh.rank < 0 || sh.rank >= sh.nranks)
        return set_error(RVK_ERR_INVALID, "dcg_plan_create: bad shard rank/nranks");
    if (A->n_rows != sh.n_own || A->n_cols != sh.halo_lo + sh.n_own + sh.halo_hi)
        return set_error(RVK_ERR_DIM, "dcg_plan_create: local CSR does not match the shard");
    if ((sh.rank > 0) != (sh.halo_lo > 0) || (sh.rank < sh.nranks - 1) != (sh.halo_hi > 0))
        return set_error(RVK_ERR_INVALID, "dcg_plan_create: halos must exist exactly at interior cuts");
    if (sh.halo_lo && sh.halo_hi && sh.halo_lo != sh.halo_hi)
        return set_error(RVK_ERR_INVALID, "dcg_plan_create: halo planes must have equal size");
    if ((sh.halo_lo > sh.n_own) || (sh.halo_hi > sh.n_own))
        return set_error(RVK_ERR_INVALID, "dcg_plan_create: shard thinner than a halo plane");
    if (cfg.max_it < 1) return set_error(RVK_ERR_INVALID, "max_it must be >= 1");
    if (!comm && !shared_gather && sh.nranks > 1)
        return set_error(RVK_ERR_INVALID, "dcg_plan_create: loopback shards need a shared gather buffer");
    int64_t maxlen = 0;
    RVK_TRY(rvk_csr_validate(ctx, A, &maxlen));
    auto P         = new rvk_dcg_plan_s();
    P->ctx         = ctx;
    P->comm        = comm;
    P->A           = *A;
    P->sh          = sh;
    P->cfg         = cfg;
    SpmvWindows win; // x-windows opt-in, leading-edge prefetch default (see rvk_cg.cu)
    if (csr_windows(ctx->stream, *A, &win) != RVK_OK) win = SpmvWindows{};
    if (!std::getenv("RVK_WINDOWS")) win.n = 0;
    if (std::getenv("RVK_NO_PREFETCH")) win.has_lead = false;
    P->sa          = make_spmv_args(*A, maxlen, &win, 2);
    P->upd_grid    = resident_grid(k_dcg_update<true>, kUpdThreads, sh.n_own);
    P->owns_gather = shared_gather == nullptr;
    P->gather      = shared_gather;
    rvk_status rc  = alloc_plan_buffers(P);
    // dinv of the owned rows: the local CSR's diagonal sits at column row + halo_lo
    if (rc == RVK_OK) {
        if (cfg.pc == RVK_PC_JACOBI) rc = diag_inverse(ctx->stream, *A, sh.halo_lo, P->dinv);
        else rc = rvk_set(ctx, sh.n_own, 1.0, P->dinv);
    }
    if (rc != RVK_OK) {
        rvk_dcg_plan_destroy(P);
        return rc;
    }
    *out = P;
    return RVK_OK;
}

rvk_status rvk_dcg_plan_destroy(rvk_dcg_plan P)
{
    if (!P) return RVK_OK;
    if (P->ctx) cudaStreamSynchronize(P->ctx->stream);
    void* bufs[] = {P->dinv, P->r, P->w, P->z, P->p[0], P->p[1], P->hist, P->beta, P->st, P->partials,
                    P->tickets};
    for (void* b : bufs)
        if (b) cudaFree(b);
    if (P->owns_gather && P->gather) cudaFree(P->gather);
    delete P;
    return RVK_OK;
}

// One shard per process (NCCL): the whole solve, stream-ordered, no host sync.
rvk_status rvk_dcg_solve_dev(rvk_dcg_plan P, const double* b_own, double* x_own)
{
    if (!P || !b_own || !x_own) return set_error(RVK_ERR_INVALID, "null argument");
    if (!P->comm && P->sh.nranks > 1)
        return set_error(RVK_ERR_INVALID, "loopback shards are solved with rvk_dcg_loopback_solve");
    const bool dist = P->comm && P->sh.nranks > 1;
    RVK_TRY(phase_setup(P, b_own, x_own));
    if (dist) RVK_TRY(nccl_allgather(P));
    for (int it = 0; it < P->cfg.max_it; ++it) {
        if (dist) RVK_TRY(nccl_halo(P, it > 0, it));
        RVK_TRY(phase_k1(P, it));
        if (dist) RVK_TRY(nccl_allgather(P));
        RVK_TRY(phase_k2(P, it, x_own));
        if (dist) RVK_TRY(nccl_allgather(P));
    }
    return phase_finish(P);
}

// All P shards on one device, enqueued phase by phase on shard 0's stream
// order (each plan's own stream; cross-shard edges via events).
rvk_status rvk_dcg_loopback_solve(rvk_dcg_plan* Ps, int np, const double* const* b, double* const* x)
{
    if (!Ps || np < 1 || !b || !x) return set_error(RVK_ERR_INVALID, "null argument");
    for (int r = 0; r < np; ++r)
        if (Ps[r]->ctx->stream != Ps[0]->ctx->stream)
            return set_error(RVK_ERR_INVALID, "loopback shards must share one context/stream");
    for (int r = 0; r < np; ++r) RVK_TRY(phase_setup(Ps[r], b[r], x[r]));
    for (int it = 0; it < Ps[0]->cfg.max_it; ++it) {
        RVK_TRY(loop_halo(Ps, np, it > 0, it));
        for (int r = 0; r < np; ++r) RVK_TRY(phase_k1(Ps[r], it));
        for (int r = 0; r < np; ++r) RVK_TRY(phase_k2(Ps[r], it, x[r]));
    }
    for (int r = 0; r < np; ++r) RVK_TRY(phase_finish(Ps[r]));
    return RVK_OK;
}

rvk_status rvk_dcg_result(rvk_dcg_plan P, double* hist_host, rvk_cg_info* info)
{
    if (!P) return set_error(RVK_ERR_INVALID, "null plan");
    CgState      h{};
    cudaStream_t s = P->ctx->stream;
    RVK_CUDA(cudaMemcpyAsync(&h, P->st, sizeof h, cudaMemcpyDeviceToHost, s));
    if (hist_host)
        RVK_CUDA(cudaMemcpyAsync(hist_host, P->hist, (P->cfg.max_it + 1) * 8, cudaMemcpyDeviceToHost, s));
    note_host_sync();
    RVK_CUDA(cudaStreamSynchronize(s));
    if (info) {
        info->state          = h.state;
        info->iterations     = h.iterations;
        info->breakdown_iter = h.breakdown_iter;
    }
    if (h.state == RVK_CG_BREAKDOWN)
        return set_error(RVK_ERR_BREAKDOWN, "cg_solve: breakdown at iteration %d", h.breakdown_iter);
    return RVK_OK;
}

} // extern "C"
