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
// Backends:
//  * PEER (the product on an NVSwitch box): every shard exports ONE device
//    window [z | p0 | p1 | flags | gather] (cudaIpc handle, mapped by every
//    other rank).  The kernels do the communication themselves, tile by tile:
//    K2/setup store the boundary planes of z straight into the neighbours'
//    halo planes while they compute them, K1 does the same for p, and each
//    kernel's last block stores its dot partials into every rank's gather
//    slot and then releases a per-source arrival flag (st.release.sys) on
//    every rank.  The next kernel's prologue waits (ld.acquire.sys) until all
//    P flags reached its phase.  No NCCL call and no separate halo/allreduce
//    step remains on the data path; the NVLink transfer overlaps the math.
//  * NCCL (one process per GPU; ncclSend/Recv for halos, ncclAllGather for
//    the partials, all stream-ordered on the solve stream, no host sync) --
//    the library-collective baseline.
//  * LOOPBACK (all P shards on one device in one process: halos are D2D
//    copies and the partials land in one shared gather buffer), and PEER
//    LOOPBACK (the PEER kernels with every "remote" window on the same
//    device) -- exercise the partition, halo indexing, the in-kernel pushes
//    and the flag protocol on a single GPU.
//
// PEER flag protocol.  Flags are 64-bit (solve_seq << 32 | phase), one per
// source rank, stored monotonically by that source only.  Phases of solve s:
// setup = 1, K1(it) = 2 + 2 it, K2(it) = 3 + 2 it, finish = 0xffffffff.
//   K1(it) waits for phase 2 it + 1 (z halos + z.z/z.r partials of z_it);
//   K2(it) waits for 2 it + 2 (p.w partials); finish waits for 2 max_it + 1;
//   setup(s) waits for every rank's finish(s - 1), so no rank overwrites a
//   slot or halo a slower peer still reads.
// Write-after-read safety of the halos / slots follows from the waits: a
// rank's K2(it) (which overwrites the neighbours' z halos and z.z slots)
// starts only after every rank's K1(it) completed reading them; K1(it)
// writes p_new = p[(it+1) % ring], whose halo was last read by K1(it-1) or
// earlier, which
// precedes every rank's K2(it-1) that K1(it) waited for.  Every block fences
// at system scope before its grid ticket, so the last block's release of the
// flag covers all blocks' remote stores.  Waits are bounded (kPeerTimeoutNs):
// a missing peer turns into RVK_CG_COMM_ERROR on every rank, never a hang.
#include "rvk_cg.cuh"
#include "rvk_common.cuh"
#include "rvk_context.hpp"
#include "rvk_spmv_march.cuh"
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
    // optional (diagnostics): the communicator's own view and its async error
    ncclResult_t (*CommCount)(const ncclComm_t, int*)           = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*)        = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
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
        sym(api.CommCount, "ncclCommCount");
        sym(api.CommUserRank, "ncclCommUserRank");
        sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
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
        for (int v = 0; v < nv; ++v) out[v] += __ldcg(g + r * 4 + j0 + v); // L2: coherent with peer stores
}

// ---- PEER backend: system-scope flag protocol ------------------------------
constexpr uint32_t kPhaseFinish   = 0xffffffffu;
constexpr uint64_t kPeerTimeoutNs = 30ull * 1000 * 1000 * 1000; // 30 s

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p)
{
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t phase_tag(uint32_t seq, uint32_t phase)
{
    return ((uint64_t)seq << 32) | phase;
}

// Everything a PEER-mode kernel needs to reach the other ranks.  Pointers are
// valid on this device (own window, or peers' windows mapped by cudaIpc).
struct DcgPeer {
    int             on;                  // 0: NCCL / loopback phases, no in-kernel comm
    int             rank, nranks;
    double* const*  gather;              // [nranks] every rank's gather slots
    uint64_t* const* flags;              // [nranks] every rank's arrival flags
    const uint64_t* my_flags;            // this rank's flags (peers store into it)
    double*         lo_z;                // where my first owned plane lands in rank-1 (or null)
    double*         lo_p[kMaxXq];        // per p ring buffer
    double*         hi_z;                // where my last owned plane lands in rank+1 (or null)
    double*         hi_p[kMaxXq];
    int64_t         plane, n_own;
};

// Block-wide wait until every rank's flag reached `tag`.  Returns false (and
// marks the solve failed) on timeout, or when another block of this rank
// already timed out.  Call from ALL threads of the block.
__device__ __forceinline__ bool peer_wait(const DcgPeer& pr, CgState* st, uint64_t tag)
{
    __shared__ int ok;
    if (threadIdx.x == 0) {
        int            good = 1;
        const uint64_t t0   = globaltimer_ns();
        for (int q = 0; q < pr.nranks && good; ++q) {
            while (ld_acquire_sys(pr.my_flags + q) < tag) {
                __nanosleep(128);
                if (globaltimer_ns() - t0 > kPeerTimeoutNs || *(volatile int*)&st->comm_error) {
                    good = 0;
                    break;
                }
            }
        }
        if (!good && atomicCAS(&st->comm_error, 0, 1) == 0) {
            st->state = RVK_CG_COMM_ERROR;
            st->done  = 1;
        }
        ok = good;
    }
    __syncthreads();
    return ok != 0;
}

// Single thread: store v[0..nv) into slot [rank*4 + j0] of every rank, then
// release phase `tag` on every rank.  The caller has fenced its block's
// remote stores (last_block<true>), so the release covers the whole grid.
__device__ __forceinline__ void peer_publish(const DcgPeer& pr, int j0, const double* v, int nv,
                                             uint64_t tag)
{
    for (int q = 0; q < pr.nranks; ++q)
        for (int k = 0; k < nv; ++k) pr.gather[q][pr.rank * 4 + j0 + k] = v[k];
    __threadfence_system();
    for (int q = 0; q < pr.nranks; ++q) st_release_sys(pr.flags[q] + pr.rank, tag);
}

// Boundary-plane push of one owned element (row i of the shard).
__device__ __forceinline__ void peer_push(double* lo, double* hi, int64_t plane, int64_t n_own,
                                          int64_t i, double v)
{
    if (lo && i < plane) lo[i] = v;
    const int64_t j = i - (n_own - plane);
    if (hi && j >= 0) hi[j] = v;
}

} // namespace

// ---------------------------------------------------------------------------
// Kernels.  PEER = true: in-kernel halo pushes, partial broadcast and flag
// waits (see the protocol at the top); false: NCCL / loopback phases do the
// exchange between kernels.
// ---------------------------------------------------------------------------
namespace {

// PC: 0 none, 1 dinv vector, 2 constant dinv (constant-coefficient diagonal,
// folded to the scalar dconst at plan time -- bit-identical, no dinv stream)
__device__ __forceinline__ double jacobi_z(int PC, const double* __restrict__ dinv, double dconst,
                                           int64_t i, double ri)
{
    return PC == 0 ? ri : mul(PC == 1 ? dinv[i] : dconst, ri);
}

// K0: r = b, x = 0, z = B b on the owned rows; partial z.z, z.r -> gather[rank][0..1]
template <int PC, bool PEER>
__global__ void __launch_bounds__(kUpdThreads)
    k_dcg_setup(int64_t n, const double* __restrict__ b, const double* __restrict__ dinv,
                double dconst, double* __restrict__ x, double* __restrict__ r,
                double* __restrict__ z, double* gather, int rank, double* partials,
                unsigned int* ticket, CgState* st, DcgPeer pr, int xw)
{
    __shared__ double smem[64];
    __shared__ int    flag;
    uint32_t          seq = 0;
    if constexpr (PEER) {
        // every rank finished the previous solve (its slots / halos are free)
        seq = st->seq;
        if (seq > 1 && !peer_wait(pr, st, phase_tag(seq - 1, kPhaseFinish))) return;
    }
    double        acc[2] = {0.0, 0.0};
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double bi = b[i];
        const double zi = jacobi_z(PC, dinv, dconst, i, bi);
        r[i] = bi;
        z[i] = zi;
        if (xw) x[i] = 0.0; // xw = 0: the whole-solve x pass starts from 0.0 itself
        if constexpr (PEER) peer_push(pr.lo_z, pr.hi_z, pr.plane, n, i, zi);
        acc[0] = add(acc[0], mul(zi, zi));
        acc[1] = add(acc[1], mul(zi, bi));
    }
    const int tid = threadIdx.x;
    block_sum<2>(acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        partials[2 * blockIdx.x]     = acc[0];
        partials[2 * blockIdx.x + 1] = acc[1];
    }
    if (!last_block<PEER>(ticket, tid, &flag, blockDim.x, 1)) return;
    fold_partials<2>(partials, gridDim.x, acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        *ticket = 0u;
        if constexpr (PEER) peer_publish(pr, 0, acc, 2, phase_tag(seq, 1));
        else {
            gather[rank * 4 + 0] = acc[0];
            gather[rank * 4 + 1] = acc[1];
        }
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

template <bool FIRST, bool PEER>
struct DcgSpmvOp {
    static constexpr bool kHasTail  = true;
    static constexpr bool kSysFence = PEER;
    static constexpr bool kNoSmall  = true; // shard plans never take the small-system K1
    const double* __restrict__ z;     // extended (halo) layout
    const double* __restrict__ p_old; // extended
    double* __restrict__ p_new;       // extended
    double* __restrict__ w;           // owned
    DcgScalars sc;
    int64_t    own_off;               // = halo_lo
    double*    gather_out;            // &gather[rank*4 + 2]
    int        it;
    double     b;
    DcgPeer    pr;                    // PEER: neighbours' p_new halo planes etc.
    double*    lo_pn;                 // PEER: pr.lo_p / hi_p of this iteration's p_new
    double*    hi_pn;
    uint32_t   seq;
    // the owned rows' slices (pre-offset by own_off): the row epilogue and its
    // operands index them directly, like the single-GPU op
    const double* __restrict__ z_own;
    const double* __restrict__ pold_own;
    double* __restrict__       pnew_own;

    __device__ __forceinline__ bool init()
    {
        CgState* st = sc.st;
        if (st->done) return false;
        if constexpr (PEER) {
            seq = st->seq;
            if (!peer_wait(pr, st, phase_tag(seq, 2 * it + 1))) return false;
        }
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
    __device__ __forceinline__ double value(const Fetch& f) const
    {
        return FIRST ? f.z : aypx1(b, f.z, f.p);
    }
    __device__ __forceinline__ int64_t own_col(int64_t i) const { return i + own_off; }
    using Own = Fetch;
    __device__ __forceinline__ Own own(int64_t i) const
    {
        return Fetch{__ldg(z_own + i), FIRST ? 0.0 : __ldg(pold_own + i)};
    }
    __device__ __forceinline__ double row(int64_t i, double sum, double acc, const Fetch& o) const
    {
        return row_p(i, sum, acc, value(o));
    }
    // k_spmv_march: cached (formed) gathered values ride in a Fetch
    static __device__ __forceinline__ Fetch  from_formed(double p) { return Fetch{p, 0.0}; }
    static __device__ __forceinline__ Fetch  raw(double z, double p) { return Fetch{z, p}; }
    static __device__ __forceinline__ double formed(const Fetch& f) { return f.z; }
    __device__ __forceinline__ double row_p(int64_t i, double sum, double acc, double p) const
    {
        pnew_own[i] = p;
        if constexpr (PEER) peer_push(lo_pn, hi_pn, pr.plane, pr.n_own, i, p);
        w[i] = sum;
        return add(acc, mul(p, sum));
    }
    __device__ __forceinline__ void tail(double pAp_local) const
    {
        if constexpr (PEER) peer_publish(pr, 2, &pAp_local, 1, phase_tag(seq, 2 * it + 2));
        else *gather_out = pAp_local;
    }
};

// K2(it): fold p.w; alpha = beta_it / pAp; updates; partial z.z, z.r.
// XM: x-update mode as the single-GPU k_cg_update (0 x += a p; 1 defer into
// pend_a[slot] -- the next iteration's pair flush, or with the whole-solve
// ring the final k_cg_xfix; 2 x = (x + a' p_prev) + a p) -- bit-identical x.
template <int PC, bool PEER, int XM = 0, bool VEC = false>
// (3 blocks per SM: the register cap keeps the update's resident wave as
// wide as the single-GPU k_cg_update's)
__global__ void __launch_bounds__(kUpdThreads, 3)
    k_dcg_update(int64_t n, const double* __restrict__ p, const double* __restrict__ w,
                 const double* __restrict__ dinv, double dconst, double* __restrict__ x,
                 double* __restrict__ r,
                 double* __restrict__ z, DcgScalars sc, int it, int rank, double* gather_out,
                 double* partials, unsigned int* ticket, DcgPeer pr,
                 const double* __restrict__ p_prev, int slot, int last)
{
    CgState* st = sc.st;
    if (st->done) return;
    uint32_t seq = 0;
    if constexpr (PEER) {
        seq = st->seq;
        if (!peer_wait(pr, st, phase_tag(seq, 2 * it + 2))) return;
    }
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
    // pend_a[slot] is only written by a DEFER (XM 1) launch, read by a later
    // XM 2 / k_cg_xfix: no race
    const double ap = XM == 2 ? st->pend_a[0] : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->pAp   = pAp;
        st->alpha = a;
        if (XM == 1) {
            st->pend_a[slot] = a;
            st->x_pending    = slot + 1;
            if (slot == 0) st->pend_it = it;
        } else if (XM == 2) {
            st->x_pending = 0;
        }
    }
    __shared__ double smem[64];
    __shared__ int    flag;
    const double      na     = -a;
    double            acc[2] = {0.0, 0.0};
    const int64_t     stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t     t0     = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if constexpr (VEC) {
        // as k_cg_update: 2 x double2 per thread per trip, all loads first
        const int64_t  n2 = n >> 1;
        const double2* p2 = reinterpret_cast<const double2*>(p);
        const double2* q2 = reinterpret_cast<const double2*>(p_prev);
        const double2* w2 = reinterpret_cast<const double2*>(w);
        const double2* d2 = reinterpret_cast<const double2*>(dinv);
        double2*       x2 = reinterpret_cast<double2*>(x);
        double2*       r2 = reinterpret_cast<double2*>(r);
        double2*       z2 = reinterpret_cast<double2*>(z);
        const double2  zero = make_double2(0.0, 0.0);
        auto ld = [&](bool use, const double2* a2, int64_t i) { return use ? ld_stream(a2 + i) : zero; };
        auto step = [&](const double2& pi, const double2& qi, const double2& wi, double2 xi,
                        double2 ri, const double2& d, int64_t i) {
            if (XM == 2) {
                xi.x = axpy1(ap, qi.x, xi.x);
                xi.y = axpy1(ap, qi.y, xi.y);
            }
            if (XM != 1) {
                xi.x = axpy1(a, pi.x, xi.x);
                xi.y = axpy1(a, pi.y, xi.y);
                st_stream(x2 + i, xi);
            }
            ri.x = axpy1(na, wi.x, ri.x);
            ri.y = axpy1(na, wi.y, ri.y);
            double2 zi = ri;
            if (PC != 0) {
                zi.x = mul(d.x, ri.x);
                zi.y = mul(d.y, ri.y);
            }
            if (!last) { // the last K2's r, z (and z halos) are dead: the next setup rewrites them
                r2[i] = ri;
                z2[i] = zi;
                if constexpr (PEER) {
                    peer_push(pr.lo_z, pr.hi_z, pr.plane, n, 2 * i, zi.x);
                    peer_push(pr.lo_z, pr.hi_z, pr.plane, n, 2 * i + 1, zi.y);
                }
            }
            acc[0] = add(acc[0], mul(zi.x, zi.x));
            acc[0] = add(acc[0], mul(zi.y, zi.y));
            acc[1] = add(acc[1], mul(zi.x, ri.x));
            acc[1] = add(acc[1], mul(zi.y, ri.y));
        };
        int64_t i = t0;
        for (; i + stride < n2; i += 2 * stride) {
            const int64_t j  = i + stride;
            const double2 pa = ld(XM != 1, p2, i), pb = ld(XM != 1, p2, j);
            const double2 qa = ld(XM == 2, q2, i), qb = ld(XM == 2, q2, j);
            const double2 wa = ld_stream(w2 + i), wb = ld_stream(w2 + j);
            const double2 xa = ld(XM != 1, x2, i), xb = ld(XM != 1, x2, j);
            const double2 ra = ld_stream(r2 + i), rb = ld_stream(r2 + j);
            double2 da = make_double2(dconst, dconst), db = da;
            if (PC == 1) {
                da = ld_stream(d2 + i);
                db = ld_stream(d2 + j);
            }
            step(pa, qa, wa, xa, ra, da, i);
            step(pb, qb, wb, xb, rb, db, j);
        }
        if (i < n2) {
            double2 d = make_double2(dconst, dconst);
            if (PC == 1) d = ld_stream(d2 + i);
            step(ld(XM != 1, p2, i), ld(XM == 2, q2, i), ld_stream(w2 + i), ld(XM != 1, x2, i),
                 ld_stream(r2 + i), d, i);
        }
    }
    for (int64_t i = (VEC ? (n & ~int64_t(1)) : 0) + t0; i < n; i += stride) {
        if (XM == 2) x[i] = axpy1(ap, p_prev[i], x[i]);
        if (XM != 1) x[i] = axpy1(a, p[i], x[i]);
        const double ri = axpy1(na, w[i], r[i]);
        const double zi = jacobi_z(PC, dinv, dconst, i, ri);
        if (!last) {
            r[i] = ri;
            z[i] = zi;
            if constexpr (PEER) peer_push(pr.lo_z, pr.hi_z, pr.plane, n, i, zi);
        }
        acc[0]          = add(acc[0], mul(zi, zi));
        acc[1]          = add(acc[1], mul(zi, ri));
    }
    const int tid = threadIdx.x;
    block_sum<2>(acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        partials[2 * blockIdx.x]     = acc[0];
        partials[2 * blockIdx.x + 1] = acc[1];
    }
    if (!last_block<PEER>(ticket, tid, &flag, blockDim.x, 1)) return;
    fold_partials<2>(partials, gridDim.x, acc, smem, tid, blockDim.x, 1);
    if (tid == 0) {
        *ticket = 0u;
        if constexpr (PEER) peer_publish(pr, 0, acc, 2, phase_tag(seq, 2 * it + 3));
        else {
            gather_out[0] = acc[0];
            gather_out[1] = acc[1];
        }
    }
    (void)rank;
}

// After the last iteration: publish hist[max_it] (the K1 prologue that would
// normally do it does not run).  PEER: then release "finished" to every rank.
template <bool PEER>
__global__ void k_dcg_finish(DcgScalars sc, int it, DcgPeer pr)
{
    CgState*       st  = sc.st;
    const uint32_t seq = st->seq;
    bool           run = !st->done; // uniform over the block
    if constexpr (PEER)
        if (run) run = peer_wait(pr, st, phase_tag(seq, 2 * it + 1));
    if (threadIdx.x != 0) return;
    if (run) {
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
    if constexpr (PEER) {
        __threadfence_system();
        for (int q = 0; q < pr.nranks; ++q)
            st_release_sys(pr.flags[q] + pr.rank, phase_tag(seq, kPhaseFinish));
    }
}

__global__ void k_dcg_reset(CgState* st)
{
    st->x_pending = 0;
    st->done = 0;
    st->state = RVK_CG_RUNNING;
    st->iterations = 0;
    st->breakdown_iter = -1;
    st->comm_error = 0;
    st->seq += 1;
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
    rvk_comm      comm = nullptr; // null: loopback group member (or PEER backend)
    rvk_csr       A{};
    rvk_shard     sh{};
    rvk_cg_config cfg{};
    SpmvArgs      sa{};
    bool          march = false; // K1 (it >= 1) is k_spmv_march (RVK_PLAN_MARCH)
    SpmvArgs      sa_m{};
    SpmvMarch     mg{};
    int           upd_grid = 0, xfix_grid = 0;
    int64_t       n_ext = 0;
    unsigned char* win = nullptr;  // [z | p0 | p1 | flags | gather], the exported PEER window
    size_t        win_bytes = 0;
    double *dinv = nullptr, *r = nullptr, *z = nullptr, *w = nullptr;
    // whole-solve CUDA graph (cfg.use_graph), captured per (b, x) pair
    cudaGraphExec_t graph   = nullptr;
    const double*   graph_b = nullptr;
    double*         graph_x = nullptr;
    double*       p[kMaxXq] = {}; // p ring in the window: iteration j writes p[(j+1) % npb]
    int           npb = 2;        // 2 (x per iteration pair) or max_it (x once per solve)
    double *hist = nullptr, *beta = nullptr, *gather = nullptr, *partials = nullptr;
    bool          owns_gather = true;
    CgState*      st = nullptr;
    unsigned int* tickets = nullptr;
    DcgPeer       peer{};          // peer.on: PEER backend attached
    bool          const_diag = false; // Jacobi diagonal is one value: dconst
    double        dconst     = 0.0;
    void**        peer_tab = nullptr; // device: gather[nranks] then flags[nranks]
};

namespace {

// Byte layout of a shard's window (identical rule on every rank, so a rank
// can address a peer's halo planes from the peer's shard geometry alone).
struct WindowLayout {
    size_t flags, gather, z, p0, vb, bytes;
    int    npb;
    size_t p(int k) const { return p0 + (size_t)k * vb; }
};
// p ring length of a shard plan: max_it (x written once per solve, every
// iteration's p kept) when 5 <= max_it <= kMaxXq and the ring takes at most
// half the device, else 2 (x per iteration pair).  A pure function of
// (max_it, n_ext, device size), so every rank can derive a peer's layout;
// attach_peers checks that the neighbours' rings match.
int ring_len(int max_it, int64_t n_ext)
{
    if (max_it < 5 || max_it > kMaxXq) return 2;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 2;
    const size_t need = (size_t)(max_it + 1) * ((size_t)n_ext * 8 + (size_t(3) << 20));
    return need <= tot / 2 ? max_it : 2;
}
WindowLayout window_layout(int64_t n_ext, int npb)
{
    // the gathered vectors start 2 MB-aligned plus 1 MB, so z[j] and p[j]
    // are not a whole number of 2 MB apart (measured: single-shard solve
    // 9.64 -> 9.45 ms); flags and gather slots after them
    auto         up  = [](size_t v) { return (v + 255) & ~size_t(255); };
    auto         up2 = [](size_t v) { return (v + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1); };
    WindowLayout L{};
    const size_t vb = up2((size_t)n_ext * 8 + 32) + (size_t(1) << 20); // + 4 doubles: x-windows round up
    L.vb            = vb;
    L.npb           = npb;
    L.z             = 0;
    L.p0            = vb;
    L.flags         = L.p(npb);
    L.gather        = up(L.flags + kMaxRanks * sizeof(uint64_t));
    L.bytes         = up(L.gather + kMaxRanks * 4 * sizeof(double));
    return L;
}

rvk_status alloc_plan_buffers(rvk_dcg_plan P)
{
    const int64_t n = P->sh.n_own;
    P->n_ext        = P->sh.halo_lo + n + P->sh.halo_hi;
    cudaError_t e   = cudaSuccess;
    auto        alloc = [&](void** p, size_t b) {
        if (e == cudaSuccess) e = cudaMalloc(p, b);
        if (e == cudaSuccess) e = cudaMemsetAsync(*p, 0, b, P->ctx->stream);
    };
    P->npb               = ring_len(P->cfg.max_it, P->n_ext);
    const WindowLayout L = window_layout(P->n_ext, P->npb);
    alloc((void**)&P->win, L.bytes);
    if (e == cudaSuccess) {
        P->win_bytes = L.bytes;
        P->z         = reinterpret_cast<double*>(P->win + L.z);
        for (int k = 0; k < P->npb; ++k) P->p[k] = reinterpret_cast<double*>(P->win + L.p(k));
        if (P->owns_gather) P->gather = reinterpret_cast<double*>(P->win + L.gather);
    }

    alloc((void**)&P->dinv, n * 8);
    alloc((void**)&P->r, n * 8);
    alloc((void**)&P->w, n * 8);
    alloc((void**)&P->hist, (P->cfg.max_it + 1) * 8);
    alloc((void**)&P->beta, (P->cfg.max_it + 1) * 8);
    alloc((void**)&P->st, sizeof(CgState));
    alloc((void**)&P->partials, 4 * kMaxReduceBlocks * 8);
    alloc((void**)&P->tickets, 16 * 4);
    if (e != cudaSuccess) return cuda_error(e, "rvk_dcg_plan_create: allocation");
    return RVK_OK;
}

DcgScalars scalars(rvk_dcg_plan P)
{
    return DcgScalars{P->st, P->hist, P->beta, P->gather, P->sh.nranks, P->cfg.rtol, P->cfg.atol};
}

int64_t plane(const rvk_dcg_plan P) { return P->sh.halo_lo ? P->sh.halo_lo : P->sh.halo_hi; }

// ---- per-phase enqueue (one shard) -----------------------------------------
// The PEER variants carry the in-kernel communication; otherwise the NCCL /
// loopback exchange is enqueued between the phases by the caller.
int pc_mode(const rvk_dcg_plan P)
{
    return P->cfg.pc != RVK_PC_JACOBI ? 0 : (P->const_diag ? 2 : 1);
}

bool x_solve(const rvk_dcg_plan P);

template <int PC, bool PEER>
void launch_setup_k(rvk_dcg_plan P, const double* b, double* x)
{
    k_dcg_setup<PC, PEER><<<P->upd_grid, kUpdThreads, 0, P->ctx->stream>>>(
        P->sh.n_own, b, P->dinv, P->dconst, x, P->r, P->z + P->sh.halo_lo, P->gather, P->sh.rank,
        P->partials, P->tickets, P->st, P->peer, x_solve(P) ? 0 : 1);
}

template <bool PEER>
void dispatch_setup(rvk_dcg_plan P, const double* b, double* x)
{
    switch (pc_mode(P)) {
    case 0: launch_setup_k<0, PEER>(P, b, x); break;
    case 1: launch_setup_k<1, PEER>(P, b, x); break;
    default: launch_setup_k<2, PEER>(P, b, x);
    }
}

rvk_status phase_setup(rvk_dcg_plan P, const double* b, double* x)
{
    k_dcg_reset<<<1, 1, 0, P->ctx->stream>>>(P->st);
    if (P->peer.on) dispatch_setup<true>(P, b, x);
    else dispatch_setup<false>(P, b, x);
    RVK_CHECK_LAUNCH("k_dcg_setup");
    return RVK_OK;
}

template <bool FIRST, bool PEER>
rvk_status launch_k1(rvk_dcg_plan P, int it)
{
    const double*  po = P->p[it % P->npb];
    double*        pn = P->p[(it + 1) % P->npb];
    const TailArgs ta{P->partials + 2 * kMaxReduceBlocks, P->tickets + 1};
    double*        go = P->gather + P->sh.rank * 4 + 2;
    const int      k  = (it + 1) % P->npb; // p_new's buffer index, also in the neighbours
    const int64_t          ho = P->sh.halo_lo;
    DcgSpmvOp<FIRST, PEER> op{P->z, po, pn, P->w, scalars(P), ho, go, it, 0.0, P->peer,
                              P->peer.lo_p[k], P->peer.hi_p[k], 0u, P->z + ho, po + ho, pn + ho};
    if constexpr (!FIRST)
        if (P->march) return launch_spmv_march(P->ctx->stream, P->sa_m, P->mg, op, ta);
    return launch_spmv(P->ctx->stream, P->sa, op, ta, sm_count());
}

rvk_status phase_k1(rvk_dcg_plan P, int it)
{
    if (P->peer.on) return it == 0 ? launch_k1<true, true>(P, it) : launch_k1<false, true>(P, it);
    return it == 0 ? launch_k1<true, false>(P, it) : launch_k1<false, false>(P, it);
}

// x update once per solve (ring = max_it: every K2 defers, k_cg_xfix applies
// them at the end) or per iteration pair (as rvk_cg.cu)
bool x_defer(const rvk_dcg_plan P) { return P->cfg.max_it >= 2; }
bool x_solve(const rvk_dcg_plan P) { return x_defer(P) && P->npb > 2; }
int x_mode(const rvk_dcg_plan P, int it)
{
    if (!x_defer(P)) return 0;
    if (x_solve(P)) return 1;
    return (it & 1) ? 2 : (it + 1 < P->cfg.max_it ? 1 : 0);
}

template <int PC, bool PEER, int XM>
void launch_update_k(rvk_dcg_plan P, int it, double* x)
{
    const double* pn = P->p[(it + 1) % P->npb] + P->sh.halo_lo;
    const double* pp = P->p[it % P->npb] + P->sh.halo_lo;
    double*       zo = P->z + P->sh.halo_lo;
    auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    const bool vec = a16(x) && a16(pn) && a16(pp) && a16(zo) && a16(P->dinv) && a16(P->r) && a16(P->w);
    auto go = [&](auto kern) {
        kern<<<P->upd_grid, kUpdThreads, 0, P->ctx->stream>>>(
            P->sh.n_own, pn, P->w, P->dinv, P->dconst, x, P->r, zo, scalars(P), it, P->sh.rank,
            P->gather + P->sh.rank * 4, P->partials, P->tickets, P->peer, pp,
            x_solve(P) ? it : 0, (it + 1 == P->cfg.max_it && !(P->cfg.opts & RVK_OPT_KEEP_WORK)) ? 1 : 0);
    };
    if (vec) go(k_dcg_update<PC, PEER, XM, true>);
    else go(k_dcg_update<PC, PEER, XM, false>);
}

template <bool PEER, int XM>
void dispatch_update(rvk_dcg_plan P, int it, double* x)
{
    switch (pc_mode(P)) {
    case 0: launch_update_k<0, PEER, XM>(P, it, x); break;
    case 1: launch_update_k<1, PEER, XM>(P, it, x); break;
    default: launch_update_k<2, PEER, XM>(P, it, x);
    }
}

template <bool PEER>
void dispatch_update_xm(rvk_dcg_plan P, int it, double* x)
{
    switch (x_mode(P, it)) {
    case 1: dispatch_update<PEER, 1>(P, it, x); break;
    case 2: dispatch_update<PEER, 2>(P, it, x); break;
    default: dispatch_update<PEER, 0>(P, it, x);
    }
}

rvk_status phase_k2(rvk_dcg_plan P, int it, double* x)
{
    if (P->peer.on) dispatch_update_xm<true>(P, it, x);
    else dispatch_update_xm<false>(P, it, x);
    RVK_CHECK_LAUNCH("k_dcg_update");
    return RVK_OK;
}

rvk_status phase_xfix(rvk_dcg_plan P, double* x)
{
    if (!x_defer(P)) return RVK_OK;
    XBufs pb{};
    for (int k = 0; k < P->npb; ++k) pb.p[k] = P->p[k] + P->sh.halo_lo;
    k_cg_xfix<4><<<P->xfix_grid, kUpdThreads, 0, P->ctx->stream>>>(P->sh.n_own, x, pb, P->npb,
                                                                   P->st, x_solve(P) ? 1 : 0);
    RVK_CHECK_LAUNCH("k_cg_xfix");
    return RVK_OK;
}

rvk_status phase_finish(rvk_dcg_plan P)
{
    if (P->peer.on) k_dcg_finish<true><<<1, 32, 0, P->ctx->stream>>>(scalars(P), P->cfg.max_it, P->peer);
    else k_dcg_finish<false><<<1, 32, 0, P->ctx->stream>>>(scalars(P), P->cfg.max_it, P->peer);
    RVK_CHECK_LAUNCH("k_dcg_finish");
    return RVK_OK;
}

// ---- NCCL collectives (one shard per process) --------------------------------
rvk_status nccl_allgather(rvk_dcg_plan P)
{
    double* mine = P->gather + P->sh.rank * 4;
    RVK_TRACE_TASK(P->ctx, "dcg.nccl_allgather");
    RVK_NCCL(nccl().AllGather(mine, P->gather, 4, ncclDouble, P->comm->comm, P->ctx->stream));
    return RVK_OK;
}

rvk_status nccl_halo(rvk_dcg_plan P, bool with_p, int it)
{
    const int64_t pl   = plane(P);
    const int     rank = P->sh.rank, np = P->sh.nranks;
    if (np == 1) return RVK_OK;
    double*     vecs[2] = {P->z, P->p[it % P->npb]};
    const int   nv      = with_p ? 2 : 1;
    auto&       api     = nccl();
    cudaStream_t s      = P->ctx->stream;
    RVK_TRACE_TASK(P->ctx, "dcg.nccl_halo");
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
            auto vec = [&](rvk_dcg_plan Q) { return v == 0 ? Q->z : Q->p[it % Q->npb]; };
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

rvk_status rvk_comm_size(rvk_comm c, int* nranks, int* rank)
{
    if (!c || !nranks || !rank) return set_error(RVK_ERR_INVALID, "comm_size: null argument");
    *nranks = c->nranks;
    *rank   = c->rank;
    // NCCL's own view of the communicator when the library exposes it
    if (c->comm && nccl().CommCount && nccl().CommUserRank) {
        RVK_NCCL(nccl().CommCount(c->comm, nranks));
        RVK_NCCL(nccl().CommUserRank(c->comm, rank));
    }
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
    RVK_TRACE_TASK(ctx, "dcg.plan_create");
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
    if (comm && shared_gather)
        return set_error(RVK_ERR_INVALID, "dcg_plan_create: shared_gather is for loopback shards only");
    int64_t maxlen = 0;
    RVK_TRY(rvk_csr_validate(ctx, A, &maxlen));
    auto P         = new rvk_dcg_plan_s();
    P->ctx         = ctx;
    P->comm        = comm;
    P->A           = *A;
    P->sh          = sh;
    P->cfg         = cfg;
    SpmvBands bands; // leading-edge L2 prefetch (see rvk_cg.cu)
    if (csr_bands(ctx->stream, *A, &bands) != RVK_OK) bands = SpmvBands{};
    P->sa          = make_spmv_args(*A, maxlen, &bands);
    {
        // plane stride: one halo = one plane (z-slab shards); a single shard
        // has no halo, its CSR diagonals give it (rvk_cg.cu csr_bands)
        const int64_t q = sh.halo_lo ? sh.halo_lo : (sh.halo_hi ? sh.halo_hi : bands.plane_q);
        if ((cfg.opts & RVK_OPT_MARCH) && q > 0)
            P->march = make_spmv_march(*A, maxlen, q, sm_count(), &P->sa_m, &P->mg);
    }
    P->upd_grid    = resident_grid(k_dcg_update<1, true, 2, true>, kUpdThreads, (sh.n_own + 1) / 2);
    P->xfix_grid   = resident_grid(k_cg_xfix<4>, kUpdThreads, (sh.n_own + 1) / 2);
    P->owns_gather = shared_gather == nullptr;
    P->gather      = shared_gather;
    rvk_status rc  = alloc_plan_buffers(P);
    // dinv of the owned rows: the local CSR's diagonal sits at column row + halo_lo
    if (rc == RVK_OK) {
        if (cfg.pc == RVK_PC_JACOBI) rc = diag_inverse(ctx->stream, *A, sh.halo_lo, P->dinv);
        else rc = rvk_set(ctx, sh.n_own, 1.0, P->dinv);
    }
    // constant diagonal -> scalar Jacobi (as rvk_cg_plan_create; RVK_OPT_DINV_VECTOR disables).
    // Every shard of a constant-coefficient operator sees the same value.
    if (rc == RVK_OK && cfg.pc == RVK_PC_JACOBI && sh.n_own > 0 && !(cfg.opts & RVK_OPT_DINV_VECTOR))
        rc = vector_is_constant(ctx->stream, sh.n_own, P->dinv, &P->const_diag, &P->dconst);
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
    // (PEER: the caller keeps every rank alive past its last solve -- a
    // barrier before destroy -- since peers store into this window)
    if (P->graph) cudaGraphExecDestroy(P->graph);
    void* bufs[] = {P->win, P->dinv, P->r, P->w, P->hist, P->beta, P->st, P->partials, P->tickets,
                    P->peer_tab};
    for (void* b : bufs)
        if (b) cudaFree(b);
    delete P;
    return RVK_OK;
}

namespace {
rvk_status enqueue_dcg(rvk_dcg_plan P, const double* b_own, double* x_own)
{
    const bool dist = !P->peer.on && P->comm && P->sh.nranks > 1;
    RVK_TRY(phase_setup(P, b_own, x_own));
    if (dist) RVK_TRY(nccl_allgather(P));
    for (int it = 0; it < P->cfg.max_it; ++it) {
        if (dist) RVK_TRY(nccl_halo(P, it > 0, it));
        RVK_TRY(phase_k1(P, it));
        if (dist) RVK_TRY(nccl_allgather(P));
        RVK_TRY(phase_k2(P, it, x_own));
        if (dist) RVK_TRY(nccl_allgather(P));
    }
    RVK_TRY(phase_finish(P));
    return phase_xfix(P, x_own);
}
} // namespace

// One shard per process: the whole solve, stream-ordered, no host sync.
// PEER: 2 kernels per iteration carry all communication; NCCL: halo
// send/recv + 2 allgathers per iteration between the kernels.  With
// cfg.use_graph the solve is captured once per (b, x) into a CUDA graph and
// replayed, in thread-local capture mode: any synchronous CUDA call this
// thread makes while the solve is enqueued fails the capture (the structural
// proof of zero host syncs, as in rvk_cg_solve_dev), while other host threads
// -- NCCL's proxy thread, other devices' threads -- are not affected.
rvk_status rvk_dcg_solve_dev(rvk_dcg_plan P, const double* b_own, double* x_own)
{
    if (!P || !b_own || !x_own) return set_error(RVK_ERR_INVALID, "null argument");
    if (!P->comm && !P->peer.on && P->sh.nranks > 1)
        return set_error(RVK_ERR_INVALID, "loopback shards are solved with rvk_dcg_loopback_solve");
    RVK_TRACE_TASK(P->ctx, "dcg.solve");
    if (!P->cfg.use_graph) return enqueue_dcg(P, b_own, x_own);
    cudaStream_t s = P->ctx->stream;
    if (!(P->graph && P->graph_b == b_own && P->graph_x == x_own)) {
        if (P->graph) cudaGraphExecDestroy(P->graph);
        P->graph          = nullptr;
        cudaGraph_t  g    = nullptr;
        RVK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        rvk_status  rc = enqueue_dcg(P, b_own, x_own);
        cudaError_t e  = cudaStreamEndCapture(s, &g);
        if (rc != RVK_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) return cuda_error(e, "cudaStreamEndCapture (sharded solve not capturable)");
        e = cudaGraphInstantiate(&P->graph, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            P->graph = nullptr;
            return cuda_error(e, "cudaGraphInstantiate (sharded solve)");
        }
        P->graph_b = b_own;
        P->graph_x = x_own;
    }
    RVK_CUDA(cudaGraphLaunch(P->graph, s));
    return RVK_OK;
}

// All P shards on one device, enqueued phase by phase on shard 0's stream
// order (each plan's own stream; cross-shard edges via events).
rvk_status rvk_dcg_loopback_solve(rvk_dcg_plan* Ps, int np, const double* const* b, double* const* x)
{
    if (!Ps || np < 1 || !b || !x) return set_error(RVK_ERR_INVALID, "null argument");
    const bool peer = Ps[0]->peer.on;
    for (int r = 0; r < np; ++r) {
        if (Ps[r]->ctx->stream != Ps[0]->ctx->stream)
            return set_error(RVK_ERR_INVALID, "loopback shards must share one context/stream");
        if (Ps[r]->peer.on != peer || Ps[r]->comm)
            return set_error(RVK_ERR_INVALID, "loopback shards: all PEER-attached or all shared-gather");
        if (!peer && np > 1 && (Ps[r]->owns_gather || Ps[r]->gather != Ps[0]->gather))
            return set_error(RVK_ERR_INVALID, "loopback shards need one shared gather buffer");
    }
    RVK_TRACE_TASK(Ps[0]->ctx, "dcg.loopback_solve");
    // phase-major order: every flag a PEER kernel waits for was released by
    // a kernel enqueued before it on this stream (no spin ever blocks)
    for (int r = 0; r < np; ++r) RVK_TRY(phase_setup(Ps[r], b[r], x[r]));
    for (int it = 0; it < Ps[0]->cfg.max_it; ++it) {
        if (!peer) RVK_TRY(loop_halo(Ps, np, it > 0, it));
        for (int r = 0; r < np; ++r) RVK_TRY(phase_k1(Ps[r], it));
        for (int r = 0; r < np; ++r) RVK_TRY(phase_k2(Ps[r], it, x[r]));
    }
    for (int r = 0; r < np; ++r) RVK_TRY(phase_finish(Ps[r]));
    for (int r = 0; r < np; ++r) RVK_TRY(phase_xfix(Ps[r], x[r]));
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
    {
        trace::HostSyncScope hs_("rvk_dcg_result");
        RVK_CUDA(cudaStreamSynchronize(s));
    }
    if (info) {
        info->state          = h.state;
        info->iterations     = h.iterations;
        info->breakdown_iter = h.breakdown_iter;
    }
    if (h.state == RVK_CG_BREAKDOWN)
        return set_error(RVK_ERR_BREAKDOWN, "cg_solve: breakdown at iteration %d", h.breakdown_iter);
    if (h.state == RVK_CG_COMM_ERROR)
        return set_error(RVK_ERR_COMM, "dcg_solve: a peer did not arrive within %llu s (PEER backend)",
                         (unsigned long long)(kPeerTimeoutNs / 1000000000ull));
    // NCCL backend: an asynchronous communicator error (a peer died, a
    // network fault) surfaces here, never as a hang in a later solve
    if (P->comm && P->comm->comm && nccl().CommGetAsyncError) {
        ncclResult_t ae = ncclSuccess;
        if (nccl().CommGetAsyncError(P->comm->comm, &ae) == ncclSuccess && ae != ncclSuccess &&
            ae != ncclInProgress)
            return nccl_error(ae, "dcg_solve: NCCL communicator async error");
    }
    return RVK_OK;
}

int rvk_dcg_plan_flags(rvk_dcg_plan P)
{
    if (!P) return -1;
    return (P->const_diag ? RVK_PLAN_CONST_DIAG : 0) |
           (x_defer(P) ? RVK_PLAN_X_DEFER : 0) | (x_solve(P) ? RVK_PLAN_X_SOLVE : 0) |
           (P->march ? RVK_PLAN_MARCH : 0);
}

// ---- PEER backend ----------------------------------------------------------
rvk_status rvk_dcg_window(rvk_dcg_plan P, void** base, size_t* bytes)
{
    if (!P || !base || !bytes) return set_error(RVK_ERR_INVALID, "null argument");
    *base  = P->win;
    *bytes = P->win_bytes;
    return RVK_OK;
}

rvk_status rvk_dcg_attach_peers(rvk_dcg_plan P, void* const* windows, const rvk_shard* shards)
{
    if (!P || !windows || !shards) return set_error(RVK_ERR_INVALID, "null argument");
    const int np = P->sh.nranks, me = P->sh.rank;
    if (P->comm || !P->owns_gather)
        return set_error(RVK_ERR_INVALID, "attach_peers: plan was created for the NCCL / shared-gather loopback backend");
    if (windows[me] != P->win)
        return set_error(RVK_ERR_INVALID, "attach_peers: windows[rank] must be this plan's own window");
    for (int q = 0; q < np; ++q) {
        const rvk_shard& s = shards[q];
        if (!windows[q] || s.rank != q || s.nranks != np)
            return set_error(RVK_ERR_INVALID, "attach_peers: shard %d does not describe rank %d of %d", q, q, np);
    }
    const int64_t pl = plane(P);
    auto ext = [&](int q) { return shards[q].halo_lo + shards[q].n_own + shards[q].halo_hi; };
    auto at  = [&](int q, size_t off) { return reinterpret_cast<unsigned char*>(windows[q]) + off; };
    std::vector<void*> tab(2 * np);
    auto lay = [&](int q) { return window_layout(ext(q), ring_len(P->cfg.max_it, ext(q))); };
    for (int q = 0; q < np; ++q) {
        const WindowLayout L = lay(q);
        if (L.npb != P->npb)
            return set_error(RVK_ERR_INVALID, "attach_peers: rank %d's p ring (%d) differs from this rank's (%d)",
                             q, L.npb, P->npb);
        tab[q]      = at(q, L.gather);
        tab[np + q] = at(q, L.flags);
    }
    DcgPeer pr{};
    pr.on     = 1;
    pr.rank   = me;
    pr.nranks = np;
    pr.plane  = pl;
    pr.n_own  = P->sh.n_own;
    const WindowLayout Lme = window_layout(P->n_ext, P->npb);
    pr.my_flags            = reinterpret_cast<const uint64_t*>(P->win + Lme.flags);
    if (me > 0) { // my first owned plane -> the upper halo of rank-1
        const rvk_shard&   d   = shards[me - 1];
        const WindowLayout L   = lay(me - 1);
        const size_t       off = (size_t)(d.halo_lo + d.n_own) * 8;
        if (d.halo_hi != pl) return set_error(RVK_ERR_DIM, "attach_peers: plane size mismatch with rank %d", me - 1);
        pr.lo_z    = reinterpret_cast<double*>(at(me - 1, L.z + off));
        for (int k = 0; k < P->npb; ++k) pr.lo_p[k] = reinterpret_cast<double*>(at(me - 1, L.p(k) + off));
    }
    if (me < np - 1) { // my last owned plane -> the lower halo of rank+1 (element 0)
        const rvk_shard&   u = shards[me + 1];
        const WindowLayout L = lay(me + 1);
        if (u.halo_lo != pl) return set_error(RVK_ERR_DIM, "attach_peers: plane size mismatch with rank %d", me + 1);
        pr.hi_z    = reinterpret_cast<double*>(at(me + 1, L.z));
        for (int k = 0; k < P->npb; ++k) pr.hi_p[k] = reinterpret_cast<double*>(at(me + 1, L.p(k)));
    }
    if (!P->peer_tab) RVK_CUDA(cudaMalloc(&P->peer_tab, 2 * kMaxRanks * sizeof(void*)));
    RVK_CUDA(cudaMemcpy(P->peer_tab, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice));
    pr.gather = reinterpret_cast<double* const*>(P->peer_tab);
    pr.flags  = reinterpret_cast<uint64_t* const*>(P->peer_tab + np);
    // fresh protocol state: flags 0, solve counter 0 (before any peer stores)
    RVK_CUDA(cudaMemsetAsync(P->win + Lme.flags, 0, kMaxRanks * sizeof(uint64_t), P->ctx->stream));
    RVK_CUDA(cudaMemsetAsync(P->st, 0, sizeof(CgState), P->ctx->stream));
    RVK_CUDA(cudaStreamSynchronize(P->ctx->stream));
    P->peer = pr;
    return RVK_OK;
}

rvk_status rvk_ipc_get_handle(const void* dev_base, void* handle_out, int handle_bytes)
{
    if (!dev_base || !handle_out || handle_bytes < (int)sizeof(cudaIpcMemHandle_t))
        return set_error(RVK_ERR_INVALID, "ipc_get_handle: need %d bytes", (int)sizeof(cudaIpcMemHandle_t));
    cudaIpcMemHandle_t h;
    RVK_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_base)));
    std::memcpy(handle_out, &h, sizeof h);
    return RVK_OK;
}

rvk_status rvk_ipc_open_handle(const void* handle, void** dev_ptr)
{
    if (!handle || !dev_ptr) return set_error(RVK_ERR_INVALID, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    RVK_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return RVK_OK;
}

rvk_status rvk_ipc_close_handle(void* dev_ptr)
{
    if (!dev_ptr) return RVK_OK;
    RVK_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return RVK_OK;
}

} // extern "C"
