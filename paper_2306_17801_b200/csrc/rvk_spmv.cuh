// rvk_spmv.cuh -- TMA-pipelined CSR SpMV mainloop for sm_100a.
//
// Computes, for every row i, sum_i = sum_k vals[k] * SRC(cols[k]) with the
// reference's exact per-row order (kernels_scalar.cpp:53-63: sum starts at
// 0.0, left to right, each product rounded before it is added), so the result
// is bit-identical to rivulet::kernels::scalar::csr_spmv when SRC(j) = x[j].
//
// Design (B200-first; HBM-bound: 12 B/nnz of streamed CSR + gathers):
//  * persistent grid, one CTA per SM (148 on B200); tiles of R consecutive
//    rows assigned round-robin, so the rows in flight chip-wide stay inside a
//    narrow window and the x-gather is served by L2;
//  * warp-specialised: warp 0 is the producer -- one lane issues
//    cp.async.bulk (TMA bulk copies, UBLKCP in SASS) of the tile's row
//    offsets, values and column indices into an S-deep shared-memory ring
//    (S, R and the stage capacity are sized per matrix at plan time), with
//    mbarrier full/empty handshakes and an L2 evict_first policy on the
//    streamed-once CSR bytes;
//  * warps 1..16 consume: lane-per-row (consecutive lanes own consecutive
//    rows, so for banded/stencil matrices every gather instruction of a warp
//    hits one contiguous run -- perfectly coalesced), reading (col, val) from
//    the stage with LDS; per batch of 8 nonzeros a thread first reads all
//    8 pairs, then issues all 8 gathers, then adds the rounded products
//    strictly left to right (the reference's order => bit-exact).  When a
//    tile is shorter than the 512 consumer threads (long rows, e.g. 27-point:
//    R = 128) the consumers split into NG groups that work on NG different
//    ring stages at once, so no thread idles;
//  * tiles that do not fit a stage (very long rows) and the last tile (whose
//    16-byte-rounded bulk range could run past the arrays) are "direct":
//    consumers read them from global memory thread-per-row;
//  * Op supplies SRC(j) (split into raw fetch + arithmetic so every gather is
//    issued before any is consumed), the per-row epilogue and the reduction
//    tail, so the same mainloop serves mat_mult and the fused CG kernel
//    (p = z + b p on the fly; w = A p; p.w partials; alpha tail).
#pragma once

#include "rvk_common.cuh"

namespace rvk {

constexpr int    kSpmvConsumerWarps = 16;
constexpr int    kSpmvConsumers     = kSpmvConsumerWarps * 32;
constexpr int    kSpmvThreads       = kSpmvConsumers + 32; // + producer warp
constexpr int    kSpmvMaxStages     = 4;
constexpr int    kSpmvChunkRows     = 32;
constexpr int    kSpmvUnroll        = 8;                   // nonzeros per lane per sweep step
constexpr size_t kSpmvHeaderBytes   = 1024;                // barriers, meta, reduction scratch
constexpr size_t kSpmvStageBudget   = 200 * 1024;          // dynamic smem for the ring

struct SpmvStageMeta {
    int64_t kv0;    // first value index held in the stage (16-B aligned)
    int64_t kc0;    // first column index held in the stage (16-B aligned)
    int     direct; // 1: read this tile from global memory
    int     pad;
};

struct SpmvArgs {
    int64_t        n_rows;
    int64_t        n_tiles;
    int            R;        // rows per tile (multiple of 32)
    int            stages;   // ring depth (<= kSpmvMaxStages)
    int            groups;   // consumer groups working on distinct stages (divides stages)
    int            cap;      // nonzeros per stage
    int            off_bytes, val_bytes, stage_bytes; // stage layout: [off | vals | cols]
    const int64_t* off;
    const int32_t* cols;
    const double*  vals;

    size_t smem_bytes() const { return kSpmvHeaderBytes + (size_t)stages * stage_bytes; }
};

// Shared reduction workspace used by Ops with a tail.
struct TailArgs {
    double*       partials;
    unsigned int* ticket;
};

__host__ __device__ inline int align16(int64_t b) { return (int)((b + 15) & ~int64_t(15)); }

// Tile geometry for a matrix whose longest row has max_row_len nonzeros: the
// largest R (multiple of 32, <= 1024) whose worst-case slab fits a stage with
// at least 3 stages in the ring, else 2.  Rows too long for any stage still
// work (direct tiles).
inline SpmvArgs make_spmv_args(const rvk_csr& A, int64_t max_row_len)
{
    if (max_row_len < 1) max_row_len = 1;
    SpmvArgs a{};
    a.n_rows = A.n_rows;
    a.off    = A.row_offsets;
    a.cols   = A.col_indices;
    a.vals   = A.values;
    auto fit = [&](int R, int min_stages) {
        const int64_t cap = ((R * max_row_len + 8) + 3) & ~int64_t(3);
        const int64_t ob = align16((int64_t)(R + 2) * 8), vb = cap * 8, cb = align16(cap * 4);
        const int64_t sb = ob + vb + cb;
        const int64_t st = std::min<int64_t>(kSpmvMaxStages, (int64_t)kSpmvStageBudget / sb);
        if (st < min_stages) return false;
        a.R = R;
        a.stages = (int)st;
        a.cap = (int)cap;
        a.off_bytes = (int)ob;
        a.val_bytes = (int)vb;
        a.stage_bytes = (int)sb;
        return true;
    };
    bool ok = false;
    for (int need = 3; need >= 2 && !ok; --need)
        for (int R = 1024; R >= 32 && !ok; R /= 2) ok = fit(R, need);
    if (!ok) { // rows longer than a stage: every tile direct, small ring
        a.R = 32;
        a.stages = 4;
        a.off_bytes = align16(34 * 8);
        a.cap = (int)(((kSpmvStageBudget / 4 - a.off_bytes) / 12) & ~size_t(3));
        a.val_bytes = a.cap * 8;
        a.stage_bytes = a.off_bytes + a.val_bytes + align16((int64_t)a.cap * 4);
    }
    a.n_tiles = (A.n_rows + a.R - 1) / a.R;
    // enough groups that every consumer thread owns a row of some tile
    a.groups = 1;
    while (a.groups * 2 <= a.stages && a.stages % (a.groups * 2) == 0 &&
           a.R * a.groups * 2 <= kSpmvConsumers)
        a.groups *= 2;
    return a;
}

// ---------------------------------------------------------------------------
// Direct tiles: thread-per-row straight from global memory (rare path).
// ---------------------------------------------------------------------------
template <class Op>
__device__ __forceinline__ double spmv_rows_direct(const Op& op, double acc, int gtid, int gsize,
                                                   int rows, int64_t r0,
                                                   const int64_t* __restrict__ O,
                                                   const int32_t* __restrict__ Cc,
                                                   const double* __restrict__ V)
{
    for (int lr = gtid; lr < rows; lr += gsize) {
        const int64_t kb = O[lr], ke = O[lr + 1];
        double        sum = 0.0;
        for (int64_t k = kb; k < ke; k += kSpmvUnroll) {
            int32_t c[kSpmvUnroll];
            double  v[kSpmvUnroll];
            bool    ok[kSpmvUnroll];
#pragma unroll
            for (int u = 0; u < kSpmvUnroll; ++u) {
                ok[u]            = k + u < ke;
                const int64_t ks = ok[u] ? k + u : ke - 1;
                c[u]             = __ldg(Cc + ks);
                v[u]             = __ldg(V + ks);
            }
            typename Op::Fetch f[kSpmvUnroll];
#pragma unroll
            for (int u = 0; u < kSpmvUnroll; ++u) f[u] = op.fetch(c[u]);
#pragma unroll
            for (int u = 0; u < kSpmvUnroll; ++u) {
                const double t = add(sum, mul(v[u], op.value(f[u])));
                sum            = ok[u] ? t : sum;
            }
        }
        acc = op.row(r0 + lr, sum, acc, op.own_fetch(r0 + lr));
    }
    return acc;
}

// ---------------------------------------------------------------------------
// Staged tiles: lane-per-row out of the shared-memory stage.
//   O  : the tile's row offsets in shared memory (global nnz indices)
//   V  : stage values, V[k - kv0];  Cc : stage columns, Cc[k - kv0]
// Stage-local 32-bit indices keep the address arithmetic cheap.
// ---------------------------------------------------------------------------
template <class Op>
__device__ __forceinline__ double spmv_rows_staged(const Op& op, double acc, int gtid, int gsize,
                                                   int rows, int64_t r0, const int64_t* O,
                                                   int64_t kv0, const int32_t* Cc,
                                                   const double* V)
{
    for (int lr = gtid; lr < rows; lr += gsize) {
        const auto own = op.own_fetch(r0 + lr); // epilogue operands, in flight early
        const int  kb  = (int)(O[lr] - kv0);
        const int  ke  = (int)(O[lr + 1] - kv0);
        double     sum = 0.0;
        for (int k = kb; k < ke; k += kSpmvUnroll) {
            int32_t c[kSpmvUnroll];
            double  v[kSpmvUnroll];
            bool    ok[kSpmvUnroll];
#pragma unroll
            for (int u = 0; u < kSpmvUnroll; ++u) {
                ok[u]        = k + u < ke;
                const int ks = ok[u] ? k + u : k; // k < ke: a valid entry
                c[u]         = Cc[ks];
                v[u]         = V[ks];
            }
            typename Op::Fetch f[kSpmvUnroll];
#pragma unroll
            for (int u = 0; u < kSpmvUnroll; ++u) f[u] = op.fetch(c[u]);
#pragma unroll
            for (int u = 0; u < kSpmvUnroll; ++u) {
                const double t = add(sum, mul(v[u], op.value(f[u])));
                sum            = ok[u] ? t : sum;
            }
        }
        acc = op.row(r0 + lr, sum, acc, own);
    }
    return acc;
}

template <class Op>
__global__ void __launch_bounds__(kSpmvThreads, 1) k_spmv_tma(SpmvArgs A, Op op_in, TailArgs tail)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t*      full   = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t*      empty  = full + kSpmvMaxStages;
    SpmvStageMeta* meta   = reinterpret_cast<SpmvStageMeta*>(smem_raw + 128);
    double*        red    = reinterpret_cast<double*>(smem_raw + 512); // 32 doubles
    int*           flag   = reinterpret_cast<int*>(smem_raw + 512 + 256);
    unsigned char* stage0 = smem_raw + kSpmvHeaderBytes;

    Op op = op_in;
    if (!op.init()) return; // device-side early exit (converged / breakdown)

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < A.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kSpmvConsumerWarps / A.groups);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (tid < 32) {
        // ===================== producer warp =====================
        if (tid == 0) {
            const uint64_t pol = policy_evict_first();
            int64_t        t   = blockIdx.x;
            int64_t        k0 = 0, k1 = 0; // slab bounds, prefetched one tile ahead
            if (t < A.n_tiles) {
                k0 = __ldg(A.off + t * A.R);
                k1 = __ldg(A.off + min(t * A.R + A.R, A.n_rows));
            }
            for (int j = 0; t < A.n_tiles; ++j, t += gridDim.x) {
                const int s = j % A.stages;
                if (j >= A.stages) mbar_wait(&empty[s], ((j / A.stages) - 1) & 1);
                const int64_t r0 = t * A.R;
                const int64_t r1 = min(r0 + A.R, A.n_rows);
                const int64_t ck0 = k0, ck1 = k1;
                const int64_t tn  = t + gridDim.x;
                if (tn < A.n_tiles) {
                    k0 = __ldg(A.off + tn * A.R);
                    k1 = __ldg(A.off + min(tn * A.R + A.R, A.n_rows));
                }
                const int64_t kv0 = ck0 & ~int64_t(1), kv1 = (ck1 + 1) & ~int64_t(1);
                const int64_t kc0 = ck0 & ~int64_t(3), kc1 = (ck1 + 3) & ~int64_t(3);
                const bool    last   = r1 >= A.n_rows;
                const bool    direct = last || (kv1 - kv0) > A.cap || (kc1 - kc0) > A.cap;
                meta[s].kv0          = kv0;
                meta[s].kc0          = kc0;
                meta[s].direct       = direct ? 1 : 0;
                if (direct) {
                    mbar_arrive(&full[s]);
                } else {
                    unsigned char* st = stage0 + (size_t)s * A.stage_bytes;
                    const uint32_t ob = (uint32_t)((A.R + 2) * 8);
                    const uint32_t vb = (uint32_t)((kv1 - kv0) * 8);
                    const uint32_t cb = (uint32_t)((kc1 - kc0) * 4);
                    mbar_arrive_expect_tx(&full[s], ob + vb + cb);
                    bulk_g2s(st, A.off + r0, ob, &full[s], pol);
                    if (vb) bulk_g2s(st + A.off_bytes, A.vals + kv0, vb, &full[s], pol);
                    if (cb)
                        bulk_g2s(st + A.off_bytes + A.val_bytes, A.cols + kc0, cb, &full[s], pol);
                }
            }
        }
        return; // the producer warp takes no part in the consumer reduction
    }

    // ===================== consumer warps =====================
    // NG groups of GS threads; group q takes the tiles j with j % NG == q
    // (NG divides the ring depth, so a group always owns the same stages).
    const int ctid  = tid - 32;
    const int gs    = kSpmvConsumers / A.groups;
    const int group = ctid / gs, gtid = ctid % gs;
    double    acc   = 0.0;
    int64_t   t     = blockIdx.x + (int64_t)group * gridDim.x;
    for (int j = group; t < A.n_tiles; j += A.groups, t += (int64_t)A.groups * gridDim.x) {
        const int s = j % A.stages;
        mbar_wait(&full[s], (j / A.stages) & 1);
        const int64_t r0   = t * A.R;
        const int     rows = (int)min((int64_t)A.R, A.n_rows - r0);
        if (meta[s].direct) {
            acc = spmv_rows_direct(op, acc, gtid, gs, rows, r0, A.off + r0, A.cols, A.vals);
        } else {
            unsigned char* st  = stage0 + (size_t)s * A.stage_bytes;
            const int64_t  kv0 = meta[s].kv0;
            // columns were copied from kc0 <= kv0: shift so both use kv0-local indices
            const int32_t* Cc = reinterpret_cast<const int32_t*>(st + A.off_bytes + A.val_bytes) +
                                (kv0 - meta[s].kc0);
            acc = spmv_rows_staged(op, acc, gtid, gs, rows, r0,
                                   reinterpret_cast<const int64_t*>(st), kv0, Cc,
                                   reinterpret_cast<const double*>(st + A.off_bytes));
        }
        __syncwarp();
        if ((ctid & 31) == 0) mbar_arrive(&empty[s]);
    }

    if constexpr (Op::kHasTail) {
        double v[1] = {acc};
        block_sum<1>(v, red, ctid, kSpmvConsumers, 1);
        if (ctid == 0) tail.partials[blockIdx.x] = v[0];
        if (!last_block(tail.ticket, ctid, flag, kSpmvConsumers, 1)) return;
        fold_partials<1>(tail.partials, gridDim.x, v, red, ctid, kSpmvConsumers, 1);
        if (ctid == 0) {
            op.tail(v[0]);
            *tail.ticket = 0u;
        }
    }
}

// Plain mat_mult: y = A x.
struct SpmvPlainOp {
    static constexpr bool kHasTail = false;
    const double* __restrict__ x;
    double* __restrict__ y;
    struct Fetch {
        double x;
    };
    __device__ __forceinline__ bool   init() { return true; }
    __device__ __forceinline__ Fetch  fetch(int32_t j) const { return Fetch{__ldg(x + j)}; }
    __device__ __forceinline__ double value(const Fetch& f) const { return f.x; }
    struct Own {};
    __device__ __forceinline__ Own    own_fetch(int64_t) const { return Own{}; }
    __device__ __forceinline__ double row(int64_t i, double sum, double acc, Own) const
    {
        y[i] = sum;
        return acc;
    }
    __device__ __forceinline__ void tail(double) const {}
};

template <class Op>
rvk_status launch_spmv(cudaStream_t stream, const SpmvArgs& a, const Op& op, TailArgs tail,
                       int grid)
{
    static bool configured = false; // per instantiation; before any graph capture
    if (!configured) {
        RVK_CUDA(cudaFuncSetAttribute(k_spmv_tma<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(kSpmvHeaderBytes + kSpmvStageBudget)));
        configured = true;
    }
    k_spmv_tma<Op><<<grid, kSpmvThreads, a.smem_bytes(), stream>>>(a, op, tail);
    RVK_CHECK_LAUNCH("k_spmv_tma");
    return RVK_OK;
}

} // namespace rvk
