// rvk_spmv.cuh -- TMA-pipelined CSR SpMV mainloop for sm_100a.
//
// Computes, for every row i, sum_i = sum_k vals[k] * SRC(cols[k]) with the
// reference's exact per-row order (kernels_scalar.cpp:53-63: sum starts at
// 0.0, left to right, each product rounded before it is added), so the result
// is bit-identical to rivulet::kernels::scalar::csr_spmv when SRC(j) = x[j].
//
// Design (B200-first, HBM-bound: ~12 B/nnz of streamed CSR + gathers):
//  * persistent grid, one CTA per SM (148 on B200), tiles of R consecutive
//    rows assigned round-robin (deterministic, and it keeps the rows in
//    flight chip-wide inside a narrow window so the x-gather reuses L2);
//  * warp-specialised: warp 0 is the producer -- one elected lane issues
//    cp.async.bulk (TMA bulk copies, UBLKCP in SASS) of the tile's row
//    offsets, values and column indices into a STAGES-deep shared-memory
//    ring, with mbarrier full/empty handshakes and an L2 evict_first policy
//    for the streamed-once CSR bytes;
//  * warps 1..8 (256 consumer threads) each own rows tid, tid+256, ... of the
//    tile and walk them sequentially out of shared memory (row stride of an
//    odd nnz/row => conflict-free 64-bit LDS), gathering SRC(j) through L1/L2;
//  * tiles that do not fit a stage (long rows) and the very last tile (whose
//    16-byte-rounded bulk range could run past the arrays) are marked
//    "direct": consumers read them straight from global memory instead.
//  * Op supplies SRC(j), the per-row epilogue and the reduction tail, so the
//    same mainloop serves mat_mult and the fused CG kernel
//    (p = z + b p on the fly; w = A p; p.w partial; alpha tail).
#pragma once

#include "rvk_common.cuh"

namespace rvk {

constexpr int kSpmvConsumers = 256;               // 8 consumer warps
constexpr int kSpmvThreads   = kSpmvConsumers + 32; // + producer warp
constexpr int kSpmvStages    = 3;
constexpr int kSpmvCapNnz    = 5120;              // per-stage nnz capacity
constexpr int kSpmvMaxRows   = 1024;              // per-tile row cap

struct SpmvStageMeta {
    int64_t kv0;    // first value index held in the stage (16-B aligned)
    int64_t kc0;    // first column index held in the stage (16-B aligned)
    int     direct; // 1: read this tile from global memory
    int     pad;
};

// Shared-memory layout of one stage.
struct SpmvLayout {
    int rows_per_tile;
    __host__ __device__ static constexpr size_t off_bytes(int R) { return (size_t)(R + 2) * 8; }
    __host__ __device__ static constexpr size_t val_bytes() { return (size_t)kSpmvCapNnz * 8; }
    __host__ __device__ static constexpr size_t col_bytes() { return (size_t)kSpmvCapNnz * 4; }
    __host__ __device__ static constexpr size_t stage_bytes(int R)
    {
        return ((off_bytes(R) + 15) & ~size_t(15)) + val_bytes() + col_bytes();
    }
    __host__ __device__ static constexpr size_t smem_bytes(int R)
    {
        return 1024 /* barriers + meta */ + kSpmvStages * stage_bytes(R);
    }
};

struct SpmvArgs {
    int64_t        n_rows;
    int64_t        n_tiles;
    int            R;    // rows per tile (even, multiple of 32)
    const int64_t* off;
    const int32_t* cols;
    const double*  vals;
};

// Shared reduction workspace used by Ops with a tail.
struct TailArgs {
    double*       partials;
    unsigned int* ticket;
};

// Rows processed concurrently per consumer thread, and columns per batch.
// Each pass a thread owns G rows (lr, lr+256, ...); for every batch of 8
// columns it first reads all G*8 (col, val) pairs (LDS from the stage, or
// LDG for direct tiles), then issues all G*8 gathers, then folds them into
// the per-row sums strictly left to right -- so the memory-level
// parallelism is G*8 gathers per thread while each row's sum keeps the
// reference's sequential order.
constexpr int kSpmvRowGroup = 2;
constexpr int kSpmvBatch    = 8;

template <int G, typename IDX, class Op>
__device__ __forceinline__ double spmv_rows(const Op& op, double acc, int ctid, int rows,
                                            int64_t r0, const int64_t* __restrict__ O,
                                            int64_t kbase, const int32_t* __restrict__ Cc,
                                            const double* __restrict__ V)
{
    // IDX = int for staged tiles (indices local to the stage: value k lives at
    // V[k - kbase], its column at Cc[k - kbase]), int64_t for direct tiles.
    for (int base = ctid; base < rows; base += G * kSpmvConsumers) {
        IDX     kb[G], ke[G], last[G];
        int32_t safe[G];
        int     len = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int  lr = base + g * kSpmvConsumers;
            const bool in = lr < rows;
            kb[g]         = in ? (IDX)(O[lr] - kbase) : (IDX)0;
            ke[g]         = in ? (IDX)(O[lr + 1] - kbase) : (IDX)0;
            len           = max(len, (int)(ke[g] - kb[g]));
            // dead slots re-read a valid entry (nnz >= 1 is guaranteed by the
            // host) and gather a valid index; they never reach the sum
            last[g] = ke[g] > kb[g] ? ke[g] - 1 : (kb[g] > 0 ? kb[g] - 1 : (IDX)0);
            const int64_t row = r0 + lr;
            safe[g]           = (int32_t)(in && row < op.n_src() ? row : 0);
        }
        double sum[G], own[G];
        bool   have_own[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            sum[g]      = 0.0;
            own[g]      = 0.0;
            have_own[g] = false;
        }
        for (int k = 0; k < len; k += kSpmvBatch) {
            // Branch-free batch: (1) all column/value reads, (2) all gathers,
            // (3) the per-row sums strictly left to right (dead slots dropped
            // by a select), so every load of the batch is in flight together.
            int32_t c[G][kSpmvBatch];
            double  v[G][kSpmvBatch];
            bool    ok[G][kSpmvBatch];
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int u = 0; u < kSpmvBatch; ++u) {
                    const IDX kk = kb[g] + (IDX)(k + u);
                    ok[g][u]     = kk < ke[g];
                    const IDX ks = ok[g][u] ? kk : last[g];
                    c[g][u]      = ok[g][u] ? Cc[ks] : safe[g];
                    v[g][u]      = V[ks];
                }
            typename Op::Fetch f[G][kSpmvBatch];
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int u = 0; u < kSpmvBatch; ++u) f[g][u] = op.fetch(c[g][u]);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int32_t row = (int32_t)(r0 + base + g * kSpmvConsumers);
#pragma unroll
                for (int u = 0; u < kSpmvBatch; ++u) {
                    const double x = op.value(f[g][u]);
                    const double t = add(sum[g], mul(v[g][u], x));
                    sum[g]         = ok[g][u] ? t : sum[g];
                    const bool d   = ok[g][u] && c[g][u] == row;
                    own[g]         = d ? x : own[g];
                    have_own[g]    = have_own[g] || d;
                }
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int lr = base + g * kSpmvConsumers;
            if (lr < rows) acc = op.row(r0 + lr, sum[g], acc, own[g], have_own[g]);
        }
    }
    return acc;
}

template <class Op>
__global__ void __launch_bounds__(kSpmvThreads, 1) k_spmv_tma(SpmvArgs A, Op op_in, TailArgs tail)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t*      full  = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t*      empty = full + kSpmvStages;
    SpmvStageMeta* meta  = reinterpret_cast<SpmvStageMeta*>(smem_raw + 128);
    double*        red   = reinterpret_cast<double*>(smem_raw + 512);  // 32 doubles
    int*           flag  = reinterpret_cast<int*>(smem_raw + 512 + 256);
    unsigned char* stage0 = smem_raw + 1024;
    const size_t   sbytes = SpmvLayout::stage_bytes(A.R);
    const size_t   obytes = (SpmvLayout::off_bytes(A.R) + 15) & ~size_t(15);

    Op op = op_in;
    if (!op.init()) return; // device-side early exit (converged / breakdown)

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < kSpmvStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kSpmvConsumers / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (tid < 32) {
        // ===================== producer warp =====================
        if (tid == 0) {
            const uint64_t pol = policy_evict_first();
            int64_t t = blockIdx.x;
            // prefetch the first tile's slab bounds
            int64_t k0 = 0, k1 = 0;
            if (t < A.n_tiles) {
                const int64_t r0 = t * A.R;
                const int64_t r1 = min(r0 + A.R, A.n_rows);
                k0 = __ldg(A.off + r0);
                k1 = __ldg(A.off + r1);
            }
            for (int j = 0; t < A.n_tiles; ++j, t += gridDim.x) {
                const int s = j % kSpmvStages;
                if (j >= kSpmvStages) mbar_wait(&empty[s], ((j / kSpmvStages) - 1) & 1);
                const int64_t r0 = t * A.R;
                const int64_t r1 = min(r0 + A.R, A.n_rows);
                const int64_t ck0 = k0, ck1 = k1;
                // prefetch the next tile's bounds (overlaps this tile's copies)
                const int64_t tn = t + gridDim.x;
                if (tn < A.n_tiles) {
                    const int64_t q0 = tn * A.R;
                    const int64_t q1 = min(q0 + A.R, A.n_rows);
                    k0 = __ldg(A.off + q0);
                    k1 = __ldg(A.off + q1);
                }
                const int64_t kv0 = ck0 & ~int64_t(1), kv1 = (ck1 + 1) & ~int64_t(1);
                const int64_t kc0 = ck0 & ~int64_t(3), kc1 = (ck1 + 3) & ~int64_t(3);
                const bool last   = r1 >= A.n_rows;
                const bool direct = last || (kv1 - kv0) > kSpmvCapNnz || (kc1 - kc0) > kSpmvCapNnz;
                meta[s].kv0    = kv0;
                meta[s].kc0    = kc0;
                meta[s].direct = direct ? 1 : 0;
                if (direct) {
                    mbar_arrive(&full[s]);
                } else {
                    unsigned char* st = stage0 + (size_t)s * sbytes;
                    const uint32_t ob = (uint32_t)((A.R + 2) * 8);
                    const uint32_t vb = (uint32_t)((kv1 - kv0) * 8);
                    const uint32_t cb = (uint32_t)((kc1 - kc0) * 4);
                    mbar_arrive_expect_tx(&full[s], ob + vb + cb);
                    bulk_g2s(st, A.off + r0, ob, &full[s], pol);
                    if (vb) bulk_g2s(st + obytes, A.vals + kv0, vb, &full[s], pol);
                    if (cb) bulk_g2s(st + obytes + SpmvLayout::val_bytes(), A.cols + kc0, cb,
                                     &full[s], pol);
                }
            }
        }
        return; // producer warp does not take part in the consumer reduction
    }

    // ===================== consumer warps =====================
    const int ctid = tid - 32;
    double    acc  = 0.0;
    int64_t   t    = blockIdx.x;
    for (int j = 0; t < A.n_tiles; ++j, t += gridDim.x) {
        const int s = j % kSpmvStages;
        mbar_wait(&full[s], (j / kSpmvStages) & 1);
        const int64_t r0   = t * A.R;
        const int     rows = (int)min((int64_t)A.R, A.n_rows - r0);
        if (meta[s].direct) {
            acc = spmv_rows<kSpmvRowGroup, int64_t>(op, acc, ctid, rows, r0, A.off + r0, 0,
                                                    A.cols, A.vals);
        } else {
            unsigned char* st  = stage0 + (size_t)s * sbytes;
            const int64_t  kv0 = meta[s].kv0;
            // columns were copied from kc0 <= kv0: shift so both share kv0-local indices
            const int32_t* cs = reinterpret_cast<const int32_t*>(st + obytes + SpmvLayout::val_bytes()) +
                                (kv0 - meta[s].kc0);
            acc = spmv_rows<kSpmvRowGroup, int>(op, acc, ctid, rows, r0,
                                                reinterpret_cast<const int64_t*>(st), kv0, cs,
                                                reinterpret_cast<const double*>(st + obytes));
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
    int64_t ncols;
    __device__ __forceinline__ bool    init() { return true; }
    __device__ __forceinline__ int64_t n_src() const { return ncols; }
    struct Fetch {
        double x;
    };
    __device__ __forceinline__ Fetch  fetch(int32_t j) const { return Fetch{__ldg(x + j)}; }
    __device__ __forceinline__ double value(const Fetch& f) const { return f.x; }
    __device__ __forceinline__ double row(int64_t i, double sum, double acc, double, bool) const
    {
        y[i] = sum;
        return acc;
    }
    __device__ __forceinline__ void tail(double) const {}
};

// Rows per tile for a matrix whose longest row has `max_row_len` entries:
// the largest multiple of 32 (<= kSpmvMaxRows) whose worst-case 16-B-rounded
// slab fits one stage.  Rows longer than a stage still work (direct tiles).
inline int spmv_rows_per_tile(int64_t max_row_len)
{
    if (max_row_len < 1) max_row_len = 1;
    int64_t r = (kSpmvCapNnz - 8) / max_row_len;
    r         = (r / 32) * 32;
    if (r < 32) r = 32;
    if (r > kSpmvMaxRows) r = kSpmvMaxRows;
    return (int)r;
}

inline SpmvArgs make_spmv_args(const rvk_csr& A, int R)
{
    SpmvArgs a;
    a.n_rows  = A.n_rows;
    a.R       = R;
    a.n_tiles = (A.n_rows + R - 1) / R;
    a.off     = A.row_offsets;
    a.cols    = A.col_indices;
    a.vals    = A.values;
    return a;
}

template <class Op>
rvk_status launch_spmv(cudaStream_t stream, const SpmvArgs& a, const Op& op, TailArgs tail,
                       int grid)
{
    const size_t smem = SpmvLayout::smem_bytes(kSpmvMaxRows);
    static bool  configured = false; // per instantiation
    if (!configured) {
        RVK_CUDA(cudaFuncSetAttribute(k_spmv_tma<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        configured = true;
    }
    k_spmv_tma<Op><<<grid, kSpmvThreads, SpmvLayout::smem_bytes(a.R), stream>>>(a, op, tail);
    RVK_CHECK_LAUNCH("k_spmv_tma");
    return RVK_OK;
}

} // namespace rvk
