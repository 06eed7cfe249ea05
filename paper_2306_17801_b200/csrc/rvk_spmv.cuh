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
//  * stencil-structured matrices (a highest diagonal band col - row, found at
//    plan time): the producer also issues an L2 bulk prefetch of the NEXT
//    tile's leading-edge columns -- the gathers' only first-touch DRAM misses;
//  * tiles that do not fit a stage (very long rows) and the last tile (whose
//    16-byte-rounded bulk range could run past the arrays) are "direct":
//    consumers read them from global memory thread-per-row;
//  * Op supplies SRC(j) (split into raw fetch + arithmetic so every gather is
//    issued before any is consumed), the per-row epilogue and the reduction
//    tail, so the same mainloop serves mat_mult and the fused CG kernel
//    (p = z + b p on the fly; w = A p; p.w partials; alpha tail).
#pragma once

#include "rvk_common.cuh"

#include <atomic>
#include <cassert>
#include <type_traits>

namespace rvk {

constexpr int    kSpmvConsumerWarps = 16;
constexpr int    kSpmvConsumers     = kSpmvConsumerWarps * 32;
constexpr int    kSpmvThreads       = kSpmvConsumers + 32; // + producer warp
constexpr int    kSpmvMaxStages     = 4;
constexpr int    kSpmvUnroll        = 8;                   // default nonzeros per lane per batch
#ifndef SPMV_FULL_FAST
#define SPMV_FULL_FAST 1                                   // warp-uniform unmasked full batches
#endif
constexpr size_t kSpmvHeaderBytes   = 2048;                // barriers, meta, reduction scratch
#ifndef RVK_SPMV_BIG_TILE_ROWS
#define RVK_SPMV_BIG_TILE_ROWS (32ll * 1024 * 1024)
#endif
constexpr int64_t kSpmvBigTileRows  = RVK_SPMV_BIG_TILE_ROWS;  // make_spmv_args: 1024-row tiles above
constexpr int64_t kSpmvPrefetchMaxLead = 128 * 1024;         // ... leading-band L2 prefetch up to
constexpr size_t kSpmvStageBudget   = 200 * 1024;          // dynamic smem for the ring
constexpr size_t kSpmvMarchSmemMax  = 227 * 1024;          // sm_100 opt-in shared memory per block
constexpr size_t kSpmvMarchSmem     = 223 * 1024;          // k_spmv_march: cache + ring (4 KB for op statics)

struct SpmvStageMeta {
    int64_t kv0;    // first value index held in the stage (16-B aligned)
    int64_t kc0;    // first column index held in the stage (16-B aligned)
    int     direct; // 1: read this tile from global memory
    int     pad;
};
static_assert(kSpmvMaxStages * sizeof(SpmvStageMeta) <= 512 - 128, "meta must fit the header");

// Plan-time structure of a stencil-like CSR: the highest diagonal band
// [lead_lo, lead_hi] of (col - row) -- the columns a tile touches FIRST in a
// row-ordered sweep, L2-prefetched one tile ahead (csr_bands).
struct SpmvBands {
    bool    has_lead = false;
    int64_t lead_lo = 0, lead_hi = 0;
    int64_t plane_q = 0; // > 0: diagonals +-Q bound two plane bands (3D stencil), Q % 32 == 0
};

struct SpmvArgs {
    int64_t        n_rows;
    int64_t        n_cols;
    int64_t        n_tiles;
    int            R;        // rows per tile (multiple of 32)
    int            stages;   // ring depth (<= kSpmvMaxStages)
    int            groups;   // consumer groups working on distinct stages (divides stages)
    int            consumers; // consumer threads (multiple of 32, <= kSpmvConsumers)
    int            unroll;    // nonzeros per lane per gather batch: 7, 8 or 9
    int            one_batch; // 1: every row fits one batch (max row length <= unroll)
    int            cap;      // nonzeros per stage
    int            off_bytes, val_bytes, col_bytes, stage_bytes; // [off | vals | cols]
    int            pf;                    // 1: L2-prefetch the next tile's leading-edge columns
    int64_t        pf_lo, pf_hi;          // ... the band [pf_lo, pf_hi] of (col - row)
    const int64_t* off;
    const int32_t* cols;
    const double*  vals;
    int64_t        small_rows; // > 0: systems up to this many rows use k_spmv_small (plan's choice)
    int            csr_keep;   // 1: the CSR stream keeps normal L2 priority (it fits the L2 with
                               //    the vectors and is re-read every iteration)

    size_t smem_bytes() const { return kSpmvHeaderBytes + (size_t)stages * stage_bytes; }
};

// Shared reduction workspace used by Ops with a tail.
struct TailArgs {
    double*       partials;
    unsigned int* ticket;
};

__host__ __device__ inline int align16(int64_t b) { return (int)((b + 15) & ~int64_t(15)); }

// Tile geometry: the largest R (power of two, <= 1024) whose worst-case slab
// (CSR rows of max_row_len) fits a stage with >= 3 stages in the ring (else
// 2).  Rows too long for any stage still work (direct tiles).  B: the
// leading diagonal band to L2-prefetch (null: none).
inline SpmvArgs make_spmv_args(const rvk_csr& A, int64_t max_row_len, const SpmvBands* B = nullptr,
                               int64_t stage_budget = (int64_t)kSpmvStageBudget)
{
    if (max_row_len < 1) max_row_len = 1;
    SpmvArgs a{};
    a.n_rows = A.n_rows;
    a.n_cols = A.n_cols;
    a.off    = A.row_offsets;
    a.cols   = A.col_indices;
    a.vals   = A.values;
    auto fit = [&](int R, int min_stages) {
        const int64_t cap = ((R * max_row_len + 8) + 3) & ~int64_t(3);
        // cb: + 48 B so a batch may read up to U - 1 + 3 columns past the
        // stage's last one (spmv_rows_staged loads every slot unmasked; the
        // values of a batch overrun into the column region)
        const int64_t ob = align16((int64_t)(R + 2) * 8), vb = cap * 8, cb = align16(cap * 4 + 48);
        const int64_t sb = ob + vb + cb;
        const int64_t st = std::min<int64_t>(kSpmvMaxStages, stage_budget / sb);
        if (st < min_stages) return false;
        a.R = R;
        a.stages = (int)st;
        a.cap = (int)cap;
        a.off_bytes = (int)ob;
        a.val_bytes = (int)vb;
        a.col_bytes = (int)cb;
        a.stage_bytes = (int)sb;
        return true;
    };
    bool ok = false;
    // large systems (> 32 M rows, i.e. 3D planes past the leading-band
    // prefetch's reach): 1024-row tiles in a 2-stage ring where they fit
    // (5- / 7-point rows).  Measured, 7-point K1 without the prefetch:
    // 384^3 1057 -> 1030 us, 512^3 2537 -> 2470 us, 768^3 8868 -> 8554 us;
    // 256-row tiles were slower (scripts/experiments/README.md)
    if (A.n_rows > kSpmvBigTileRows) ok = fit(1024, 2);
    for (int need = 3; need >= 2 && !ok; --need)
        for (int R = 1024; R >= 32 && !ok; R /= 2) ok = fit(R, need);
    if (!ok) { // rows longer than a stage: every tile direct, small ring
        a.R = 32;
        a.stages = 4;
        a.off_bytes = align16(34 * 8);
        a.cap = (int)(((kSpmvStageBudget / 4 - a.off_bytes - 64) / 12) & ~size_t(3));
        a.val_bytes = a.cap * 8;
        a.col_bytes = align16((int64_t)a.cap * 4 + 48);
        a.stage_bytes = a.off_bytes + a.val_bytes + a.col_bytes;
    }
    // (the ring must fit the dynamic shared memory launch_spmv configures)
    assert(a.smem_bytes() <= kSpmvHeaderBytes + kSpmvStageBudget);
    a.n_tiles = (A.n_rows + a.R - 1) / a.R;
    // the leading-edge L2 prefetch pays while the +plane band is near
    // (2D grids, 3D planes <= 128 K rows: 256^3 7-point K1 318.9 -> 316.5 us,
    // 27-point 960.8 -> 930.4 us); for larger planes it costs DRAM bandwidth
    // (7-point K1 without it: 384^3 1074 -> 1062 us, 512^3 2735 -> 2541 us,
    // 768^3 9554 -> 8566 us; scripts/experiments/README.md)
    a.pf = (B && B->has_lead && B->lead_lo > 0 && B->lead_lo <= kSpmvPrefetchMaxLead) ? 1 : 0;
    a.pf_lo   = a.pf ? B->lead_lo : 0;
    a.pf_hi   = a.pf ? B->lead_hi : 0;
    // enough groups that every consumer thread owns a row of some tile
    a.consumers = kSpmvConsumers;
    a.groups    = 1;
    while (a.groups * 2 <= a.stages && a.stages % (a.groups * 2) == 0 &&
           a.R * a.groups * 2 <= a.consumers)
        a.groups *= 2;
    // gather batch size: one batch per 7- / 9-point row (and 3 per 27-point
    // row) instead of batches of 8 with masked-off slots
    a.unroll = 8;
    if (max_row_len <= 7) a.unroll = 7;
    else if (max_row_len == 9 || max_row_len % 9 == 0) a.unroll = 9;
    a.one_batch = max_row_len <= a.unroll ? 1 : 0;
    return a;
}

// Epilogue operands of row i, loaded before the row's gathers so their
// latency hides under the products: Op::own(i) when the op declares an `Own`
// type (row-owned vectors the epilogue reads), else the op's gathered
// operands at its own column.
template <class Op, class = void>
struct spmv_has_own : std::false_type {};
template <class Op>
struct spmv_has_own<Op, std::void_t<typename Op::Own>> : std::true_type {};

template <class Op, class G>
__device__ __forceinline__ auto spmv_own(const Op& op, int64_t i, const G& gather)
{
    if constexpr (spmv_has_own<Op>::value) return op.own(i);
    else return gather(op.own_col(i));
}

// ---------------------------------------------------------------------------
// Direct tiles: thread-per-row straight from global memory (rare path).
// ---------------------------------------------------------------------------
template <int U, class Op, class Acc>
__device__ __forceinline__ Acc spmv_rows_direct(const Op& op, Acc acc, int gtid, int gsize,
                                                   int rows, int64_t r0,
                                                   const int64_t* __restrict__ O,
                                                   const int32_t* __restrict__ Cc,
                                                   const double* __restrict__ V)
{
    for (int lr = gtid; lr < rows; lr += gsize) {
        const auto    own = spmv_own(op, r0 + lr, [&](int64_t c) { return op.fetch((int32_t)c); });
        const int64_t kb = (int64_t)O[lr], ke = (int64_t)O[lr + 1];
        double        sum = 0.0;
        for (int64_t k = kb; k < ke; k += U) {
            int32_t c[U];
            double  v[U];
            bool    ok[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                ok[u]            = k + u < ke;
                const int64_t ks = ok[u] ? k + u : ke - 1;
                c[u]             = __ldg(Cc + ks);
                v[u]             = __ldg(V + ks);
            }
            typename Op::Fetch f[U];
#pragma unroll
            for (int u = 0; u < U; ++u) f[u] = op.fetch(c[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double t = add(sum, mul(v[u], op.value(f[u])));
                sum            = ok[u] ? t : sum;
            }
        }
        acc = op.row(r0 + lr, sum, acc, own);
    }
    return acc;
}

// ---------------------------------------------------------------------------
// Staged tiles: lane-per-row out of the shared-memory stage.
//   O  : the tile's row offsets in shared memory (global nnz indices)
//   V  : stage values, V[k - kv0];  Cc : stage columns, Cc[k - kv0]
// Stage-local 32-bit indices keep the address arithmetic cheap.
// ---------------------------------------------------------------------------
template <int U, class Op, class Acc>
__device__ __forceinline__ Acc spmv_rows_staged(const Op& op, Acc acc, int gtid, int gsize,
                                                   int rows, int64_t r0, const int64_t* O,
                                                   int64_t kv0, const int32_t* Cc, const double* V)
{
    auto gather = [&](int64_t c) { return op.fetch((int32_t)c); };
    for (int lr = gtid; lr < rows; lr += gsize) {
        const auto own = spmv_own(op, r0 + lr, gather); // epilogue operands, in flight early
        const int  kb  = (int)((int64_t)O[lr] - kv0);
        const int  ke  = (int)((int64_t)O[lr + 1] - kv0);
        double     sum = 0.0;
        for (int k = kb; k < ke; k += U) {
            int32_t c[U];
            double  v[U];
            typename Op::Fetch f[U];
            // warp-uniform fast path: every active lane has a full batch
            // (interior stencil rows when U matches the row length) -- no
            // per-slot masking selects.  Measured: 9-batches (9/27-point)
            // K1 387 -> 377 / 1018 -> 939 us; the 7-batch (7-point) kernel
            // got SLOWER (318 -> 332 us), so only U == 9 takes it.
            if (SPMV_FULL_FAST && U == 9 && __all_sync(__activemask(), k + U <= ke)) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    c[u] = Cc[k + u];
                    v[u] = V[k + u];
                }
#pragma unroll
                for (int u = 0; u < U; ++u) f[u] = gather(c[u]);
#pragma unroll
                for (int u = 0; u < U; ++u) sum = add(sum, mul(v[u], op.value(f[u])));
                continue;
            }
            // every slot is loaded from a fixed offset of one stage address
            // (no per-slot address registers: a re-used LDS address register
            // stalls the next address computation until the queued LDS has
            // read it -- measured 7% on the 7-point K1); slots past the row's
            // end gather the row's first column instead and are not summed
            bool ok[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                c[u] = Cc[k + u];
                v[u] = V[k + u];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                ok[u] = k + u < ke;
                c[u]  = ok[u] ? c[u] : c[0]; // k < ke: c[0] is a valid column
            }
#pragma unroll
            for (int u = 0; u < U; ++u) f[u] = gather(c[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double t = add(sum, mul(v[u], op.value(f[u])));
                sum            = ok[u] ? t : sum;
            }
        }
        acc = op.row(r0 + lr, sum, acc, own);
    }
    return acc;
}

// Staged tiles, software-pipelined over the thread's stream of (row, batch)
// steps: the NEXT step's columns are read from the stage while the current
// step's gathers are in flight, so every gather address is ready when a step
// starts and all U x nsrc gathers issue back to back.  (Measured on B200: a
// column read consumed right before its gather stalls the issue of the
// remaining gathers behind the LSU queue -- 7-point K1 319 -> 344 us.)  Per
// row the sum is the same left-to-right chain over its batches as the
// reference's loop (bit-identical).  Slots past the row's end gather column
// 0 (always valid) and are not summed; stage reads past the end stay inside
// the stage's 48-byte column slack.
template <int U, class Op, class Acc>
__device__ __forceinline__ Acc spmv_rows_pipe(const Op& op, Acc acc, int gtid, int gsize,
                                                 int rows, int64_t r0, const int64_t* O,
                                                 int64_t kv0, const int32_t* Cc, const double* V)
{
    auto gather = [&](int64_t c) { return op.fetch((int32_t)c); };
    if (gtid >= rows) return acc;
    int     lr = gtid;
    int     k  = (int)((int64_t)O[lr] - kv0), ke = (int)((int64_t)O[lr + 1] - kv0);
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = k + u < ke ? Cc[k + u] : 0;
    auto   own = spmv_own(op, r0 + lr, gather); // epilogue operands, in flight early
    double sum = 0.0;
    while (true) {
        typename Op::Fetch f[U];
#pragma unroll
        for (int u = 0; u < U; ++u) f[u] = gather(c[u]);
        // the next step: this row's next batch, or the thread's next row
        const bool row_done = k + U >= ke;
        const int  ln       = row_done ? lr + gsize : lr;
        const bool more     = ln < rows;
        int        kn = k + U, ken = ke;
        if (row_done && more) {
            kn  = (int)((int64_t)O[ln] - kv0);
            ken = (int)((int64_t)O[ln + 1] - kv0);
        }
        if (more) {
#pragma unroll
            for (int u = 0; u < U; ++u) c[u] = kn + u < ken ? Cc[kn + u] : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double t = add(sum, mul(V[k + u], op.value(f[u])));
            sum            = k + u < ke ? t : sum;
        }
        if (row_done) {
            acc = op.row(r0 + lr, sum, acc, own);
            if (!more) break;
            own = spmv_own(op, r0 + ln, gather);
            sum = 0.0;
        }
        lr = ln;
        k  = kn;
        ke = ken;
    }
    return acc;
}

// Number of fused reductions an op accumulates (Op::kSums, default 1): the
// row() accumulator is a double, or SumVec<N> for N > 1, and tail() receives
// the folded sums (double, or const double (&)[N]).
template <int N>
struct SumVec {
    double v[N];
};
template <class Op, class = void>
struct spmv_sums {
    static constexpr int value = 1;
};
template <class Op>
struct spmv_sums<Op, std::void_t<decltype(Op::kSums)>> {
    static constexpr int value = Op::kSums;
};
// Op::kSysFence: the op stores into peer GPUs' memory (PEER backend).
template <class Op, class = void>
struct spmv_sys_fence : std::false_type {};
template <class Op>
struct spmv_sys_fence<Op, std::void_t<decltype(Op::kSysFence)>>
    : std::integral_constant<bool, Op::kSysFence> {};
// Op::kNoSmall: the op is never launched on a small_rows plan (row-sharded
// and TFQMR plans), so k_spmv_small is not instantiated for it.
template <class Op, class = void>
struct spmv_no_small : std::false_type {};
template <class Op>
struct spmv_no_small<Op, std::void_t<decltype(Op::kNoSmall)>> : std::integral_constant<bool, Op::kNoSmall> {};
template <class Op>
using spmv_acc_t = std::conditional_t<spmv_sums<Op>::value == 1, double, SumVec<spmv_sums<Op>::value>>;

// U: nonzeros per lane per gather batch (SpmvArgs::unroll).
template <class Op, int U = kSpmvUnroll>
__global__ void __launch_bounds__(kSpmvThreads, 1) k_spmv_tma(SpmvArgs A, Op op_in, TailArgs tail)
{
    const int64_t* __restrict__ OFF = A.off;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t*      full   = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t*      empty  = full + kSpmvMaxStages;
    SpmvStageMeta* meta   = reinterpret_cast<SpmvStageMeta*>(smem_raw + 128);
    double*        red    = reinterpret_cast<double*>(smem_raw + 512); // 32 doubles per sum (<= 4)
    int*           flag   = reinterpret_cast<int*>(smem_raw + 512 + 1024);
    unsigned char* stage0 = smem_raw + kSpmvHeaderBytes;

    Op op = op_in;
    if (!op.init()) return; // device-side early exit (converged / breakdown)

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < A.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (A.consumers / 32) / A.groups);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (tid < 32) {
        // ===================== producer warp =====================
        if (tid == 0) {
            // CSR: read once per launch -- evict first, unless the whole
            // matrix stays L2-resident across the solve's launches
            const uint64_t pol_stream = A.csr_keep ? policy_evict_normal() : policy_evict_first();
            int64_t        v   = blockIdx.x;
            int64_t        k0 = 0, k1 = 0; // slab bounds, prefetched one tile ahead
            if (v < A.n_tiles) {
                const int64_t t = v;
                k0 = (int64_t)__ldg(OFF + t * A.R);
                k1 = (int64_t)__ldg(OFF + min(t * A.R + A.R, A.n_rows));
            }
            // stage / phase counters kept incrementally: a run-time division
            // per tile costs more than the tile's address arithmetic
            int s = 0, ph = 0;
            for (int j = 0; v < A.n_tiles; ++j, v += gridDim.x) {
                if (j >= A.stages) mbar_wait(&empty[s], ph ^ 1);
                const int64_t t  = v;
                const int64_t r0 = t * A.R;
                const int64_t r1 = min(r0 + A.R, A.n_rows);
                const int64_t ck0 = k0, ck1 = k1;
                const int64_t tn  = v + gridDim.x; // this CTA's next tile
                if (tn < A.n_tiles) {
                    k0 = (int64_t)__ldg(OFF + tn * A.R);
                    k1 = (int64_t)__ldg(OFF + min(tn * A.R + A.R, A.n_rows));
                }
                const int64_t kv0 = ck0 & ~int64_t(1), kv1 = (ck1 + 1) & ~int64_t(1);
                const int64_t kc0 = ck0 & ~int64_t(3), kc1 = (ck1 + 3) & ~int64_t(3);
                const bool    last   = r1 >= A.n_rows;
                const bool    direct = last || (kv1 - kv0) > A.cap || (kc1 - kc0) > A.cap;
                SpmvStageMeta& m     = meta[s];
                m.kv0                = kv0;
                m.kc0                = kc0;
                m.direct             = direct ? 1 : 0;
                const int cur        = s;
                if (++s == A.stages) {
                    s  = 0;
                    ph ^= 1;
                }
                if (direct) {
                    mbar_arrive(&full[cur]);
                    continue;
                }
                unsigned char* st = stage0 + (size_t)cur * A.stage_bytes;
                // R+2 offsets (a 16-B multiple; the last tile is direct)
                const uint32_t ob = (uint32_t)((A.R + 2) * 8);
                const uint32_t vb = (uint32_t)((kv1 - kv0) * 8);
                const uint32_t cb = (uint32_t)((kc1 - kc0) * 4);
                mbar_arrive_expect_tx(&full[cur], ob + vb + cb);
                bulk_g2s(st, OFF + r0, ob, &full[cur], pol_stream);
                if (vb) bulk_g2s(st + A.off_bytes, A.vals + kv0, vb, &full[cur], pol_stream);
                if (cb) bulk_g2s(st + A.off_bytes + A.val_bytes, A.cols + kc0, cb, &full[cur], pol_stream);
                // leading edge of this CTA's NEXT tile: its highest-diagonal
                // columns are first-touch DRAM misses for the gathers; start
                // them now (L2 prefetch, no smem, no barrier)
                if (A.pf && tn < A.n_tiles) {
                    const int64_t q0 = tn * A.R, q1 = min(q0 + A.R, A.n_rows);
                    int64_t       lo = max(q0 + A.pf_lo, (int64_t)0) & ~int64_t(1);
                    int64_t       hi = min(q1 + A.pf_hi, A.n_cols) & ~int64_t(1);
                    if (hi > lo) {
                        const int nps = op.num_src();
                        for (int k = 0; k < nps; ++k)
                            bulk_prefetch_l2(op.src_ptr(k) + lo, (uint32_t)(hi - lo) * 8);
                    }
                }
            }
        }
        return; // the producer warp takes no part in the consumer reduction
    }

    // ===================== consumer warps =====================
    // NG groups of GS threads; group q takes the tiles j with j % NG == q
    // (NG divides the ring depth, so a group always owns the same stages).
    const int ctid  = tid - 32;
    const int gs    = A.consumers / A.groups;
    const int group = ctid / gs, gtid = ctid % gs;
    constexpr int NS = spmv_sums<Op>::value;
    static_assert(NS >= 1 && NS <= 4, "at most 4 fused reductions");
    spmv_acc_t<Op> acc{};
    int64_t   v     = blockIdx.x + (int64_t)group * gridDim.x;
    int       s     = group, ph = 0; // stage / phase, advanced by the group count (it divides the ring)
    for (; v < A.n_tiles; v += (int64_t)A.groups * gridDim.x) {
        mbar_wait(&full[s], ph);
        const SpmvStageMeta& m = meta[s];
        const int64_t t    = v;
        const int64_t r0   = t * A.R;
        const int     rows = (int)min((int64_t)A.R, A.n_rows - r0);
        if (m.direct) {
            acc = spmv_rows_direct<U>(op, acc, gtid, gs, rows, r0, OFF + r0, A.cols, A.vals);
        } else {
            unsigned char* st  = stage0 + (size_t)s * A.stage_bytes;
            const int64_t  kv0 = m.kv0;
            // columns were copied from kc0 <= kv0: shift so both use kv0-local indices
            const int32_t* Cc = reinterpret_cast<const int32_t*>(st + A.off_bytes + A.val_bytes) +
                                (kv0 - m.kc0);
            const int64_t* O = reinterpret_cast<const int64_t*>(st);
            const double*  V = reinterpret_cast<const double*>(st + A.off_bytes);
            acc = spmv_rows_pipe<U>(op, acc, gtid, gs, rows, r0, O, kv0, Cc, V);
        }
        __syncwarp();
        if ((ctid & 31) == 0) mbar_arrive(&empty[s]);
        if ((s += A.groups) >= A.stages) {
            s -= A.stages;
            ph ^= 1;
        }
    }

    if constexpr (Op::kHasTail) {
        double v[NS];
        if constexpr (NS == 1) v[0] = acc;
        else {
#pragma unroll
            for (int j = 0; j < NS; ++j) v[j] = acc.v[j];
        }
        block_sum<NS>(v, red, ctid, A.consumers, 1);
        if (ctid == 0) {
#pragma unroll
            for (int j = 0; j < NS; ++j) tail.partials[(size_t)blockIdx.x * NS + j] = v[j];
        }
        if (!last_block<spmv_sys_fence<Op>::value>(tail.ticket, ctid, flag, A.consumers, 1)) return;
        fold_partials<NS>(tail.partials, gridDim.x, v, red, ctid, A.consumers, 1);
        if (ctid == 0) {
            if constexpr (NS == 1) op.tail(v[0]);
            else op.tail(v);
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
    __device__ __forceinline__ bool          init() { return true; }
    __device__ __forceinline__ int           num_src() const { return 1; }
    __device__ __forceinline__ const double* src_ptr(int) const { return x; }
    __device__ __forceinline__ Fetch         fetch(int32_t j) const { return Fetch{__ldg(x + j)}; }
    __device__ __forceinline__ double  value(const Fetch& f) const { return f.x; }
    __device__ __forceinline__ int64_t own_col(int64_t) const { return 0; } // unused by row()
    __device__ __forceinline__ double  row(int64_t i, double sum, double acc, const Fetch&) const
    {
        y[i] = sum;
        return acc;
    }
    __device__ __forceinline__ void tail(double) const {}
};

// Plain SpMV that is a no-op once a device flag is set (the early-exit of
// the op-per-kernel solver sequences).
struct SpmvGuardedOp : SpmvPlainOp {
    const int* guard;
    __device__ __forceinline__ bool init() { return *guard == 0; }
};

// Small systems: no TMA ring, no warp specialisation -- plain blocks of
// kSpmvSmallThreads, one row per thread through the same per-row code as the
// TMA kernel's direct tiles (identical row sums), then the same block-sum /
// last-block tail.  A 544-thread warp-specialised CTA per SM with its
// mbarrier ring is pure ramp-up latency when the whole operand set is a few
// MB in L2 (SpmvArgs::small_rows).
constexpr int kSpmvSmallThreads = 256;
template <class Op, int U>
__global__ void __launch_bounds__(kSpmvSmallThreads) k_spmv_small(SpmvArgs A, Op op_in, TailArgs tail)
{
    __shared__ double red[32 * 4];
    __shared__ int    flag;
    Op op = op_in;
    if (!op.init()) return;
    constexpr int NS = spmv_sums<Op>::value;
    spmv_acc_t<Op> acc{};
    const int64_t r0   = (int64_t)blockIdx.x * kSpmvSmallThreads;
    const int     rows = (int)min((int64_t)kSpmvSmallThreads, A.n_rows - r0);
    acc = spmv_rows_direct<U>(op, acc, (int)threadIdx.x, kSpmvSmallThreads, rows, r0, A.off + r0, A.cols,
                              A.vals);
    if constexpr (Op::kHasTail) {
        const int tid = threadIdx.x;
        double    v[NS];
        if constexpr (NS == 1) v[0] = acc;
        else {
#pragma unroll
            for (int j = 0; j < NS; ++j) v[j] = acc.v[j];
        }
        block_sum<NS>(v, red, tid, kSpmvSmallThreads, 1);
        if (tid == 0) {
#pragma unroll
            for (int j = 0; j < NS; ++j) tail.partials[(size_t)blockIdx.x * NS + j] = v[j];
        }
        if (!last_block<spmv_sys_fence<Op>::value>(tail.ticket, tid, &flag, kSpmvSmallThreads, 1)) return;
        fold_partials<NS>(tail.partials, gridDim.x, v, red, tid, kSpmvSmallThreads, 1);
        if (tid == 0) {
            if constexpr (NS == 1) op.tail(v[0]);
            else op.tail(v);
            *tail.ticket = 0u;
        }
    }
}

template <class Op>
rvk_status launch_spmv(cudaStream_t stream, const SpmvArgs& a, const Op& op, TailArgs tail,
                       int grid)
{
    // (the tail's partial slots: the plans reserve 2 x kMaxReduceBlocks doubles)
    if constexpr (!spmv_no_small<Op>::value)
    if (a.small_rows && a.n_rows <= a.small_rows &&
        ((a.n_rows + kSpmvSmallThreads - 1) / kSpmvSmallThreads) * spmv_sums<Op>::value <=
            2 * (int64_t)kMaxReduceBlocks) {
        const int g = (int)((a.n_rows + kSpmvSmallThreads - 1) / kSpmvSmallThreads);
        if (a.unroll == 7) k_spmv_small<Op, 7><<<g, kSpmvSmallThreads, 0, stream>>>(a, op, tail);
        else if (a.unroll == 9) k_spmv_small<Op, 9><<<g, kSpmvSmallThreads, 0, stream>>>(a, op, tail);
        else k_spmv_small<Op, 8><<<g, kSpmvSmallThreads, 0, stream>>>(a, op, tail);
        RVK_CHECK_LAUNCH("k_spmv_small");
        return RVK_OK;
    }
    // > 48 KB of dynamic shared memory is a per-device function attribute:
    // set once per instantiation and device (idempotent, so a race between
    // two host threads only repeats it)
    static std::atomic<uint64_t> configured{0};
    if (device_first_use(configured)) {
        const int smax = (int)(kSpmvHeaderBytes + kSpmvStageBudget);
        RVK_CUDA(cudaFuncSetAttribute(k_spmv_tma<Op, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
        RVK_CUDA(cudaFuncSetAttribute(k_spmv_tma<Op, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
        RVK_CUDA(cudaFuncSetAttribute(k_spmv_tma<Op, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
        device_mark_done(configured);
    }
    const int    th = 32 + a.consumers;
    const size_t sm = a.smem_bytes();
    if (a.unroll == 7) k_spmv_tma<Op, 7><<<grid, th, sm, stream>>>(a, op, tail);
    else if (a.unroll == 9) k_spmv_tma<Op, 9><<<grid, th, sm, stream>>>(a, op, tail);
    else k_spmv_tma<Op, 8><<<grid, th, sm, stream>>>(a, op, tail);
    RVK_CHECK_LAUNCH("k_spmv_tma");
    return RVK_OK;
}

// Stencil structure of a CSR (plan time, one host sync): the highest band of
// diagonals (col - row), for the leading-edge L2 prefetch.  has_lead = false
// when the matrix is not stencil-like (more than 128 diagonals).
// Implemented in rvk_cg.cu.
rvk_status csr_bands(cudaStream_t s, const rvk_csr& A, SpmvBands* out);

} // namespace rvk
