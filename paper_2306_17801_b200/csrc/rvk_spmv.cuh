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
//  * stencil-structured matrices (few distinct diagonals col - row, found at
//    plan time) also get the tile's x-windows -- the contiguous ranges of the
//    gathered vectors the tile's diagonals touch -- bulk-copied into the
//    stage, so every gather is a conflict-free LDS instead of an L1/L2 round
//    trip (other columns still fall back to a global load);
//  * tiles that do not fit a stage (very long rows) and the last tile (whose
//    16-byte-rounded bulk range could run past the arrays) are "direct":
//    consumers read them from global memory thread-per-row;
//  * Op supplies SRC(j) (split into raw fetch + arithmetic so every gather is
//    issued before any is consumed), the per-row epilogue and the reduction
//    tail, so the same mainloop serves mat_mult and the fused CG kernel
//    (p = z + b p on the fly; w = A p; p.w partials; alpha tail).
#pragma once

#include "rvk_common.cuh"

#include <cstdlib>
#include <cstring>
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
constexpr int    kSpmvMaxWin        = 4;                   // x-windows per tile
constexpr int    kSpmvMaxSrc        = 2;                   // gathered vectors per column
constexpr size_t kSpmvHeaderBytes   = 2048;                // barriers, meta, reduction scratch
constexpr size_t kSpmvStageBudget   = 200 * 1024;          // dynamic smem for the ring

struct SpmvStageMeta {
    int64_t kv0;    // first value index held in the stage (16-B aligned)
    int64_t kc0;    // first column index held in the stage (16-B aligned)
    int     direct; // 1: read this tile from global memory
    int     pad;
    int64_t wlo[kSpmvMaxWin]; // global column range [wlo, whi) held by window w
    int64_t whi[kSpmvMaxWin];
};
static_assert(kSpmvMaxStages * sizeof(SpmvStageMeta) <= 512 - 128, "meta must fit the header");

// Plan-time structure of a stencil-like CSR: every nonzero's (col - row)
// falls in one of n diagonal bands [lo_w, hi_w].  Only used with gathered
// sources the plan allocated itself, 16-B aligned and padded by >= 2 doubles.
struct SpmvWindows {
    int     n = 0;
    int64_t lo[kSpmvMaxWin] = {0, 0, 0, 0};
    int64_t hi[kSpmvMaxWin] = {0, 0, 0, 0};
    // highest diagonal band [lead_lo, lead_hi] (any band count): the columns a
    // tile touches FIRST in a row-ordered sweep -- prefetched into L2 one tile ahead
    bool    has_lead = false;
    int64_t lead_lo = 0, lead_hi = 0;
    // lowest diagonal band: (lead centre - trail centre) / 2 = the plane
    // stride of a symmetric stencil, in any (shifted, halo-extended) column space
    int64_t trail_lo = 0, trail_hi = 0;
};

struct SpmvArgs {
    int64_t        n_rows;
    int64_t        n_cols;
    int64_t        n_tiles;
    int            R;        // rows per tile (multiple of 32)
    int            stages;   // ring depth (<= kSpmvMaxStages)
    int            groups;   // consumer groups working on distinct stages (divides stages)
    int            consumers; // consumer threads (multiple of 32, <= kSpmvConsumers)
    int            unroll;    // nonzeros per lane per gather batch: 7, 8 or 9 (spmv_unroll)
    int            cap;      // nonzeros per stage
    int            off_bytes, val_bytes, col_bytes, stage_bytes; // [off | vals | cols | windows]
    int            nwin;                  // 0: no x-windows
    int64_t        win_lo[kSpmvMaxWin];   // diagonal bands (col - row)
    int64_t        win_hi[kSpmvMaxWin];
    int            win_base[kSpmvMaxWin]; // element offset of window w inside one source's area
    int            win_elems;             // doubles per source per stage
    int            pf;                    // 1: L2-prefetch the next tile's leading-edge columns
    int64_t        pf_lo, pf_hi;          // ... the band [pf_lo, pf_hi] of (col - row)
    // tile ORDER (spmv_set_order): ord_tc == 0 = row order; else 2.5D
    // blocking -- each plane (ord_tp tiles) is cut into chunks of ord_tc
    // consecutive tiles, and the grid sweeps chunk 0 through all ord_np
    // planes, then chunk 1, ...  The frontier stays one contiguous chunk of
    // one plane, and the +-plane gathers are reused from L2 one CHUNK later
    // instead of one plane later
    int64_t        ord_tp, ord_tc, ord_np;
    const int64_t* off;
    const int32_t* cols;
    const double*  vals;
    // plan-owned int32 copy of the row offsets (nnz < 2^31; padded by >= 4
    // entries) or null: the mainloop then streams 4 instead of 8 B per row
    const int32_t* off32;
    int64_t        small_rows; // > 0: systems up to this many rows use k_spmv_small (plan's choice)

    size_t smem_bytes() const { return kSpmvHeaderBytes + (size_t)stages * stage_bytes; }
};

// Shared reduction workspace used by Ops with a tail.
struct TailArgs {
    double*       partials;
    unsigned int* ticket;
};

__host__ __device__ inline int align16(int64_t b) { return (int)((b + 15) & ~int64_t(15)); }

// Virtual tile index -> tile (row block) index.
__host__ __device__ __forceinline__ int64_t spmv_tile(const SpmvArgs& a, int64_t v)
{
    if (!a.ord_tc) return v;
    const int64_t per_chunk = a.ord_np * a.ord_tc;
    const int64_t c = v / per_chunk, rem = v - c * per_chunk;
    const int64_t k = rem / a.ord_tc, u = rem - k * a.ord_tc;
    return k * a.ord_tp + c * a.ord_tc + u;
}

// Tile geometry: the largest R (power of two, <= 1024) whose worst-case slab
// (CSR rows of max_row_len, plus nsrc x-windows when W is given) fits a stage
// with >= 3 stages in the ring (else 2).  Rows too long for any stage still
// work (direct tiles).
inline SpmvArgs make_spmv_args(const rvk_csr& A, int64_t max_row_len,
                               const SpmvWindows* W = nullptr, int nsrc = 1)
{
    if (max_row_len < 1) max_row_len = 1;
    SpmvArgs a{};
    a.n_rows = A.n_rows;
    a.n_cols = A.n_cols;
    a.off    = A.row_offsets;
    a.cols   = A.col_indices;
    a.vals   = A.values;
    const int nwin = (W && W->n > 0 && W->n <= kSpmvMaxWin) ? W->n : 0;
    auto fit = [&](int R, int min_stages) {
        const int64_t cap = ((R * max_row_len + 8) + 3) & ~int64_t(3);
        const int64_t ob = align16((int64_t)(R + 2) * 8), vb = cap * 8, cb = align16(cap * 4);
        int64_t we = 0;
        int     base[kSpmvMaxWin] = {0, 0, 0, 0};
        for (int w = 0; w < nwin; ++w) {
            base[w] = (int)we;
            // R + band width + 16-B rounding at both ends, kept 16-B aligned
            we += ((R + (W->hi[w] - W->lo[w]) + 4) + 1) & ~int64_t(1);
        }
        const int64_t sb = ob + vb + cb + (int64_t)nsrc * we * 8;
        const int64_t st = std::min<int64_t>(kSpmvMaxStages, (int64_t)kSpmvStageBudget / sb);
        if (st < min_stages) return false;
        a.R = R;
        a.stages = (int)st;
        a.cap = (int)cap;
        a.off_bytes = (int)ob;
        a.val_bytes = (int)vb;
        a.col_bytes = (int)cb;
        a.stage_bytes = (int)sb;
        a.nwin = nwin;
        a.win_elems = (int)we;
        for (int w = 0; w < kSpmvMaxWin; ++w) {
            a.win_lo[w]   = w < nwin ? W->lo[w] : 0;
            a.win_hi[w]   = w < nwin ? W->hi[w] : 0;
            a.win_base[w] = base[w];
        }
        return true;
    };
    bool ok = false;
    for (int need = 3; need >= 2 && !ok; --need)
        for (int R = 1024; R >= 32 && !ok; R /= 2) ok = fit(R, need);
    if (!ok) { // rows longer than a stage: every tile direct, small ring
        a.R = 32;
        a.stages = 4;
        a.nwin = 0;
        a.off_bytes = align16(34 * 8);
        a.cap = (int)(((kSpmvStageBudget / 4 - a.off_bytes) / 12) & ~size_t(3));
        a.val_bytes = a.cap * 8;
        a.col_bytes = align16((int64_t)a.cap * 4);
        a.stage_bytes = a.off_bytes + a.val_bytes + a.col_bytes;
    }
    a.n_tiles = (A.n_rows + a.R - 1) / a.R;
    a.pf      = (W && W->has_lead && W->lead_lo > 0) ? 1 : 0;
    a.pf_lo   = a.pf ? W->lead_lo : 0;
    a.pf_hi   = a.pf ? W->lead_hi : 0;
    // enough groups that every consumer thread owns a row of some tile
    auto set_groups = [&] {
        a.groups = 1;
        while (a.groups * 2 <= a.stages && a.stages % (a.groups * 2) == 0 &&
               a.R * a.groups * 2 <= a.consumers)
            a.groups *= 2;
    };
    a.consumers = kSpmvConsumers;
    set_groups();
    // gather batch size: one batch per 7- / 9-point row (and 3 per 27-point
    // row) instead of batches of 8 with masked-off slots (RVK_SPMV_UNROLL=8
    // restores the fixed batch)
    const char* un = std::getenv("RVK_SPMV_UNROLL");
    a.unroll = 8;
    if (!(un && un[0] == '8')) {
        if (max_row_len <= 7) a.unroll = 7;
        else if (max_row_len == 9 || max_row_len % 9 == 0) a.unroll = 9;
    }
    // Long rows (short tiles): every ring stage is consumed at once, so the
    // producer has no stage to fill ahead.  Opt-in (RVK_SPMV_SLACK=1): halve
    // the consumer warps so half the ring is always in flight.  Measured
    // slower on B200 (27-point 256^3 K1 1288 vs 1066 us): the gathers need
    // the thread-level parallelism more than the TMA needs the slack.
    const char* slack = std::getenv("RVK_SPMV_SLACK");
    if (ok && a.groups == a.stages && a.stages >= 2 && slack && slack[0] == '1') {
        a.consumers = kSpmvConsumers / 2;
        set_groups();
    }
    return a;
}

// Tile order policy (plan time).  Row order is the default: it keeps the
// chip-wide frontier one contiguous window.  Opt-in (RVK_CHUNK_MB=<budget>):
// when two planes of streamed bytes (CSR + vectors) exceed the budget, the
// planes are cut into the fewest chunks that bring two CHUNKS under it
// (>= RVK_CHUNK_MIN_TILES tiles per chunk, default one per SM).  Measured on
// B200 at 768^3 (profiles/r01_summary.md): chunking removes the -plane
// re-reads (K1 DRAM reads 55.3 -> 49.8 GB vs 48.9 algorithmic) but the DRAM
// throughput drops more (5.29 -> 4.51 TB/s), and a pure pencil sweep (one
// tile per plane) is slower still -- so it stays off by default.  The plane
// is half the distance between the centres of the highest and lowest
// diagonal bands (7/5-point: exactly nx*ny / nx; 27/9-point: the bands
// around them; also in a shard's halo-extended column space).
// RVK_TILE_ORDER=row forces row order.
inline void spmv_set_order(SpmvArgs& a, const SpmvWindows& W, int64_t nnz, int nsrc, int sms)
{
    a.ord_tp = a.ord_tc = a.ord_np = 0;
    const char* env = std::getenv("RVK_TILE_ORDER");
    if (env && std::strcmp(env, "row") == 0) return;
    if (!W.has_lead || W.lead_lo <= 0 || a.n_rows <= 0) return;
    const int64_t plane = ((W.lead_lo + W.lead_hi) - (W.trail_lo + W.trail_hi)) / 4;
    if (plane < a.R || plane % a.R) return;
    const int64_t tp = plane / a.R;
    if (a.n_tiles % tp || a.n_tiles / tp < 3) return;
    const char*  mb        = std::getenv("RVK_CHUNK_MB");
    if (!mb) return;
    const double budget    = std::atof(mb) * 1024 * 1024;
    const double row_bytes = 12.0 * (double)nnz / (double)a.n_rows + 8.0 + 16.0 * (nsrc + 1);
    if (2.0 * (double)plane * row_bytes <= budget) return; // row order already reuses
    const char*   mt     = std::getenv("RVK_CHUNK_MIN_TILES"); // tests: chunk small grids
    const int64_t min_tc = mt ? std::atoll(mt) : sms;
    // fewest chunks under the budget; if none, the smallest chunk allowed
    int64_t best = 0;
    for (int64_t cp = 2; cp <= tp; ++cp) {
        if (tp % cp) continue;
        const int64_t tc = tp / cp;
        if (tc < min_tc) break;
        best = tc;
        if (2.0 * (double)(tc * a.R) * row_bytes <= budget) break;
    }
    if (best) {
        a.ord_tp = tp;
        a.ord_tc = best;
        a.ord_np = a.n_tiles / tp;
    }
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
template <int U, class Op, class Acc, class OffT>
__device__ __forceinline__ Acc spmv_rows_direct(const Op& op, Acc acc, int gtid, int gsize,
                                                   int rows, int64_t r0,
                                                   const OffT* __restrict__ O,
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

// x-windows of one stage: window w holds global columns [lo[w], hi[w]) of
// every gathered source at element base[w] of that source's area.
struct StageWindows {
    int           n;
    int64_t       lo[kSpmvMaxWin], hi[kSpmvMaxWin];
    int           base[kSpmvMaxWin];
    const double* s0; // window area of source 0 / 1
    const double* s1;
};

// Branch-free window lookup.  Every column of a staged tile lies in some
// window by construction (the bands come from a scan of all nonzeros and the
// loaded ranges are rounded outward into padded buffers), so no fallback.
__device__ __forceinline__ int window_index(const StageWindows& W, int64_t c)
{
    int idx = 0;
#pragma unroll
    for (int w = 0; w < kSpmvMaxWin; ++w) {
        const bool in = w < W.n && c >= W.lo[w] && c < W.hi[w];
        idx           = in ? W.base[w] + (int)(c - W.lo[w]) : idx;
    }
    return idx;
}

// ---------------------------------------------------------------------------
// Staged tiles: lane-per-row out of the shared-memory stage.
//   O  : the tile's row offsets in shared memory (global nnz indices)
//   V  : stage values, V[k - kv0];  Cc : stage columns, Cc[k - kv0]
// Stage-local 32-bit indices keep the address arithmetic cheap.  WIN: the
// gathers read the stage's x-windows (LDS) instead of global memory.
// ---------------------------------------------------------------------------
template <bool WIN, int U, class Op, class Acc, class OffT>
__device__ __forceinline__ Acc spmv_rows_staged(const Op& op, Acc acc, int gtid, int gsize,
                                                   int rows, int64_t r0, const OffT* O,
                                                   int64_t kv0, const int32_t* Cc,
                                                   const double* V, const StageWindows& W)
{
    auto gather = [&](int64_t c) {
        if constexpr (WIN) return op.fetch_smem(W.s0, W.s1, window_index(W, c));
        else return op.fetch((int32_t)c);
    };
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
            bool ok[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                ok[u]        = k + u < ke;
                const int ks = ok[u] ? k + u : k; // k < ke: a valid entry
                c[u]         = Cc[ks];
                v[u]         = V[ks];
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
template <class Op>
using spmv_acc_t = std::conditional_t<spmv_sums<Op>::value == 1, double, SumVec<spmv_sums<Op>::value>>;

template <class OffT>
__device__ __forceinline__ const OffT* spmv_offsets(const SpmvArgs& A)
{
    if constexpr (sizeof(OffT) == 4) return A.off32;
    else return A.off;
}

// OffT: int64_t (the matrix's own offsets) or int32_t (SpmvArgs::off32).
// U: nonzeros per lane per gather batch (SpmvArgs::unroll).
template <class Op, class OffT = int64_t, int U = kSpmvUnroll>
__global__ void __launch_bounds__(kSpmvThreads, 1) k_spmv_tma(SpmvArgs A, Op op_in, TailArgs tail)
{
    const OffT* __restrict__ OFF = spmv_offsets<OffT>(A);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t*      full   = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t*      empty  = full + kSpmvMaxStages;
    SpmvStageMeta* meta   = reinterpret_cast<SpmvStageMeta*>(smem_raw + 128);
    double*        red    = reinterpret_cast<double*>(smem_raw + 512); // 32 doubles per sum (<= 4)
    int*           flag   = reinterpret_cast<int*>(smem_raw + 512 + 1024);
    unsigned char* stage0 = smem_raw + kSpmvHeaderBytes;

    pdl_trigger(); // the successor may start launching (it waits for our completion)
    pdl_wait();    // our predecessor's writes are visible from here on
    Op op = op_in;
    if (!op.init()) return; // device-side early exit (converged / breakdown)

    const int tid  = threadIdx.x;
    const int nsrc = A.nwin ? op.num_src() : 0;
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
            const uint64_t pol_stream = policy_evict_first(); // CSR: read once
            const uint64_t pol_keep   = policy_evict_last();  // x-windows: reused by 3 tiles
            int64_t        v   = blockIdx.x;
            int64_t        k0 = 0, k1 = 0; // slab bounds, prefetched one tile ahead
            if (v < A.n_tiles) {
                const int64_t t = spmv_tile(A, v);
                k0 = (int64_t)__ldg(OFF + t * A.R);
                k1 = (int64_t)__ldg(OFF + min(t * A.R + A.R, A.n_rows));
            }
            for (int j = 0; v < A.n_tiles; ++j, v += gridDim.x) {
                const int s = j % A.stages;
                if (j >= A.stages) mbar_wait(&empty[s], ((j / A.stages) - 1) & 1);
                const int64_t t  = spmv_tile(A, v);
                const int64_t r0 = t * A.R;
                const int64_t r1 = min(r0 + A.R, A.n_rows);
                const int64_t ck0 = k0, ck1 = k1;
                const int64_t vn  = v + gridDim.x;
                const int64_t tn  = vn < A.n_tiles ? spmv_tile(A, vn) : A.n_tiles;
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
                if (direct) {
                    mbar_arrive(&full[s]);
                    continue;
                }
                // x-windows: columns [r0 + lo_w, r1 - 1 + hi_w] clipped to
                // [0, n_cols) and rounded OUTWARD to 16-B boundaries -- the
                // gathered sources are plan-owned buffers padded by >= 2
                // doubles, so the rounded end stays inside the allocation
                uint32_t wbytes = 0;
                for (int w = 0; w < A.nwin; ++w) {
                    int64_t lo = r0 + A.win_lo[w], hi = r1 + A.win_hi[w]; // exclusive hi
                    lo = max(lo, (int64_t)0);
                    hi = min(hi, A.n_cols);
                    lo = lo & ~int64_t(1);
                    hi = (hi + 1) & ~int64_t(1);
                    if (hi < lo) hi = lo;
                    m.wlo[w] = lo;
                    m.whi[w] = hi;
                    wbytes += (uint32_t)(hi - lo) * 8;
                }
                unsigned char* st = stage0 + (size_t)s * A.stage_bytes;
                // R+2 offsets (R+4 for int32: 16-B multiple; off32 is padded)
                const uint32_t ob = sizeof(OffT) == 8 ? (uint32_t)((A.R + 2) * 8) : (uint32_t)((A.R + 4) * 4);
                const uint32_t vb = (uint32_t)((kv1 - kv0) * 8);
                const uint32_t cb = (uint32_t)((kc1 - kc0) * 4);
                mbar_arrive_expect_tx(&full[s], ob + vb + cb + wbytes * nsrc);
                bulk_g2s(st, OFF + r0, ob, &full[s], pol_stream);
                if (vb) bulk_g2s(st + A.off_bytes, A.vals + kv0, vb, &full[s], pol_stream);
                if (cb) bulk_g2s(st + A.off_bytes + A.val_bytes, A.cols + kc0, cb, &full[s], pol_stream);
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
                double* win0 = reinterpret_cast<double*>(st + A.off_bytes + A.val_bytes + A.col_bytes);
                for (int k = 0; k < nsrc; ++k) {
                    const double* src = op.src_ptr(k);
                    double*       dst = win0 + (size_t)k * A.win_elems;
                    for (int w = 0; w < A.nwin; ++w) {
                        const uint32_t b = (uint32_t)(m.whi[w] - m.wlo[w]) * 8;
                        if (b) bulk_g2s(dst + A.win_base[w], src + m.wlo[w], b, &full[s], pol_keep);
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
    for (int j = group; v < A.n_tiles; j += A.groups, v += (int64_t)A.groups * gridDim.x) {
        const int s = j % A.stages;
        const int64_t t = spmv_tile(A, v);
        mbar_wait(&full[s], (j / A.stages) & 1);
        const int64_t r0   = t * A.R;
        const int     rows = (int)min((int64_t)A.R, A.n_rows - r0);
        const SpmvStageMeta& m = meta[s];
        if (m.direct) {
            acc = spmv_rows_direct<U>(op, acc, gtid, gs, rows, r0, OFF + r0, A.cols, A.vals);
        } else {
            unsigned char* st  = stage0 + (size_t)s * A.stage_bytes;
            const int64_t  kv0 = m.kv0;
            // columns were copied from kc0 <= kv0: shift so both use kv0-local indices
            const int32_t* Cc = reinterpret_cast<const int32_t*>(st + A.off_bytes + A.val_bytes) +
                                (kv0 - m.kc0);
            StageWindows W;
            W.n = nsrc ? A.nwin : 0;
            const double* win0 =
                reinterpret_cast<const double*>(st + A.off_bytes + A.val_bytes + A.col_bytes);
            W.s0 = win0;
            W.s1 = win0 + A.win_elems;
#pragma unroll
            for (int w = 0; w < kSpmvMaxWin; ++w) {
                W.lo[w]   = m.wlo[w];
                W.hi[w]   = m.whi[w];
                W.base[w] = A.win_base[w];
            }
            const OffT* O = reinterpret_cast<const OffT*>(st);
            const double*  V = reinterpret_cast<const double*>(st + A.off_bytes);
            if (W.n) acc = spmv_rows_staged<true, U>(op, acc, gtid, gs, rows, r0, O, kv0, Cc, V, W);
            else acc = spmv_rows_staged<false, U>(op, acc, gtid, gs, rows, r0, O, kv0, Cc, V, W);
        }
        __syncwarp();
        if ((ctid & 31) == 0) mbar_arrive(&empty[s]);
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
    __device__ __forceinline__ Fetch fetch_smem(const double* s0, const double*, int i) const
    {
        return Fetch{s0[i]};
    }
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
    pdl_trigger();
    pdl_wait();
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
    if (a.small_rows && a.n_rows <= a.small_rows && !a.off32 &&
        ((a.n_rows + kSpmvSmallThreads - 1) / kSpmvSmallThreads) * spmv_sums<Op>::value <=
            2 * (int64_t)kMaxReduceBlocks) {
        const int g = (int)((a.n_rows + kSpmvSmallThreads - 1) / kSpmvSmallThreads);
        cudaError_t e;
        if (a.unroll == 7) e = launch_pdl(k_spmv_small<Op, 7>, g, kSpmvSmallThreads, 0, stream, a, op, tail);
        else if (a.unroll == 9) e = launch_pdl(k_spmv_small<Op, 9>, g, kSpmvSmallThreads, 0, stream, a, op, tail);
        else e = launch_pdl(k_spmv_small<Op, 8>, g, kSpmvSmallThreads, 0, stream, a, op, tail);
        if (e != cudaSuccess) return cuda_error(e, "k_spmv_small launch");
        RVK_CHECK_LAUNCH("k_spmv_small");
        return RVK_OK;
    }
    static bool configured = false; // per instantiation; before any graph capture
    const int   smax       = (int)(kSpmvHeaderBytes + kSpmvStageBudget);
    if (!configured) {
        RVK_CUDA(cudaFuncSetAttribute(k_spmv_tma<Op, int64_t, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
        RVK_CUDA(cudaFuncSetAttribute(k_spmv_tma<Op, int64_t, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
        RVK_CUDA(cudaFuncSetAttribute(k_spmv_tma<Op, int64_t, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
        RVK_CUDA(cudaFuncSetAttribute(k_spmv_tma<Op, int32_t, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
        configured = true;
    }
    const int th = 32 + a.consumers;
    const size_t sm = a.smem_bytes();
    cudaError_t e;
    if (a.off32) e = launch_pdl(k_spmv_tma<Op, int32_t, 8>, grid, th, sm, stream, a, op, tail);
    else if (a.unroll == 7) e = launch_pdl(k_spmv_tma<Op, int64_t, 7>, grid, th, sm, stream, a, op, tail);
    else if (a.unroll == 9) e = launch_pdl(k_spmv_tma<Op, int64_t, 9>, grid, th, sm, stream, a, op, tail);
    else e = launch_pdl(k_spmv_tma<Op, int64_t, 8>, grid, th, sm, stream, a, op, tail);
    if (e != cudaSuccess) return cuda_error(e, "k_spmv_tma launch");
    RVK_CHECK_LAUNCH("k_spmv_tma");
    return RVK_OK;
}

// Stencil structure of a CSR (plan time, one host sync): the distinct
// diagonals (col - row), clustered into at most kSpmvMaxWin bands.  n = 0
// when the matrix is not stencil-like (more than 64 diagonals, or bands that
// would not fit).  Implemented in rvk_cg.cu.
rvk_status csr_windows(cudaStream_t s, const rvk_csr& A, SpmvWindows* out);

} // namespace rvk
