// rvk_spmv_march.cuh -- plane-marching CSR SpMV for large 3D stencil grids.
//
// Same row sums as k_spmv_tma (kernels_scalar.cpp:53-63 order, each product
// rounded before it is added: bit-identical), different tile order and a
// shared-memory cache of the gathered operand.
//
// Why: in row order the grid sweeps z-planes with the whole chip, so a
// gathered value is used three times one plane of streamed bytes apart (as
// the +plane neighbour, as the row's own plane, as the -plane neighbour).
// At 768^3 two planes of streamed CSR (146 MB) exceed the 126 MB L2 and the
// -plane gathers come back from DRAM: +13% traffic (profiles/
// r01_plane_study.md), and every gathered nonzero is an L2 request.
//
// Here CTA g owns the in-plane row range [a_g, a_g + L_g) (Q rows per plane,
// split into 148 contiguous ranges) and marches it through the planes
// k = 0 .. K-1 (tiles of <= R rows of plane k, TMA-staged exactly like
// k_spmv_tma).  The CTA keeps the FORMED gathered value p_j (for the CG K1:
// p = z + b p_old, the same single rounding every gather would compute) of
// its range for planes k-1, k and k+1 in a 3-slot shared-memory ring:
//   * the thread of row i = kQ + a + o loads z/p_old at i + Q (the +plane
//     element at its own offset, a coalesced first-touch DRAM read that the
//     producer L2-prefetched one tile ahead), forms p and stores it in slot
//     (k+1) % 3 -- every slot entry is written by exactly one thread;
//   * a gathered column inside the CTA's range of plane k or k-1 is read from
//     its slot (LDS), the row's own +plane column from the register, anything
//     else (range halos, far columns of a general CSR) from global memory;
//   * one consumer barrier per plane step orders the slot writes of step k
//     before the reads of steps k+1 and k+2.
// Correctness needs no stencil structure (a miss is a global gather); the
// structure only decides the hit rate.  DRAM sees every gathered value once.
#pragma once

#include "rvk_spmv.cuh"

namespace rvk {

struct SpmvMarch {
    int64_t Q;      // rows per plane (a multiple of 32)
    int64_t K;      // planes (ceil(n / Q))
    int     Lmax;   // largest range (rows; multiple of 32)
    int     grid;   // CTAs
    int     stage_bytes; // SpmvArgs::stage_bytes + the staged +plane z / p_old (16 B per row)
    int     passes; // ranges per CTA: the plane is split into grid x passes ranges, CTA g
                    // marches ranges g, g + grid, ... one after the other (a smaller cache
                    // leaves room for a deeper TMA ring)
    size_t  smem_bytes(const SpmvArgs& a) const
    {
        return kSpmvHeaderBytes + (size_t)3 * Lmax * 8 + (size_t)a.stages * stage_bytes;
    }
};

// Range r's in-plane rows: [a, a + L), 32-row aligned.
__host__ __device__ inline void march_range(const SpmvMarch& M, int r, int64_t* a, int* L)
{
    const int64_t q32 = M.Q / 32, nr = (int64_t)M.grid * M.passes;
    const int64_t b0 = q32 * r / nr, b1 = q32 * (r + 1) / nr;
    *a = b0 * 32;
    *L = (int)((b1 - b0) * 32);
}

// Row tile t of plane k for a CTA with range [a, a + L): rows [r0, r1).
__device__ __forceinline__ void march_tile(const SpmvArgs& A, const SpmvMarch& M, int64_t a, int L,
                                           int64_t k, int t, int64_t* r0, int64_t* r1)
{
    const int64_t base = k * M.Q + a;
    *r0                = base + (int64_t)t * A.R;
    *r1                = min(min(*r0 + A.R, base + L), A.n_rows);
    if (*r0 > A.n_rows) *r0 = A.n_rows;
}

// One row of plane k: gathers classified against the slot ring.
//   Ck / Cm : slots of planes k and k-1 (index = column - (kQ + a) [+ Q])
//   Cn      : slot of plane k+1 (this row stores its own +plane value there)
// Row and column indices fit 32 bits (int32 columns), so the classification
// runs in 32-bit arithmetic.  A cache hit is carried in the op's Fetch slot
// (Op::from_formed / Op::formed) so hits and misses share registers: the
// LDS of a hit and the LDG of a miss are predicated alternatives.
//   cs      : column of row 0 (0; a row-sharded plan's local columns start
//             after the lower halo plane)
//   zq / pq : this row's +plane z / p_old, TMA-staged with the tile (null:
//             the tile has none staged -- fetch from global memory if the
//             +plane exists)
template <int U, class Op, class Acc, class ColF, class ValF>
__device__ __forceinline__ Acc march_row(const Op& op, Acc acc, int i, int base, int L, int Q,
                                         int ncols, int cs, const double* Ck, const double* Cm,
                                         double* Cn, const double* zq, const double* pqr, int kb,
                                         int ke, ColF col, ValF val)
{
    const int  o     = i - base; // offset in the range, 0 <= o < L
    const bool has_q = i + cs < ncols - Q;
    base += cs;                  // from here on: column space
    // the row's own +plane value: formed once from the staged raw operands,
    // cached for steps k+1 (own plane) and k+2 (-plane)
    double pq = 0.0;
    if (has_q) {
        pq    = zq ? op.value(Op::raw(zq[0], pqr[0])) : op.value(op.fetch(base + o + Q));
        Cn[o] = pq;
    }
    double sum = 0.0;
    for (int k = kb; k < ke; k += U) {
        typename Op::Fetch f[U];
        unsigned           miss = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c   = k + u < ke ? col(k + u) : base + o; // past the row's end: a harmless slot
            const int rel = c - base;
            if ((unsigned)rel < (unsigned)L) f[u] = Op::from_formed(Ck[rel]);
            else if ((unsigned)(rel + Q) < (unsigned)L) f[u] = Op::from_formed(Cm[rel + Q]);
            else if (rel - Q == o) f[u] = Op::from_formed(pq);
            else {
                f[u] = op.fetch(c);
                miss |= 1u << u;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double v = (miss >> u) & 1u ? op.value(f[u]) : Op::formed(f[u]);
            // slots past the row's end re-read the batch's first value (in
            // bounds for the direct path's global arrays) and are not summed
            const double t = add(sum, mul(val(k + u < ke ? k + u : k), v));
            sum            = k + u < ke ? t : sum;
        }
    }
    return op.row_p(i, sum, acc, Ck[o]);
}

template <class Op, int U>
__global__ void __launch_bounds__(kSpmvThreads, 1)
    k_spmv_march(SpmvArgs A, SpmvMarch M, Op op_in, TailArgs tail)
{
    const int64_t* __restrict__ OFF = A.off;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t*      full   = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t*      empty  = full + kSpmvMaxStages;
    SpmvStageMeta* meta   = reinterpret_cast<SpmvStageMeta*>(smem_raw + 128);
    double*        red    = reinterpret_cast<double*>(smem_raw + 512);
    int*           flag   = reinterpret_cast<int*>(smem_raw + 512 + 1024);
    double*        cache  = reinterpret_cast<double*>(smem_raw + kSpmvHeaderBytes);
    unsigned char* stage0 = smem_raw + kSpmvHeaderBytes + (size_t)3 * M.Lmax * 8;

    Op op = op_in;
    if (!op.init()) return;

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
            const uint64_t pol_stream = policy_evict_first();
            const uint64_t pol_keep   = policy_evict_normal();
            int            j          = 0;
            int            s = 0, ph = 0; // ring slot / phase of tile j (no per-tile division)
            for (int pass = 0; pass < M.passes; ++pass) {
            int64_t a;
            int     L;
            march_range(M, blockIdx.x + pass * M.grid, &a, &L);
            const int T = (L + A.R - 1) / A.R; // tiles per plane step
            for (int64_t k = 0; k < M.K; ++k) {
                for (int t = 0; t < T; ++t, ++j) {
                    if (j >= A.stages) mbar_wait(&empty[s], ph ^ 1);
                    int64_t r0, r1;
                    march_tile(A, M, a, L, k, t, &r0, &r1);
                    SpmvStageMeta& m = meta[s];
                    // offsets of R + 2 rows (16-B multiple) must stay inside
                    // off[0..n]; the matrix's last tile is direct (rounded
                    // value / column ranges could pass nnz)
                    const bool direct = r1 >= A.n_rows || r0 + A.R + 2 > A.n_rows + 1;
                    int64_t    ck0 = 0, ck1 = 0;
                    if (!direct) {
                        ck0 = (int64_t)__ldg(OFF + r0);
                        ck1 = (int64_t)__ldg(OFF + r1);
                    }
                    const int64_t kv0 = ck0 & ~int64_t(1), kv1 = (ck1 + 1) & ~int64_t(1);
                    const int64_t kc0 = ck0 & ~int64_t(3), kc1 = (ck1 + 3) & ~int64_t(3);
                    const bool    dir = direct || (kv1 - kv0) > A.cap || (kc1 - kc0) > A.cap;
                    m.kv0             = kv0;
                    m.kc0             = kc0;
                    m.direct          = dir ? 1 : 0;
                    // +plane segment of the tile (z, p_old at rows + cs + Q):
                    // contiguous, so TMA-staged with the CSR -- the rows' only
                    // first-touch gathers leave the consumers' critical path
                    const int64_t cs   = op.own_col(0);
                    const bool    plus = !dir && r1 + cs + M.Q <= A.n_cols && op.num_src() == 2;
                    m.pad              = plus ? 1 : 0;
                    if (dir) {
                        mbar_arrive(&full[s]);
                    } else {
                        unsigned char* st = stage0 + (size_t)s * M.stage_bytes;
                        const uint32_t ob = (uint32_t)((A.R + 2) * 8);
                        const uint32_t vb = (uint32_t)((kv1 - kv0) * 8);
                        const uint32_t cb = (uint32_t)((kc1 - kc0) * 4);
                        const uint32_t qb = plus ? (uint32_t)((r1 - r0) * 8) : 0u;
                        mbar_arrive_expect_tx(&full[s], ob + vb + cb + 2 * qb);
                        bulk_g2s(st, OFF + r0, ob, &full[s], pol_stream);
                        if (vb) bulk_g2s(st + A.off_bytes, A.vals + kv0, vb, &full[s], pol_stream);
                        if (cb) bulk_g2s(st + A.off_bytes + A.val_bytes, A.cols + kc0, cb, &full[s], pol_stream);
                        if (qb) {
                            unsigned char* q = st + A.stage_bytes;
                            // normal L2 priority: the neighbouring ranges read
                            // these lines again as their halo gathers
                            bulk_g2s(q, op.src_ptr(0) + r0 + cs + M.Q, qb, &full[s], pol_keep);
                            bulk_g2s(q + (size_t)A.R * 8, op.src_ptr(1) + r0 + cs + M.Q, qb, &full[s],
                                     pol_keep);
                        }
                    }
                    if (++s == A.stages) {
                        s  = 0;
                        ph ^= 1;
                    }
                }
            }
            }
        }
        return;
    }

    // ===================== consumer warps =====================
    const int ctid  = tid - 32;
    const int gs    = A.consumers / A.groups;
    const int group = ctid / gs, gtid = ctid % gs;
    constexpr int NS = spmv_sums<Op>::value;
    spmv_acc_t<Op> acc{};

    const int cs = (int)op.own_col(0);
    int       j  = 0;
    int       rs = 0, rph = 0, rg = 0; // ring slot, phase and owning group of tile j
    for (int pass = 0; pass < M.passes; ++pass) {
    int64_t a;
    int     L;
    march_range(M, blockIdx.x + pass * M.grid, &a, &L);
    const int T = (L + A.R - 1) / A.R; // tiles per plane step
    // prologue: plane 0 of the range into slot 0, and the plane below it into
    // slot 2 when the column space has one (a row shard's lower halo plane)
    for (int o = ctid; o < L; o += A.consumers) {
        const int64_t i = a + o;
        if (i < A.n_rows) cache[o] = op.value(op.fetch((int32_t)(i + cs)));
        if (i + cs - M.Q >= 0) cache[(size_t)2 * M.Lmax + o] = op.value(op.fetch((int32_t)(i + cs - M.Q)));
    }
    asm volatile("bar.sync 2, %0;" ::"r"(A.consumers) : "memory");

    for (int64_t k = 0; k < M.K; ++k) {
        const double* Ck   = cache + (size_t)(k % 3) * M.Lmax;
        const double* Cm   = cache + (size_t)((k + 2) % 3) * M.Lmax;
        double*       Cn   = cache + (size_t)((k + 1) % 3) * M.Lmax;
        const int64_t base = k * M.Q + a;
        for (int t = 0; t < T; ++t, ++j) {
            const int s = rs, mine = rg == group;
            const int phs = rph;
            if (++rs == A.stages) {
                rs  = 0;
                rph ^= 1;
            }
            if (++rg == A.groups) rg = 0;
            if (!mine) continue;
            mbar_wait(&full[s], phs);
            int64_t r0, r1;
            march_tile(A, M, a, L, k, t, &r0, &r1);
            const int            rows = (int)(r1 - r0);
            const SpmvStageMeta& m    = meta[s];
            if (m.direct) {
                const int32_t* __restrict__ Cg = A.cols;
                const double* __restrict__ Vg  = A.vals;
                for (int lr = gtid; lr < rows; lr += gs) {
                    const int64_t kb = OFF[r0 + lr], ke = OFF[r0 + lr + 1];
                    acc = march_row<U>(op, acc, (int)(r0 + lr), (int)base, L, (int)M.Q, (int)A.n_cols, cs,
                                       Ck, Cm, Cn, nullptr, nullptr, 0, (int)(ke - kb),
                                       [&](int q) { return __ldg(Cg + kb + q); },
                                       [&](int q) { return __ldg(Vg + kb + q); });
                }
            } else {
                unsigned char* st  = stage0 + (size_t)s * M.stage_bytes;
                const int64_t  kv0 = m.kv0;
                const double*  Zq  = m.pad ? reinterpret_cast<const double*>(st + A.stage_bytes) : nullptr;
                const double*  Pq  = Zq ? Zq + A.R : nullptr;
                const int32_t* Cc  = reinterpret_cast<const int32_t*>(st + A.off_bytes + A.val_bytes) +
                                    (kv0 - m.kc0);
                const int64_t* O   = reinterpret_cast<const int64_t*>(st);
                const double*  V   = reinterpret_cast<const double*>(st + A.off_bytes);
                for (int lr = gtid; lr < rows; lr += gs) {
                    const int kb = (int)(O[lr] - kv0), ke = (int)(O[lr + 1] - kv0);
                    acc = march_row<U>(op, acc, (int)(r0 + lr), (int)base, L, (int)M.Q, (int)A.n_cols, cs,
                                       Ck, Cm, Cn, Zq ? Zq + lr : nullptr, Pq ? Pq + lr : nullptr,
                                       kb, ke, [&](int q) { return Cc[q]; },
                                       [&](int q) { return V[q]; });
                }
            }
            __syncwarp();
            if ((ctid & 31) == 0) mbar_arrive(&empty[s]);
        }
        // slot (k+1) complete before step k+1 reads it; slot (k-1) free
        asm volatile("bar.sync 2, %0;" ::"r"(A.consumers) : "memory");
    }
    } // pass

    if constexpr (Op::kHasTail) {
        double v[NS];
        if constexpr (NS == 1) v[0] = acc;
        else {
#pragma unroll
            for (int q = 0; q < NS; ++q) v[q] = acc.v[q];
        }
        block_sum<NS>(v, red, ctid, A.consumers, 1);
        if (ctid == 0) {
#pragma unroll
            for (int q = 0; q < NS; ++q) tail.partials[(size_t)blockIdx.x * NS + q] = v[q];
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

// Plan-time geometry: Q = the plane stride (from the CSR's diagonals), one
// range per SM.  Returns false when the matrix has no plane structure or the
// cache + a ring of >= 2 stages does not fit the shared memory.
bool make_spmv_march(const rvk_csr& A, int64_t max_row_len, int64_t Q, int grid, SpmvArgs* a,
                     SpmvMarch* M);

template <class Op>
rvk_status launch_spmv_march(cudaStream_t stream, const SpmvArgs& a, const SpmvMarch& M,
                             const Op& op, TailArgs tail)
{
    static std::atomic<uint64_t> configured{0};
    if (device_first_use(configured)) {
        // dynamic + static shared memory <= the opt-in maximum (an op may
        // bring static shared memory of its own)
        auto set = [](auto fn) -> rvk_status {
            cudaFuncAttributes fa{};
            RVK_CUDA(cudaFuncGetAttributes(&fa, fn));
            const int smax = (int)(kSpmvMarchSmemMax - fa.sharedSizeBytes);
            RVK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
            return RVK_OK;
        };
        if (rvk_status st = set(k_spmv_march<Op, 7>); st != RVK_OK) return st;
        if (rvk_status st = set(k_spmv_march<Op, 8>); st != RVK_OK) return st;
        if (rvk_status st = set(k_spmv_march<Op, 9>); st != RVK_OK) return st;
        device_mark_done(configured);
    }
    const int    th = 32 + a.consumers;
    const size_t sm = M.smem_bytes(a);
    if (a.unroll == 7) k_spmv_march<Op, 7><<<M.grid, th, sm, stream>>>(a, M, op, tail);
    else if (a.unroll == 9) k_spmv_march<Op, 9><<<M.grid, th, sm, stream>>>(a, M, op, tail);
    else k_spmv_march<Op, 8><<<M.grid, th, sm, stream>>>(a, M, op, tail);
    RVK_CHECK_LAUNCH("k_spmv_march");
    return RVK_OK;
}

} // namespace rvk
