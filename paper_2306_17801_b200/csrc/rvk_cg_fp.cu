// rvk_cg_fp.cu -- the fused 2-phase Jacobi-CG iteration as ONE persistent
// cooperative launch that keeps k_spmv_tma's TMA ring alive across the
// whole solve (RVK_PLAN_FPERSIST).
//
// For systems past the one-launch grid solves (rvk_cg_small.cu, <= ~606 K
// rows) and small enough that per-launch ramp / tail latency, not HBM,
// bounds the fused graph (1 M rows: K1 23 us with 62 MB from DRAM, K2 11 us
// with 8 MB -- DESIGN.md section 9), each iteration runs in one kernel:
//
//   K1 phase   the consumer warps run the same lane-per-row mainloop as
//              k_spmv_tma (spmv_rows_pipe / spmv_rows_direct) over this
//              CTA's tiles: p = z + b p_old per gathered column, w = A p,
//              p and w stored, p.w partial;
//   barrier    consumer thread 0 publishes the block partial, releases a
//              monotonic arrival counter and spins on it (ld.acquire.gpu);
//              every CTA folds the partials in the same fixed order (same
//              code as the grid solve), so all hold the same alpha;
//   K2 phase   the same rows (each consumer thread owns the rows it just
//              wrote): x += a p, r += (-a) w, z = d r; z.z, z.r partials;
//   barrier    as above -> dp (hist), beta; the exit decision is identical
//              in every CTA.
//
// The producer warp streams the CSR tiles of EVERY iteration back to back
// (the matrix does not change), so the next iteration's first stages are
// already in shared memory while the K2 phase and the barriers run.  After
// an exit (breakdown / convergence) the consumers keep draining the ring
// without computing, so no bulk copy is left in flight at kernel exit.
// Element arithmetic is the reference's (mul-then-add, operand order of
// kernels_scalar.cpp:11-63); only the reduction trees differ from the fused
// graph (hist within 1e-10 of the oracle, tests/test_gpu_fp.py).
#include "rvk_cg.cuh"
#include "rvk_context.hpp"
#include "rvk_internal.hpp"
#include "rvk_spmv.cuh"

namespace rvk {

namespace {

// gathers of vectors other CTAs wrote inside this launch: L2 (coherent)
template <bool FIRST>
struct FpOp {
    const double* z;
    const double* po;
    double*       pn;
    double*       w;
    double        b;
    struct Fetch {
        double z, p;
    };
    __device__ __forceinline__ Fetch fetch(int32_t j) const
    {
        return Fetch{__ldcg(z + j), FIRST ? 0.0 : __ldcg(po + j)};
    }
    __device__ __forceinline__ double  value(const Fetch& f) const { return FIRST ? f.z : aypx1(b, f.z, f.p); }
    __device__ __forceinline__ int64_t own_col(int64_t i) const { return i; }
    __device__ __forceinline__ double  row(int64_t i, double sum, double acc, const Fetch& o) const
    {
        const double p = value(o);
        pn[i]          = p;
        w[i]           = sum;
        return add(acc, mul(p, sum));
    }
};

__device__ __forceinline__ unsigned fp_ld_acquire(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// mbarrier wait with a watchdog: a protocol bug traps (a launch error the
// host reports) instead of hanging the GPU
__device__ __forceinline__ void fp_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t ok = 0;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (spin > (1u << 22)) __trap();
    }
}

constexpr int kFpBar = 1; // named barrier of the 512 consumer threads
constexpr int kFpB   = 4; // update-phase rows per thread per batch

// Block-sum v over the consumers, publish, grid barrier, fold every CTA's
// partials in block order (lane l: blocks l, l+32, ... ascending, then a
// shuffle tree) -- identical in every CTA.
template <int NV>
__device__ __forceinline__ void fp_reduce(double (&v)[NV], double* partials, unsigned* bar, unsigned target,
                                          double* red, double* out_sh, int ctid)
{
    block_sum<NV>(v, red, ctid, kSpmvConsumers, kFpBar);
    if (ctid == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) partials[blockIdx.x * 4 + j] = v[j];
        __threadfence();
        atomicAdd(bar, 1u);
        for (uint32_t spin = 0; fp_ld_acquire(bar) < target; ++spin)
            if (spin > (1u << 24)) __trap();
    }
    asm volatile("bar.sync %0, %1;" ::"r"(kFpBar), "r"(kSpmvConsumers) : "memory");
    if (ctid < 32) {
        constexpr int kPer = (148 + 31) / 32;
        double        pv[kPer][NV];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int blk = ctid + 32 * q;
#pragma unroll
            for (int j = 0; j < NV; ++j) pv[q][j] = blk < (int)gridDim.x ? __ldcg(partials + blk * 4 + j) : 0.0;
        }
        double f[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) f[j] = 0.0;
#pragma unroll
        for (int q = 0; q < kPer; ++q)
            if (ctid + 32 * q < (int)gridDim.x) {
#pragma unroll
                for (int j = 0; j < NV; ++j) f[j] = add(f[j], pv[q][j]);
            }
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            f[j] = warp_sum(f[j]);
            if (ctid == 0) out_sh[j] = f[j];
        }
    }
    asm volatile("bar.sync %0, %1;" ::"r"(kFpBar), "r"(kSpmvConsumers) : "memory");
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = out_sh[j];
    asm volatile("bar.sync %0, %1;" ::"r"(kFpBar), "r"(kSpmvConsumers) : "memory");
}

template <int U>
__global__ void __launch_bounds__(kSpmvThreads, 1) k_cg_fp(SpmvArgs A, FpArgs f)
{
    const int64_t* __restrict__ OFF = A.off;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t*      full   = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t*      empty  = full + kSpmvMaxStages;
    SpmvStageMeta* meta   = reinterpret_cast<SpmvStageMeta*>(smem_raw + 128);
    unsigned char* stage0 = smem_raw + kSpmvHeaderBytes;
    __shared__ double red[128], out_sh[4];

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < A.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], A.consumers / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (tid < 32) {
        // ===================== producer: every iteration's tiles =============
        if (tid == 0) {
            const uint64_t pol = A.csr_keep ? policy_evict_normal() : policy_evict_first();
            int            s = 0, ph = 0, j = 0;
            for (int it = 0; it < f.max_it; ++it) {
                for (int64_t v = blockIdx.x; v < A.n_tiles; v += gridDim.x, ++j) {
                    if (j >= A.stages) fp_wait(&empty[s], ph ^ 1);
                    const int64_t r0 = v * A.R;
                    const int64_t r1 = min(r0 + A.R, A.n_rows);
                    const int64_t k0 = __ldg(OFF + r0), k1 = __ldg(OFF + r1);
                    const int64_t kv0 = k0 & ~int64_t(1), kv1 = (k1 + 1) & ~int64_t(1);
                    const int64_t kc0 = k0 & ~int64_t(3), kc1 = (k1 + 3) & ~int64_t(3);
                    const bool    direct = r1 >= A.n_rows || (kv1 - kv0) > A.cap || (kc1 - kc0) > A.cap;
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
                    const uint32_t ob = (uint32_t)((A.R + 2) * 8);
                    const uint32_t vb = (uint32_t)((kv1 - kv0) * 8);
                    const uint32_t cb = (uint32_t)((kc1 - kc0) * 4);
                    mbar_arrive_expect_tx(&full[cur], ob + vb + cb);
                    bulk_g2s(st, OFF + r0, ob, &full[cur], pol);
                    if (vb) bulk_g2s(st + A.off_bytes, A.vals + kv0, vb, &full[cur], pol);
                    if (cb) bulk_g2s(st + A.off_bytes + A.val_bytes, A.cols + kc0, cb, &full[cur], pol);
                }
            }
        }
        return;
    }

    // ===================== consumers =====================
    const int      ctid = tid - 32;
    const unsigned G    = gridDim.x;
    const double   dc   = f.dconst;
    const int      rpt  = (A.R + A.consumers - 1) / A.consumers; // rows per thread per tile
    auto dval = [&](int64_t i) { return f.dvec ? __ldg(f.dinv + i) : dc; };
    unsigned nbar = 0;

    // ---- setup on this CTA's rows: r = b, z = d b, x = 0; z.z, z.r ---------
    double acc2[2] = {0.0, 0.0};
    for (int64_t v = blockIdx.x; v < A.n_tiles; v += G) {
        const int64_t r0 = v * A.R, r1 = min(r0 + A.R, A.n_rows);
        for (int64_t i = r0 + ctid; i < r1; i += A.consumers) {
            const double bi = f.b[i];
            const double zi = mul(dval(i), bi);
            f.r[i]          = bi;
            f.z[i]          = zi;
            f.x[i]          = 0.0;
            acc2[0]         = add(acc2[0], mul(zi, zi));
            acc2[1]         = add(acc2[1], mul(zi, bi));
        }
    }
    fp_reduce<2>(acc2, f.partials, f.bar, ++nbar * G, red, out_sh, ctid);
    double       beta = acc2[1];
    const double dp0  = sqrt(acc2[0]);
    double       betaold = 0.0, alpha = 0.0, pAp = 0.0, dp = dp0;
    int          state = RVK_CG_RUNNING, iters = 0, bk = -1;
    if (cg_converged(dp0, dp0, f.rtol, f.atol)) state = RVK_CG_CONVERGED;

    int s = 0, ph = 0;
    // one pass over this CTA's stages of an iteration; compute = false drains
    auto k1_phase = [&](auto op, bool compute) {
        double acc = 0.0;
        for (int64_t v = blockIdx.x; v < A.n_tiles; v += G) {
            fp_wait(&full[s], ph);
            if (compute) {
                const SpmvStageMeta& m    = meta[s];
                const int64_t        r0   = v * A.R;
                const int            rows = (int)min((int64_t)A.R, A.n_rows - r0);
                if (m.direct) {
                    acc = spmv_rows_direct<U>(op, acc, ctid, A.consumers, rows, r0, OFF + r0, A.cols, A.vals);
                } else {
                    unsigned char* st  = stage0 + (size_t)s * A.stage_bytes;
                    const int64_t  kv0 = m.kv0;
                    const int32_t* Cc =
                        reinterpret_cast<const int32_t*>(st + A.off_bytes + A.val_bytes) + (kv0 - m.kc0);
                    const int64_t* O = reinterpret_cast<const int64_t*>(st);
                    const double*  V = reinterpret_cast<const double*>(st + A.off_bytes);
                    acc = spmv_rows_pipe<U>(op, acc, ctid, A.consumers, rows, r0, O, kv0, Cc, V);
                }
            }
            __syncwarp();
            if ((ctid & 31) == 0) mbar_arrive(&empty[s]);
            if (++s == A.stages) {
                s  = 0;
                ph ^= 1;
            }
        }
        return acc;
    };

    for (int it = 0; it < f.max_it; ++it) {
        const bool live = state == RVK_CG_RUNNING;
        double     bb   = 0.0;
        if (live && it > 0) {
            if (betaold == 0.0) {
                state = RVK_CG_BREAKDOWN;
                bk    = it;
            } else {
                bb = beta / betaold;
            }
        }
        const bool    run = state == RVK_CG_RUNNING;
        const double* po  = (it & 1) ? f.p1 : f.p0;
        double*       pn  = (it & 1) ? f.p0 : f.p1;
        double        pw  = it == 0 ? k1_phase(FpOp<true>{f.z, po, pn, f.w, bb}, run)
                                    : k1_phase(FpOp<false>{f.z, po, pn, f.w, bb}, run);
        if (!run) continue; // drain the remaining iterations' stages
        double v1[1] = {pw};
        fp_reduce<1>(v1, f.partials, f.bar, ++nbar * G, red, out_sh, ctid);
        pAp             = v1[0];
        const double al = beta / pAp;
        if (pAp == 0.0 || !isfinite(al)) {
            state = RVK_CG_BREAKDOWN;
            bk    = it;
            continue;
        }
        alpha   = al;
        betaold = beta;
        // ---- K2 phase: the rows this thread just wrote p / w for -------------
        // (slots q = tile-major over this CTA's tiles; batches of kFpB rows
        // with every load issued before the first store)
        const double na = -al;
        acc2[0] = acc2[1] = 0.0;
        for (int q0 = 0;; q0 += kFpB) {
            int64_t ii[kFpB];
            double  wv[kFpB], rv[kFpB], pv[kFpB], xv[kFpB], dv[kFpB];
            bool    any = false;
#pragma unroll
            for (int u = 0; u < kFpB; ++u) {
                const int     q  = q0 + u;
                const int64_t v  = blockIdx.x + (int64_t)(q / rpt) * G;
                const int64_t i  = v * A.R + ctid + (int64_t)(q % rpt) * A.consumers;
                const bool    ok = v < A.n_tiles && i < min(v * A.R + A.R, A.n_rows);
                ii[u]            = ok ? i : -1;
                any |= ok;
                wv[u] = ok ? f.w[i] : 0.0;
                rv[u] = ok ? f.r[i] : 0.0;
                pv[u] = ok ? pn[i] : 0.0;
                xv[u] = ok ? f.x[i] : 0.0;
                dv[u] = ok ? dval(i) : 0.0;
            }
            if (!any && blockIdx.x + (int64_t)((q0 + kFpB) / rpt) * G >= A.n_tiles) break;
#pragma unroll
            for (int u = 0; u < kFpB; ++u) {
                if (ii[u] < 0) continue;
                const int64_t i  = ii[u];
                const double  ri = axpy1(na, wv[u], rv[u]);
                const double  zi = mul(dv[u], ri);
                f.x[i]           = axpy1(al, pv[u], xv[u]);
                f.r[i]           = ri;
                f.z[i]           = zi;
                acc2[0]          = add(acc2[0], mul(zi, zi));
                acc2[1]          = add(acc2[1], mul(zi, ri));
            }
        }
        fp_reduce<2>(acc2, f.partials, f.bar, ++nbar * G, red, out_sh, ctid);
        dp    = sqrt(acc2[0]);
        iters = it + 1;
        if (blockIdx.x == 0 && ctid == 0) f.hist[it + 1] = dp;
        if (cg_converged(dp, dp0, f.rtol, f.atol)) state = RVK_CG_CONVERGED;
        beta = acc2[1];
    }
    if (blockIdx.x == 0 && ctid == 0) {
        f.hist[0]            = dp0;
        f.st->dp0            = dp0;
        f.st->dp             = dp;
        f.st->alpha          = alpha;
        f.st->pAp            = pAp;
        f.st->beta           = beta;
        f.st->betaold        = betaold;
        f.st->iterations     = iters;
        f.st->breakdown_iter = bk;
        f.st->state          = state;
        f.st->done           = 1;
    }
}

} // namespace

bool fp_eligible(const SpmvArgs& a) { return a.groups == 1 && a.consumers == kSpmvConsumers; }

rvk_status launch_fp(cudaStream_t s, const SpmvArgs& a, const FpArgs& f)
{
    RVK_CUDA(cudaMemsetAsync(f.bar, 0, sizeof(unsigned), s));
    const int    grid = (int)std::min<int64_t>(sm_count(), a.n_tiles);
    const size_t smem = a.smem_bytes();
    void*        kargs[] = {const_cast<SpmvArgs*>(&a), const_cast<FpArgs*>(&f)};
    auto go = [&](auto fn) -> rvk_status {
        // > 48 KB dynamic shared memory: per device and instantiation (idempotent)
        RVK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(kSpmvHeaderBytes + kSpmvStageBudget)));
        RVK_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kSpmvThreads), kargs, smem, s));
        return RVK_OK;
    };
    if (a.unroll == 7) return go(k_cg_fp<7>);
    if (a.unroll == 9) return go(k_cg_fp<9>);
    return go(k_cg_fp<8>);
}

} // namespace rvk
