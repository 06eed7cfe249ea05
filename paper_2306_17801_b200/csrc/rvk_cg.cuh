// rvk_cg.cuh -- pieces shared by the single-GPU (rvk_cg.cu) and the
// row-sharded (rvk_dcg.cu) Jacobi-CG.
#pragma once

#include "rvk_common.cuh"

namespace rvk {

// Device-resident solver scalars (the reference's Managed a, b, beta,
// betaold, dp of PAPER.md:108-109) plus the exit state.
struct CgState {
    double beta, betaold, alpha, pAp, dp0, dp;
    int    done, state, iterations, breakdown_iter;
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

} // namespace rvk
