// rvk_stencil.cu -- device-side assembly of the benchmark Laplacians
// and the synthetic RHS.
//
// Bit-exact with the CPU builder (oracle/rvk_oracle.c:ro_build_laplacian):
// lexicographic ordering with x fastest, Dirichlet by truncation, columns
// ascending, centre = points-1 and -1 for every neighbour.  The row offset of
// every row has a closed form (the per-row count is separable: box stencils
// count cx*cy*cz, star stencils cx+cy+cz-2 with c = 1 + #in-grid neighbours
// along that axis), so each thread writes its rows independently -- no scan,
// no host round trip, and 768^3 (3.17e9 nnz, int64 offsets) assembles at
// HBM speed instead of ~2 minutes on the host.
#include "rvk_common.cuh"
#include "rvk_context.hpp"

namespace rvk {

namespace {

struct Grid3 {
    int64_t nx, ny, nz;
    int     box; // 1: 9/27-point, 0: 5/7-point
    int     zr;  // 1 in 3D
    double  centre;
};

// number of in-grid positions {k-1,k,k+1} along an axis of length n
__host__ __device__ __forceinline__ int64_t axis_count(int64_t k, int64_t n)
{
    return 1 + (k > 0) + (k < n - 1);
}
// sum_{k' < k} axis_count(k', n)
__host__ __device__ __forceinline__ int64_t axis_prefix(int64_t k, int64_t n)
{
    if (n == 1) return k; // only k in {0, 1}
    if (k <= 0) return 0;
    if (k >= n) return 3 * n - 2;
    return 3 * k - 1;
}

__host__ __device__ __forceinline__ int64_t row_offset(const Grid3& g, int64_t x, int64_t y,
                                                       int64_t z)
{
    const int64_t TX = axis_prefix(g.nx, g.nx), TY = axis_prefix(g.ny, g.ny);
    const int64_t cy = axis_count(y, g.ny), cz = axis_count(z, g.nz);
    if (g.box) {
        return axis_prefix(z, g.nz) * TY * TX + cz * (axis_prefix(y, g.ny) * TX + cy * axis_prefix(x, g.nx));
    }
    // star: count = cx + cy + cz - 2
    const int64_t planes = z * (g.ny * TX + g.nx * TY - 2 * g.nx * g.ny) + g.nx * g.ny * axis_prefix(z, g.nz);
    const int64_t lines  = y * (TX + g.nx * (cz - 2)) + g.nx * axis_prefix(y, g.ny);
    const int64_t cells  = axis_prefix(x, g.nx) + x * (cy + cz - 2);
    return planes + lines + cells;
}

__host__ __device__ __forceinline__ int64_t row_offset_lin(const Grid3& g, int64_t row)
{
    const int64_t t = row / g.nx;
    return row_offset(g, row % g.nx, t % g.ny, t / g.ny); // row == n gives nnz
}

// Rows [r_begin, r_end) of the global operator; offsets rebased to 0 and
// columns shifted by -col_shift (a shard's local CSR for row sharding).
__global__ void k_build_laplacian(Grid3 g, int64_t r_begin, int64_t r_end, int64_t col_shift,
                                  int64_t* __restrict__ off, int32_t* __restrict__ cols,
                                  double* __restrict__ vals)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n      = r_end - r_begin;
    const int64_t k_base = row_offset_lin(g, r_begin);
    for (int64_t lr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lr < n; lr += stride) {
        const int64_t row = r_begin + lr;
        const int64_t x = row % g.nx;
        const int64_t t = row / g.nx;
        const int64_t y = t % g.ny;
        const int64_t z = t / g.ny;
        int64_t       k = row_offset(g, x, y, z) - k_base;
        off[lr]         = k;
        if (lr == n - 1) off[n] = row_offset_lin(g, r_end) - k_base;
        for (int dz = -g.zr; dz <= g.zr; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if (!g.box && (dx != 0) + (dy != 0) + (dz != 0) > 1) continue;
                    const int64_t xx = x + dx, yy = y + dy, zz = z + dz;
                    if (xx < 0 || xx >= g.nx || yy < 0 || yy >= g.ny || zz < 0 || zz >= g.nz)
                        continue;
                    cols[k] = (int32_t)(xx + g.nx * (yy + g.ny * zz) - col_shift);
                    vals[k] = (dx == 0 && dy == 0 && dz == 0) ? g.centre : -1.0;
                    ++k;
                }
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_fill_rhs(uint64_t seed, int64_t n, double* __restrict__ b)
{
    const double  scale  = 1.0 / 4503599627370496.0; // 2^-52 (exact)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        b[i] = (double)(splitmix64(seed + (uint64_t)i) >> 11) * scale - 1.0;
}

bool stencil_valid(int dim, int points, int64_t nx, int64_t ny, int64_t nz)
{
    if (dim == 2) return (points == 5 || points == 9) && nx >= 2 && ny >= 2;
    if (dim == 3) return (points == 7 || points == 27) && nx >= 2 && ny >= 2 && nz >= 2;
    return false;
}

int grid_for(int64_t n)
{
    const int64_t want = (n + 255) / 256;
    const int64_t cap  = (int64_t)sm_count() * 16;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

} // namespace
} // namespace rvk

using namespace rvk;

extern "C" {

rvk_status rvk_laplacian_size(int dim, int points, int64_t nx, int64_t ny, int64_t nz,
                              int64_t* n_rows, int64_t* nnz)
{
    if (dim == 2) nz = 1;
    if (!stencil_valid(dim, points, nx, ny, dim == 2 ? 2 : nz))
        return set_error(RVK_ERR_INVALID, "invalid stencil spec dim=%d points=%d grid=%lldx%lldx%lld",
                         dim, points, (long long)nx, (long long)ny, (long long)nz);
    const int64_t n = nx * ny * nz;
    if (nx * ny > INT32_MAX || n > INT32_MAX)
        return set_error(RVK_ERR_INVALID, "grid too large for int32 column indices");
    Grid3 g{nx, ny, nz, (points == 9 || points == 27) ? 1 : 0, dim == 3 ? 1 : 0,
            (double)(points - 1)};
    if (n_rows) *n_rows = n;
    if (nnz) *nnz = row_offset(g, 0, 0, nz);
    return RVK_OK;
}

rvk_status rvk_build_laplacian(rvk_ctx ctx, int dim, int points, int64_t nx, int64_t ny,
                               int64_t nz, int64_t* off, int32_t* cols, double* vals)
{
    if (!ctx || !off || !cols || !vals) return set_error(RVK_ERR_INVALID, "null argument");
    if (dim == 2) nz = 1;
    int64_t n = 0, nnz = 0;
    rvk_status rc = rvk_laplacian_size(dim, points, nx, ny, nz, &n, &nnz);
    if (rc != RVK_OK) return rc;
    RVK_TRACE_TASK(ctx, "rvk_build_laplacian");
    Grid3 g{nx, ny, nz, (points == 9 || points == 27) ? 1 : 0, dim == 3 ? 1 : 0,
            (double)(points - 1)};
    k_build_laplacian<<<grid_for(n), 256, 0, ctx->stream>>>(g, 0, n, 0, off, cols, vals);
    RVK_CHECK_LAUNCH("k_build_laplacian");
    return RVK_OK;
}

rvk_status rvk_laplacian_rows_nnz(int dim, int points, int64_t nx, int64_t ny, int64_t nz,
                                  int64_t row_begin, int64_t row_end, int64_t* nnz)
{
    if (dim == 2) nz = 1;
    int64_t n = 0;
    rvk_status rc = rvk_laplacian_size(dim, points, nx, ny, nz, &n, nullptr);
    if (rc != RVK_OK) return rc;
    if (row_begin < 0 || row_end > n || row_begin >= row_end)
        return set_error(RVK_ERR_INVALID, "invalid row range [%lld, %lld) of %lld rows",
                         (long long)row_begin, (long long)row_end, (long long)n);
    Grid3 g{nx, ny, nz, (points == 9 || points == 27) ? 1 : 0, dim == 3 ? 1 : 0,
            (double)(points - 1)};
    if (nnz) *nnz = row_offset_lin(g, row_end) - row_offset_lin(g, row_begin);
    return RVK_OK;
}

rvk_status rvk_build_laplacian_rows(rvk_ctx ctx, int dim, int points, int64_t nx, int64_t ny,
                                    int64_t nz, int64_t row_begin, int64_t row_end,
                                    int64_t col_shift, int64_t* off, int32_t* cols, double* vals)
{
    if (!ctx || !off || !cols || !vals) return set_error(RVK_ERR_INVALID, "null argument");
    if (dim == 2) nz = 1;
    int64_t    nnz = 0;
    rvk_status rc  = rvk_laplacian_rows_nnz(dim, points, nx, ny, nz, row_begin, row_end, &nnz);
    if (rc != RVK_OK) return rc;
    RVK_TRACE_TASK(ctx, "rvk_build_laplacian_rows");
    Grid3 g{nx, ny, nz, (points == 9 || points == 27) ? 1 : 0, dim == 3 ? 1 : 0,
            (double)(points - 1)};
    k_build_laplacian<<<grid_for(row_end - row_begin), 256, 0, ctx->stream>>>(
        g, row_begin, row_end, col_shift, off, cols, vals);
    RVK_CHECK_LAUNCH("k_build_laplacian");
    return RVK_OK;
}

rvk_status rvk_fill_rhs(rvk_ctx ctx, uint64_t seed, int64_t n, double* b)
{
    if (!ctx || (n > 0 && !b)) return set_error(RVK_ERR_INVALID, "null argument");
    if (n <= 0) return RVK_OK;
    RVK_TRACE_TASK(ctx, "rvk_fill_rhs");
    k_fill_rhs<<<grid_for(n), 256, 0, ctx->stream>>>(seed, n, b);
    RVK_CHECK_LAUNCH("k_fill_rhs");
    return RVK_OK;
}

} // extern "C"
