// Probe: 3D TMA tile load of doubles (box 34x10x1, OOB zero fill) from a
// __grid_constant__ descriptor vs a descriptor in global memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, double* out, int x, int y, int z, int bytes)
{
    __shared__ __align__(128) double buf[352];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const CUtensorMap* m = MODE == 0 ? &tm : gtm;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(bytes) : "memory");
        if (MODE == 2)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(s32(buf)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y), "r"(z), "r"(s32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(s32(buf)), "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(s32(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(s32(&bar)) : "memory");
    for (int i = threadIdx.x; i < 340; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv)
{
    const int mode_sel = argc > 1 ? atoi(argv[1]) : 0;
    const int cx = argc > 2 ? atoi(argv[2]) : -1, cy = argc > 3 ? atoi(argv[3]) : -1;
    const int dtype = argc > 4 ? atoi(argv[4]) : 0; // 0 f64, 1 u64
    const int bw = argc > 5 ? atoi(argv[5]) : 34;
    const int nx = 64, ny = 24, nz = 10;
    std::vector<double> h(nx * ny * nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i + 1;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8 + 32);
    cudaMalloc(&o, 340 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    printf("entry %p q=%d\n", f, (int)q);
    CUtensorMap tm;
    cuuint64_t dims[3] = {nx, ny, nz}, strides[2] = {nx * 8, nx * ny * 8};
    cuuint32_t box[3] = {(cuuint32_t)bw, 10, 1}, es[3] = {1, 1, 1};
    CUresult r = ((EncodeFn)f)(&tm, dtype ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    CUtensorMap* g;
    cudaMalloc(&g, sizeof tm);
    cudaMemcpy(g, &tm, sizeof tm, cudaMemcpyHostToDevice);
    for (int mode = mode_sel; mode <= mode_sel; ++mode) {
        cudaMemset(o, 0, 340 * 8);
        if (mode == 0) k<0><<<1, 128>>>(tm, g, o, cx, cy, 0, bw * 10 * 8);
        else if (mode == 1) k<1><<<1, 128>>>(tm, g, o, cx, cy, 0, bw * 10 * 8);
        else k<2><<<1, 128>>>(tm, g, o, cx, cy, 0, bw * 10 * 8);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> ho(340);
        cudaMemcpy(ho.data(), o, 340 * 8, cudaMemcpyDeviceToHost);
        printf("mode %d: %s  [0]=%g [35]=%g [36]=%g [339]=%g\n", mode, cudaGetErrorString(e), ho[0], ho[35], ho[36], ho[339]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
