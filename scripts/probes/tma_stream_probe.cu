// TMA bulk-stream probe: does the ORDER in which 148 persistent CTAs stream
// their tiles change the HBM throughput a cp.async.bulk ring reaches?
// Patterns over one big read-only buffer (tiles of `tile` bytes):
//   interleaved : CTA g takes tiles g, g+G, g+2G, ...          (k_spmv_tma's row order)
//   regions     : CTA g streams its own contiguous 1/G slice    (one long stream per SM)
//   march       : the buffer is planes of G slices of `slice` bytes; CTA g
//                 reads its slice of plane 0, then of plane 1, ... (k_spmv_march)
// One producer thread per CTA issues each tile as 3 bulk copies (offset /
// value / column-like split 1:6:3) into an S-deep mbarrier ring; 16 consumer
// warps wait for a stage, touch one word per warp and release it.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b)
{
    asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.shared::cta.b64 s, [%0];\n\t}" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t tx)
{
    asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;\n\t}" ::"r"(su32(b)),
                 "r"(tx) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par)
{
    asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra W_%=;\n\t}" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}

// pattern 0 interleaved, 1 regions, 2 march
__global__ void __launch_bounds__(544, 1)
    k_probe(const char* buf, long tiles, int tile, int S, int pattern, long slice_tiles, int* sink)
{
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full  = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + 8;
    unsigned char* ring = sm + 1024;
    const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
    // the CTA's tile sequence
    const long per = tiles / G; // tiles per CTA
    auto tile_of = [&](long j) -> long {
        if (pattern == 0) return g + j * G;
        if (pattern == 1) return (long)g * per + j;
        // march: planes of G slices of slice_tiles tiles
        const long plane = j / slice_tiles, t = j % slice_tiles;
        return (plane * G + g) * slice_tiles + t;
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], 16);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid < 32) {
        if (tid == 0) {
            for (long j = 0; j < per; ++j) {
                const int s = (int)(j % S);
                if (j >= S) mb_wait(&empty[s], (uint32_t)(((j / S) - 1) & 1));
                const char*    src = buf + tile_of(j) * (long)tile;
                unsigned char* dst = ring + (size_t)s * tile;
                const uint32_t a = (tile / 10) & ~15, b = (tile * 6 / 10) & ~15, c = tile - a - b;
                mb_expect(&full[s], tile);
                bulk(dst, src, a, &full[s]);
                bulk(dst + a, src + a, b, &full[s]);
                bulk(dst + a + b, src + a + b, c, &full[s]);
            }
        }
        return;
    }
    int acc = 0;
    for (long j = 0; j < per; ++j) {
        const int s = (int)(j % S);
        mb_wait(&full[s], (uint32_t)((j / S) & 1));
        acc += ring[(size_t)s * tile + ((tid - 32) * 64) % tile];
        __syncwarp();
        if ((tid & 31) == 0) mb_arrive(&empty[s]);
    }
    if (acc == 123456789) *sink = acc;
}

int main(int argc, char** argv)
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long bytes = (argc > 1 ? atol(argv[1]) : 24L) << 30; // GiB (default 24)
    char* buf;
    int*  sink;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&sink, 4);
    cudaMemset(buf, 1, bytes);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const char* names[] = {"interleaved", "regions", "march"};
    for (int tile : {24576, 47104, 55296}) {
        for (int S : {2, 3, 4}) {
            if (1024 + (long)S * tile > 227 * 1024) continue;
            const long tiles = (bytes / tile) / sms * sms;
            for (int pat = 0; pat < 3; ++pat) {
                // march slices: ~367 KB of a 768^2 plane's CSR per SM per step
                const long slice = (pat == 2) ? (367 * 1024) / tile : 1;
                long       use   = tiles;
                if (pat == 2) use = (tiles / (sms * slice)) * sms * slice;
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                k_probe<<<sms, 544, 1024 + S * tile>>>(buf, use, tile, S, pat, slice, sink);
                cudaEventRecord(a);
                k_probe<<<sms, 544, 1024 + S * tile>>>(buf, use, tile, S, pat, slice, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                printf("tile %6d B  stages %d  %-11s  %7.1f GB/s  (%s)\n", tile, S, names[pat],
                       (double)use * tile / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
