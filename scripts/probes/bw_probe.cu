// HBM ceiling probe: what a read-dominated stream (K1's 88/12 read/write mix)
// can reach on this B200, vs the 1:1 copy figure in MEASURED_PEAKS.json.
// Prints GB/s for: read-only reduction, 1:1 copy, 7:1 read:write, at 2 GB.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ double4 ldv(const double4* p)
{
    double4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ldv2(const double2* p)
{
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

// RS read streams (each n2 double2), WS write streams; U loads in flight per thread
template <int RS, int WS, int U>
__global__ void k_mix(const double2* __restrict__ in, double2* __restrict__ out, long n2, double* sink)
{
    double acc = 0;
    const long stride = (long)gridDim.x * blockDim.x;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride * U) {
        double2 v[RS][U];
#pragma unroll
        for (int s = 0; s < RS; ++s)
#pragma unroll
            for (int u = 0; u < U; ++u)
                v[s][u] = (i + u * stride < n2) ? ldv2(in + s * n2 + i + u * stride) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double2 t = make_double2(0, 0);
#pragma unroll
            for (int s = 0; s < RS; ++s) { t.x += v[s][u].x; t.y += v[s][u].y; }
#pragma unroll
            for (int w = 0; w < WS; ++w)
                if (i + u * stride < n2) out[w * n2 + i + u * stride] = t;
            acc += t.x;
        }
    }
    if (acc == 12345.678) *sink = acc;
}

template <int RS, int WS, int U>
void run(const char* name, double2* in, double2* out, long n2, double* sink, int blocks, int threads)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k_mix<RS, WS, U><<<blocks, threads>>>(in, out, n2, sink);
    cudaEventRecord(a);
    const int reps = 20;
    for (int r = 0; r < reps; ++r) k_mix<RS, WS, U><<<blocks, threads>>>(in, out, n2, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 16.0 * n2 * (RS + WS);
    printf("%-28s blocks %5d x %4d  %8.1f GB/s  (%.1f us)\n", name, blocks, threads, bytes * reps / (ms * 1e-3) / 1e9,
           ms * 1e3 / reps);
}

int main(int argc, char** argv)
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // argv[1]: GiB per stream (default 1; the footprint test runs 1, 4, 8)
    const long gib = argc > 1 ? atol(argv[1]) : 1;
    const long n2 = (1L << 26) * gib;
    printf("stream size %ld GiB\n", gib);
    double2 *in, *out;
    double*  sink;
    cudaMalloc(&in, 8 * n2 * 16);
    cudaMalloc(&out, 2 * n2 * 16);
    cudaMalloc(&sink, 8);
    cudaMemset(in, 0, 8 * n2 * 16);
    cudaMemset(out, 0, 2 * n2 * 16);
    for (int occ : {8}) {
        const int bl = sms * occ;
        run<2, 0, 4>("read 2 streams", in, out, n2, sink, bl, 256);
        run<1, 1, 4>("copy 1:1", in, out, n2, sink, bl, 256);
        run<7, 1, 2>("7 read : 1 write", in, out, n2, sink, bl, 256);
        run<4, 1, 4>("4 read : 1 write", in, out, n2, sink, bl, 256);
        run<2, 2, 4>("2 read : 2 write (K2-like)", in, out, n2, sink, bl, 256);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
