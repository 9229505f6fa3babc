// Microbenchmark (dev tool): GPU-initiated reads of pinned host memory over
// PCIe at different request shapes; how many useful GB/s each reaches.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// mode 0: thread reads 4 B of a random 32-B sector; 1: 16 B (ld.v4) of one;
// 2: a warp reads a random 128-B line (lane 4 B); 3: a warp reads 512 B (lane 16 B)
__global__ void k_gather(const float *__restrict__ src, size_t n_floats, int mode, int iters, float *sink)
{
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31;
    const uint32_t warp = tid >> 5;
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) {
            const size_t sec = hash32(tid * 1315423911u + i) % (n_floats / 8);
            acc += src[sec * 8];
        } else if (mode == 1) {
            const size_t sec = hash32(tid * 1315423911u + i) % (n_floats / 8);
            const float4 v = *reinterpret_cast<const float4 *>(src + sec * 8);
            acc += v.x + v.w;
        } else if (mode == 2) {
            const size_t line = hash32(warp * 2654435761u + i) % (n_floats / 32);
            acc += src[line * 32 + lane];
        } else {
            const size_t blk = hash32(warp * 2654435761u + i) % (n_floats / 128);
            const float4 v = reinterpret_cast<const float4 *>(src + blk * 128)[lane];
            acc += v.x + v.w;
        }
    }
    if (acc == 123.456f) sink[0] = acc;
}

extern "C" float run_gather(const float *src, size_t n_floats, int mode, int blocks, int threads, int iters)
{
    float *sink;
    cudaMalloc(&sink, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_gather<<<blocks, threads>>>(src, n_floats, mode, 2, sink);
    cudaEventRecord(a);
    k_gather<<<blocks, threads>>>(src, n_floats, mode, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(sink);
    return ms;
}
