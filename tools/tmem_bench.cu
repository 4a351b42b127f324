// Microbenchmark: tcgen05.ld throughput (TMEM -> registers) per SM.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k(int iters, float* out, long long* cyc) {
    __shared__ uint32_t slot;
    int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    float acc = 0.f;
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[64];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(r[q*16+0]), "=r"(r[q*16+1]), "=r"(r[q*16+2]), "=r"(r[q*16+3]), "=r"(r[q*16+4]), "=r"(r[q*16+5]),
                           "=r"(r[q*16+6]), "=r"(r[q*16+7]), "=r"(r[q*16+8]), "=r"(r[q*16+9]), "=r"(r[q*16+10]), "=r"(r[q*16+11]),
                           "=r"(r[q*16+12]), "=r"(r[q*16+13]), "=r"(r[q*16+14]), "=r"(r[q*16+15])
                         : "r"(t + q * 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 64; ++q) acc += __uint_as_float(r[q]);
    }
    long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot));
}
template <int NW> void run(int blocks) {
    int iters = 20000;
    float* o; long long* c; cudaMalloc(&o, 4 * blocks * NW * 32); cudaMalloc(&c, 8 * blocks);
    k<NW><<<blocks, NW * 32>>>(100, o, c);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<NW><<<blocks, NW * 32>>>(iters, o, c); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double bytes_per_blk_iter = NW * 32.0 * 64 * 4;
    printf("warps=%d blocks=%d: %.1f cycles/iter/block -> %.1f B/cycle/block; %s\n", NW, blocks, (double)h / iters,
           bytes_per_blk_iter / ((double)h / iters), cudaGetErrorString(cudaGetLastError()));
}
int main() { run<4>(148); run<8>(148); run<4>(296); run<16>(148); return 0; }
