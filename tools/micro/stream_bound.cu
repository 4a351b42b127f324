// Streaming bound for the C2 SpMV data volume: 55M (val fp64, col int32)
// pairs + x gathers x[col] with col = i / 55 (the "self" pattern: every
// gather an L1/L2 hit), reduced per 128-element block into one double.
// Times a flat grid-stride kernel (no rows): the rate the CSR kernels would
// reach if their row structure cost nothing.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void flat(long n, const double* __restrict__ v, const int* __restrict__ c, const double* __restrict__ x,
                     double* __restrict__ out) {
    double a = 0.0;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        a = fma(__ldg(v + i), __ldg(x + __ldg(c + i)), a);
    out[(long)blockIdx.x * blockDim.x + threadIdx.x] = a;
}
__global__ void flat4(long n, const double* __restrict__ v, const int* __restrict__ c, const double* __restrict__ x,
                      double* __restrict__ out) {
    double a = 0.0;
    const long T = (long)gridDim.x * blockDim.x;
    for (long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += T * 4) {
        const double2 v0 = *reinterpret_cast<const double2*>(v + i), v1 = *reinterpret_cast<const double2*>(v + i + 2);
        const int4 cc = *reinterpret_cast<const int4*>(c + i);
        a = fma(v0.x, __ldg(x + cc.x), a);
        a = fma(v0.y, __ldg(x + cc.y), a);
        a = fma(v1.x, __ldg(x + cc.z), a);
        a = fma(v1.y, __ldg(x + cc.w), a);
    }
    out[(long)blockIdx.x * blockDim.x + threadIdx.x] = a;
}
__global__ void init(long n, double* v, int* c) {
    long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        v[i] = 1.0 / (1 + i % 7);
        c[i] = (int)(i / 55);
    }
}
int main() {
    const long n = 54916340L / 4 * 4, nx = 1000000;
    double *v, *x, *out;
    int* c;
    cudaMalloc(&v, n * 8);
    cudaMalloc(&c, n * 4);
    cudaMalloc(&x, nx * 8);
    cudaMalloc(&out, 148L * 2048 * 8 * 8);
    cudaMemset(x, 0, nx * 8);
    init<<<(n + 255) / 256, 256>>>(n, v, c);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int variant = 0; variant < 2; ++variant)
        for (int bps : {4, 8, 16}) {
            const int grid = 148 * bps;
            for (int w = 0; w < 3; ++w) {
                if (variant == 0) flat<<<grid, 256>>>(n, v, c, x, out); else flat4<<<grid, 256>>>(n, v, c, x, out);
            }
            cudaEventRecord(e0);
            for (int r = 0; r < 20; ++r) {
                if (variant == 0) flat<<<grid, 256>>>(n, v, c, x, out); else flat4<<<grid, 256>>>(n, v, c, x, out);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            ms /= 20;
            printf("%s blocks/SM %d: %.4f ms  %.0f GB/s (12 B per nonzero)\n", variant ? "flat4" : "flat", bps, ms,
                   n * 12.0 / ms / 1e6);
        }
    return 0;
}
