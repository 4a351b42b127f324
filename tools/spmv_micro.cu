// Microbenchmark: where does the CSR SpMV time go on B200?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/spmv_micro.cu -o tools/spmv_micro
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

template <int MODE>  // 0 full, 1 no gather, 2 no vals, 3 no col (x[row])
__global__ void __launch_bounds__(256) k_rows(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                              const double* __restrict__ vals, const double* __restrict__ x,
                                              double* __restrict__ y) {
    const int G = 16;
    int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t row = gid / G;
    int lane = threadIdx.x % G;
    if (row >= n) return;
    int64_t b = __ldg(rp + row), e = __ldg(rp + row + 1);
    double a0 = 0, a1 = 0;
    int64_t p = b + lane;
    for (; p + G < e; p += 2 * G) {
        if (MODE == 0) { a0 = fma(__ldg(vals + p), __ldg(x + __ldg(col + p)), a0); a1 = fma(__ldg(vals + p + G), __ldg(x + __ldg(col + p + G)), a1); }
        if (MODE == 1) { a0 = fma(__ldg(vals + p), (double)__ldg(col + p), a0); a1 = fma(__ldg(vals + p + G), (double)__ldg(col + p + G), a1); }
        if (MODE == 2) { a0 += __ldg(x + __ldg(col + p)); a1 += __ldg(x + __ldg(col + p + G)); }
        if (MODE == 3) { a0 = fma(__ldg(vals + p), __ldg(x + (p & 1048575)), a0); a1 = fma(__ldg(vals + p + G), __ldg(x + ((p + G) & 1048575)), a1); }
    }
    if (p < e) {
        if (MODE == 0) a0 = fma(__ldg(vals + p), __ldg(x + __ldg(col + p)), a0);
        if (MODE == 1) a0 = fma(__ldg(vals + p), (double)__ldg(col + p), a0);
        if (MODE == 2) a0 += __ldg(x + __ldg(col + p));
        if (MODE == 3) a0 = fma(__ldg(vals + p), __ldg(x + (p & 1048575)), a0);
    }
    a0 += a1;
    for (int o = G / 2; o > 0; o >>= 1) a0 += __shfl_xor_sync(0xffffffffu, a0, o, G);
    if (lane == 0) y[row] = a0;
}

__global__ void k_read(int64_t nv, const double2* __restrict__ v, int64_t nc, const int4* __restrict__ c, double* out) {
    double acc = 0;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = i; j < nv; j += st) { double2 t = __ldg(v + j); acc += t.x + t.y; }
    for (int64_t j = i; j < nc; j += st) { int4 t = __ldg(c + j); acc += t.x + t.w; }
    if (acc == 1.2345) out[0] = acc;
}

int main(int argc, char** argv) {
    const int64_t n = 1000000;
    const int deg = 55;
    const int window = argc > 1 ? atoi(argv[1]) : 10000;  // 0 = uniform random
    std::mt19937_64 rng(1);
    std::vector<int64_t> rp(n + 1);
    std::vector<int32_t> col;
    col.reserve(n * deg);
    for (int64_t i = 0; i < n; ++i) {
        rp[i] = (int64_t)col.size();
        std::vector<int32_t> c;
        for (int j = 0; j < deg; ++j) {
            int64_t v = window ? (i - window / 2 + (int64_t)(rng() % window)) : (int64_t)(rng() % n);
            if (v < 0) v += n;
            if (v >= n) v -= n;
            c.push_back((int32_t)v);
        }
        std::sort(c.begin(), c.end());
        col.insert(col.end(), c.begin(), c.end());
    }
    rp[n] = (int64_t)col.size();
    const int64_t nnz = rp[n];
    std::vector<double> vals(nnz, 0.5), xh(n, 1.0);
    int64_t *drp; int32_t* dcol; double *dv, *dx, *dy;
    cudaMalloc(&drp, 8 * (n + 1)); cudaMalloc(&dcol, 4 * nnz + 64); cudaMalloc(&dv, 8 * nnz + 64); cudaMalloc(&dx, 8 * n); cudaMalloc(&dy, 8 * n);
    cudaMemcpy(drp, rp.data(), 8 * (n + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(dcol, col.data(), 4 * nnz, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, vals.data(), 8 * nnz, cudaMemcpyHostToDevice);
    cudaMemcpy(dx, xh.data(), 8 * n, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double bytes = 12.0 * nnz + 8.0 * (n + 1) + 16.0 * n;
    auto run = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        printf("window=%d %-10s %.4f ms  %.0f GB/s(alg)\n", window, name, ms, bytes / ms / 1e6);
    };
    unsigned grid = (unsigned)((n * 16 + 255) / 256);
    run("full", [&] { k_rows<0><<<grid, 256>>>(n, drp, dcol, dv, dx, dy); });
    run("nogather", [&] { k_rows<1><<<grid, 256>>>(n, drp, dcol, dv, dx, dy); });
    run("novals", [&] { k_rows<2><<<grid, 256>>>(n, drp, dcol, dv, dx, dy); });
    run("nocol", [&] { k_rows<3><<<grid, 256>>>(n, drp, dcol, dv, dx, dy); });
    run("read", [&] { k_read<<<148 * 8, 256>>>(nnz / 2, (const double2*)dv, nnz / 4, (const int4*)dcol, dy); });
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
