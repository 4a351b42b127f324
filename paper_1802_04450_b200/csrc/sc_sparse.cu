// CSR kernels: SpMV (sequential-order and vectorised), degrees, symmetric
// scaling, exact symmetry check, non-positive degree search.
//
// Device CSR layout: row_ptr int64[n+1],
// col int32[nnz] (n < 2^31), vals f64[nnz]; rows sorted, columns strictly
// increasing within a row (sparse.py:110-138).
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#include "sc_common.cuh"
#include "sc_sparse.cuh"

namespace sc {

// y_i = sum_p vals[p] * x[col[p]], each row accumulated sequentially in column
// order with separately rounded products: bit-identical to the reference's
// np.bincount(rows, vals * x[col]) (sparse.py:205-207).
__global__ void spmv_seq_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                const int32_t* __restrict__ col, const double* __restrict__ vals,
                                const double* __restrict__ x, double* __restrict__ y) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t p = row_ptr[i], e = row_ptr[i + 1];
    double acc = 0.0;
    for (; p < e; ++p) acc = __dadd_rn(acc, __dmul_rn(vals[p], __ldg(x + col[p])));
    y[i] = acc;
}

// Vectorised CSR SpMV: G lanes per row, strided products, shuffle tree.
// Used inside the eigensolver where the reduction order is free (eigenvalue
// parity is a 1e-5 tolerance).
template <int G>
__global__ void __launch_bounds__(256) spmv_vec_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                                       const int32_t* __restrict__ col,
                                                       const double* __restrict__ vals,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y) {
    int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t row = gid / G;
    int lane = threadIdx.x % G;
    if (row >= n) return;
    int64_t b = row_ptr[row], e = row_ptr[row + 1];
    double acc = 0.0;
    int64_t p = b + lane;
    // two independent chains for memory-level parallelism
    double acc2 = 0.0;
    for (; p + G < e; p += 2 * G) {
        int32_t c0 = __ldg(col + p), c1 = __ldg(col + p + G);
        double v0 = __ldg(vals + p), v1 = __ldg(vals + p + G);
        acc = fma(v0, __ldg(x + c0), acc);
        acc2 = fma(v1, __ldg(x + c1), acc2);
    }
    if (p < e) acc = fma(__ldg(vals + p), __ldg(x + __ldg(col + p)), acc);
    acc += acc2;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
    if (lane == 0) y[row] = acc;
}

// Cache-policy loads for the SpMV: the col/vals/row_ptr streams are read once
// and must not evict the x entries the rows gather (L1::no_allocate), while x
// is kept (L1::evict_last) so a row block's neighbourhood stays in L1.
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int64_t ld_stream(const int64_t* p) {
    int64_t v;
    asm("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_keep(const double* p) {
    double v;
    asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// Locality SpMV.  The rows are cut into kNumSMs contiguous ranges; block b
// works on range b % kNumSMs, which for a grid of exactly one resident wave
// (kNumSMs x SPMV_LOCAL_BPS blocks) is the SM the block scheduler puts it on.
// All warps of that SM walk their range together, G lanes per row and 32/G
// rows per warp, so once the operator is in locality order (a row's columns
// lie in a window of nearby rows, pipeline.py / sc_knn.cu pivot chain) the
// x gathers are served by the SM's L1 (no shared memory: the whole unified
// carve-out is L1) instead of one random L2 sector per nonzero.  Correctness
// does not depend on the block -> SM placement, only the hit rate does.
template <int G>
__global__ void __launch_bounds__(256) spmv_local_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ vals,
                                                         const double* __restrict__ x, double* __restrict__ y) {
    constexpr int RPW = 32 / G;
    const int grp = blockIdx.x % kNumSMs, sub = blockIdx.x / kNumSMs;
    const int64_t r0 = n * grp / kNumSMs, r1 = n * (grp + 1) / kNumSMs;
    const int lane = threadIdx.x & 31, sl = lane % G;
    const int wpb = blockDim.x >> 5;
    const int64_t stride = (int64_t)(gridDim.x / kNumSMs) * wpb * RPW;
    for (int64_t base = r0 + ((int64_t)sub * wpb + (threadIdx.x >> 5)) * RPW; base < r1; base += stride) {
        const int64_t row = base + lane / G;
        const bool valid = row < r1;
        int64_t p = 0, e = 0;
        if (valid) {
            p = ld_stream(row_ptr + row) + sl;
            e = ld_stream(row_ptr + row + 1);
        }
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (; p + 3 * G < e; p += 4 * G) {
            const int32_t c0 = ld_stream(col + p), c1 = ld_stream(col + p + G), c2 = ld_stream(col + p + 2 * G),
                          c3 = ld_stream(col + p + 3 * G);
            const double v0 = ld_stream(vals + p), v1 = ld_stream(vals + p + G), v2 = ld_stream(vals + p + 2 * G),
                         v3 = ld_stream(vals + p + 3 * G);
            a0 = fma(v0, ld_keep(x + c0), a0);
            a1 = fma(v1, ld_keep(x + c1), a1);
            a2 = fma(v2, ld_keep(x + c2), a2);
            a3 = fma(v3, ld_keep(x + c3), a3);
        }
        if (p + G < e) {
            const int32_t c0 = ld_stream(col + p), c1 = ld_stream(col + p + G);
            const double v0 = ld_stream(vals + p), v1 = ld_stream(vals + p + G);
            a0 = fma(v0, ld_keep(x + c0), a0);
            a1 = fma(v1, ld_keep(x + c1), a1);
            p += 2 * G;
        }
        if (p < e) a2 = fma(ld_stream(vals + p), ld_keep(x + ld_stream(col + p)), a2);
        double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
        if (valid && sl == 0) y[row] = acc;
    }
}

// Batched warp-per-row SpMV: a warp owns R consecutive rows and issues the
// first two 32-wide strips of all R rows (2R col + 2R val loads per lane, then
// 2R independent x gathers) before consuming any of them, so each warp keeps
// ~R times the bytes in flight of a one-row warp.  (The one-row kernel is
// long-scoreboard bound at ~2.2 TB/s: row_ptr -> col/vals -> x is a chain of
// three dependent round trips per ~55 nonzeros.)  Longer rows finish in a
// strip loop; lane sums go through one shuffle tree per row.
template <int R>
__global__ void __launch_bounds__(256) spmv_batch_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ vals,
                                                         const double* __restrict__ x, double* __restrict__ y) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t row0 = warp * R;
    if (row0 >= n) return;
    const int64_t nr = imin64(R, n - row0);
    const int64_t rp = lane <= nr ? __ldg(row_ptr + row0 + lane) : 0;
    int64_t b[R], e[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        b[r] = __shfl_sync(0xffffffffu, rp, r);
        e[r] = r < nr ? __shfl_sync(0xffffffffu, rp, r + 1) : b[r];
    }
    int32_t c[R][2];
    double v[R][2];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int64_t p = b[r] + lane + 32 * u;
            const bool ok = p < e[r];
            c[r][u] = ok ? __ldg(col + p) : -1;
            v[r][u] = ok ? __ldg(vals + p) : 0.0;
        }
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double a = 0.0;
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (c[r][u] >= 0) a = fma(v[r][u], __ldg(x + c[r][u]), a);
        for (int64_t p = b[r] + lane + 64; p < e[r]; p += 32) a = fma(__ldg(vals + p), __ldg(x + __ldg(col + p)), a);
        acc[r] = a;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const double s = warp_sum(acc[r]);
        if (lane == r && r < nr) y[row0 + r] = s;
    }
}

// Software-pipelined warp-per-row SpMV over per-SM row ranges (as in
// spmv_local_kernel).  While a warp's x gathers for row t are in flight it
// already holds the first two 32-wide col/val strips of row t+1 and the
// row_ptr pair of row t+2, so the HBM stream (col, vals, row_ptr) never
// waits behind the gathers.  Rows longer than 64 finish in a strip loop.
__global__ void __launch_bounds__(256) spmv_pipe_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                                        const int32_t* __restrict__ col,
                                                        const double* __restrict__ vals,
                                                        const double* __restrict__ x, double* __restrict__ y) {
    const int grp = blockIdx.x % kNumSMs, sub = blockIdx.x / kNumSMs;
    const int64_t r0 = n * grp / kNumSMs, r1 = n * (grp + 1) / kNumSMs;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)(gridDim.x / kNumSMs) * (blockDim.x >> 5);
    int64_t row = r0 + (int64_t)sub * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= r1) return;
    auto bounds = [&](int64_t r, int64_t& b, int64_t& e) {
        if (r < r1) {
            const int64_t v = __ldg(row_ptr + r + (lane & 1));
            b = __shfl_sync(0xffffffffu, v, 0);
            e = __shfl_sync(0xffffffffu, v, 1);
        } else {
            b = e = 0;
        }
    };
    auto strips = [&](int64_t b, int64_t e, int32_t& c0, int32_t& c1, double& v0, double& v1) {
        const int64_t p = b + lane;
        c0 = p < e ? __ldg(col + p) : -1;
        v0 = p < e ? __ldg(vals + p) : 0.0;
        c1 = p + 32 < e ? __ldg(col + p + 32) : -1;
        v1 = p + 32 < e ? __ldg(vals + p + 32) : 0.0;
    };
    int64_t b, e, nb, ne;
    bounds(row, b, e);
    bounds(row + stride, nb, ne);
    int32_t c0, c1;
    double v0, v1;
    strips(b, e, c0, c1, v0, v1);
    for (; row < r1; row += stride) {
        // prefetch: strips of the next row, bounds of the one after
        int32_t d0, d1;
        double w0, w1;
        strips(nb, ne, d0, d1, w0, w1);
        int64_t nnb, nne;
        bounds(row + 2 * stride, nnb, nne);
        double acc = 0.0, acc2 = 0.0;
        if (c0 >= 0) acc = v0 * __ldg(x + c0);
        if (c1 >= 0) acc2 = v1 * __ldg(x + c1);
        for (int64_t p = b + 64 + lane; p < e; p += 32) acc = fma(__ldg(vals + p), __ldg(x + __ldg(col + p)), acc);
        const double s = warp_sum(acc + acc2);
        if (lane == 0) y[row] = s;
        b = nb;
        e = ne;
        nb = nnb;
        ne = nne;
        c0 = d0;
        c1 = d1;
        v0 = w0;
        v1 = w1;
    }
}

// SM-affine SpMV: the rows are cut into one contiguous range per SM id
// (%nsmid ranges); a warp first drains the range of the SM it runs on
// (atomic per-range cursor, SPMV_GRAB rows per grab) and then steals from the
// other ranges, so every row is done exactly once whatever the block
// placement, and in locality order an SM's gathers stay inside its range's
// x neighbourhood (its L1).  cursors: nsmid ints, zero at launch.
constexpr int SPMV_GRAB_ITERS = 16;
constexpr int SPMV_MAX_RANGES = kNumSMs;
__device__ __forceinline__ uint32_t sm_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t sm_count() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(r));
    return r;
}
template <int G>
__global__ void __launch_bounds__(256) spmv_affine_kernel(int64_t n, int nranges, const int64_t* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ vals,
                                                          const double* __restrict__ x, double* __restrict__ y,
                                                          int* __restrict__ cursors) {
    constexpr int RPW = 32 / G;
    constexpr int GRAB = RPW * SPMV_GRAB_ITERS;
    const int lane = threadIdx.x & 31, sl = lane % G;
    const int home = (int)(sm_id() % (uint32_t)nranges);
    for (int t = 0; t < nranges; ++t) {
        const int rg = (home + t) % nranges;
        const int64_t r0 = n * rg / nranges, r1 = n * (rg + 1) / nranges;
        const int len = (int)(r1 - r0);
        while (true) {
            int start = 0;
            if (lane == 0) start = *((volatile int*)cursors + rg) >= len ? len : atomicAdd(cursors + rg, GRAB);
            start = __shfl_sync(0xffffffffu, start, 0);
            if (start >= len) break;
            const int64_t end = imin64(r1, r0 + start + GRAB);
            for (int64_t base = r0 + start; base < end; base += RPW) {
                const int64_t row = base + lane / G;
                const bool valid = row < end;
                int64_t p = 0, e = 0;
                if (valid) {
                    p = ld_stream(row_ptr + row) + sl;
                    e = ld_stream(row_ptr + row + 1);
                }
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                for (; p + 3 * G < e; p += 4 * G) {
                    const int32_t c0 = ld_stream(col + p), c1 = ld_stream(col + p + G),
                                  c2 = ld_stream(col + p + 2 * G), c3 = ld_stream(col + p + 3 * G);
                    const double v0 = ld_stream(vals + p), v1 = ld_stream(vals + p + G),
                                 v2 = ld_stream(vals + p + 2 * G), v3 = ld_stream(vals + p + 3 * G);
                    a0 = fma(v0, ld_keep(x + c0), a0);
                    a1 = fma(v1, ld_keep(x + c1), a1);
                    a2 = fma(v2, ld_keep(x + c2), a2);
                    a3 = fma(v3, ld_keep(x + c3), a3);
                }
                if (p + G < e) {
                    const int32_t c0 = ld_stream(col + p), c1 = ld_stream(col + p + G);
                    const double v0 = ld_stream(vals + p), v1 = ld_stream(vals + p + G);
                    a0 = fma(v0, ld_keep(x + c0), a0);
                    a1 = fma(v1, ld_keep(x + c1), a1);
                    p += 2 * G;
                }
                if (p < e) a2 = fma(ld_stream(vals + p), ld_keep(x + ld_stream(col + p)), a2);
                double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
                if (valid && sl == 0) y[row] = acc;
            }
        }
    }
}

template <int G>
static int spmv_affine_launch(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                              const double* x, double* y, int* cursors, cudaStream_t st) {
    static int bps = 0, nsm = 0;
    if (!bps) {
        cudaFuncSetAttribute(spmv_affine_kernel<G>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, spmv_affine_kernel<G>, 256, 0);
        if (bps < 1) bps = 1;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    SC_CUDA(cudaMemsetAsync(cursors, 0, sizeof(int) * SPMV_MAX_RANGES, st));
    spmv_affine_kernel<G><<<nsm * bps, 256, 0, st>>>(n, SPMV_MAX_RANGES, row_ptr, col, vals, x, y, cursors);
    return SC_OK;
}

template <int G>
static void spmv_local_launch(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                              const double* x, double* y, cudaStream_t st) {
    static int bps = 0;
    if (!bps) {  // all of the unified L1/shared array as L1; one resident wave
        cudaFuncSetAttribute(spmv_local_kernel<G>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, spmv_local_kernel<G>, 256, 0);
        if (bps < 1) bps = 1;
    }
    spmv_local_kernel<G><<<kNumSMs * bps, 256, 0, st>>>(n, row_ptr, col, vals, x, y);
}

// "placed": spmv_local_kernel's per-SM row ranges with the block -> SM
// placement MEASURED instead of assumed.  A probe kernel with the identical
// launch configuration records %smid per block once; the host turns it into
// per-block descriptors (range = the SM the block ran on, sub-index among
// that SM's blocks), so the blocks sharing an SM (and its L1) share one
// contiguous row range and its x working set.  Correctness does not depend
// on the placement repeating (every range is covered by its descriptors);
// only the L1 hit rate does.
__global__ void smid_probe_kernel(int* __restrict__ out) {
    if (threadIdx.x == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        out[blockIdx.x] = (int)sm;
    }
}

template <int G>
__global__ void __launch_bounds__(256) spmv_placed_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ vals,
                                                          const double* __restrict__ x, double* __restrict__ y,
                                                          const int4* __restrict__ desc) {
    constexpr int RPW = 32 / G;
    const int4 dsc = desc[blockIdx.x];  // (range, sub-index, blocks in the range, ranges)
    const int64_t r0 = n * dsc.x / dsc.w, r1 = n * (dsc.x + 1) / dsc.w;
    const int lane = threadIdx.x & 31, sl = lane % G;
    const int wpb = blockDim.x >> 5;
    const int64_t stride = (int64_t)dsc.z * wpb * RPW;
    for (int64_t base = r0 + ((int64_t)dsc.y * wpb + (threadIdx.x >> 5)) * RPW; base < r1; base += stride) {
        const int64_t row = base + lane / G;
        const bool valid = row < r1;
        int64_t p = 0, e = 0;
        if (valid) {
            p = ld_stream(row_ptr + row) + sl;
            e = ld_stream(row_ptr + row + 1);
        }
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (; p + 3 * G < e; p += 4 * G) {
            const int32_t c0 = ld_stream(col + p), c1 = ld_stream(col + p + G), c2 = ld_stream(col + p + 2 * G),
                          c3 = ld_stream(col + p + 3 * G);
            const double v0 = ld_stream(vals + p), v1 = ld_stream(vals + p + G), v2 = ld_stream(vals + p + 2 * G),
                         v3 = ld_stream(vals + p + 3 * G);
            a0 = fma(v0, ld_keep(x + c0), a0);
            a1 = fma(v1, ld_keep(x + c1), a1);
            a2 = fma(v2, ld_keep(x + c2), a2);
            a3 = fma(v3, ld_keep(x + c3), a3);
        }
        if (p + G < e) {
            const int32_t c0 = ld_stream(col + p), c1 = ld_stream(col + p + G);
            const double v0 = ld_stream(vals + p), v1 = ld_stream(vals + p + G);
            a0 = fma(v0, ld_keep(x + c0), a0);
            a1 = fma(v1, ld_keep(x + c1), a1);
            p += 2 * G;
        }
        if (p < e) a2 = fma(ld_stream(vals + p), ld_keep(x + ld_stream(col + p)), a2);
        double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
        if (valid && sl == 0) y[row] = acc;
    }
}

template <int G>
static int spmv_placed_launch(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                              const double* x, double* y, cudaStream_t st) {
    static int bps = 0, nblk = 0;
    static int4* desc = nullptr;  // device, built once per process (same launch configuration)
    if (!desc) {
        cudaFuncSetAttribute(spmv_placed_kernel<G>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
        cudaFuncSetAttribute(smid_probe_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, spmv_placed_kernel<G>, 256, 0);
        if (bps < 1) bps = 1;
        int dev = 0, nsm = kNumSMs;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        nblk = nsm * bps;
        int* dsm = nullptr;
        SC_CUDA(cudaMalloc(&dsm, sizeof(int) * nblk));
        SC_CUDA(cudaStreamSynchronize(st));
        smid_probe_kernel<<<nblk, 256, 0, st>>>(dsm);
        std::vector<int> sm(nblk);
        SC_CUDA(d2h_sync(sm.data(), dsm, sizeof(int) * nblk, st));
        cudaFree(dsm);
        // ranges: the distinct SMs seen, in id order; blocks numbered within each
        std::vector<int> ids(sm), cnt;
        std::sort(ids.begin(), ids.end());
        ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
        cnt.assign(ids.size(), 0);
        std::vector<int4> h(nblk);
        for (int b = 0; b < nblk; ++b) {
            const int r = (int)(std::lower_bound(ids.begin(), ids.end(), sm[b]) - ids.begin());
            h[b] = make_int4(r, cnt[r]++, 0, (int)ids.size());
        }
        for (int b = 0; b < nblk; ++b) h[b].z = cnt[h[b].x];
        SC_CUDA(cudaMalloc(&desc, sizeof(int4) * nblk));
        SC_CUDA(cudaMemcpy(desc, h.data(), sizeof(int4) * nblk, cudaMemcpyHostToDevice));
    }
    spmv_placed_kernel<G><<<nblk, 256, 0, st>>>(n, row_ptr, col, vals, x, y, desc);
    return SC_OK;
}

// SpMV kernel choice.  Default: "placed" (per-SM row ranges on the measured
// block placement); "local" assumes block b runs on SM b % 148.
// SPECLUST_SPMV_KERNEL overrides it (tuning and tests): "vec" (one row per
// warp, flat grid), "affine" (SM-id ranges with stealing), "pipe"
// (software-pipelined), "batch2"/"batch4"/"batch8" (R rows per warp),
// "bulk" (SpmvPlan only: cp.async.bulk staged chunks).
int spmv_kind() {
    const char* kenv = std::getenv("SPECLUST_SPMV_KERNEL");
    if (!kenv) return 10;  // "placed": 0.26 vs 0.29 ms per C2 matvec for "local" (tools/spmv_c2.py)
    if (!std::strcmp(kenv, "vec")) return 0;
    if (!std::strcmp(kenv, "affine")) return 1;
    if (!std::strcmp(kenv, "batch2")) return 2;
    if (!std::strcmp(kenv, "batch4")) return 4;
    if (!std::strcmp(kenv, "pipe")) return 5;
    if (!std::strcmp(kenv, "batch8")) return 8;
    if (!std::strcmp(kenv, "bulk")) return 9;
    if (!std::strcmp(kenv, "local")) return 6;
    if (!std::strcmp(kenv, "placed")) return 10;
    return 6;
}

int spmv_launch(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                const double* vals, const double* x, double* y, bool deterministic,
                cudaStream_t st) {
    if (n == 0) return SC_OK;
    double bytes = (double)nnz * 12.0 + (double)(n + 1) * 8.0 + 2.0 * (double)n * 8.0;
    ProfScope prof(deterministic ? "spmv_seq" : "spmv", st, bytes);
    const int kind = spmv_kind();
    const double mean_len = (double)nnz / (double)n;
    if (deterministic) {
        spmv_seq_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, row_ptr, col, vals, x, y);
    } else if (kind == 5 && mean_len > 24 && n >= 4096) {
        static int bps = 0;
        if (!bps) {  // one resident wave: blocks per SM from the occupancy calculator
            cudaFuncSetAttribute(spmv_pipe_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, spmv_pipe_kernel, 256, 0);
            if (bps < 1) bps = 1;
        }
        spmv_pipe_kernel<<<kNumSMs * bps, 256, 0, st>>>(n, row_ptr, col, vals, x, y);
    } else if ((kind == 2 || kind == 4 || kind == 8 || kind == 9) && mean_len > 24) {
        if (kind == 2)
            spmv_batch_kernel<2><<<(unsigned)ceil_div(ceil_div(n, 2) * 32, 256), 256, 0, st>>>(n, row_ptr, col, vals, x, y);
        else if (kind == 8)
            spmv_batch_kernel<8><<<(unsigned)ceil_div(ceil_div(n, 8) * 32, 256), 256, 0, st>>>(n, row_ptr, col, vals, x, y);
        else
            spmv_batch_kernel<4><<<(unsigned)ceil_div(ceil_div(n, 4) * 32, 256), 256, 0, st>>>(n, row_ptr, col, vals, x, y);
    } else if (kind == 6 && n >= 4096) {
        if (mean_len > 24)
            spmv_local_launch<16>(n, row_ptr, col, vals, x, y, st);
        else
            spmv_local_launch<8>(n, row_ptr, col, vals, x, y, st);
    } else if (kind == 10 && n >= 4096) {
        const int rc = mean_len > 24 ? spmv_placed_launch<16>(n, row_ptr, col, vals, x, y, st)
                                     : spmv_placed_launch<8>(n, row_ptr, col, vals, x, y, st);
        if (rc) return rc;
    } else if (kind == 1 && n >= 4096) {
        DevBuf<int> cur;
        int rc;
        if ((rc = cur.alloc(SPMV_MAX_RANGES))) return rc;
        if (mean_len > 24)
            rc = spmv_affine_launch<16>(n, row_ptr, col, vals, x, y, cur.p, st);
        else
            rc = spmv_affine_launch<8>(n, row_ptr, col, vals, x, y, cur.p, st);
        if (rc) return rc;
    } else {
        double mean = n ? (double)nnz / (double)n : 0.0;
        static const char* genv = std::getenv("SPECLUST_SPMV_G");  // tuning override
        if (genv) mean = std::atoi(genv) == 32 ? 100 : std::atoi(genv) == 16 ? 20 : std::atoi(genv) == 8 ? 8 : 1;
        if (mean > 24) {
            spmv_vec_kernel<32><<<(unsigned)ceil_div(n * 32, 256), 256, 0, st>>>(n, row_ptr, col, vals, x, y);
        } else if (mean > 10) {
            spmv_vec_kernel<16><<<(unsigned)ceil_div(n * 16, 256), 256, 0, st>>>(n, row_ptr, col, vals, x, y);
        } else if (mean > 4) {
            spmv_vec_kernel<8><<<(unsigned)ceil_div(n * 8, 256), 256, 0, st>>>(n, row_ptr, col, vals, x, y);
        } else {
            spmv_vec_kernel<4><<<(unsigned)ceil_div(n * 4, 256), 256, 0, st>>>(n, row_ptr, col, vals, x, y);
        }
    }
    SC_LAUNCHED(1);
    return SC_OK;
}

// d_i = sequential row sum (laplacian.py:27-31 = spmv(w, ones)).
__global__ void degrees_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                               const double* __restrict__ vals, double* __restrict__ d) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int64_t p = row_ptr[i], e = row_ptr[i + 1]; p < e; ++p) acc = __dadd_rn(acc, vals[p]);
    d[i] = acc;
}

int degrees_launch(int64_t n, const int64_t* row_ptr, const double* vals, double* d,
                   cudaStream_t st) {
    if (n == 0) return SC_OK;
    degrees_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, row_ptr, vals, d);
    SC_LAUNCHED(1);
    return SC_OK;
}

// a_ij = w_ij / sqrt(d_i * d_j)  (laplacian.py:89-91: one product, one sqrt,
// one division, all IEEE round-to-nearest -> bit-identical to numpy).
// (row_offset: the CSR holds rows row_offset .. row_offset+n-1 of the global
// matrix; d is the global degree vector)
__global__ void sym_scale_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ col, const double* __restrict__ vals,
                                 const double* __restrict__ d, double* __restrict__ out, int64_t row_offset = 0) {
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (i >= n) return;
    double di = d[row_offset + i];
    for (int64_t p = row_ptr[i] + (threadIdx.x & 31), e = row_ptr[i + 1]; p < e; p += 32) {
        double s = __dsqrt_rn(__dmul_rn(di, __ldg(d + col[p])));
        out[p] = __ddiv_rn(vals[p], s);
    }
}

// Every entry (i, j, v) must have a mirror (j, i, v); rows hold unique
// columns, so this is equivalent to A == A^T (sparse.py:210-222).
// Only the strictly upper entries (i, j > i) look up their mirror (j, i);
// the lower ones are counted: every upper entry has an equal mirror and
// #upper == #lower  <=>  the matrix is symmetric (the mirror map is then a
// bijection onto the lower entries).
__global__ void symmetric_check_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                       const int32_t* __restrict__ col,
                                       const double* __restrict__ vals, int* __restrict__ bad,
                                       unsigned long long* __restrict__ ul) {
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (i >= n) return;
    unsigned long long nu = 0, nl = 0;
    for (int64_t p = row_ptr[i] + (threadIdx.x & 31), e = row_ptr[i + 1]; p < e; p += 32) {
        int64_t j = col[p];
        if (j <= i) {
            nl += j < i;
            continue;
        }
        ++nu;
        int64_t lo = row_ptr[j], hi = row_ptr[j + 1];
        // binary search for column i in row j
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (col[mid] < i) lo = mid + 1; else hi = mid;
        }
        if (lo >= row_ptr[j + 1] || col[lo] != i || !(vals[lo] == vals[p])) atomicOr(bad, 1);
    }
    for (int o = 16; o > 0; o >>= 1) {
        nu += __shfl_xor_sync(0xffffffffu, nu, o);
        nl += __shfl_xor_sync(0xffffffffu, nl, o);
    }
    if ((threadIdx.x & 31) == 0 && (nu | nl)) {
        atomicAdd(ul, nu);
        atomicAdd(ul + 1, nl);
    }
}

__global__ void count_nonpositive_kernel(int64_t n, const double* __restrict__ d, int mode,
                                         unsigned long long* __restrict__ count) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool hit = false;
    if (i < n) hit = mode == 0 ? (d[i] == 0.0) : !(d[i] > 0.0);
    unsigned ballot = __ballot_sync(0xffffffffu, hit);
    if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(count, (unsigned long long)__popc(ballot));
}

// ordered compaction of matching indices (error path only; one block)
__global__ void list_nonpositive_kernel(int64_t n, const double* __restrict__ d, int mode,
                                        int64_t* __restrict__ out, int64_t cap) {
    __shared__ int warp_tot[32];
    __shared__ int64_t base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int64_t off = 0; off < n && base < cap; off += blockDim.x) {
        int64_t i = off + threadIdx.x;
        bool hit = false;
        if (i < n) hit = mode == 0 ? (d[i] == 0.0) : !(d[i] > 0.0);
        unsigned ballot = __ballot_sync(0xffffffffu, hit);
        int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 0) warp_tot[w] = __popc(ballot);
        __syncthreads();
        int before = 0;
        for (int q = 0; q < w; ++q) before += warp_tot[q];
        int rank = before + __popc(ballot & ((1u << l) - 1u));
        if (hit && base + rank < cap) out[base + rank] = i;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot += warp_tot[q];
            base += tot;
        }
        __syncthreads();
    }
}

}  // namespace sc

using namespace sc;

extern "C" {

int sc_spmv_f64(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int32_t* col,
                const double* vals, const double* x, double* y, int deterministic,
                sc_stream_t stream) {
    if (n_rows < 0 || n_cols < 0) return fail(SC_ERR_VALUE, "negative dimension");
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    int64_t nnz = 0;
    if (n_rows > 0) SC_CUDA(d2h_sync(&nnz, row_ptr + n_rows, sizeof(int64_t), st));
    return spmv_launch(n_rows, nnz, row_ptr, col, vals, x, y, deterministic != 0, st);
}

int sc_degrees_f64(int64_t n, const int64_t* row_ptr, const double* vals, double* d,
                   sc_stream_t stream) {
    if (n < 0) return fail(SC_ERR_VALUE, "negative dimension");
    return degrees_launch(n, row_ptr, vals, d, as_stream(stream));
}

int sc_find_nonpositive(int64_t n, const double* d, int mode, int64_t* count_out,
                        int64_t* idx_out, int64_t max_idx, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    *count_out = 0;
    if (n <= 0) return SC_OK;
    DevBuf<unsigned long long> cnt;
    if (int rc = cnt.alloc(1)) return rc;
    SC_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
    count_nonpositive_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d, mode, cnt.p);
    SC_LAUNCHED(1);
    unsigned long long h = 0;
    SC_CUDA(d2h_sync(&h, cnt.p, sizeof(h), st));
    *count_out = (int64_t)h;
    if (h > 0 && idx_out && max_idx > 0) {
        list_nonpositive_kernel<<<1, 1024, 0, st>>>(n, d, mode, idx_out, max_idx);
        SC_LAUNCHED(1);
        SC_CUDA(cudaStreamSynchronize(st));
    }
    return SC_OK;
}

int sc_sym_scale_f64(int64_t n, const int64_t* row_ptr, const int32_t* col,
                     const double* vals, const double* d, double* out, sc_stream_t stream) {
    if (n <= 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    sym_scale_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, col, vals, d, out);
    SC_LAUNCHED(1);
    return SC_OK;
}

int sc_sym_scale_shard_f64(int64_t n_local, int64_t row_offset, const int64_t* row_ptr, const int32_t* col,
                           const double* vals, const double* d_global, double* out, sc_stream_t stream) {
    if (n_local <= 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    sym_scale_kernel<<<(unsigned)ceil_div(n_local, 8), 256, 0, st>>>(n_local, row_ptr, col, vals, d_global, out,
                                                                     row_offset);
    SC_LAUNCHED(1);
    return SC_OK;
}

}  // extern "C"

// CSR container invariants (sparse.py:83-142 CsrMatrix checks) on the device:
// row_ptr non-decreasing inside [0, nnz], columns in [0, n_cols) and strictly
// increasing within a row, values finite.  Warp per row; the first violation
// of each kind is counted (flags[0..3]).
__global__ void __launch_bounds__(256) csr_validate_kernel(int64_t n, int64_t n_cols, int64_t nnz,
                                                           const int64_t* __restrict__ row_ptr,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ vals,
                                                           unsigned long long* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (row >= n) return;
    const int64_t a = row_ptr[row], b = row_ptr[row + 1];
    if (a > b || a < 0 || b > nnz) {
        if (lane == 0) atomicAdd(&flags[0], 1ull);
        return;
    }
    bool bad_range = false, bad_order = false, bad_val = false;
    for (int64_t e = a + lane; e < b; e += 32) {
        const int32_t c = col[e];
        bad_range |= c < 0 || (int64_t)c >= n_cols;
        bad_order |= e > a && col[e - 1] >= c;
        bad_val |= !isfinite(vals[e]);
    }
    bad_range = __any_sync(0xffffffffu, bad_range);
    bad_order = __any_sync(0xffffffffu, bad_order);
    bad_val = __any_sync(0xffffffffu, bad_val);
    if (lane == 0) {
        if (bad_range) atomicAdd(&flags[1], 1ull);
        if (bad_order) atomicAdd(&flags[2], 1ull);
        if (bad_val) atomicAdd(&flags[3], 1ull);
    }
}

extern "C" {

int sc_csr_validate(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                    const double* vals, sc_stream_t stream) {
    if (n_rows < 0 || n_cols < 0 || nnz < 0) return fail(SC_ERR_FORMAT, "negative CSR dimension");
    if (n_cols > INT32_MAX) return fail(SC_ERR_FORMAT, "device CSR columns must fit int32");
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    int64_t ends[2] = {0, 0};
    SC_CUDA(d2h_sync(&ends[0], row_ptr, sizeof(int64_t), st));
    SC_CUDA(d2h_sync(&ends[1], row_ptr + n_rows, sizeof(int64_t), st));
    if (ends[0] != 0 || ends[1] != nnz) return fail(SC_ERR_FORMAT, "row_ptr must start at 0 and end at nnz");
    if (n_rows == 0) return SC_OK;
    DevBuf<unsigned long long> flags;
    if (int rc = flags.alloc(4)) return rc;
    SC_CUDA(cudaMemsetAsync(flags.p, 0, 4 * sizeof(unsigned long long), st));
    csr_validate_kernel<<<(unsigned)ceil_div(n_rows, 8), 256, 0, st>>>(n_rows, n_cols, nnz, row_ptr, col, vals,
                                                                       flags.p);
    SC_LAUNCHED(1);
    unsigned long long h[4];
    SC_CUDA(d2h_sync(h, flags.p, sizeof(h), st));
    if (h[0]) return fail(SC_ERR_FORMAT, "row_ptr must be non-decreasing");
    if (h[1]) return fail(SC_ERR_FORMAT, "column index out of range");
    if (h[2]) return fail(SC_ERR_FORMAT, "column indices must strictly increase within rows");
    if (h[3]) return fail(SC_ERR_FORMAT, "values must be finite");
    return SC_OK;
}

int sc_csr_is_symmetric(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                        const double* vals, int* result, sc_stream_t stream) {
    (void)nnz;
    *result = 1;
    if (n <= 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    DevBuf<int> bad;
    DevBuf<unsigned long long> ul;
    if (int rc = bad.alloc(1)) return rc;
    if (int rc = ul.alloc(2)) return rc;
    SC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    SC_CUDA(cudaMemsetAsync(ul.p, 0, 2 * sizeof(unsigned long long), st));
    symmetric_check_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, col, vals, bad.p, ul.p);
    SC_LAUNCHED(1);
    int h = 0;
    unsigned long long hul[2] = {0, 0};
    SC_CUDA(d2h_sync(&h, bad.p, sizeof(int), st));
    SC_CUDA(d2h_sync(hul, ul.p, sizeof(hul), st));
    *result = (h || hul[0] != hul[1]) ? 0 : 1;
    return SC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Symmetric permutation B = P A P^T of a CSR matrix: row p of B is row perm[p]
// of A with every column c relabelled pos[c] (pos = perm^-1) and the row
// re-sorted.  The eigensolver runs on the locality-ordered operator so the
// SpMV gathers of x hit nearby cache lines (stage 2).
#include "sc_scan.cuh"

namespace sc {
__global__ void perm_row_len_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ perm,
                                    int64_t* __restrict__ len) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t i = perm[p];
    len[p] = row_ptr[i + 1] - row_ptr[i];
}

// warp per output row: rows of <= 64 entries are sorted by their new column
// with a register bitonic network (2 keys per lane, key = new column << 32 |
// source slot, all keys distinct), rows of <= PERM_SMEM by a bitonic sort in
// shared memory; longer rows are listed for perm_long_kernel
__device__ __forceinline__ int64_t cas64(int64_t v, int64_t o, bool keep_min) {
    return keep_min ? (v < o ? v : o) : (v > o ? v : o);
}
constexpr int PERM_SMEM = 512;  // rows up to this length sort in shared memory (8 warps x 4 KB)
__global__ void __launch_bounds__(256) perm_row_fill_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                     const double* __restrict__ vals, const int32_t* __restrict__ perm,
                                     const int32_t* __restrict__ pos, const int64_t* __restrict__ out_ptr,
                                     int32_t* __restrict__ out_col, double* __restrict__ out_vals,
                                     int64_t* __restrict__ long_rows, unsigned int* __restrict__ nlong) {
    __shared__ int64_t perm_keys[8][PERM_SMEM];
    const int64_t p = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (p >= n) return;
    const int64_t i = perm[p];
    const int64_t b = row_ptr[i], len = row_ptr[i + 1] - b, o = out_ptr[p];
    if (len <= 64) {
        int64_t v0 = lane < len ? ((int64_t)pos[col[b + lane]] << 32) | lane : INT64_MAX;
        int64_t v1 = lane + 32 < len ? ((int64_t)pos[col[b + lane + 32]] << 32) | (lane + 32) : INT64_MAX;
#pragma unroll
        for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                if (j == 32) {  // partners are the two keys of this lane
                    const bool up = (lane & k) == 0;  // k == 64: always ascending
                    const int64_t lo = v0 < v1 ? v0 : v1, hi = v0 < v1 ? v1 : v0;
                    v0 = up ? lo : hi;
                    v1 = up ? hi : lo;
                } else {
                    const int64_t o0 = __shfl_xor_sync(0xffffffffu, v0, j);
                    const int64_t o1 = __shfl_xor_sync(0xffffffffu, v1, j);
                    const bool lower = (lane & j) == 0;
                    v0 = cas64(v0, o0, lower == ((lane & k) == 0));
                    v1 = cas64(v1, o1, lower == (((lane + 32) & k) == 0));
                }
            }
        }
        if (lane < len) {
            out_col[o + lane] = (int32_t)(v0 >> 32);
            out_vals[o + lane] = vals[b + (int32_t)(v0 & 0xffffffff)];
        }
        if (lane + 32 < len) {
            out_col[o + lane + 32] = (int32_t)(v1 >> 32);
            out_vals[o + lane + 32] = vals[b + (int32_t)(v1 & 0xffffffff)];
        }
        return;
    }
    if (len <= PERM_SMEM) {
        // shared-memory bitonic sort of the keys, padded to a power of two
        int64_t* K = perm_keys[threadIdx.x / 32];
        int np2 = 128;
        while (np2 < len) np2 <<= 1;
        for (int e = lane; e < np2; e += 32) K[e] = e < len ? ((int64_t)pos[col[b + e]] << 32) | e : INT64_MAX;
        __syncwarp();
        for (int k = 2; k <= np2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int q = lane; q < np2; q += 32) {
                    const int pq = q ^ j;
                    if (pq > q) {
                        const int64_t a = K[q], c = K[pq];
                        if ((a > c) == ((q & k) == 0)) {
                            K[q] = c;
                            K[pq] = a;
                        }
                    }
                }
                __syncwarp();
            }
        for (int e = lane; e < len; e += 32) {
            const int64_t v = K[e];
            out_col[o + e] = (int32_t)(v >> 32);
            out_vals[o + e] = vals[b + (int32_t)(v & 0xffffffff)];
        }
        return;
    }
    if (lane == 0) long_rows[atomicAdd(nlong, 1u)] = p;  // perm_long_kernel
}

// rows longer than PERM_SMEM (hubs), a block per row: bitonic sort of up to
// PERM_LONG keys in (dynamic) shared memory, counting beyond
constexpr int PERM_LONG = 8192;
__global__ void __launch_bounds__(512) perm_long_kernel(const int64_t* __restrict__ row_ptr,
                                                        const int32_t* __restrict__ col,
                                                        const double* __restrict__ vals,
                                                        const int32_t* __restrict__ perm,
                                                        const int32_t* __restrict__ pos,
                                                        const int64_t* __restrict__ out_ptr,
                                                        int32_t* __restrict__ out_col, double* __restrict__ out_vals,
                                                        const int64_t* __restrict__ long_rows,
                                                        const unsigned int* __restrict__ nlong) {
    extern __shared__ int64_t K[];
    const int tid = threadIdx.x;
    const unsigned nrows = *nlong;
    for (unsigned f = blockIdx.x; f < nrows; f += gridDim.x) {
        const int64_t p = long_rows[f];
        const int64_t i = perm[p];
        const int64_t b = row_ptr[i], len = row_ptr[i + 1] - b, o = out_ptr[p];
        __syncthreads();
        if (len <= PERM_LONG) {
            int np2 = 1;
            while (np2 < len) np2 <<= 1;
            for (int e = tid; e < np2; e += blockDim.x)
                K[e] = e < len ? ((int64_t)pos[col[b + e]] << 32) | e : INT64_MAX;
            __syncthreads();
            for (int k = 2; k <= np2; k <<= 1)
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int q = tid; q < np2; q += blockDim.x) {
                        const int pq = q ^ j;
                        if (pq > q) {
                            const int64_t a = K[q], c = K[pq];
                            if ((a > c) == ((q & k) == 0)) {
                                K[q] = c;
                                K[pq] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
            for (int e = tid; e < len; e += blockDim.x) {
                const int64_t v = K[e];
                out_col[o + e] = (int32_t)(v >> 32);
                out_vals[o + e] = vals[b + (int32_t)(v & 0xffffffff)];
            }
        } else {
            for (int64_t e = tid; e < len; e += blockDim.x) {
                const int32_t key = pos[col[b + e]];
                int64_t r = 0;
                for (int64_t q = 0; q < len; ++q) r += pos[col[b + q]] < key;
                out_col[o + r] = key;
                out_vals[o + r] = vals[b + e];
            }
        }
    }
}
}  // namespace sc

extern "C" int sc_csr_permute_f64(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                                  const int32_t* perm, const int32_t* pos, int64_t* out_row_ptr, int32_t* out_col,
                                  double* out_vals, sc_stream_t stream) {
    using namespace sc;
    if (n <= 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    DevBuf<int64_t> len, tmp;
    int rc;
    if ((rc = len.alloc(n)) || (rc = tmp.alloc(ceil_div(n, SCAN_BLK) + 1))) return rc;
    perm_row_len_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, row_ptr, perm, len.p);
    SC_LAUNCHED(1);
    if ((rc = exclusive_scan_i64(n, len.p, out_row_ptr, tmp.p, st))) return rc;
    DevBuf<int64_t> long_rows;
    DevBuf<unsigned int> nlong;
    if ((rc = long_rows.alloc(n)) || (rc = nlong.alloc(1))) return rc;
    SC_CUDA(cudaMemsetAsync(nlong.p, 0, sizeof(unsigned int), st));
    perm_row_fill_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, col, vals, perm, pos, out_row_ptr,
                                                                   out_col, out_vals, long_rows.p, nlong.p);
    constexpr int long_smem = PERM_LONG * (int)sizeof(int64_t);
    SC_CUDA(cudaFuncSetAttribute(perm_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, long_smem));
    perm_long_kernel<<<(unsigned)(2 * kNumSMs), 512, long_smem, st>>>(row_ptr, col, vals, perm, pos, out_row_ptr,
                                                                       out_col, out_vals, long_rows.p, nlong.p);
    SC_LAUNCHED(2);
    return SC_OK;
}

// pos[perm[p]] = p
namespace sc {
__global__ void invert_perm_kernel(int64_t n, const int32_t* __restrict__ perm, int32_t* __restrict__ pos) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) pos[perm[p]] = (int32_t)p;
}
// dst row r = src row idx[r] (row-major n x k)
__global__ void gather_rows_kernel(int64_t n, int64_t k, const double* __restrict__ src, const int32_t* __restrict__ idx,
                                   double* __restrict__ dst) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * k) return;
    const int64_t r = e / k, c = e - r * k;
    dst[e] = src[(int64_t)idx[r] * k + c];
}
}  // namespace sc

extern "C" int sc_invert_perm(int64_t n, const int32_t* perm, int32_t* pos, sc_stream_t stream) {
    using namespace sc;
    if (n <= 0) return SC_OK;
    invert_perm_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, perm, pos);
    SC_LAUNCHED(1);
    return SC_OK;
}

extern "C" int sc_gather_rows_f64(int64_t n, int64_t k, const double* src, const int32_t* idx, double* dst,
                                  sc_stream_t stream) {
    using namespace sc;
    if (n <= 0 || k <= 0) return SC_OK;
    gather_rows_kernel<<<(unsigned)ceil_div(n * k, 256), 256, 0, as_stream(stream)>>>(n, k, src, idx, dst);
    SC_LAUNCHED(1);
    return SC_OK;
}

// ---------------------------------------------------------------------------
// SELL-32-sigma (see sc_sparse.cuh)
namespace sc {
// one block per window of SELL_SIGMA rows: rank rows by (length desc, row asc)
__global__ void __launch_bounds__(SELL_SIGMA) sell_sort_kernel(int64_t n, int64_t lcap,
                                                               const int64_t* __restrict__ row_ptr,
                                                               int32_t* __restrict__ srow, int32_t* __restrict__ slen,
                                                               int32_t* __restrict__ lrows,
                                                               unsigned long long* __restrict__ nlong) {
    __shared__ int32_t L[SELL_SIGMA];
    const int64_t r = (int64_t)blockIdx.x * SELL_SIGMA + threadIdx.x;
    int64_t full = r < n ? row_ptr[r + 1] - row_ptr[r] : -1;
    if (full > lcap) {  // hub row: empty in the slices, listed for the long-row kernel
        lrows[atomicAdd(nlong, 1ull)] = (int32_t)r;
        full = 0;
    }
    const int32_t len = (int32_t)full;
    L[threadIdx.x] = len;
    __syncthreads();
    int rank = 0;
    for (int u = 0; u < SELL_SIGMA; ++u) {
        const int32_t lu = L[u];
        rank += (lu > len) || (lu == len && u < (int)threadIdx.x);
    }
    const int64_t o = (int64_t)blockIdx.x * SELL_SIGMA + rank;
    srow[o] = (int32_t)r;
    slen[o] = len < 0 ? 0 : len;
}

__global__ void sell_width_kernel(int64_t nslices, const int32_t* __restrict__ slen, int32_t* __restrict__ width,
                                  int64_t* __restrict__ size) {
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nslices) return;
    const int32_t w = slen[s * 32];  // longest row of the slice (sorted descending)
    width[s] = w;
    size[s] = (int64_t)w * 32;
}

// warp per slice
__global__ void sell_fill_kernel(int64_t nslices, const int64_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ col_in, const double* __restrict__ vals_in,
                                 const int64_t* __restrict__ slice_ptr, const int32_t* __restrict__ width,
                                 const int32_t* __restrict__ srow, const int32_t* __restrict__ slen,
                                 int32_t* __restrict__ col, double* __restrict__ vals) {
    const int64_t s = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int t = threadIdx.x & 31;
    if (s >= nslices) return;
    const int64_t idx = s * 32 + t;
    const int32_t len = slen[idx];
    const int64_t src = len > 0 ? row_ptr[srow[idx]] : 0;
    const int64_t base = slice_ptr[s] + t;
    const int32_t w = width[s];
    for (int32_t j = 0; j < w; ++j) {
        const bool in = j < len;
        col[base + (int64_t)j * 32] = in ? col_in[src + j] : 0;
        vals[base + (int64_t)j * 32] = in ? vals_in[src + j] : 0.0;
    }
}

// warp per slice, lane per row; the block's 8 slices are one sorting window
__global__ void __launch_bounds__(256) spmv_sell_kernel(int64_t n, int64_t nslices,
                                                        const int64_t* __restrict__ slice_ptr,
                                                        const int32_t* __restrict__ width,
                                                        const int32_t* __restrict__ srow,
                                                        const int32_t* __restrict__ slen,
                                                        const int32_t* __restrict__ col,
                                                        const double* __restrict__ vals,
                                                        const double* __restrict__ x, double* __restrict__ y) {
    const int64_t s = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int t = threadIdx.x & 31;
    if (s >= nslices) return;
    const int64_t idx = s * 32 + t;
    const int32_t len = slen[idx];
    const int32_t w = width[s];
    const int32_t* c = col + slice_ptr[s] + t;
    const double* v = vals + slice_ptr[s] + t;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int32_t j = 0;
    for (; j + 4 <= w; j += 4) {
        // every lane issues its loads for 4 entries before the first use
        int32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        if (j < len) { c0 = __ldg(c + (int64_t)j * 32); v0 = __ldg(v + (int64_t)j * 32); }
        if (j + 1 < len) { c1 = __ldg(c + (int64_t)(j + 1) * 32); v1 = __ldg(v + (int64_t)(j + 1) * 32); }
        if (j + 2 < len) { c2 = __ldg(c + (int64_t)(j + 2) * 32); v2 = __ldg(v + (int64_t)(j + 2) * 32); }
        if (j + 3 < len) { c3 = __ldg(c + (int64_t)(j + 3) * 32); v3 = __ldg(v + (int64_t)(j + 3) * 32); }
        if (j < len) a0 = fma(v0, __ldg(x + c0), a0);
        if (j + 1 < len) a1 = fma(v1, __ldg(x + c1), a1);
        if (j + 2 < len) a2 = fma(v2, __ldg(x + c2), a2);
        if (j + 3 < len) a3 = fma(v3, __ldg(x + c3), a3);
    }
    for (; j < w; ++j)
        if (j < len) a0 = fma(__ldg(v + (int64_t)j * 32), __ldg(x + __ldg(c + (int64_t)j * 32)), a0);
    const int32_t r = srow[idx];
    if (r < n) y[r] = (a0 + a1) + (a2 + a3);
}

// warp per long row (after spmv_sell_kernel, which wrote 0 for it)
__global__ void __launch_bounds__(256) spmv_long_rows_kernel(int64_t nlong, const int32_t* __restrict__ lrows,
                                                             const int64_t* __restrict__ row_ptr,
                                                             const int32_t* __restrict__ col,
                                                             const double* __restrict__ vals,
                                                             const double* __restrict__ x, double* __restrict__ y) {
    const int64_t q = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= nlong) return;
    const int32_t r = lrows[q];
    const int64_t b = row_ptr[r], e = row_ptr[r + 1];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t p = b + lane;
    for (; p + 96 < e; p += 128) {
        const int32_t c0 = __ldg(col + p), c1 = __ldg(col + p + 32), c2 = __ldg(col + p + 64), c3 = __ldg(col + p + 96);
        const double v0 = __ldg(vals + p), v1 = __ldg(vals + p + 32), v2 = __ldg(vals + p + 64),
                     v3 = __ldg(vals + p + 96);
        a0 = fma(v0, __ldg(x + c0), a0);
        a1 = fma(v1, __ldg(x + c1), a1);
        a2 = fma(v2, __ldg(x + c2), a2);
        a3 = fma(v3, __ldg(x + c3), a3);
    }
    for (; p < e; p += 32) a0 = fma(__ldg(vals + p), __ldg(x + __ldg(col + p)), a0);
    double acc = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) y[r] = acc;
}

int SellMatrix::build(int64_t n_, const int64_t* row_ptr_in, const int32_t* col_in, const double* vals_in,
                      cudaStream_t st) {
    n = n_;
    row_ptr = row_ptr_in;
    csr_col = col_in;
    csr_vals = vals_in;
    const int64_t nwin = ceil_div(n, SELL_SIGMA);
    nslices = nwin * (SELL_SIGMA / 32);
    int64_t nnz = 0;
    SC_CUDA(d2h_sync(&nnz, row_ptr + n, sizeof(int64_t), st));
    // hub threshold: twice the mean row length (at least 64)
    lcap = std::max<int64_t>(64, 2 * ceil_div(nnz, std::max<int64_t>(n, 1)));
    DevBuf<int64_t> size, tmp;
    DevBuf<unsigned long long> cnt;
    int rc;
    if ((rc = slice_ptr.alloc(nslices + 1)) || (rc = width.alloc(nslices)) || (rc = srow.alloc(nslices * 32)) ||
        (rc = slen.alloc(nslices * 32)) || (rc = size.alloc(nslices)) || (rc = lrows.alloc(n)) ||
        (rc = cnt.alloc(1)) || (rc = tmp.alloc(ceil_div(nslices, SCAN_BLK) + 1)))
        return rc;
    SC_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
    sell_sort_kernel<<<(unsigned)nwin, SELL_SIGMA, 0, st>>>(n, lcap, row_ptr, srow.p, slen.p, lrows.p, cnt.p);
    sell_width_kernel<<<(unsigned)ceil_div(nslices, 256), 256, 0, st>>>(nslices, slen.p, width.p, size.p);
    SC_LAUNCHED(2);
    if ((rc = exclusive_scan_i64(nslices, size.p, slice_ptr.p, tmp.p, st))) return rc;
    unsigned long long hl = 0;
    SC_CUDA(d2h_sync(&stored, slice_ptr.p + nslices, sizeof(int64_t), st));
    SC_CUDA(d2h_sync(&hl, cnt.p, sizeof(hl), st));
    nlong = (int64_t)hl;
    if ((rc = col.alloc(std::max<int64_t>(stored, 1))) || (rc = vals.alloc(std::max<int64_t>(stored, 1)))) return rc;
    sell_fill_kernel<<<(unsigned)ceil_div(nslices, 8), 256, 0, st>>>(nslices, row_ptr_in, col_in, vals_in, slice_ptr.p,
                                                                    width.p, srow.p, slen.p, col.p, vals.p);
    SC_LAUNCHED(1);
    return SC_OK;
}

int SellMatrix::spmv(const double* x, double* y, cudaStream_t st) const {
    if (n == 0) return SC_OK;
    ProfScope prof("spmv", st, 12.0 * (double)stored + 8.0 * 4.0 * (double)n);  // + long rows (small)
    spmv_sell_kernel<<<(unsigned)ceil_div(nslices, 8), 256, 0, st>>>(n, nslices, slice_ptr.p, width.p, srow.p, slen.p,
                                                                     col.p, vals.p, x, y);
    SC_LAUNCHED(1);
    if (nlong > 0) {
        spmv_long_rows_kernel<<<(unsigned)ceil_div(nlong, 8), 256, 0, st>>>(nlong, lrows.p, row_ptr, csr_col, csr_vals,
                                                                            x, y);
        SC_LAUNCHED(1);
    }
    return SC_OK;
}
}  // namespace sc

// ---- C ABI: SELL operator handle (built once, applied many times) ----------
struct sc_sell {
    sc::SellMatrix m;
};
extern "C" int sc_sell_create(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                              sc_stream_t stream, sc_sell** out) {
    using namespace sc;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    auto* h = new sc_sell();
    if (int rc = h->m.build(n, row_ptr, col, vals, st)) {
        delete h;
        return rc;
    }
    *out = h;
    return SC_OK;
}
extern "C" int sc_sell_spmv(const sc_sell* h, const double* x, double* y, sc_stream_t stream) {
    return h->m.spmv(x, y, sc::as_stream(stream));
}
extern "C" int sc_sell_info(const sc_sell* h, int64_t* stored, int64_t* nlong) {
    *stored = h->m.stored;
    *nlong = h->m.nlong;
    return SC_OK;
}
extern "C" void sc_sell_destroy(sc_sell* h) { delete h; }

// ---------------------------------------------------------------------------
// Bulk-staged SpMV (see SpmvPlan in sc_sparse.cuh).
#include "sc_tc.cuh"

namespace sc {

// chunk c = the rows whose first nonzero index lies in [c*CH, (c+1)*CH)
__device__ __forceinline__ int64_t first_row_at_or_after(const int64_t* __restrict__ row_ptr, int64_t n, int64_t p) {
    int64_t lo = 0, hi = n + 1;  // first r in [0, n] with row_ptr[r] >= p (n if none)
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (row_ptr[mid] < p) lo = mid + 1; else hi = mid;
    }
    return lo > n ? n : lo;
}

__global__ void spmv_plan_kernel(int64_t n, int64_t nnz, int64_t nch, const int64_t* __restrict__ row_ptr,
                                 SpmvChunk* __restrict__ chunks) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const int64_t ra = first_row_at_or_after(row_ptr, n, c * SPMV_CH);
    const int64_t rb = c + 1 == nch ? n : first_row_at_or_after(row_ptr, n, (c + 1) * SPMV_CH);
    SpmvChunk ch;
    ch.row_begin = ra;
    ch.row_end = rb;
    ch.p_begin = row_ptr[ra];
    ch.p_end = row_ptr[rb];
    // staged iff it fits the stage and the 16-byte-rounded bulk reads stay
    // inside the arrays (only the matrix tail can fail the latter)
    const int64_t pa = ch.p_begin & ~3ll, pv = ch.p_begin & ~1ll, rr = ra & ~1ll;
    const int64_t ncol = (ch.p_end - pa + 3) & ~3ll, nval = (ch.p_end - pv + 1) & ~1ll,
                  nrp = (rb + 1 - rr + 1) & ~1ll;
    ch.staged = ch.p_end - ch.p_begin <= SPMV_CAP && rb - ra <= SPMV_RCAP && pa + ncol <= nnz && pv + nval <= nnz &&
                rr + nrp <= n + 1;
    chunks[c] = ch;
}

struct SpmvStage {
    int32_t col[SPMV_CAP + 4];
    double vals[SPMV_CAP + 2];
    int64_t rp[SPMV_RCAP + 2];
};

// one CTA per SM: warp 0 streams chunk after chunk of (col, vals, row_ptr)
// into a SPMV_STAGES-deep shared-memory ring with cp.async.bulk (completion on
// the stage's mbarrier); warps 1.. consume the staged chunk G lanes per row,
// gather x (L1 / L2) and write y, then release the stage.  The CTA's chunks
// are one contiguous range, so in locality order its x window stays in L1.
template <int G>
__global__ void __launch_bounds__(SPMV_THREADS, 1) spmv_bulk_kernel(int64_t n, int64_t nch,
                                                                    const SpmvChunk* __restrict__ chunks,
                                                                    const int64_t* __restrict__ row_ptr,
                                                                    const int32_t* __restrict__ col,
                                                                    const double* __restrict__ vals,
                                                                    const double* __restrict__ x,
                                                                    double* __restrict__ y) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SpmvStage* stages = reinterpret_cast<SpmvStage*>(smem_raw);
    __shared__ uint64_t full[SPMV_STAGES], empty[SPMV_STAGES];
    __shared__ SpmvChunk hdr[SPMV_STAGES];
    constexpr int NCW = SPMV_THREADS / 32 - 1;  // consumer warps
    constexpr int RPW = 32 / G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c0 = nch * blockIdx.x / gridDim.x, c1 = nch * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SPMV_STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], NCW);
        }
        tc::fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane != 0) return;
        for (int64_t c = c0; c < c1; ++c) {
            const int64_t i = c - c0;
            const int s = (int)(i % SPMV_STAGES);
            tc::mbar_wait(&empty[s], (uint32_t)(((i / SPMV_STAGES) & 1) ^ 1));
            const SpmvChunk ch = chunks[c];
            hdr[s] = ch;
            if (ch.staged && ch.p_end > ch.p_begin) {
                const int64_t pa = ch.p_begin & ~3ll, pv = ch.p_begin & ~1ll, rr = ch.row_begin & ~1ll;
                const uint32_t bc = (uint32_t)(((ch.p_end - pa + 3) & ~3ll) * 4);
                const uint32_t bv = (uint32_t)(((ch.p_end - pv + 1) & ~1ll) * 8);
                const uint32_t br = (uint32_t)(((ch.row_end + 1 - rr + 1) & ~1ll) * 8);
                tc::mbar_expect_tx(&full[s], bc + bv + br);
                tc::bulk_g2s(stages[s].col, col + pa, bc, &full[s]);
                tc::bulk_g2s(stages[s].vals, vals + pv, bv, &full[s]);
                tc::bulk_g2s(stages[s].rp, row_ptr + rr, br, &full[s]);
            } else {
                tc::mbar_arrive(&full[s]);  // direct chunk: consumers read global memory
            }
        }
        return;
    }
    const int cw = warp - 1, sl = lane % G;
    for (int64_t c = c0; c < c1; ++c) {
        const int64_t i = c - c0;
        const int s = (int)(i % SPMV_STAGES);
        tc::mbar_wait(&full[s], (uint32_t)((i / SPMV_STAGES) & 1));
        const SpmvChunk ch = hdr[s];
        const SpmvStage& st = stages[s];
        const bool staged = ch.staged != 0;
        const int64_t pa = ch.p_begin & ~3ll, pv = ch.p_begin & ~1ll, rr = ch.row_begin & ~1ll;
        for (int64_t base = ch.row_begin + (int64_t)cw * RPW; base < ch.row_end; base += (int64_t)NCW * RPW) {
            const int64_t row = base + lane / G;
            const bool valid = row < ch.row_end;
            int64_t p = 0, e = 0;
            if (valid) {
                if (staged) {
                    p = st.rp[row - rr];
                    e = st.rp[row + 1 - rr];
                } else {
                    p = row_ptr[row];
                    e = row_ptr[row + 1];
                }
            }
            p += sl;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            if (staged) {
                for (; p + 3 * G < e; p += 4 * G) {
                    const int32_t q0 = st.col[p - pa], q1 = st.col[p + G - pa], q2 = st.col[p + 2 * G - pa],
                                  q3 = st.col[p + 3 * G - pa];
                    a0 = fma(st.vals[p - pv], __ldg(x + q0), a0);
                    a1 = fma(st.vals[p + G - pv], __ldg(x + q1), a1);
                    a2 = fma(st.vals[p + 2 * G - pv], __ldg(x + q2), a2);
                    a3 = fma(st.vals[p + 3 * G - pv], __ldg(x + q3), a3);
                }
                for (; p < e; p += G) a0 = fma(st.vals[p - pv], __ldg(x + st.col[p - pa]), a0);
            } else {
                for (; p < e; p += G) a0 = fma(__ldg(vals + p), __ldg(x + __ldg(col + p)), a0);
            }
            double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
            if (valid && sl == 0) y[row] = acc;
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[s]);
    }
}

int SpmvPlan::build(int64_t n_, const int64_t* row_ptr_, const int32_t* col_, const double* vals_, cudaStream_t st) {
    n = n_;
    row_ptr = row_ptr_;
    col = col_;
    vals = vals_;
    nnz = 0;
    if (n > 0) {
        SC_CUDA(d2h_sync(&nnz, row_ptr + n, sizeof(int64_t), st));
    }
    nch = std::max<int64_t>(1, ceil_div(nnz, SPMV_CH));
    int rc;
    if ((rc = chunks.alloc(nch))) return rc;
    if (n > 0) {
        spmv_plan_kernel<<<(unsigned)ceil_div(nch, 256), 256, 0, st>>>(n, nnz, nch, row_ptr, chunks.p);
        SC_LAUNCHED(1);
    }
    return SC_OK;
}

int SpmvPlan::apply(const double* x, double* y, cudaStream_t st) const {
    if (n == 0) return SC_OK;
    const double mean = (double)nnz / (double)n;
    if (spmv_kind() != 9 || mean <= 8) return spmv_launch(n, nnz, row_ptr, col, vals, x, y, false, st);
    ProfScope prof("spmv", st, (double)nnz * 12.0 + (double)(n + 1) * 8.0 + 2.0 * (double)n * 8.0);
    const size_t smem = sizeof(SpmvStage) * SPMV_STAGES;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(spmv_bulk_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const int64_t grid = std::min<int64_t>(kNumSMs, nch);
    spmv_bulk_kernel<8><<<(unsigned)grid, SPMV_THREADS, smem, st>>>(n, nch, chunks.p, row_ptr, col, vals, x, y);
    SC_LAUNCHED(1);
    return SC_OK;
}

}  // namespace sc

// ---- C ABI: SpMV plan handle (built once per operator, applied per matvec) --
struct sc_spmv_plan {
    sc::SpmvPlan p;
};
extern "C" int sc_spmv_plan_create(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                                   sc_stream_t stream, sc_spmv_plan** out) {
    using namespace sc;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    auto* h = new sc_spmv_plan();
    if (int rc = h->p.build(n, row_ptr, col, vals, st)) {
        delete h;
        return rc;
    }
    *out = h;
    return SC_OK;
}
extern "C" int sc_spmv_plan_apply(const sc_spmv_plan* h, const double* x, double* y, sc_stream_t stream) {
    return h->p.apply(x, y, sc::as_stream(stream));
}
extern "C" void sc_spmv_plan_destroy(sc_spmv_plan* h) { delete h; }

// ---------------------------------------------------------------------------
// Input cleaning and row scaling (laplacian.py:34-81)
namespace sc {
__global__ void keep_flags_kernel(int64_t n, const double* __restrict__ d, int64_t* __restrict__ flag) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = d[i] != 0.0;
}
// remap[i] = new index of node i (exclusive scan of keep flags) or -1
__global__ void remap_kernel(int64_t n, const double* __restrict__ d, const int64_t* __restrict__ scan,
                             int64_t* __restrict__ remap, double* __restrict__ d_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (d[i] != 0.0) {
        remap[i] = scan[i];
        d_out[scan[i]] = d[i];
    } else {
        remap[i] = -1;
    }
}
// kept entries per kept row (warp per row)
__global__ void induced_count_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                     const int64_t* __restrict__ remap, int64_t* __restrict__ len) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (i >= n || remap[i] < 0) return;
    int64_t c = 0;
    for (int64_t p = row_ptr[i] + lane; p < row_ptr[i + 1]; p += 32) c += remap[col[p]] >= 0;
    c = warp_sum_i64(c);
    if (lane == 0) len[remap[i]] = c;
}
// entries of kept rows with kept columns, order preserved (warp ballot scan)
__global__ void induced_fill_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                    const double* __restrict__ vals, const int64_t* __restrict__ remap,
                                    const int64_t* __restrict__ out_ptr, int32_t* __restrict__ out_col,
                                    double* __restrict__ out_vals) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (i >= n || remap[i] < 0) return;
    int64_t o = out_ptr[remap[i]];
    for (int64_t p0 = row_ptr[i]; p0 < row_ptr[i + 1]; p0 += 32) {
        const int64_t p = p0 + lane;
        const int64_t rc = p < row_ptr[i + 1] ? remap[col[p]] : -1;
        const unsigned m = __ballot_sync(0xffffffffu, rc >= 0);
        if (rc >= 0) {
            const int64_t q = o + __popc(m & ((1u << lane) - 1u));
            out_col[q] = (int32_t)rc;
            out_vals[q] = vals[p];
        }
        o += __popc(m);
    }
}
__global__ void row_scale_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const double* __restrict__ vals,
                                 const double* __restrict__ d, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (i >= n) return;
    const double di = d[i];
    for (int64_t p = row_ptr[i] + (threadIdx.x & 31); p < row_ptr[i + 1]; p += 32) out[p] = __ddiv_rn(vals[p], di);
}
}  // namespace sc

// Induced submatrix on the nonzero-degree nodes (handle_isolated 'remove'):
// outputs are caller-allocated with the input sizes (n + 1, nnz, n); the new
// sizes come back in *n_new / *nnz_new.
extern "C" int sc_csr_remove_isolated(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                                      const double* d, int64_t* remap, int64_t* out_row_ptr, int32_t* out_col,
                                      double* out_vals, double* out_d, int64_t* n_new, int64_t* nnz_new,
                                      sc_stream_t stream) {
    using namespace sc;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    *n_new = 0;
    *nnz_new = 0;
    if (n <= 0) return SC_OK;
    DevBuf<int64_t> flag, scan, len, tmp;
    int rc;
    if ((rc = flag.alloc(n)) || (rc = scan.alloc(n + 1)) || (rc = len.alloc(n)) ||
        (rc = tmp.alloc(ceil_div(n, SCAN_BLK) + 1)))
        return rc;
    keep_flags_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d, flag.p);
    SC_LAUNCHED(1);
    if ((rc = exclusive_scan_i64(n, flag.p, scan.p, tmp.p, st))) return rc;
    SC_CUDA(cudaMemcpyAsync(n_new, scan.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    remap_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d, scan.p, remap, out_d);
    induced_count_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, col, remap, len.p);
    SC_LAUNCHED(2);
    SC_CUDA(cudaStreamSynchronize(st));
    if (*n_new == 0) {
        SC_CUDA(cudaMemsetAsync(out_row_ptr, 0, sizeof(int64_t), st));
        SC_CUDA(cudaStreamSynchronize(st));
        return SC_OK;
    }
    if ((rc = exclusive_scan_i64(*n_new, len.p, out_row_ptr, tmp.p, st))) return rc;
    induced_fill_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, col, vals, remap, out_row_ptr, out_col,
                                                                  out_vals);
    SC_LAUNCHED(1);
    SC_CUDA(d2h_sync(nnz_new, out_row_ptr + *n_new, sizeof(int64_t), st));
    return SC_OK;
}

// out[p] = vals[p] / d[row(p)] (row_scale, laplacian.py:75-81; IEEE division,
// bit-identical to the reference)
extern "C" int sc_row_scale_f64(int64_t n, const int64_t* row_ptr, const double* vals, const double* d, double* out,
                                sc_stream_t stream) {
    using namespace sc;
    if (n <= 0) return SC_OK;
    row_scale_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, as_stream(stream)>>>(n, row_ptr, vals, d, out);
    SC_LAUNCHED(1);
    return SC_OK;
}
