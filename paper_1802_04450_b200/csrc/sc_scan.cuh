// Device exclusive scan of int64 counts (used for CSR row pointers).
#pragma once
#include "sc_common.cuh"

namespace sc {

constexpr int SCAN_BLK = 1024;

static __global__ void scan_block_sums_kernel(int64_t n, const int64_t* __restrict__ in, int64_t* __restrict__ bsum) {
    __shared__ int64_t red[32];
    int64_t i = (int64_t)blockIdx.x * SCAN_BLK + threadIdx.x;
    int64_t v = i < n ? in[i] : 0;
    v = warp_sum_i64(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        int64_t t = red[threadIdx.x];
        t = warp_sum_i64(t);
        if (threadIdx.x == 0) bsum[blockIdx.x] = t;
    }
}

// single block: exclusive scan of nb block sums in place, total into *total
static __global__ void scan_top_kernel(int64_t nb, int64_t* __restrict__ bsum, int64_t* __restrict__ total) {
    __shared__ int64_t carry;
    __shared__ int64_t wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nb; base += blockDim.x) {
        int64_t i = base + threadIdx.x;
        int64_t v = i < nb ? bsum[i] : 0;
        // inclusive warp scan
        int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        int64_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            int64_t s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                int64_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        int64_t incl = x + (w > 0 ? wsum[w - 1] : 0) + carry;
        if (i < nb) bsum[i] = incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

static __global__ void scan_apply_kernel(int64_t n, const int64_t* __restrict__ in, const int64_t* __restrict__ boff,
                                  int64_t* __restrict__ out) {
    __shared__ int64_t wsum[32];
    int64_t i = (int64_t)blockIdx.x * SCAN_BLK + threadIdx.x;
    int64_t v = i < n ? in[i] : 0;
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t s = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        wsum[lane] = s;
    }
    __syncthreads();
    int64_t incl = x + (w > 0 ? wsum[w - 1] : 0) + boff[blockIdx.x];
    if (i < n) out[i] = incl - v;
}

// out[0..n] = exclusive scan of in[0..n), out[n] = total.  tmp >= ceil(n/1024)+1.
inline int exclusive_scan_i64(int64_t n, const int64_t* in, int64_t* out, int64_t* tmp, cudaStream_t st) {
    int64_t nb = ceil_div(n, SCAN_BLK);
    if (n == 0) {
        cudaMemsetAsync(out, 0, sizeof(int64_t), st);
        return SC_OK;
    }
    scan_block_sums_kernel<<<(unsigned)nb, SCAN_BLK, 0, st>>>(n, in, tmp);
    scan_top_kernel<<<1, 1024, 0, st>>>(nb, tmp, out + n);
    scan_apply_kernel<<<(unsigned)nb, SCAN_BLK, 0, st>>>(n, in, tmp, out);
    SC_LAUNCHED(3);
    return SC_OK;
}

}  // namespace sc
