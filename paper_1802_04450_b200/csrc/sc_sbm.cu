// Planted-partition stochastic block model generated straight into CSR on
// the device (reference sbm.py:68-108).
//
// The reference draws, per block pair, a Binomial(pair count, p) edge count
// and a uniform subset of that size -- distributionally identical to an
// independent coin per unordered pair.  Here every row i flips the coins of
// its pairs (i, j > i) by geometric skipping (Philox stream keyed by
// (seed, i)): with probability p_in inside i's block, p_out beyond it, the
// gap to the next edge is floor(log u / log(1 - p)); by memorylessness the
// walk restarts at the block boundary.  Work is O(edges), so the C4 graph
// (16M nodes, ~512M edges) never materialises the reference's triu_indices.
// The upper triangle is emitted row by row (columns ascending), mirrored
// into the lower triangle through per-row counters, and each row's lower
// segment is sorted, giving a canonical symmetric unit-weight CSR.
// Deterministic for a given seed (the counter-based stream does not depend
// on scheduling); the numpy stream of the reference is not reproduced.
#include <algorithm>
#include <cmath>

#include "sc_common.cuh"
#include "sc_scan.cuh"

namespace sc {

// uniform in (0, 1] from the Philox block (row, step) of `seed`
__device__ __forceinline__ double philox_u01(uint64_t seed, uint64_t row, uint64_t step) {
    uint4 c = make_uint4((uint32_t)step, (uint32_t)(step >> 32), (uint32_t)row, (uint32_t)(row >> 32) ^ 0x5B3Du);
    uint2 k = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    uint4 r = Philox::gen(c, k);
    const uint64_t a = ((uint64_t)r.x << 21) ^ ((uint64_t)r.y >> 11);
    return ((double)(a & ((1ull << 53) - 1)) + 1.0) * (1.0 / 9007199254740992.0);
}

struct SbmRow {
    int64_t i, own_end, n;
    double lq_in, lq_out;  // log(1 - p); 0 when p == 0 (no edges), -inf when p == 1
    bool in_zero, out_zero;
};

// visit the upper-triangle edges (i, j > i) of row i in ascending j
template <class F>
__device__ __forceinline__ void sbm_walk(const SbmRow& r, uint64_t seed, F emit) {
    uint64_t step = 0;
    // own block (p_in), then the rest (p_out)
    for (int seg = 0; seg < 2; ++seg) {
        const bool zero = seg == 0 ? r.in_zero : r.out_zero;
        const double lq = seg == 0 ? r.lq_in : r.lq_out;
        int64_t j = seg == 0 ? r.i + 1 : r.own_end;
        const int64_t end = seg == 0 ? r.own_end : r.n;
        if (zero) continue;
        while (true) {
            // gap ~ Geometric(p) on {0, 1, ...}: number of failures before a success
            const double u = philox_u01(seed, (uint64_t)r.i, step++);
            const double g = isinf(lq) ? 0.0 : floor(log(u) / lq);
            if (g >= (double)(end - j)) break;
            j += (int64_t)g;
            emit(j);
            ++j;
            if (j >= end) break;
        }
    }
}

__device__ __forceinline__ SbmRow sbm_row(int64_t i, int64_t n, const int64_t* __restrict__ offsets, int64_t nblocks,
                                          double p_in, double p_out) {
    // block of i: binary search in offsets[0..nblocks]
    int64_t lo = 0, hi = nblocks;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (offsets[mid] <= i) lo = mid; else hi = mid;
    }
    SbmRow r;
    r.i = i;
    r.n = n;
    r.own_end = offsets[lo + 1];
    r.in_zero = !(p_in > 0.0);
    r.out_zero = !(p_out > 0.0);
    r.lq_in = p_in >= 1.0 ? -INFINITY : log1p(-p_in);
    r.lq_out = p_out >= 1.0 ? -INFINITY : log1p(-p_out);
    return r;
}

__global__ void sbm_count_kernel(int64_t n, const int64_t* __restrict__ offsets, int64_t nblocks, double p_in,
                                 double p_out, uint64_t seed, int64_t* __restrict__ up_cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const SbmRow r = sbm_row(i, n, offsets, nblocks, p_in, p_out);
    int64_t c = 0;
    sbm_walk(r, seed, [&](int64_t) { ++c; });
    up_cnt[i] = c;
}

__global__ void sbm_fill_upper_kernel(int64_t n, const int64_t* __restrict__ offsets, int64_t nblocks, double p_in,
                                      double p_out, uint64_t seed, const int64_t* __restrict__ up_ptr,
                                      int32_t* __restrict__ up_col, unsigned int* __restrict__ low_cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const SbmRow r = sbm_row(i, n, offsets, nblocks, p_in, p_out);
    int64_t o = up_ptr[i];
    sbm_walk(r, seed, [&](int64_t j) {
        up_col[o++] = (int32_t)j;
        atomicAdd(low_cnt + j, 1u);
    });
}

__global__ void sbm_row_len_kernel(int64_t n, const int64_t* __restrict__ up_ptr,
                                   const unsigned int* __restrict__ low_cnt, int64_t* __restrict__ len,
                                   unsigned int* __restrict__ maxlow) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    len[i] = (int64_t)low_cnt[i] + (up_ptr[i + 1] - up_ptr[i]);
    atomicMax(maxlow, low_cnt[i]);
}

// row i = [lower entries (unsorted for now)][upper entries (ascending)]
__global__ void sbm_scatter_kernel(int64_t n, const int64_t* __restrict__ up_ptr, const int32_t* __restrict__ up_col,
                                   const unsigned int* __restrict__ low_cnt, const int64_t* __restrict__ row_ptr,
                                   unsigned int* __restrict__ cursor, int32_t* __restrict__ col,
                                   double* __restrict__ vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t base = row_ptr[i] + low_cnt[i];
    for (int64_t p = up_ptr[i]; p < up_ptr[i + 1]; ++p) {
        const int32_t j = up_col[p];
        col[base + (p - up_ptr[i])] = j;
        vals[base + (p - up_ptr[i])] = 1.0;
        const unsigned int slot = atomicAdd(cursor + j, 1u);
        col[row_ptr[j] + slot] = (int32_t)i;
        vals[row_ptr[j] + slot] = 1.0;
    }
}

// sort each row's lower segment: warp per row for <= 64 entries (registers);
// longer rows are appended to `longs` for sbm_sort_long_kernel
__global__ void sbm_sort_lower_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                      const unsigned int* __restrict__ low_cnt, int32_t* __restrict__ col,
                                      int64_t* __restrict__ longs, unsigned int* __restrict__ nlong) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    int32_t* c = col + row_ptr[i];
    const int len = (int)low_cnt[i];
    if (len <= 1) return;
    if (len > 64) {
        if (lane == 0) longs[atomicAdd(nlong, 1u)] = i;
        return;
    }
    int32_t v0 = lane < len ? c[lane] : INT32_MAX;
    int32_t v1 = lane + 32 < len ? c[lane + 32] : INT32_MAX;
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {
                const bool up = (lane & k) == 0;
                const int32_t lo = min(v0, v1), hi = max(v0, v1);
                v0 = up ? lo : hi;
                v1 = up ? hi : lo;
            } else {
                const int32_t o0 = __shfl_xor_sync(0xffffffffu, v0, j);
                const int32_t o1 = __shfl_xor_sync(0xffffffffu, v1, j);
                const bool lower = (lane & j) == 0;
                const bool a0 = lower == ((lane & k) == 0), a1 = lower == (((lane + 32) & k) == 0);
                v0 = a0 ? min(v0, o0) : max(v0, o0);
                v1 = a1 ? min(v1, o1) : max(v1, o1);
            }
        }
    }
    __syncwarp();
    if (lane < len) c[lane] = v0;
    if (lane + 32 < len) c[lane + 32] = v1;
}

// one CTA per long row (any length): shared-memory bitonic sort up to
// kSbmSmemSort entries, rank counting (distinct values) beyond
constexpr int kSbmSmemSort = 16384;
__global__ void __launch_bounds__(1024) sbm_sort_long_kernel(const int64_t* __restrict__ longs,
                                                             const unsigned int* __restrict__ nlong,
                                                             const int64_t* __restrict__ row_ptr,
                                                             const unsigned int* __restrict__ low_cnt,
                                                             int32_t* __restrict__ col, int32_t* __restrict__ scratch) {
    extern __shared__ int32_t sk[];
    for (unsigned int t = blockIdx.x; t < *nlong; t += gridDim.x) {
        const int64_t i = longs[t];
        int32_t* c = col + row_ptr[i];
        const int len = (int)low_cnt[i];
        if (len <= kSbmSmemSort) {
            int np2 = 1;
            while (np2 < len) np2 <<= 1;
            for (int e = threadIdx.x; e < np2; e += blockDim.x) sk[e] = e < len ? c[e] : INT32_MAX;
            __syncthreads();
            for (int size = 2; size <= np2; size <<= 1)
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int q = threadIdx.x; q < np2 / 2; q += blockDim.x) {
                        const int lo = 2 * q - (q & (stride - 1)), hi = lo + stride;
                        const bool up = (lo & size) == 0;
                        const int32_t a = sk[lo], b = sk[hi];
                        if ((a > b) == up) {
                            sk[lo] = b;
                            sk[hi] = a;
                        }
                    }
                    __syncthreads();
                }
            for (int e = threadIdx.x; e < len; e += blockDim.x) c[e] = sk[e];
        } else {
            // sources of one row are distinct: rank = number of smaller ones
            int32_t* out = scratch + row_ptr[i];
            for (int e = threadIdx.x; e < len; e += blockDim.x) {
                const int32_t v = c[e];
                int r = 0;
                for (int f = 0; f < len; ++f) r += c[f] < v;
                out[r] = v;
            }
            __syncthreads();
            for (int e = threadIdx.x; e < len; e += blockDim.x) c[e] = out[e];
        }
        __syncthreads();
    }
}

}  // namespace sc

using namespace sc;

extern "C" {

// Two calls: with col == NULL the total nnz comes back in *nnz_out (host);
// then with caller-allocated row_ptr (n+1), col / vals (nnz) (dev).  offsets
// (dev int64, nblocks + 1): block boundaries.  Any row length.
int sc_sbm_csr(int64_t n, const int64_t* offsets, int64_t nblocks, double p_in, double p_out, uint64_t seed,
               int64_t* row_ptr, int32_t* col, double* vals, int64_t* nnz_out, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    *nnz_out = 0;
    if (n <= 0) return SC_OK;
    if (!(0.0 <= p_out && p_out <= p_in && p_in <= 1.0)) return fail(SC_ERR_VALUE, "need 0 <= p_out <= p_in <= 1");
    if (n >= (int64_t)INT32_MAX) return fail(SC_ERR_VALUE, "n must be < 2^31");
    DevBuf<int64_t> up_cnt, up_ptr, len, tmp;
    int rc;
    if ((rc = up_cnt.alloc(n)) || (rc = up_ptr.alloc(n + 1)) || (rc = tmp.alloc(ceil_div(n, SCAN_BLK) + 1))) return rc;
    sbm_count_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, offsets, nblocks, p_in, p_out, seed, up_cnt.p);
    SC_LAUNCHED(1);
    if ((rc = exclusive_scan_i64(n, up_cnt.p, up_ptr.p, tmp.p, st))) return rc;
    int64_t nup = 0;
    SC_CUDA(d2h_sync(&nup, up_ptr.p + n, sizeof(int64_t), st));
    *nnz_out = 2 * nup;
    if (!col) return SC_OK;
    DevBuf<int32_t> up_col;
    DevBuf<unsigned int> low_cnt, cursor;
    if ((rc = up_col.alloc(std::max<int64_t>(nup, 1))) || (rc = low_cnt.alloc(n)) || (rc = cursor.alloc(n)) ||
        (rc = len.alloc(n)))
        return rc;
    SC_CUDA(cudaMemsetAsync(low_cnt.p, 0, sizeof(unsigned int) * n, st));
    SC_CUDA(cudaMemsetAsync(cursor.p, 0, sizeof(unsigned int) * n, st));
    DevBuf<unsigned int> maxlow;
    if ((rc = maxlow.alloc(1))) return rc;
    SC_CUDA(cudaMemsetAsync(maxlow.p, 0, sizeof(unsigned int), st));
    sbm_fill_upper_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, offsets, nblocks, p_in, p_out, seed, up_ptr.p,
                                                                      up_col.p, low_cnt.p);
    sbm_row_len_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, up_ptr.p, low_cnt.p, len.p, maxlow.p);
    SC_LAUNCHED(2);
    unsigned int hmax = 0;
    SC_CUDA(d2h_sync(&hmax, maxlow.p, sizeof(hmax), st));
    if ((rc = exclusive_scan_i64(n, len.p, row_ptr, tmp.p, st))) return rc;
    sbm_scatter_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, up_ptr.p, up_col.p, low_cnt.p, row_ptr, cursor.p,
                                                                   col, vals);
    // lower segments in ascending column order (unbounded length)
    DevBuf<int64_t> longs;
    DevBuf<unsigned int> nlong;
    DevBuf<int32_t> scratch;
    if ((rc = longs.alloc(n)) || (rc = nlong.alloc(1))) return rc;
    if (hmax > (unsigned)kSbmSmemSort && (rc = scratch.alloc(2 * nup + 1))) return rc;
    SC_CUDA(cudaMemsetAsync(nlong.p, 0, sizeof(unsigned int), st));
    sbm_sort_lower_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, low_cnt.p, col, longs.p, nlong.p);
    if (hmax > 64) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(sbm_sort_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSbmSmemSort * (int)sizeof(int32_t));
            attr = true;
        }
        sbm_sort_long_kernel<<<4 * kNumSMs, 1024, kSbmSmemSort * sizeof(int32_t), st>>>(longs.p, nlong.p, row_ptr,
                                                                                      low_cnt.p, col, scratch.p);
    }
    SC_LAUNCHED(2);
    SC_CUDA(cudaStreamSynchronize(st));
    return SC_OK;
}

}  // extern "C"
