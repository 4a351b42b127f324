// CSR kernels: SpMV (sequential-order and vectorised), degrees, symmetric
// scaling, exact symmetry check, non-positive degree search.
//
// Device CSR layout: row_ptr int64[n+1],
// col int32[nnz] (n < 2^31), vals f64[nnz]; rows sorted, columns strictly
// increasing within a row (sparse.py:110-138).
#include <cstdlib>

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

int spmv_launch(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                const double* vals, const double* x, double* y, bool deterministic,
                cudaStream_t st) {
    if (n == 0) return SC_OK;
    double bytes = (double)nnz * 12.0 + (double)(n + 1) * 8.0 + 2.0 * (double)n * 8.0;
    ProfScope prof(deterministic ? "spmv_seq" : "spmv", st, bytes);
    if (deterministic) {
        spmv_seq_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, row_ptr, col, vals, x, y);
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
__global__ void symmetric_check_kernel(int64_t n, const int64_t* __restrict__ row_ptr,
                                       const int32_t* __restrict__ col,
                                       const double* __restrict__ vals, int* __restrict__ bad) {
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (i >= n) return;
    for (int64_t p = row_ptr[i] + (threadIdx.x & 31), e = row_ptr[i + 1]; p < e; p += 32) {
        int64_t j = col[p];
        int64_t lo = row_ptr[j], hi = row_ptr[j + 1];
        // binary search for column i in row j
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (col[mid] < i) lo = mid + 1; else hi = mid;
        }
        if (lo >= row_ptr[j + 1] || col[lo] != i || !(vals[lo] == vals[p])) atomicOr(bad, 1);
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
    if (n_rows > 0) SC_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SC_CUDA(cudaStreamSynchronize(st));
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
    SC_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    SC_CUDA(cudaStreamSynchronize(st));
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

int sc_csr_is_symmetric(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                        const double* vals, int* result, sc_stream_t stream) {
    (void)nnz;
    *result = 1;
    if (n <= 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    DevBuf<int> bad;
    if (int rc = bad.alloc(1)) return rc;
    SC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    symmetric_check_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, col, vals, bad.p);
    SC_LAUNCHED(1);
    int h = 0;
    SC_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    SC_CUDA(cudaStreamSynchronize(st));
    *result = h ? 0 : 1;
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

// warp per output row; entries ranked by their new column (distinct keys)
__global__ void perm_row_fill_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                     const double* __restrict__ vals, const int32_t* __restrict__ perm,
                                     const int32_t* __restrict__ pos, const int64_t* __restrict__ out_ptr,
                                     int32_t* __restrict__ out_col, double* __restrict__ out_vals) {
    const int64_t p = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (p >= n) return;
    const int64_t i = perm[p];
    const int64_t b = row_ptr[i], len = row_ptr[i + 1] - b, o = out_ptr[p];
    for (int64_t e = lane; e < len; e += 32) {
        const int32_t key = pos[col[b + e]];
        int64_t r = 0;
        for (int64_t f = 0; f < len; ++f) r += pos[col[b + f]] < key;
        out_col[o + r] = key;
        out_vals[o + r] = vals[b + e];
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
    perm_row_fill_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, col, vals, perm, pos, out_row_ptr,
                                                                   out_col, out_vals);
    SC_LAUNCHED(1);
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
    SC_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SC_CUDA(cudaStreamSynchronize(st));
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
    SC_CUDA(cudaMemcpyAsync(&stored, slice_ptr.p + nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SC_CUDA(cudaMemcpyAsync(&hl, cnt.p, sizeof(hl), cudaMemcpyDeviceToHost, st));
    SC_CUDA(cudaStreamSynchronize(st));
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
