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
