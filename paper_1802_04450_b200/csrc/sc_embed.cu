// Spectral embedding: v = u / sqrt(d) rowwise, unit columns, optional unit
// rows (laplacian.py:94-106; pipeline.py:242-245).  Row-major n x k.
#include "sc_common.cuh"

namespace sc {

constexpr int EMB_ROWS = 256;  // rows per column-norm partial block

// out = u / sqrt(d) (rowwise) and per-block column sums of squares
__global__ void emb_scale_kernel(int64_t n, int64_t k, const double* __restrict__ u,
                                 const double* __restrict__ d, double* __restrict__ out,
                                 double* __restrict__ part) {
    // block: 256 threads; columns strided by thread, rows [r0, r0 + EMB_ROWS)
    int64_t r0 = (int64_t)blockIdx.x * EMB_ROWS;
    int64_t r1 = imin64(n, r0 + EMB_ROWS);
    for (int64_t c = threadIdx.x; c < k; c += blockDim.x) {
        double acc = 0.0;
        for (int64_t r = r0; r < r1; ++r) {
            double x = __ddiv_rn(u[r * k + c], __dsqrt_rn(d[r]));
            out[r * k + c] = x;
            acc = __dadd_rn(acc, __dmul_rn(x, x));
        }
        part[blockIdx.x * k + c] = acc;
    }
}

__global__ void emb_colnorm_kernel(int64_t nb, int64_t k, const double* __restrict__ part,
                                   double* __restrict__ norms) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k) return;
    double acc = 0.0;
    for (int64_t b = 0; b < nb; ++b) acc = __dadd_rn(acc, part[b * k + c]);
    double nv = __dsqrt_rn(acc);
    norms[c] = nv == 0.0 ? 1.0 : nv;  // laplacian.py:105 norms[norms == 0] = 1
}

__global__ void emb_colsum_kernel(int64_t nb, int64_t k, const double* __restrict__ part, double* __restrict__ colsq) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k) return;
    double acc = 0.0;
    for (int64_t b = 0; b < nb; ++b) acc = __dadd_rn(acc, part[b * k + c]);
    colsq[c] = acc;
}

__global__ void emb_norms_from_sq_kernel(int64_t k, const double* __restrict__ colsq, double* __restrict__ norms) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k) return;
    double nv = __dsqrt_rn(colsq[c]);
    norms[c] = nv == 0.0 ? 1.0 : nv;
}

// divide by column norms, then (optionally) each row by its 2-norm; warp per row
__global__ void emb_finish_kernel(int64_t n, int64_t k, const double* __restrict__ norms,
                                  int normalize_rows, double* __restrict__ out) {
    int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (r >= n) return;
    double* row = out + r * k;
    double acc = 0.0;
    for (int64_t c = lane; c < k; c += 32) {
        double x = __ddiv_rn(row[c], norms ? norms[c] : 1.0);
        row[c] = x;
        acc = fma(x, x, acc);
    }
    if (!normalize_rows) return;
    acc = warp_sum(acc);
    double rn = sqrt(acc);
    if (rn == 0.0) rn = 1.0;  // pipeline.py:244
    for (int64_t c = lane; c < k; c += 32) row[c] = __ddiv_rn(row[c], rn);
}

// column-major input (element (r, c) at u[c * ld + r]): the column sums of
// squares of u / sqrt(d) in emb_scale_kernel's order, without the output
__global__ void emb_colsq_cm_kernel(int64_t n, int64_t k, int64_t ld, const double* __restrict__ u,
                                    const double* __restrict__ d, double* __restrict__ part) {
    int64_t r0 = (int64_t)blockIdx.x * EMB_ROWS;
    int64_t r1 = imin64(n, r0 + EMB_ROWS);
    for (int64_t c = threadIdx.x; c < k; c += blockDim.x) {
        double acc = 0.0;
        for (int64_t r = r0; r < r1; ++r) {
            double x = __ddiv_rn(u[c * ld + r], __dsqrt_rn(d[r]));
            acc = __dadd_rn(acc, __dmul_rn(x, x));
        }
        part[blockIdx.x * k + c] = acc;
    }
}

// out (row-major n x k) = u (column-major) / sqrt(d) rowwise: 32 x 32 tiles
// through shared memory (coalesced on both sides)
__global__ void emb_transpose_scale_kernel(int64_t n, int64_t k, int64_t ld, const double* __restrict__ u,
                                           const double* __restrict__ d, double* __restrict__ out) {
    __shared__ double t[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    for (int cc = threadIdx.y; cc < 32; cc += blockDim.y) {
        const int64_t r = r0 + threadIdx.x, c = c0 + cc;
        if (r < n && c < k) t[cc][threadIdx.x] = __ddiv_rn(u[c * ld + r], __dsqrt_rn(d[r]));
    }
    __syncthreads();
    for (int rr = threadIdx.y; rr < 32; rr += blockDim.y) {
        const int64_t r = r0 + rr, c = c0 + threadIdx.x;
        if (r < n && c < k) out[r * k + c] = t[threadIdx.x][rr];
    }
}

}  // namespace sc

using namespace sc;

extern "C" {

int sc_recover_embedding(int64_t n, int64_t k, const double* u, const double* d,
                         int normalize_rows, double* out, sc_stream_t stream) {
    if (n < 0 || k < 0) return fail(SC_ERR_VALUE, "negative dimension");
    if (n == 0 || k == 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    int64_t nb = ceil_div(n, EMB_ROWS);
    DevBuf<double> part, norms;
    int rc;
    if ((rc = part.alloc(nb * k)) || (rc = norms.alloc(k))) return rc;
    ProfScope prof("embed", st, 3.0 * n * k * 8.0);
    emb_scale_kernel<<<(unsigned)nb, 256, 0, st>>>(n, k, u, d, out, part.p);
    emb_colnorm_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, st>>>(nb, k, part.p, norms.p);
    emb_finish_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, k, norms.p, normalize_rows, out);
    SC_LAUNCHED(3);
    SC_CUDA(cudaStreamSynchronize(st));
    return SC_OK;
}

// sc_recover_embedding for eigenvectors stored column-major with leading
// dimension ld (the Lanczos basis columns, sc_eigensolve_csr_basis); out is
// row-major n x k and must not overlap u.  Bit-identical to
// sc_recover_embedding on the same values.
int sc_recover_embedding_cm(int64_t n, int64_t k, const double* u, int64_t ld, const double* d, int normalize_rows,
                            double* out, sc_stream_t stream) {
    if (n < 0 || k < 0 || ld < n) return fail(SC_ERR_VALUE, "bad dimensions");
    if (n == 0 || k == 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    int64_t nb = ceil_div(n, EMB_ROWS);
    DevBuf<double> part, norms;
    int rc;
    if ((rc = part.alloc(nb * k)) || (rc = norms.alloc(k))) return rc;
    ProfScope prof("embed", st, 4.0 * n * k * 8.0);
    emb_colsq_cm_kernel<<<(unsigned)nb, 256, 0, st>>>(n, k, ld, u, d, part.p);
    emb_colnorm_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, st>>>(nb, k, part.p, norms.p);
    emb_transpose_scale_kernel<<<dim3((unsigned)ceil_div(n, 32), (unsigned)ceil_div(k, 32)), dim3(32, 8), 0, st>>>(
        n, k, ld, u, d, out);
    emb_finish_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, k, norms.p, normalize_rows, out);
    SC_LAUNCHED(4);
    SC_CUDA(cudaStreamSynchronize(st));
    return SC_OK;
}

// Row-sharded embedding: phase 1 scales the local rows and returns their
// column sums of squares (dev k; all-reduced by the caller), phase 2 divides
// by the global column norms and optionally normalises rows.
int sc_embed_scale(int64_t n, int64_t k, const double* u, const double* d, double* out, double* colsq,
                   sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    if (k <= 0) return SC_OK;
    if (n <= 0) {
        SC_CUDA(cudaMemsetAsync(colsq, 0, sizeof(double) * k, st));
        return SC_OK;
    }
    int64_t nb = ceil_div(n, EMB_ROWS);
    DevBuf<double> part;
    if (int rc = part.alloc(nb * k)) return rc;
    emb_scale_kernel<<<(unsigned)nb, 256, 0, st>>>(n, k, u, d, out, part.p);
    emb_colsum_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, st>>>(nb, k, part.p, colsq);
    SC_LAUNCHED(2);
    return SC_OK;
}

int sc_embed_finish(int64_t n, int64_t k, const double* colsq, int normalize_rows, double* out, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    if (n <= 0 || k <= 0) return SC_OK;
    DevBuf<double> norms;
    if (int rc = norms.alloc(k)) return rc;
    emb_norms_from_sq_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, st>>>(k, colsq, norms.p);
    emb_finish_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, k, norms.p, normalize_rows, out);
    SC_LAUNCHED(2);
    return SC_OK;
}

int sc_normalize_rows(int64_t n, int64_t k, const double* v, double* out, sc_stream_t stream) {
    if (n <= 0 || k <= 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    if (out != v) SC_CUDA(cudaMemcpyAsync(out, v, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, st));
    emb_finish_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, k, nullptr, 1, out);
    SC_LAUNCHED(1);
    return SC_OK;
}

}  // extern "C"
