// The graph stage's other measures and patterns:
//   * cosine / cross-correlation edge similarities over a given edge list
//     (graph.py:136-147, the paper's given-edge-list path),
//   * the epsilon-distance pattern (graph.py:160-176),
//   * the similarity-threshold pattern (graph.py:206-211).
//
// Numerics follow the reference's numpy primitives: row means in numpy's
// pairwise-sum order (x.mean(axis=1)), squared norms and dot products in the
// einsum order (NpDot, sc_common.cuh), one IEEE sqrt of the product of the
// squared norms and one division, then the clip.  Edge similarities and the
// eps pattern are therefore bit-identical to the reference; the threshold
// pattern is bit-identical for exp_decay up to the last-ulp difference of
// CUDA's exp at the threshold itself, and for cosine / cross-correlation it
// uses the einsum order where the reference forms the full n x n matrix with a
// BLAS GEMM (pairs within rounding of the threshold may differ).
#include <cmath>
#include <vector>

#include "sc_common.cuh"
#include "sc_scan.cuh"

namespace sc {

// xc = x - mean(x, axis=1) (centre = 1) or x; sq = einsum(xc, xc)
__global__ void centre_rows_kernel(int64_t n, int64_t d, const double* __restrict__ x, int centre,
                                   double* __restrict__ xc, double* __restrict__ sq) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* xi = x + i * d;
    double* oi = xc + i * d;
    // np.add.reduce starts from the identity: 0.0 + pairwise(row)
    const double mu = centre ? __ddiv_rn(__dadd_rn(0.0, np_pairwise_sum_dev(xi, d)), (double)d) : 0.0;
    for (int64_t l = 0; l < d; ++l) oi[l] = centre ? __dsub_rn(xi[l], mu) : xi[l];
    sq[i] = np_sqnorm(oi, d);
}

// smallest degenerate (zero-norm) point among the edge endpoints
__global__ void degenerate_kernel(int64_t m, const int64_t* __restrict__ pairs, const double* __restrict__ sq,
                                  unsigned long long* __restrict__ first) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * m) return;
    const int64_t i = pairs[t];
    if (sq[i] == 0.0) atomicMin(first, (unsigned long long)i);
}

__device__ __forceinline__ double np_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t d) {
    NpDot s;
    np_dot_span(s, 0, d, [&](int64_t l) { return __dmul_rn(a[l], b[l]); });
    return s.result();
}

// clip(dot / sqrt(sq_i * sq_j), -1, 1) (graph.py:145-147)
__device__ __forceinline__ double corr_value(const double* __restrict__ xc, const double* __restrict__ sq, int64_t d,
                                             int64_t i, int64_t j) {
    const double v = __ddiv_rn(np_dot(xc + i * d, xc + j * d, d), __dsqrt_rn(__dmul_rn(sq[i], sq[j])));
    return v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
}

__global__ void edge_corr_kernel(int64_t m, int64_t d, const int64_t* __restrict__ pairs,
                                 const double* __restrict__ xc, const double* __restrict__ sq, int policy,
                                 double* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    double v = corr_value(xc, sq, d, pairs[2 * t], pairs[2 * t + 1]);
    if (policy == 0) v = v > 0.0 ? v : 0.0;  // clamp_zero: np.maximum(v, 0.0)
    else if (policy == 1) v = fabs(v);       // abs
    out[t] = v;
}

// pattern predicate for the pair (i, j), i < j
//   mode 0: eps      d2(x_j - x_i) <= a            (a = eps^2)
//   mode 1: thr-exp  exp(b * d2(x - x_i)[j]) > a   (b = -1 / (2 sigma^2))
//   mode 2: thr-corr corr(i, j) > a on xc / sq
__device__ __forceinline__ bool pattern_hit(int mode, const double* __restrict__ x, const double* __restrict__ sq,
                                            int64_t d, int64_t i, int64_t j, double a, double b) {
    if (mode == 2) return corr_value(x, sq, d, i, j) > a;
    const double d2 = np_sqdist(x + j * d, x + i * d, d);
    return mode == 0 ? d2 <= a : exp(b * d2) > a;
}

// warp per row i: counts[i] = #{j > i : hit}
__global__ void pattern_count_kernel(int64_t n, int64_t d, const double* __restrict__ x,
                                     const double* __restrict__ sq, int mode, double a, double b,
                                     int64_t* __restrict__ counts) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    int64_t c = 0;
    for (int64_t j = i + 1 + lane; j < n; j += 32) c += pattern_hit(mode, x, sq, d, i, j, a, b);
    c = warp_sum_i64(c);
    if (lane == 0) counts[i] = c;
}

// warp per row i: the hits as (i, j) pairs, j ascending, from offsets[i]
__global__ void pattern_fill_kernel(int64_t n, int64_t d, const double* __restrict__ x,
                                    const double* __restrict__ sq, int mode, double a, double b,
                                    const int64_t* __restrict__ offsets, int64_t* __restrict__ pairs) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    int64_t o = offsets[i];
    for (int64_t j0 = i + 1; j0 < n; j0 += 32) {
        const int64_t j = j0 + lane;
        const bool hit = j < n && pattern_hit(mode, x, sq, d, i, j, a, b);
        const unsigned msk = __ballot_sync(0xffffffffu, hit);
        if (hit) {
            const int64_t q = o + __popc(msk & ((1u << lane) - 1u));
            pairs[2 * q] = i;
            pairs[2 * q + 1] = j;
        }
        o += __popc(msk);
    }
}

}  // namespace sc

using namespace sc;

extern "C" {

int sc_edge_similarity_f64(int64_t n, int64_t d, const double* x, int64_t m, const int64_t* pairs, int kind,
                           int negative_policy, double* out, int64_t* degenerate, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    *degenerate = -1;
    if (kind != 1 && kind != 2) return fail(SC_ERR_VALUE, "edge similarity kind must be 1 (cosine) or 2 (cross_correlation)");
    if (m <= 0 || n <= 0) return SC_OK;
    DevBuf<double> xc, sq;
    DevBuf<unsigned long long> first;
    int rc;
    if ((rc = xc.alloc((size_t)n * d)) || (rc = sq.alloc(n)) || (rc = first.alloc(1))) return rc;
    SC_CUDA(cudaMemsetAsync(first.p, 0xff, sizeof(unsigned long long), st));
    centre_rows_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(n, d, x, kind == 2, xc.p, sq.p);
    degenerate_kernel<<<(unsigned)ceil_div(2 * m, 256), 256, 0, st>>>(m, pairs, sq.p, first.p);
    SC_LAUNCHED(2);
    unsigned long long h = 0;
    SC_CUDA(d2h_sync(&h, first.p, sizeof(h), st));
    if (h != ~0ull) {
        *degenerate = (int64_t)h;
        return fail(SC_ERR_VALUE, "degenerate vector at point index " + std::to_string(h));
    }
    edge_corr_kernel<<<(unsigned)ceil_div(m, 128), 128, 0, st>>>(m, d, pairs, xc.p, sq.p, negative_policy, out);
    SC_LAUNCHED(1);
    SC_CUDA(cudaStreamSynchronize(st));
    return SC_OK;
}

// Pattern edges (i < j, row-major).  mode 0 eps (a = eps), 1 threshold with
// exp_decay (a = lambda, b = sigma), 2 threshold with cosine, 3 threshold with
// cross-correlation (a = lambda).  Two calls: pairs == NULL returns the edge
// count in *m_out; then the caller allocates pairs (m x 2 int64, dev) and calls
// again.  For modes 2-3 *degenerate receives the first zero-norm point.
int sc_pattern_edges_f64(int64_t n, int64_t d, const double* x, int mode, double a, double b, int64_t* pairs,
                         int64_t* m_out, int64_t* degenerate, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    *degenerate = -1;
    if (mode < 0 || mode > 3) return fail(SC_ERR_VALUE, "pattern mode must be 0..3");
    if (n <= 1) {
        *m_out = 0;
        return SC_OK;
    }
    DevBuf<double> xc, sq;
    DevBuf<int64_t> counts, offs, tmp;
    int rc;
    if ((rc = counts.alloc(n)) || (rc = offs.alloc(n + 1)) || (rc = tmp.alloc(ceil_div(n, SCAN_BLK) + 1))) return rc;
    const double* xs = x;
    int kmode = mode;
    double pa = a, pb = 0.0;
    if (mode == 0) {
        pa = a * a;  // graph.py:166: eps2 = eps * eps
    } else if (mode == 1) {
        pb = -1.0 / (2.0 * (b * b));  // graph.py:154: inv = -1.0 / (2.0 * sigma**2)
    } else {
        if ((rc = xc.alloc((size_t)n * d)) || (rc = sq.alloc(n))) return rc;
        centre_rows_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(n, d, x, mode == 3, xc.p, sq.p);
        SC_LAUNCHED(1);
        // the reference checks every point (graph.py:153: _check_nondegenerate(sq, kind))
        std::vector<double> hsq(n);
        SC_CUDA(d2h_sync(hsq.data(), sq.p, sizeof(double) * n, st));
        for (int64_t i = 0; i < n; ++i)
            if (hsq[i] == 0.0) {
                *degenerate = i;
                return fail(SC_ERR_VALUE, "degenerate vector at point index " + std::to_string(i));
            }
        xs = xc.p;
        kmode = 2;
    }
    pattern_count_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, d, xs, sq.p, kmode, pa, pb, counts.p);
    SC_LAUNCHED(1);
    if ((rc = exclusive_scan_i64(n, counts.p, offs.p, tmp.p, st))) return rc;
    SC_CUDA(d2h_sync(m_out, offs.p + n, sizeof(int64_t), st));
    if (!pairs || *m_out == 0) return SC_OK;
    pattern_fill_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, d, xs, sq.p, kmode, pa, pb, offs.p, pairs);
    SC_LAUNCHED(1);
    SC_CUDA(cudaStreamSynchronize(st));
    return SC_OK;
}

}  // extern "C"
