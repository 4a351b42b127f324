// Thick-restart Lanczos on device (eigen.py:86-302), usable both through the
// reverse-communication session API (caller applies the operator) and as a
// device-resident eigensolve whose SpMV never leaves the GPU.
//
// Data layout: the Krylov basis B is column-major n x (m+1) fp64
// with leading dimension ld = round_up(n, 32) so every basis vector is a
// contiguous, 256-byte aligned array (it is both the SpMV input and a GEMV
// column).  The projected matrix T is m x m column-major.
//
// Per Lanczos step (reference: eigen.py:152-179):
//   h1 = B^T w (alpha = h1[j]);  w -= B h1;  [h2 = B^T w;  w -= B h2;]  beta = |w|
// i.e. a full classical Gram-Schmidt pass over the raw product, which subsumes
// the reference's three-term subtraction (eigen.py:160) — every component
// that subtraction removes is also removed by the full pass — and a second
// pass only when the first cancelled most of |w| (DGKS criterion, see
// advance()).  T, the breakdown rule, the convergence/verification logic and
// the thick restart follow eigen.py:166-239 exactly.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "sc_common.cuh"
#include "sc_sparse.cuh"
#include "sc_block.cuh"
#include "sc_dc.cuh"
#include "sc_symeig.cuh"
#include "sc_scan.cuh"

namespace sc {

constexpr int GT_ROWS = 2048;     // rows per gemv_t partial block (max)
constexpr int GN_THREADS = 256;   // rows per gemv_n block
constexpr double kBreakdownRtol = 1e-13;  // eigen.py:50
// windowed orthogonalisation only from this many rows on: below it the cost
// of the reference's full CGS2 is negligible, and tiny operators (many
// repeated / zero eigenvalues, exact breakdowns) are where a window's loss
// grows fastest (reference acceptance criteria 1 and 6)
constexpr int64_t kWindowMinN = 32768;
// convergence test of a sweep: est_i <= margin * tol * max(1, |theta_i|)
// (eigen.py:198-200 uses tol itself).  Below kWindowMinN rows margin =
// kConvMargin: the estimates come from a different start vector than
// numpy's, so the converged residuals land elsewhere in [0, tol], and a 4x
// margin keeps them clear of tol for the reference's row-operator acceptance
// check (residual of D^-1/2 u under D^-1 W, <= 1e-8) at negligible cost.
// From kWindowMinN rows on the reference's own test (margin 1): at C3h the
// 4x margin cost 10 of 21 restarts (all 1000 estimates were below tol from
// restart 11 on, one straggler hovered between 0.25 tol and tol)
constexpr double kConvMargin = 0.25;
// windowed mode: a window pass that leaves |w| below this fraction of its
// input norm has cancelled to rounding level -> two passes over the basis
constexpr double kWindowCancel = 1e-6;
// SELL-32-sigma matvecs are opt-in (SPECLUST_SPMV_FORMAT=sell): on the C2
// kNN operator the x gathers are L2-sector bound and the warp-per-row CSR
// kernel measured faster (161 vs 183 ms per 500 matvecs, profiles/)
constexpr int64_t kSellMinRows = INT64_MAX;
constexpr int64_t kMaxWindow = 16;
constexpr int64_t kMaxSweepWindow = 32;  // <= WCG_MAX - 8: the per-step window spans it

// ---- kernels ------------------------------------------------------------------
__global__ void fill_normal_kernel(int64_t n, uint64_t seed, uint64_t stream_id, double* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = philox_normal(seed, stream_id, (uint64_t)i);
}

// element i of a shard starting at global row `offset` (shard-independent draws)
__global__ void fill_normal_offset_kernel(int64_t n, int64_t offset, uint64_t seed, uint64_t stream_id,
                                          double* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = philox_normal(seed, stream_id, (uint64_t)(offset + i));
}

// part[b * ncols + c] = sum_{r in block b} B[c * ld + r] * w[r];
// optional sq_part[b] = sum_{r in block b} w[r]^2 (|w| before the projection)
__global__ void __launch_bounds__(256) gemv_t_partial_kernel(int64_t n, int64_t ld, int ncols, int rpb,
                                                             const double* __restrict__ B,
                                                             const double* __restrict__ w,
                                                             double* __restrict__ part,
                                                             double* __restrict__ sq_part) {
    // rpb rows per block (<= GT_ROWS); the grid is sized to one balanced wave
    // of kNumSMs x 8 blocks when n allows (Lanczos::init)
    __shared__ double ws[GT_ROWS];
    const int64_t r0 = (int64_t)blockIdx.x * rpb;
    const int rows = (int)imin64(rpb, n - r0);
    for (int i = threadIdx.x; i < rows; i += blockDim.x) ws[i] = w[r0 + i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (sq_part && warp == 0) {
        double s = 0.0;
        for (int t = lane; t < rows; t += 32) s = fma(ws[t], ws[t], s);
        s = warp_sum(s);
        if (lane == 0) sq_part[blockIdx.x] = s;
    }
    // two columns per warp pass (twice the loads in flight per warp, one
    // shuffle tree per column as before); per-column arithmetic unchanged
    int c = warp * 2;
    for (; c + 1 < ncols; c += 16) {
        const double* col = B + (int64_t)c * ld + r0;
        const double* col2 = col + ld;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
        int t = lane;
#pragma unroll 2
        for (; t + 96 < rows; t += 128) {
            const double x0 = __ldg(col + t), x1 = __ldg(col + t + 32), x2 = __ldg(col + t + 64),
                         x3 = __ldg(col + t + 96);
            const double y0 = __ldg(col2 + t), y1 = __ldg(col2 + t + 32), y2 = __ldg(col2 + t + 64),
                         y3 = __ldg(col2 + t + 96);
            const double w0 = ws[t], w1 = ws[t + 32], w2 = ws[t + 64], w3 = ws[t + 96];
            a0 = fma(x0, w0, a0);
            a1 = fma(x1, w1, a1);
            a2 = fma(x2, w2, a2);
            a3 = fma(x3, w3, a3);
            b0 = fma(y0, w0, b0);
            b1 = fma(y1, w1, b1);
            b2 = fma(y2, w2, b2);
            b3 = fma(y3, w3, b3);
        }
        for (; t < rows; t += 32) {
            a0 = fma(__ldg(col + t), ws[t], a0);
            b0 = fma(__ldg(col2 + t), ws[t], b0);
        }
        const double acc = warp_sum((a0 + a1) + (a2 + a3));
        const double acc2 = warp_sum((b0 + b1) + (b2 + b3));
        if (lane == 0) {
            part[blockIdx.x * (int64_t)ncols + c] = acc;
            part[blockIdx.x * (int64_t)ncols + c + 1] = acc2;
        }
    }
    if (c < ncols) {  // the odd last column
        const double* col = B + (int64_t)c * ld + r0;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int t = lane;
        for (; t + 96 < rows; t += 128) {
            a0 = fma(__ldg(col + t), ws[t], a0);
            a1 = fma(__ldg(col + t + 32), ws[t + 32], a1);
            a2 = fma(__ldg(col + t + 64), ws[t + 64], a2);
            a3 = fma(__ldg(col + t + 96), ws[t + 96], a3);
        }
        for (; t < rows; t += 32) a0 = fma(__ldg(col + t), ws[t], a0);
        const double acc = warp_sum((a0 + a1) + (a2 + a3));
        if (lane == 0) part[blockIdx.x * (int64_t)ncols + c] = acc;
    }
}

// rows per gemv_t block: one balanced wave at the kernel's real occupancy,
// 32-row granules
static int gemv_t_rows_per_block(int64_t n) {
    static int bps = 0;
    if (!bps) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, gemv_t_partial_kernel, 256, 0);
        if (bps < 1) bps = 1;
    }
    return (int)std::min<int64_t>(GT_ROWS, std::max<int64_t>(32, ceil_div(ceil_div(n, kNumSMs * bps), 32) * 32));
}

// h[c] = sum_b part[b * ncols + c] (fixed order), warp per column
__global__ void reduce_cols_kernel(int64_t nb, int ncols, const double* __restrict__ part,
                                   double* __restrict__ h) {
    int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    int lane = threadIdx.x & 31;
    if (c >= ncols) return;
    double acc = 0.0;
#pragma unroll 8
    for (int64_t b = lane; b < nb; b += 32) acc += part[b * ncols + c];
    acc = warp_sum(acc);
    if (lane == 0) h[c] = acc;
}

// w[r] -= sum_c B[c * ld + r] * h[c]; optional per-block sum of w_new^2
__global__ void __launch_bounds__(GN_THREADS) gemv_n_update_kernel(int64_t n, int64_t ld, int ncols,
                                                                   const double* __restrict__ B,
                                                                   const double* __restrict__ h,
                                                                   double* __restrict__ w,
                                                                   double* __restrict__ sq_part) {
    extern __shared__ double hs[];
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) hs[c] = h[c];
    __syncthreads();
    int64_t r = (int64_t)blockIdx.x * GN_THREADS + threadIdx.x;
    double v = 0.0;
    if (r < n) {
        const double* p = B + r;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int c = 0;
#pragma unroll 8
        for (; c + 4 <= ncols; c += 4) {  // unrolled: 32 column loads in flight per row
            a0 = fma(__ldg(p + (int64_t)c * ld), hs[c], a0);
            a1 = fma(__ldg(p + (int64_t)(c + 1) * ld), hs[c + 1], a1);
            a2 = fma(__ldg(p + (int64_t)(c + 2) * ld), hs[c + 2], a2);
            a3 = fma(__ldg(p + (int64_t)(c + 3) * ld), hs[c + 3], a3);
        }
        for (; c < ncols; ++c) a0 = fma(__ldg(p + (int64_t)c * ld), hs[c], a0);
        v = w[r] - ((a0 + a1) + (a2 + a3));
        w[r] = v;
    }
    if (sq_part) {
        __shared__ double red[GN_THREADS / 32];
        double s = warp_sum(v * v);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int i = 0; i < GN_THREADS / 32; ++i) t += red[i];
            sq_part[blockIdx.x] = t;
        }
    }
}

// Two classical Gram-Schmidt passes of w against the window columns
// B[:, lo .. lo+cnt) in ONE cooperative launch (the window is short: the
// per-step cost was launch latency, ~10 kernels):
//   h1 = Bw^T w;  w -= Bw h1;  h2 = Bw^T w;  w -= Bw h2;  beta = |w|
// with the second projection accumulated in the same row sweep as the first
// update (Bw read three times, not four).  Fixed-order reductions (every
// block sums the per-block partials in block order), so the result does not
// depend on scheduling.  Outputs: T[j,j] = scal[2] = alpha = h1[cnt-1]
// (q_j is the last window column), scal[0] = |w|, scal[3] = |w0|.
#define WCG_BLOCK_REDUCE_STORE(ACC, NCOL)                                       \
    do {                                                                        \
        _Pragma("unroll") for (int c_ = 0; c_ <= NC; ++c_) {                    \
            if (c_ < (NCOL)) {                                                  \
                const double v_ = warp_sum(ACC[c_]);                            \
                if (lane == 0) red[warp][c_] = v_;                              \
            }                                                                   \
        }                                                                       \
        __syncthreads();                                                        \
        for (int c_ = threadIdx.x; c_ < (NCOL); c_ += blockDim.x) {             \
            double t_ = 0.0;                                                    \
            for (int q_ = 0; q_ < 8; ++q_) t_ += red[q_][c_];                   \
            part[(int64_t)blockIdx.x * stride + c_] = t_;                       \
        }                                                                       \
        __syncthreads();                                                        \
    } while (0)
constexpr int WCG_MAX = 40;
template <int NC>
__global__ void __launch_bounds__(256) window_cgs2_kernel(int64_t n, int64_t ld, const double* __restrict__ Bw, int cnt,
                                                          double* __restrict__ w, double* __restrict__ part,
                                                          int64_t m, int64_t j, double* __restrict__ T,
                                                          double* __restrict__ scal) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    constexpr int WCG_U = NC <= 8 ? 4 : (NC <= 16 ? 2 : 1);  // rows per thread per load group (registers)
    __shared__ double red[8][NC + 1];
    __shared__ double hs[NC + 1];
    const int nb = gridDim.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t per = ceil_div_dev(n, nb);
    const int64_t r0 = (int64_t)blockIdx.x * per, r1 = r0 + per < n ? r0 + per : n;
    const int stride = WCG_MAX + 1;  // part[b * stride + c], c == WCG_MAX: |w|^2
    // sum of column `col` over the blocks' partials, fixed order: lane-strided
    // partial sums (4 loads in flight per lane), then the warp's xor tree.
    // (One thread per column looping over all blocks was a serial chain of
    // ~300 L2 loads after every grid barrier: ~half of the kernel's time.)
    auto col_sum = [&](int col) {
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        int b = lane;
        for (; b + 96 < nb; b += 128)
#pragma unroll
            for (int u = 0; u < 4; ++u) t[u] += __ldcg(part + (int64_t)(b + 32 * u) * stride + col);
        for (; b < nb; b += 32) t[0] += __ldcg(part + (int64_t)b * stride + col);
        return warp_sum((t[0] + t[1]) + (t[2] + t[3]));
    };
    // hs[c] = column sums c < ncol (and hs[NC] = the |w|^2 column): warp q
    // takes columns q, q + 8, ...
    auto gather_h = [&](int ncol, bool with_w) {
        const int tot = ncol + (with_w ? 1 : 0);
        for (int q = warp; q < tot; q += 8) {
            const double v = col_sum(q < ncol ? q : WCG_MAX);
            if (lane == 0) hs[q < ncol ? q : NC] = v;
        }
        __syncthreads();
    };
    double acc[NC + 1];
    // pass 1: projections of the raw w and |w0|^2
#pragma unroll
    for (int c = 0; c <= NC; ++c) acc[c] = 0.0;
    // rows in groups of WCG_U per thread (stride blockDim.x), every load of a
    // group issued before its FMAs: WCG_U x (cnt + 1) loads in flight
    int64_t r = r0 + threadIdx.x;
    for (; r + (WCG_U - 1) * 256 < r1; r += WCG_U * 256) {
        double x[WCG_U], b[WCG_U][NC];
#pragma unroll
        for (int u = 0; u < WCG_U; ++u) {
            x[u] = w[r + u * 256];
#pragma unroll
            for (int c = 0; c < NC; ++c) b[u][c] = c < cnt ? __ldg(Bw + (int64_t)c * ld + r + u * 256) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < WCG_U; ++u) {
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c] = fma(b[u][c], x[u], acc[c]);
            acc[NC] = fma(x[u], x[u], acc[NC]);
        }
    }
    for (; r < r1; r += blockDim.x) {
        const double x = w[r];
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (c < cnt) acc[c] = fma(__ldg(Bw + (int64_t)c * ld + r), x, acc[c]);
        acc[NC] = fma(x, x, acc[NC]);
    }
    {
        const double v = warp_sum(acc[NC]);
        if (lane == 0) red[warp][NC] = v;
    }
    WCG_BLOCK_REDUCE_STORE(acc, cnt);  // (its barriers also publish red[][NC])
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < 8; ++q) t += red[q][NC];
        part[(int64_t)blockIdx.x * stride + WCG_MAX] = t;
    }
    grid.sync();
    gather_h(cnt, true);
    const double w0sq = hs[NC];
    const double alpha = hs[cnt - 1];
    // update 1 fused with the projections of the updated w (pass 2)
#pragma unroll
    for (int c = 0; c <= NC; ++c) acc[c] = 0.0;
    r = r0 + threadIdx.x;
    for (; r + (WCG_U - 1) * 256 < r1; r += WCG_U * 256) {
        double x[WCG_U], b[WCG_U][NC];
#pragma unroll
        for (int u = 0; u < WCG_U; ++u) {
            x[u] = w[r + u * 256];
#pragma unroll
            for (int c = 0; c < NC; ++c) b[u][c] = c < cnt ? __ldg(Bw + (int64_t)c * ld + r + u * 256) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < WCG_U; ++u) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < NC; ++c) s = fma(b[u][c], hs[c < cnt ? c : 0] * (c < cnt ? 1.0 : 0.0), s);
            const double xv = x[u] - s;
            w[r + u * 256] = xv;
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c] = fma(b[u][c], xv, acc[c]);
        }
    }
    for (; r < r1; r += blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (c < cnt) s = fma(__ldg(Bw + (int64_t)c * ld + r), hs[c], s);
        const double x = w[r] - s;
        w[r] = x;
#pragma unroll
        for (int c = 0; c < NC; ++c)  // the same lines again: L1 hits
            if (c < cnt) acc[c] = fma(__ldg(Bw + (int64_t)c * ld + r), x, acc[c]);
    }
    grid.sync();  // every block has read hs-dependent part[] before it is overwritten
    WCG_BLOCK_REDUCE_STORE(acc, cnt);
    grid.sync();
    gather_h(cnt, false);
    // update 2 and |w|^2
    double sq = 0.0;
    r = r0 + threadIdx.x;
    for (; r + (WCG_U - 1) * 256 < r1; r += WCG_U * 256) {
        double x[WCG_U], b[WCG_U][NC];
#pragma unroll
        for (int u = 0; u < WCG_U; ++u) {
            x[u] = w[r + u * 256];
#pragma unroll
            for (int c = 0; c < NC; ++c) b[u][c] = c < cnt ? __ldg(Bw + (int64_t)c * ld + r + u * 256) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < WCG_U; ++u) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < NC; ++c) s = fma(b[u][c], hs[c < cnt ? c : 0] * (c < cnt ? 1.0 : 0.0), s);
            const double xv = x[u] - s;
            w[r + u * 256] = xv;
            sq = fma(xv, xv, sq);
        }
    }
    for (; r < r1; r += blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (c < cnt) s = fma(__ldg(Bw + (int64_t)c * ld + r), hs[c], s);
        const double x = w[r] - s;
        w[r] = x;
        sq = fma(x, x, sq);
    }
    {
        const double v = warp_sum(sq);
        if (lane == 0) red[warp][0] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < 8; ++q) t += red[q][0];
            part[(int64_t)blockIdx.x * stride + WCG_MAX] = t;
        }
    }
    grid.sync();
    if (blockIdx.x == 0 && warp == 0) {
        const double t = col_sum(WCG_MAX);
        if (lane == 0) {
            scal[0] = sqrt(t);
            scal[2] = alpha;
            scal[3] = sqrt(w0sq);
            T[j * m + j] = alpha;
        }
    }
}

// per-block partial sums of x^2 and non-finite detection
__global__ void sumsq_partial_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ part,
                                     int* __restrict__ nonfinite) {
    __shared__ double red[8];
    int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    double v = i < n ? x[i] : 0.0;
    if (nonfinite && !isfinite(v)) atomicOr(nonfinite, 1);
    double s = warp_sum(v * v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        part[blockIdx.x] = t;
    }
}

// scal[out] = sqrt(sum part) (fixed order)
__global__ void finish_norm_kernel(int64_t nb, const double* __restrict__ part, double* __restrict__ scal, int out) {
    __shared__ double red[1024];
    double a = 0.0;
    for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) a += part[b];
    red[threadIdx.x] = a;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) scal[out] = sqrt(red[0]);
}

__global__ void div_copy_kernel(int64_t n, const double* __restrict__ src, double div, double* __restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i] / div;
}

// dst = src / scal[idx]
__global__ void scale_copy_kernel(int64_t n, const double* __restrict__ src, const double* __restrict__ scal,
                                  int idx, double* __restrict__ dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i] / scal[idx];
}

// One launch for the end of a Lanczos step's first CGS pass: scal[0] = |w|
// (sqp partials), scal[3] = |w0| (sq0 partials), T[j,j] = scal[2] = alpha =
// h[j] -- the arithmetic of finish_norm_kernel x 2 + commit_alpha_kernel.
__global__ void __launch_bounds__(1024) step_norms_kernel(int64_t nb_n, const double* __restrict__ sqp, int64_t nb_t,
                                                          const double* __restrict__ sq0, int64_t m, int64_t j,
                                                          const double* __restrict__ h, int64_t hidx,
                                                          double* __restrict__ T, double* __restrict__ scal) {
    __shared__ double red[1024];
    for (int pass = 0; pass < 2; ++pass) {
        const double* part = pass ? sq0 : sqp;
        const int64_t nb = pass ? nb_t : nb_n;
        double a = 0.0;
        for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) a += part[b];
        red[threadIdx.x] = a;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
            __syncthreads();
        }
        if (threadIdx.x == 0) scal[pass ? 3 : 0] = sqrt(red[0]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        T[j * m + j] = h[hidx];
        scal[2] = h[hidx];
    }
}

// next = w / scal[0] and T[j,j+1] = T[j+1,j] = beta in one launch
__global__ void scale_copy_couple_kernel(int64_t n, const double* __restrict__ src, const double* __restrict__ scal,
                                         double* __restrict__ dst, int64_t m, int64_t j, double* __restrict__ T) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i] / scal[0];
    if (i == 0) {
        const double b = scal[0];
        T[j * m + j + 1] = b;
        T[(j + 1) * m + j] = b;
    }
}

// The common step's couple, decided on the device (one-step lookahead,
// sc_lanczos::spec_launch): with beta = scal[0], alpha = scal[2], |w0| =
// scal[3] and the host's running scale, the host's tests -- no window
// cancellation (beta >= wcancel |w0|) and no breakdown (beta > rtol *
// max(1, max(scale, |alpha|, beta))) -- are evaluated on the same doubles; if
// both pass, q_{j+1} = w / beta and the couplings are written exactly as
// scale_copy_couple_kernel does, else nothing is written.  scal[6] = 0 / 1
// tells the host which.
__global__ void couple_guarded_kernel(int64_t n, const double* __restrict__ src, double* __restrict__ scal,
                                      double* __restrict__ dst, int64_t m, int64_t j, double* __restrict__ T,
                                      double scale, double wcancel, double rtol) {
    const double beta = scal[0], alpha = scal[2], w0 = scal[3];
    const double sc = fmax(scale, fmax(fabs(alpha), beta));
    const bool ok = !(beta < wcancel * w0) && beta > rtol * fmax(1.0, sc);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ok && i < n) dst[i] = src[i] / beta;
    if (i == 0) {
        if (ok) {
            T[j * m + j + 1] = beta;
            T[(j + 1) * m + j] = beta;
        }
        scal[6] = ok ? 0.0 : 1.0;
    }
}

// T[j,j] = alpha (= h[j] after the first projection), scal[2] = alpha
__global__ void commit_alpha_kernel(int64_t m, int64_t j, const double* __restrict__ h,
                                    double* __restrict__ T, double* __restrict__ scal) {
    if (threadIdx.x != 0) return;
    T[j * m + j] = h[j];
    scal[2] = h[j];
}

// T[j,j+1] = T[j+1,j] = beta (mode 1) or 0 (mode 0: breakdown, eigen.py:174-176)
__global__ void set_coupling_kernel(int64_t m, int64_t j, const double* __restrict__ scal,
                                    double* __restrict__ T, int mode) {
    if (threadIdx.x != 0) return;
    double b = mode ? scal[0] : 0.0;
    T[j * m + j + 1] = b;
    T[(j + 1) * m + j] = b;
}

// thick restart of T: diag(theta[:k]) plus (optionally) the arrowhead column
__global__ void restart_T_kernel(int64_t m, int64_t k, const double* __restrict__ theta,
                                 const double* __restrict__ S, const double* __restrict__ scal,
                                 int coupled, double* __restrict__ T) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < m * m;
         idx += (int64_t)gridDim.x * blockDim.x)
        T[idx] = 0.0;
    __syncthreads();  // single block launch
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
        T[i * m + i] = theta[i];
        if (coupled) {
            double cpl = scal[0] * S[i * m + (m - 1)];  // beta * s[m-1, i]
            T[k * m + i] = cpl;
            T[i * m + k] = cpl;
        }
    }
}

// gather S[m-1, :k] (last row of the sorted eigenvector block)
__global__ void last_row_kernel(int64_t m, int64_t k, const double* __restrict__ S, double* __restrict__ out) {
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) out[i] = S[i * m + (m - 1)];
}

// C = A (n x kk, col-major ld lda) * S (kk x kc, col-major ld lds);
// out col-major (ldc) if rowmajor == 0 else row-major n x kc
constexpr int GB_M = 64, GB_N = 64, GB_K = 16;
__global__ void __launch_bounds__(256) dgemm_tall_kernel(int64_t n, int kk, int kc, const double* __restrict__ A,
                                                         int64_t lda, const double* __restrict__ S, int64_t lds,
                                                         double* __restrict__ C, int64_t ldc, int rowmajor) {
    __shared__ double As[GB_K][GB_M + 1];
    __shared__ double Ss[GB_K][GB_N + 1];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t r0 = (int64_t)blockIdx.x * GB_M;
    const int c0 = blockIdx.y * GB_N;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < kk; k0 += GB_K) {
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            int idx = tid + 256 * t;
            // A tile: 16 columns x 64 rows, rows fastest (coalesced)
            int rr = idx & 63, kq = idx >> 6;
            int64_t gr = r0 + rr;
            int gk = k0 + kq;
            As[kq][rr] = (gr < n && gk < kk) ? A[(int64_t)gk * lda + gr] : 0.0;
            // S tile: 64 columns x 16 k, k fastest
            int kq2 = idx & 15, cc = idx >> 4;
            int gc = c0 + cc, gk2 = k0 + kq2;
            Ss[kq2][cc] = (gc < kc && gk2 < kk) ? S[(int64_t)gc * lds + gk2] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < GB_K; ++q) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[q][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Ss[q][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int64_t r = r0 + ty + 16 * i;
        if (r >= n) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int c = c0 + tx + 16 * j;
            if (c >= kc) continue;
            if (rowmajor) C[r * kc + c] = acc[i][j];
            else C[(int64_t)c * ldc + r] = acc[i][j];
        }
    }
}

// The same product on the fp64 tensor path (mma.sync m8n8k4 f64, 37 TFLOP/s
// measured on this part vs ~16 for the register-tiled FMA kernel above):
// CTA tile 128 rows x 128 output columns, K chunks of 16 basis columns
// through a 3-stage cp.async ring; 8 warps as 4 (rows) x 2 (columns), each
// 32 x 64 = 4 x 8 m8n8 accumulators.  Grid x = output column tiles, so the
// CTAs sharing a row tile of A run together and A is read from HBM once.
// Requires lda, lds even and A, S 16-byte aligned (dgemm_launch checks).
constexpr int DG_M = 128, DG_N = 128, DG_K = 16, DG_STAGES = 3;
constexpr int DG_LDA = DG_M + 4;   // As[k][row]: conflict-free a-fragment loads
constexpr int DG_LDS = DG_K + 4;   // Ss[col][k]: conflict-free b-fragment loads
constexpr int DG_STAGE = DG_K * DG_LDA + DG_N * DG_LDS;

__device__ __forceinline__ void dg_cp16(double* smem, const double* gmem, int bytes) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(256) dgemm_dmma_kernel(int64_t n, int kk, int kc, const double* __restrict__ A,
                                                         int64_t lda, const double* __restrict__ S, int64_t lds,
                                                         double* __restrict__ C, int64_t ldc, int rowmajor) {
    extern __shared__ __align__(16) double dg_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wr = warp & 3, wc = warp >> 2;
    const int c0 = blockIdx.x * DG_N;
    const int64_t r0 = (int64_t)blockIdx.y * DG_M;
    const int nch = (kk + DG_K - 1) / DG_K;
    auto load = [&](int ch, int stage) {
        double* As = dg_smem + stage * DG_STAGE;
        double* Ss = As + DG_K * DG_LDA;
        const int k0 = ch * DG_K;
        // A: 16 basis columns x 64 row pairs
        for (int e = threadIdx.x; e < DG_K * (DG_M / 2); e += 256) {
            const int kq = e / (DG_M / 2), rp = (e % (DG_M / 2)) * 2;
            const int k = k0 + kq;
            const int64_t r = r0 + rp;
            const int bytes = (k < kk && r < n) ? (r + 1 < n ? 16 : 8) : 0;
            dg_cp16(As + kq * DG_LDA + rp, bytes ? A + (int64_t)k * lda + r : A, bytes);
        }
        // S: 128 output columns x 8 k pairs
        for (int e = threadIdx.x; e < DG_N * (DG_K / 2); e += 256) {
            const int cc = e / (DG_K / 2), kp = (e % (DG_K / 2)) * 2;
            const int col = c0 + cc, k = k0 + kp;
            const int bytes = (col < kc && k < kk) ? (k + 1 < kk ? 16 : 8) : 0;
            dg_cp16(Ss + cc * DG_LDS + kp, bytes ? S + (int64_t)col * lds + k : S, bytes);
        }
    };
    double acc[4][8][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int st = 0; st < DG_STAGES - 1; ++st) {
        if (st < nch) load(st, st);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    for (int ch = 0; ch < nch; ++ch) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(DG_STAGES - 2) : "memory");
        __syncthreads();
        if (ch + DG_STAGES - 1 < nch) load(ch + DG_STAGES - 1, (ch + DG_STAGES - 1) % DG_STAGES);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        const double* As = dg_smem + (ch % DG_STAGES) * DG_STAGE;
        const double* Ss = As + DG_K * DG_LDA;
        const double* ap = As + (lane & 3) * DG_LDA + wr * 32 + (lane >> 2);
        const double* bp = Ss + (wc * 64 + (lane >> 2)) * DG_LDS + (lane & 3);
#pragma unroll
        for (int k4 = 0; k4 < DG_K; k4 += 4) {
            double a[4], b[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = ap[k4 * DG_LDA + i * 8];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = bp[j * 8 * DG_LDS + k4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                 : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                                 : "d"(a[i]), "d"(b[j]));
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = r0 + wr * 32 + i * 8 + (lane >> 2);
        if (r >= n) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = c0 + wc * 64 + j * 8 + 2 * (lane & 3) + h;
                if (c >= kc) continue;
                if (rowmajor) C[r * kc + c] = acc[i][j][h];
                else C[(int64_t)c * ldc + r] = acc[i][j][h];
            }
        }
    }
}

// C = A S (dgemm_tall_kernel's contract) on the DMMA kernel when the operands
// allow 16-byte copies, else on the FMA kernel
static int dgemm_launch(int64_t n, int kk, int kc, const double* A, int64_t lda, const double* S, int64_t lds,
                        double* C, int64_t ldc, int rowmajor, cudaStream_t st) {
    if (n <= 0 || kc <= 0) return SC_OK;
    const bool dmma = !(lda & 1) && !(lds & 1) && !(reinterpret_cast<uintptr_t>(A) & 15) &&
                      !(reinterpret_cast<uintptr_t>(S) & 15) && !std::getenv("SPECLUST_DGEMM_FMA");
    if (dmma) {
        static bool attr = false;
        const int smem = DG_STAGES * DG_STAGE * (int)sizeof(double);
        if (!attr) {
            SC_CUDA(cudaFuncSetAttribute(dgemm_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr = true;
        }
        dim3 grid((unsigned)ceil_div(kc, DG_N), (unsigned)ceil_div(n, DG_M));
        dgemm_dmma_kernel<<<grid, 256, smem, st>>>(n, kk, kc, A, lda, S, lds, C, ldc, rowmajor);
    } else {
        dim3 grid((unsigned)ceil_div(n, GB_M), (unsigned)ceil_div(kc, GB_N));
        dgemm_tall_kernel<<<grid, 256, 0, st>>>(n, kk, kc, A, lda, S, lds, C, ldc, rowmajor);
    }
    SC_LAUNCHED(1);
    return SC_OK;
}

// copy n x k col-major (ld) block between two buffers with the same ld
__global__ void copy_cols_kernel(int64_t n, int64_t k, int64_t ld, const double* __restrict__ src,
                                 double* __restrict__ dst) {
    int64_t total = k * ld;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        if ((i % ld) < n) dst[i] = src[i];
}
// dst[c * ldd + r] = src[c * lds + r], r < rows, c < k (row chunk of a column-major block)
__global__ void copy_chunk_cols_kernel(int64_t rows, int64_t k, const double* __restrict__ src, int64_t lds,
                                       double* __restrict__ dst, int64_t ldd) {
    const int64_t total = rows * k;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / rows, r = i - c * rows;
        dst[c * ldd + r] = src[c * lds + r];
    }
}

// per-block column sums of squares of a row-major n x k matrix
constexpr int CN_ROWS = 256;
// element (r, c) of V at V[r * rs + c * cs]: row-major (rs = k, cs = 1) or
// column-major with leading dimension ld (rs = 1, cs = ld); same arithmetic
__global__ void colsq_partial_kernel(int64_t n, int64_t k, const double* __restrict__ V, int64_t rs, int64_t cs,
                                     double* __restrict__ part) {
    int64_t r0 = (int64_t)blockIdx.x * CN_ROWS, r1 = imin64(n, r0 + CN_ROWS);
    for (int64_t c = threadIdx.x; c < k; c += blockDim.x) {
        double a = 0.0;
        for (int64_t r = r0; r < r1; ++r) a = fma(V[r * rs + c * cs], V[r * rs + c * cs], a);
        part[blockIdx.x * k + c] = a;
    }
}
__global__ void scale_cols_colmajor_kernel(int64_t n, int64_t k, int64_t ld, const double* __restrict__ norms,
                                           double* __restrict__ V) {
    const int64_t total = k * ld;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        if (i % ld < n) V[i] = V[i] / norms[i / ld];
}
// partial sums of (y_i - theta_c v_i)^2 for one column (residual of a
// column-major eigenvector from its own SpMV)
__global__ void resid_col_partial_kernel(int64_t n, const double* __restrict__ y, const double* __restrict__ v,
                                         const double* __restrict__ theta, int64_t c, double* __restrict__ part) {
    __shared__ double red[256];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double a = 0.0;
    if (i < n) {
        const double r = y[i] - theta[c] * v[i];
        a = r * r;
    }
    red[threadIdx.x] = a;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void colnorm_finish_kernel(int64_t nb, int64_t k, const double* __restrict__ part,
                                      double* __restrict__ norms) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k) return;
    double a = 0.0;
    for (int64_t b = 0; b < nb; ++b) a += part[b * k + c];
    norms[c] = sqrt(a);
}
__global__ void scale_cols_rowmajor_kernel(int64_t n, int64_t k, const double* __restrict__ norms, double* __restrict__ V) {
    int64_t total = n * k;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        V[i] = V[i] / norms[i % k];
}

// residual partials: R[i, c] = (A V)[i, c] - theta_c V[i, c]; part[b, c] = sum_i R^2
constexpr int RS_ROWS = 64;
__global__ void residual_partial_kernel(int64_t n, int64_t k, const int64_t* __restrict__ row_ptr,
                                        const int32_t* __restrict__ col, const double* __restrict__ vals,
                                        const double* __restrict__ V, const double* __restrict__ theta,
                                        double* __restrict__ part) {
    // block: 256 threads = 8 warps; rows [r0, r0 + RS_ROWS); columns chunked by 32
    __shared__ double red[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * RS_ROWS;
    for (int64_t c0 = 0; c0 < k; c0 += 32) {
        int64_t c = c0 + lane;
        double acc2 = 0.0;
        for (int64_t r = r0 + warp; r < imin64(n, r0 + RS_ROWS); r += 8) {
            double a = 0.0;
            if (c < k) {
                for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) a = fma(vals[p], V[(int64_t)col[p] * k + c], a);
                double res = a - theta[c] * V[r * k + c];
                acc2 = fma(res, res, acc2);
            }
        }
        red[warp][lane] = acc2;
        __syncthreads();
        if (warp == 0 && c < k) {
            double t = 0.0;
            for (int q = 0; q < 8; ++q) t += red[q][lane];
            part[blockIdx.x * k + c] = t;
        }
        __syncthreads();
    }
}

// The same partials with every column of a row in one pass (k <= 32 KC):
// lane c accumulates columns c, c + 32, ..., so A is read once and each
// neighbour's V row (k doubles) is read whole.  Per-column arithmetic and
// order are those of residual_partial_kernel.
template <int KC>
__global__ void __launch_bounds__(256) residual_rows_kernel(int64_t n, int64_t k, const int64_t* __restrict__ row_ptr,
                                                            const int32_t* __restrict__ col,
                                                            const double* __restrict__ vals,
                                                            const double* __restrict__ V,
                                                            const double* __restrict__ theta,
                                                            double* __restrict__ part) {
    __shared__ double red[8][32 * KC];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * RS_ROWS;
    double acc2[KC];
#pragma unroll
    for (int q = 0; q < KC; ++q) acc2[q] = 0.0;
    for (int64_t r = r0 + warp; r < imin64(n, r0 + RS_ROWS); r += 8) {
        double a[KC];
#pragma unroll
        for (int q = 0; q < KC; ++q) a[q] = 0.0;
        const int64_t pe = row_ptr[r + 1];
        for (int64_t p = row_ptr[r]; p < pe; ++p) {
            const double v = vals[p];
            const double* vr = V + (int64_t)col[p] * k;
#pragma unroll
            for (int q = 0; q < KC; ++q)
                if (lane + 32 * q < k) a[q] = fma(v, vr[lane + 32 * q], a[q]);
        }
#pragma unroll
        for (int q = 0; q < KC; ++q) {
            const int64_t c = lane + 32 * q;
            if (c < k) {
                const double res = a[q] - theta[c] * V[r * k + c];
                acc2[q] = fma(res, res, acc2[q]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < KC; ++q) red[warp][lane + 32 * q] = acc2[q];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < KC; ++q) {
            const int64_t c = lane + 32 * q;
            if (c < k) {
                double t = 0.0;
                for (int w = 0; w < 8; ++w) t += red[w][lane + 32 * q];
                part[blockIdx.x * k + c] = t;
            }
        }
    }
}

// max |v| as ordered bits of a non-negative double
__global__ void absmax_kernel(int64_t m, const double* __restrict__ v, unsigned long long* __restrict__ out) {
    double a = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        a = fmax(a, fabs(v[i]));
    for (int o = 16; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(a));
}

// per-block partial of x.ay - y.ax (symmetry probe)
__global__ void dot_partial_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ ay,
                                   const double* __restrict__ y, const double* __restrict__ ax,
                                   double* __restrict__ part) {
    __shared__ double red[8];
    int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    double v = i < n ? (x[i] * ay[i] - y[i] * ax[i]) : 0.0;
    double s = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < 8; ++q) t += red[q];
        part[blockIdx.x] = t;
    }
}

__global__ void finish_sum_kernel(int64_t nb, const double* __restrict__ part, double* __restrict__ out, int idx) {
    __shared__ double red[1024];
    double a = 0.0;
    for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) a += part[b];
    red[threadIdx.x] = a;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[idx] = red[0];
}

}  // namespace sc

using namespace sc;

// ---------------------------------------------------------------------------
// ---- locked eigenvalue-1 eigenspace of a normalized adjacency -----------------
// A = D^-1/2 W D^-1/2 has eigenvalue 1 with multiplicity = the number of
// connected components of W, eigenvectors u_C = D^1/2 1_C / |D^1/2 1_C|
// (disjoint supports).  The reference discovers every copy by Lanczos sweeps
// from fresh directions (eigen.py:195-206, one copy of a degenerate value
// per verification sweep: 10 of C3h's 21 restarts); here they are locked up
// front and the Lanczos recurrence runs on their orthogonal complement.

// one min-label propagation step with pointer jumping: lab2[i] =
// min(lab[i], lab[j] over row i), then lab2[i] = lab[lab2[i]] (one jump)
__global__ void cc_propagate_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                    const int32_t* __restrict__ lab, int32_t* __restrict__ lab2,
                                    int* __restrict__ changed) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t mn = lab[i];
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) mn = min(mn, lab[col[e]]);
    mn = min(mn, lab[mn]);
    lab2[i] = mn;
    if (mn != lab[i]) *changed = 1;
}
// root flags (label == own index) for the component numbering
__global__ void cc_roots_kernel(int64_t n, const int32_t* __restrict__ lab, int64_t* __restrict__ flag) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = lab[i] == (int32_t)i ? 1 : 0;
}
// component id of node i = rank of its root among the roots (roots in index order)
__global__ void cc_number_kernel(int64_t n, const int32_t* __restrict__ lab, const int64_t* __restrict__ rank,
                                 int64_t* __restrict__ comp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) comp[i] = rank[lab[i]];
}
// per component C: sum over its members (member order) of a[i] * (b ? b[i] :
// 1), in two fixed-order passes over chunks of at most SEG_CH members (one
// block per component would leave C3's 164K-node component to one block's
// serial loop every Lanczos step): chunk partials, then each component's
// chunks in order
constexpr int64_t SEG_CH = 4096;
__global__ void seg_dot_chunks_kernel(const int64_t* __restrict__ cbeg, const int64_t* __restrict__ cend,
                                      const int32_t* __restrict__ members, const double* __restrict__ a,
                                      const double* __restrict__ b, double* __restrict__ part) {
    __shared__ double red[256];
    const int64_t q = blockIdx.x;
    double acc = 0.0;
    for (int64_t t = cbeg[q] + threadIdx.x; t < cend[q]; t += blockDim.x) {
        const int64_t i = members[t];
        acc = fma(a[i], b ? b[i] : 1.0, acc);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[q] = red[0];
}
__global__ void seg_dot_combine_kernel(int64_t c, const int64_t* __restrict__ qoff, const double* __restrict__ part,
                                       double* __restrict__ out) {
    const int64_t C = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (C >= c) return;
    double t = 0.0;
    for (int64_t q = qoff[C]; q < qoff[C + 1]; ++q) t += part[q];
    out[C] = t;
}

// u[i] = sqrt(d[i]) / sqrt(dsum[comp[i]])
__global__ void locked_vec_kernel(int64_t n, const double* __restrict__ d, const int64_t* __restrict__ comp,
                                  const double* __restrict__ dsum, double* __restrict__ u) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) u[i] = sqrt(d[i]) / sqrt(dsum[comp[i]]);
}
// x[i] -= h[comp[i]] * u[i]
__global__ void deflate_sub_kernel(int64_t n, const int64_t* __restrict__ comp, const double* __restrict__ u,
                                   const double* __restrict__ h, double* __restrict__ x) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] -= h[comp[i]] * u[i];
}
// r[i] = (y[i] - theta[comp[i]] u[i])^2
__global__ void locked_resid_kernel(int64_t n, const int64_t* __restrict__ comp, const double* __restrict__ u,
                                    const double* __restrict__ y, const double* __restrict__ theta,
                                    double* __restrict__ r) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const double t = y[i] - theta[comp[i]] * u[i];
        r[i] = t * t;
    }
}
// out (row-major n x k): columns [0, c) the locked vectors in the order
// col_of[comp] (dense, zero off their component), columns [c, k) from
// rv (row-major n x (k - c))
__global__ void assemble_vectors_kernel(int64_t n, int64_t k, int64_t c, const int64_t* __restrict__ comp,
                                        const int64_t* __restrict__ col_of, const double* __restrict__ u,
                                        const double* __restrict__ rv, double* __restrict__ out) {
    const int64_t total = n * k;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / k, j = e - i * k;
        double v;
        if (j < c)
            v = col_of[comp[i]] == j ? u[i] : 0.0;
        else
            v = rv[i * (k - c) + (j - c)];
        out[e] = v;
    }
}

__global__ void iota_i32_kernel(int64_t n, int32_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)i;
}

// SPECLUST_SLOW_MS=t (diagnostics): Lanczos steps whose host wall time
// exceeds t ms are reported with their step index and phase
struct SlowWatch {
    double ms = -1.0;
    std::chrono::steady_clock::time_point t0;
    SlowWatch() {
        const char* e = std::getenv("SPECLUST_SLOW_MS");
        if (e) ms = std::atof(e);
        t0 = std::chrono::steady_clock::now();
    }
    void lap(const char* what, int64_t a, int64_t b) {
        if (ms < 0) return;
        const auto t1 = std::chrono::steady_clock::now();
        const double dt = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (dt > ms) fprintf(stderr, "[slow] lanczos %s %lld/%lld %.1f ms\n", what, (long long)a, (long long)b, dt);
        t0 = t1;
    }
};

struct LockedSet {
    int64_t c = 0, nq = 0;
    DevBuf<int64_t> comp;   // n: component id
    DevBuf<double> u, h;    // n: the locked vectors (disjoint supports); c: projections
    Bucketer bk;            // members grouped by component
    DevBuf<int64_t> cbeg, cend, qoff;  // member chunks (<= SEG_CH) and each component's first chunk
    DevBuf<double> part;
    // chunk table from the component sizes (bk.start, after bk.run)
    int plan(cudaStream_t st) {
        std::vector<int64_t> hs(c + 1);
        SC_CUDA(d2h_sync(hs.data(), bk.start.p, sizeof(int64_t) * (c + 1), st));
        std::vector<int64_t> hb, he, hq(c + 1, 0);
        for (int64_t C = 0; C < c; ++C) {
            for (int64_t t = hs[C]; t < hs[C + 1]; t += SEG_CH) {
                hb.push_back(t);
                he.push_back(std::min(hs[C + 1], t + SEG_CH));
            }
            if (hs[C + 1] == hs[C]) {  // (no empty component exists; keep the table total)
                hb.push_back(hs[C]);
                he.push_back(hs[C]);
            }
            hq[C + 1] = (int64_t)hb.size();
        }
        nq = (int64_t)hb.size();
        int rc;
        if ((rc = cbeg.alloc(nq)) || (rc = cend.alloc(nq)) || (rc = qoff.alloc(c + 1)) || (rc = part.alloc(nq)))
            return rc;
        SC_CUDA(cudaMemcpyAsync(cbeg.p, hb.data(), sizeof(int64_t) * nq, cudaMemcpyHostToDevice, st));
        SC_CUDA(cudaMemcpyAsync(cend.p, he.data(), sizeof(int64_t) * nq, cudaMemcpyHostToDevice, st));
        SC_CUDA(cudaMemcpyAsync(qoff.p, hq.data(), sizeof(int64_t) * (c + 1), cudaMemcpyHostToDevice, st));
        SC_CUDA(cudaStreamSynchronize(st));
        return SC_OK;
    }
    // out[C] = sum over component C's members of a[i] * (b ? b[i] : 1), fixed order
    int seg_dot(const double* a, const double* b, double* out, cudaStream_t st) {
        seg_dot_chunks_kernel<<<(unsigned)nq, 256, 0, st>>>(cbeg.p, cend.p, bk.members.p, a, b, part.p);
        seg_dot_combine_kernel<<<(unsigned)ceil_div(c, 256), 256, 0, st>>>(c, qoff.p, part.p, out);
        SC_LAUNCHED(2);
        return SC_OK;
    }
    int deflate(int64_t n, double* x, cudaStream_t st) {
        if (int rc = seg_dot(u.p, x, h.p, st)) return rc;
        deflate_sub_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, comp.p, u.p, h.p, x);
        SC_LAUNCHED(1);
        return SC_OK;
    }
};

struct sc_lanczos {
    int64_t n = 0, k = 0, m = 0, ld = 0, max_restarts = 0;
    double tol = 0.0;
    uint64_t seed = 0;
    cudaStream_t st = nullptr;
    int state = 0;  // 0 need_matvec, 1 converged, 2 failed
    int64_t j = 0;
    int64_t restarts = 0, breakdowns = 0, matvecs = 0, second_passes = 0;
    // windowed reorthogonalisation: columns < j0 are orthogonalised against
    // each other; win = current window length
    bool windowed = true;
    int64_t j0 = 0, win = 6, flushes = 0, window_sum = 0;
    // two-tier flushes after a restart (SPECLUST_REORTH=onetier disables):
    // the window's loss is measured against the retained Ritz block (it grows
    // there: converged Ritz vectors) and against the sweep's own older
    // vectors (it stays at rounding level, profiles/r02_flush_losses.md), so
    // the Ritz block is flushed every `win` steps and the sweep's older
    // vectors only every `win_s` steps; js = first column not yet flushed
    // against the sweep's older vectors
    bool tiered = true;
    int64_t js = 0, win_s = 16, sweep_flushes = 0;
    double max_loss = 0.0;
    DevBuf<double> bpart, bH, wpart;
    DevBuf<unsigned long long> bmax;
    uint64_t rng_stream = 0;
    double scale = 0.0;
    std::vector<double> history, pending, theta_k, est_k;
    bool has_pending = false;
    // one-step lookahead (internal drivers only; SPECLUST_LOOKAHEAD=0 off): a
    // common windowed step launches its couple guarded on the device
    // (couple_guarded_kernel), swaps the work vector and returns, so the
    // driver's next SpMV runs while the host reads this step's scalars; the
    // next advance() settles them first and, if the device declined (window
    // cancellation or breakdown), swaps back and takes this step's host path
    bool spec_on = false, spec_pending = false;
    DevBuf<double> w2;
    double* spec_host = nullptr;  // pinned: scal[0..6] of the pending step
    cudaEvent_t spec_ev = nullptr;
    int64_t spec_hits = 0, spec_aborts = 0;
    ~sc_lanczos() {
        if (spec_host) cudaFreeHost(spec_host);
        if (spec_ev) cudaEventDestroy(spec_ev);
    }

    DevBuf<double> B, T, w, part, h, sqp, sq0, scal, Y, A, Z, wraw, wsort, S, lastrow, vectors;
    double* vec_out = nullptr;  // converged Ritz vectors (row-major n x k): `vectors` or a caller buffer
    bool in_basis = false;      // caller-owned basis; the result stays in its columns 0..k-1
    LockedSet* locked = nullptr;  // deflated eigenvalue-1 eigenspace (orthogonal complement only)
    DevBuf<int> info, nonfinite;
    int64_t nb_t = 0, nb_n = 0;
    int rpb_t = GT_ROWS;  // rows per gemv_t block
    static constexpr int64_t fz_blocks = 4 * kNumSMs;  // persistent grid of the fused pass

    // ---- building blocks
    int project(const double* x, int ncols, double* sq_part = nullptr, int64_t col0 = 0) {
        gemv_t_partial_kernel<<<(unsigned)nb_t, 256, 0, st>>>(n, ld, ncols, rpb_t, B.p + col0 * ld, x, part.p,
                                                               sq_part);
        reduce_cols_kernel<<<(unsigned)ceil_div((int64_t)ncols * 32, 256), 256, 0, st>>>(nb_t, ncols, part.p, h.p);
        SC_LAUNCHED(2);
        return SC_OK;
    }
    int subtract(double* x, int ncols, bool with_norm, int64_t col0 = 0) {
        gemv_n_update_kernel<<<(unsigned)nb_n, GN_THREADS, sizeof(double) * (size_t)ncols, st>>>(
            n, ld, ncols, B.p + col0 * ld, h.p, x, with_norm ? sqp.p : nullptr);
        SC_LAUNCHED(1);
        return SC_OK;
    }
    // two CGS passes against the first `count` basis vectors; scal[0] = |x|
    int cgs2(double* x, int count) {
        double bytes = 4.0 * (double)n * count * 8.0;
        ProfScope prof("reorth", st, bytes);
        int rc;
        if (count == 0) {
            sumsq_partial_kernel<<<(unsigned)nb_n, 256, 0, st>>>(n, x, sqp.p, nullptr);
            SC_LAUNCHED(1);
        } else {
            if ((rc = project(x, count)) || (rc = subtract(x, count, false))) return rc;
            if ((rc = project(x, count)) || (rc = subtract(x, count, true))) return rc;
        }
        finish_norm_kernel<<<1, 1024, 0, st>>>(nb_n, sqp.p, scal.p, 0);
        SC_LAUNCHED(1);
        return SC_OK;
    }
    double read_scal(int idx) {
        double v = 0.0;
        d2h_sync(&v, scal.p + idx, sizeof(double), st);
        return v;
    }
    // unit vector orthogonal to B[:, :count] into column `dst` (eigen.py:137-150)
    int fresh(int64_t count, int64_t dst, bool is_breakdown) {
        for (int attempt = 0; attempt < 3; ++attempt) {
            double* x = B.p + dst * ld;
            fill_normal_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, seed, ++rng_stream, x);
            SC_LAUNCHED(1);
            if (locked) {
                int rc0 = locked->deflate(n, x, st);
                if (!rc0) rc0 = locked->deflate(n, x, st);
                if (rc0) return rc0;
            }
            // the first `count` columns are the basis; CGS2 against them
            // (x lives in column dst >= count, so it is not projected on itself)
            int rc = cgs2(x, (int)count);
            if (rc) return rc;
            double nv = read_scal(0);
            if (nv > 1e-6 * std::sqrt((double)n)) {
                if (is_breakdown) ++breakdowns;
                scale_copy_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, x, scal.p, 0, x);
                SC_LAUNCHED(1);
                return SC_OK;
            }
        }
        state = 2;
        return fail(SC_ERR_BREAKDOWN, "could not extend the basis past " + std::to_string(count) + " vectors");
    }

    int init(int64_t n_, int64_t k_, int64_t m_, double tol_, int64_t maxr, uint64_t seed_, cudaStream_t st_,
             double* basis = nullptr) {
        n = n_;
        k = k_;
        m = m_ > 0 ? m_ : imin64(n_, std::max<int64_t>(2 * k_, k_ + 8));  // eigen.py:53-55
        if (!(1 <= k && k < m && m <= n))
            return fail(SC_ERR_VALUE, "need 1 <= k < m <= n, got k=" + std::to_string(k) + ", m=" +
                                          std::to_string(m) + ", n=" + std::to_string(n));
        if (!(tol_ > 0)) return fail(SC_ERR_VALUE, "tol must be positive");
        if (maxr < 0) return fail(SC_ERR_VALUE, "max_restarts must be nonnegative");
        tol = tol_;
        max_restarts = maxr;
        seed = seed_;
        st = st_;
        ld = (n + 31) / 32 * 32;
        // one balanced wave at the kernel occupancy while the rows fit, 32-row granules
        rpb_t = gemv_t_rows_per_block(n);
        nb_t = ceil_div(n, rpb_t);
        nb_n = ceil_div(n, GN_THREADS);
        int rc;
        if (basis) {
            B.borrow(basis, (size_t)ld * (m + 1));
            in_basis = true;
        }
        if ((!basis && (rc = B.alloc((size_t)ld * (m + 1)))) || (rc = T.alloc((size_t)m * m)) || (rc = w.alloc(ld)) ||
            (rc = part.alloc((size_t)std::max<int64_t>(nb_t, fz_blocks) * (m + 1))) || (rc = h.alloc(m + 1)) ||
            (rc = sqp.alloc(nb_n)) || (rc = sq0.alloc(nb_t)) ||
            (rc = scal.alloc(8)) || (rc = A.alloc((size_t)m * m)) || (rc = Z.alloc((size_t)m * m)) ||
            (rc = wraw.alloc(m)) || (rc = wsort.alloc(m)) || (rc = S.alloc((size_t)m * k)) ||
            (rc = lastrow.alloc(k)) || (rc = info.alloc(1)) || (rc = nonfinite.alloc(1)) || (rc = bmax.alloc(1)))
            return rc;
        {
            const char* e = std::getenv("SPECLUST_REORTH");
            windowed = !(e && std::strcmp(e, "full") == 0) && (n >= kWindowMinN || (e && std::strcmp(e, "window") == 0));
            tiered = !(e && std::strcmp(e, "onetier") == 0);
        }
        SC_CUDA(cudaMemsetAsync(T.p, 0, sizeof(double) * m * m, st));
        SC_CUDA(cudaMemsetAsync(w.p, 0, sizeof(double) * ld, st));
        // start vector: normal draws, normalised (eigen.py:113-115)
        double* q0 = B.p;
        fill_normal_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, seed, 0, q0);
        SC_LAUNCHED(1);
        if ((rc = cgs2(q0, 0))) return rc;
        scale_copy_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, q0, scal.p, 0, q0);
        SC_LAUNCHED(1);
        j = 0;
        state = 0;
        SC_CUDA(cudaStreamSynchronize(st));
        return SC_OK;
    }

    const double* in_slot() const { return B.p + j * ld; }

    int enable_lookahead() {
        const char* e = std::getenv("SPECLUST_LOOKAHEAD");
        if (spec_on || (e && e[0] == '0')) return SC_OK;
        int rc;
        if ((rc = w2.alloc(ld))) return rc;
        SC_CUDA(cudaMemsetAsync(w2.p, 0, sizeof(double) * ld, st));
        if (cudaMallocHost(&spec_host, 8 * sizeof(double)) != cudaSuccess) {
            spec_host = nullptr;
            cudaGetLastError();
            return SC_OK;  // no lookahead
        }
        if (cudaEventCreateWithFlags(&spec_ev, cudaEventDisableTiming) != cudaSuccess) {
            spec_ev = nullptr;
            cudaGetLastError();
            return SC_OK;
        }
        spec_on = true;
        return SC_OK;
    }
    // the step may be decided on the device: not the sweep's last, and no
    // flush falls due after it (both need the host between the steps)
    bool spec_can() const {
        if (!spec_on || j + 1 >= m) return false;
        const int64_t jn = j + 1;
        if (windowed && tiered && restarts > 0) return !(jn - j0 >= win || jn + 1 - js >= win_s);
        return !(windowed && jn - j0 >= win);
    }
    int spec_launch() {
        double* next = B.p + (j + 1) * ld;
        couple_guarded_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, w.p, scal.p, next, m, j, T.p, scale,
                                                                          kWindowCancel, kBreakdownRtol);
        SC_LAUNCHED(1);
        SC_CUDA(cudaMemcpyAsync(spec_host, scal.p, 7 * sizeof(double), cudaMemcpyDeviceToHost, st));
        SC_CUDA(cudaEventRecord(spec_ev, st));
        std::swap(w.p, w2.p);
        ++j;
        spec_pending = true;
        return SC_OK;
    }
    int spec_resolve(double* ab, bool* ok) {
        spec_pending = false;
        SC_CUDA(cudaEventSynchronize(spec_ev));
        for (int i = 0; i < 4; ++i) ab[i] = spec_host[i];
        *ok = spec_host[6] == 0.0;
        if (*ok) {
            ++spec_hits;
            scale = std::max(scale, std::max(std::fabs(ab[2]), ab[0]));
        } else {
            ++spec_aborts;
            std::swap(w.p, w2.p);
            --j;
        }
        return SC_OK;
    }

    // one Lanczos step on w = A q_j (eigen.py:152-179)
    int advance(bool check_finite) {
        if (state != 0) return fail(SC_ERR_STATE, "advance called in a finished session");
        if (spec_pending) {
            double ab[4];
            bool ok = false;
            int rc = spec_resolve(ab, &ok);
            if (rc) return rc;
            // declined: the pending step's host path; the driver's SpMV of
            // the unwritten q_{j+1} (in the other work vector) is discarded
            if (!ok) return tail(ab);
        }
        ++matvecs;
        int rc;
        if (check_finite) {
            SC_CUDA(cudaMemsetAsync(nonfinite.p, 0, sizeof(int), st));
            sumsq_partial_kernel<<<(unsigned)nb_n, 256, 0, st>>>(n, w.p, sqp.p, nonfinite.p);
            SC_LAUNCHED(1);
            int bad = 0;
            SC_CUDA(d2h_sync(&bad, nonfinite.p, sizeof(int), st));
            if (bad) return fail(SC_ERR_VALUE, "out_slot contains non-finite values");
        }
        if (locked && (rc = locked->deflate(n, w.p, st))) return rc;
        // Orthogonalisation (reference: recurrence + CGS2 over the whole
        // basis every step, eigen.py:157-163).  Windowed mode (default): two
        // CGS passes over the window [lo, j] of recent vectors (it always
        // holds q_{j-1} and q_j, so the three-term components are removed;
        // the first step after a restart projects on the whole retained block
        // for the arrowhead couplings), and every `win` steps the window is
        // orthogonalised against the older basis with two DMMA GEMMs
        // (flush()).  The loss of orthogonality a window accumulates is
        // measured exactly at each flush and the window length adapts to
        // keep it below 1e-9 (semi-orthogonality is sqrt(eps) ~ 1.5e-8).
        // SPECLUST_REORTH=full: one CGS pass over the whole basis every step
        // (+ a DGKS-guarded second pass), the round-1 scheme.
        const bool arrow_step = restarts > 0 && j == k;
        const bool two = windowed && tiered && restarts > 0;
        const int64_t lo = (!windowed || arrow_step) ? 0
                           : std::max<int64_t>(0, std::min<int64_t>(two ? js : j0, j - 1));
        const int cnt = (int)(j + 1 - lo);
        double ab[4];
        if (windowed && !arrow_step && cnt <= WCG_MAX) {
            ProfScope prof("reorth", st, 3.0 * (double)n * cnt * 8.0);
            if ((rc = window_cgs2(lo, cnt))) return rc;
            if (spec_can()) return spec_launch();
            SC_CUDA(d2h_sync(ab, scal.p, sizeof(double) * 4, st));
        } else {
            ProfScope prof("reorth", st, 2.0 * (double)n * cnt * 8.0);
            if ((rc = project(w.p, cnt, sq0.p, lo))) return rc;
            if ((rc = subtract(w.p, cnt, true, lo))) return rc;
            step_norms_kernel<<<1, 1024, 0, st>>>(nb_n, sqp.p, nb_t, sq0.p, m, j, h.p, j - lo, T.p, scal.p);
            SC_LAUNCHED(1);
            if (windowed) {  // second pass over the (short) window, always
                if ((rc = project(w.p, cnt, nullptr, lo)) || (rc = subtract(w.p, cnt, true, lo))) return rc;
                finish_norm_kernel<<<1, 1024, 0, st>>>(nb_n, sqp.p, scal.p, 0);
                SC_LAUNCHED(1);
            }
            SC_CUDA(d2h_sync(ab, scal.p, sizeof(double) * 4, st));
        }
        return tail(ab);
    }

    // the rest of a step once its scalars are on the host: cancellation
    // passes, end of sweep, couple or breakdown, flushes
    int tail(const double* ab_in) {
        int rc;
        double ab[4] = {ab_in[0], ab_in[1], ab_in[2], ab_in[3]};
        const bool two = windowed && tiered && restarts > 0;
        // second pass over the WHOLE basis: always in full mode (the
        // reference's unconditional CGS2, eigen.py:131-135); in windowed mode
        // when the window pass cancelled w to rounding level (a breakdown or
        // near-breakdown: the new direction is made of rounding errors and
        // is not orthogonal to the older basis the window does not cover)
        const bool cancelled = windowed && ab[0] < kWindowCancel * ab[3];
        if (!windowed || cancelled) {
            ProfScope prof("reorth", st, 4.0 * (double)n * (j + 1) * 8.0);
            ++second_passes;
            for (int pass = 0; pass < (cancelled ? 2 : 1); ++pass) {
                if ((rc = project(w.p, (int)(j + 1))) || (rc = subtract(w.p, (int)(j + 1), true))) return rc;
            }
            finish_norm_kernel<<<1, 1024, 0, st>>>(nb_n, sqp.p, scal.p, 0);
            SC_LAUNCHED(1);
            SC_CUDA(d2h_sync(ab, scal.p, sizeof(double), st));
        }
        if (windowed && j + 1 == m) {
            // end of the sweep: the last window against the older basis, then
            // one pass of w over the whole (now orthonormal) basis -- w seeds
            // the next sweep (eigen.py:232) and its norm is the residual scale
            if (two) {
                if ((rc = flush_range(0, k, j0, m - 1, win, kMaxWindow))) return rc;
                if ((rc = flush_range(k, js, js, m - 1, win_s, kMaxSweepWindow))) return rc;
            } else if ((rc = flush(j0, m - 1))) {
                return rc;
            }
            ProfScope prof("reorth", st, 2.0 * (double)n * m * 8.0);
            if ((rc = project(w.p, (int)m)) || (rc = subtract(w.p, (int)m, true))) return rc;
            finish_norm_kernel<<<1, 1024, 0, st>>>(nb_n, sqp.p, scal.p, 0);
            SC_LAUNCHED(1);
            SC_CUDA(d2h_sync(ab, scal.p, sizeof(double), st));
        }
        const double beta = ab[0], alpha = ab[2];
        scale = std::max(scale, std::max(std::fabs(alpha), beta));
        if (j + 1 == m) return finish_sweep(beta);
        double* next = B.p + (j + 1) * ld;
        if (beta > kBreakdownRtol * std::max(1.0, scale)) {
            scale_copy_couple_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, w.p, scal.p, next, m, j, T.p);
            SC_LAUNCHED(1);
        } else {
            set_coupling_kernel<<<1, 32, 0, st>>>(m, j, scal.p, T.p, 0);
            SC_LAUNCHED(1);
            if ((rc = fresh(j + 1, j + 1, true))) return rc;
        }
        ++j;
        if (two) {
            if (j - j0 >= win || j + 1 - js >= win_s) {
                if ((rc = flush_range(0, k, j0, j, win, kMaxWindow))) return rc;
                j0 = j + 1;
            }
            if (j + 1 - js >= win_s) {
                if ((rc = flush_range(k, js, js, j, win_s, kMaxSweepWindow))) return rc;
                ++sweep_flushes;
                js = j + 1;
            }
        } else if (windowed && j - j0 >= win) {
            if ((rc = flush(j0, j))) return rc;
            j0 = j + 1;
        }
        return SC_OK;
    }

    int window_cgs2(int64_t lo, int cnt) {
        void* fn = cnt <= 8    ? (void*)window_cgs2_kernel<8>
                   : cnt <= 16 ? (void*)window_cgs2_kernel<16>
                   : cnt <= 24 ? (void*)window_cgs2_kernel<24>
                               : (void*)window_cgs2_kernel<40>;
        const int bucket = cnt <= 8 ? 0 : cnt <= 16 ? 1 : cnt <= 24 ? 2 : 3;
        static int bps_tab[4] = {0, 0, 0, 0};
        int& bps = bps_tab[bucket];
        if (!bps) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, 256, 0);
            if (bps < 1) bps = 1;
        }
        int dev = 0, nsm = kNumSMs;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)bps * nsm, ceil_div(n, 256)));
        int rc;
        if (wpart.n < (size_t)grid * (WCG_MAX + 1) && (rc = wpart.alloc((size_t)grid * (WCG_MAX + 1)))) return rc;
        const double* Bw = B.p + lo * ld;
        double* wp = w.p;
        double* pp = wpart.p;
        double* Tp = T.p;
        double* sp = scal.p;
        int64_t nn = n, ldd = ld, mm = m, jj = j;
        int c = cnt;
        void* args[] = {&nn, &ldd, (void*)&Bw, &c, &wp, &pp, &mm, &jj, &Tp, &sp};
        SC_CUDA(cudaLaunchCooperativeKernel(fn, grid, 256, args, 0, st));
        SC_LAUNCHED(1);
        return SC_OK;
    }

    // columns [c0, c1] -= B[:, :c0] (B[:, :c0]^T B[:, c0..c1]): one block CGS
    // pass (the window is within ~1e-9 of orthogonal to the older basis, so a
    // second pass would change nothing at working precision); the measured
    // loss adapts the window length
    int flush(int64_t c0, int64_t c1) { return flush_range(0, c0, c0, c1, win, kMaxWindow); }
    // columns [c0, c1] -= B[:, ob:oe] (B[:, ob:oe]^T B[:, c0..c1]); the
    // measured loss adapts `wv` (capped at wmax)
    double flush_ms[2] = {0.0, 0.0};  // SPECLUST_TIMING_DEBUG: flushes against the Ritz block / the sweep
    int64_t flush_n[2] = {0, 0};
    int flush_range(int64_t ob, int64_t oe, int64_t c0, int64_t c1, int64_t& wv, int64_t wmax) {
        static const bool fdbg = std::getenv("SPECLUST_TIMING_DEBUG") != nullptr;
        if (!fdbg) return flush_range_(ob, oe, c0, c1, wv, wmax);
        cudaStreamSynchronize(st);
        const auto t0 = std::chrono::steady_clock::now();
        const int rc = flush_range_(ob, oe, c0, c1, wv, wmax);
        cudaStreamSynchronize(st);
        const int kind = ob == 0 ? 0 : 1;
        flush_ms[kind] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ++flush_n[kind];
        return rc;
    }
    int flush_range_(int64_t ob, int64_t oe, int64_t c0, int64_t c1, int64_t& wv, int64_t wmax) {
        const int64_t nb = oe - ob;
        if (nb <= 0 || c1 < c0) return SC_OK;
        const int c = (int)(c1 - c0 + 1);
        int rc;
        ProfScope prof("reorth", st, 2.0 * (double)n * (double)(nb + c) * 8.0);
        const size_t need = block_part_size(n, (int)nb, c);
        if (bpart.n < need && (rc = bpart.alloc(need))) return rc;
        if (bH.n < (size_t)nb * c && (rc = bH.alloc((size_t)m * 48))) return rc;
        SC_CUDA(cudaMemsetAsync(bmax.p, 0, sizeof(unsigned long long), st));
        if ((rc = block_tn(n, ld, (int)nb, B.p + ob * ld, B.p + c0 * ld, c, bH.p, bpart.p, bmax.p, st))) return rc;
        if ((rc = block_nn(n, ld, (int)nb, B.p + ob * ld, bH.p, c, B.p + c0 * ld, st))) return rc;
        unsigned long long bits = 0;
        SC_CUDA(d2h_sync(&bits, bmax.p, sizeof(bits), st));
        double loss;
        memcpy(&loss, &bits, sizeof(loss));
        static const bool dbg = std::getenv("SPECLUST_FLUSH_DEBUG") != nullptr;
        if (dbg && restarts > 0 && flushes % 10 == 0) {
            // loss against the retained Ritz block (rows < k of H) vs the sweep's vectors
            std::vector<double> hh((size_t)nb * c);
            SC_CUDA(cudaMemcpy(hh.data(), bH.p, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost));
            double lr = 0.0, ls = 0.0;
            for (int64_t r = 0; r < nb; ++r)
                for (int o = 0; o < c; ++o)
                    (ob + r < k ? lr : ls) = std::max(ob + r < k ? lr : ls, std::fabs(hh[r * c + o]));
            fprintf(stderr, "[flush] restart %lld j %lld c %d old [%lld, %lld) loss_ritz %.2e loss_sweep %.2e\n",
                    (long long)restarts, (long long)c1, c, (long long)ob, (long long)oe, lr, ls);
            // loss against the Ritz block by column decile (columns in descending Ritz value order)
            if (ob == 0 && nb >= 10) {
                fprintf(stderr, "[flush]   ritz deciles:");
                const int64_t kk = std::min<int64_t>(k, nb);
                for (int dcl = 0; dcl < 10; ++dcl) {
                    double mx = 0.0;
                    for (int64_t r = kk * dcl / 10; r < kk * (dcl + 1) / 10; ++r)
                        for (int o = 0; o < c; ++o) mx = std::max(mx, std::fabs(hh[r * c + o]));
                    fprintf(stderr, " %.1e", mx);
                }
                int64_t nconv = 0;
                for (int64_t i = 0; i < (int64_t)est_k.size(); ++i)
                    if (est_k[i] <= tol * std::max(1.0, std::fabs(theta_k[i]))) ++nconv;
                fprintf(stderr, "  (converged at the last restart: %lld)\n", (long long)nconv);
            }
        }
        ++flushes;
        window_sum += c;
        max_loss = std::max(max_loss, loss);
        if (loss > 1e-8) {
            // far from orthogonal: re-orthonormalise the window in order
            for (int64_t col = c0; col <= c1; ++col) {
                double* x = B.p + col * ld;
                const int cc = (int)(col - c0);
                if (cc > 0) {
                    for (int pass = 0; pass < 2; ++pass)
                        if ((rc = project(x, cc, nullptr, c0)) || (rc = subtract(x, cc, false, c0))) return rc;
                }
                sumsq_partial_kernel<<<(unsigned)nb_n, 256, 0, st>>>(n, x, sqp.p, nullptr);
                finish_norm_kernel<<<1, 1024, 0, st>>>(nb_n, sqp.p, scal.p, 5);
                scale_copy_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, x, scal.p, 5, x);
                SC_LAUNCHED(3);
            }
        }
        // the loss grows geometrically with the window length: aim the next
        // window from the growth rate this one showed, growing by at most
        // one vector per flush.  Aim at 1e-10, a decade and a half below
        // semi-orthogonality (sqrt(eps) ~ 1.5e-8; windows above 1e-8 are
        // re-orthonormalised): the growth rate is not steady -- it rises as
        // Ritz values converge inside a sweep.  (Measured: aiming at 1e-11
        // C3 eigen 7.92 s / 719 flushes / max loss 6e-10; at 1e-10 7.49 s /
        // 571 / 5e-9; at 1e-9 7.56 s / 552 / 6e-6, tools/gpu_r2df.sh.)
        double target = (double)wmax;
        if (loss > 1e-16) target = (double)c * 6.0 / std::log10(loss / 1e-16);
        if (loss > 1e-9) target = std::min(target, (double)c / 2);
        wv = std::max<int64_t>(2, std::min<int64_t>({wmax, (int64_t)target, (int64_t)c + 1}));
        return SC_OK;
    }
    // Y = B[:, :m] S[:, :k]
    int ritz(double* out, int64_t ldc, int rowmajor, int64_t r0 = 0, int64_t rows = -1) {
        if (rows < 0) rows = n;
        ProfScope prof("ritz", st, 2.0 * (double)rows * m * k);
        return dgemm_launch(rows, (int)m, (int)k, B.p + r0, ld, S.p, m, out, ldc, rowmajor, st);
    }

    // eigen.py:187-239
    std::chrono::steady_clock::time_point sweep_t0 = std::chrono::steady_clock::now();
    int finish_sweep(double beta) {
        int rc;
        static const bool tdbg = std::getenv("SPECLUST_TIMING_DEBUG") != nullptr;
        if (tdbg) {
            cudaStreamSynchronize(st);
            const auto t1 = std::chrono::steady_clock::now();
            fprintf(stderr, "[lanczos] sweep %lld: %.3f ms, matvecs %lld, flushes %lld (from-0 %lld: %.1f ms, sweep %lld: %.1f ms), lookahead %lld / declined %lld\n",
                    (long long)restarts, std::chrono::duration<double, std::milli>(t1 - sweep_t0).count(),
                    (long long)matvecs, (long long)flushes, (long long)flush_n[0], flush_ms[0],
                    (long long)flush_n[1], flush_ms[1], (long long)spec_hits, (long long)spec_aborts);
            flush_ms[0] = flush_ms[1] = 0.0;
            flush_n[0] = flush_n[1] = 0;
            sweep_t0 = t1;
        }
        // T is diag(theta) + arrow at row k after a restart, tridiagonal
        // before the first one: arrowhead divide and conquer (sc_dc.cu);
        // SPECLUST_SYMEIG=dense keeps the dense Householder + QL solver
        static const bool dense = [] {
            const char* e = std::getenv("SPECLUST_SYMEIG");
            return e && std::strcmp(e, "dense") == 0;
        }();
        if (dense) {
            SC_CUDA(cudaMemcpyAsync(A.p, T.p, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
            if ((rc = symeig_launch((int)m, (int)k, A.p, Z.p, wraw.p, wsort.p, S.p, info.p, st))) return rc;
        } else {
            SC_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), st));
            if ((rc = dc_symeig_launch((int)m, restarts > 0 ? (int)k : 0, T.p, (int)k, wsort.p, S.p, st))) return rc;
        }
        last_row_kernel<<<1, 256, 0, st>>>(m, k, S.p, lastrow.p);
        SC_LAUNCHED(1);
        theta_k.assign(k, 0.0);
        std::vector<double> lr(k);
        int hinfo = 0;
        SC_CUDA(d2h_sync(theta_k.data(), wsort.p, sizeof(double) * k, st));
        SC_CUDA(d2h_sync(lr.data(), lastrow.p, sizeof(double) * k, st));
        SC_CUDA(d2h_sync(&hinfo, info.p, sizeof(int), st));
        if (hinfo) {
            state = 2;
            return fail(SC_ERR_INTERNAL, "projected eigenproblem: QL did not converge");
        }
        est_k.assign(k, 0.0);
        double worst = 0.0;
        bool converged = true;
        const double margin = n >= kWindowMinN ? 1.0 : kConvMargin;
        for (int64_t i = 0; i < k; ++i) {
            est_k[i] = beta * std::fabs(lr[i]);
            worst = std::max(worst, est_k[i]);
            if (!(est_k[i] <= margin * tol * std::max(1.0, std::fabs(theta_k[i])))) converged = false;
        }
        history.push_back(worst);
        bool verified = false;
        if (has_pending) {
            verified = true;
            for (int64_t i = 0; i < k; ++i) {
                double slack = std::max(1.0, std::fabs(theta_k[i])) * std::max(tol, 1e-12);
                if (!(std::fabs(theta_k[i] - pending[i]) <= slack)) verified = false;
            }
        }
        static const bool sweep_dbg = std::getenv("SPECLUST_TIMING_DEBUG") != nullptr;
        if (sweep_dbg) {
            int64_t nconv = 0, iworst = 0;
            double dmax = 0.0;
            for (int64_t i = 0; i < k; ++i) {
                if (est_k[i] <= margin * tol * std::max(1.0, std::fabs(theta_k[i]))) ++nconv;
                if (est_k[i] > est_k[iworst]) iworst = i;
                if (has_pending) dmax = std::max(dmax, std::fabs(theta_k[i] - pending[i]));
            }
            fprintf(stderr, "[lanczos] restart %lld: converged %lld / %lld, worst est %.2e at %lld (theta %.12f), "
                            "pending %d, max |theta - pending| %.2e, verified %d\n",
                    (long long)restarts, (long long)nconv, (long long)k, est_k[iworst], (long long)iworst,
                    theta_k[iworst], (int)has_pending, dmax, (int)verified);
        }
        if (converged && (m == n || verified)) {
            if (in_basis) {
                // result in the caller's basis memory: Ritz vectors into
                // columns 0..k-1 in place (the restart's row-chunked product)
                if ((rc = ritz_in_place())) return rc;
                Y.free();
                if ((rc = normalize_vectors())) return rc;
                state = 1;
                return SC_OK;
            }
            Y.free();
            if (!vec_out) {
                if ((rc = vectors.alloc((size_t)n * k))) return rc;
                vec_out = vectors.p;
            }
            if ((rc = ritz(vec_out, k, 1))) return rc;
            if ((rc = normalize_vectors())) return rc;
            state = 1;
            return SC_OK;
        }
        if (restarts >= max_restarts) {
            state = 2;
            char buf[160];
            snprintf(buf, sizeof(buf), "%lld restarts without verified convergence; worst residual estimate %.3e",
                     (long long)restarts, worst);
            return fail(SC_ERR_MAX_RESTARTS, buf);
        }
        ++restarts;
        if ((rc = ritz_in_place())) return rc;
        const bool coupled = !converged && beta > kBreakdownRtol * std::max(1.0, scale);
        restart_T_kernel<<<1, 1024, 0, st>>>(m, k, wsort.p, S.p, scal.p, coupled ? 1 : 0, T.p);
        SC_LAUNCHED(1);
        if (converged) {
            pending = theta_k;
            has_pending = true;
            if ((rc = fresh(k, k, false))) return rc;
        } else {
            has_pending = false;
            if (coupled) {
                scale_copy_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, w.p, scal.p, 0, B.p + k * ld);
                SC_LAUNCHED(1);
            } else {
                if ((rc = fresh(k, k, true))) return rc;
            }
        }
        j = k;
        j0 = k;
        js = k;
        return SC_OK;
    }

    // lock a deflated eigenspace after init: q0 projected off it, renormalised
    int set_locked(LockedSet* lk) {
        locked = lk;
        double* q0 = B.p;
        int rc;
        if ((rc = lk->deflate(n, q0, st)) || (rc = lk->deflate(n, q0, st)) || (rc = cgs2(q0, 0))) return rc;
        scale_copy_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, q0, scal.p, 0, q0);
        SC_LAUNCHED(1);
        SC_CUDA(cudaStreamSynchronize(st));
        return SC_OK;
    }

    // B[:, :k] = B[:, :m] S[:, :k] in place, one row chunk at a time
    // through a chunk-sized temporary (rows of the product depend only on
    // the same rows of B), so the restart needs no n x k copy
    int ritz_in_place() {
        int rc;
        const int64_t chunk = std::min<int64_t>(n, std::max<int64_t>(GB_M, ((int64_t)1 << 28) / (8 * k) / GB_M * GB_M));
        if (!Y.p && (rc = Y.alloc((size_t)chunk * k))) return rc;
        for (int64_t r0 = 0; r0 < n; r0 += chunk) {
            const int64_t rows = std::min<int64_t>(chunk, n - r0);
            if ((rc = ritz(Y.p, chunk, 0, r0, rows))) return rc;
            copy_chunk_cols_kernel<<<4 * kNumSMs, 256, 0, st>>>(rows, k, Y.p, chunk, B.p + r0, ld);
            SC_LAUNCHED(1);
        }
        return SC_OK;
    }

    int normalize_vectors() {
        int64_t nb = ceil_div(n, CN_ROWS);
        DevBuf<double> p, nr;
        int rc;
        if ((rc = p.alloc((size_t)nb * k)) || (rc = nr.alloc(k))) return rc;
        if (vec_out) {
            colsq_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(n, k, vec_out, k, 1, p.p);
            colnorm_finish_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, st>>>(nb, k, p.p, nr.p);
            scale_cols_rowmajor_kernel<<<4 * kNumSMs, 256, 0, st>>>(n, k, nr.p, vec_out);
        } else {  // the vectors in the basis columns 0..k-1
            colsq_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(n, k, B.p, 1, ld, p.p);
            colnorm_finish_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, st>>>(nb, k, p.p, nr.p);
            scale_cols_colmajor_kernel<<<4 * kNumSMs, 256, 0, st>>>(n, k, ld, nr.p, B.p);
        }
        SC_LAUNCHED(3);
        SC_CUDA(cudaStreamSynchronize(st));
        return SC_OK;
    }
};

static int residuals_launch(int64_t n, int64_t k, const int64_t* row_ptr, const int32_t* col, const double* vals,
                            const double* V, const double* theta_dev, double* res_host, cudaStream_t st) {
    int64_t nb = ceil_div(n, RS_ROWS);
    DevBuf<double> p, nr;
    int rc;
    if ((rc = p.alloc((size_t)nb * k)) || (rc = nr.alloc(k))) return rc;
    if (k <= 32)
        residual_rows_kernel<1><<<(unsigned)nb, 256, 0, st>>>(n, k, row_ptr, col, vals, V, theta_dev, p.p);
    else if (k <= 64)
        residual_rows_kernel<2><<<(unsigned)nb, 256, 0, st>>>(n, k, row_ptr, col, vals, V, theta_dev, p.p);
    else if (k <= 128)
        residual_rows_kernel<4><<<(unsigned)nb, 256, 0, st>>>(n, k, row_ptr, col, vals, V, theta_dev, p.p);
    else
        residual_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(n, k, row_ptr, col, vals, V, theta_dev, p.p);
    colnorm_finish_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, st>>>(nb, k, p.p, nr.p);
    SC_LAUNCHED(2);
    SC_CUDA(d2h_sync(res_host, nr.p, sizeof(double) * k, st));
    return SC_OK;
}

extern "C" {

int sc_lanczos_create(int64_t n, int64_t k, int64_t m, double tol, int64_t max_restarts, uint64_t seed,
                      sc_stream_t stream, sc_lanczos_t** out) {
    StreamScope stream_scope(as_stream(stream));
    auto* s = new sc_lanczos();
    int rc = s->init(n, k, m, tol, max_restarts, seed, as_stream(stream));
    if (rc) {
        delete s;
        return rc;
    }
    *out = s;
    return SC_OK;
}

void sc_lanczos_destroy(sc_lanczos_t* s) { delete s; }
int sc_lanczos_state(const sc_lanczos_t* s) { return s->state; }
const double* sc_lanczos_in_slot(const sc_lanczos_t* s) { return s->in_slot(); }
double* sc_lanczos_out_slot(sc_lanczos_t* s) { return s->w.p; }

int sc_lanczos_advance(sc_lanczos_t* s) {
    StreamScope stream_scope(s->st);
    int rc = s->advance(true);
    if (rc && rc != SC_ERR_VALUE && rc != SC_ERR_STATE) s->state = 2;
    return rc;
}

int sc_lanczos_get_stats(const sc_lanczos_t* s, sc_lanczos_stats* st) {
    st->restarts = s->restarts;
    st->breakdowns = s->breakdowns;
    st->matvecs = s->matvecs;
    st->n_history = (int64_t)std::min<size_t>(s->history.size(), 512);
    st->second_passes = s->second_passes;
    st->flushes = s->flushes;
    st->max_loss = s->max_loss;
    st->mean_window = s->flushes ? (double)s->window_sum / (double)s->flushes : 0.0;
    for (int64_t i = 0; i < st->n_history; ++i) st->history[i] = s->history[i];
    return SC_OK;
}

int sc_lanczos_ritz(const sc_lanczos_t* s, double* values, double* estimates) {
    if (s->theta_k.empty()) return fail(SC_ERR_NOT_CONVERGED, "no completed sweep");
    for (int64_t i = 0; i < s->k; ++i) {
        values[i] = s->theta_k[i];
        estimates[i] = s->est_k[i];
    }
    return SC_OK;
}

int sc_lanczos_extract(sc_lanczos_t* s, double* values, double* vectors) {
    if (s->state != 1) return fail(SC_ERR_NOT_CONVERGED, "extract called before convergence");
    for (int64_t i = 0; i < s->k; ++i) values[i] = s->theta_k[i];
    SC_CUDA(cudaMemcpyAsync(vectors, s->vec_out, sizeof(double) * s->n * s->k, cudaMemcpyDeviceToDevice, s->st));
    SC_CUDA(cudaStreamSynchronize(s->st));
    return SC_OK;
}

int sc_eigensolve_csr(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals, int64_t k,
                      int64_t m, double tol, int64_t max_restarts, uint64_t seed, double* values, double* vectors,
                      double* residuals, sc_lanczos_stats* stats, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    sc_lanczos s;
    int rc = s.init(n, k, m, tol, max_restarts, seed, st);
    if (rc) return rc;
    if ((rc = s.enable_lookahead())) return rc;
    s.vec_out = vectors;  // the converged Ritz vectors go straight to the caller's buffer
    int64_t nnz = 0;
    SC_CUDA(d2h_sync(&nnz, row_ptr + n, sizeof(int64_t), st));
    // large operators: SELL-32-sigma copy for the hundreds of matvecs
    SellMatrix sell;
    const char* fenv = std::getenv("SPECLUST_SPMV_FORMAT");
    const bool use_sell = fenv ? std::strcmp(fenv, "sell") == 0 : n >= kSellMinRows;
    if (use_sell && (rc = sell.build(n, row_ptr, col, vals, st))) return rc;
    SlowWatch sw;
    sw.lap("init", 0, 0);
    while (s.state == 0) {
        if (use_sell)
            rc = sell.spmv(s.in_slot(), s.w.p, st);
        else
            rc = spmv_launch(n, nnz, row_ptr, col, vals, s.in_slot(), s.w.p, false, st);
        if (rc) return rc;
        rc = s.advance(false);
        sw.lap("step", s.restarts, s.j);
        if (rc) {
            if (stats) sc_lanczos_get_stats(&s, stats);
            if (rc == SC_ERR_MAX_RESTARTS) {
                for (int64_t i = 0; i < k; ++i) {
                    values[i] = s.theta_k[i];
                    residuals[i] = s.est_k[i];
                }
            }
            return rc;
        }
    }
    for (int64_t i = 0; i < k; ++i) values[i] = s.theta_k[i];
    // true residuals |A v - theta v| (eigen.py:241-248)
    if ((rc = residuals_launch(n, k, row_ptr, col, vals, vectors, s.wsort.p, residuals, st))) return rc;
    if (stats) sc_lanczos_get_stats(&s, stats);
    return SC_OK;
}

int sc_eigensolve_csr_basis(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals, int64_t k,
                            int64_t m, double tol, int64_t max_restarts, uint64_t seed, double* values, double* basis,
                            double* residuals, sc_lanczos_stats* stats, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    if (!basis) return fail(SC_ERR_VALUE, "basis workspace required");
    sc_lanczos s;
    int rc = s.init(n, k, m, tol, max_restarts, seed, st, basis);
    if (rc) return rc;
    if ((rc = s.enable_lookahead())) return rc;
    int64_t nnz = 0;
    SC_CUDA(d2h_sync(&nnz, row_ptr + n, sizeof(int64_t), st));
    while (s.state == 0) {
        if ((rc = spmv_launch(n, nnz, row_ptr, col, vals, s.in_slot(), s.w.p, false, st))) return rc;
        rc = s.advance(false);
        if (rc) {
            if (stats) sc_lanczos_get_stats(&s, stats);
            if (rc == SC_ERR_MAX_RESTARTS) {
                for (int64_t i = 0; i < k; ++i) {
                    values[i] = s.theta_k[i];
                    residuals[i] = s.est_k[i];
                }
            }
            return rc;
        }
    }
    for (int64_t i = 0; i < k; ++i) values[i] = s.theta_k[i];
    // true residuals |A v - theta v| per column (eigen.py:241-248): one SpMV each
    {
        const int64_t nb = ceil_div(n, 256);
        DevBuf<double> p, nr;
        if ((rc = p.alloc(nb)) || (rc = nr.alloc(k))) return rc;
        for (int64_t c = 0; c < k; ++c) {
            const double* v = basis + c * s.ld;
            if ((rc = spmv_launch(n, nnz, row_ptr, col, vals, v, s.w.p, false, st))) return rc;
            resid_col_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(n, s.w.p, v, s.wsort.p, c, p.p);
            finish_norm_kernel<<<1, 1024, 0, st>>>(nb, p.p, nr.p, (int)c);
            SC_LAUNCHED(2);
        }
        SC_CUDA(d2h_sync(residuals, nr.p, sizeof(double) * k, st));
    }
    if (stats) sc_lanczos_get_stats(&s, stats);
    return SC_OK;
}

int64_t sc_lanczos_basis_ld(int64_t n) { return (n + 31) / 32 * 32; }

int sc_eigensolve_csr_deflate(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                              const double* d, int64_t k, int64_t m, double tol, int64_t max_restarts, uint64_t seed,
                              double* values, double* vectors, double* residuals, sc_lanczos_stats* stats,
                              int64_t* locked_out, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    *locked_out = 0;
    if (m <= 0) m = imin64(n, std::max<int64_t>(2 * k, k + 8));
    auto plain = [&]() {
        return sc_eigensolve_csr(n, row_ptr, col, vals, k, m, tol, max_restarts, seed, values, vectors, residuals,
                                 stats, stream);
    };
    if (n < kWindowMinN || k < 2 || !d) return plain();
    int rc;
    // ---- connected components of the sparsity graph (min-label propagation)
    LockedSet lk;
    int64_t c = 0;
    {
        DevBuf<int32_t> lab, lab2;
        DevBuf<int> changed;
        if ((rc = lab.alloc(n)) || (rc = lab2.alloc(n)) || (rc = changed.alloc(1))) return rc;
        iota_i32_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, lab.p);
        SC_LAUNCHED(1);
        for (int it = 0; it < 100000; ++it) {
            SC_CUDA(cudaMemsetAsync(changed.p, 0, sizeof(int), st));
            cc_propagate_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, row_ptr, col, lab.p, lab2.p, changed.p);
            SC_LAUNCHED(1);
            std::swap(lab.p, lab2.p);
            int h = 0;
            SC_CUDA(d2h_sync(&h, changed.p, sizeof(int), st));
            if (!h) break;
        }
        DevBuf<int64_t> flag, rank, tmp;
        if ((rc = flag.alloc(n)) || (rc = rank.alloc(n + 1)) || (rc = tmp.alloc(ceil_div(n, 1024) + 2))) return rc;
        cc_roots_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, lab.p, flag.p);
        SC_LAUNCHED(1);
        if ((rc = exclusive_scan_i64(n, flag.p, rank.p, tmp.p, st))) return rc;
        SC_CUDA(d2h_sync(&c, rank.p + n, sizeof(int64_t), st));
        // one component (nothing to lock), or at least k copies of eigenvalue 1
        // (the wanted set is then a subset of the degenerate space): the
        // reference's procedure unchanged
        if (c <= 1 || c >= k) return plain();
        if ((rc = lk.comp.alloc(n))) return rc;
        cc_number_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, lab.p, rank.p, lk.comp.p);
        SC_LAUNCHED(1);
    }
    lk.c = c;
    if ((rc = lk.u.alloc(n)) || (rc = lk.h.alloc(c)) || (rc = lk.bk.init(n, c)) || (rc = lk.bk.run(lk.comp.p, st)) ||
        (rc = lk.plan(st)))
        return rc;
    DevBuf<double> dsum, y, r, theta_l, res_l;
    if ((rc = dsum.alloc(c)) || (rc = y.alloc(n)) || (rc = r.alloc(n)) || (rc = theta_l.alloc(c)) ||
        (rc = res_l.alloc(c)))
        return rc;
    if ((rc = lk.seg_dot(d, nullptr, dsum.p, st))) return rc;
    locked_vec_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d, lk.comp.p, dsum.p, lk.u.p);
    SC_LAUNCHED(1);
    int64_t nnz = 0;
    SC_CUDA(d2h_sync(&nnz, row_ptr + n, sizeof(int64_t), st));
    // Rayleigh quotients and true residuals of the locked vectors; the
    // operator must be D^-1/2 W D^-1/2 for this d (else: the plain solve)
    if ((rc = spmv_launch(n, nnz, row_ptr, col, vals, lk.u.p, y.p, false, st))) return rc;
    if ((rc = lk.seg_dot(lk.u.p, y.p, theta_l.p, st))) return rc;
    locked_resid_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, lk.comp.p, lk.u.p, y.p, theta_l.p, r.p);
    if ((rc = lk.seg_dot(r.p, nullptr, res_l.p, st))) return rc;
    SC_LAUNCHED(1);
    std::vector<double> th(c), rs(c);
    SC_CUDA(d2h_sync(th.data(), theta_l.p, sizeof(double) * c, st));
    SC_CUDA(d2h_sync(rs.data(), res_l.p, sizeof(double) * c, st));
    for (int64_t q = 0; q < c; ++q) {
        rs[q] = std::sqrt(rs[q]);
        if (!(rs[q] <= 1e-3 * tol && std::fabs(th[q] - 1.0) <= 1e-10)) return plain();
    }
    // ---- Lanczos on the orthogonal complement: k - c pairs, subspace m - c
    const int64_t kr = k - c, mr = m - c;
    sc_lanczos s;
    if ((rc = s.init(n, kr, mr, tol, max_restarts, seed, st))) return rc;
    if ((rc = s.enable_lookahead())) return rc;
    if ((rc = s.set_locked(&lk))) return rc;
    DevBuf<double> rv;
    if ((rc = rv.alloc((size_t)n * kr))) return rc;
    s.vec_out = rv.p;
    SlowWatch sw;
    while (s.state == 0) {
        if ((rc = spmv_launch(n, nnz, row_ptr, col, vals, s.in_slot(), s.w.p, false, st))) return rc;
        rc = s.advance(false);
        sw.lap("step", s.restarts, s.j);
        if (rc) {
            if (stats) sc_lanczos_get_stats(&s, stats);
            if (rc == SC_ERR_MAX_RESTARTS) {
                for (int64_t i = 0; i < k; ++i) {
                    values[i] = i < c ? th[i] : s.theta_k[i - c];
                    residuals[i] = i < c ? rs[i] : s.est_k[i - c];
                }
            }
            return rc;
        }
    }
    // ---- assemble: locked pairs first (eigenvalue 1 >= every other), in
    // descending Rayleigh quotient (ties by component order), then the rest
    std::vector<int64_t> ord(c), col_of(c);
    for (int64_t q = 0; q < c; ++q) ord[q] = q;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return th[a] > th[b]; });
    for (int64_t j = 0; j < c; ++j) col_of[ord[j]] = j;
    DevBuf<int64_t> dcol;
    if ((rc = dcol.alloc(c))) return rc;
    SC_CUDA(cudaMemcpyAsync(dcol.p, col_of.data(), sizeof(int64_t) * c, cudaMemcpyHostToDevice, st));
    assemble_vectors_kernel<<<8 * kNumSMs, 256, 0, st>>>(n, k, c, lk.comp.p, dcol.p, lk.u.p, rv.p, vectors);
    SC_LAUNCHED(1);
    std::vector<double> res_r(kr);
    if ((rc = residuals_launch(n, kr, row_ptr, col, vals, rv.p, s.wsort.p, res_r.data(), st))) return rc;
    for (int64_t j = 0; j < c; ++j) {
        values[j] = th[ord[j]];
        residuals[j] = rs[ord[j]];
    }
    for (int64_t j = 0; j < kr; ++j) {
        values[c + j] = s.theta_k[j];
        residuals[c + j] = res_r[j];
    }
    if (stats) sc_lanczos_get_stats(&s, stats);
    SC_CUDA(cudaStreamSynchronize(st));
    *locked_out = c;
    return SC_OK;
}

int sc_symmetry_probe(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                      uint64_t seed, double* ratio_out, sc_stream_t stream) {
    // eigen.py:279-288: three random (x, y) pairs; ratio = |x'Ay - y'Ax| / (|x| |y|)
    // (the caller multiplies the tolerance by max(1, max|a|))
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    *ratio_out = 0.0;
    if (n <= 0) return SC_OK;
    int64_t nnz = 0;
    SC_CUDA(d2h_sync(&nnz, row_ptr + n, sizeof(int64_t), st));
    DevBuf<double> x, y, ax, ay, part, out;
    int64_t nb = ceil_div(n, 256);
    int rc;
    if ((rc = x.alloc(n)) || (rc = y.alloc(n)) || (rc = ax.alloc(n)) || (rc = ay.alloc(n)) ||
        (rc = part.alloc(nb)) || (rc = out.alloc(4)))
        return rc;
    double worst = 0.0;
    for (int t = 0; t < 3; ++t) {
        uint64_t sid = (1ull << 40) + 2 * (uint64_t)t;
        fill_normal_kernel<<<(unsigned)nb, 256, 0, st>>>(n, seed, sid, x.p);
        fill_normal_kernel<<<(unsigned)nb, 256, 0, st>>>(n, seed, sid + 1, y.p);
        SC_LAUNCHED(2);
        if ((rc = spmv_launch(n, nnz, row_ptr, col, vals, y.p, ay.p, false, st))) return rc;
        if ((rc = spmv_launch(n, nnz, row_ptr, col, vals, x.p, ax.p, false, st))) return rc;
        dot_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(n, x.p, ay.p, y.p, ax.p, part.p);
        finish_sum_kernel<<<1, 1024, 0, st>>>(nb, part.p, out.p, 0);
        sumsq_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(n, x.p, part.p, nullptr);
        finish_norm_kernel<<<1, 1024, 0, st>>>(nb, part.p, out.p, 1);
        sumsq_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(n, y.p, part.p, nullptr);
        finish_norm_kernel<<<1, 1024, 0, st>>>(nb, part.p, out.p, 2);
        SC_LAUNCHED(6);
        double h[3];
        SC_CUDA(d2h_sync(h, out.p, sizeof(double) * 3, st));
        double denom = h[1] * h[2];
        double r = denom > 0 ? std::fabs(h[0]) / denom : 0.0;
        worst = std::max(worst, r);
    }
    // scale by max(1, max|a|) (eigen.py:282, 285)
    DevBuf<unsigned long long> vmax;
    if ((rc = vmax.alloc(1))) return rc;
    SC_CUDA(cudaMemsetAsync(vmax.p, 0, sizeof(unsigned long long), st));
    if (nnz > 0) {
        absmax_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nnz, 256), 4 * kNumSMs), 256, 0, st>>>(nnz, vals, vmax.p);
        SC_LAUNCHED(1);
    }
    unsigned long long vb = 0;
    SC_CUDA(d2h_sync(&vb, vmax.p, sizeof(vb), st));
    double vm;
    std::memcpy(&vm, &vb, sizeof(vm));
    *ratio_out = worst / std::max(1.0, vm);
    return SC_OK;
}

// ---- per-shard building blocks of the row-sharded eigensolver -------------------
int sc_gemv_t_f64(int64_t n, int64_t ld, int64_t ncols, const double* B, const double* w, double* h,
                  sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    if (ncols <= 0) return SC_OK;
    if (n <= 0) {
        SC_CUDA(cudaMemsetAsync(h, 0, sizeof(double) * ncols, st));
        return SC_OK;
    }
    const int rpb = gemv_t_rows_per_block(n);
    const int64_t nb = ceil_div(n, rpb);
    DevBuf<double> part;
    if (int rc = part.alloc((size_t)nb * ncols)) return rc;
    ProfScope prof("reorth", st, (double)n * ncols * 8.0);
    gemv_t_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(n, ld, (int)ncols, rpb, B, w, part.p, nullptr);
    reduce_cols_kernel<<<(unsigned)ceil_div(ncols * 32, 256), 256, 0, st>>>(nb, (int)ncols, part.p, h);
    SC_LAUNCHED(2);
    return SC_OK;
}

int sc_gemv_n_f64(int64_t n, int64_t ld, int64_t ncols, const double* B, const double* h, double* w, double* sq_out,
                  sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    if (n <= 0) {
        if (sq_out) SC_CUDA(cudaMemsetAsync(sq_out, 0, sizeof(double), st));
        return SC_OK;
    }
    const int64_t nb = ceil_div(n, GN_THREADS);
    DevBuf<double> sq, scal;
    if (sq_out) {
        if (int rc = sq.alloc(nb)) return rc;
    }
    ProfScope prof("reorth", st, (double)n * ncols * 8.0);
    if (ncols > 0) {
        gemv_n_update_kernel<<<(unsigned)nb, GN_THREADS, sizeof(double) * (size_t)ncols, st>>>(
            n, ld, (int)ncols, B, h, w, sq_out ? sq.p : nullptr);
        SC_LAUNCHED(1);
    } else if (sq_out) {
        sumsq_partial_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, w, sq.p, nullptr);
        SC_LAUNCHED(1);
    }
    if (sq_out) {
        const int64_t parts = ncols > 0 ? nb : ceil_div(n, 256);
        finish_sum_kernel<<<1, 1024, 0, st>>>(parts, sq.p, sq_out, 0);
        SC_LAUNCHED(1);
    }
    return SC_OK;
}

// dst = src / div (IEEE division, as `w / beta` in eigen.py:172)
int sc_div_copy_f64(int64_t n, const double* src, double div, double* dst, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    if (n <= 0) return SC_OK;
    div_copy_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, src, div, dst);
    SC_LAUNCHED(1);
    return SC_OK;
}

int sc_fill_normal(int64_t n, int64_t offset, uint64_t seed, uint64_t stream_id, double* out, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    if (n <= 0) return SC_OK;
    fill_normal_offset_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, offset, seed, stream_id, out);
    SC_LAUNCHED(1);
    return SC_OK;
}

int sc_symeig_f64(int64_t m, int64_t kout, const double* T, double* theta, double* S, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    if (m < 1 || kout < 1 || kout > m) return fail(SC_ERR_VALUE, "symeig needs 1 <= kout <= m");
    DevBuf<double> A, Z, wraw;
    DevBuf<int> info;
    int rc;
    if ((rc = A.alloc((size_t)m * m)) || (rc = Z.alloc((size_t)m * m)) || (rc = wraw.alloc(m)) ||
        (rc = info.alloc(1)))
        return rc;
    SC_CUDA(cudaMemcpyAsync(A.p, T, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
    if ((rc = symeig_launch((int)m, (int)kout, A.p, Z.p, wraw.p, theta, S, info.p, st))) return rc;
    int h = 0;
    SC_CUDA(d2h_sync(&h, info.p, sizeof(int), st));
    if (h) return fail(SC_ERR_INTERNAL, "projected eigenproblem: QL did not converge");
    return SC_OK;
}

int sc_dgemm_tall(int64_t n, int64_t kk, int64_t kc, const double* A, int64_t lda, const double* S, int64_t lds,
                  double* C, int64_t ldc, int rowmajor, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    if (n <= 0 || kc <= 0) return SC_OK;
    ProfScope prof("ritz", st, 2.0 * (double)n * kk * kc);
    return dgemm_launch(n, (int)kk, (int)kc, A, lda, S, lds, C, ldc, rowmajor, st);
}

}  // extern "C"
