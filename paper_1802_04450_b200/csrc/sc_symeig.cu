// Dense symmetric eigensolver for the Lanczos projected matrix (m x m),
// entirely on device:
//   1. Householder tridiagonalisation (one CTA, matrix in global/L2);
//   2. eigenvectors by row blocks: each of C CTAs owns RB rows of Z in shared
//      memory, forms its rows of Q = H_0 ... H_{m-3} (row-local: z <- z H_k),
//      then runs the implicit QL iteration with Wilkinson-type shifts on its
//      own copy of (d, e) — every CTA computes the identical rotation chains,
//      so no inter-CTA traffic — and applies each chain to its rows;
//   3. a stable descending sort.
// The row-block split keeps the rotation sweeps in shared memory (the
// serial carry of a QL chain through global memory was the cost of the
// single-CTA version: 13 ms per m=200 solve).
//
// Replaces np.linalg.eigh(proj) + argsort(-theta, kind="stable") in
// eigen.py:189-192 (the reference's LAPACK dsyevd call on the host).
#include <algorithm>

#include "sc_common.cuh"
#include "sc_symeig.cuh"

namespace sc {

constexpr int SE_THREADS = 1024;
constexpr int SE_SMEM_MAX = 200 * 1024;

__device__ __forceinline__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = (int)threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// a: m x m column-major symmetric.  On exit reflector k (unit v, H = I - 2vv^T
// acting on rows k+1..) is in a[k*m + k+1 ..] (all zero: no reflection), the
// diagonal d_i in a[i*m + i] and the off-diagonal e_i in a[(i+1)*m + i].
__global__ void __launch_bounds__(SE_THREADS, 1) symeig_tridiag_kernel(int m, double* __restrict__ a) {
    extern __shared__ double sm[];
    double* v = sm;      // m
    double* q = v + m;   // m
    double* red = q + m; // 40
    __shared__ double s_alpha, s_beta;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;

    for (int k = 0; k + 2 < m; ++k) {
        const int len = m - k - 1;  // rows k+1 .. m-1
        double* col = a + (size_t)k * m;
        double part = 0.0;
        for (int i = k + 2 + tid; i < m; i += nt) part = fma(col[i], col[i], part);
        double sigma = block_sum(part, red);
        if (tid == 0) {
            double x0 = col[k + 1];
            if (sigma == 0.0) {
                s_alpha = x0;
                s_beta = 0.0;  // no reflection
            } else {
                double nx = sqrt(x0 * x0 + sigma);
                double alpha = x0 >= 0.0 ? -nx : nx;
                double v0 = x0 - alpha;
                s_alpha = alpha;
                s_beta = 1.0 / sqrt(v0 * v0 + sigma);  // normaliser of v
                col[k + 1] = v0;
            }
        }
        __syncthreads();
        const double beta = s_beta;
        if (tid == 0) a[(size_t)(k + 1) * m + k] = s_alpha;  // e_k (row k, column k+1)
        if (beta == 0.0) {
            for (int i = k + 1 + tid; i < m; i += nt) col[i] = 0.0;
            __syncthreads();
            continue;
        }
        for (int i = tid; i < len; i += nt) {
            double vi = col[k + 1 + i] * beta;
            v[i] = vi;
            col[k + 1 + i] = vi;
        }
        __syncthreads();
        // p = A22 v  (warp per output row, lanes along the contiguous column)
        for (int i = warp; i < len; i += nw) {
            const double* ci = a + (size_t)(k + 1 + i) * m + (k + 1);
            double acc = 0.0;
            for (int j = lane; j < len; j += 32) acc = fma(ci[j], v[j], acc);
            acc = warp_sum(acc);
            if (lane == 0) q[i] = acc;
        }
        __syncthreads();
        double kp = 0.0;
        for (int i = tid; i < len; i += nt) kp = fma(v[i], q[i], kp);
        double K = block_sum(kp, red);
        for (int i = tid; i < len; i += nt) q[i] = q[i] - K * v[i];
        __syncthreads();
        // A22 -= 2 (v q^T + q v^T)
        for (int idx = tid; idx < len * len; idx += nt) {
            int cI = idx / len, r = idx - cI * len;
            double* p = a + (size_t)(k + 1 + cI) * m + (k + 1 + r);
            *p -= 2.0 * (v[r] * q[cI] + q[r] * v[cI]);
        }
        __syncthreads();
    }
    if (m >= 2 && tid == 0) a[(size_t)(m - 1) * m + (m - 2)] = a[(size_t)(m - 2) * m + (m - 1)];
}

// named CTA barriers (non-.aligned forms, after a warp reconvergence)
__device__ __forceinline__ void named_sync(int id, int n) {
    __syncwarp();
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    __syncwarp();
    asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// CTA b: rows [b*rb, b*rb + rb) of the eigenvector matrix Z = Q * (QL rotations)
__global__ void __launch_bounds__(256) symeig_ql_kernel(int m, int rb, const double* __restrict__ a,
                                                        double* __restrict__ z, double* __restrict__ w,
                                                        int* __restrict__ info, double* __restrict__ zglob) {
    extern __shared__ double sm[];
    // the CTA's rows of Z: shared memory, or (large m, one wave) a private
    // global block that stays L2-resident
    double* zb = zglob ? zglob + (size_t)blockIdx.x * m * rb : sm;  // zb[i * rb + rr] = Z[r0 + rr][i]
    double* d = zglob ? sm : zb + (size_t)m * rb;                   // m
    double* e = d + m;                     // m
    double* v = e + m;                     // m
    double* cs2 = v + m;                   // 2 x m (double-buffered rotation chains)
    double* sn2 = cs2 + 2 * (size_t)m;     // 2 x m
    __shared__ int s_lo2[2], s_hi2[2], s_zero;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int r0 = blockIdx.x * rb;
    const int rows = min(rb, m - r0);

    for (int i = tid; i < m; i += nt) {
        d[i] = a[(size_t)i * m + i];
        e[i] = i + 1 < m ? a[(size_t)(i + 1) * m + i] : 0.0;
    }
    for (int idx = tid; idx < m * rb; idx += nt) {
        const int i = idx / rb, rr = idx - i * rb;
        zb[idx] = (r0 + rr == i) ? 1.0 : 0.0;
    }
    __syncthreads();

    // ---- Q rows: z <- z H_k for k = 0 .. m-3 (Q = H_0 H_1 ... H_{m-3})
    for (int k = 0; k + 2 < m; ++k) {
        const int len = m - k - 1;
        const double* vk = a + (size_t)k * m + (k + 1);
        if (tid == 0) s_zero = 1;
        __syncthreads();
        for (int i = tid; i < len; i += nt) {
            const double x = vk[i];
            v[i] = x;
            if (x != 0.0) s_zero = 0;
        }
        __syncthreads();
        const int zero = s_zero;
        __syncthreads();  // everyone has read s_zero before thread 0 resets it
        if (zero) continue;  // uniform
        // warp-cooperative per row: 8 lanes per row, rows strided over the CTA
        // (the loop bound is CTA-uniform so every lane reaches the shuffles)
        const int g = tid >> 3, sub = tid & 7, ng = nt >> 3;
        for (int rbase = 0; rbase < rb; rbase += ng) {
            const int rr = rbase + g;
            double dot = 0.0;
            if (rr < rows)
                for (int i = sub; i < len; i += 8) dot = fma(zb[(size_t)(k + 1 + i) * rb + rr], v[i], dot);
            dot += __shfl_xor_sync(0xffffffffu, dot, 1);
            dot += __shfl_xor_sync(0xffffffffu, dot, 2);
            dot += __shfl_xor_sync(0xffffffffu, dot, 4);
            if (rr < rows)
                for (int i = sub; i < len; i += 8) zb[(size_t)(k + 1 + i) * rb + rr] -= 2.0 * dot * v[i];
        }
        __syncthreads();
    }

    // ---- implicit QL on (d, e), pipelined: warp 0 forms the rotation chains
    // (lane 0 the serial chain, the whole warp the search for the next
    // negligible off-diagonal) into a double buffer while warps 1..7 apply
    // the previous chain to the CTA's rows; named barriers FULL[b] / EMPTY[b]
    // hand the buffers over.  Same rotations in the same order as a serial
    // compute-then-apply loop.
    if (tid == 0 && blockIdx.x == 0) *info = 0;
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    constexpr int BAR_FULL = 1, BAR_EMPTY = 3;  // ids 1,2 and 3,4
    if (warp == 0) {
        int l = 0, iter = 0, c = 0;
        bool pending[2] = {false, false};  // a handed-over chain whose EMPTY is not yet awaited
        while (true) {
            const int buf = c & 1;
            if (pending[buf]) {
                named_sync(BAR_EMPTY + buf, nt);
                pending[buf] = false;
            }
            double* csb = cs2 + (size_t)buf * m;
            double* snb = sn2 + (size_t)buf * m;
            int lo = -1, hi = -1;
            while (l < m) {
                int mm = m - 1;
                for (int base = l; base < m - 1; base += 32) {
                    const int idx = base + lane;
                    bool neg = false;
                    if (idx < m - 1) {
                        const double dd = fabs(d[idx]) + fabs(d[idx + 1]);
                        neg = fabs(e[idx]) + dd == dd;
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, neg);
                    if (bal) {
                        mm = base + __ffs(bal) - 1;
                        break;
                    }
                }
                if (mm == l) {
                    ++l;
                    iter = 0;
                    continue;
                }
                if (++iter > 60) {
                    if (lane == 0 && blockIdx.x == 0) *info = l + 1;
                    l = m;
                    break;
                }
                int cnt = 0;
                if (lane == 0) {
                    double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                    double r = hypot(g, 1.0);
                    g = d[mm] - d[l] + e[l] / (g + (g >= 0.0 ? fabs(r) : -fabs(r)));
                    double s = 1.0, c2 = 1.0, p = 0.0;
                    int i;
                    bool early = false;
                    // The chain is serial, so its latency is the QL cost: d[i],
                    // e[i] are prefetched into registers one rotation ahead, and
                    // one rsqrt (1 ulp) replaces sqrt + reciprocal; c, s stay
                    // orthonormal to ~1 ulp.  |f|, |g| are O(|T|): no rescaling.
                    double ei = e[mm - 1], di = d[mm - 1], di1 = d[mm];
                    for (i = mm - 1; i >= l; --i) {
                        const double e_nx = i > l ? e[i - 1] : 0.0;
                        const double d_nx = i > l ? d[i - 1] : 0.0;
                        const double f = s * ei, b = c2 * ei;
                        const double r2 = fma(f, f, g * g);
                        if (r2 == 0.0) {
                            e[i + 1] = 0.0;
                            d[i + 1] = di1 - p;
                            e[mm] = 0.0;
                            early = true;
                            break;
                        }
                        const double ri = rsqrt(r2);
                        e[i + 1] = r2 * ri;
                        s = f * ri;
                        c2 = g * ri;
                        g = di1 - p;
                        r = (di - g) * s + 2.0 * c2 * b;
                        p = s * r;
                        d[i + 1] = g + p;
                        g = c2 * r - b;
                        csb[cnt] = c2;
                        snb[cnt] = s;
                        ++cnt;
                        di1 = di;  // d[i] is untouched by this rotation
                        di = d_nx;
                        ei = e_nx;
                    }
                    if (!(early && i >= l)) {
                        d[l] -= p;
                        e[l] = g;
                        e[mm] = 0.0;
                    }
                }
                cnt = __shfl_sync(0xffffffffu, cnt, 0);
                __syncwarp();  // lane 0's d / e updates before the next search
                if (cnt > 0) {
                    hi = mm - 1;    // first rotation acts on (mm-1, mm)
                    lo = mm - cnt;  // last rotation acts on (mm-cnt, mm-cnt+1)
                    break;
                }
            }
            if (lane == 0) {
                s_lo2[buf] = lo;
                s_hi2[buf] = hi;
            }
            named_arrive(BAR_FULL + buf, nt);
            if (lo < 0) {  // finished: settle the other buffer's hand-over
                if (pending[buf ^ 1]) named_sync(BAR_EMPTY + (buf ^ 1), nt);
                break;
            }
            pending[buf] = true;
            ++c;
        }
    } else {
        for (int c = 0;; ++c) {
            const int buf = c & 1;
            named_sync(BAR_FULL + buf, nt);
            const int hi = s_hi2[buf], lo = s_lo2[buf];
            if (lo < 0) break;
            const double* csb = cs2 + (size_t)buf * m;
            const double* snb = sn2 + (size_t)buf * m;
            for (int rr = tid - 32; rr < rows; rr += nt - 32) {
                double carry = zb[(size_t)(hi + 1) * rb + rr];
                int t = 0;
                for (int i = hi; i >= lo; --i, ++t) {
                    const double c2 = csb[t], s = snb[t];
                    const double zi = zb[(size_t)i * rb + rr];
                    zb[(size_t)(i + 1) * rb + rr] = s * zi + c2 * carry;
                    carry = c2 * zi - s * carry;
                }
                zb[(size_t)lo * rb + rr] = carry;
            }
            named_arrive(BAR_EMPTY + buf, nt);
        }
    }
    __syncthreads();
    for (int idx = tid; idx < m * rows; idx += nt) {
        const int i = idx / rows, rr = idx - i * rows;
        z[(size_t)i * m + r0 + rr] = zb[(size_t)i * rb + rr];
    }
    if (blockIdx.x == 0)
        for (int i = tid; i < m; i += nt) w[i] = d[i];
}

// stable descending order: rank_i = #{j : w_j > w_i or (w_j == w_i and j < i)}
__global__ void symeig_sort_kernel(int m, int kout, const double* __restrict__ w,
                                   const double* __restrict__ z, double* __restrict__ ws,
                                   double* __restrict__ zs) {
    extern __shared__ int rank_of[];  // m
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        double wi = w[i];
        int r = 0;
        for (int j = 0; j < m; ++j) {
            double wj = w[j];
            r += (wj > wi) || (wj == wi && j < i);
        }
        rank_of[i] = r;
        ws[r] = wi;
    }
    __syncthreads();
    // copy the first kout sorted columns
    for (int i = 0; i < m; ++i) {
        int r = rank_of[i];
        if (r >= kout) continue;
        for (int row = threadIdx.x; row < m; row += blockDim.x)
            zs[(size_t)r * m + row] = z[(size_t)i * m + row];
    }
}

int symeig_launch(int m, int kout, double* a, double* z, double* w_raw, double* w_sorted,
                  double* z_sorted, int* info, cudaStream_t st) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(symeig_tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SE_SMEM_MAX);
        cudaFuncSetAttribute(symeig_ql_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SE_SMEM_MAX);
        cudaFuncSetAttribute(symeig_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SE_SMEM_MAX);
        attr_set = true;
    }
    // rows per CTA: as many as fit (at most 64) next to the 7 m-vectors
    int rb = 64;
    while (rb > 1 && sizeof(double) * ((size_t)m * rb + 7 * (size_t)m) > (size_t)SE_SMEM_MAX) rb >>= 1;
    // every CTA recomputes the same rotation chains: when the shared-memory
    // row blocks need more CTAs than one wave, the rows go to global blocks
    // (L2-resident) with one CTA per SM instead
    const bool global_z = (m + rb - 1) / rb > kNumSMs;
    if (global_z) rb = (m + kNumSMs - 1) / kNumSMs;
    const size_t ql_smem = sizeof(double) * ((global_z ? 0 : (size_t)m * rb) + 7 * (size_t)m);
    if (ql_smem > (size_t)SE_SMEM_MAX) return fail(SC_ERR_VALUE, "projected matrix too large for the device eigensolver");
    const int nblk = (m + rb - 1) / rb;
    DevBuf<double> zglob;
    if (global_z)
        if (int rc = zglob.alloc((size_t)nblk * m * rb)) return rc;
    {
        ProfScope prof("symeig", st, 0.0);
        symeig_tridiag_kernel<<<1, SE_THREADS, sizeof(double) * (2 * (size_t)m + 40), st>>>(m, a);
        symeig_ql_kernel<<<nblk, 256, ql_smem, st>>>(m, rb, a, z, w_raw, info, zglob.p);
        symeig_sort_kernel<<<1, 1024, sizeof(int) * (size_t)m, st>>>(m, kout, w_raw, z, w_sorted, z_sorted);
    }
    SC_LAUNCHED(3);
    return SC_OK;
}

}  // namespace sc
