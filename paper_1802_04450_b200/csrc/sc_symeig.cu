// Dense symmetric eigensolver for the Lanczos projected matrix (m x m),
// entirely on device: Householder tridiagonalisation, explicit Q, implicit
// QL with Wilkinson-type shifts (rotation chains computed by one thread and
// applied to the rows of Q by the whole CTA), then a stable descending sort.
//
// Replaces np.linalg.eigh(proj) + argsort(-theta, kind="stable") in
// eigen.py:189-192 (the reference's LAPACK dsyevd call on the host).
#include "sc_common.cuh"
#include "sc_symeig.cuh"

namespace sc {

constexpr int SE_THREADS = 1024;

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

// a: m x m column-major symmetric (destroyed); z: m x m output eigenvectors
// (column j <-> eigenvalue w[j], unsorted); info: 0 ok, >0 QL failure.
__global__ void __launch_bounds__(SE_THREADS, 1) symeig_kernel(int m, double* __restrict__ a,
                                                                double* __restrict__ z,
                                                                double* __restrict__ w, int* info) {
    extern __shared__ double sm[];
    double* d = sm;            // m
    double* e = d + m;         // m
    double* v = e + m;         // m (Householder vector / rotation cos)
    double* q = v + m;         // m (p, q vectors / rotation sin)
    double* red = q + m;       // 40
    __shared__ double s_alpha, s_beta;
    __shared__ int s_lo, s_hi, s_state;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;

    // ---- 1. tridiagonalisation; reflector k stored in a[k+1.., k]
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
        e[k] = s_alpha;  // every thread writes the same value
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
    for (int i = tid; i < m; i += nt) d[i] = a[(size_t)i * m + i];
    if (tid == 0) {
        if (m >= 2) e[m - 2] = a[(size_t)(m - 2) * m + (m - 1)];
        e[m - 1] = 0.0;
    }
    __syncthreads();

    // ---- 2. Q = H_0 H_1 ... H_{m-3}, accumulated backwards into z
    for (int idx = tid; idx < m * m; idx += nt) z[idx] = (idx % (m + 1) == 0) ? 1.0 : 0.0;
    __syncthreads();
    for (int k = m - 3; k >= 0; --k) {
        const int len = m - k - 1;
        const double* vk = a + (size_t)k * m + (k + 1);
        bool zero = true;
        for (int i = 0; i < len && zero; ++i) zero = vk[i] == 0.0;  // uniform branch
        if (zero) continue;
        for (int i = tid; i < len; i += nt) v[i] = vk[i];
        __syncthreads();
        // w_j = v^T Q[k+1:, j] for columns j >= k+1  (warp per column)
        for (int j = warp; j < len; j += nw) {
            const double* cj = z + (size_t)(k + 1 + j) * m + (k + 1);
            double acc = 0.0;
            for (int i = lane; i < len; i += 32) acc = fma(v[i], cj[i], acc);
            acc = warp_sum(acc);
            if (lane == 0) q[j] = acc;
        }
        __syncthreads();
        for (int idx = tid; idx < len * len; idx += nt) {
            int cJ = idx / len, r = idx - cJ * len;
            z[(size_t)(k + 1 + cJ) * m + (k + 1 + r)] -= 2.0 * v[r] * q[cJ];
        }
        __syncthreads();
    }

    // ---- 3. implicit QL on (d, e); rotations applied to the rows of z
    double* cs = v;
    double* sn = q;
    if (tid == 0) {
        s_state = 0;
        *info = 0;
    }
    __syncthreads();
    int l = 0, iter = 0;  // only meaningful in thread 0
    while (true) {
        if (tid == 0) {
            s_lo = s_hi = -1;
            while (l < m) {
                int mm;
                for (mm = l; mm < m - 1; ++mm) {
                    double dd = fabs(d[mm]) + fabs(d[mm + 1]);
                    if (fabs(e[mm]) + dd == dd) break;
                }
                if (mm == l) {
                    ++l;
                    iter = 0;
                    continue;
                }
                if (++iter > 60) {
                    *info = l + 1;
                    l = m;
                    break;
                }
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = hypot(g, 1.0);
                g = d[mm] - d[l] + e[l] / (g + (g >= 0.0 ? fabs(r) : -fabs(r)));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                bool early = false;
                int cnt = 0;
                for (i = mm - 1; i >= l; --i) {
                    double f = s * e[i], b = c * e[i];
                    // |f|, |g| are O(|T|) here: plain sqrt instead of hypot's
                    // rescaling, one reciprocal instead of two divisions
                    r = sqrt(fma(f, f, g * g));
                    e[i + 1] = r;
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[mm] = 0.0;
                        early = true;
                        break;
                    }
                    const double ri = 1.0 / r;
                    s = f * ri;
                    c = g * ri;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    p = s * r;
                    d[i + 1] = g + p;
                    g = c * r - b;
                    cs[cnt] = c;
                    sn[cnt] = s;
                    ++cnt;
                }
                if (!(early && i >= l)) {
                    d[l] -= p;
                    e[l] = g;
                    e[mm] = 0.0;
                }
                if (cnt > 0) {
                    s_hi = mm - 1;          // first rotation acts on (mm-1, mm)
                    s_lo = mm - cnt;        // last rotation acts on (mm-cnt, mm-cnt+1)
                    break;                  // hand the chain to the CTA
                }
            }
            if (l >= m && s_hi < 0) s_state = 1;
        }
        __syncthreads();
        if (s_state) break;
        const int hi = s_hi, lo = s_lo;
        for (int r = tid; r < m; r += nt) {
            double carry = z[(size_t)(hi + 1) * m + r];  // z[r][i+1]
            int t = 0;
            for (int i = hi; i >= lo; --i, ++t) {
                double c = cs[t], s = sn[t];
                double zi = z[(size_t)i * m + r];
                z[(size_t)(i + 1) * m + r] = s * zi + c * carry;
                carry = c * zi - s * carry;
            }
            z[(size_t)lo * m + r] = carry;
        }
        __syncthreads();
    }
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
    size_t smem = sizeof(double) * (4 * (size_t)m + 40);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(symeig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(symeig_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    if (smem > 200 * 1024) return fail(SC_ERR_VALUE, "projected matrix too large for the device eigensolver");
    {
        ProfScope prof("symeig", st, 0.0);
        symeig_kernel<<<1, SE_THREADS, smem, st>>>(m, a, z, w_raw, info);
        symeig_sort_kernel<<<1, 1024, sizeof(int) * (size_t)m, st>>>(m, kout, w_raw, z, w_sorted, z_sorted);
    }
    SC_LAUNCHED(2);
    return SC_OK;
}

}  // namespace sc
