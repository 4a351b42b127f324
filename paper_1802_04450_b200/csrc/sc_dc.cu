// Projected eigensolver of the thick-restart Lanczos (replaces
// np.linalg.eigh(proj) + argsort(-theta, kind="stable"), eigen.py:189-192)
// by an arrowhead divide and conquer that uses the structure of proj:
//
//   rows/cols 0..p-1 : diag(theta) (the retained Ritz values, eigen.py:226)
//   row/col p        : the couplings beta*s[m-1,:k] (eigen.py:233-235)
//   rows p..m-1      : the tridiagonal Lanczos recurrence (eigen.py:159, 173)
//
// (p = 0 in the first sweep: T is tridiagonal).  Tearing T at row p gives an
// arrowhead whose left part is already diagonal and whose right part is the
// tridiagonal tail; the tail is solved recursively by tearing at its middle
// row (Gu & Eisenstat), so every merge is one arrowhead eigenproblem
//
//   [[diag(d), z], [z^T, alpha]]  with  d = eigenvalues of the two children,
//   z = coupling * (last row of the left / first row of the right child's
//   eigenvectors),  alpha = the torn diagonal entry,
//
// solved by: stable sort of d, deflation of tiny z and of (nearly) equal d
// (Givens rotation, LAPACK dlaed2's test), one warp per root of the secular
// equation alpha - lam + sum z_i^2/(lam - d_i) = 0 (origin shifted to the
// nearer pole, two-pole rational model with a bisection safeguard), Loewner
// recomputation of z from the computed roots (numerically orthogonal
// eigenvectors), and a batched fp64 GEMM with the children's eigenvector
// blocks.  Only the wanted kout eigenvectors are formed at the top level.
//
// Work: O(m^2) for the secular equations and O(sum over merges of n^3) in the
// GEMMs (~2e9 flops at m = 2000), all parallel, instead of the serial
// rotation chain of an implicit QL (m^2 dependent rotations).  tools/dc_proto.py
// is the numpy model of the same algorithm (checked against LAPACK there).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <math_constants.h>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "sc_common.cuh"
#include "sc_dc.cuh"

namespace sc {

namespace {

constexpr double kEps = 2.220446049250313e-16;
constexpr int kDcMaxN = 8192;

struct DcNode {
    int s, n, mid;  // rows [s, s+n) of T, torn at row mid
    int sL, nL;     // left child rows (kindL 1: rows [0, nL) of diag(theta))
    int sR, nR;     // right child rows (nR == 0: none)
    int kindL;      // 0 tree child, 1 diagonal (retained Ritz values), 2 none
    int bufL, bufR; // Q buffer holding each child's eigenvectors
    int out;        // 0/1: Q buffer; 2: the caller's S (top)
    int ncol;       // eigenvectors produced (n, or kout at the top)
};

struct DcTile {
    int node, part;  // part 0: rows of the left child, 1: right child
    int r0, c0;      // first output row (absolute) and column (node-relative)
};

struct DcCopy {
    int s, n, from;
};

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ double dc_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// a root of a x^2 + b x + c inside (lo, hi), else NaN
__device__ double quad_in(double a, double b, double c, double lo, double hi) {
    if (a == 0.0) {
        if (b == 0.0) return CUDART_NAN;
        double x = -c / b;
        return (x > lo && x < hi) ? x : CUDART_NAN;
    }
    double disc = b * b - 4.0 * a * c;
    if (!(disc >= 0.0)) return CUDART_NAN;
    double sq = sqrt(disc);
    double q = -0.5 * (b + copysign(sq, b));
    if (q == 0.0) return (0.0 > lo && 0.0 < hi) ? 0.0 : CUDART_NAN;
    double x1 = q / a, x2 = c / q;
    if (x1 > lo && x1 < hi) return x1;
    if (x2 > lo && x2 < hi) return x2;
    return CUDART_NAN;
}

// ---- kernels ------------------------------------------------------------------
// a[i] = T[i,i], b[i] = T[i,i+1] (0 past the end), c[i] = T[i,p] for i < p
__global__ void dc_extract_kernel(int m, int p, const double* __restrict__ T, double* __restrict__ a,
                                  double* __restrict__ b, double* __restrict__ c) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        a[i] = T[(size_t)i * m + i];
        b[i] = i + 1 < m ? T[(size_t)(i + 1) * m + i] : 0.0;
        if (i < p) c[i] = T[(size_t)p * m + i];
    }
}

// leaves (single rows of the tail): lam = a, Q = 1
__global__ void dc_leaf_kernel(int nleaf, const int* __restrict__ rows, const double* __restrict__ a,
                               double* __restrict__ lam, double* __restrict__ Q0, int m) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nleaf) return;
    int s = rows[i];
    lam[s] = a[s];
    Q0[(size_t)s * m + s] = 1.0;
}

// move child eigenvector blocks that sit in the buffer their parent writes
__global__ void dc_copy_kernel(const DcCopy* __restrict__ cp, double* __restrict__ Q0, double* __restrict__ Q1,
                               int m) {
    DcCopy c = cp[blockIdx.y];
    const double* src = c.from ? Q1 : Q0;
    double* dst = c.from ? Q0 : Q1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)c.n * c.n;
         e += (int64_t)gridDim.x * blockDim.x) {
        int col = (int)(e / c.n), row = (int)(e % c.n);
        size_t off = (size_t)(c.s + col) * m + c.s + row;
        dst[off] = src[off];
    }
}

// One CTA per node: gather (d, z), stable sort of d, deflation (dlaed2's
// tests: |z_i| <= tol, or a Givens rotation that zeroes one z of a close
// pair whose off-diagonal remainder |(d_j - d_i) c s| <= tol).
struct DcWork {
    double *lam, *a, *b, *carr, *Q0, *Q1;
    double *dsrt, *zsrt, *dk, *zk, *rot_c, *rot_s, *zn2, *tau, *zhat, *U;
    int *perm, *ipos, *kept, *rot_p, *rot_q, *nkept, *nrot, *root_o, *colsrc;
    const DcNode* nodes;
    int m;
};

__global__ void __launch_bounds__(1024) dc_setup_kernel(DcWork W, int node0) {
    extern __shared__ double smem[];
    const DcNode nd = W.nodes[node0 + blockIdx.x];
    const int nd_d = nd.n - 1;  // number of d's
    int np2 = 1;
    while (np2 < nd_d) np2 <<= 1;
    double* key = smem;                                      // np2
    double* zc = key + np2;                                  // nd_d (by coordinate)
    int* idx = reinterpret_cast<int*>(zc + nd_d);            // np2
    __shared__ double red[33];
    const int m = W.m;
    double amax = 0.0;
    for (int c = threadIdx.x; c < np2; c += blockDim.x) {
        if (c < nd_d) {
            double d, z;
            if (c < nd.nL) {
                if (nd.kindL == 1) {
                    d = W.a[c];
                    z = W.carr[c];
                } else {
                    const double* QL = nd.bufL ? W.Q1 : W.Q0;
                    d = W.lam[nd.sL + c];
                    z = W.b[nd.mid - 1] * QL[(size_t)(nd.sL + c) * m + (nd.mid - 1)];
                }
            } else {
                const int cc = c - nd.nL;
                const double* QR = nd.bufR ? W.Q1 : W.Q0;
                d = W.lam[nd.sR + cc];
                z = W.b[nd.mid] * QR[(size_t)(nd.sR + cc) * m + (nd.mid + 1)];
            }
            key[c] = d;
            zc[c] = z;
            idx[c] = c;
            amax = fmax(amax, fmax(fabs(d), fabs(z)));
        } else {
            key[c] = CUDART_INF;
            idx[c] = c;
        }
    }
    // max |d|, |z| for the deflation tolerance
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
    __syncthreads();
    // bitonic sort of (key, idx) ascending, ties by index (stable)
    for (int size = 2; size <= np2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < np2 / 2; t += blockDim.x) {
                int lo = 2 * t - (t & (stride - 1));
                int hi = lo + stride;
                bool up = ((lo & size) == 0);
                double k0 = key[lo], k1 = key[hi];
                int i0 = idx[lo], i1 = idx[hi];
                bool gt = (k0 > k1) || (k0 == k1 && i0 > i1);
                if (gt == up) {
                    key[lo] = k1;
                    key[hi] = k0;
                    idx[lo] = i1;
                    idx[hi] = i0;
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        double mx = fabs(W.a[nd.mid]);
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
        const double tol = 8.0 * kEps * mx;
        const int s = nd.s;
        double* ds = W.dsrt + s;
        double* zs = W.zsrt + s;
        for (int i = 0; i < nd_d; ++i) {
            ds[i] = key[i];
            zs[i] = zc[idx[i]];
            W.perm[s + i] = idx[i];
            W.ipos[s + idx[i]] = i;
        }
        int r = 0, nrot = 0, pj = -1;
        int* kept = W.kept + s;
        for (int jj = 0; jj < nd_d; ++jj) {
            const double zj = zs[jj];
            if (fabs(zj) <= tol) continue;
            if (pj >= 0) {
                const double zp = zs[pj];
                const double t = hypot(zp, zj);
                const double cc = zj / t, ss = zp / t;
                const double tau = (ds[jj] - ds[pj]) * cc * ss;
                if (fabs(tau) <= tol) {
                    const double dp = ds[pj] * cc * cc + ds[jj] * ss * ss;
                    const double dj = ds[pj] * ss * ss + ds[jj] * cc * cc;
                    ds[pj] = dp;
                    ds[jj] = dj;
                    zs[pj] = 0.0;
                    zs[jj] = t;
                    W.rot_p[s + nrot] = pj;
                    W.rot_q[s + nrot] = jj;
                    W.rot_c[s + nrot] = cc;
                    W.rot_s[s + nrot] = ss;
                    ++nrot;
                    --r;  // pj leaves the kept list
                }
            }
            kept[r++] = jj;
            pj = jj;
        }
        double z2 = 0.0;
        for (int t = 0; t < r; ++t) {
            W.dk[s + t] = ds[kept[t]];
            W.zk[s + t] = zs[kept[t]];
            z2 = fma(zs[kept[t]], zs[kept[t]], z2);
        }
        W.nkept[node0 + blockIdx.x] = r;
        W.nrot[node0 + blockIdx.x] = nrot;
        W.zn2[node0 + blockIdx.x] = z2;
    }
}

// One warp per root: (origin, tau) with lam = dk[origin] + tau
__global__ void __launch_bounds__(256) dc_roots_kernel(DcWork W, int node0, const int* __restrict__ slot_node) {
    const int slot = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (slot >= W.m) return;
    const int id = slot_node[slot];
    if (id < 0) return;
    const DcNode nd = W.nodes[node0 + id];
    const int j = slot - nd.s;
    const int r = W.nkept[node0 + id];
    if (j > r) return;
    const double alpha = W.a[nd.mid];
    if (r == 0) {
        if (lane == 0) {
            W.root_o[slot] = -1;
            W.tau[slot] = 0.0;
        }
        return;
    }
    const double* dk = W.dk + nd.s;
    const double* zk = W.zk + nd.s;
    const double znorm = sqrt(W.zn2[node0 + id]);
    int o;
    double lo, hi;
    if (j == 0) {
        o = 0;
        lo = fmin(dk[0], alpha) - znorm - dk[0];
        hi = 0.0;
    } else if (j == r) {
        o = r - 1;
        lo = 0.0;
        hi = fmax(dk[r - 1], alpha) + znorm - dk[r - 1];
    } else {
        const double dl = dk[j - 1], dh = dk[j];
        const double mid = 0.5 * (dl + dh);
        double sacc = 0.0;
        for (int i = lane; i < r; i += 32) {
            const double z = zk[i];
            sacc += z * z / (mid - dk[i]);
        }
        sacc = dc_warp_sum(sacc);
        if (alpha - mid + sacc > 0.0) {
            o = j;
            lo = mid - dh;
            hi = 0.0;
        } else {
            o = j - 1;
            lo = 0.0;
            hi = mid - dl;
        }
    }
    const double dor = dk[o];
    const double a0 = alpha - dor;
    const int ilo = j - 1, ihi = j < r ? j : -1;
    const double del_lo = ilo >= 0 ? dk[ilo] - dor : 0.0;
    const double del_hi = ihi >= 0 ? dk[ihi] - dor : 0.0;
    double tau = 0.5 * (lo + hi);
    double w1 = CUDART_INF, w2 = CUDART_INF;
    for (int it = 0; it < 200; ++it) {
        double sf = 0.0, sa = 0.0, sl = 0.0, sh = 0.0;
        for (int i = lane; i < r; i += 32) {
            const double z = zk[i];
            const double t = tau - (dk[i] - dor);
            const double q = z / t;
            const double term = z * q;
            sf += term;
            sa += fabs(term);
            if (i <= ilo)
                sl = fma(q, q, sl);
            else
                sh = fma(q, q, sh);
        }
        sf = dc_warp_sum(sf);
        sa = dc_warp_sum(sa);
        sl = dc_warp_sum(sl);
        sh = dc_warp_sum(sh);
        const double f = a0 - tau + sf;
        const double err = fabs(a0) + fabs(tau) + sa;
        if (f == 0.0 || fabs(f) <= 4.0 * kEps * err) break;
        if (f > 0.0)
            lo = tau;
        else
            hi = tau;
        if (hi - lo <= 2.0 * kEps * fmax(fabs(lo), fabs(hi))) break;
        double nw;
        if (ilo >= 0 && ihi >= 0) {
            const double tl = tau - del_lo, th = tau - del_hi;
            const double s_lo = (sl + 0.5) * tl * tl;
            const double s_hi = (sh + 0.5) * th * th;
            const double c = f - s_lo / tl - s_hi / th;
            nw = quad_in(c, -c * (del_lo + del_hi) + s_lo + s_hi, c * del_lo * del_hi - s_lo * del_hi - s_hi * del_lo,
                         lo, hi);
        } else if (ihi >= 0) {
            const double th = tau - del_hi;
            const double s_hi = sh * th * th;
            const double c = f + tau - s_hi / th;
            nw = quad_in(-1.0, c + del_hi, -c * del_hi + s_hi, lo, hi);
        } else {
            const double tl = tau - del_lo;
            const double s_lo = sl * tl * tl;
            const double c = f + tau - s_lo / tl;
            nw = quad_in(-1.0, c + del_lo, -c * del_lo + s_lo, lo, hi);
        }
        const double width = hi - lo;
        if (!(nw > lo && nw < hi) || width > 0.5 * w2) nw = 0.5 * (lo + hi);
        w2 = w1;
        w1 = width;
        tau = nw;
    }
    if (lane == 0) {
        W.root_o[slot] = o;
        W.tau[slot] = tau;
    }
}

__device__ __forceinline__ double dc_diff(const double* dk, const int* ro, const double* tau, int j, int t) {
    // lam_j - d_t from the origin representation
    return (dk[ro[j]] - dk[t]) + tau[j];
}

// Loewner: zhat_t^2 = (d_t - lam_0)(lam_r - d_t) prod_{j=1}^{t} (d_t - lam_j)/(d_t - d_{j-1})
//                     prod_{j=t+1}^{r-1} (lam_j - d_t)/(d_j - d_t)
__global__ void dc_zhat_kernel(DcWork W, int node0, const int* __restrict__ slot_node) {
    const int slot = blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= W.m) return;
    const int id = slot_node[slot];
    if (id < 0) return;
    const DcNode nd = W.nodes[node0 + id];
    const int t = slot - nd.s;
    const int r = W.nkept[node0 + id];
    if (t >= r) return;
    const double* dk = W.dk + nd.s;
    const int* ro = W.root_o + nd.s;
    const double* tau = W.tau + nd.s;
    const double dt = dk[t];
    double p = -dc_diff(dk, ro, tau, 0, t) * dc_diff(dk, ro, tau, r, t);
    for (int j = 1; j <= t; ++j) p *= -dc_diff(dk, ro, tau, j, t) / (dt - dk[j - 1]);
    for (int j = t + 1; j < r; ++j) p *= dc_diff(dk, ro, tau, j, t) / (dk[j] - dt);
    W.zhat[nd.s + t] = copysign(sqrt(p), W.zk[nd.s + t]);
}

// One CTA per node: the node's n eigenvalues (r+1 roots and the deflated d's)
// in ascending order -> lam, and the source of each output column
__global__ void __launch_bounds__(1024) dc_order_kernel(DcWork W, int node0, double* __restrict__ wsort) {
    extern __shared__ double smem[];
    const DcNode nd = W.nodes[node0 + blockIdx.x];
    const int n = nd.n, nd_d = n - 1, s = nd.s;
    const int r = W.nkept[node0 + blockIdx.x];
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    double* key = smem;
    int* tag = reinterpret_cast<int*>(key + np2);
    int* flag = tag + np2;  // nd_d kept flags
    for (int i = threadIdx.x; i < nd_d; i += blockDim.x) flag[i] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < r; t += blockDim.x) flag[W.kept[s + t]] = 1;
    __syncthreads();
    // slots 0..r: roots; r+1..n-1: deflated positions in sorted order
    for (int e = threadIdx.x; e < np2; e += blockDim.x) {
        if (e <= r) {
            const int o = W.root_o[s + e];
            key[e] = (o >= 0 ? W.dk[s + o] : W.a[nd.mid]) + W.tau[s + e];
            tag[e] = e;
        } else if (e < n) {
            key[e] = CUDART_NAN;  // filled below
            tag[e] = 0;
        } else {
            key[e] = CUDART_INF;
            tag[e] = INT_MAX;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int e = r + 1;
        for (int i = 0; i < nd_d; ++i)
            if (!flag[i]) {
                key[e] = W.dsrt[s + i];
                tag[e] = -1 - i;
                ++e;
            }
    }
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < np2 / 2; t += blockDim.x) {
                int lo = 2 * t - (t & (stride - 1));
                int hi = lo + stride;
                bool up = ((lo & size) == 0);
                double k0 = key[lo], k1 = key[hi];
                int i0 = tag[lo], i1 = tag[hi];
                bool gt = (k0 > k1) || (k0 == k1 && i0 > i1);
                if (gt == up) {
                    key[lo] = k1;
                    key[hi] = k0;
                    tag[lo] = i1;
                    tag[hi] = i0;
                }
            }
            __syncthreads();
        }
    }
    if (nd.out == 2) {
        // top: all eigenvalues descending; columns = the kout largest, descending
        for (int c = threadIdx.x; c < n; c += blockDim.x) wsort[c] = key[n - 1 - c];
        for (int c = threadIdx.x; c < nd.ncol; c += blockDim.x) W.colsrc[s + c] = tag[n - 1 - c];
    } else {
        for (int c = threadIdx.x; c < n; c += blockDim.x) {
            W.lam[s + c] = key[c];
            W.colsrc[s + c] = tag[c];
        }
    }
}

// One warp per output column: the arrowhead eigenvector in sorted d
// coordinates (apex last), the deflation rotations applied in reverse order,
// stored in U (rows s.., column s+c; top: column c)
__global__ void __launch_bounds__(128) dc_vec_kernel(DcWork W, int node0, const int* __restrict__ slot_node,
                                                     int max_n) {
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = blockIdx.x * (blockDim.x >> 5) + warp;
    if (slot >= W.m) return;
    const int id = slot_node[slot];
    if (id < 0) return;
    const DcNode nd = W.nodes[node0 + id];
    const int c = slot - nd.s;
    if (c >= nd.ncol) return;
    const int n = nd.n, nd_d = n - 1, s = nd.s;
    const int r = W.nkept[node0 + id];
    double* y = smem + (size_t)warp * max_n;
    for (int i = lane; i < n; i += 32) y[i] = 0.0;
    __syncwarp();
    const int src = W.colsrc[s + c];
    if (src >= 0) {
        const int j = src;
        double nrm = 0.0;
        if (r > 0) {
            const double* dk = W.dk + s;
            const int* ro = W.root_o + s;
            const double* tau = W.tau + s;
            for (int t = lane; t < r; t += 32) {
                const double v = W.zhat[s + t] / dc_diff(dk, ro, tau, j, t);
                y[W.kept[s + t]] = v;
                nrm = fma(v, v, nrm);
            }
        }
        nrm = dc_warp_sum(nrm) + 1.0;
        const double inv = 1.0 / sqrt(nrm);
        __syncwarp();
        for (int i = lane; i < nd_d; i += 32) y[i] *= inv;
        if (lane == 0) y[nd_d] = inv;
    } else {
        if (lane == 0) y[-1 - src] = 1.0;
    }
    __syncwarp();
    const int nrot = W.nrot[node0 + id];
    if (lane == 0) {
        for (int t = nrot - 1; t >= 0; --t) {
            const int pj = W.rot_p[s + t], qj = W.rot_q[s + t];
            const double cc = W.rot_c[s + t], ss = W.rot_s[s + t];
            const double yp = y[pj], yq = y[qj];
            y[pj] = cc * yp + ss * yq;
            y[qj] = -ss * yp + cc * yq;
        }
    }
    __syncwarp();
    const int col = nd.out == 2 ? c : s + c;
    double* u = W.U + (size_t)col * W.m + s;
    for (int i = lane; i < n; i += 32) u[i] = y[i];
}

// Rows of the node's eigenvectors that need no product: the torn row mid
// (apex coordinate) and, at the top, the rows of diag(theta) (identity child)
__global__ void dc_rows_kernel(DcWork W, int node0, double* __restrict__ S) {
    const DcNode nd = W.nodes[node0 + blockIdx.y];
    const int m = W.m;
    double* out = nd.out == 2 ? S : (nd.out ? W.Q1 : W.Q0);
    const int colbase = nd.out == 2 ? 0 : nd.s;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nd.ncol; c += gridDim.x * blockDim.x) {
        const double* u = W.U + (size_t)(colbase + c) * m + nd.s;
        double* o = out + (size_t)(colbase + c) * m;
        o[nd.mid] = u[nd.n - 1];
        if (nd.kindL == 1)
            for (int i = 0; i < nd.nL; ++i) o[i] = u[W.ipos[nd.s + i]];
    }
}

// Batched fp64 GEMM: out[rows of child, cols] = Q_child * U[child coords, cols],
// U rows gathered through ipos (coordinate -> sorted position).  64 x 64
// output tile per CTA, 256 threads x (4 x 4) accumulators, K in steps of 16.
constexpr int GT_M = 64, GT_N = 64, GT_K = 16;
__global__ void __launch_bounds__(256) dc_gemm_kernel(DcWork W, const DcTile* __restrict__ tiles, double* __restrict__ S) {
    __shared__ double As[GT_K][GT_M + 1];
    __shared__ double Bs[GT_K][GT_N + 1];
    const DcTile tl = tiles[blockIdx.x];
    const DcNode nd = W.nodes[tl.node];
    const int m = W.m;
    const int cs = tl.part == 0 ? nd.sL : nd.sR;  // child row/col start
    const int cn = tl.part == 0 ? nd.nL : nd.nR;  // child size (= K)
    const int coord0 = tl.part == 0 ? 0 : nd.nL;  // arrowhead coordinate of child col 0
    const double* Qc = (tl.part == 0 ? nd.bufL : nd.bufR) ? W.Q1 : W.Q0;
    double* out = nd.out == 2 ? S : (nd.out ? W.Q1 : W.Q0);
    const int colbase = nd.out == 2 ? 0 : nd.s;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < cn; k0 += GT_K) {
        // A tile: rows r0..r0+63 of the child, columns k0..k0+15 (child-relative)
        for (int e = threadIdx.x; e < GT_M * GT_K; e += 256) {
            const int rr = e % GT_M, kk = e / GT_M;
            const int row = tl.r0 + rr, k = k0 + kk;
            As[kk][rr] = (row < cs + cn && k < cn) ? Qc[(size_t)(cs + k) * m + row] : 0.0;
        }
        for (int e = threadIdx.x; e < GT_N * GT_K; e += 256) {
            const int kk = e % GT_K, cc = e / GT_K;
            const int k = k0 + kk, col = tl.c0 + cc;
            double v = 0.0;
            if (k < cn && col < nd.ncol) {
                const int pos = W.ipos[nd.s + coord0 + k];
                v = W.U[(size_t)(colbase + col) * m + nd.s + pos];
            }
            Bs[kk][cc] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GT_K; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = tl.r0 + ty + 16 * i;
        if (row >= cs + cn) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = tl.c0 + tx + 16 * j;
            if (col < nd.ncol) out[(size_t)(colbase + col) * m + row] = acc[i][j];
        }
    }
}

// ---- host side ------------------------------------------------------------------
struct DcLevel {
    int node0 = 0, count = 0, max_n = 0;
    std::vector<int> slot_node;  // m entries
    std::vector<DcTile> tiles;
    std::vector<DcCopy> copies;
    int slot_off = 0, tile_off = 0, copy_off = 0;
};

struct DcPlan {
    int m = 0, p = 0, kout = 0;
    std::vector<DcNode> nodes;
    std::vector<int> leaves;
    std::vector<DcLevel> levels;  // tail levels bottom-up, then the top
    DevBuf<DcNode> d_nodes;
    DevBuf<int> d_slot, d_leaves;
    DevBuf<DcTile> d_tiles;
    DevBuf<DcCopy> d_copies;
};

struct DcTmp {
    int s, n, mid, h, idL, idR;
};

int build_tail(std::vector<DcTmp>& tmp, std::vector<int>& leaves, int s, int n) {
    if (n <= 0) return -1;
    if (n == 1) {
        leaves.push_back(s);
        tmp.push_back({s, 1, s, 0, -1, -1});
        return (int)tmp.size() - 1;
    }
    const int nl = (n - 1) / 2;
    const int mid = s + nl;
    int l = build_tail(tmp, leaves, s, nl);
    int r = build_tail(tmp, leaves, mid + 1, n - 1 - nl);
    int h = 1 + std::max(l >= 0 ? tmp[l].h : 0, r >= 0 ? tmp[r].h : 0);
    tmp.push_back({s, n, mid, h, l, r});
    return (int)tmp.size() - 1;
}

void add_tiles(DcLevel& L, int id, const DcNode& nd) {
    for (int part = 0; part < 2; ++part) {
        const int cs = part == 0 ? nd.sL : nd.sR;
        const int cn = part == 0 ? nd.nL : nd.nR;
        if (cn <= 0 || (part == 0 && nd.kindL != 0)) continue;
        for (int r0 = cs; r0 < cs + cn; r0 += GT_M)
            for (int c0 = 0; c0 < nd.ncol; c0 += GT_N) L.tiles.push_back({id, part, r0, c0});
    }
}

int make_plan(DcPlan& P, int m, int p, int kout, cudaStream_t st) {
    P.m = m;
    P.p = p;
    P.kout = kout;
    std::vector<DcTmp> tmp;
    P.leaves.clear();
    const int troot = build_tail(tmp, P.leaves, p + 1, m - p - 1);
    int H = troot >= 0 ? tmp[troot].h : 0;
    std::vector<int> buf(tmp.size(), 0);
    // tail nodes by height
    P.nodes.clear();
    P.levels.clear();
    std::vector<int> node_id(tmp.size(), -1);
    for (int h = 1; h <= H; ++h) {
        DcLevel L;
        L.node0 = (int)P.nodes.size();
        L.slot_node.assign(m, -1);
        for (size_t t = 0; t < tmp.size(); ++t) {
            if (tmp[t].h != h) continue;
            const DcTmp& T = tmp[t];
            DcNode nd{};
            nd.s = T.s;
            nd.n = T.n;
            nd.mid = T.mid;
            nd.sL = T.s;
            nd.nL = T.idL >= 0 ? tmp[T.idL].n : 0;
            nd.sR = T.mid + 1;
            nd.nR = T.idR >= 0 ? tmp[T.idR].n : 0;
            nd.kindL = nd.nL > 0 ? 0 : 2;
            nd.out = h & 1;
            nd.ncol = T.n;
            // children in the buffer this node writes move to the other one
            for (int side = 0; side < 2; ++side) {
                const int c = side == 0 ? T.idL : T.idR;
                if (c < 0) continue;
                if (buf[c] == nd.out) {
                    L.copies.push_back({tmp[c].s, tmp[c].n, buf[c]});
                    buf[c] = 1 - buf[c];
                }
                (side == 0 ? nd.bufL : nd.bufR) = buf[c];
            }
            buf[t] = nd.out;
            const int id = (int)P.nodes.size() - L.node0;
            for (int i = 0; i < T.n; ++i) L.slot_node[T.s + i] = id;
            P.nodes.push_back(nd);
            add_tiles(L, L.node0 + id, nd);
            L.max_n = std::max(L.max_n, T.n);
            ++L.count;
            node_id[t] = (int)P.nodes.size() - 1;
        }
        P.levels.push_back(std::move(L));
    }
    // top: diag(theta) rows [0, p) | row p | tail (p, m)
    {
        DcLevel L;
        L.node0 = (int)P.nodes.size();
        L.slot_node.assign(m, -1);
        DcNode nd{};
        nd.s = 0;
        nd.n = m;
        nd.mid = p;
        nd.sL = 0;
        nd.nL = p;
        nd.kindL = p > 0 ? 1 : 2;
        nd.sR = p + 1;
        nd.nR = m - p - 1;
        nd.bufL = 0;
        nd.bufR = troot >= 0 ? buf[troot] : 0;
        nd.out = 2;
        nd.ncol = kout;
        for (int i = 0; i < m; ++i) L.slot_node[i] = 0;
        P.nodes.push_back(nd);
        add_tiles(L, L.node0, nd);
        L.max_n = m;
        L.count = 1;
        P.levels.push_back(std::move(L));
    }
    // upload
    size_t nslot = 0, ntile = 0, ncopy = 0;
    for (auto& L : P.levels) {
        L.slot_off = (int)nslot;
        L.tile_off = (int)ntile;
        L.copy_off = (int)ncopy;
        nslot += L.slot_node.size();
        ntile += L.tiles.size();
        ncopy += L.copies.size();
    }
    std::vector<int> hs;
    std::vector<DcTile> ht;
    std::vector<DcCopy> hc;
    for (auto& L : P.levels) {
        hs.insert(hs.end(), L.slot_node.begin(), L.slot_node.end());
        ht.insert(ht.end(), L.tiles.begin(), L.tiles.end());
        hc.insert(hc.end(), L.copies.begin(), L.copies.end());
    }
    int rc;
    if ((rc = P.d_nodes.alloc(P.nodes.size())) || (rc = P.d_slot.alloc(std::max<size_t>(1, hs.size()))) ||
        (rc = P.d_leaves.alloc(std::max<size_t>(1, P.leaves.size()))) ||
        (rc = P.d_tiles.alloc(std::max<size_t>(1, ht.size()))) || (rc = P.d_copies.alloc(std::max<size_t>(1, hc.size()))))
        return rc;
    SC_CUDA(cudaMemcpyAsync(P.d_nodes.p, P.nodes.data(), sizeof(DcNode) * P.nodes.size(), cudaMemcpyHostToDevice, st));
    if (!hs.empty()) SC_CUDA(cudaMemcpyAsync(P.d_slot.p, hs.data(), sizeof(int) * hs.size(), cudaMemcpyHostToDevice, st));
    if (!P.leaves.empty())
        SC_CUDA(cudaMemcpyAsync(P.d_leaves.p, P.leaves.data(), sizeof(int) * P.leaves.size(), cudaMemcpyHostToDevice, st));
    if (!ht.empty()) SC_CUDA(cudaMemcpyAsync(P.d_tiles.p, ht.data(), sizeof(DcTile) * ht.size(), cudaMemcpyHostToDevice, st));
    if (!hc.empty()) SC_CUDA(cudaMemcpyAsync(P.d_copies.p, hc.data(), sizeof(DcCopy) * hc.size(), cudaMemcpyHostToDevice, st));
    // the host vectors must outlive the async copies
    SC_CUDA(cudaStreamSynchronize(st));
    return SC_OK;
}

struct DcWorkspace {
    int m = 0;
    DevBuf<double> dbl;  // 13 m-vectors + U + Q0 + Q1
    DevBuf<int> ints;    // 11 m-vectors + per-node counters
    DcWork w{};
    int alloc(int m_, cudaStream_t st) {
        if (m_ <= m) return SC_OK;
        m = m_;
        int rc;
        const size_t mm = (size_t)m * m;
        if ((rc = dbl.alloc(13 * (size_t)m + 3 * mm)) || (rc = ints.alloc(11 * (size_t)m + 3 * (size_t)(2 * m + 2))))
            return rc;
        double* d = dbl.p;
        w.lam = d; d += m;
        w.a = d; d += m;
        w.b = d; d += m;
        w.carr = d; d += m;
        w.dsrt = d; d += m;
        w.zsrt = d; d += m;
        w.dk = d; d += m;
        w.zk = d; d += m;
        w.rot_c = d; d += m;
        w.rot_s = d; d += m;
        w.zn2 = d; d += m;
        w.tau = d; d += m;
        w.zhat = d; d += m;
        w.U = d; d += mm;
        w.Q0 = d; d += mm;
        w.Q1 = d; d += mm;
        int* q = ints.p;
        w.perm = q; q += m;
        w.ipos = q; q += m;
        w.kept = q; q += m;
        w.rot_p = q; q += m;
        w.rot_q = q; q += m;
        w.root_o = q; q += m;
        w.colsrc = q; q += m;
        q += 4 * m;
        w.nkept = q; q += 2 * m + 2;
        w.nrot = q; q += 2 * m + 2;
        (void)st;
        return SC_OK;
    }
};

struct DcCache {
    std::mutex mu;
    std::map<std::tuple<int, int, int>, std::unique_ptr<DcPlan>> plans;
    DcWorkspace ws;
};
DcCache& dc_cache() {
    static DcCache* c = new DcCache();
    return *c;
}

}  // namespace

int dc_symeig_launch(int m, int p, const double* T, int kout, double* wsort, double* S, cudaStream_t st) {
    if (m < 1 || m > kDcMaxN) return fail(SC_ERR_VALUE, "arrowhead eigensolver needs 1 <= m <= 8192");
    if (p < 0 || p >= m) return fail(SC_ERR_VALUE, "arrow size p must satisfy 0 <= p < m");
    if (kout < 1 || kout > m) return fail(SC_ERR_VALUE, "symeig needs 1 <= kout <= m");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(dc_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(dc_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(dc_vec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    DcCache& C = dc_cache();
    std::lock_guard<std::mutex> lock(C.mu);
    int rc;
    if ((rc = C.ws.alloc(m, st))) return rc;
    auto key = std::make_tuple(m, p, kout);
    auto it = C.plans.find(key);
    if (it == C.plans.end()) {
        auto plan = std::make_unique<DcPlan>();
        if ((rc = make_plan(*plan, m, p, kout, st))) return rc;
        it = C.plans.emplace(key, std::move(plan)).first;
    }
    DcPlan& P = *it->second;
    DcWork w = C.ws.w;
    w.m = m;
    w.nodes = P.d_nodes.p;
    ProfScope prof("symeig", st, 0.0);
    int launches = 0;
    dc_extract_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(m, p, T, w.a, w.b, w.carr);
    ++launches;
    if (!P.leaves.empty()) {
        dc_leaf_kernel<<<(unsigned)ceil_div((int64_t)P.leaves.size(), 256), 256, 0, st>>>(
            (int)P.leaves.size(), P.d_leaves.p, w.a, w.lam, w.Q0, m);
        ++launches;
    }
    for (const DcLevel& L : P.levels) {
        const int* slot = P.d_slot.p + L.slot_off;
        if (!L.copies.empty()) {
            dim3 g(64, (unsigned)L.copies.size());
            dc_copy_kernel<<<g, 256, 0, st>>>(P.d_copies.p + L.copy_off, w.Q0, w.Q1, m);
            ++launches;
        }
        int np2 = 1;
        while (np2 < L.max_n) np2 <<= 1;
        const size_t sm_setup = (size_t)np2 * 12 + (size_t)L.max_n * 8 + 64;
        const int thr = std::min(1024, std::max(64, np2 / 2));
        dc_setup_kernel<<<L.count, thr, sm_setup, st>>>(w, L.node0);
        dc_roots_kernel<<<(unsigned)ceil_div((int64_t)m * 32, 256), 256, 0, st>>>(w, L.node0, slot);
        dc_zhat_kernel<<<(unsigned)ceil_div(m, 128), 128, 0, st>>>(w, L.node0, slot);
        const size_t sm_order = (size_t)np2 * 12 + (size_t)L.max_n * 4 + 64;
        dc_order_kernel<<<L.count, thr, sm_order, st>>>(w, L.node0, wsort);
        const int wpb = std::max(1, std::min(4, (int)((200 * 1024) / ((size_t)L.max_n * 8))));
        dc_vec_kernel<<<(unsigned)ceil_div(m, wpb), 32 * wpb, (size_t)wpb * L.max_n * 8, st>>>(w, L.node0, slot,
                                                                                                   L.max_n);
        dim3 gr((unsigned)std::max<int64_t>(1, ceil_div(L.max_n, 256)), (unsigned)L.count);
        dc_rows_kernel<<<gr, 256, 0, st>>>(w, L.node0, S);
        launches += 6;
        if (!L.tiles.empty()) {
            dc_gemm_kernel<<<(unsigned)L.tiles.size(), 256, 0, st>>>(w, P.d_tiles.p + L.tile_off, S);
            ++launches;
        }
    }
    SC_LAUNCHED(launches);
    return SC_OK;
}

}  // namespace sc

extern "C" int sc_symeig_arrow_f64(int64_t m, int64_t p, int64_t kout, const double* T, double* theta, double* S,
                                   sc_stream_t stream) {
    cudaStream_t st = sc::as_stream(stream);
    sc::StreamScope scope(st);
    return sc::dc_symeig_launch((int)m, (int)p, T, (int)kout, theta, S, st);
}
