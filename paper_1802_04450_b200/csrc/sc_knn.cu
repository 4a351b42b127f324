// Stage 1: kNN + exp_decay similarity graph, emitted straight into CSR.
//
// Reference semantics (graph.py:149-157, 185-204, 136-141, 214-237):
//   row i ranks every j != i by (similarity desc, index asc) with
//   s_ij = exp(inv * d2_ij), inv = -1/(2 sigma^2), d2 from direct differences;
//   the first knn are selected; edge {i,j} exists iff j in top(i) or i in
//   top(j); its weight exp(-d2/(2 sigma^2)) is evaluated once per pair.
//
// Pipeline:
//   prep      centre X (fp64 column means), fp32 copy + fp32 norms, fp64 norms
//   candidates  distance tiles |x_j|^2 - 2 x_i.x_j (low precision) with a
//             streaming per-row top-R list (append + quickselect compaction)
//   recheck   exact fp64 d2 and s for the R..CAP candidates, rank by
//             (-s, j), certify with an error bound that no non-candidate can
//             enter the top knn; uncertified rows -> exact fallback
//   fallback  fp64 scan of all n points + radix select on (s, -j)
//   union     reverse lists, duplicate removal, scan, CSR fill with fp64 values
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sc_common.cuh"
#include "sc_knn.cuh"
#include "sc_list.cuh"
#include "sc_knn_tc2.cuh"
#include "sc_tma.cuh"
#include "sc_knn_tc.cuh"
#include "sc_scan.cuh"
#include "sc_sparse.cuh"

namespace sc {

// ---------------------------------------------------------------------------
// prep
__global__ void colsum_partial_kernel(int64_t n, int64_t d, const double* __restrict__ x, double* __restrict__ part) {
    // block b: rows [b*256, b*256+256); thread t handles columns t, t+blockDim...
    int64_t r0 = (int64_t)blockIdx.x * 256, r1 = imin64(n, r0 + 256);
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
        double a = 0.0;
        for (int64_t r = r0; r < r1; ++r) a += x[r * d + c];
        part[blockIdx.x * d + c] = a;
    }
}
__global__ void colmean_finish_kernel(int64_t nb, int64_t n, int64_t d, const double* __restrict__ part,
                                      double* __restrict__ mean) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d) return;
    double a = 0.0;
    for (int64_t b = 0; b < nb; ++b) a += part[b * d + c];
    mean[c] = a / (double)n;
}

// pivots for the scan order: rows floor(c * n / C), c < C
__global__ void gather_strided_rows_kernel(int64_t n, int64_t d, int64_t C, const double* __restrict__ x,
                                           double* __restrict__ out) {
    const int64_t c = blockIdx.x;
    const int64_t r = c * n / C;
    for (int64_t l = threadIdx.x; l < d; l += blockDim.x) out[c * d + l] = x[r * d + l];
}

// squared distances between the C pivots (fp32 is plenty for ordering them)
__global__ void pivot_dist_kernel(int64_t C, int64_t d, const double* __restrict__ piv, float* __restrict__ D) {
    const int64_t a = blockIdx.y, b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= C) return;
    double s = 0.0;
    for (int64_t l = 0; l < d; ++l) {
        const double t = piv[a * d + l] - piv[b * d + l];
        s = fma(t, t, s);
    }
    D[a * C + b] = (float)s;
}

// out row r = x row idx[r] (n x d)
__global__ void gather_rows_i32_kernel(int64_t n, int64_t d, const double* __restrict__ x,
                                       const int32_t* __restrict__ idx, double* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * d) return;
    const int64_t r = e / d;
    out[e] = x[(int64_t)idx[r] * d + (e - r * d)];
}

__global__ void gather_pivots_kernel(int64_t C, int64_t d, const double* __restrict__ src,
                                     const int32_t* __restrict__ order, double* __restrict__ dst) {
    const int64_t c = blockIdx.x;
    for (int64_t l = threadIdx.x; l < d; l += blockDim.x) dst[c * d + l] = src[(int64_t)order[c] * d + l];
}

// Greedy nearest-neighbour tour over the pivots (start at pivot 0, always
// step to the closest unvisited one; ties -> lower index).  Pivots of one
// dense region are mutual near neighbours, so the tour visits them in a run
// and their buckets become one contiguous range of the scan order.
// SPECLUST_TIMING_DEBUG=1: host wall time of the ordering phases on stderr
struct PhaseClock {
    cudaStream_t st;
    bool on;
    std::chrono::steady_clock::time_point t0;
    explicit PhaseClock(cudaStream_t s) : st(s), on(std::getenv("SPECLUST_TIMING_DEBUG") != nullptr) {
        if (on) {
            cudaStreamSynchronize(st);
            t0 = std::chrono::steady_clock::now();
        }
    }
    void lap(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[knn_order] %s %.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

static void pivot_tour(int64_t C, const std::vector<float>& D, std::vector<int32_t>& order) {
    std::vector<char> used((size_t)C, 0);
    order.assign(1, 0);
    used[0] = 1;
    int64_t cur = 0;
    for (int64_t t = 1; t < C; ++t) {
        float best = INFINITY;
        int64_t bi = -1;
        const float* row = D.data() + cur * C;
        for (int64_t b = 0; b < C; ++b)
            if (!used[(size_t)b] && (bi < 0 || row[b] < best)) {
                best = row[b];
                bi = b;
            }
        used[(size_t)bi] = 1;
        order.push_back((int32_t)bi);
        cur = bi;
    }
}

// xf = fp32(x - mean) padded to dp columns; cnf = fp32(|xf|^2) (computed in
// fp64 from the fp32 values); rn = |x - mean| (fp64); rmax = max rn
__global__ void knn_prep_kernel(int64_t n, int64_t d, int64_t dp, const double* __restrict__ x,
                                const double* __restrict__ mean, float* __restrict__ xf,
                                float* __restrict__ cnf, double* __restrict__ rn, double* __restrict__ qn,
                                unsigned long long* __restrict__ rmax_bits) {
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    double a64 = 0.0, a32 = 0.0;
    for (int64_t c = lane; c < dp; c += 32) {
        float f = 0.f;
        if (c < d) {
            double v = x[i * d + c] - mean[c];
            a64 = fma(v, v, a64);
            f = (float)v;
        }
        xf[i * dp + c] = f;
        a32 = fma((double)f, (double)f, a32);
    }
    a64 = warp_sum(a64);
    a32 = warp_sum(a32);
    if (lane == 0) {
        cnf[i] = (float)a32;
        double r = sqrt(a64);
        rn[i] = r;
        qn[i] = a32;
        atomicMax(rmax_bits, (unsigned long long)__double_as_longlong(r));
    }
}

// ---------------------------------------------------------------------------
// candidate generation, SIMT fp32 tiles (reference kernel for A/B checks of
// the tcgen05 path; selected with SPECLUST_KNN_KERNEL=simt) (128 query rows x 128 columns)
constexpr int KM = 128, KN = 128, KK = 16;

__global__ void __launch_bounds__(256) knn_cand_simt_kernel(int64_t n, int64_t qtile0, int dp,
                                                            const float* __restrict__ xf,
                                                            const float* __restrict__ cnf, int cap, int R,
                                                            float2* __restrict__ lists, int* __restrict__ counts,
                                                            float* __restrict__ taus) {
    extern __shared__ float smem[];
    float* As = smem;                    // KK x KM
    float* Bs = As + KK * KM;            // KK x KN
    float* Ks = Bs + KK * KN;            // KM x (KN + 1)
    float* cns = Ks + KM * (KN + 1);     // KN
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t r0 = (qtile0 + blockIdx.x) * KM;
    const int64_t myrow = r0 + tid;
    const int64_t lrow = (int64_t)blockIdx.x * KM + tid;  // list slot
    const bool selector = tid < KM && myrow < n;
    int cnt = 0;
    float tau = INFINITY;
    float2* L = lists + (selector ? lrow : 0) * (int64_t)cap;

    for (int64_t c0 = 0; c0 < n; c0 += KN) {
        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        for (int k0 = 0; k0 < dp; k0 += KK) {
            __syncthreads();
            // 128 rows x 16 floats each for A and B: 512 float4 each, 2 per thread
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                int idx = tid + 256 * t;
                int rr = idx >> 2, q4 = (idx & 3) * 4;
                int64_t ga = r0 + rr, gb = c0 + rr;
                float4 va = ga < n ? *reinterpret_cast<const float4*>(xf + ga * dp + k0 + q4) : make_float4(0, 0, 0, 0);
                float4 vb = gb < n ? *reinterpret_cast<const float4*>(xf + gb * dp + k0 + q4) : make_float4(0, 0, 0, 0);
                As[(q4 + 0) * KM + rr] = va.x;
                As[(q4 + 1) * KM + rr] = va.y;
                As[(q4 + 2) * KM + rr] = va.z;
                As[(q4 + 3) * KM + rr] = va.w;
                Bs[(q4 + 0) * KN + rr] = vb.x;
                Bs[(q4 + 1) * KN + rr] = vb.y;
                Bs[(q4 + 2) * KN + rr] = vb.z;
                Bs[(q4 + 3) * KN + rr] = vb.w;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < KK; ++k) {
                float4 a0 = *reinterpret_cast<const float4*>(As + k * KM + ty * 4);
                float4 a1 = *reinterpret_cast<const float4*>(As + k * KM + 64 + ty * 4);
                float4 b0 = *reinterpret_cast<const float4*>(Bs + k * KN + tx * 4);
                float4 b1 = *reinterpret_cast<const float4*>(Bs + k * KN + 64 + tx * 4);
                float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
        }
        if (tid < KN) cns[tid] = (c0 + tid < n) ? cnf[c0 + tid] : 0.f;
        __syncthreads();
        // keys = |x_j|^2 - 2 x_i.x_j into the smem tile
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            int m = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int nn = j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4);
                Ks[m * (KN + 1) + nn] = fmaf(-2.f, acc[i][j], cns[nn]);
            }
        }
        __syncthreads();
        if (selector) {
            int cmax = (int)imin64(KN, n - c0);
            const float* krow = Ks + tid * (KN + 1);
            for (int c = 0; c < cmax; ++c) {
                float key = krow[c];
                if (key < tau) {
                    int64_t col = c0 + c;
                    if (col == myrow) continue;
                    L[cnt++] = make_float2(key, __int_as_float((int)col));
                    if (cnt == cap) {
                        tau = list_compact(L, cap, R);
                        cnt = R;
                    }
                }
            }
        }
    }
    if (selector) {
        counts[lrow] = cnt;
        taus[lrow] = tau;
    }
}

// ---------------------------------------------------------------------------
// exact recheck: warp per row
// |x_j - x_i|^2 in the summation order of the reference's
// np.einsum("ij,ij->i", diff, diff) (graph.py:92, 156; 136-141), so ranking
// keys and edge values are bit-identical (NpDot, sc_common.cuh)
__device__ __forceinline__ double exact_d2(const double* __restrict__ xi, const double* __restrict__ xj, int64_t d) {
    return np_sqdist(xj, xi, d);
}

// Measure of the kNN ranking / edge values.  kind 0: exp_decay (the ranking
// value is exp(inv * d2) over x, graph.py:149-157); kind 1: cosine or
// cross-correlation: clip(dot(xc_i, xc_j) / sqrt(sq_i sq_j), -1, 1) with xc
// the (centred) rows and sq their squared norms (graph.py:143-147, 158-163),
// while the candidate search runs on the row-normalised xc (|a - b|^2 =
// 2 - 2 cos for unit rows).  policy: negative policy of the edge values
// (0 clamp_zero, 1 abs, 2 keep).
struct KnnMeasure {
    int kind = 0;
    const double* xc = nullptr;
    const double* sq = nullptr;
    int policy = 0;
};
__device__ __forceinline__ double knn_corr(const KnnMeasure& ms, int64_t d, int64_t i, int64_t j) {
    const double* a = ms.xc + i * d;
    const double* b = ms.xc + j * d;
    NpDot acc;
    np_dot_span(acc, 0, d, [&](int64_t l) { return __dmul_rn(a[l], b[l]); });
    const double v = __ddiv_rn(acc.result(), __dsqrt_rn(__dmul_rn(ms.sq[i], ms.sq[j])));
    return v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
}
// clip(dot / sqrt(sq_i sq_j), -1, 1) of a dot product in the einsum order
__device__ __forceinline__ double knn_corr_of(const KnnMeasure& ms, double dot, int64_t i, int64_t j) {
    const double v = __ddiv_rn(dot, __dsqrt_rn(__dmul_rn(ms.sq[i], ms.sq[j])));
    return v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
}

// Warp-cooperative einsum-order reductions of up to 32 rows (lane t owns the
// row rt, nullptr = none) against the warp-uniform row ri.  The rows are
// staged through shared memory (stage: 32 x 33 doubles per warp) 32 columns
// at a time with coalesced loads; a lane-per-row loop would spend one L1
// wavefront per lane per element.  DIFF: |rt - ri|^2 (np_sqdist(rt, ri));
// else dot(ri, rt).  Bit-identical to the per-lane forms.  The row pointers
// are exchanged through shared memory (after the 32 x 33 tile) rather than
// shuffles, which would need a converged warp the compiler cannot prove.
constexpr int kStageLd = 33;
constexpr int kStageWarp = 32 * kStageLd + 32;  // doubles per warp
template <bool DIFF>
__device__ __forceinline__ double warp_rows_np(const double* __restrict__ ri, const double* rt, int64_t d,
                                               double* __restrict__ stage) {
    const int lane = threadIdx.x & 31;
    const double** rows = reinterpret_cast<const double**>(stage + 32 * kStageLd);
    __syncwarp();
    rows[lane] = rt;
    NpDot acc;
    for (int64_t c0 = 0; c0 < d; c0 += 32) {
        const int w = (int)(d - c0 < 32 ? d - c0 : 32);
        __syncwarp();
#pragma unroll
        for (int r0 = 0; r0 < 32; r0 += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double* pr = rows[r0 + q];
                v[q] = (pr && lane < w) ? __ldg(pr + c0 + lane) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) stage[(r0 + q) * kStageLd + lane] = v[q];
        }
        __syncwarp();
        if (rt) {
            const double* srow = stage + lane * kStageLd - c0;
            np_dot_span(acc, c0, c0 + w, [&](int64_t l) {
                if (DIFF) {
                    const double t = __dsub_rn(srow[l], ri[l]);
                    return __dmul_rn(t, t);
                }
                return __dmul_rn(ri[l], srow[l]);
            });
        }
    }
    return acc.result();
}

// order-preserving 64-bit key of a double (any sign), 0 reserved
__device__ __forceinline__ unsigned long long ordered_key(double s) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(s);
    return (u >> 63) ? ~u : (u | (1ull << 63));
}

// (s desc, j asc) ordering: a precedes b
__device__ __forceinline__ bool precedes(double sa, int ja, double sb, int jb) {
    return sa > sb || (sa == sb && ja < jb);
}

__global__ void __launch_bounds__(256) knn_recheck_kernel(int64_t n, int64_t p0, int64_t p1, int64_t d,
                                                          const double* __restrict__ x,
                                                          int64_t knn, double inv, int cap,
                                                          const float2* __restrict__ lists,
                                                          const int* __restrict__ counts,
                                                          const float* __restrict__ taus,
                                                          const double* __restrict__ rn, const double* __restrict__ qn,
                                                          const unsigned long long* __restrict__ rmax_bits,
                                                          double cdelta, const int32_t* __restrict__ perm,
                                                          int32_t* __restrict__ sel,
                                                          int32_t* __restrict__ flagged,
                                                          unsigned long long* __restrict__ nflag, KnnMeasure ms,
                                                          const double* __restrict__ xs, double* __restrict__ selv) {
    // lists/counts/taus/sel are in scan order relative to p0 (position ip
    // holds point perm[ip]); distances, norms and the (-s, j) tie-break use
    // original indices; flagged rows are recorded by scan position
    extern __shared__ unsigned char rsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* stage = reinterpret_cast<double*>(rsm) + (size_t)warp * kStageWarp;
    double* S = reinterpret_cast<double*>(rsm) + (size_t)8 * kStageWarp + (size_t)warp * cap;
    double* D = reinterpret_cast<double*>(rsm) + (size_t)8 * kStageWarp + (size_t)8 * cap + (size_t)warp * cap;
    int* J = reinterpret_cast<int*>(reinterpret_cast<double*>(rsm) + (size_t)8 * kStageWarp + (size_t)16 * cap) +
             (size_t)warp * cap;
    const int64_t lp = (int64_t)blockIdx.x * 8 + warp;
    const int64_t ip = p0 + lp;
    if (ip >= p1) return;
    const int64_t i = perm ? (int64_t)perm[ip] : ip;
    const int cnt = counts[lp];
    const float2* L = lists + lp * (int64_t)cap;
    // xs: the points in scan order (row p = point perm[p]); the candidates of a
    // row are its scan-order neighbours, so their rows are L2-resident there
    const double* xi = xs ? xs + ip * d : x + i * d;
    const float tau = taus[lp];
    const double rr = rn[i] + __longlong_as_double((long long)*rmax_bits);
    const double delta = cdelta * rr * rr;  // |approximate key - exact (d2 - qn_i)| bound
    // Prune the list with its approximate keys: with T the knn-th smallest
    // key, at least knn candidates have d2 <= qn + T + delta, so a candidate
    // whose key exceeds T + 2 delta (+ slack) cannot be selected.  The dropped
    // keys join the non-candidates in the certificate below (lower bound
    // qn + key - delta), so a wrong prune is caught there like a short list.
    constexpr int PL = TC_LIST_P / 32;
    float kv[PL];
    unsigned uk[PL];
#pragma unroll
    for (int q = 0; q < PL; ++q) {
        const int t = lane + 32 * q;
        kv[q] = t < cnt ? L[t].x : INFINITY;
        const unsigned u = __float_as_uint(kv[q]);
        uk[q] = t < cnt ? ((u >> 31) ? ~u : (u | 0x80000000u)) : 0xffffffffu;
    }
    float kdrop = INFINITY;  // smallest dropped key
    int* K = J;              // kept list positions (J is rewritten in place below)
    int m = cnt;
    if (cnt > knn + 8) {
        unsigned pre = 0;  // knn-th smallest ordered key (radix select over the warp)
        for (int b = 31; b >= 0; --b) {
            const unsigned trial = pre | ((1u << b) - 1u);
            int c = 0;
#pragma unroll
            for (int q = 0; q < PL; ++q) c += (lane + 32 * q < cnt) && uk[q] <= trial;
            if (__reduce_add_sync(0xffffffffu, c) < (int)knn) pre |= 1u << b;
        }
        const unsigned tb = (pre >> 31) ? (pre & 0x7fffffffu) : ~pre;
        const double T = (double)__uint_as_float(tb);
        const double thr = T + 2.0 * delta + 1e-9 * (fabs(qn[i] + T) + delta);
        m = 0;
#pragma unroll
        for (int q = 0; q < PL; ++q) {
            const int t = lane + 32 * q;
            const bool keep = t < cnt && (double)kv[q] <= thr;
            if (t < cnt && !keep) kdrop = fminf(kdrop, kv[q]);
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) K[m + __popc(bal & ((1u << lane) - 1u))] = t;
            m += __popc(bal);
        }
        for (int o = 16; o > 0; o >>= 1) kdrop = fminf(kdrop, __shfl_xor_sync(0xffffffffu, kdrop, o));
    } else {
        for (int t = lane; t < cnt; t += 32) K[t] = t;
    }
    __syncwarp();
    for (int t0 = 0; t0 < m; t0 += 32) {
        const int t = t0 + lane;
        int js = 0, j = 0;
        if (t < m) {
            js = __float_as_int(L[K[t]].y);
            j = perm ? perm[js] : js;
        }
        if (ms.kind == 0) {
            const double* rt = t < m ? (xs ? xs + (int64_t)js * d : x + (int64_t)j * d) : nullptr;
            const double d2 = warp_rows_np<true>(xi, rt, d, stage);
            if (t < m) {
                S[t] = exp(inv * d2);
                D[t] = d2;
            }
        } else {
            const double dot = warp_rows_np<false>(ms.xc + i * d, t < m ? ms.xc + (int64_t)j * d : nullptr, d, stage);
            if (t < m) S[t] = D[t] = knn_corr_of(ms, dot, i, j);
        }
        __syncwarp();
        if (t < m) J[t] = j;
    }
    __syncwarp();
    // rank each kept candidate; the knn first ranks are selected (s_k: the
    // knn-th value).  The selection is written in ascending j order: its
    // slot is the number of selected candidates with a smaller index.
    double s_k = INFINITY;
    int ranks[TC_LIST_P / 32];
#pragma unroll
    for (int q = 0; q < TC_LIST_P / 32; ++q) {
        const int t = lane + 32 * q;
        ranks[q] = INT_MAX;
        if (t < m) {
            const double st = S[t];
            const int jt = J[t];
            int r = 0;
            for (int u = 0; u < m; ++u) r += precedes(S[u], J[u], st, jt);
            ranks[q] = r;
            if (r == knn - 1) s_k = st;
        }
    }
    // broadcast s_k (held by exactly one lane)
    for (int o = 16; o > 0; o >>= 1) s_k = fmin(s_k, __shfl_xor_sync(0xffffffffu, s_k, o));
    __syncwarp();
#pragma unroll
    for (int q = 0; q < TC_LIST_P / 32; ++q)  // non-selected candidates leave the index order
        if (lane + 32 * q < m && ranks[q] >= knn) J[lane + 32 * q] = INT_MAX;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < TC_LIST_P / 32; ++q) {
        const int t = lane + 32 * q;
        if (t < m && ranks[q] < knn) {
            const int jt = J[t];
            int slot = 0;
            for (int u = 0; u < m; ++u) slot += J[u] < jt;
            sel[lp * knn + slot] = jt;
            if (selv) selv[lp * knn + slot] = D[t];  // the edge's d2 (exp_decay) or correlation
        }
    }
    if (lane != 0) return;
    bool ok;
    const float tlow = fminf(tau, kdrop);  // smallest key of any point not evaluated exactly
    if (m < knn) {
        ok = false;
    } else if (isinf(tlow)) {
        ok = true;  // never compacted, nothing dropped: every other point was evaluated
    } else {
        double lower = qn[i] + (double)tlow - delta;  // lower bound of d2 for the others
        lower = lower * (1.0 - 1e-12) - 1e-300;
        // cosine: unit rows, so a non-candidate has cos <= 1 - lower / 2
        ok = ms.kind == 0 ? (lower > 0.0 && s_k > exp(inv * lower)) : s_k > 1.0 - 0.5 * lower + 1e-12;
    }
    if (!ok) {
        unsigned long long slot = atomicAdd(nflag, 1ull);
        flagged[slot] = (int32_t)ip;
    }
}

// ---------------------------------------------------------------------------
// exact fallback: block per flagged row, radix select on the (s, -j) order
__global__ void __launch_bounds__(512) knn_fallback_kernel(int64_t n, int64_t p0, int64_t d,
                                                           const double* __restrict__ x, int64_t knn, double inv,
                                                           const int32_t* __restrict__ perm,
                                                           const int32_t* __restrict__ flagged, int64_t nflag,
                                                           unsigned long long* __restrict__ scratch,
                                                           int32_t* __restrict__ sel, KnnMeasure ms,
                                                           double* __restrict__ selv) {
    __shared__ unsigned int hist[256];
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_remaining;
    __shared__ int s_out;
    __shared__ int wcount[16];
    __shared__ long long s_base;
    unsigned long long* key = scratch + (size_t)blockIdx.x * n;
    for (int64_t f = blockIdx.x; f < nflag; f += gridDim.x) {
        const int64_t ip = flagged[f];
        const int64_t i = perm ? (int64_t)perm[ip] : ip;
        int32_t* srow = sel + (ip - p0) * knn;
        const double* xi = x + i * d;
        for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
            if (j == i) {
                key[j] = 0ull;
            } else {
                if (ms.kind == 0) {
                    double s = exp(inv * exact_d2(xi, x + j * d, d));
                    key[j] = (unsigned long long)__double_as_longlong(s) + 1ull;  // s >= 0 -> monotone bits
                } else {
                    key[j] = ordered_key(knn_corr(ms, d, i, j));
                }
            }
        }
        if (threadIdx.x == 0) {
            s_prefix = 0ull;
            s_remaining = knn;
        }
        __syncthreads();
        unsigned long long mask = 0ull;
        for (int pass = 7; pass >= 0; --pass) {
            const int shift = pass * 8;
            for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
            __syncthreads();
            const unsigned long long pre = s_prefix;
            for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
                unsigned long long kj = key[j];
                if ((kj & mask) == pre) atomicAdd(&hist[(kj >> shift) & 255ull], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                long long rem = s_remaining;
                long long above = 0;
                int g = 255;
                for (; g > 0; --g) {
                    if (above + (long long)hist[g] >= rem) break;
                    above += hist[g];
                }
                s_remaining = rem - above;
                s_prefix = pre | ((unsigned long long)g << shift);
            }
            mask |= 255ull << shift;
            __syncthreads();
        }
        const unsigned long long T = s_prefix;
        const long long take_eq = s_remaining;  // elements == T to take, lowest index first
        if (threadIdx.x == 0) {
            s_out = 0;
            s_base = 0;
        }
        __syncthreads();
        for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
            if (key[j] > T) {
                int slot = atomicAdd(&s_out, 1);
                srow[slot] = (int32_t)j;
            }
        }
        __syncthreads();
        const int above_cnt = s_out;
        for (int64_t base = 0; base < n; base += blockDim.x) {
            int64_t j = base + threadIdx.x;
            bool hit = j < n && key[j] == T;
            unsigned bal = __ballot_sync(0xffffffffu, hit);
            int w = threadIdx.x >> 5, l = threadIdx.x & 31;
            if (l == 0) wcount[w] = __popc(bal);
            __syncthreads();
            long long before = s_base;
            for (int q = 0; q < w; ++q) before += wcount[q];
            long long r = before + __popc(bal & ((1u << l) - 1u));
            if (hit && r < take_eq) srow[above_cnt + r] = (int32_t)j;
            __syncthreads();
            if (threadIdx.x == 0) {
                long long tot = 0;
                for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot += wcount[q];
                s_base += tot;
            }
            __syncthreads();
            if (s_base >= take_eq) break;
        }
        __syncthreads();
        if (selv)
            for (int64_t t = threadIdx.x; t < knn; t += blockDim.x) {
                const int64_t j = srow[t];
                selv[(ip - p0) * knn + t] = ms.kind == 0 ? exact_d2(xi, x + j * d, d) : knn_corr(ms, d, i, j);
            }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// union + CSR
// ascending j order of the fallback rows (the recheck writes its rows sorted)
__global__ void sort_rows_kernel(int64_t nrows, const int32_t* __restrict__ rows, int64_t p0, int64_t knn,
                                 int32_t* __restrict__ sel, double* __restrict__ selv) {
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nrows) return;
    const int64_t i = rows[f] - p0;
    int32_t* r = sel + i * knn;
    double* w = selv ? selv + i * knn : nullptr;  // values travel with their columns
    for (int64_t a = 1; a < knn; ++a) {
        int32_t v = r[a];
        const double wv = w ? w[a] : 0.0;
        int64_t b = a - 1;
        while (b >= 0 && r[b] > v) {
            r[b + 1] = r[b];
            if (w) w[b + 1] = w[b];
            --b;
        }
        r[b + 1] = v;
        if (w) w[b + 1] = wv;
    }
}

// The union works on the selections of ALL points (sel: n x knn in scan
// order, row q = point perm[q]) and emits the CSR rows [r0, r1) only, so
// each shard of a multi-GPU build produces its own row block.
__global__ void pos_of_kernel(int64_t n, const int32_t* __restrict__ perm, int32_t* __restrict__ pos) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n) pos[perm ? perm[q] : q] = (int32_t)q;
}

__global__ void rev_count_kernel(int64_t total, int64_t r0, int64_t r1, const int32_t* __restrict__ sel,
                                 int64_t* __restrict__ rc) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= total) return;
    const int64_t j = sel[p];
    if (j >= r0 && j < r1) atomicAdd(reinterpret_cast<unsigned long long*>(rc + (j - r0)), 1ull);
}

__global__ void rev_fill_kernel(int64_t n, int64_t knn, int64_t r0, int64_t r1, const int32_t* __restrict__ sel,
                                const int32_t* __restrict__ perm, const int64_t* __restrict__ rev_ptr,
                                unsigned int* __restrict__ fill, int32_t* __restrict__ rev,
                                int64_t* __restrict__ rev_src) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n * knn) return;
    const int64_t j = sel[p];
    if (j < r0 || j >= r1) return;
    unsigned int slot = atomicAdd(fill + (j - r0), 1u);
    const int64_t q = p / knn;
    rev[rev_ptr[j - r0] + slot] = perm ? perm[q] : (int32_t)q;
    if (rev_src) rev_src[rev_ptr[j - r0] + slot] = p;  // the selection slot (its value)
}

__device__ __forceinline__ bool in_sorted(const int32_t* __restrict__ a, int64_t len, int32_t v) {
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo < len && a[lo] == v;
}

// len_i = knn + #(reverse entries not already selected); marks duplicates
__global__ void row_count_kernel(int64_t nl, int64_t r0, int64_t knn, const int32_t* __restrict__ sel,
                                 const int32_t* __restrict__ pos, const int64_t* __restrict__ rev_ptr,
                                 const int32_t* __restrict__ rev, uint8_t* __restrict__ dup,
                                 int64_t* __restrict__ len) {
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;  // local row
    int lane = threadIdx.x & 31;
    if (i >= nl) return;
    const int32_t* s = sel + (int64_t)pos[r0 + i] * knn;
    int64_t c = 0;
    for (int64_t p = rev_ptr[i] + lane; p < rev_ptr[i + 1]; p += 32) {
        bool dp = in_sorted(s, knn, rev[p]);
        dup[p] = dp;
        c += !dp;
    }
    c = warp_sum_i64(c);
    if (lane == 0) len[i] = knn + c;
}

// CSR fill from the exact values the recheck kept (selv: the d2 or the
// correlation of every selection slot, rev_src: the slot of each reverse
// entry): no distances are recomputed.  The value of a reverse entry comes
// from the other endpoint's slot, which is the same number (|a - b|^2 and the
// dot product are symmetric bit for bit in the einsum order).  Warp per row;
// the row's non-duplicate reverse entries are counted from shared memory.
__global__ void __launch_bounds__(256) row_fill_vals_kernel(
    int64_t nl, int64_t r0, int64_t knn, double den, const int32_t* __restrict__ sel, const double* __restrict__ selv,
    const int32_t* __restrict__ pos, const int64_t* __restrict__ rev_ptr, const int32_t* __restrict__ rev,
    const int64_t* __restrict__ rev_src, const uint8_t* __restrict__ dup, const int64_t* __restrict__ row_ptr,
    int32_t* __restrict__ col, double* __restrict__ vals, const int32_t* __restrict__ order, int kind, int policy,
    int64_t* __restrict__ long_rows, unsigned int* __restrict__ nlong) {
    constexpr int FILL_CAP = 192;
    __shared__ int32_t cin_all[8][FILL_CAP];
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    int32_t* C = cin_all[threadIdx.x / 32];
    if (i >= nl) return;
    if (order) i = order[i];
    const int64_t slot0 = (int64_t)pos[r0 + i] * knn;
    const int32_t* s = sel + slot0;
    const int64_t rb = rev_ptr[i], re = rev_ptr[i + 1];
    const int64_t out0 = row_ptr[i];
    auto value = [&](double v) {
        if (kind == 0) return exp(-v / den);
        return policy == 0 ? (v > 0.0 ? v : 0.0) : (policy == 1 ? fabs(v) : v);
    };
    // the non-duplicate reverse columns (shared memory when they fit; longer
    // rows -- hubs selected by many points -- go to row_fill_long_kernel)
    int nr = 0;
    const bool fits = re - rb <= FILL_CAP;
    if (!fits && long_rows) {
        if (lane == 0) long_rows[atomicAdd(nlong, 1u)] = i;
        return;
    }
    if (fits) {
        for (int64_t p0 = rb; p0 < re; p0 += 32) {
            const int64_t p = p0 + lane;
            const bool a = p < re && !dup[p];
            const unsigned bal = __ballot_sync(0xffffffffu, a);
            if (a) C[nr + __popc(bal & ((1u << lane) - 1u))] = rev[p];
            nr += __popc(bal);
        }
        __syncwarp();
    }
    auto rev_less = [&](int32_t e) {
        int64_t r = 0;
        if (fits)
            for (int q = 0; q < nr; ++q) r += C[q] < e;
        else
            for (int64_t q = rb; q < re; ++q) r += (!dup[q] && rev[q] < e);
        return r;
    };
    for (int64_t t = lane; t < knn; t += 32) {
        const int32_t e = s[t];
        const int64_t r = t + rev_less(e);
        col[out0 + r] = e;
        vals[out0 + r] = value(selv[slot0 + t]);
    }
    for (int64_t p = rb + lane; p < re; p += 32) {
        if (dup[p]) continue;
        const int32_t e = rev[p];
        int64_t lo = 0, hi = knn;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (s[mid] < e) lo = mid + 1; else hi = mid;
        }
        const int64_t r = lo + rev_less(e);
        col[out0 + r] = e;
        vals[out0 + r] = value(selv[rev_src[p]]);
    }
}

// The long rows of row_fill_vals_kernel, a block per row: the row's
// non-duplicate reverse entries are sorted in shared memory (bitonic, with
// their positions as payload) and merged with the sorted selection, instead
// of the warp kernel's per-entry counting, which is quadratic in the row
// length.  Rows longer than FILL_LONG fall back to counting.
constexpr int FILL_LONG = 4096;
__global__ void __launch_bounds__(256) row_fill_long_kernel(
    int64_t r0, int64_t knn, double den, const int32_t* __restrict__ sel, const double* __restrict__ selv,
    const int32_t* __restrict__ pos, const int64_t* __restrict__ rev_ptr, const int32_t* __restrict__ rev,
    const int64_t* __restrict__ rev_src, const uint8_t* __restrict__ dup, const int64_t* __restrict__ row_ptr,
    int32_t* __restrict__ col, double* __restrict__ vals, int kind, int policy, const int64_t* __restrict__ long_rows,
    const unsigned int* __restrict__ nlong) {
    __shared__ int32_t E[FILL_LONG];
    __shared__ int32_t P[FILL_LONG];  // offsets in the row's reverse list
    __shared__ int s_nr;
    const int tid = threadIdx.x, lane = tid & 31;
    auto value = [&](double v) {
        if (kind == 0) return exp(-v / den);
        return policy == 0 ? (v > 0.0 ? v : 0.0) : (policy == 1 ? fabs(v) : v);
    };
    const unsigned nrows = *nlong;
    for (unsigned f = blockIdx.x; f < nrows; f += gridDim.x) {
        const int64_t i = long_rows[f];
        const int64_t slot0 = (int64_t)pos[r0 + i] * knn;
        const int32_t* s = sel + slot0;
        const int64_t rb = rev_ptr[i], re = rev_ptr[i + 1];
        const int64_t out0 = row_ptr[i];
        __syncthreads();
        if (tid < 32) {  // warp 0 compacts the non-duplicate entries
            int nr = 0;
            for (int64_t p0 = rb; p0 < re; p0 += 32) {
                const int64_t p = p0 + lane;
                const bool a = p < re && !dup[p];
                const unsigned bal = __ballot_sync(0xffffffffu, a);
                const int q = nr + __popc(bal & ((1u << lane) - 1u));
                if (a && q < FILL_LONG) {
                    E[q] = rev[p];
                    P[q] = (int32_t)(p - rb);
                }
                nr += __popc(bal);
            }
            if (lane == 0) s_nr = nr;
        }
        __syncthreads();
        const int nr = s_nr;
        if (nr <= FILL_LONG) {
            int np2 = 1;
            while (np2 < nr) np2 <<= 1;
            for (int q = nr + tid; q < np2; q += blockDim.x) E[q] = INT_MAX;
            __syncthreads();
            for (int k = 2; k <= np2; k <<= 1)
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int q = tid; q < np2; q += blockDim.x) {
                        const int o = q ^ j;
                        if (o > q) {
                            const bool up = (q & k) == 0;
                            if ((E[q] > E[o]) == up) {
                                const int32_t te = E[q];
                                E[q] = E[o];
                                E[o] = te;
                                const int32_t tp = P[q];
                                P[q] = P[o];
                                P[o] = tp;
                            }
                        }
                    }
                    __syncthreads();
                }
            for (int q = tid; q < nr; q += blockDim.x) {
                const int32_t e = E[q];
                int64_t lo = 0, hi = knn;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (s[mid] < e) lo = mid + 1; else hi = mid;
                }
                col[out0 + q + lo] = e;
                vals[out0 + q + lo] = value(selv[rev_src[rb + P[q]]]);
            }
            for (int64_t t = tid; t < knn; t += blockDim.x) {
                const int32_t e = s[t];
                int lo = 0, hi = nr;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (E[mid] < e) lo = mid + 1; else hi = mid;
                }
                col[out0 + t + lo] = e;
                vals[out0 + t + lo] = value(selv[slot0 + t]);
            }
        } else {
            for (int64_t t = tid; t < knn; t += blockDim.x) {
                const int32_t e = s[t];
                int64_t r = t;
                for (int64_t q = rb; q < re; ++q) r += (!dup[q] && rev[q] < e);
                col[out0 + r] = e;
                vals[out0 + r] = value(selv[slot0 + t]);
            }
            for (int64_t p = rb + tid; p < re; p += blockDim.x) {
                if (dup[p]) continue;
                const int32_t e = rev[p];
                int64_t lo = 0, hi = knn;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (s[mid] < e) lo = mid + 1; else hi = mid;
                }
                int64_t r = lo;
                for (int64_t q = rb; q < re; ++q) r += (!dup[q] && rev[q] < e);
                col[out0 + r] = e;
                vals[out0 + r] = value(selv[rev_src[p]]);
            }
        }
    }
}

__global__ void __launch_bounds__(128) row_fill_kernel(int64_t nl, int64_t r0, int64_t d, int64_t knn,
                                                       const double* __restrict__ x, double den,
                                                       const int32_t* __restrict__ sel, const int32_t* __restrict__ pos,
                                                       const int64_t* __restrict__ rev_ptr,
                                                       const int32_t* __restrict__ rev, const uint8_t* __restrict__ dup,
                                                       const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col,
                                                       double* __restrict__ vals, const int32_t* __restrict__ order,
                                                       KnnMeasure ms, const double* __restrict__ xs) {
    // warp per local row; with `order` (whole graph only) the rows are visited
    // in the kNN locality order, and with xs (the points in that order) the x
    // rows of a row's neighbours sit next to its own
    constexpr int FILL_CAP = 256;
    __shared__ double stage_all[4][kStageWarp];
    __shared__ int32_t cin_all[4][FILL_CAP], cout_all[4][FILL_CAP];
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    double* stage = stage_all[threadIdx.x / 32];
    int32_t* C = cin_all[threadIdx.x / 32];
    int32_t* O = cout_all[threadIdx.x / 32];
    if (i >= nl) return;
    if (order) i = order[i];
    const int64_t gi = r0 + i;
    const int32_t* s = sel + (int64_t)pos[gi] * knn;
    const int64_t rb = rev_ptr[i], re = rev_ptr[i + 1];
    const int64_t out0 = row_ptr[i];
    const double* ri = ms.kind == 0 ? (xs ? xs + (int64_t)pos[gi] * d : x + gi * d) : ms.xc + gi * d;
    // value of the edge (gi, e) for the active lanes (warp-collective)
    auto edge = [&](bool act, int32_t e) {
        const double* rt =
            act ? (ms.kind == 0 ? (xs ? xs + (int64_t)pos[e] * d : x + (int64_t)e * d) : ms.xc + (int64_t)e * d)
                : nullptr;
        if (ms.kind == 0) return exp(-warp_rows_np<true>(ri, rt, d, stage) / den);
        const double v = act ? knn_corr_of(ms, warp_rows_np<false>(ri, rt, d, stage), gi, e)
                             : warp_rows_np<false>(ri, rt, d, stage);
        return ms.policy == 0 ? (v > 0.0 ? v : 0.0) : (ms.policy == 1 ? fabs(v) : v);
    };
    const int64_t len = row_ptr[i + 1] - out0;
    if (len <= FILL_CAP) {
        // merge in shared memory: C = the sorted selection, then the reverse
        // entries not already selected; O = the row's columns in order
        for (int t = lane; t < knn; t += 32) C[t] = s[t];
        int nr = 0;
        for (int64_t p0 = rb; p0 < re; p0 += 32) {
            const int64_t p = p0 + lane;
            const bool a = p < re && !dup[p];
            const unsigned bal = __ballot_sync(0xffffffffu, a);
            if (a) C[knn + nr + __popc(bal & ((1u << lane) - 1u))] = rev[p];
            nr += __popc(bal);
        }
        __syncwarp();
        const int32_t* Rv = C + knn;
        for (int t = lane; t < len; t += 32) {
            const int32_t e = C[t];
            int r = 0;
            if (t < knn) {
                r = t;
            } else {
                int lo = 0, hi = (int)knn;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (C[mid] < e) lo = mid + 1; else hi = mid;
                }
                r = lo;
            }
            for (int q = 0; q < nr; ++q) r += Rv[q] < e;
            O[r] = e;
        }
        __syncwarp();
        for (int t0 = 0; t0 < len; t0 += 32) {
            const int t = t0 + lane;
            const bool act = t < len;
            const int32_t e = act ? O[t] : 0;
            const double v = edge(act, e);
            if (act) {
                col[out0 + t] = e;
                vals[out0 + t] = v;
            }
        }
        return;
    }
    // long rows: selected entries
    for (int64_t t0 = 0; t0 < knn; t0 += 32) {
        const int64_t t = t0 + lane;
        const bool act = t < knn;
        int32_t e = 0;
        int64_t r = t;
        if (act) {
            e = s[t];
            for (int64_t p = rb; p < re; ++p) r += (!dup[p] && rev[p] < e);
        }
        const double v = edge(act, e);
        if (act) {
            col[out0 + r] = e;
            vals[out0 + r] = v;
        }
    }
    // reverse-only entries
    for (int64_t p0 = rb; p0 < re; p0 += 32) {
        const int64_t p = p0 + lane;
        const bool act = p < re && !dup[p];
        int32_t e = 0;
        int64_t r = 0;
        if (act) {
            e = rev[p];
            int64_t lo = 0, hi = knn;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if (s[mid] < e) lo = mid + 1; else hi = mid;
            }
            r = lo;
            for (int64_t q = rb; q < re; ++q) r += (!dup[q] && rev[q] < e);
        }
        const double v = edge(act, e);
        if (act) {
            col[out0 + r] = e;
            vals[out0 + r] = v;
        }
    }
}

}  // namespace sc

using namespace sc;

namespace sc {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D map over a rows x dp fp16 row-major matrix: 64 x 128 boxes, 128-byte
// swizzle (the K-major UMMA operand layout of sc_tc.cuh)
int make_f16_tile_map(CUtensorMap* map, const __half* base, int64_t rows, int64_t dp) {
    auto encode = tensor_map_encoder();
    if (!encode) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t gdim[2] = {(cuuint64_t)dp, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)dp * sizeof(__half)};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
    return SC_OK;
}

template <int NKB, int STAGES, bool LSMEM>
static int launch_tc(const CUtensorMap& map, int64_t n, int64_t ntiles, int64_t qtile0, int64_t nq, const float* cnk,
                     float key_scale, int cap, int R, float2* lists, int* counts, float* taus, cudaStream_t st) {
    const uint32_t smem = TcLayout<NKB, STAGES, LSMEM>::total;
    SC_CUDA(cudaFuncSetAttribute(knn_cand_tc_kernel<NKB, STAGES, LSMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    DevBuf<long long> dbg;
    const bool want_dbg = std::getenv("SPECLUST_KNN_DEBUG") != nullptr;
    if (want_dbg) {
        if (int rc = dbg.alloc((size_t)nq * 16)) return rc;
        SC_CUDA(cudaMemsetAsync(dbg.p, 0, sizeof(long long) * nq * 16, st));
    }
    knn_cand_tc_kernel<NKB, STAGES, LSMEM><<<(unsigned)nq, TC_THREADS, smem, st>>>(map, n, ntiles, qtile0, cnk,
                                                                                   key_scale, cap, R, lists, counts,
                                                                                   taus, dbg.p);
    SC_LAUNCHED(1);
    if (want_dbg) {
        std::vector<long long> h((size_t)nq * 16);
        SC_CUDA(d2h_sync(h.data(), dbg.p, sizeof(long long) * h.size(), st));
        double acc[16] = {0};
        for (int64_t b = 0; b < nq; ++b)
            for (int q = 0; q < 16; ++q) acc[q] += (double)h[b * 16 + q];
        fprintf(stderr, "[knn_tc dbg] warp2 per tile: fired halves %.4f, quarters %.4f, appends/row %.2f (total), "
                        "compactions/row %.2f (total)\n",
                acc[12] / nq / ntiles, acc[15] / nq / ntiles, acc[13] / nq / 32, acc[14] / nq / 32);
        const char* names[12] = {"tma.wait_empty", "-", "-", "tma.total", "mma.wait_tempty", "mma.wait_full",
                                 "mma.latency64", "mma.total", "epi.wait_tfull", "epi.ldtm", "epi.work", "epi.fast"};
        for (int q = 0; q < 12; ++q)
            if (names[q][0] != '-')
                fprintf(stderr, "[knn_tc dbg] %-16s %.1f cycles/tile\n", names[q],
                        q == 6 ? acc[q] / nq / 64 : acc[q] / nq / ntiles);
    }
    return SC_OK;
}

static uint32_t tc2_heap_bytes(int R) { return 16 + 256u * (uint32_t)R * 8u + 8u * 32u * 16u * 4u; }

template <int NKB, int STAGES, int WMODE, bool HEAP>
static int launch_tc2_w(const CUtensorMap& map, int64_t n, int64_t ntiles, int64_t qtile0, int64_t nq, const float* cnk,
                        float key_scale, int cap, int R, float2* lists, int* counts, float* taus, cudaStream_t st) {
    const int64_t grid = ceil_div(nq, 2);
    // heap variant: + per-row heaps; list variant: at least 114 KB so that
    // exactly one CTA (holding all 512 TMEM columns) fits an SM
    const uint32_t smem = HEAP ? Tc2Layout<NKB, STAGES>::total + tc2_heap_bytes(R)
                               : std::max<uint32_t>(Tc2Layout<NKB, STAGES>::total, 116u * 1024u);
    SC_CUDA(cudaFuncSetAttribute(knn_cand_tc2_kernel<NKB, STAGES, WMODE, HEAP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DevBuf<long long> dbg;
    if (WMODE & 64) {
        if (int rc = dbg.alloc(8)) return rc;
        SC_CUDA(cudaMemsetAsync(dbg.p, 0, 8 * sizeof(long long), st));
    }
    knn_cand_tc2_kernel<NKB, STAGES, WMODE, HEAP><<<(unsigned)grid, TC2_THREADS, smem, st>>>(
        map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts, taus, dbg.p);
    SC_LAUNCHED(1);
    if (WMODE & 64) {
        long long h[8];
        SC_CUDA(d2h_sync(h, dbg.p, sizeof(h), st));
        const double warps = (double)grid * 8;
        fprintf(stderr, "[knn_tc2 list path] per warp: cycles t<16 %.3g, 16<=t<128 %.3g, t>=128 %.3g; "
                        "fired halves %.0f / %.0f / %.0f\n",
                h[0] / warps, h[1] / warps, h[2] / warps, h[3] / warps, h[4] / warps, h[5] / warps);
    }
    return SC_OK;
}

// WMODE bit 0: producer / MMA waits with a suspend hint; bit 1: epilogue waits
// with it; bits 2-4 are profiling switches (skip epilogue / MMA / list path:
// SPECLUST_KNN_WAIT=7, 11, 15, 19, 27 with SPECLUST_KNN_TILE_ONLY=1, results
// invalid) used to separate the MMA, epilogue and list-maintenance costs
template <int NKB, int STAGES>
static int launch_tc2(const CUtensorMap& map, int64_t n, int64_t ntiles, int64_t qtile0, int64_t nq, const float* cnk,
                      float key_scale, int cap, int R, float2* lists, int* counts, float* taus, cudaStream_t st) {
    const char* wenv = std::getenv("SPECLUST_KNN_WAIT");
    const int w = wenv ? std::atoi(wenv) : 3;
    if (std::getenv("SPECLUST_KNN_NOLIST")) cap = -cap;  // profiling only: results invalid
    // opt-in (SPECLUST_KNN_HEAP=1): candidate lists as shared-memory max-heaps
    // (d <= 64: the 256 x R heaps fit beside a 3- or 2-deep operand ring).
    // Measured at C2 it is slower than the global lists with warp compaction
    // (319 vs 271 ms: each replacement is a chain of ~6 dependent shared loads
    // on the inserting lane while its warp waits), so it is off by default.
    const char* henv = std::getenv("SPECLUST_KNN_HEAP");
    const bool heap_ok = NKB == 1 && henv && std::strcmp(henv, "1") == 0;
    constexpr uint32_t kMax = 227u * 1024u;
    if (heap_ok && w == 3) {
        if (Tc2Layout<NKB, 3>::total + tc2_heap_bytes(R) <= kMax)
            return launch_tc2_w<NKB, 3, 3, true>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts,
                                                 taus, st);
        if (Tc2Layout<NKB, 2>::total + tc2_heap_bytes(R) <= kMax)
            return launch_tc2_w<NKB, 2, 3, true>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts,
                                                 taus, st);
    }
#define SC_TC2(W) \
    case W: return launch_tc2_w<NKB, STAGES, W, false>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts, taus, st)
    switch (w) {
        SC_TC2(0);
        SC_TC2(7);
        SC_TC2(11);
        SC_TC2(15);
        SC_TC2(19);
        SC_TC2(27);
        SC_TC2(67);
        default: return launch_tc2_w<NKB, STAGES, 3, false>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists,
                                                            counts, taus, st);
    }
#undef SC_TC2
}

// tensor-core candidate lists: query tiles [qtile0, qtile0 + nq) against every
// candidate tile
int knn_candidates_tc(int64_t n, int64_t n_pad, int64_t dp64, const __half* xh, const float* cnk, float key_scale,
                      int64_t qtile0, int64_t nq, int cap, int R, float2* lists, int* counts, float* taus,
                      cudaStream_t st) {
    auto encode = tensor_map_encoder();
    if (!encode) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)dp64, (cuuint64_t)n_pad};
    cuuint64_t gstride[1] = {(cuuint64_t)dp64 * sizeof(__half)};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(xh), gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
    const int64_t ntiles = n_pad / 128;
    ProfScope prof("knn_tile", st, 2.0 * (double)imin64(n, nq * 128) * (double)n * (double)dp64);
    // query-pair kernel for d <= 128 (SPECLUST_KNN_TC=1 selects the one-tile kernel)
    const char* tenv = std::getenv("SPECLUST_KNN_TC");
    if (!(tenv && std::strcmp(tenv, "1") == 0) && dp64 <= 128) {
        if (dp64 == 64)
            return launch_tc2<1, 6>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts, taus, st);
        return launch_tc2<2, 2>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts, taus, st);
    }
    switch (dp64 / 64) {
        case 1: return launch_tc<1, 4, false>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts, taus, st);
        case 2: return launch_tc<2, 3, false>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts, taus, st);
        case 3: return launch_tc<3, 2, false>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts, taus, st);
        default: return launch_tc<4, 2, false>(map, n, ntiles, qtile0, nq, cnk, key_scale, cap, R, lists, counts, taus, st);
    }
}

__global__ void iota_kernel(int64_t n, int32_t* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)i;
}

// Selection stage: the top-knn of every point at scan positions [p0, p1),
// written to sel ((p1 - p0) x knn, each row ascending), plus the scan order
// perm (n entries; identical on every caller for the same x).
int knn_select(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq, int64_t p0, int64_t p1,
               int32_t* sel, int32_t* perm_out, int64_t* stats, cudaStream_t st, KnnMeasure ms = KnnMeasure(),
               double* selv = nullptr) {
    const double inv = -1.0 / two_sigma_sq;  // graph.py:154
    const int64_t dp = (d + 15) / 16 * 16;
    const char* kenv = std::getenv("SPECLUST_KNN_KERNEL");
    const int64_t dp64 = (d + 63) / 64 * 64;
    // candidate margin beyond knn for the fp16 keys (tuning knob for experiments)
    const char* menv = std::getenv("SPECLUST_KNN_MARGIN");
    const int64_t tc_margin = menv ? std::max<int64_t>(1, std::atoll(menv)) : std::max<int64_t>(12, knn / 2 + 8);
    // the tensor-core path sorts lists of <= TC_LIST_P slots and needs R + 16 <= cap
    const bool use_tc = dp64 <= 256 && knn + tc_margin + 16 <= TC_LIST_P && n > 2 * (knn + tc_margin) + 1 &&
                        !(kenv && std::strcmp(kenv, "simt") == 0);
    // list budget: R kept candidates per row, 2R append capacity.  The fp16
    // tensor-core keys carry a larger error bound than fp32, so keep more.
    const int64_t margin = use_tc ? tc_margin : std::max<int64_t>(8, knn / 2);
    const int R = (int)imin64(n - 1, knn + margin);
    int cap;
    if (use_tc) {
        // a compaction leaves R entries and must leave room for one 16-column chunk
        // capacity 2R + 16 (<= the sort width): each warp compaction frees
        // R + 16 slots (C2: 128 -> -9 ms of list maintenance vs 2R); tuning knob
        const char* cenv = std::getenv("SPECLUST_KNN_CAP");
        // the query-pair kernel (d <= 128) compacts by radix select up to
        // TC2_LIST_MAX entries and hands the recheck <= TC_LIST_P: a longer
        // append list means ~3x fewer compactions (each frees cap - R slots)
        const char* tenv = std::getenv("SPECLUST_KNN_TC");
        const bool tc2 = dp64 <= 128 && !(tenv && std::strcmp(tenv, "1") == 0);
        const int64_t cmax = tc2 ? TC2_LIST_MAX : TC_LIST_P;
        cap = (int)std::min<int64_t>(std::max<int64_t>(cenv ? std::atoll(cenv) : 2 * R + 16, R + 16),
                                     cmax);
    } else {
        cap = 2 * R;
        if (cap > n - 1) cap = (int)(n - 1);  // lists can hold every other point
        if (cap < R) cap = R;
    }
    const int64_t np = p1 - p0;  // positions of this call
    const int64_t qtile0 = p0 / 128, qtile1 = ceil_div(p1, 128), nq = qtile1 - qtile0;
    const int64_t nslots = nq * 128;  // list slots (whole query tiles)
    int rc;
    DevBuf<double> part, mean, rn, qn;
    DevBuf<float> xf, cnf, taus;
    DevBuf<__half> xh;
    DevBuf<unsigned long long> rmax, nflag;
    DevBuf<float2> lists;
    DevBuf<int> counts;
    DevBuf<int32_t> flagged;
    const int64_t nbc = ceil_div(n, 256);
    const int64_t n_pad = (n + 127) / 128 * 128;
    if ((rc = part.alloc((size_t)nbc * d)) || (rc = mean.alloc(d)) || (rc = rn.alloc(n)) || (rc = qn.alloc(n)) ||
        (rc = taus.alloc(nslots)) || (rc = rmax.alloc(1)) || (rc = nflag.alloc(1)) ||
        (rc = lists.alloc((size_t)nslots * cap)) || (rc = counts.alloc(nslots)) || (rc = flagged.alloc(np)))
        return rc;
    // ---- prep: fp64 column means (the key is translation invariant; centring
    // shrinks |x| and with it the error bound)
    colsum_partial_kernel<<<(unsigned)nbc, 128, 0, st>>>(n, d, x, part.p);
    colmean_finish_kernel<<<(unsigned)ceil_div(d, 128), 128, 0, st>>>(nbc, n, d, part.p, mean.p);
    SC_CUDA(cudaMemsetAsync(rmax.p, 0, sizeof(unsigned long long), st));
    SC_CUDA(cudaMemsetAsync(nflag.p, 0, sizeof(unsigned long long), st));
    SC_LAUNCHED(2);
    double cdelta;
    const int32_t* perm = nullptr;  // scan order -> original index (nullptr: identity)
    DevBuf<double> piv;
    DevBuf<int64_t> plab;
    Bucketer bk;
    if (use_tc) {
        knn_rownorm_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, d, x, mean.p, rn.p, rmax.p);
        SC_LAUNCHED(1);
        unsigned long long rb = 0;
        SC_CUDA(d2h_sync(&rb, rmax.p, sizeof(rb), st));
        double rm;
        std::memcpy(&rm, &rb, sizeof(rm));
        // power-of-two scale: every |element| <= 128, |row|^2 stays far from overflow
        const double scale = rm > 0 ? std::ldexp(1.0, (int)std::floor(std::log2(128.0 / rm))) : 1.0;
        // locality order for the scan: points bucketed (stably) by their nearest
        // of C strided pivots, so a query tile's neighbours sit in nearby
        // candidate tiles and its threshold tightens within the first tiles
        if (n >= 4096 && !std::getenv("SPECLUST_KNN_NOSORT")) {
            const int64_t C = std::min<int64_t>(1024, std::max<int64_t>(8, n / 1024));
            if ((rc = piv.alloc((size_t)C * d)) || (rc = plab.alloc(n)) || (rc = bk.init(n, C))) return rc;
            ProfScope prof_order("knn_order", st, 0.0);
            PhaseClock pc(st);
            gather_strided_rows_kernel<<<(unsigned)C, 128, 0, st>>>(n, d, C, x, piv.p);
            SC_LAUNCHED(1);
            if (!std::getenv("SPECLUST_KNN_NOREFINE")) {
                // a few Lloyd steps of the pivots on a strided subsample: raw
                // strided pivots in high dimension split a dense region among
                // the pivots of other regions (nearest-pivot distances are all
                // alike); refined pivots sit inside the regions
                const int64_t ns = std::min<int64_t>(n, 32 * C);
                DevBuf<double> sub, cent;
                DevBuf<int64_t> slab;
                if ((rc = sub.alloc((size_t)ns * d)) || (rc = cent.alloc((size_t)C * d)) || (rc = slab.alloc(ns)))
                    return rc;
                gather_strided_rows_kernel<<<(unsigned)ns, 128, 0, st>>>(n, d, ns, x, sub.p);
                SC_LAUNCHED(1);
                std::vector<double> hist(8);
                int64_t its = 0;
                ProfMute mute;
                if ((rc = sc_lloyd(ns, d, C, sub.p, piv.p, 4, 0, slab.p, cent.p, hist.data(), &its,
                                   reinterpret_cast<sc_stream_t>(st))))
                    return rc;
                SC_CUDA(cudaMemcpyAsync(piv.p, cent.p, sizeof(double) * C * d, cudaMemcpyDeviceToDevice, st));
                pc.lap("refine (lloyd on pivots)");
            }
            if (!std::getenv("SPECLUST_KNN_NOTOUR")) {
                // renumber the pivots along a nearest-neighbour tour: bucket
                // b's points then sit next to those of the pivots closest to
                // b, so a dense region is one index range (kNN scan order and
                // the eigensolver's SpMV locality)
                DevBuf<float> pd;
                DevBuf<double> piv2;
                DevBuf<int32_t> ord;
                if ((rc = pd.alloc((size_t)C * C)) || (rc = piv2.alloc((size_t)C * d)) || (rc = ord.alloc(C)))
                    return rc;
                pivot_dist_kernel<<<dim3((unsigned)ceil_div(C, 128), (unsigned)C), 128, 0, st>>>(C, d, piv.p, pd.p);
                SC_LAUNCHED(1);
                std::vector<float> hd((size_t)C * C);
                SC_CUDA(d2h_sync(hd.data(), pd.p, sizeof(float) * C * C, st));
                std::vector<int32_t> order;
                pivot_tour(C, hd, order);
                SC_CUDA(cudaMemcpyAsync(ord.p, order.data(), sizeof(int32_t) * C, cudaMemcpyHostToDevice, st));
                gather_pivots_kernel<<<(unsigned)C, 128, 0, st>>>(C, d, piv.p, ord.p, piv2.p);
                SC_CUDA(cudaMemcpyAsync(piv.p, piv2.p, sizeof(double) * C * d, cudaMemcpyDeviceToDevice, st));
                SC_CUDA(cudaStreamSynchronize(st));  // `order` leaves scope
                SC_LAUNCHED(1);
            }
            pc.lap("tour");
            if ((rc = assign_nearest(n, d, x, C, piv.p, plab.p, st)) || (rc = bk.run(plab.p, st))) return rc;
            pc.lap("assign + buckets");
            perm = bk.members.p;
        }
        if ((rc = xh.alloc((size_t)n_pad * dp64)) || (rc = cnf.alloc(n_pad))) return rc;
        knn_prep_f16_kernel<<<(unsigned)ceil_div(n_pad, 8), 256, 0, st>>>(n, n_pad, d, dp64, x, mean.p, scale, perm,
                                                                          xh.p, cnf.p, qn.p);
        SC_LAUNCHED(1);
        PhaseClock pct(st);
        if ((rc = knn_candidates_tc(n, n_pad, dp64, xh.p, cnf.p, (float)(-2.0 / (scale * scale)), qtile0, nq, cap, R,
                                    lists.p, counts.p, taus.p, st)))
            return rc;
        pct.lap("candidate tiles");
        if (std::getenv("SPECLUST_KNN_TILE_ONLY"))  // profiling: stop after the candidate kernel
            return fail(SC_ERR_VALUE, "SPECLUST_KNN_TILE_ONLY set");
        // fp16 rounding of both operands (u = 2^-11) + fp32 accumulation of
        // dp64 products + fp32 rounding of |x_j|^2 and of the key, relative to
        // (|x_i| + |x_j|)^2; 10% slack on top.
        cdelta = 1.1 * (2.0 * std::ldexp(1.0, -11) + (double)(dp64 + 8) * std::ldexp(1.0, -24));
    } else {
        if ((rc = xf.alloc((size_t)n * dp)) || (rc = cnf.alloc(n))) return rc;
        knn_prep_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, d, dp, x, mean.p, xf.p, cnf.p, rn.p, qn.p,
                                                                  rmax.p);
        SC_LAUNCHED(1);
        size_t smem = sizeof(float) * (KK * KM + KK * KN + KM * (KN + 1) + KN);
        cudaFuncSetAttribute(knn_cand_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        ProfScope prof("knn_tile", st, 2.0 * (double)np * (double)n * (double)d);
        knn_cand_simt_kernel<<<(unsigned)nq, 256, smem, st>>>(n, qtile0, (int)dp, xf.p, cnf.p, cap, R, lists.p,
                                                              counts.p, taus.p);
        SC_LAUNCHED(1);
        // fp32 inputs (u = 2^-24) and a dp-term fp32 accumulation
        cdelta = (2.0 * (double)dp + 16.0) * std::ldexp(1.0, -24);
    }
    // list slots start at tile qtile0; the recheck addresses them from p0
    const int64_t slot0 = p0 - qtile0 * 128;
    // ---- exact recheck + certificate
    DevBuf<double> xs;  // points in scan order (exp_decay with a locality order)
    if (perm && ms.kind == 0) {
        if ((rc = xs.alloc((size_t)n * d))) return rc;
        gather_rows_i32_kernel<<<(unsigned)ceil_div(n * d, 256), 256, 0, st>>>(n, d, x, perm, xs.p);
        SC_LAUNCHED(1);
    }
    {
        size_t smem = (size_t)8 * (kStageWarp * sizeof(double) + cap * (2 * sizeof(double) + sizeof(int)));
        cudaFuncSetAttribute(knn_recheck_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        ProfScope prof("knn_recheck", st, (double)np * cap * d * 8.0);
        knn_recheck_kernel<<<(unsigned)ceil_div(np, 8), 256, smem, st>>>(
            n, p0, p1, d, x, knn, inv, cap, lists.p + slot0 * cap, counts.p + slot0, taus.p + slot0, rn.p, qn.p,
            rmax.p, cdelta, perm, sel, flagged.p, nflag.p, ms, xs.p, selv);
        SC_LAUNCHED(1);
    }
    PhaseClock pcr(st);
    unsigned long long hflag = 0;
    SC_CUDA(d2h_sync(&hflag, nflag.p, sizeof(hflag), st));
    if (pcr.on) fprintf(stderr, "[knn_order] flagged rows %llu\n", hflag);
    lists.free();
    xf.free();
    xh.free();
    if (hflag > 0) {
        int64_t grid = imin64((int64_t)hflag, kNumSMs);
        DevBuf<unsigned long long> scratch;
        if ((rc = scratch.alloc((size_t)grid * n))) return rc;
        ProfScope prof("knn_fallback", st, (double)hflag * n * d * 8.0);
        knn_fallback_kernel<<<(unsigned)grid, 512, 0, st>>>(n, p0, d, x, knn, inv, perm, flagged.p, (int64_t)hflag,
                                                            scratch.p, sel, ms, selv);
        SC_LAUNCHED(1);
    }
    {
        ProfScope prof("knn_union", st, 0.0);
        if (hflag > 0)
            sort_rows_kernel<<<(unsigned)ceil_div((int64_t)hflag, 128), 128, 0, st>>>((int64_t)hflag, flagged.p, p0,
                                                                                     knn, sel, selv);
        if (perm)
            SC_CUDA(cudaMemcpyAsync(perm_out, perm, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
        else
            iota_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, perm_out);
        SC_LAUNCHED((hflag > 0 ? 1 : 0) + (perm ? 0 : 1));
    }
    pcr.lap("fallback + sort");
    // the pooled scratch above is released on st; callers see sel/perm ordered on st
    if (stats) {
        stats[0] = R;
        stats[1] = cap;
        stats[2] = (int64_t)hflag;
        for (int q = 3; q < 8; ++q) stats[q] = 0;
    }
    return SC_OK;
}

// Union stage: CSR rows [r0, r1) (local row_ptr, global columns) of the
// symmetrised kNN graph from the selections of all n points.
int knn_union(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq, const int32_t* sel,
              const int32_t* perm, int64_t r0, int64_t r1, int64_t* row_ptr, int32_t* col, double* vals, int64_t cap,
              int64_t* nnz_out, cudaStream_t st, KnnMeasure ms = KnnMeasure(), const double* selv = nullptr) {
    const int64_t nl = r1 - r0;
    int rc;
    DevBuf<int32_t> pos, rev;
    DevBuf<int64_t> rc_cnt, rev_ptr, len, tmp;
    DevBuf<unsigned int> fill;
    DevBuf<uint8_t> dup;
    if ((rc = pos.alloc(n)) || (rc = rc_cnt.alloc(nl)) || (rc = rev_ptr.alloc(nl + 1)) || (rc = len.alloc(nl)) ||
        (rc = tmp.alloc(ceil_div(std::max<int64_t>(n, nl), SCAN_BLK) + 1)) || (rc = fill.alloc(nl)))
        return rc;
    ProfScope prof("knn_union", st, 0.0);
    pos_of_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, perm, pos.p);
    SC_CUDA(cudaMemsetAsync(rc_cnt.p, 0, sizeof(int64_t) * nl, st));
    SC_CUDA(cudaMemsetAsync(fill.p, 0, sizeof(unsigned int) * nl, st));
    rev_count_kernel<<<(unsigned)ceil_div(n * knn, 256), 256, 0, st>>>(n * knn, r0, r1, sel, rc_cnt.p);
    SC_LAUNCHED(2);
    if ((rc = exclusive_scan_i64(nl, rc_cnt.p, rev_ptr.p, tmp.p, st))) return rc;
    int64_t nrev = 0;
    SC_CUDA(d2h_sync(&nrev, rev_ptr.p + nl, sizeof(int64_t), st));
    DevBuf<int64_t> rev_src;  // with selv: the selection slot of each reverse entry
    if ((rc = rev.alloc(std::max<int64_t>(nrev, 1))) || (rc = dup.alloc(std::max<int64_t>(nrev, 1)))) return rc;
    if (selv && (rc = rev_src.alloc(std::max<int64_t>(nrev, 1)))) return rc;
    rev_fill_kernel<<<(unsigned)ceil_div(n * knn, 256), 256, 0, st>>>(n, knn, r0, r1, sel, perm, rev_ptr.p, fill.p,
                                                                      rev.p, rev_src.p);
    row_count_kernel<<<(unsigned)ceil_div(nl, 8), 256, 0, st>>>(nl, r0, knn, sel, pos.p, rev_ptr.p, rev.p, dup.p,
                                                                len.p);
    SC_LAUNCHED(2);
    if ((rc = exclusive_scan_i64(nl, len.p, row_ptr, tmp.p, st))) return rc;
    int64_t nnz = 0;
    SC_CUDA(d2h_sync(&nnz, row_ptr + nl, sizeof(int64_t), st));
    *nnz_out = nnz;
    if (nnz > cap)
        return fail(SC_ERR_VALUE, "knn union: " + std::to_string(nnz) + " entries exceed the output capacity " +
                                      std::to_string(cap));
    if (selv) {
        DevBuf<int64_t> long_rows;
        DevBuf<unsigned int> nlong;
        if ((rc = long_rows.alloc(nl)) || (rc = nlong.alloc(1))) return rc;
        SC_CUDA(cudaMemsetAsync(nlong.p, 0, sizeof(unsigned int), st));
        row_fill_vals_kernel<<<(unsigned)ceil_div(nl, 8), 256, 0, st>>>(
            nl, r0, knn, two_sigma_sq, sel, selv, pos.p, rev_ptr.p, rev.p, rev_src.p, dup.p, row_ptr, col, vals,
            (r0 == 0 && nl == n) ? perm : nullptr, ms.kind, ms.policy, long_rows.p, nlong.p);
        row_fill_long_kernel<<<(unsigned)(2 * kNumSMs), 256, 0, st>>>(r0, knn, two_sigma_sq, sel, selv, pos.p,
                                                                      rev_ptr.p, rev.p, rev_src.p, dup.p, row_ptr, col,
                                                                      vals, ms.kind, ms.policy, long_rows.p, nlong.p);
        SC_LAUNCHED(2);
        return SC_OK;
    }
    DevBuf<double> xs;  // points in scan order: the neighbours of a row are close there
    if (perm && r0 == 0 && nl == n && ms.kind == 0) {
        if ((rc = xs.alloc((size_t)n * d))) return rc;
        gather_rows_i32_kernel<<<(unsigned)ceil_div(n * d, 256), 256, 0, st>>>(n, d, x, perm, xs.p);
        SC_LAUNCHED(1);
    }
    row_fill_kernel<<<(unsigned)ceil_div(nl, 4), 128, 0, st>>>(nl, r0, d, knn, x, two_sigma_sq, sel, pos.p, rev_ptr.p,
                                                               rev.p, dup.p, row_ptr, col, vals,
                                                               (r0 == 0 && nl == n) ? perm : nullptr, ms, xs.p);
    SC_LAUNCHED(1);
    return SC_OK;
}

int knn_graph_build(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq, int64_t* row_ptr,
                    int32_t* col, double* vals, int64_t* nnz_out, int64_t* stats, cudaStream_t st) {
    DevBuf<int32_t> sel, perm;
    DevBuf<double> selv;  // exact d2 of every selection slot, reused by the CSR fill
    int rc;
    if ((rc = sel.alloc((size_t)n * knn)) || (rc = perm.alloc(n)) || (rc = selv.alloc((size_t)n * knn))) return rc;
    PhaseClock pc(st);
    if ((rc = knn_select(n, d, x, knn, two_sigma_sq, 0, n, sel.p, perm.p, stats, st, KnnMeasure(), selv.p)))
        return rc;
    pc.lap("select total");
    if ((rc = knn_union(n, d, x, knn, two_sigma_sq, sel.p, perm.p, 0, n, row_ptr, col, vals, 2 * n * knn, nnz_out,
                        st, KnnMeasure(), selv.p)))
        return rc;
    pc.lap("union");
    if (stats) stats[3] = *nnz_out;
    return SC_OK;
}

}  // namespace sc

static int check_knn_args(int64_t n, int64_t d, int64_t knn, double two_sigma_sq) {
    if (n < 2 || d < 1) return fail(SC_ERR_FORMAT, "point matrix must be 2-D with n >= 2, d >= 1");
    if (!(knn >= 1 && knn < n))
        return fail(SC_ERR_VALUE, "knn must satisfy 1 <= knn < n, got " + std::to_string(knn) + " for n=" +
                                      std::to_string(n));
    if (!(two_sigma_sq > 0)) return fail(SC_ERR_VALUE, "exp_decay requires sigma > 0");
    if (n >= (int64_t)INT32_MAX) return fail(SC_ERR_VALUE, "n must be < 2^31 for int32 column indices");
    return SC_OK;
}

extern "C" int sc_knn_graph_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq,
                                int64_t* row_ptr, int32_t* col, double* vals, int64_t* nnz_out, int64_t* stats_out,
                                sc_stream_t stream) {
    if (int rc = check_knn_args(n, d, knn, two_sigma_sq)) return rc;
    StreamScope stream_scope(as_stream(stream));
    return knn_graph_build(n, d, x, knn, two_sigma_sq, row_ptr, col, vals, nnz_out, stats_out, as_stream(stream));
}

extern "C" int sc_knn_select_vals_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq,
                                      int64_t p0, int64_t p1, int32_t* sel, double* sel_vals, int32_t* perm,
                                      int64_t* stats_out, sc_stream_t stream) {
    if (int rc = check_knn_args(n, d, knn, two_sigma_sq)) return rc;
    if (!(0 <= p0 && p0 <= p1 && p1 <= n) || p0 % 128 != 0)
        return fail(SC_ERR_VALUE, "scan range [p0, p1) must lie in [0, n] with p0 a multiple of 128");
    StreamScope stream_scope(as_stream(stream));
    if (p0 == p1) {  // empty shard: still provide the scan order
        int64_t tmp[8];
        DevBuf<int32_t> s1;
        if (int rc = s1.alloc((size_t)128 * knn)) return rc;
        const int64_t q0 = std::min<int64_t>(p0, n - 1) / 128 * 128;
        return knn_select(n, d, x, knn, two_sigma_sq, q0, q0 + 1, s1.p, perm, stats_out ? stats_out : tmp,
                          as_stream(stream));
    }
    return knn_select(n, d, x, knn, two_sigma_sq, p0, p1, sel, perm, stats_out, as_stream(stream), KnnMeasure(),
                      sel_vals);
}

extern "C" int sc_knn_select_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq, int64_t p0,
                                 int64_t p1, int32_t* sel, int32_t* perm, int64_t* stats_out, sc_stream_t stream) {
    return sc_knn_select_vals_f64(n, d, x, knn, two_sigma_sq, p0, p1, sel, nullptr, perm, stats_out, stream);
}

extern "C" int sc_knn_union_vals_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq,
                                     const int32_t* sel, const double* sel_vals, const int32_t* perm, int64_t r0,
                                     int64_t r1, int64_t* row_ptr, int32_t* col, double* vals, int64_t cap,
                                     int64_t* nnz_out, sc_stream_t stream) {
    if (int rc = check_knn_args(n, d, knn, two_sigma_sq)) return rc;
    if (!(0 <= r0 && r0 <= r1 && r1 <= n)) return fail(SC_ERR_VALUE, "row range [r0, r1) must lie in [0, n]");
    StreamScope stream_scope(as_stream(stream));
    if (r0 == r1) {
        *nnz_out = 0;
        const int64_t z = 0;
        SC_CUDA(cudaMemcpyAsync(row_ptr, &z, sizeof(z), cudaMemcpyHostToDevice, as_stream(stream)));
        SC_CUDA(cudaStreamSynchronize(as_stream(stream)));
        return SC_OK;
    }
    return knn_union(n, d, x, knn, two_sigma_sq, sel, perm, r0, r1, row_ptr, col, vals, cap, nnz_out,
                     as_stream(stream), KnnMeasure(), sel_vals);
}

extern "C" int sc_knn_union_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq,
                                const int32_t* sel, const int32_t* perm, int64_t r0, int64_t r1, int64_t* row_ptr,
                                int32_t* col, double* vals, int64_t cap, int64_t* nnz_out, sc_stream_t stream) {
    return sc_knn_union_vals_f64(n, d, x, knn, two_sigma_sq, sel, nullptr, perm, r0, r1, row_ptr, col, vals, cap,
                                 nnz_out, stream);
}

// exp(-d2 / (2 sigma^2)) per given pair (graph.py:136-141; build_similarity)
namespace sc {
__global__ void pair_weights_kernel(int64_t m, int64_t d, const double* __restrict__ x, const int64_t* __restrict__ e,
                                    double den, double* __restrict__ out) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= m) return;
    int64_t a = e[2 * p], b = e[2 * p + 1];
    out[p] = exp(-exact_d2(x + a * d, x + b * d, d) / den);
}
}  // namespace sc

extern "C" int sc_pair_weights(int64_t n, int64_t d, const double* x, int64_t m, const int64_t* pairs,
                               double two_sigma_sq, double* out, sc_stream_t stream) {
    (void)n;
    if (m <= 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    pair_weights_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(m, d, x, pairs, two_sigma_sq, out);
    SC_LAUNCHED(1);
    return SC_OK;
}

// ---- kNN graph with the cosine / cross-correlation measures ------------------
namespace sc {
// xc = x - mean(x, axis=1) (centre) or x, sq = einsum(xc, xc), xn = xc / sqrt(sq)
__global__ void corr_prep_kernel(int64_t n, int64_t d, const double* __restrict__ x, int centre,
                                 double* __restrict__ xc, double* __restrict__ sq, double* __restrict__ xn,
                                 unsigned long long* __restrict__ first_bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* xi = x + i * d;
    double* oi = xc + i * d;
    const double mu = centre ? __ddiv_rn(__dadd_rn(0.0, np_pairwise_sum_dev(xi, d)), (double)d) : 0.0;
    for (int64_t l = 0; l < d; ++l) oi[l] = centre ? __dsub_rn(xi[l], mu) : xi[l];
    const double q = np_sqnorm(oi, d);
    sq[i] = q;
    if (q == 0.0) atomicMin(first_bad, (unsigned long long)i);
    const double r = q > 0.0 ? 1.0 / sqrt(q) : 0.0;
    for (int64_t l = 0; l < d; ++l) xn[i * d + l] = oi[l] * r;
}
}  // namespace sc

// Union-kNN similarity graph for any measure (graph.py:149-163, 185-237):
// kind 0 exp_decay (sigma), 1 cosine, 2 cross_correlation; negative_policy
// 0 clamp_zero, 1 abs, 2 keep.  The candidate search runs on the
// row-normalised (centred) points; ranking, the certificate and the edge
// values use the reference's formula.  A degenerate point returns
// SC_ERR_VALUE with *degenerate (host) = its index.
extern "C" int sc_knn_graph_measure_f64(int64_t n, int64_t d, const double* x, int64_t knn, int kind, double sigma,
                                        int negative_policy, int64_t* row_ptr, int32_t* col, double* vals,
                                        int64_t* nnz_out, int64_t* stats_out, int64_t* degenerate,
                                        sc_stream_t stream) {
    *degenerate = -1;
    if (kind == 0) return sc_knn_graph_f64(n, d, x, knn, 2.0 * (sigma * sigma), row_ptr, col, vals, nnz_out,
                                           stats_out, stream);
    if (kind != 1 && kind != 2) return fail(SC_ERR_VALUE, "measure kind must be 0, 1 or 2");
    if (int rc = check_knn_args(n, d, knn, 1.0)) return rc;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    DevBuf<double> xc, sq, xn;
    DevBuf<unsigned long long> bad;
    DevBuf<int32_t> sel, perm;
    DevBuf<double> selv;
    int rc;
    if ((rc = xc.alloc((size_t)n * d)) || (rc = sq.alloc(n)) || (rc = xn.alloc((size_t)n * d)) || (rc = bad.alloc(1)) ||
        (rc = sel.alloc((size_t)n * knn)) || (rc = perm.alloc(n)) || (rc = selv.alloc((size_t)n * knn)))
        return rc;
    SC_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
    corr_prep_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(n, d, x, kind == 2, xc.p, sq.p, xn.p, bad.p);
    SC_LAUNCHED(1);
    unsigned long long hb = 0;
    SC_CUDA(d2h_sync(&hb, bad.p, sizeof(hb), st));
    if (hb != ~0ull) {  // graph.py:158-163: every point is checked
        *degenerate = (int64_t)hb;
        return fail(SC_ERR_VALUE, "degenerate vector at point index " + std::to_string(hb));
    }
    KnnMeasure ms;
    ms.kind = 1;
    ms.xc = xc.p;
    ms.sq = sq.p;
    ms.policy = negative_policy;
    int64_t tmp[8];
    int64_t* stats = stats_out ? stats_out : tmp;
    if ((rc = knn_select(n, d, xn.p, knn, 1.0, 0, n, sel.p, perm.p, stats, st, ms, selv.p))) return rc;
    if ((rc = knn_union(n, d, xn.p, knn, 1.0, sel.p, perm.p, 0, n, row_ptr, col, vals, 2 * n * knn, nnz_out, st,
                        ms, selv.p)))
        return rc;
    stats[3] = *nnz_out;
    return SC_OK;
}
