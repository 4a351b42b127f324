// k-means: fp64 Gram-expansion distance tiles with fused argmin epilogue,
// stable label bucketing + point-order centroid sums, farthest-point reseed,
// k-means++ device steps, Lloyd driver, and the ncut metric.
//
// Reference semantics (kmeans.py:84-196, metrics.py:59-67):
//   S = (|v|^2 + |c|^2) - 2 v.c, clamped at 0; argmin ties -> lowest index;
//   centroid = (sum of members in point order) / count; empty clusters take
//   the rows with the largest current cost (stable: ties -> lower index).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include "sc_common.cuh"
#include "sc_sparse.cuh"
#include "sc_scan.cuh"

namespace sc {

__device__ __forceinline__ int64_t ceil_div_dev(int64_t d) { return (d + 31) / 32; }

// ---------------------------------------------------------------------------
// row squared norms in numpy's einsum order (kmeans.py:92-97): the same
// order the distance tile uses for v.c, so the expansion is bit-identical to
// the reference and identical rows give an exact zero (test_kmeans.py:23-27)
__global__ void rownorm_kernel(int64_t n, int64_t d, const double* __restrict__ v,
                               double* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = np_sqnorm(v + i * d, d);
}

constexpr int TP = 64, TQ = 64, KC = 16;

// MODE 0: assignment (argmin epilogue); MODE 1: write the clamped n x k matrix.
template <int MODE>
__global__ void __launch_bounds__(256) dist_tile_kernel(
    int64_t n, int64_t k, int64_t d, const double* __restrict__ v, const double* __restrict__ vn,
    const double* __restrict__ c, const double* __restrict__ cn, double* __restrict__ out,
    int64_t* __restrict__ labels, const int64_t* __restrict__ old_labels,
    double* __restrict__ cost, unsigned long long* __restrict__ changes,
    double* __restrict__ cost_partial) {
    __shared__ double Vs[KC][TP + 1];
    __shared__ double Cs[KC][TQ + 1];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t p0 = (int64_t)blockIdx.x * TP;

    double best[4];
    int64_t arg[4];
    double vnr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        best[i] = INFINITY;
        arg[i] = 0;
        int64_t p = p0 + ty + 16 * i;
        vnr[i] = p < n ? vn[p] : 0.0;
    }

    for (int64_t q0 = 0; q0 < k; q0 += TQ) {
        // v.c in numpy's einsum order (NpDot): even / odd lane accumulators
        double acc[4][4], acc1[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = acc1[i][j] = 0.0;
        for (int64_t l0 = 0; l0 < d; l0 += KC) {
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                int idx = tid + 256 * r;
                int pp = idx >> 4, ll = idx & 15;
                int64_t gp = p0 + pp, gl = l0 + ll;
                Vs[ll][pp] = (gp < n && gl < d) ? v[gp * d + gl] : 0.0;
                int64_t gq = q0 + pp;
                Cs[ll][pp] = (gq < k && gl < d) ? c[gq * d + gl] : 0.0;
            }
            __syncthreads();
            const int lmax = (int)imin64(KC, d - l0);
            // acc += p_l for element l (unfused), into the even or odd lane
            auto step = [&](int l, bool odd) {
                double a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = Vs[l][ty + 16 * i];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = Cs[l][tx + 16 * j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        double& r = odd ? acc1[i][j] : acc[i][j];
                        r = __dadd_rn(__dmul_rn(a[i], b[j]), r);
                    }
            };
            int l = 0;
            for (; l + 8 <= lmax; l += 8) {  // whole block: p0 + (p2 + (p4 + (p6 + acc)))
#pragma unroll
                for (int t = 6; t >= 0; t -= 2) {
                    step(l + t, false);
                    step(l + t + 1, true);
                }
            }
            for (; l + 2 <= lmax; l += 2) {
                step(l, false);
                step(l + 1, true);
            }
            if (l < lmax) step(l, false);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], acc1[i][j]);
        // epilogue for this centroid tile
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t q = q0 + tx + 16 * j;
            if (q >= k) continue;
            double cq = cn[q];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double s = __dsub_rn(__dadd_rn(vnr[i], cq), __dmul_rn(2.0, acc[i][j]));
                s = s > 0.0 ? s : 0.0;  // np.maximum(s, 0.0)
                if (MODE == 1) {
                    int64_t p = p0 + ty + 16 * i;
                    if (p < n) out[p * k + q] = s;
                } else if (s < best[i]) {
                    best[i] = s;
                    arg[i] = q;
                }
            }
        }
    }
    if (MODE == 1) return;
    // reduce (best, arg) over the 16 lanes sharing a point: lexicographic min
    double blk_cost = 0.0;
    int nchg = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        double b = best[i];
        int64_t a = arg[i];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            double ob = __shfl_xor_sync(0xffffffffu, b, o);
            int64_t oa = __shfl_xor_sync(0xffffffffu, a, o);
            if (ob < b || (ob == b && oa < a)) {
                b = ob;
                a = oa;
            }
        }
        int64_t p = p0 + ty + 16 * i;
        if (tx == 0 && p < n) {
            labels[p] = a;
            cost[p] = b;
            if (old_labels) nchg += (old_labels[p] != a);
        }
    }
    // per-block cost sum in fixed order (deterministic)
    __shared__ double red[TP];
    __shared__ int chg[TP];
    if (tx == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int64_t p = p0 + ty + 16 * i;
            red[ty + 16 * i] = p < n ? cost[p] : 0.0;
        }
        chg[ty] = nchg;
    }
    __syncthreads();
    if (tid == 0) {
        for (int i = 0; i < TP; ++i) blk_cost += red[i];
        int tot = 0;
        for (int i = 0; i < 16; ++i) tot += chg[i];
        cost_partial[blockIdx.x] = blk_cost;
        if (tot) atomicAdd(changes, (unsigned long long)tot);
    }
}

// sum of a partial array in fixed order by one block (deterministic)
__global__ void sum_partials_kernel(int64_t m, const double* __restrict__ part, double* __restrict__ out) {
    __shared__ double red[1024];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc += part[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// ---------------------------------------------------------------------------
// Stable bucketing by label.
constexpr int BK_ITEMS = 2048;  // items per bucketing block (one warp per block)

__global__ void bucket_count_kernel(int64_t n, int64_t k, const int64_t* __restrict__ labels,
                                    int32_t* __restrict__ blkcount) {
    int64_t b = blockIdx.x;
    int32_t* row = blkcount + b * k;
    for (int64_t c = threadIdx.x; c < k; c += blockDim.x) row[c] = 0;
    __syncthreads();
    int64_t lo = b * BK_ITEMS, hi = imin64(n, lo + BK_ITEMS);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(row + labels[i], 1);
}

// per label: exclusive offsets over blocks in block order; start[] over labels
__global__ void bucket_offsets_kernel(int64_t nblk, int64_t k, const int32_t* __restrict__ blkcount,
                                      int64_t* __restrict__ blkoff, int64_t* __restrict__ total) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k) return;
    int64_t run = 0;
    for (int64_t b = 0; b < nblk; ++b) {
        blkoff[b * k + c] = run;
        run += blkcount[b * k + c];
    }
    total[c] = run;
}

__global__ void exclusive_scan_small_kernel(int64_t k, int64_t* __restrict__ start) {
    // start[0..k) holds totals on entry; converts in place to offsets, start[k] = sum
    if (threadIdx.x != 0) return;
    int64_t run = 0;
    for (int64_t c = 0; c < k; ++c) {
        int64_t t = start[c];
        start[c] = run;
        run += t;
    }
    start[k] = run;
}

__global__ void bucket_scatter_kernel(int64_t n, int64_t k, const int64_t* __restrict__ labels,
                                      const int64_t* __restrict__ blkoff,
                                      const int64_t* __restrict__ start,
                                      int32_t* __restrict__ members) {
    extern __shared__ int32_t run[];  // k counters
    int64_t b = blockIdx.x;
    for (int64_t c = threadIdx.x; c < k; c += 32) run[c] = 0;
    __syncwarp();
    int lane = threadIdx.x;
    int64_t lo = b * BK_ITEMS, hi = imin64(n, lo + BK_ITEMS);
    const int64_t* off = blkoff + b * k;
    for (int64_t base = lo; base < hi; base += 32) {
        int64_t i = base + lane;
        bool valid = i < hi;
        int64_t lab = valid ? labels[i] : -1 - lane;
        unsigned peers = __match_any_sync(0xffffffffu, lab);
        int rank = __popc(peers & ((1u << lane) - 1u));
        int32_t before = valid ? run[lab] : 0;
        if (valid) members[start[lab] + off[lab] + before + rank] = (int32_t)i;
        __syncwarp();
        if (valid && rank == 0) run[lab] = before + __popc(peers);
        __syncwarp();
    }
}

int Bucketer::init(int64_t n_, int64_t k_) {
    n = n_;
    k = k_;
    nblk = ceil_div(n, BK_ITEMS);
    if (int rc = blkcount.alloc((size_t)std::max<int64_t>(1, nblk * k))) return rc;
    if (int rc = blkoff.alloc((size_t)std::max<int64_t>(1, nblk * k))) return rc;
    if (int rc = start.alloc((size_t)k + 1)) return rc;
    if (int rc = members.alloc((size_t)std::max<int64_t>(1, n))) return rc;
    return SC_OK;
}

int Bucketer::run(const int64_t* labels, cudaStream_t st) {
    if (n == 0) {
        SC_CUDA(cudaMemsetAsync(start.p, 0, sizeof(int64_t) * (k + 1), st));
        return SC_OK;
    }
    bucket_count_kernel<<<(unsigned)nblk, 256, 0, st>>>(n, k, labels, blkcount.p);
    bucket_offsets_kernel<<<(unsigned)ceil_div(k, 128), 128, 0, st>>>(nblk, k, blkcount.p, blkoff.p, start.p);
    exclusive_scan_small_kernel<<<1, 32, 0, st>>>(k, start.p);
    size_t smem = sizeof(int32_t) * (size_t)k;
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(bucket_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    bucket_scatter_kernel<<<(unsigned)nblk, 32, smem, st>>>(n, k, labels, blkoff.p, start.p, members.p);
    SC_LAUNCHED(4);
    return SC_OK;
}

// centroid = point-order member sum / count (kmeans.py:144-148; np.add.at is a
// sequential scatter-add in point order, reproduced exactly per (cluster, dim)).
__global__ void centroid_mean_kernel(int64_t k, int64_t d, const double* __restrict__ v,
                                     const int64_t* __restrict__ start,
                                     const int32_t* __restrict__ members,
                                     double* __restrict__ cent, int* __restrict__ empty_flag) {
    int64_t dchunks = ceil_div_dev(d);
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (w >= k * dchunks) return;
    int64_t cl = w / dchunks;
    int64_t dim = (w % dchunks) * 32 + lane;
    int64_t b = start[cl], e = start[cl + 1];
    if (e == b) {
        if (lane == 0 && (w % dchunks) == 0) empty_flag[cl] = 1;
        if (dim < d) cent[cl * d + dim] = 0.0;
        return;
    }
    if (dim >= d) return;
    // the sum is a strictly sequential chain (point order); only the loads are
    // batched, 16 in flight per thread, so the chain runs at add latency
    double acc = 0.0;
    int64_t m = b;
    constexpr int B = 16;
    for (; m + B <= e; m += B) {
        double x[B];
#pragma unroll
        for (int u = 0; u < B; ++u) x[u] = __ldg(v + (int64_t)__ldg(members + m + u) * d + dim);
#pragma unroll
        for (int u = 0; u < B; ++u) acc = __dadd_rn(acc, x[u]);
    }
    for (; m < e; ++m) acc = __dadd_rn(acc, v[(int64_t)members[m] * d + dim]);
    cent[cl * d + dim] = __ddiv_rn(acc, (double)(e - b));
}

// Segmented variant for large clusters: each cluster's member list (point
// order) is cut into segments of CM_SEG members; level 1 sums a segment
// sequentially (warp = segment x 32 features), level 2 adds the segment sums
// of a cluster in segment order and divides by the count.  Deterministic;
// identical to the point-order chain for clusters of <= CM_SEG members.
constexpr int64_t CM_SEG = INT64_MAX / 4;  // one segment per cluster: the exact point-order chain
__global__ void centroid_segsum_kernel(int64_t k, int64_t d, int64_t nseg, const double* __restrict__ v,
                                       const int64_t* __restrict__ start, const int32_t* __restrict__ members,
                                       const int64_t* __restrict__ seg_off, double* __restrict__ part) {
    const int64_t dchunks = ceil_div_dev(d);
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nseg * dchunks) return;
    const int64_t s = w / dchunks;
    const int64_t dim = (w % dchunks) * 32 + lane;
    // cluster owning global segment s: last c with seg_off[c] <= s
    int64_t lo = 0, hi = k;
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (seg_off[mid] <= s) lo = mid; else hi = mid;
    }
    const int64_t cl = lo;
    const int64_t b = start[cl] + (s - seg_off[cl]) * CM_SEG;
    const int64_t e = imin64(start[cl + 1], b + CM_SEG);
    // the chain is strictly sequential in point order (np.add.at); the warp
    // loads 64 member indices per batch (two coalesced loads, shuffled to
    // every lane) and then the 64 rows' values of its 32 features, so 64
    // independent loads are in flight per lane ahead of the dependent adds
    const bool on = dim < d;
    double acc = 0.0;
    int64_t m = b;
    constexpr int B = 64;
    for (; m + B <= e; m += B) {
        const int32_t i0 = __ldg(members + m + lane), i1 = __ldg(members + m + 32 + lane);
        double x[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int32_t r = __shfl_sync(0xffffffffu, u < 32 ? i0 : i1, u & 31);
            x[u] = on ? __ldg(v + (int64_t)r * d + dim) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < B; ++u) acc = __dadd_rn(acc, x[u]);
    }
    for (; m < e; ++m) acc = __dadd_rn(acc, on ? v[(int64_t)members[m] * d + dim] : 0.0);
    if (on) part[s * d + dim] = acc;
}

// The same point-order chains with the member rows staged in shared memory:
// one warp per CTA (one cluster x 32 features), batches of CS_BATCH member
// rows gathered with 8-byte cp.async into a double buffer while the previous
// batch is summed from shared memory; member indices are loaded one batch
// ahead of their gathers.  One gather latency is exposed per CS_BATCH rows
// instead of two per 64, and the add chain never waits on global memory.
constexpr int CS_BATCH = 128;
__device__ __forceinline__ void cs_cp8(double* dst, const double* src, bool pred) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(pred ? 8 : 0) : "memory");
}
__global__ void __launch_bounds__(32) centroid_segsum_smem_kernel(int64_t k, int64_t d, int64_t nseg,
                                                                 const double* __restrict__ v,
                                                                 const int64_t* __restrict__ start,
                                                                 const int32_t* __restrict__ members,
                                                                 const int64_t* __restrict__ seg_off,
                                                                 double* __restrict__ part) {
    extern __shared__ __align__(16) double cs_buf[];  // [2][CS_BATCH][32]
    const int64_t dchunks = ceil_div_dev(d);
    const int64_t w = blockIdx.x;
    const int lane = threadIdx.x;
    if (w >= nseg * dchunks) return;
    const int64_t s = w / dchunks;
    const int64_t dim = (w % dchunks) * 32 + lane;
    int64_t lo = 0, hi = k;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (seg_off[mid] <= s) lo = mid; else hi = mid;
    }
    const int64_t cl = lo;
    const int64_t b = start[cl] + (s - seg_off[cl]) * CM_SEG;
    const int64_t e = imin64(start[cl + 1], b + CM_SEG);
    const bool on = dim < d;
    const int64_t nb = (e - b + CS_BATCH - 1) / CS_BATCH;
    constexpr int PL = CS_BATCH / 32;  // member indices per lane per batch
    auto load_idx = [&](int64_t t, int32_t (&ix)[PL]) {
#pragma unroll
        for (int q = 0; q < PL; ++q) {
            const int64_t m = b + t * CS_BATCH + q * 32 + lane;
            ix[q] = (t < nb && m < e) ? __ldg(members + m) : -1;
        }
    };
    auto gather = [&](int64_t t, const int32_t (&ix)[PL]) {
        double* dst = cs_buf + (t & 1) * CS_BATCH * 32;
#pragma unroll
        for (int q = 0; q < PL; ++q) {
#pragma unroll 8
            for (int r = 0; r < 32; ++r) {
                const int32_t row = __shfl_sync(0xffffffffu, ix[q], r);
                cs_cp8(dst + (q * 32 + r) * 32 + lane, row >= 0 && on ? v + (int64_t)row * d + dim : v, row >= 0 && on);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    int32_t ia[PL], ib[PL];
    load_idx(0, ia);
    gather(0, ia);
    load_idx(1, ib);
    double acc = 0.0;
    for (int64_t t = 0; t < nb; ++t) {
        // gathers of batch t + 1 (indices already in ib), then the indices of t + 2
        if (t + 1 < nb) gather(t + 1, ib);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        load_idx(t + 2, ia);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncwarp();
        const double* src = cs_buf + (t & 1) * CS_BATCH * 32 + lane;
        const int rows = (int)imin64(CS_BATCH, e - (b + t * CS_BATCH));
        for (int r = 0; r < rows; ++r) acc = __dadd_rn(acc, src[r * 32]);
        __syncwarp();  // the buffer is refilled by the gathers of batch t + 2
#pragma unroll
        for (int q = 0; q < PL; ++q) ib[q] = ia[q];
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if (on) part[s * d + dim] = acc;
}
static int segsum_smem_attr() {
    static bool done = false;
    if (!done) {
        SC_CUDA(cudaFuncSetAttribute(centroid_segsum_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     2 * CS_BATCH * 32 * (int)sizeof(double)));
        done = true;
    }
    return SC_OK;
}


__global__ void centroid_segmean_kernel(int64_t k, int64_t d, const int64_t* __restrict__ start,
                                        const int64_t* __restrict__ seg_off, const double* __restrict__ part,
                                        double* __restrict__ cent) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= k * d) return;
    const int64_t cl = idx / d, dim = idx % d;
    const int64_t cnt = start[cl + 1] - start[cl];
    if (cnt == 0) {
        cent[idx] = 0.0;
        return;
    }
    double acc = 0.0;
    for (int64_t s = seg_off[cl]; s < seg_off[cl + 1]; ++s) acc = __dadd_rn(acc, part[s * d + dim]);
    cent[idx] = __ddiv_rn(acc, (double)cnt);
}

// unnormalised cluster totals + counts (shard partials for an all-reduce)
__global__ void centroid_segtotal_kernel(int64_t k, int64_t d, const int64_t* __restrict__ start,
                                         const int64_t* __restrict__ seg_off, const double* __restrict__ part,
                                         double* __restrict__ sums, int64_t* __restrict__ counts) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= k * d) return;
    const int64_t cl = idx / d, dim = idx % d;
    double acc = 0.0;
    for (int64_t s = seg_off[cl]; s < seg_off[cl + 1]; ++s) acc = __dadd_rn(acc, part[s * d + dim]);
    sums[idx] = acc;
    if (dim == 0) counts[cl] = start[cl + 1] - start[cl];
}

__global__ void centroid_divide_kernel(int64_t k, int64_t d, const double* __restrict__ sums,
                                       const int64_t* __restrict__ counts, double* __restrict__ cent) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= k * d) return;
    const int64_t c = counts[idx / d];
    cent[idx] = c > 0 ? __ddiv_rn(sums[idx], (double)c) : 0.0;
}

// argmax of cost over unmarked points, ties -> lowest index (one reseed slot)
__global__ void argmax_partial_kernel(int64_t n, const double* __restrict__ cost,
                                      const uint8_t* __restrict__ used, double* __restrict__ pv,
                                      int64_t* __restrict__ pi) {
    __shared__ double sv[256];
    __shared__ int64_t si[256];
    double bv = -INFINITY;
    int64_t bi = INT64_MAX;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (used[i]) continue;
        double c = cost[i];
        if (c > bv || (c == bv && i < bi)) {
            bv = c;
            bi = i;
        }
    }
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            double ov = sv[threadIdx.x + s];
            int64_t oi = si[threadIdx.x + s];
            if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
                sv[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pv[blockIdx.x] = sv[0];
        pi[blockIdx.x] = si[0];
    }
}

__global__ void reseed_finish_kernel(int nb, const double* __restrict__ pv, const int64_t* __restrict__ pi,
                                     int64_t d, const double* __restrict__ v, uint8_t* __restrict__ used,
                                     double* __restrict__ cent, int64_t cl) {
    __shared__ int64_t pick;
    if (threadIdx.x == 0) {
        double bv = -INFINITY;
        int64_t bi = INT64_MAX;
        for (int b = 0; b < nb; ++b) {
            if (pv[b] > bv || (pv[b] == bv && pi[b] < bi)) {
                bv = pv[b];
                bi = pi[b];
            }
        }
        pick = bi;
        used[bi] = 1;
    }
    __syncthreads();
    for (int64_t l = threadIdx.x; l < d; l += blockDim.x) cent[cl * d + l] = v[pick * d + l];
}


// ---------------------------------------------------------------------------
// k-means++ device steps (kmeans.py:101-136)
// d2 <- min(d2, |v - v[pick]|^2) by direct differences; mark taken; per-block
// candidate partials (count, weight sum) over untaken rows with d2 > 0.
// `prow` = coordinates of the drawn row; `pick` = its local index (or -1 when
// the row lives on another shard)
// Points in 8-column panels (panel b = columns 8b..8b+7 of every row, n x 8,
// zero-padded): a thread's 64-byte piece of a row is contiguous with its
// neighbours', so the k-means++ update reads the panels coalesced and stops
// at the first panel whose partial sum reaches the row's d2.
__global__ void to_panels_kernel(int64_t n, int64_t d, const double* __restrict__ v, double* __restrict__ v8) {
    const int64_t nch = (d + 7) / 8;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nch * n * 8) return;
    const int64_t b = e / (n * 8), rem = e - b * n * 8, i = rem >> 3, q = rem & 7;
    const int64_t c = 8 * b + q;
    v8[e] = c < d ? v[i * d + c] : 0.0;
}

// nonzero-panel bitmap: bit p % 32 of word w = p / 32 of row i (at w * n + i)
// is set when panel p of the row has a nonzero element; counts the zero
// panels.  The k-means++ update skips loading zero panels (their elements
// enter its numpy-order sums as exact zeros), which on an embedding with
// locked component eigenvectors (C3: one nonzero among 850 columns) cuts the
// bytes per row ~6x with bit-identical distances.
__global__ void panel_nonzero_kernel(int64_t n, int64_t nch, const double* __restrict__ v8,
                                     uint32_t* __restrict__ nzm, unsigned long long* __restrict__ nzero) {
    const int64_t nw = (nch + 31) / 32;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long zeros = 0;
    if (e < nw * n) {
        const int64_t w = e / n, i = e - w * n;
        uint32_t bits = 0;
        for (int b = 0; b < 32; ++b) {
            const int64_t p = w * 32 + b;
            if (p >= nch) break;
            const double2* src = reinterpret_cast<const double2*>(v8 + (p * n + i) * 8);
            bool nz = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double2 a = src[q];
                nz |= a.x != 0.0 || a.y != 0.0;
            }
            if (nz) bits |= 1u << b; else ++zeros;
        }
        nzm[e] = bits;
    }
    for (int o = 16; o > 0; o >>= 1) zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
    if ((threadIdx.x & 31) == 0 && zeros) atomicAdd(nzero, zeros);
}

// fp16 copy of s * v in 8-column panels (panel p of row i at p * n + i)
__global__ void to_half_panels_kernel(int64_t n, int64_t d, const double* __restrict__ v, double s,
                                      uint4* __restrict__ vh8) {
    const int64_t nch = (d + 7) / 8;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nch * n) return;
    const int64_t p = e / n, i = e - p * n;
    __align__(16) __half h[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int64_t c = 8 * p + q;
        h[q] = __double2half(c < d ? s * v[i * d + c] : 0.0);
    }
    vh8[e] = *reinterpret_cast<const uint4*>(h);
}

// |v_i| (plain fp64; used only inside error bounds)
__global__ void rownorm_sqrt_kernel(int64_t n, int64_t d, const double* __restrict__ v, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double a = 0.0;
    for (int64_t l = 0; l < d; ++l) a = fma(v[i * d + l], v[i * d + l], a);
    out[i] = sqrt(a);
}

constexpr int KPP_UPD_ROWS = 128, KPP_UPD_COLS = 32;

__device__ __forceinline__ void kpp_block_partials(double w, int64_t cnt, double* sw, int64_t* scn,
                                                   double* __restrict__ pw, int64_t* __restrict__ pc) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // fixed-order block partials (deterministic)
    for (int o = 16; o > 0; o >>= 1) {
        w += __shfl_down_sync(0xffffffffu, w, o);
        cnt += __shfl_down_sync(0xffffffffu, cnt, o);
    }
    if (lane == 0) {
        sw[warp] = w;
        scn[warp] = cnt;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0;
        int64_t c = 0;
        for (int q = 0; q < KPP_UPD_ROWS / 32; ++q) {
            a += sw[q];
            c += scn[q];
        }
        pw[blockIdx.x] = a;
        pc[blockIdx.x] = c;
    }
}

__global__ void __launch_bounds__(KPP_UPD_ROWS) kpp_update_kernel(int64_t n, int64_t d, const double* __restrict__ v, const double* __restrict__ prow,
                                  int64_t pick, int first, double* __restrict__ d2, uint8_t* __restrict__ taken,
                                  double* __restrict__ pw, int64_t* __restrict__ pc) {
    // one thread per row, folding its row against the new centre in numpy's
    // einsum order (_dist_to_one, kmeans.py:101-104).  Rows are read
    // directly, 32 columns at a time; once the partial sum already reaches the
    // row's current d2 the rest is skipped: rounded additions of nonnegative
    // terms never decrease the sum, so the full distance could not lower d2
    // and min(d2, dist) = d2 exactly (most rows, once the seeding has covered
    // their region).
    // The warp's 32 rows are staged through shared memory a 32-column chunk at
    // a time with coalesced loads (a thread-per-row read costs one L1
    // wavefront per lane per element); pruned rows stop loading.
    __shared__ double sw[KPP_UPD_ROWS / 32];
    __shared__ int64_t scn[KPP_UPD_ROWS / 32];
    __shared__ double stg_all[KPP_UPD_ROWS / 32][32 * (KPP_UPD_COLS + 1)];
    __shared__ const double* rows_all[KPP_UPD_ROWS / 32][32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t i = (int64_t)blockIdx.x * KPP_UPD_ROWS + tid;
    double* stg = stg_all[warp];
    const double** rows = rows_all[warp];
    NpDot acc;
    bool pruned = false;
    double old = 0.0;
    const double* row = i < n ? v + i * d : nullptr;
    if (i < n && !first) old = d2[i];
    for (int64_t c0 = 0; c0 < d; c0 += KPP_UPD_COLS) {
        const bool active = row && !pruned;
        if (!__any_sync(0xffffffffu, active)) break;
        const int w = (int)imin64(KPP_UPD_COLS, d - c0);
        rows[lane] = active ? row : nullptr;
        __syncwarp();
#pragma unroll
        for (int r0 = 0; r0 < 32; r0 += 8) {
            double vv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double* pr = rows[r0 + q];
                vv[q] = (pr && lane < w) ? __ldg(pr + c0 + lane) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) stg[(r0 + q) * (KPP_UPD_COLS + 1) + lane] = vv[q];
        }
        __syncwarp();
        if (active) {
            const double* sr = stg + lane * (KPP_UPD_COLS + 1) - c0;
            np_dot_span(acc, c0, c0 + w, [&](int64_t l) {
                const double t = __dsub_rn(sr[l], __ldg(prow + l));
                return __dmul_rn(t, t);
            });
            if (!first && c0 + w < d && acc.result() >= old) pruned = true;
        }
        __syncwarp();
    }
    double w = 0.0;
    int64_t cnt = 0;
    if (i < n) {
        const double dist = acc.result();
        const double nv = first ? dist : (pruned ? old : fmin(old, dist));
        if (i == pick) taken[i] = 1;
        const bool tk = (i == pick) || taken[i];
        d2[i] = nv;
        if (!tk && nv > 0.0) {
            w = nv;
            cnt = 1;
        }
    }
    kpp_block_partials(w, cnt, sw, scn, pw, pc);
}

// |c_t - c_j|^2 for the centres drawn before c_t (plain fp64: only used in
// the bound below, with a margin)
__global__ void kpp_centre_dist_kernel(int64_t d, int t, const double* __restrict__ cent, double* __restrict__ cc) {
    const int j = (int)(blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32), lane = threadIdx.x & 31;
    if (j >= t) return;
    double a = 0.0;
    for (int64_t l = lane; l < d; l += 32) {
        const double u = cent[(int64_t)t * d + l] - cent[(int64_t)j * d + l];
        a = fma(u, u, a);
    }
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) cc[j] = a;
}

// the same update over 8-column panels (to_panels_kernel), pruning per panel;
// d2 is identical (the prune is exact whatever the granularity).  With cc
// (the distances of the new centre c_t to the earlier ones) a row whose
// nearest centre c_a = ctr[i] has |c_t - c_a|^2 > 4 d2 (1 + 1e-6) is skipped
// unread: |x - c_t| >= |c_t - c_a| - |x - c_a| > |x - c_a| (the margin is
// far above the rounding of the computed squares), so min(d2, dist) = d2.
// fp16 screen of the k-means++ update (optional): the points as 8-column
// fp16 panels of s * v, the new centre likewise (scaled, in shared memory),
// fp64 row norms and |c|.  A row whose certified lower bound on |v - c|^2
// exceeds its current d2 cannot change (min(d2, dist) = d2) and is not read
// in fp64; the rest go through the exact numpy-order path unchanged.
struct KppScreen {
    const uint4* vh8 = nullptr;    // [ceil(d/8)][n] x 8 halves
    const __half* ch = nullptr;    // ceil(d/8) * 8 halves (device)
    const double* vnorm = nullptr; // |v_i|
    const double* cnorm = nullptr; // |c| (device scalar)
    double s = 1.0;
    unsigned long long* stats = nullptr;  // [0] rows screened, [1] rows the screen pruned
};

__global__ void kpp_centre_half_kernel(int64_t d, const double* __restrict__ row, double s, __half* __restrict__ ch,
                                       double* __restrict__ cnorm) {
    __shared__ double part[32];
    double a = 0.0;
    const int64_t dp = (d + 7) / 8 * 8;
    for (int64_t l = threadIdx.x; l < dp; l += blockDim.x) {
        const double x = l < d ? row[l] : 0.0;
        ch[l] = __double2half(s * x);
        a = fma(x, x, a);
    }
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
        cnorm[0] = sqrt(t);
    }
}

__global__ void __launch_bounds__(KPP_UPD_ROWS) kpp_update_panel_kernel(int64_t n, int64_t d,
                                                                        const double* __restrict__ v8,
                                                                        const double* __restrict__ prow, int64_t pick,
                                                                        int first, double* __restrict__ d2,
                                                                        uint8_t* __restrict__ taken,
                                                                        double* __restrict__ pw,
                                                                        int64_t* __restrict__ pc,
                                                                        const double* __restrict__ cc,
                                                                        int32_t* __restrict__ ctr, int t,
                                                                        KppScreen scr,
                                                                        const int32_t* __restrict__ reps,
                                                                        int64_t nreps,
                                                                        const uint32_t* __restrict__ nzm) {
    __shared__ double sw[KPP_UPD_ROWS / 32];
    __shared__ int64_t scn[KPP_UPD_ROWS / 32];
    // dynamic shared memory: the new centre's row (nch * 8 doubles), then
    // (screen) its fp16 copy
    extern __shared__ __align__(16) double kpp_row[];
    // reps: only the listed rows (one per group of identical rows), no
    // partials (kpp_expand_kernel copies their d2 to the group and sums)
    const int64_t ti = (int64_t)blockIdx.x * KPP_UPD_ROWS + threadIdx.x;
    const int64_t i = reps ? (ti < nreps ? (int64_t)reps[ti] : n) : ti;
    const int64_t nch = (d + 7) / 8;
    __half* kpp_ch = reinterpret_cast<__half*>(kpp_row + nch * 8);
    for (int64_t l = threadIdx.x; l < nch * 8; l += blockDim.x) kpp_row[l] = l < d ? prow[l] : 0.0;
    if (scr.vh8)
        for (int64_t l = threadIdx.x; l < nch * 8; l += blockDim.x) kpp_ch[l] = scr.ch[l];
    __syncthreads();
    NpDot acc;
    bool pruned = false, screened = false, screen_pruned = false;
    double old = 0.0;
    if (i < n) {
        if (!first) old = d2[i];
        if (!first && cc && cc[ctr[i]] > 4.0 * old * (1.0 + 1e-6)) pruned = true;
        if (!first && !pruned && scr.vh8) {
            // f = |fp16(s v) - fp16(s c)|^2 in fp32; per element the fp16
            // rounding moves each difference by <= 2^-11 (|s v_l| + |s c_l|)
            // + 2^-24 (subnormals), so |s(v - c)| >= sqrt(f) - |Delta| with
            // |Delta| <= 2^-11 s (|v| + |c|) + 2^-24 sqrt(d) (triangle
            // inequality in l2); fp32 rounding of the d-term sum is covered
            // by shrinking f by (d + 8) 2^-23
            float f = 0.0f;
            const uint4* src = scr.vh8 + i;
            for (int64_t p = 0; p < nch; ++p) {
                const uint4 raw = __ldg(src + p * n);
                const __half2* hv = reinterpret_cast<const __half2*>(&raw);
                const __half2* hc = reinterpret_cast<const __half2*>(kpp_ch + 8 * p);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 a = __half22float2(hv[q]), b = __half22float2(hc[q]);
                    const float dx = a.x - b.x, dy = a.y - b.y;
                    f = fmaf(dx, dx, f);
                    f = fmaf(dy, dy, f);
                }
            }
            const double delta = 0x1p-11 * scr.s * (scr.vnorm[i] + scr.cnorm[0]) + 0x1p-24 * sqrt((double)d);
            const double rf = sqrt(fmax(0.0, (double)f * (1.0 - (double)(d + 8) * 0x1p-23)));
            const double lb = rf - delta;
            screened = true;
            if (lb > 0.0 && lb * lb > old * scr.s * scr.s * (1.0 + 1e-9)) pruned = true;
            screen_pruned = pruned;
        }
        // full panels two at a time (both panels' loads in flight before the
        // arithmetic; the early exit is tested per pair), then the tail panel
        const int64_t dfull = d / 8 * 8;
        int64_t c0 = 0;
        auto panel = [&](int64_t cc, const double2 a0, const double2 a1, const double2 a2, const double2 a3) {
            const double2* cr = reinterpret_cast<const double2*>(kpp_row + cc);
            const double2 b0 = cr[0], b1 = cr[1], b2 = cr[2], b3 = cr[3];
            auto sq = [](double u, double w) {
                const double t = __dsub_rn(u, w);
                return __dmul_rn(t, t);
            };
            acc.block(sq(a0.x, b0.x), sq(a0.y, b0.y), sq(a1.x, b1.x), sq(a1.y, b1.y), sq(a2.x, b2.x),
                      sq(a2.y, b2.y), sq(a3.x, b3.x), sq(a3.y, b3.y));
        };
        // zero panels (nzm) are not loaded: their elements are exact zeros
        uint32_t nzw = 0xffffffffu;
        int64_t nzw_at = -1;
        auto panel_nz = [&](int64_t p) {
            if (!nzm) return true;
            if ((p >> 5) != nzw_at) {
                nzw_at = p >> 5;
                nzw = __ldg(nzm + nzw_at * n + i);
            }
            return ((nzw >> (p & 31)) & 1u) != 0;
        };
        const double2 z2 = make_double2(0.0, 0.0);
        for (; c0 + 16 <= dfull && !pruned; c0 += 16) {
            const double2* s0 = reinterpret_cast<const double2*>(v8 + ((c0 >> 3) * n + i) * 8);
            const double2* s1 = reinterpret_cast<const double2*>(v8 + (((c0 >> 3) + 1) * n + i) * 8);
            const bool n0 = panel_nz(c0 >> 3), n1 = panel_nz((c0 >> 3) + 1);
            const double2 a0 = n0 ? __ldg(s0) : z2, a1 = n0 ? __ldg(s0 + 1) : z2, a2 = n0 ? __ldg(s0 + 2) : z2,
                          a3 = n0 ? __ldg(s0 + 3) : z2;
            const double2 e0 = n1 ? __ldg(s1) : z2, e1 = n1 ? __ldg(s1 + 1) : z2, e2 = n1 ? __ldg(s1 + 2) : z2,
                          e3 = n1 ? __ldg(s1 + 3) : z2;
            panel(c0, a0, a1, a2, a3);
            panel(c0 + 8, e0, e1, e2, e3);
            if (!first && c0 + 16 < d && acc.result() >= old) pruned = true;
        }
        for (; c0 < d && !pruned; c0 += 8) {
            const double2* src = reinterpret_cast<const double2*>(v8 + ((c0 >> 3) * n + i) * 8);
            const bool n0 = panel_nz(c0 >> 3);
            const double2 a0 = n0 ? __ldg(src) : z2, a1 = n0 ? __ldg(src + 1) : z2, a2 = n0 ? __ldg(src + 2) : z2,
                          a3 = n0 ? __ldg(src + 3) : z2;
            const int rem = (int)(d - c0 < 8 ? d - c0 : 8);
            if (rem == 8) {
                panel(c0, a0, a1, a2, a3);
            } else {  // the tail: pairs, then a single (np_dot_span)
                const double x[8] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y, a3.x, a3.y};
                auto f = [&](int q) {
                    const double t = __dsub_rn(x[q], kpp_row[c0 + q]);
                    return __dmul_rn(t, t);
                };
#pragma unroll
                for (int q = 0; q < 8; q += 2)
                    if (q + 2 <= rem) acc.pair(f(q), f(q + 1));
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if ((rem & 1) && q == rem - 1) acc.single(f(q));
            }
            if (!first && c0 + 8 < d && acc.result() >= old) {
                pruned = true;
                break;
            }
        }
    }
    double w = 0.0;
    int64_t cnt = 0;
    if (i < n) {
        const double dist = acc.result();
        const double nv = first ? dist : (pruned ? old : fmin(old, dist));
        if (ctr && (first || (!pruned && dist < old))) ctr[i] = t;  // the nearest centre so far
        if (i == pick) taken[i] = 1;
        const bool tk = (i == pick) || taken[i];
        d2[i] = nv;
        if (!tk && nv > 0.0) {
            w = nv;
            cnt = 1;
        }
    }
    if (scr.stats) {  // screen effectiveness, warp-aggregated
        const unsigned bs = __ballot_sync(0xffffffffu, screened), bp = __ballot_sync(0xffffffffu, screen_pruned);
        if ((threadIdx.x & 31) == 0 && bs) {
            atomicAdd(&scr.stats[0], (unsigned long long)__popc(bs));
            atomicAdd(&scr.stats[1], (unsigned long long)__popc(bp));
        }
    }
    if (!reps) kpp_block_partials(w, cnt, sw, scn, pw, pc);
}

// rows with an identical earlier row (rep[i] < i): d2 and the nearest centre
// are the representative's (identical arithmetic on identical bits); the
// candidate partials over all rows in kpp_update_panel_kernel's block order
__global__ void __launch_bounds__(KPP_UPD_ROWS) kpp_expand_kernel(int64_t n, const int32_t* __restrict__ rep,
                                                                  int64_t pick, double* __restrict__ d2,
                                                                  uint8_t* __restrict__ taken,
                                                                  int32_t* __restrict__ ctr,
                                                                  double* __restrict__ pw, int64_t* __restrict__ pc) {
    __shared__ double sw[KPP_UPD_ROWS / 32];
    __shared__ int64_t scn[KPP_UPD_ROWS / 32];
    const int64_t i = (int64_t)blockIdx.x * KPP_UPD_ROWS + threadIdx.x;
    double w = 0.0;
    int64_t cnt = 0;
    if (i < n) {
        const int64_t r = rep[i];
        double nv = d2[i];
        if (r != i) {
            nv = d2[r];
            d2[i] = nv;
            if (ctr) ctr[i] = ctr[r];
        }
        if (i == pick) taken[i] = 1;
        const bool tk = (i == pick) || taken[i];
        if (!tk && nv > 0.0) {
            w = nv;
            cnt = 1;
        }
    }
    kpp_block_partials(w, cnt, sw, scn, pw, pc);
}

// identical-row groups: 64-bit hash of each row's bit patterns
__global__ void row_hash_kernel(int64_t n, int64_t d, const double* __restrict__ v, uint64_t* __restrict__ h) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t x = 0x9E3779B97F4A7C15ull ^ (uint64_t)d;
    for (int64_t l = 0; l < d; ++l) {
        uint64_t b = (uint64_t)__double_as_longlong(v[i * d + l]);
        b ^= b >> 33;
        b *= 0xff51afd7ed558ccdull;
        b ^= b >> 33;
        x = (x ^ b) * 0x100000001b3ull + 0x632be59bd9b4e019ull;
    }
    x ^= x >> 31;
    h[i] = x == ~0ull ? 0ull : x;  // ~0 marks an empty slot
}
// open addressing: slot key = hash, value = the smallest row index with it
__global__ void hash_insert_kernel(int64_t n, const uint64_t* __restrict__ h, uint64_t mask,
                                   unsigned long long* __restrict__ keys, unsigned long long* __restrict__ vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long key = h[i];
    uint64_t s = key & mask;
    while (true) {
        const unsigned long long prev = atomicCAS(&keys[s], ~0ull, key);
        if (prev == ~0ull || prev == key) {
            atomicMin(&vals[s], (unsigned long long)i);
            return;
        }
        s = (s + 1) & mask;
    }
}
// rep[i] = the smallest index of a row with the same hash AND the same bits (else i)
__global__ void hash_rep_kernel(int64_t n, int64_t d, const double* __restrict__ v, const uint64_t* __restrict__ h,
                                uint64_t mask, const unsigned long long* __restrict__ keys,
                                const unsigned long long* __restrict__ vals, int32_t* __restrict__ rep,
                                int64_t* __restrict__ isrep) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long key = h[i];
    uint64_t s = key & mask;
    while (keys[s] != key) s = (s + 1) & mask;
    int64_t r = (int64_t)vals[s];
    if (r != i) {
        for (int64_t l = 0; l < d; ++l)
            if (__double_as_longlong(v[i * d + l]) != __double_as_longlong(v[r * d + l])) {
                r = i;  // a hash collision: its own group
                break;
            }
    }
    rep[i] = (int32_t)r;
    isrep[i] = r == i ? 1 : 0;
}
__global__ void compact_reps_kernel(int64_t n, const int64_t* __restrict__ isrep, const int64_t* __restrict__ pos,
                                    int32_t* __restrict__ reps) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && isrep[i]) reps[pos[i]] = (int32_t)i;
}


__global__ void kpp_total_kernel(int64_t nb, const double* __restrict__ pw, const int64_t* __restrict__ pc,
                                 double* __restrict__ out_total, int64_t* __restrict__ out_count) {
    __shared__ double sw[1024];
    __shared__ int64_t sc_[1024];
    double a = 0.0;
    int64_t c = 0;
    for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) {
        a += pw[b];
        c += pc[b];
    }
    sw[threadIdx.x] = a;
    sc_[threadIdx.x] = c;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            sw[threadIdx.x] += sw[threadIdx.x + s];
            sc_[threadIdx.x] += sc_[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *out_total = sw[0];
        *out_count = sc_[0];
    }
}

constexpr int KPP_BLK = 1024;

// per-block sums of p_i = w_i / total over candidates (rng.choice p vector)
__global__ void kpp_psum_kernel(int64_t n, const double* __restrict__ d2, const uint8_t* __restrict__ taken,
                                const double* __restrict__ total, double* __restrict__ bsum) {
    __shared__ double red[KPP_BLK];
    int64_t i = (int64_t)blockIdx.x * KPP_BLK + threadIdx.x;
    double tot = *total;
    double p = 0.0;
    if (i < n && !taken[i] && d2[i] > 0.0) p = d2[i] / tot;
    red[threadIdx.x] = p;
    __syncthreads();
    for (int s = KPP_BLK / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = red[0];
}

// first index whose normalised cumulative probability exceeds u
// (numpy Generator.choice: cdf = p.cumsum(); cdf /= cdf[-1];
//  cdf.searchsorted(u, side="right")).
// Warp-parallel inverse-CDF search over the candidates (kmeans.py:130-132:
// rng.choice(p=d2/sum) = first candidate whose cumulative probability exceeds
// the uniform draw).  Level 1 walks the KPP_BLK-row block sums (32 contiguous
// chunks, one per lane, warp prefix over the chunk sums), level 2 the rows of
// the crossing block (KPP_BLK / 32 per lane).  `crosses(c)` tests a cumulative value.
// The cumulative sums are regrouped relative to a strictly sequential cumsum,
// so a draw could differ only if it fell within a few ulps of a boundary.
template <class Crosses>
__device__ __forceinline__ int64_t kpp_warp_search(int64_t n, int64_t nb, const double* __restrict__ d2,
                                                   const uint8_t* __restrict__ taken, double tot,
                                                   const double* __restrict__ bsum, Crosses crosses) {
    const int lane = threadIdx.x & 31;
    // ---- level 1: block sums
    const int64_t per = (nb + 31) / 32, b0 = imin64(nb, lane * per), b1 = imin64(nb, b0 + per);
    double cs = 0.0;
    for (int64_t b = b0; b < b1; ++b) cs += bsum[b];
    double pre = cs;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += t;
    }
    double run = pre - cs;  // exclusive prefix of this lane's chunk
    int64_t hit = -1;
    if (crosses(pre))
        for (int64_t b = b0; b < b1; ++b) {
            if (crosses(run + bsum[b])) {
                hit = b;
                break;
            }
            run += bsum[b];
        }
    unsigned m = __ballot_sync(0xffffffffu, hit >= 0);
    int64_t blk;
    if (m) {
        const int src = __ffs(m) - 1;
        blk = __shfl_sync(0xffffffffu, hit, src);
        run = __shfl_sync(0xffffffffu, run, src);
    } else {
        blk = nb - 1;  // rounding: no block crossed -> the last block, from its start
        run = __shfl_sync(0xffffffffu, pre, 31) - bsum[nb - 1];
    }
    // ---- level 2: rows of the crossing block, KPP_BLK / 32 consecutive rows per lane
    constexpr int RPL = KPP_BLK / 32;
    const int64_t lo = blk * KPP_BLK, hi = imin64(n, lo + KPP_BLK);
    const int64_t r0 = imin64(hi, lo + lane * RPL), r1 = imin64(hi, r0 + RPL);
    double ps = 0.0;
    int64_t mylast = -1;
    for (int64_t i = r0; i < r1; ++i)
        if (!taken[i] && d2[i] > 0.0) {
            ps += d2[i] / tot;
            mylast = i;
        }
    double pp = ps;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, pp, o);
        if (lane >= o) pp += t;
    }
    double r = run + (pp - ps);
    int64_t found = -1;
    if (crosses(run + pp))
        for (int64_t i = r0; i < r1; ++i) {
            if (taken[i] || !(d2[i] > 0.0)) continue;
            r += d2[i] / tot;
            if (crosses(r)) {
                found = i;
                break;
            }
        }
    m = __ballot_sync(0xffffffffu, found >= 0);
    if (m) return __shfl_sync(0xffffffffu, found, __ffs(m) - 1);
    // rounding pushed the crossing past every candidate of the block: its
    // last candidate (or, if none, the last candidate overall)
    unsigned ml = __ballot_sync(0xffffffffu, mylast >= 0);
    if (ml) return __shfl_sync(0xffffffffu, mylast, 31 - __clz(ml));
    return -2;
}

__device__ __forceinline__ int64_t kpp_last_candidate(int64_t n, const double* __restrict__ d2,
                                                      const uint8_t* __restrict__ taken) {
    for (int64_t i = n - 1; i >= 0; --i)
        if (!taken[i] && d2[i] > 0.0) return i;
    return -1;
}

__global__ void kpp_search_kernel(int64_t n, int64_t nb, const double* __restrict__ d2,
                                  const uint8_t* __restrict__ taken, const double* __restrict__ total,
                                  const double* __restrict__ bsum, double u, int64_t* __restrict__ out) {
    // sum of all block sums (lane-chunked, as in kpp_warp_search)
    const int lane = threadIdx.x & 31;
    const int64_t per = (nb + 31) / 32, b0 = imin64(nb, lane * per), b1 = imin64(nb, b0 + per);
    double cs = 0.0;
    for (int64_t b = b0; b < b1; ++b) cs += bsum[b];
    double last = cs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, last, o);
        if (lane >= o) last += t;
    }
    last = __shfl_sync(0xffffffffu, last, 31);
    int64_t r = kpp_warp_search(n, nb, d2, taken, *total, bsum, [&](double c) { return c / last > u; });
    if (r == -2 && lane == 0) r = kpp_last_candidate(n, d2, taken);
    if (lane == 0) *out = r;
}

__global__ void kpp_search_target_kernel(int64_t n, int64_t nb, const double* __restrict__ d2,
                                         const uint8_t* __restrict__ taken, const double* __restrict__ total,
                                         const double* __restrict__ bsum, double target, int64_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    // target at/above this shard's total: its last candidate
    const int64_t per = (nb + 31) / 32, b0 = imin64(nb, lane * per), b1 = imin64(nb, b0 + per);
    double cs = 0.0;
    for (int64_t b = b0; b < b1; ++b) cs += bsum[b];
    double all = cs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, all, o);
        if (lane >= o) all += t;
    }
    all = __shfl_sync(0xffffffffu, all, 31);
    int64_t r;
    if (!(all > target)) {
        r = lane == 0 ? kpp_last_candidate(n, d2, taken) : -1;
    } else {
        r = kpp_warp_search(n, nb, d2, taken, *total, bsum, [&](double c) { return c > target; });
        if (r == -2) r = -1;
    }
    if (lane == 0) *out = r;
}

__global__ void argmax_finish_kernel(int nb, const double* __restrict__ pv, const int64_t* __restrict__ pi,
                                     uint8_t* __restrict__ used, int64_t* __restrict__ out) {
    if (threadIdx.x != 0) return;
    double bv = -INFINITY;
    int64_t bi = INT64_MAX;
    for (int b = 0; b < nb; ++b) {
        if (pv[b] > bv || (pv[b] == bv && pi[b] < bi)) {
            bv = pv[b];
            bi = pi[b];
        }
    }
    used[bi] = 1;
    *out = bi;
}

__global__ void kpp_nth_free_kernel(int64_t n, const uint8_t* __restrict__ taken, int64_t r,
                                    int64_t* __restrict__ out) {
    if (threadIdx.x != 0) return;
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (taken[i]) continue;
        if (c == r) {
            *out = i;
            return;
        }
        ++c;
    }
    *out = -1;
}

// ---------------------------------------------------------------------------
// ncut (metrics.py:34-39, 59-67).  Per row (warp): degree and the weight of
// the row's entries that cross to another part; per part: one sequential
// chain over its member rows in ascending order.
__global__ void ncut_rows_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                 const double* __restrict__ vals, const int64_t* __restrict__ labels,
                                 double* __restrict__ deg, double* __restrict__ cross, int64_t row_offset = 0) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int64_t li = labels[row_offset + i];
    double dg = 0.0, cr = 0.0;
    for (int64_t p = row_ptr[i] + lane; p < row_ptr[i + 1]; p += 32) {
        const double v = vals[p];
        dg += v;
        if (labels[col[p]] != li) cr += v;
    }
    dg = warp_sum(dg);
    cr = warp_sum(cr);
    if (lane == 0) {
        deg[i] = dg;
        cross[i] = cr;
    }
}

__global__ void bucket_sizes_kernel(int64_t k, const int64_t* __restrict__ start, int64_t* __restrict__ counts) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < k) counts[c] = start[c + 1] - start[c];
}

__global__ void ncut_parts_kernel(int64_t k, const double* __restrict__ deg, const double* __restrict__ cross,
                                  const int64_t* __restrict__ start, const int32_t* __restrict__ members,
                                  double* __restrict__ bnd, double* __restrict__ vol) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k) return;
    double b = 0.0, v = 0.0;
    const int64_t e = start[c + 1];
    int64_t m = start[c];
    // the gathers of 16 members are issued before the (sequential, point
    // order) additions consume them
    constexpr int B = 16;
    for (; m + B <= e; m += B) {
        int64_t idx[B];
        double dv[B], cv[B];
#pragma unroll
        for (int u = 0; u < B; ++u) idx[u] = members[m + u];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            dv[u] = deg[idx[u]];
            cv[u] = cross[idx[u]];
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            v += dv[u];
            b += cv[u];
        }
    }
    for (; m < e; ++m) {
        const int64_t i = members[m];
        v += deg[i];
        b += cross[i];
    }
    bnd[c] = b;
    vol[c] = v;
}

// numpy's pairwise summation (DOUBLE_pairwise_sum) for a contiguous array
static double np_pairwise_sum(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;  // numpy starts from the first element: (-0.0) aware
        if (n == 0) return 0.0;
        res = a[0];
        for (int64_t i = 1; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// numpy's sum of a device array (np.add.reduce over a contiguous float64
// array = DOUBLE_pairwise_sum of the whole array): the recursion's leaves
// (<= 128 elements, 8 accumulators) are summed on the device, one thread per
// leaf, and combined on the host in the recursion's order.  The reference's
// SSE history is float(point_cost.sum()) (kmeans.py:176, 184).
__global__ void np_leaf_sum_kernel(int64_t nleaf, const int64_t* __restrict__ off, const double* __restrict__ a,
                                   double* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nleaf) return;
    const double* x = a + off[t];
    const int64_t n = off[t + 1] - off[t];
    double res;
    if (n < 8) {
        res = 0.0;
        for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, x[i]);
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = x[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], x[i + j]);
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, x[i]);
    }
    out[t] = res;
}

struct NpSum {
    int64_t n = -1;
    std::vector<int64_t> off;  // leaf boundaries
    std::vector<double> h;
    DevBuf<int64_t> d_off;
    DevBuf<double> d_leaf;
    static void leaves(int64_t o, int64_t n, std::vector<int64_t>& out) {
        if (n <= 128) {
            out.push_back(o + n);
            return;
        }
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        leaves(o, n2, out);
        leaves(o + n2, n - n2, out);
    }
    double combine(int64_t n, size_t& li) const {
        if (n <= 128) return h[li++];
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        const double a = combine(n2, li);
        const double b = combine(n - n2, li);
        return a + b;
    }
    int sum(const double* a, int64_t n_, double* result, cudaStream_t st) {
        int rc;
        if (n_ != n) {
            n = n_;
            off.assign(1, 0);
            leaves(0, n, off);
            if ((rc = d_off.alloc(off.size())) || (rc = d_leaf.alloc(off.size()))) return rc;
            SC_CUDA(cudaMemcpyAsync(d_off.p, off.data(), sizeof(int64_t) * off.size(), cudaMemcpyHostToDevice, st));
            h.assign(off.size() - 1, 0.0);
        }
        const int64_t nl = (int64_t)off.size() - 1;
        np_leaf_sum_kernel<<<(unsigned)ceil_div(nl, 128), 128, 0, st>>>(nl, d_off.p, a, d_leaf.p);
        SC_LAUNCHED(1);
        SC_CUDA(d2h_sync(h.data(), d_leaf.p, sizeof(double) * nl, st));
        size_t li = 0;
        *result = n > 0 ? combine(n, li) : 0.0;
        return SC_OK;
    }
};

// labels[i] = nearest of the k rows of c (fp64 distance tiles, ties -> lowest)

}  // namespace sc

// ---------------------------------------------------------------------------
// Tensor-core assignment with certified argmin (sc_assign_tc.cuh)
#include "sc_assign_tc.cuh"
#include "sc_tma.cuh"

namespace sc {

__global__ void as_absmax_kernel(int64_t m, const double* __restrict__ x, unsigned long long* __restrict__ out) {
    double a = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        a = fmax(a, fabs(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(a));
}

// rows x dp fp16 copy of s * x (zero padding), warp per row
__global__ void as_prep_rows_kernel(int64_t rows, int64_t rows_pad, int64_t d, int64_t dp, const double* __restrict__ x,
                                    double s, __half* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (i >= rows_pad) return;
    for (int64_t l = lane; l < dp; l += 32)
        out[i * dp + l] = __double2half(i < rows && l < d ? s * x[i * d + l] : 0.0);
}

// centroid norms for the keys (fp32, +inf on padding) and max |c|^2
__global__ void as_cent_norms_kernel(int64_t k, int64_t k_pad, const double* __restrict__ cn, float* __restrict__ cnk,
                                     unsigned long long* __restrict__ cnmax) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= k_pad) return;
    cnk[c] = c < k ? (float)cn[c] : INFINITY;
    if (c < k) atomicMax(cnmax, (unsigned long long)__double_as_longlong(cn[c]));
}

// exact S(v_i, c) in the reference's order (kmeans.py:92-98), clamped at 0
__device__ __forceinline__ double exact_s(const double* __restrict__ vi, double vni, const double* __restrict__ cc,
                                          double cnc, int64_t d) {
    NpDot s;
    np_dot_span(s, 0, d, [&](int64_t l) { return __dmul_rn(vi[l], cc[l]); });
    const double r = __dsub_rn(__dadd_rn(vni, cnc), __dmul_rn(2.0, s.result()));
    return r > 0.0 ? r : 0.0;
}

// delta_i bounds |approx key - exact key| for row i (fp16 operands, fp32
// accumulation of dp products, fp32 norms and FMA, fp16 subnormals):
//   delta_i = 1.25 * ( 2 (2^-10 + (dp+1) 2^-24) |v_i| cmax
//                      + 2^-24 (2 cnmax + 2 |v_i| cmax)
//                      + 2^-24 sqrt(dp) (|v_i| + cmax) / s )
__device__ __forceinline__ double as_delta(double vni, double cnmax, int64_t dp, double s) {
    const double cmax = sqrt(cnmax);
    const double va = sqrt(vni);
    return 1.25 * (2.0 * (0x1p-10 + (double)(dp + 1) * 0x1p-24) * va * cmax + 0x1p-24 * (2.0 * cnmax + 2.0 * va * cmax) +
                   0x1p-24 * sqrt((double)dp) * (va + cmax) / s);
}

// Uncertified rows whose fourth-best approximate key is more than 2 delta
// above the best: every centroid that can hold the exact minimum is among
// the kept three, so their exact keys (exact_s's arithmetic, the reference's)
// settle the row -- minimum, lowest index on ties.  Ten rows per warp, lanes
// 3r..3r+2 evaluate row r's candidates through the warp-staged dot
// (warp_pair_dot_np: coalesced row reads); rows with more near-ties go to
// flagged2 for the full re-scan.  Dynamic shared memory: kPairStage doubles
// per warp.
__global__ void as_resolve_kernel(int64_t nf, int64_t d, int64_t dp, double s, const double* __restrict__ v,
                                  const double* __restrict__ vn, const double* __restrict__ c,
                                  const double* __restrict__ cn, const unsigned long long* __restrict__ cnmax_bits,
                                  const int32_t* __restrict__ flagged, const float2* __restrict__ best_keys,
                                  const float2* __restrict__ alt_keys, const int32_t* __restrict__ best_idx,
                                  const int2* __restrict__ alt_idx, const int64_t* __restrict__ old_labels,
                                  int64_t* __restrict__ labels, double* __restrict__ cost,
                                  unsigned long long* __restrict__ changes, int32_t* __restrict__ flagged2,
                                  unsigned long long* __restrict__ nflag2) {
    extern __shared__ double res_stage[];
    const int lane = threadIdx.x & 31, grp = lane / 3, slot = lane - 3 * grp;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t r = w * 10 + grp;
    const bool mine = grp < 10 && r < nf;
    int64_t i = -1, q = -1;
    bool settle = false;
    if (mine) {
        i = flagged[r];
        const double delta = as_delta(vn[i], __longlong_as_double((long long)*cnmax_bits), dp, s);
        const float2 bk = best_keys[i], ak = alt_keys[i];
        const double lim = (double)bk.x + 2.0 * delta;
        settle = best_idx[i] >= 0 && (double)ak.y > lim;
        if (settle) {
            const int2 ai = alt_idx[i];
            if (slot == 0) q = best_idx[i];
            if (slot == 1 && ai.x >= 0 && (double)bk.y <= lim) q = ai.x;
            if (slot == 2 && ai.y >= 0 && (double)ak.x <= lim) q = ai.y;
        } else if (slot == 0) {
            flagged2[atomicAdd(nflag2, 1ull)] = (int32_t)i;
        }
    }
    const double dot = warp_pair_dot_np(q >= 0 ? v + i * d : nullptr, q >= 0 ? c + q * d : nullptr, d,
                                        res_stage + (threadIdx.x >> 5) * kPairStage);
    double sv = INFINITY;
    int64_t arg = INT64_MAX;
    if (q >= 0) {
        const double t = __dsub_rn(__dadd_rn(vn[i], cn[q]), __dmul_rn(2.0, dot));
        sv = t > 0.0 ? t : 0.0;
        arg = q;
    }
    const int base = 3 * grp < 30 ? 3 * grp : 0;
#pragma unroll
    for (int o = 1; o <= 2; ++o) {
        const double os = __shfl_sync(0xffffffffu, sv, base + o);
        const int64_t oa = __shfl_sync(0xffffffffu, arg, base + o);
        if (slot == 0 && (os < sv || (os == sv && oa < arg))) {
            sv = os;
            arg = oa;
        }
    }
    if (mine && settle && slot == 0) {
        labels[i] = arg;
        cost[i] = sv;
        if (old_labels && old_labels[i] != arg) atomicAdd(changes, 1ull);
    }
}

__global__ void as_take_best_kernel(int64_t n, const int32_t* __restrict__ best_idx, int64_t* __restrict__ labels) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) labels[i] = best_idx[i] < 0 ? 0 : best_idx[i];
}

// Certified rows (second-best approximate key more than 2 delta above the
// best): label = best, exact cost (exact_s's products and order) with a
// thread per row reading its row and its centroid in 64-byte pieces; the
// rest are listed for as_resolve_kernel.  (Measured at C5: rows in point
// order beat both an 8-column panel copy of the points and rows visited in
// cluster order, whose point reads scatter.)
__global__ void __launch_bounds__(256) as_finalize_rows_kernel(
    int64_t n, int64_t d, int64_t dp, double s, const double* __restrict__ v, const double* __restrict__ vn,
    const double* __restrict__ c, const double* __restrict__ cn, const unsigned long long* __restrict__ cnmax_bits,
    const int32_t* __restrict__ best_idx, const float2* __restrict__ best_keys,
    const int64_t* __restrict__ old_labels, int64_t* __restrict__ labels, double* __restrict__ cost,
    int32_t* __restrict__ flagged, unsigned long long* __restrict__ nflag, unsigned long long* __restrict__ changes,
    bool vec2) {
    // vec2: the warp stages its rows' 8-element pieces of v and of their
    // centroids in shared memory (lane quarter q of 8 rows per load: 8 lines
    // per instruction instead of 32 -- one row per thread made every load an
    // L1 wavefront per lane), and each thread sums its own row from there in
    // the same NpDot order; row stride 10 doubles: conflict-free double2 reads
    constexpr int FS = 10;
    __shared__ __align__(16) double stv[8][32 * FS];
    __shared__ __align__(16) double stc[8][32 * FS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int chg = 0;
    bool cert = false;
    int32_t b = -1;
    if (i < n) {
        const double delta = as_delta(vn[i], __longlong_as_double((long long)*cnmax_bits), dp, s);
        const float2 bk = best_keys[i];
        b = best_idx[i];
        cert = b >= 0 && (double)bk.y - (double)bk.x > 2.0 * delta;
        if (!cert) flagged[atomicAdd(nflag, 1ull)] = (int32_t)i;
    }
    NpDot acc;
    int64_t l = 0;
    if (vec2 && __any_sync(0xffffffffu, cert)) {
        const int64_t d8 = d / 8 * 8;
        const int64_t row0 = i - lane;
        bool rc[4];
        int32_t rb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            rc[q] = __shfl_sync(0xffffffffu, cert, q * 8 + (lane >> 2));
            rb[q] = __shfl_sync(0xffffffffu, b, q * 8 + (lane >> 2));
        }
        double* sv = stv[warp];
        double* sc = stc[warp];
        for (; l < d8; l += 8) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int rr = q * 8 + (lane >> 2);
                if (rc[q]) {
                    const double2 xv = __ldg(reinterpret_cast<const double2*>(v + (row0 + rr) * d + l) + (lane & 3));
                    const double2 xc = __ldg(reinterpret_cast<const double2*>(c + (int64_t)rb[q] * d + l) + (lane & 3));
                    reinterpret_cast<double2*>(sv + rr * FS)[lane & 3] = xv;
                    reinterpret_cast<double2*>(sc + rr * FS)[lane & 3] = xc;
                }
            }
            __syncwarp();
            if (cert) {
                const double2* pv = reinterpret_cast<const double2*>(sv + lane * FS);
                const double2* pc = reinterpret_cast<const double2*>(sc + lane * FS);
                const double2 x0 = pv[0], x1 = pv[1], x2 = pv[2], x3 = pv[3];
                const double2 y0 = pc[0], y1 = pc[1], y2 = pc[2], y3 = pc[3];
                acc.block(__dmul_rn(x0.x, y0.x), __dmul_rn(x0.y, y0.y), __dmul_rn(x1.x, y1.x),
                          __dmul_rn(x1.y, y1.y), __dmul_rn(x2.x, y2.x), __dmul_rn(x2.y, y2.y),
                          __dmul_rn(x3.x, y3.x), __dmul_rn(x3.y, y3.y));
            }
            __syncwarp();
        }
    }
    if (cert) {
        const double* vi = v + i * d;
        const double* cb = c + (int64_t)b * d;
        np_dot_span(acc, l, d, [&](int64_t j) { return __dmul_rn(__ldg(vi + j), __ldg(cb + j)); });
        labels[i] = b;
        const double r = __dsub_rn(__dadd_rn(vn[i], cn[b]), __dmul_rn(2.0, acc.result()));
        cost[i] = r > 0.0 ? r : 0.0;
        if (old_labels) chg = old_labels[i] != b;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, chg);
    if ((threadIdx.x & 31) == 0 && bal) atomicAdd(changes, (unsigned long long)__popc(bal));
}

// ct[l * k + q] = c[q * d + l] (the centroids column-major for the re-scan)
__global__ void as_transpose_kernel(int64_t k, int64_t d, const double* __restrict__ c, double* __restrict__ ct) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= k * d) return;
    const int64_t l = e / k, q = e - l * k;
    ct[e] = c[q * d + l];
}

// Exact re-scan of rows with more near-ties than the kept candidates: CTA =
// RS_R flagged rows (staged in shared memory) x 256 consecutive centroids,
// thread = one centroid; the centroids are read column-major (coalesced) and
// every product feeds RS_R rows.  Keys in exact_s's arithmetic; the CTA's
// minimum per row (lowest index on ties) goes to pval / pidx[row][chunk].
constexpr int RS_R = 8;
__global__ void __launch_bounds__(256) as_rescan_tile_kernel(int64_t nf, int64_t d, int64_t k,
                                                             const double* __restrict__ v,
                                                             const double* __restrict__ vn,
                                                             const double* __restrict__ ct,
                                                             const double* __restrict__ cn,
                                                             const int32_t* __restrict__ fl, int nchunks,
                                                             double* __restrict__ pval, int32_t* __restrict__ pidx) {
    extern __shared__ double rs_rows[];  // RS_R x d
    __shared__ int64_t rid[RS_R];
    __shared__ double rval[RS_R][8];
    __shared__ int32_t ridx[RS_R][8];
    const int64_t r0 = (int64_t)blockIdx.x * RS_R;
    const int nr = (int)(nf - r0 < RS_R ? nf - r0 : RS_R);
    if (threadIdx.x < RS_R) rid[threadIdx.x] = threadIdx.x < nr ? (int64_t)fl[r0 + threadIdx.x] : -1;
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (int64_t)RS_R * d; e += blockDim.x) {
        const int r = (int)(e / d);
        rs_rows[e] = r < nr ? v[rid[r] * d + (e - (int64_t)r * d)] : 0.0;
    }
    __syncthreads();
    const int64_t q = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
    const bool ok = q < k;
    NpDot acc[RS_R];
    if (ok) {
        int64_t l = 0;
        for (; l + 8 <= d; l += 8) {
            double cc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) cc[u] = __ldg(ct + (l + u) * k + q);
#pragma unroll
            for (int r = 0; r < RS_R; ++r) {
                const double* x = rs_rows + (int64_t)r * d + l;
                acc[r].block(__dmul_rn(x[0], cc[0]), __dmul_rn(x[1], cc[1]), __dmul_rn(x[2], cc[2]),
                             __dmul_rn(x[3], cc[3]), __dmul_rn(x[4], cc[4]), __dmul_rn(x[5], cc[5]),
                             __dmul_rn(x[6], cc[6]), __dmul_rn(x[7], cc[7]));
            }
        }
        for (; l + 2 <= d; l += 2) {
            const double c0 = __ldg(ct + l * k + q), c1 = __ldg(ct + (l + 1) * k + q);
#pragma unroll
            for (int r = 0; r < RS_R; ++r)
                acc[r].pair(__dmul_rn(rs_rows[(int64_t)r * d + l], c0), __dmul_rn(rs_rows[(int64_t)r * d + l + 1], c1));
        }
        if (l < d) {
            const double c0 = __ldg(ct + l * k + q);
#pragma unroll
            for (int r = 0; r < RS_R; ++r) acc[r].single(__dmul_rn(rs_rows[(int64_t)r * d + l], c0));
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < RS_R; ++r) {
        double sv = INFINITY;
        int32_t a = INT32_MAX;
        if (ok && r < nr) {
            const double t = __dsub_rn(__dadd_rn(vn[rid[r]], cn[q]), __dmul_rn(2.0, acc[r].result()));
            sv = t > 0.0 ? t : 0.0;
            a = (int32_t)q;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double os = __shfl_xor_sync(0xffffffffu, sv, o);
            const int32_t oa = __shfl_xor_sync(0xffffffffu, a, o);
            if (os < sv || (os == sv && oa < a)) {
                sv = os;
                a = oa;
            }
        }
        if (lane == 0) {
            rval[r][warp] = sv;
            ridx[r][warp] = a;
        }
    }
    __syncthreads();
    if (threadIdx.x < nr) {
        const int r = threadIdx.x;
        double sv = rval[r][0];
        int32_t a = ridx[r][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (rval[r][w] < sv || (rval[r][w] == sv && ridx[r][w] < a)) {
                sv = rval[r][w];
                a = ridx[r][w];
            }
        pval[(r0 + r) * nchunks + blockIdx.y] = sv;
        pidx[(r0 + r) * nchunks + blockIdx.y] = a;
    }
}

// per re-scanned row: minimum over the chunks (ascending centroid order,
// strict < keeps the lowest index on ties); labels / cost / change count
__global__ void as_rescan_merge_kernel(int64_t nf, int nchunks, const int32_t* __restrict__ fl,
                                       const double* __restrict__ pval, const int32_t* __restrict__ pidx,
                                       const int64_t* __restrict__ old_labels, int64_t* __restrict__ labels,
                                       double* __restrict__ cost, unsigned long long* __restrict__ changes) {
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int chg = 0;
    if (f < nf) {
        double sv = pval[f * nchunks];
        int32_t a = pidx[f * nchunks];
        for (int j = 1; j < nchunks; ++j)
            if (pval[f * nchunks + j] < sv) {
                sv = pval[f * nchunks + j];
                a = pidx[f * nchunks + j];
            }
        const int64_t i = fl[f];
        labels[i] = a;
        cost[i] = sv;
        if (old_labels) chg = old_labels[i] != a;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, chg);
    if ((threadIdx.x & 31) == 0 && bal) atomicAdd(changes, (unsigned long long)__popc(bal));
}

// flagged rows: exact scan over all centroids (warp per row, lowest index on ties)
__global__ void as_rescan_kernel(int64_t d, int64_t k, const double* __restrict__ v, const double* __restrict__ vn,
                                 const double* __restrict__ c, const double* __restrict__ cn,
                                 const int32_t* __restrict__ flagged, const unsigned long long* __restrict__ nflag,
                                 const int64_t* __restrict__ old_labels, int64_t* __restrict__ labels,
                                 double* __restrict__ cost, unsigned long long* __restrict__ changes) {
    const int64_t nf = (int64_t)*nflag;
    const int lane = threadIdx.x & 31;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nf;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t i = flagged[w];
        double best = INFINITY;
        int64_t arg = 0;
        for (int64_t q = lane; q < k; q += 32) {
            const double sv = exact_s(v + i * d, vn[i], c + q * d, cn[q], d);
            if (sv < best) {
                best = sv;
                arg = q;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int64_t oa = __shfl_xor_sync(0xffffffffu, arg, o);
            if (ob < best || (ob == best && oa < arg)) {
                best = ob;
                arg = oa;
            }
        }
        if (lane == 0) {
            labels[i] = arg;
            cost[i] = best;
            if (old_labels && old_labels[i] != arg) atomicAdd(changes, 1ull);
        }
    }
}

// compact copy of the flagged rows (and their norms / old labels)
__global__ void as_gather_kernel(int64_t nf, int64_t d, const int32_t* __restrict__ flagged,
                                 const double* __restrict__ v, const double* __restrict__ vn,
                                 const int64_t* __restrict__ old_labels, double* __restrict__ vf,
                                 double* __restrict__ vnf, int64_t* __restrict__ oldf) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nf * d) return;
    const int64_t r = e / d, l = e - r * d;
    const int64_t i = flagged[r];
    vf[e] = v[i * d + l];
    if (l == 0) {
        vnf[r] = vn[i];
        if (old_labels) oldf[r] = old_labels[i];
    }
}
__global__ void as_scatter_kernel(int64_t nf, const int32_t* __restrict__ flagged, const int64_t* __restrict__ labf,
                                  const double* __restrict__ costf, int64_t* __restrict__ labels,
                                  double* __restrict__ cost) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nf) return;
    labels[flagged[r]] = labf[r];
    cost[flagged[r]] = costf[r];
}

// part[b] = cost[64 b] + ... + cost[64 b + 63], sequential (the same fixed
// order as dist_tile_kernel's per-block sum, so the SSE is path-independent)
__global__ void cost_block_sum_kernel(int64_t n, const double* __restrict__ cost, double* __restrict__ part) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b * TP >= n) return;
    double acc = 0.0;
    for (int64_t i = b * TP; i < imin64(n, (b + 1) * TP); ++i) acc += cost[i];
    part[b] = acc;
}

template <int NKB, int STAGES, int QT>
static int launch_assign_tc(const CUtensorMap& vmap, const CUtensorMap& cmap, int64_t n, int64_t nptiles,
                            int64_t nctiles, const float* cnk, float key_scale, int32_t* best_idx, float2* best_keys,
                            int2* alt_idx, float2* alt_keys, cudaStream_t st) {
    const uint32_t smem = AsLayout<NKB, STAGES, QT>::total;
    SC_CUDA(cudaFuncSetAttribute(assign_tc_kernel<NKB, STAGES, QT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    assign_tc_kernel<NKB, STAGES, QT><<<(unsigned)ceil_div(nptiles, QT), 64 + QT * 128, smem, st>>>(
        vmap, cmap, n, nptiles, nctiles, cnk, key_scale, best_idx, best_keys, alt_idx, alt_keys);
    SC_LAUNCHED(1);
    return SC_OK;
}

template <int STAGES, int QT>
static int launch_assign_tc_kl(const CUtensorMap& vmap, const CUtensorMap& cmap, int64_t n, int64_t nptiles,
                               int64_t nctiles, int nkb, const float* cnk, float key_scale, int32_t* best_idx,
                               float2* best_keys, int2* alt_idx, float2* alt_keys, cudaStream_t st) {
    const uint32_t smem = AsKlLayout<STAGES, QT>::total;
    SC_CUDA(cudaFuncSetAttribute(assign_tc_kl_kernel<STAGES, QT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    assign_tc_kl_kernel<STAGES, QT><<<(unsigned)ceil_div(nptiles, QT), 64 + QT * 128, smem, st>>>(
        vmap, cmap, n, nptiles, nctiles, nkb, cnk, key_scale, best_idx, best_keys, alt_idx, alt_keys);
    SC_LAUNCHED(1);
    return SC_OK;
}

// Per-lloyd-call state of the tensor-core assignment (V converted once).
struct AssignTc {
    int64_t n = 0, d = 0, dp = 0, n_pad = 0;
    double s = 1.0;
    bool active = false;
    DevBuf<__half> vh;
    CUtensorMap vmap;
    DevBuf<int32_t> bidx, flagged;
    DevBuf<float2> bkeys, akeys;
    DevBuf<int2> aidx;
    DevBuf<int32_t> flagged2;
    DevBuf<unsigned long long> scal;  // [0] nflag, [1] cnmax bits, [2] absmax bits, [3] nflag after resolve
    // eligible: enough rows to pay for the conversion; SPECLUST_ASSIGN=fp64 disables.
    // dp <= 256: point tiles resident in shared memory; wider: K-chunk ring
    int init(int64_t n_, int64_t d_, int64_t k, const double* v, cudaStream_t st) {
        n = n_;
        d = d_;
        dp = (d + 63) / 64 * 64;
        const char* env = std::getenv("SPECLUST_ASSIGN");
        active = !(env && std::strcmp(env, "fp64") == 0) && d >= 1 && n >= 4096 && k >= 8;
        if (!active) return SC_OK;
        n_pad = (n + 127) / 128 * 128;
        int rc;
        if ((rc = vh.alloc((size_t)n_pad * dp)) || (rc = bidx.alloc(n)) || (rc = bkeys.alloc(n)) ||
            (rc = flagged.alloc(n)) || (rc = scal.alloc(4)) || (rc = akeys.alloc(n)) || (rc = aidx.alloc(n)) ||
            (rc = flagged2.alloc(n)))
            return rc;
        SC_CUDA(cudaMemsetAsync(scal.p, 0, sizeof(unsigned long long) * 4, st));
        as_absmax_kernel<<<kNumSMs * 4, 256, 0, st>>>(n * d, v, scal.p + 2);
        SC_LAUNCHED(1);
        unsigned long long hb = 0;
        SC_CUDA(d2h_sync(&hb, scal.p + 2, sizeof(hb), st));
        double amax;
        std::memcpy(&amax, &hb, sizeof(amax));
        // power-of-two scale: |s x| <= 128 for every element of V (centroids
        // are means / copies of rows, so the same bound holds for them)
        s = amax > 0 ? std::ldexp(1.0, (int)std::floor(std::log2(128.0 / amax))) : 1.0;
        as_prep_rows_kernel<<<(unsigned)ceil_div(n_pad, 8), 256, 0, st>>>(n, n_pad, d, dp, v, s, vh.p);
        SC_LAUNCHED(1);
        return make_f16_tile_map(&vmap, vh.p, n_pad, dp);
    }
    // labels / cost / change count of one assignment step
    // certify = false: labels are the approximate argmin (no exact costs, no
    // rescan) -- for callers that only need a heuristic grouping
    int assign(int64_t k, const double* v, const double* vn, const double* c, const double* cn,
               const int64_t* old_labels, int64_t* labels, double* cost, unsigned long long* changes,
               cudaStream_t st, bool certify = true) {
        const int64_t k_pad = (k + 127) / 128 * 128;
        DevBuf<__half> ch;
        DevBuf<float> cnk;
        int rc;
        if ((rc = ch.alloc((size_t)k_pad * dp)) || (rc = cnk.alloc(k_pad))) return rc;
        SC_CUDA(cudaMemsetAsync(scal.p, 0, sizeof(unsigned long long) * 2, st));
        SC_CUDA(cudaMemsetAsync(scal.p + 3, 0, sizeof(unsigned long long), st));
        as_prep_rows_kernel<<<(unsigned)ceil_div(k_pad, 8), 256, 0, st>>>(k, k_pad, d, dp, c, s, ch.p);
        as_cent_norms_kernel<<<(unsigned)ceil_div(k_pad, 256), 256, 0, st>>>(k, k_pad, cn, cnk.p, scal.p + 1);
        SC_LAUNCHED(2);
        CUtensorMap cmap;
        if ((rc = make_f16_tile_map(&cmap, ch.p, k_pad, dp))) return rc;
        const int64_t nptiles = n_pad / 128, nctiles = k_pad / 128;
        const float key_scale = (float)(-2.0 / (s * s));
        static const bool dbg = std::getenv("SPECLUST_ASSIGN_DEBUG") != nullptr;
        // SPECLUST_ASSIGN_DEBUG: per-phase device times on stderr
        struct PhaseEv {
            bool on;
            cudaStream_t st;
            int m = 0;
            cudaEvent_t ev[8];
            const char* name[8];
            void mark(const char* nm) {
                if (!on || m >= 8) return;
                cudaEventCreate(&ev[m]);
                cudaEventRecord(ev[m], st);
                name[m++] = nm;
            }
            ~PhaseEv() {
                if (!on) return;
                mark("end");
                cudaEventSynchronize(ev[m - 1]);
                fprintf(stderr, "[assign_tc]");
                for (int j = 1; j < m; ++j) {
                    float t = 0;
                    cudaEventElapsedTime(&t, ev[j - 1], ev[j]);
                    fprintf(stderr, " %s %.3f ms", name[j - 1], t);
                }
                fprintf(stderr, "\n");
                for (int j = 0; j < m; ++j) cudaEventDestroy(ev[j]);
            }
        } evp{dbg, st};
        evp.mark("tc");
        // STAGES counts 64-column centroid chunks (16 KB each)
        int2* ai = aidx.p;
        float2* ak = akeys.p;
        switch (dp / 64) {
            case 1: rc = launch_assign_tc<1, 8, 2>(vmap, cmap, n, nptiles, nctiles, cnk.p, key_scale, bidx.p, bkeys.p, ai, ak, st); break;
            case 2: rc = launch_assign_tc<2, 8, 2>(vmap, cmap, n, nptiles, nctiles, cnk.p, key_scale, bidx.p, bkeys.p, ai, ak, st); break;
            case 3: rc = launch_assign_tc<3, 6, 2>(vmap, cmap, n, nptiles, nctiles, cnk.p, key_scale, bidx.p, bkeys.p, ai, ak, st); break;
            case 4: rc = launch_assign_tc<4, 4, 2>(vmap, cmap, n, nptiles, nctiles, cnk.p, key_scale, bidx.p, bkeys.p, ai, ak, st); break;
            default: rc = launch_assign_tc_kl<4, 2>(vmap, cmap, n, nptiles, nctiles, (int)(dp / 64), cnk.p, key_scale, bidx.p, bkeys.p, ai, ak, st); break;
        }
        if (rc) return rc;
        evp.mark("finalize");
        if (!certify) {
            as_take_best_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, bidx.p, labels);
            SC_LAUNCHED(1);
            return SC_OK;
        }
        as_finalize_rows_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
            n, d, dp, s, v, vn, c, cn, scal.p + 1, bidx.p, bkeys.p, old_labels, labels, cost, flagged.p, scal.p,
            changes, d % 2 == 0 && ((reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(c)) & 15) == 0);
        SC_LAUNCHED(1);
        // uncertified rows: exact re-scan.  Few rows or few centroids: a warp
        // per row; otherwise the rows are gathered and run through the tiled
        // fp64 assignment kernel (the same arithmetic as the fp64 path)
        int64_t nf = flagged_count(st);
        if (nf == 0) return SC_OK;
        evp.mark("resolve");
        // at most three candidates within 2 delta of the best: exact keys of those
        constexpr int res_smem = 8 * kPairStage * (int)sizeof(double);
        SC_CUDA(cudaFuncSetAttribute(as_resolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, res_smem));
        as_resolve_kernel<<<(unsigned)ceil_div(nf, 80), 256, res_smem, st>>>(
            nf, d, dp, s, v, vn, c, cn, scal.p + 1, flagged.p, bkeys.p, akeys.p, bidx.p, aidx.p, old_labels, labels,
            cost, changes, flagged2.p, scal.p + 3);
        SC_LAUNCHED(1);
        {
            unsigned long long h = 0;
            SC_CUDA(d2h_sync(&h, scal.p + 3, sizeof(h), st));
            if (dbg) fprintf(stderr, "[assign_tc] uncertified %lld, after the three-candidate resolve %llu\n",
                             (long long)nf, h);
            nf = (int64_t)h;
        }
        if (nf == 0) return SC_OK;
        evp.mark("rescan");
        const int32_t* fl = flagged2.p;
        DevBuf<double> ct, pval;
        DevBuf<int32_t> pidx;
        const int nchunks = (int)ceil_div(k, 256);
        const int64_t batch = std::min<int64_t>(nf, std::max<int64_t>(RS_R, ((int64_t)1 << 24) / nchunks));
        if ((rc = ct.alloc((size_t)k * d)) || (rc = pval.alloc((size_t)batch * nchunks)) ||
            (rc = pidx.alloc((size_t)batch * nchunks)))
            return rc;
        as_transpose_kernel<<<(unsigned)ceil_div(k * d, 256), 256, 0, st>>>(k, d, c, ct.p);
        SC_LAUNCHED(1);
        const int rs_smem = (int)(RS_R * d * sizeof(double));
        if (rs_smem > 200 * 1024) {  // very wide rows: warp per row
            as_rescan_kernel<<<kNumSMs * 4, 256, 0, st>>>(d, k, v, vn, c, cn, fl, scal.p + 3, old_labels, labels,
                                                          cost, changes);
            SC_LAUNCHED(1);
            return SC_OK;
        }
        SC_CUDA(cudaFuncSetAttribute(as_rescan_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, rs_smem));
        for (int64_t f0 = 0; f0 < nf; f0 += batch) {
            const int64_t nb = std::min(batch, nf - f0);
            as_rescan_tile_kernel<<<dim3((unsigned)ceil_div(nb, RS_R), (unsigned)nchunks), 256, rs_smem, st>>>(
                nb, d, k, v, vn, ct.p, cn, fl + f0, nchunks, pval.p, pidx.p);
            as_rescan_merge_kernel<<<(unsigned)ceil_div(nb, 256), 256, 0, st>>>(nb, nchunks, fl + f0, pval.p, pidx.p,
                                                                              old_labels, labels, cost, changes);
            SC_LAUNCHED(2);
        }
        return SC_OK;
    }
    int64_t flagged_count(cudaStream_t st) {
        unsigned long long h = 0;
        d2h_sync(&h, scal.p, sizeof(h), st);
        return (int64_t)h;
    }
};

}  // namespace sc

namespace sc {
// labels[i] = index of the nearest of the k rows of c: exact fp64 Gram
// expansion, or (eligible shapes) the tensor-core argmin without the exact
// certificate -- used only for the kNN scan-order grouping, where any
// near-nearest pivot serves
int assign_nearest(int64_t n, int64_t d, const double* v, int64_t k, const double* c, int64_t* labels,
                   cudaStream_t st) {
    const int64_t nb = ceil_div(n, TP);
    DevBuf<double> vn, cn, cost, part;
    DevBuf<unsigned long long> changes;
    int rc;
    if ((rc = vn.alloc(n)) || (rc = cn.alloc(k)) || (rc = cost.alloc(n)) || (rc = part.alloc(nb)) ||
        (rc = changes.alloc(1)))
        return rc;
    SC_CUDA(cudaMemsetAsync(changes.p, 0, sizeof(unsigned long long), st));
    rownorm_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d, v, vn.p);
    rownorm_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(k, d, c, cn.p);
    SC_LAUNCHED(2);
    AssignTc atc;
    if ((rc = atc.init(n, d, k, v, st))) return rc;
    if (atc.active) return atc.assign(k, v, vn.p, c, cn.p, nullptr, labels, cost.p, changes.p, st, false);
    dist_tile_kernel<0><<<(unsigned)nb, 256, 0, st>>>(n, k, d, v, vn.p, c, cn.p, nullptr, labels, nullptr, cost.p,
                                                      changes.p, part.p);
    SC_LAUNCHED(1);
    return SC_OK;
}

}  // namespace sc

using namespace sc;

// ---------------------------------------------------------------------------
// host entry points
struct sc_kmeanspp {
    int64_t n = 0, d = 0, nb_upd = 0, nb_p = 0;
    const double* v = nullptr;
    cudaStream_t st = nullptr;
    bool first = true;
    int64_t taken_count = 0;
    DevBuf<double> d2, pw, bsum, total, v8;  // v8: the points in 8-column panels
    DevBuf<int64_t> pc, count, pick;
    DevBuf<uint8_t> taken;
    // centres drawn so far (up to ccap), their distances to the newest one and
    // each row's nearest centre: the triangle-inequality skip of the update
    static constexpr int ccap = 1024;
    DevBuf<double> cent, cc;
    DevBuf<int32_t> ctr;
    int ncent = 0;
    bool bound = false;
    // fp16 screen (KppScreen): points as fp16 panels, the centre in fp16
    // groups of identical rows (rep[i]: smallest index with the same bits):
    // the update computes one distance per group
    DevBuf<int32_t> rep, reps;
    int64_t nreps = 0;
    DevBuf<uint32_t> nzm;  // nonzero-panel bitmap (only when >= 1/4 of the panels are zero)
    DevBuf<uint4> vh8;
    DevBuf<__half> ch;
    DevBuf<double> vnorm, cnorm;
    DevBuf<unsigned long long> sstat;  // screened / pruned row counts (kpp_update_panel_kernel)
    double hs = 1.0;
    bool screen = false;
    int screened_draws = 0;
    // the screen only pays when it prunes: on embeddings whose clusters are
    // all at the same distance (orthogonal unit rows, e.g. C3) the fp16 bound
    // cannot separate a new distance from the old one and every row still
    // needs the exact pass -- after a few draws such a screen is switched off
    void screen_review() {
        if (!screen || ++screened_draws != 8) return;
        unsigned long long h[2] = {0, 0};
        d2h_sync(h, sstat.p, sizeof(h), st);
        if (h[0] > 0 && (double)h[1] < 0.25 * (double)h[0]) screen = false;
    }

    // d2 <- min(d2, |v - row|^2) and the candidate partials (row: the drawn
    // point's coordinates, device; pick: its local index or -1)
    int update(const double* row, int64_t pick_index) {
        ProfScope prof("kmeanspp", st, (double)n * d * 8.0);
        if (v8.p) {
            const double* ccp = nullptr;
            int t = -1;
            if (bound && ncent < ccap) {
                t = ncent++;
                SC_CUDA(cudaMemcpyAsync(cent.p + (int64_t)t * d, row, sizeof(double) * d, cudaMemcpyDeviceToDevice,
                                        st));
                if (t > 0) {
                    kpp_centre_dist_kernel<<<(unsigned)ceil_div(t, 8), 256, 0, st>>>(d, t, cent.p, cc.p);
                    SC_LAUNCHED(1);
                    ccp = cc.p;
                }
            } else {
                bound = false;  // past ccap centres: plain updates from here on
            }
            KppScreen scr;
            size_t smem = (size_t)ceil_div(d, 8) * 8 * sizeof(double);
            static size_t smem_attr = 48 * 1024;
            if (screen && !first) {
                kpp_centre_half_kernel<<<1, 256, 0, st>>>(d, row, hs, ch.p, cnorm.p);
                SC_LAUNCHED(1);
                scr.vh8 = vh8.p;
                scr.ch = ch.p;
                scr.vnorm = vnorm.p;
                scr.cnorm = cnorm.p;
                scr.s = hs;
                scr.stats = sstat.p;
                smem += (size_t)ceil_div(d, 8) * 8 * sizeof(__half);
            }
            if (smem > smem_attr) {
                SC_CUDA(cudaFuncSetAttribute(kpp_update_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
                smem_attr = smem;
            }
            if (reps.p) {
                kpp_update_panel_kernel<<<(unsigned)ceil_div(nreps, KPP_UPD_ROWS), KPP_UPD_ROWS, smem, st>>>(
                    n, d, v8.p, row, -1, first ? 1 : 0, d2.p, taken.p, nullptr, nullptr, ccp,
                    bound ? ctr.p : nullptr, t, scr, reps.p, nreps, nzm.p);
                kpp_expand_kernel<<<(unsigned)nb_upd, KPP_UPD_ROWS, 0, st>>>(n, rep.p, pick_index, d2.p, taken.p,
                                                                           bound ? ctr.p : nullptr, pw.p, pc.p);
                SC_LAUNCHED(1);
            } else {
                kpp_update_panel_kernel<<<(unsigned)nb_upd, KPP_UPD_ROWS, smem, st>>>(
                    n, d, v8.p, row, pick_index, first ? 1 : 0, d2.p, taken.p, pw.p, pc.p, ccp,
                    bound ? ctr.p : nullptr, t, scr, nullptr, 0, nzm.p);
            }
        } else {
            kpp_update_kernel<<<(unsigned)nb_upd, KPP_UPD_ROWS, 0, st>>>(n, d, v, row, pick_index, first ? 1 : 0, d2.p,
                                                                         taken.p, pw.p, pc.p);
        }
        SC_LAUNCHED(1);
        return SC_OK;
    }
};

extern "C" {

int sc_pairwise_sq_dist(int64_t n, int64_t k, int64_t d, const double* v, const double* c,
                        double* out, sc_stream_t stream) {
    if (n < 0 || k < 0 || d < 0) return fail(SC_ERR_VALUE, "negative dimension");
    if (n == 0 || k == 0) return SC_OK;
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    DevBuf<double> vn, cn;
    if (int rc = vn.alloc(n)) return rc;
    if (int rc = cn.alloc(k)) return rc;
    rownorm_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d, v, vn.p);
    rownorm_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(k, d, c, cn.p);
    dist_tile_kernel<1><<<(unsigned)ceil_div(n, TP), 256, 0, st>>>(n, k, d, v, vn.p, c, cn.p, out,
                                                                   nullptr, nullptr, nullptr, nullptr, nullptr);
    SC_LAUNCHED(3);
    SC_CUDA(cudaStreamSynchronize(st));
    return SC_OK;
}

int sc_lloyd(int64_t n, int64_t d, int64_t k, const double* v, const double* c_init,
             int64_t max_iters, int64_t tol_changes, int64_t* labels, double* centroids,
             double* sse_history, int64_t* iters_out, sc_stream_t stream) {
    if (n < 1 || k < 1 || d < 0) return fail(SC_ERR_VALUE, "lloyd requires n >= 1, k >= 1");
    if (max_iters < 1) return fail(SC_ERR_VALUE, "max_iters must be >= 1");
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    const int64_t nb = ceil_div(n, TP);
    DevBuf<double> vn, cn, cost, part, sse;
    DevBuf<int64_t> lab2;
    DevBuf<unsigned long long> changes;
    DevBuf<int> empty;
    DevBuf<uint8_t> used;
    DevBuf<double> pv;
    DevBuf<int64_t> pi;
    Bucketer bk;
    int rc;
    if ((rc = vn.alloc(n)) || (rc = cn.alloc(k)) || (rc = cost.alloc(n)) || (rc = part.alloc(nb)) ||
        (rc = sse.alloc(1)) || (rc = lab2.alloc(n)) || (rc = changes.alloc(1)) || (rc = empty.alloc(k)) ||
        (rc = bk.init(n, k)))
        return rc;
    SC_CUDA(cudaMemcpyAsync(centroids, c_init, sizeof(double) * k * d, cudaMemcpyDeviceToDevice, st));
    rownorm_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d, v, vn.p);
    rownorm_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(k, d, centroids, cn.p);
    double flops = 2.0 * (double)n * (double)k * (double)d;
    // tensor-core assignment with certified argmin when eligible (any width)
    AssignTc atc;
    if ((rc = atc.init(n, d, k, v, st))) return rc;
    auto assign_step = [&](const int64_t* old_lab, int64_t* out_lab) -> int {
        ProfScope prof("kmeans_assign", st, flops);
        if (atc.active) {
            int r = atc.assign(k, v, vn.p, centroids, cn.p, old_lab, out_lab, cost.p, changes.p, st);
            if (r) return r;
            if (std::getenv("SPECLUST_ASSIGN_DEBUG"))
                fprintf(stderr, "[assign_tc] n=%lld k=%lld d=%lld rescanned rows %lld\n", (long long)n, (long long)k,
                        (long long)d, (long long)atc.flagged_count(st));
            cost_block_sum_kernel<<<(unsigned)ceil_div(nb, 256), 256, 0, st>>>(n, cost.p, part.p);
        } else {
            dist_tile_kernel<0><<<(unsigned)nb, 256, 0, st>>>(n, k, d, v, vn.p, centroids, cn.p, nullptr, out_lab,
                                                              old_lab, cost.p, changes.p, part.p);
        }
        SC_LAUNCHED(1);
        return SC_OK;
    };
    SC_LAUNCHED(2);
    if ((rc = assign_step(nullptr, labels))) return rc;
    NpSum npsum;
    if ((rc = npsum.sum(cost.p, n, &sse_history[0], st))) return rc;

    int64_t* cur = labels;
    int64_t* nxt = lab2.p;
    int64_t iters = 0;
    const int64_t dchunks = ceil_div(d, 32);
    std::vector<int64_t> hseg(k + 1, 0);
    DevBuf<int64_t> seg_off;
    DevBuf<double> segpart;
    if ((rc = seg_off.alloc(k + 1)) || (rc = segpart.alloc((size_t)(n / CM_SEG + k + 1) * d))) return rc;
    while (iters < max_iters) {
        // ---- update (kmeans.py:139-156)
        if ((rc = bk.run(cur, st))) return rc;
        // cluster sizes (host): segment plan + empty clusters
        std::vector<int64_t> hstart(k + 1);
        SC_CUDA(d2h_sync(hstart.data(), bk.start.p, sizeof(int64_t) * (k + 1), st));
        for (int64_t c = 0; c < k; ++c) hseg[c + 1] = hseg[c] + ceil_div(hstart[c + 1] - hstart[c], CM_SEG);
        const int64_t nseg = hseg[k];
        {
            ProfScope prof("kmeans_update", st, (double)n * d * 8.0 + 12.0 * n + 16.0 * k * d);
            SC_CUDA(cudaMemcpyAsync(seg_off.p, hseg.data(), sizeof(int64_t) * (k + 1), cudaMemcpyHostToDevice, st));
            if (nseg > 0)
                if ((rc = segsum_smem_attr())) return rc;
                centroid_segsum_smem_kernel<<<(unsigned)(nseg * dchunks), 32, 2 * CS_BATCH * 32 * sizeof(double),
                                              st>>>(k, d, nseg, v, bk.start.p, bk.members.p, seg_off.p, segpart.p);
            centroid_segmean_kernel<<<(unsigned)ceil_div(k * d, 256), 256, 0, st>>>(k, d, bk.start.p, seg_off.p,
                                                                                    segpart.p, centroids);
        }
        SC_LAUNCHED(2);
        std::vector<int64_t> empties;
        for (int64_t c = 0; c < k; ++c)
            if (hstart[c + 1] == hstart[c]) empties.push_back(c);
        if (!empties.empty()) {
            if (!used.p) {
                if ((rc = used.alloc(n)) || (rc = pv.alloc(256)) || (rc = pi.alloc(256))) return rc;
            }
            SC_CUDA(cudaMemsetAsync(used.p, 0, n, st));
            for (size_t s = 0; s < empties.size() && (int64_t)s < n; ++s) {
                argmax_partial_kernel<<<256, 256, 0, st>>>(n, cost.p, used.p, pv.p, pi.p);
                reseed_finish_kernel<<<1, 128, 0, st>>>(256, pv.p, pi.p, d, v, used.p, centroids, empties[s]);
                SC_LAUNCHED(2);
            }
        }
        // ---- assign
        rownorm_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(k, d, centroids, cn.p);
        SC_CUDA(cudaMemsetAsync(changes.p, 0, sizeof(unsigned long long), st));
        if ((rc = assign_step(cur, nxt))) return rc;
        SC_LAUNCHED(1);
        unsigned long long hchg = 0;
        SC_CUDA(d2h_sync(&hchg, changes.p, sizeof(hchg), st));
        if ((rc = npsum.sum(cost.p, n, &sse_history[iters + 1], st))) return rc;
        ++iters;
        std::swap(cur, nxt);
        if ((int64_t)hchg <= tol_changes) break;
    }
    if (cur != labels) SC_CUDA(cudaMemcpyAsync(labels, cur, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));
    SC_CUDA(cudaStreamSynchronize(st));
    *iters_out = iters;
    return SC_OK;
}

int sc_kmeanspp_create(int64_t n, int64_t d, const double* v, sc_stream_t stream, sc_kmeanspp_t** out) {
    if (n < 1) return fail(SC_ERR_VALUE, "k-means++ needs n >= 1");
    StreamScope stream_scope(as_stream(stream));
    auto* s = new sc_kmeanspp();
    s->n = n;
    s->d = d;
    s->v = v;
    s->st = as_stream(stream);
    s->nb_upd = ceil_div(n, KPP_UPD_ROWS);
    s->nb_p = ceil_div(n, KPP_BLK);
    int rc;
    if ((rc = s->d2.alloc(n)) || (rc = s->taken.alloc(n)) || (rc = s->pw.alloc(s->nb_upd)) ||
        (rc = s->pc.alloc(s->nb_upd)) || (rc = s->bsum.alloc(s->nb_p)) || (rc = s->total.alloc(1)) ||
        (rc = s->count.alloc(1)) || (rc = s->pick.alloc(1))) {
        delete s;
        return rc;
    }
    cudaMemsetAsync(s->taken.p, 0, n, s->st);
    // 8-column panels of the points for the update (skipped when memory is short)
    const int64_t nch = ceil_div(d, 8);
    // (the panel update stages the centre row in shared memory: d <= 24576)
    if (d <= 24576 && s->v8.alloc((size_t)nch * n * 8) == SC_OK) {
        // identical rows (e.g. the constant rows of a graph component whose
        // eigenvalue-1 eigenvector is locked): one distance per group;
        // used when it saves at least a quarter of the rows
        const char* denv = std::getenv("SPECLUST_KPP_DEDUP");
        if (!(denv && denv[0] == '0') && n >= 4096 && d >= 8 && n < ((int64_t)1 << 31)) {
            uint64_t tsz = 1;
            while (tsz < (uint64_t)(2 * n)) tsz <<= 1;
            DevBuf<uint64_t> hsh;
            DevBuf<unsigned long long> keys, vals;
            DevBuf<int64_t> isrep, pos, tmp;
            if (hsh.alloc(n) == SC_OK && keys.alloc(tsz) == SC_OK && vals.alloc(tsz) == SC_OK &&
                isrep.alloc(n) == SC_OK && pos.alloc(n + 1) == SC_OK && tmp.alloc(ceil_div(n, 1024) + 2) == SC_OK &&
                s->rep.alloc(n) == SC_OK) {
                cudaMemsetAsync(keys.p, 0xff, sizeof(unsigned long long) * tsz, s->st);
                cudaMemsetAsync(vals.p, 0xff, sizeof(unsigned long long) * tsz, s->st);
                const unsigned nbk = (unsigned)ceil_div(n, 256);
                row_hash_kernel<<<nbk, 256, 0, s->st>>>(n, d, v, hsh.p);
                hash_insert_kernel<<<nbk, 256, 0, s->st>>>(n, hsh.p, tsz - 1, keys.p, vals.p);
                hash_rep_kernel<<<nbk, 256, 0, s->st>>>(n, d, v, hsh.p, tsz - 1, keys.p, vals.p, s->rep.p, isrep.p);
                SC_LAUNCHED(3);
                int64_t nr = n;
                if (exclusive_scan_i64(n, isrep.p, pos.p, tmp.p, s->st) == SC_OK) {
                    SC_CUDA(d2h_sync(&nr, pos.p + n, sizeof(int64_t), s->st));
                    if (nr <= n - n / 4 && s->reps.alloc(std::max<int64_t>(nr, 1)) == SC_OK) {
                        compact_reps_kernel<<<nbk, 256, 0, s->st>>>(n, isrep.p, pos.p, s->reps.p);
                        SC_LAUNCHED(1);
                        s->nreps = nr;
                    }
                }
                if (std::getenv("SPECLUST_TIMING_DEBUG"))
                    fprintf(stderr, "[kmeans++] identical-row groups: %lld of %lld rows (%s)\n", (long long)nr,
                            (long long)n, s->reps.p ? "used" : "not used");
            }
            if (!s->reps.p) s->rep.free();
        }
        to_panels_kernel<<<(unsigned)ceil_div(nch * n * 8, 256), 256, 0, s->st>>>(n, d, v, s->v8.p);
        SC_LAUNCHED(1);
        {
            const char* zenv = std::getenv("SPECLUST_KPP_ZERO_PANELS");
            const int64_t nw = ceil_div(nch, 32);
            DevBuf<unsigned long long> nzero;
            if (!(zenv && zenv[0] == '0') && nch >= 4 && s->nzm.alloc((size_t)nw * n) == SC_OK &&
                nzero.alloc(1) == SC_OK) {
                cudaMemsetAsync(nzero.p, 0, sizeof(unsigned long long), s->st);
                panel_nonzero_kernel<<<(unsigned)ceil_div(nw * n, 256), 256, 0, s->st>>>(n, nch, s->v8.p, s->nzm.p,
                                                                                        nzero.p);
                SC_LAUNCHED(1);
                unsigned long long hz = 0;
                SC_CUDA(d2h_sync(&hz, nzero.p, sizeof(hz), s->st));
                if (std::getenv("SPECLUST_TIMING_DEBUG"))
                    fprintf(stderr, "[kmeans++] zero panels: %llu of %lld\n", hz, (long long)(nch * n));
                if ((double)hz < 0.25 * (double)(nch * n)) s->nzm.free();
            } else {
                s->nzm.free();
            }
        }
        s->bound = s->cent.alloc((size_t)sc_kmeanspp::ccap * d) == SC_OK &&
                   s->cc.alloc(sc_kmeanspp::ccap) == SC_OK && s->ctr.alloc(n) == SC_OK;
        // the fp16 screen pays for itself once a row is wider than a few
        // panels; optional (memory) and off with SPECLUST_KPP_SCREEN=0
        const char* env = std::getenv("SPECLUST_KPP_SCREEN");
        const bool want = !(env && env[0] == '0') && d >= 32 && d <= 8192;
        if (want && s->vh8.alloc((size_t)nch * n) == SC_OK && s->ch.alloc((size_t)nch * 8) == SC_OK &&
            s->vnorm.alloc(n) == SC_OK && s->cnorm.alloc(1) == SC_OK && s->sstat.alloc(2) == SC_OK) {
            cudaMemsetAsync(s->sstat.p, 0, 2 * sizeof(unsigned long long), s->st);
            DevBuf<unsigned long long> amax;
            if (amax.alloc(1) == SC_OK) {
                cudaMemsetAsync(amax.p, 0, sizeof(unsigned long long), s->st);
                as_absmax_kernel<<<kNumSMs * 4, 256, 0, s->st>>>(n * d, v, amax.p);
                rownorm_sqrt_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s->st>>>(n, d, v, s->vnorm.p);
                SC_LAUNCHED(2);
                unsigned long long hb = 0;
                SC_CUDA(d2h_sync(&hb, amax.p, sizeof(hb), s->st));
                double am;
                std::memcpy(&am, &hb, sizeof(am));
                // |s v| <= 2^14: far from the fp16 overflow at 65504
                s->hs = am > 0 ? std::ldexp(1.0, (int)std::floor(std::log2(16384.0 / am))) : 1.0;
                to_half_panels_kernel<<<(unsigned)ceil_div(nch * n, 256), 256, 0, s->st>>>(n, d, v, s->hs,
                                                                                            s->vh8.p);
                SC_LAUNCHED(1);
                s->screen = true;
            }
        }
    }
    *out = s;
    return SC_OK;
}

void sc_kmeanspp_destroy(sc_kmeanspp_t* s) { delete s; }

int sc_kmeanspp_take(sc_kmeanspp_t* s, int64_t index) {
    if (index < 0 || index >= s->n) return fail(SC_ERR_VALUE, "k-means++ index out of range");
    if (int rc = s->update(s->v + index * s->d, index)) return rc;
    if (!s->first) s->screen_review();
    kpp_total_kernel<<<1, 1024, 0, s->st>>>(s->nb_upd, s->pw.p, s->pc.p, s->total.p, s->count.p);
    SC_LAUNCHED(1);
    s->first = false;
    s->taken_count += 1;
    return SC_OK;
}

int sc_kmeanspp_candidates(sc_kmeanspp_t* s, int64_t* count, int64_t* n_free) {
    SC_CUDA(d2h_sync(count, s->count.p, sizeof(int64_t), s->st));
    *n_free = s->n - s->taken_count;
    return SC_OK;
}

int sc_kmeanspp_pick(sc_kmeanspp_t* s, int mode, double u, int64_t r, int64_t* index) {
    if (mode == 0) {
        kpp_psum_kernel<<<(unsigned)s->nb_p, KPP_BLK, 0, s->st>>>(s->n, s->d2.p, s->taken.p, s->total.p, s->bsum.p);
        kpp_search_kernel<<<1, 32, 0, s->st>>>(s->n, s->nb_p, s->d2.p, s->taken.p, s->total.p, s->bsum.p, u,
                                               s->pick.p);
        SC_LAUNCHED(2);
    } else {
        kpp_nth_free_kernel<<<1, 32, 0, s->st>>>(s->n, s->taken.p, r, s->pick.p);
        SC_LAUNCHED(1);
    }
    int64_t h = -1;
    SC_CUDA(d2h_sync(&h, s->pick.p, sizeof(int64_t), s->st));
    if (h < 0) return fail(SC_ERR_INTERNAL, "k-means++ draw found no row");
    *index = h;
    return sc_kmeanspp_take(s, h);
}

// ---- shard-aware k-means++ steps (point shards, global draw order = rank order)
int sc_kmeanspp_take_row(sc_kmeanspp_t* s, const double* row, int64_t local_index) {
    if (int rc = s->update(row, local_index)) return rc;
    kpp_total_kernel<<<1, 1024, 0, s->st>>>(s->nb_upd, s->pw.p, s->pc.p, s->total.p, s->count.p);
    SC_LAUNCHED(1);
    s->first = false;
    if (local_index >= 0) s->taken_count += 1;
    return SC_OK;
}

// local candidate weight sum (sum of d2 over untaken rows with d2 > 0), count, untaken rows
int sc_kmeanspp_weight(sc_kmeanspp_t* s, double* wsum, int64_t* count, int64_t* n_free) {
    SC_CUDA(d2h_sync(wsum, s->total.p, sizeof(double), s->st));
    SC_CUDA(d2h_sync(count, s->count.p, sizeof(int64_t), s->st));
    *n_free = s->n - s->taken_count;
    return SC_OK;
}

// local sum of p = w / total_global over candidates (host *psum)
int sc_kmeanspp_psum(sc_kmeanspp_t* s, double total_global, double* psum) {
    SC_CUDA(cudaMemcpyAsync(s->total.p, &total_global, sizeof(double), cudaMemcpyHostToDevice, s->st));
    kpp_psum_kernel<<<(unsigned)s->nb_p, KPP_BLK, 0, s->st>>>(s->n, s->d2.p, s->taken.p, s->total.p, s->bsum.p);
    DevBuf<double> out;
    if (int rc = out.alloc(1)) return rc;
    sum_partials_kernel<<<1, 1024, 0, s->st>>>(s->nb_p, s->bsum.p, out.p);
    SC_LAUNCHED(2);
    SC_CUDA(d2h_sync(psum, out.p, sizeof(double), s->st));
    return SC_OK;
}

// first local candidate whose cumulative p exceeds `target` (after sc_kmeanspp_psum);
// *index = -1 when the crossing is not on this shard
int sc_kmeanspp_search(sc_kmeanspp_t* s, double target, int64_t* index) {
    kpp_search_target_kernel<<<1, 32, 0, s->st>>>(s->n, s->nb_p, s->d2.p, s->taken.p, s->total.p, s->bsum.p, target,
                                                  s->pick.p);
    SC_LAUNCHED(1);
    SC_CUDA(d2h_sync(index, s->pick.p, sizeof(int64_t), s->st));
    return SC_OK;
}

int sc_kmeanspp_nth_free(sc_kmeanspp_t* s, int64_t r, int64_t* index) {
    kpp_nth_free_kernel<<<1, 32, 0, s->st>>>(s->n, s->taken.p, r, s->pick.p);
    SC_LAUNCHED(1);
    SC_CUDA(d2h_sync(index, s->pick.p, sizeof(int64_t), s->st));
    return SC_OK;
}

// ---- per-shard building blocks of point-sharded Lloyd -------------------------------
// labels/cost for the local points; *changes (host) vs old_labels (or -1 when
// old_labels is null), *sse (host) = local sum of costs
int sc_kmeans_assign(int64_t n, int64_t d, int64_t k, const double* v, const double* c, const int64_t* old_labels,
                     int64_t* labels, double* cost, int64_t* changes, double* sse, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    *changes = 0;
    *sse = 0.0;
    if (n <= 0) return SC_OK;
    const int64_t nb = ceil_div(n, TP);
    DevBuf<double> vn, cn, part, out;
    DevBuf<unsigned long long> chg;
    int rc;
    if ((rc = vn.alloc(n)) || (rc = cn.alloc(k)) || (rc = part.alloc(nb)) || (rc = out.alloc(1)) ||
        (rc = chg.alloc(1)))
        return rc;
    SC_CUDA(cudaMemsetAsync(chg.p, 0, sizeof(unsigned long long), st));
    rownorm_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d, v, vn.p);
    rownorm_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(k, d, c, cn.p);
    SC_LAUNCHED(2);
    {
        ProfScope prof("kmeans_assign", st, 2.0 * (double)n * k * d);
        // tensor-core certified argmin when eligible (the shard's rows are
        // converted to fp16 per call: one extra pass over v)
        AssignTc atc;
        if ((rc = atc.init(n, d, k, v, st))) return rc;
        if (atc.active) {
            if ((rc = atc.assign(k, v, vn.p, c, cn.p, old_labels, labels, cost, chg.p, st))) return rc;
            cost_block_sum_kernel<<<(unsigned)ceil_div(nb, 256), 256, 0, st>>>(n, cost, part.p);
        } else {
            dist_tile_kernel<0><<<(unsigned)nb, 256, 0, st>>>(n, k, d, v, vn.p, c, cn.p, nullptr, labels, old_labels,
                                                              cost, chg.p, part.p);
        }
    }
    sum_partials_kernel<<<1, 1024, 0, st>>>(nb, part.p, out.p);
    SC_LAUNCHED(2);
    unsigned long long hc = 0;
    SC_CUDA(d2h_sync(&hc, chg.p, sizeof(hc), st));
    SC_CUDA(d2h_sync(sse, out.p, sizeof(double), st));
    *changes = (int64_t)hc;
    return SC_OK;
}

// unnormalised per-cluster sums of the local points (point order, segmented)
// and counts (dev int64)
int sc_kmeans_local_sums(int64_t n, int64_t d, int64_t k, const double* v, const int64_t* labels, double* sums,
                         int64_t* counts, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    if (n <= 0) {
        SC_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * k * d, st));
        SC_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * k, st));
        return SC_OK;
    }
    Bucketer bk;
    DevBuf<int64_t> seg_off;
    DevBuf<double> segpart;
    int rc;
    if ((rc = bk.init(n, k)) || (rc = seg_off.alloc(k + 1)) ||
        (rc = segpart.alloc((size_t)(n / CM_SEG + k + 1) * d)))
        return rc;
    if ((rc = bk.run(labels, st))) return rc;
    std::vector<int64_t> hstart(k + 1), hseg(k + 1, 0);
    SC_CUDA(d2h_sync(hstart.data(), bk.start.p, sizeof(int64_t) * (k + 1), st));
    for (int64_t c = 0; c < k; ++c) hseg[c + 1] = hseg[c] + ceil_div(hstart[c + 1] - hstart[c], CM_SEG);
    const int64_t nseg = hseg[k];
    SC_CUDA(cudaMemcpyAsync(seg_off.p, hseg.data(), sizeof(int64_t) * (k + 1), cudaMemcpyHostToDevice, st));
    const int64_t dchunks = ceil_div(d, 32);
    if (nseg > 0)
        if (int rc = segsum_smem_attr()) return rc;
        centroid_segsum_smem_kernel<<<(unsigned)(nseg * dchunks), 32, 2 * CS_BATCH * 32 * sizeof(double), st>>>(
            k, d, nseg, v, bk.start.p, bk.members.p, seg_off.p, segpart.p);
    centroid_segtotal_kernel<<<(unsigned)ceil_div(k * d, 256), 256, 0, st>>>(k, d, bk.start.p, seg_off.p, segpart.p,
                                                                            sums, counts);
    SC_LAUNCHED(2);
    SC_CUDA(cudaStreamSynchronize(st));
    return SC_OK;
}

// cent = sums / counts (0 for empty clusters)
int sc_centroid_divide(int64_t k, int64_t d, const double* sums, const int64_t* counts, double* cent,
                       sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    if (k * d <= 0) return SC_OK;
    centroid_divide_kernel<<<(unsigned)ceil_div(k * d, 256), 256, 0, st>>>(k, d, sums, counts, cent);
    SC_LAUNCHED(1);
    return SC_OK;
}

// first e indices of the stable descending order of cost (kmeans.py:151)
int sc_farthest(int64_t n, const double* cost, int64_t e, int64_t* idx_out, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    DevBuf<uint8_t> used;
    DevBuf<double> pv;
    DevBuf<int64_t> pi, pick;
    int rc;
    if ((rc = used.alloc(n)) || (rc = pv.alloc(256)) || (rc = pi.alloc(256)) || (rc = pick.alloc(e > 0 ? e : 1)))
        return rc;
    SC_CUDA(cudaMemsetAsync(used.p, 0, n, st));
    for (int64_t s = 0; s < e && s < n; ++s) {
        argmax_partial_kernel<<<256, 256, 0, st>>>(n, cost, used.p, pv.p, pi.p);
        argmax_finish_kernel<<<1, 32, 0, st>>>(256, pv.p, pi.p, used.p, pick.p + s);
        SC_LAUNCHED(2);
    }
    SC_CUDA(d2h_sync(idx_out, pick.p, sizeof(int64_t) * e, st));
    return SC_OK;
}

// row-sharded ncut partials: rows row_offset.. of W, labels of ALL points;
// per part boundary weight / volume of the local rows and member counts (dev)
int sc_ncut_partials(int64_t n_local, int64_t row_offset, const int64_t* row_ptr, const int32_t* col,
                     const double* vals, const int64_t* labels_global, int64_t k, double* bnd, double* vol,
                     int64_t* counts, sc_stream_t stream) {
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    if (k < 1) return fail(SC_ERR_VALUE, "ncut needs k >= 1");
    if (n_local <= 0) {
        SC_CUDA(cudaMemsetAsync(bnd, 0, sizeof(double) * k, st));
        SC_CUDA(cudaMemsetAsync(vol, 0, sizeof(double) * k, st));
        SC_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * k, st));
        return SC_OK;
    }
    DevBuf<double> deg, cross;
    Bucketer bk;
    int rc;
    if ((rc = deg.alloc(n_local)) || (rc = cross.alloc(n_local)) || (rc = bk.init(n_local, k))) return rc;
    if ((rc = bk.run(labels_global + row_offset, st))) return rc;
    ncut_rows_kernel<<<(unsigned)ceil_div(n_local, 8), 256, 0, st>>>(n_local, row_ptr, col, vals, labels_global,
                                                                     deg.p, cross.p, row_offset);
    ncut_parts_kernel<<<(unsigned)ceil_div(k, 64), 64, 0, st>>>(k, deg.p, cross.p, bk.start.p, bk.members.p, bnd, vol);
    bucket_sizes_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(k, bk.start.p, counts);
    SC_LAUNCHED(3);
    return SC_OK;
}

int sc_ncut(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
            const int64_t* labels, int64_t k, int skip_empty, double* out, int64_t* occupied,
            sc_stream_t stream) {
    *out = -1.0;
    if (n < 1 || k < 1) return fail(SC_ERR_VALUE, "ncut needs n >= 1 and k >= 1");
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    DevBuf<double> deg, cross, bnd, vol;
    Bucketer bk;
    int rc;
    if ((rc = deg.alloc(n)) || (rc = cross.alloc(n)) || (rc = bnd.alloc(k)) || (rc = vol.alloc(k)) ||
        (rc = bk.init(n, k)))
        return rc;
    ProfScope prof("ncut", st, 0.0);
    if ((rc = bk.run(labels, st))) return rc;
    ncut_rows_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, col, vals, labels, deg.p, cross.p);
    ncut_parts_kernel<<<(unsigned)ceil_div(k, 64), 64, 0, st>>>(k, deg.p, cross.p, bk.start.p, bk.members.p, bnd.p,
                                                                 vol.p);
    SC_LAUNCHED(2);
    std::vector<double> hb(k), hv(k);
    std::vector<int64_t> hs(k + 1);
    SC_CUDA(d2h_sync(hb.data(), bnd.p, sizeof(double) * k, st));
    SC_CUDA(d2h_sync(hv.data(), vol.p, sizeof(double) * k, st));
    SC_CUDA(d2h_sync(hs.data(), bk.start.p, sizeof(int64_t) * (k + 1), st));
    // parts in label order; empty parts are dropped when compacting (the
    // pipeline's np.unique relabelling, pipeline.py:256-257)
    std::vector<double> q;
    q.reserve(k);
    for (int64_t c = 0; c < k; ++c) {
        const bool empty = hs[c + 1] == hs[c];
        if (empty && skip_empty) continue;
        if (!(hv[c] > 0.0)) return fail(SC_ERR_VALUE, "part " + std::to_string(c) + " has zero volume");
        q.push_back(hb[c] / hv[c]);
    }
    if (occupied) *occupied = (int64_t)q.size();
    *out = 0.5 * np_pairwise_sum(q.data(), (int64_t)q.size());
    return SC_OK;
}

// cut and ratio_cut (metrics.py:34-56): per-row crossing weights, per-part
// boundary sums in member order, sizes from the label buckets.
// cut = 1/2 sum_i cross_i; ratio_cut = 1/2 sum_c bnd_c / size_c (numpy's
// pairwise order over parts).  *empty_part = first empty part (ratio_cut's
// EmptyPart) or -1.
int sc_partition_cuts(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                      const int64_t* labels, int64_t k, double* cut_out, double* ratio_out, int64_t* empty_part,
                      sc_stream_t stream) {
    if (n < 1 || k < 1) return fail(SC_ERR_VALUE, "cut metrics need n >= 1 and k >= 1");
    cudaStream_t st = as_stream(stream);
    StreamScope stream_scope(st);
    DevBuf<double> deg, cross, bnd, vol, tot;
    Bucketer bk;
    int rc;
    if ((rc = deg.alloc(n)) || (rc = cross.alloc(n)) || (rc = bnd.alloc(k)) || (rc = vol.alloc(k)) ||
        (rc = tot.alloc(1)) || (rc = bk.init(n, k)))
        return rc;
    if ((rc = bk.run(labels, st))) return rc;
    ncut_rows_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, row_ptr, col, vals, labels, deg.p, cross.p);
    ncut_parts_kernel<<<(unsigned)ceil_div(k, 64), 64, 0, st>>>(k, deg.p, cross.p, bk.start.p, bk.members.p, bnd.p,
                                                                 vol.p);
    sum_partials_kernel<<<1, 1024, 0, st>>>(n, cross.p, tot.p);
    SC_LAUNCHED(3);
    std::vector<double> hb(k);
    std::vector<int64_t> hs(k + 1);
    double htot = 0.0;
    SC_CUDA(d2h_sync(hb.data(), bnd.p, sizeof(double) * k, st));
    SC_CUDA(d2h_sync(hs.data(), bk.start.p, sizeof(int64_t) * (k + 1), st));
    SC_CUDA(d2h_sync(&htot, tot.p, sizeof(double), st));
    *cut_out = 0.5 * htot;
    *empty_part = -1;
    std::vector<double> q(k);
    for (int64_t c = 0; c < k; ++c) {
        const int64_t size = hs[c + 1] - hs[c];
        if (size == 0) {
            if (*empty_part < 0) *empty_part = c;
            q[c] = 0.0;
        } else {
            q[c] = hb[c] / (double)size;
        }
    }
    *ratio_out = *empty_part >= 0 ? -1.0 : 0.5 * np_pairwise_sum(q.data(), k);
    return SC_OK;
}

}  // extern "C"


