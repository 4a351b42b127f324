// kNN candidate generation on the 5th-generation tensor cores.
//
// One CTA owns 128 query rows and streams every candidate tile of 128 rows:
//   warp 0     TMA producer: query tile once, candidate tiles through a ring
//   warp 1     TMEM allocation + single-thread tcgen05.mma issuer
//              (M=128, N=128, K=16 per instruction, fp16 in / fp32 out)
//   warps 2-5  epilogue: thread <-> query row (TMEM lane); tcgen05.ld of the
//              accumulator, key = |x_j|^2 - 2 x_i.x_j, min-of-16 filter against
//              the row's running threshold, rare appends to the row's list
// Two TMEM accumulators (2 x 128 columns) let the MMA of tile t+1 overlap the
// epilogue of tile t.  Operands are K-major fp16 in 128-byte swizzled rows,
// staged by TMA (SWIZZLE_128B) and described to UMMA with matching
// descriptors.
//
// Candidate lists: each row appends (key, column) pairs with key < tau into
// a list of `cap` slots; a list that could overflow is compacted by the
// whole warp (bitonic sort of the row's list in shared memory, keep the R
// smallest, tau = R-th key), so compaction never serialises 32 divergent
// lanes.  For d <= 64 the lists live in shared memory for the whole scan;
// wider rows keep them in global memory and sort through a per-warp scratch.
#pragma once
#include <cuda_fp16.h>

#include "sc_tc.cuh"

namespace sc {

constexpr int TC_THREADS = 192;
constexpr uint32_t TC_TILE_BYTES = 128 * 128;  // 128 rows x 64 fp16
constexpr int TC_LIST_P = 128;                 // sort width (power of two >= cap)

template <int NKB, int STAGES, bool LSMEM>
struct TcLayout {
    static constexpr uint32_t kA = NKB * TC_TILE_BYTES;
    static constexpr uint32_t kB = NKB * TC_TILE_BYTES;
    // lists: 128 rows x P slots (smem-resident) or 4 warps x P scratch
    static constexpr uint32_t kL = (LSMEM ? 128 : 4) * TC_LIST_P * 8;
    static constexpr uint32_t kCn = 2 * 128 * 4;  // column norms of the two in-flight tiles
    static constexpr uint32_t kBar = 8 * (2 * STAGES + 5) + 8;
    static constexpr uint32_t total = 1024 + kA + STAGES * kB + kL + kCn + kBar;
};

// warp-cooperative: sort S[0..P) ascending by key (entries >= cnt are +inf)
__device__ __forceinline__ void warp_bitonic_sort(float2* S, int lane) {
#pragma unroll 1
    for (int k = 2; k <= TC_LIST_P; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int t = 0; t < TC_LIST_P / 64; ++t) {
                // pair index p in [0, P/2): element i = ((p & ~(j-1)) << 1) | (p & (j-1)), partner i + j
                int p = lane + 32 * t;
                int i = ((p & ~(j - 1)) << 1) | (p & (j - 1));
                int q = i + j;
                float2 a = S[i], b = S[q];
                bool up = (i & k) == 0;
                bool swap = up ? (a.x > b.x) : (a.x < b.x);
                if (swap) {
                    S[i] = b;
                    S[q] = a;
                }
            }
            __syncwarp();
        }
    }
}

template <int NKB, int STAGES, bool LSMEM>
__global__ void __launch_bounds__(TC_THREADS, LSMEM ? 1 : 2)
    knn_cand_tc_kernel(const __grid_constant__ CUtensorMap xmap, int64_t n, int64_t ntiles, int64_t qtile0,
                       const float* __restrict__ cnk, float key_scale, int cap, int R, float2* __restrict__ lists,
                       int* __restrict__ counts, float* __restrict__ taus, long long* __restrict__ dbg) {
    using Lay = TcLayout<NKB, STAGES, LSMEM>;
    long long d_wait0 = 0, d_wait1 = 0, d_work = 0, d_fast = 0, d_t0 = clock64();
    long long n_fire = 0, n_app = 0, n_comp = 0, n_quart = 0;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;
    uint8_t* sB = base + Lay::kA;
    float2* sL = reinterpret_cast<float2*>(sB + STAGES * Lay::kB);
    float* sCn = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sL) + Lay::kL);  // [2][128]
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sCn) + Lay::kCn);
    uint64_t* empty = full + STAGES;
    uint64_t* afull = empty + STAGES;
    uint64_t* tfull = afull + 1;   // [2]
    uint64_t* tempty = tfull + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // query tile qt (scan positions row0..row0+127); lists/counts/taus are
    // indexed by position relative to the first query tile of the launch
    const int64_t qt = qtile0 + blockIdx.x;
    const int64_t row0 = qt * 128;
    const int64_t lrow0 = (int64_t)blockIdx.x * 128;

    if (warp == 0 && lane == 0) tc::tma_prefetch(&xmap);
    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s) {
                tc::mbar_init(&full[s], 1);
                tc::mbar_init(&empty[s], 1);
            }
            tc::mbar_init(afull, 1);
            for (int b = 0; b < 2; ++b) {
                // two arrivals per use: the column-norm bulk copy (expect_tx) and the MMA commit
                tc::mbar_init(&tfull[b], 2);
                tc::mbar_init(&tempty[b], 4);
            }
            tc::fence_mbar_init();
        }
        __syncwarp();
        tc::tmem_alloc(tmem_slot, 256);
    }
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            tc::mbar_expect_tx(afull, Lay::kA);
            for (int kb = 0; kb < NKB; ++kb) tc::tma_load_2d(sA + kb * TC_TILE_BYTES, &xmap, afull, kb * 64, (int)row0);
            for (int64_t t = 0; t < ntiles; ++t) {
                const int s = (int)(t % STAGES);
                const uint32_t ph = (uint32_t)((t / STAGES) & 1);
                long long c0 = clock64();
                tc::mbar_wait(&empty[s], ph ^ 1);
                d_wait0 += clock64() - c0;
                tc::mbar_expect_tx(&full[s], Lay::kB);
                for (int kb = 0; kb < NKB; ++kb)
                    tc::tma_load_2d(sB + s * Lay::kB + kb * TC_TILE_BYTES, &xmap, &full[s], kb * 64,
                                    (int)(((qt + t) % ntiles) * 128));
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_f16_f32(128, 128);
            tc::mbar_wait(afull, 0);
            for (int64_t t = 0; t < ntiles; ++t) {
                const int s = (int)(t % STAGES);
                const uint32_t ph = (uint32_t)((t / STAGES) & 1);
                const int buf = (int)(t & 1);
                const uint32_t bph = (uint32_t)((t >> 1) & 1);
                long long c0 = clock64();
                tc::mbar_wait(&tempty[buf], bph ^ 1);
                long long c1 = clock64();
                tc::mbar_wait(&full[s], ph);
                long long c2 = clock64();
                d_wait0 += c1 - c0;
                d_wait1 += c2 - c1;
                // the accumulator slot is free, so is its column-norm slot
                tc::mbar_expect_tx(&tfull[buf], 128 * 4);
                tc::bulk_g2s(sCn + buf * 128, cnk + ((qt + t) % ntiles) * 128, 128 * 4, &tfull[buf]);
                tc::fence_after();
#pragma unroll
                for (int kb = 0; kb < NKB; ++kb) {
                    const uint64_t ad = tc::desc_k_sw128(sA + kb * TC_TILE_BYTES);
                    const uint64_t bd = tc::desc_k_sw128(sB + s * Lay::kB + kb * TC_TILE_BYTES);
#pragma unroll
                    for (int k = 0; k < 4; ++k)  // 4 x K=16 per 64-element swizzle row (32 B steps)
                        tc::umma_f16(tmem + buf * 128, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                }
                tc::umma_commit(&empty[s]);
                tc::umma_commit(&tfull[buf]);
                if (dbg && t < 64) {  // debug: raw MMA completion latency (first tiles)
                    long long c3 = clock64();
                    tc::mbar_wait(&tfull[buf], bph);
                    d_work += clock64() - c3;
                }
            }
        }
    } else {
        const int quad = warp & 3;
        const int lrow = quad * 32 + lane;
        const int64_t row = row0 + lrow;
        const bool valid = row < n;
        // list of this row: smem-resident or global (with a per-warp smem scratch)
        float2* L = LSMEM ? sL + (size_t)lrow * TC_LIST_P : lists + (valid ? lrow0 + lrow : 0) * (int64_t)cap;
        float2* scratch = LSMEM ? nullptr : sL + (size_t)quad * TC_LIST_P;
        int cnt = 0;
        float tau = INFINITY;
        for (int64_t t = 0; t < ntiles; ++t) {
            const int buf = (int)(t & 1);
            const uint32_t bph = (uint32_t)((t >> 1) & 1);
            long long c0 = clock64();
            tc::mbar_wait(&tfull[buf], bph);
            long long c1 = clock64();
            d_wait0 += c1 - c0;
            tc::fence_after();
            // scan order: the query tile's own (locality-sorted) neighbourhood first
            const int64_t col0 = ((qt + t) % ntiles) * 128;
            const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * 128);
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
                float v[64];
                const long long h0 = clock64();
                tc::tmem_ld64(taddr + half * 64, v);
                tc::tmem_wait_ld();
                const long long h1 = clock64();
                d_wait1 += h1 - h0;
                const float4* cp = reinterpret_cast<const float4*>(sCn + buf * 128 + half * 64);
                float m0 = INFINITY, m1 = INFINITY;
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const float4 cn4 = cp[u];  // smem broadcast
                    v[4 * u + 0] = fmaf(key_scale, v[4 * u + 0], cn4.x);
                    v[4 * u + 1] = fmaf(key_scale, v[4 * u + 1], cn4.y);
                    v[4 * u + 2] = fmaf(key_scale, v[4 * u + 2], cn4.z);
                    v[4 * u + 3] = fmaf(key_scale, v[4 * u + 3], cn4.w);
                    m0 = fminf(m0, fminf(v[4 * u + 0], v[4 * u + 1]));
                    m1 = fminf(m1, fminf(v[4 * u + 2], v[4 * u + 3]));
                }
                // steady state: no row of the warp improves -> one vote per 64 columns
                const bool any = __any_sync(0xffffffffu, valid && fminf(m0, m1) < tau);
                d_fast += clock64() - h1;
                if (!any) continue;
                ++n_fire;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int c = half * 64 + q * 16;
                    const float* keys = v + q * 16;
                    float m = INFINITY;
#pragma unroll
                    for (int u = 0; u < 16; ++u) m = fminf(m, keys[u]);
                    const bool pass = valid && m < tau;
                    // make room: warp-cooperative compaction of every list
                    // that could overflow while taking this chunk
                    unsigned want = __ballot_sync(0xffffffffu, pass && cnt > cap - 16);
                    n_quart += __any_sync(0xffffffffu, pass);
                    n_comp += __popc(want);
                    while (want) {
                        __syncwarp();  // make lane src's appends visible
                        const int src = __ffs(want) - 1;
                        want &= want - 1;
                        const int c_src = __shfl_sync(0xffffffffu, cnt, src);
                        float2* Ls = LSMEM ? sL + (size_t)(quad * 32 + src) * TC_LIST_P : scratch;
                        const float2* Lg = lists + (lrow0 + quad * 32 + src) * (int64_t)cap;
                        for (int e = lane; e < TC_LIST_P; e += 32) {
                            float2 val = make_float2(INFINITY, __int_as_float(-1));
                            if (e < c_src) val = LSMEM ? Ls[e] : Lg[e];
                            Ls[e] = val;
                        }
                        __syncwarp();
                        warp_bitonic_sort(Ls, lane);
                        if (!LSMEM) {
                            float2* Lw = lists + (lrow0 + quad * 32 + src) * (int64_t)cap;
                            for (int e = lane; e < R; e += 32) Lw[e] = Ls[e];
                        }
                        const float new_tau = Ls[R - 1].x;
                        __syncwarp();
                        if (lane == src) {
                            cnt = R;
                            tau = new_tau;
                        }
                    }
                    if (pass) {
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const int64_t col = col0 + c + u;
                            if (keys[u] < tau && col != row && col < n) {
                                L[cnt++] = make_float2(keys[u], __int_as_float((int)col));
                                ++n_app;
                            }
                        }
                    }
                }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[buf]);
            d_work += clock64() - c1;
        }
        if (valid) {
            if (LSMEM) {
                float2* Lg = lists + (lrow0 + lrow) * (int64_t)cap;
                for (int e = 0; e < cnt; ++e) Lg[e] = L[e];
            }
            counts[lrow0 + lrow] = cnt;
            taus[lrow0 + lrow] = tau;
        }
    }
    if (dbg && lane == 0 && warp < 3) {
        long long* o = dbg + (size_t)blockIdx.x * 16 + warp * 4;
        o[0] = d_wait0;
        o[1] = d_wait1;
        o[2] = d_work;
        o[3] = warp == 2 ? d_fast : clock64() - d_t0;
    }
    if (dbg && warp == 2) {
        const long long a = warp_sum_i64(n_app);
        if (lane == 0) {
            long long* o = dbg + (size_t)blockIdx.x * 16;
            o[12] = n_fire;
            o[13] = a;
            o[14] = n_comp;
            o[15] = n_quart;
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, 256);
    }
}

// fp16 operand prep: xh = fp16(scale * (x - mean)) padded to (n_pad x dp);
// cnk = |xh|^2 / scale^2 (fp64 sum of the fp16 values, +inf on padding rows);
// qn = same in fp64 for query rows.
// Rows are written in scan order: position i holds original point perm[i]
// (perm == nullptr: identity); qn is indexed by the original point.
static __global__ void knn_prep_f16_kernel(int64_t n, int64_t n_pad, int64_t d, int64_t dp, const double* __restrict__ x,
                                    const double* __restrict__ mean, double scale, const int32_t* __restrict__ perm,
                                    __half* __restrict__ xh, float* __restrict__ cnk, double* __restrict__ qn) {
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (i >= n_pad) return;
    const int64_t src = (i < n && perm) ? (int64_t)perm[i] : i;
    double acc = 0.0;
    for (int64_t c = lane; c < dp; c += 32) {
        __half h = __float2half_rn(0.f);
        if (i < n && c < d) h = __double2half((x[src * d + c] - mean[c]) * scale);
        xh[i * dp + c] = h;
        double hv = (double)__half2float(h);
        acc = fma(hv, hv, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
        double inv_s2 = 1.0 / (scale * scale);
        if (i < n) {
            cnk[i] = (float)(acc * inv_s2);
            qn[src] = acc * inv_s2;
        } else {
            cnk[i] = INFINITY;
        }
    }
}

// fp64 centred row norms and their maximum (pass 1 of the prep)
static __global__ void knn_rownorm_kernel(int64_t n, int64_t d, const double* __restrict__ x, const double* __restrict__ mean,
                                   double* __restrict__ rn, unsigned long long* __restrict__ rmax_bits) {
    int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    double a = 0.0;
    for (int64_t c = lane; c < d; c += 32) {
        double v = x[i * d + c] - mean[c];
        a = fma(v, v, a);
    }
    a = warp_sum(a);
    if (lane == 0) {
        double r = sqrt(a);
        rn[i] = r;
        atomicMax(rmax_bits, (unsigned long long)__double_as_longlong(r));
    }
}

}  // namespace sc
