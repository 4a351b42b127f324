// k-means assignment on the 5th-generation tensor cores: certified argmin.
//
// The reference assigns every point to argmin_c S(v, c) with
// S = (|v|^2 + |c|^2) - 2 einsum(v, c) in fp64, clamped at 0, ties to the
// lowest index (kmeans.py:84-98, 175, 182).  Here the n x k cross term is a
// tcgen05 GEMM on fp16 operands (fp32 accumulate) and every row keeps only
// (best key, its centroid, second-best key) of key_c = |c|^2 - 2 v.c.  A
// row whose second-best approximate key exceeds the best by more than twice
// the rounding bound delta(|v|, max|c|) has a certified, unique exact argmin;
// its label is final and only its exact fp64 cost is recomputed (one dot
// product in numpy's summation order).  The rest (near ties, exact
// duplicates, clamp cases) are re-scanned exactly over all centroids.
//
// Every row also keeps its third-best key and centroid and the fourth-best
// key: a row that misses the certificate but has at most three candidates
// within 2 delta of its best (a point between two or three centroids of a
// split cluster) is settled by exact fp64 keys of those candidates alone
// (as_resolve_kernel); only the rest are re-scanned.
//
// Layout: CTA = QT point tiles of 128 rows (A, loaded once by TMA) against
// the centroid tiles (B, a STAGES-deep TMA ring of 64-column K chunks, so two
// resident point tiles fit next to it at d = 256 and every centroid chunk
// read from L2 feeds M = 256 rows of MMA); a single thread issues the
// M=128 x N=128 x K=16 fp16 MMAs into QT x 2 TMEM accumulators; 4*QT
// epilogue warps (thread <-> point row, TMEM lane quarter warp % 4) turn a
// tile into keys with packed f32x2 FMAs against the centroid norms (their
// own ring) and take 16-column minima; only a quarter whose minimum beats the
// row's second-best is walked element by element.
#pragma once
#include <cuda_fp16.h>

#include "sc_knn_tc2.cuh"
#include "sc_tc.cuh"

namespace sc {

constexpr int AS_CN_RING = 8;

// best three approximate keys (and centroids) of a row plus the fourth-best
// key; a key equal to a kept one goes behind it
struct AsTop3 {
    float b1 = INFINITY, b2 = INFINITY, b3 = INFINITY, b4 = INFINITY;
    int32_t i1 = -1, i2 = -1, i3 = -1;
    __device__ __forceinline__ void push(float k, int32_t j) {
        if (k < b2) {
            b4 = b3;
            b3 = b2;
            i3 = i2;
            if (k < b1) {
                b2 = b1;
                i2 = i1;
                b1 = k;
                i1 = j;
            } else {
                b2 = k;
                i2 = j;
            }
        } else if (k < b3) {
            b4 = b3;
            b3 = k;
            i3 = j;
        } else if (k < b4) {
            b4 = k;
        }
    }
    __device__ __forceinline__ void store(int64_t row, int32_t* best_idx, float2* best_keys, int2* alt_idx,
                                          float2* alt_keys) const {
        best_idx[row] = i1;
        best_keys[row] = make_float2(b1, b2);
        alt_idx[row] = make_int2(i2, i3);
        alt_keys[row] = make_float2(b3, b4);
    }
};

// One 16-column quarter whose minimum beat the row's fourth-best key: the
// columns below it as a bit mask (compares on the registers), then only
// those are pushed, read back from the thread's stage slots (layout
// [4][32 lanes] float4 per warp: conflict-free stores).
__device__ __forceinline__ void as_walk_quarter(AsTop3& top, const float* e, uint32_t stage, int32_t cb) {
    uint32_t mask = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) mask |= (e[u] < top.b4 ? 1u : 0u) << u;
    if (!mask) return;
#pragma unroll
    for (int u4 = 0; u4 < 4; ++u4)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stage + u4 * 512), "f"(e[4 * u4]),
                     "f"(e[4 * u4 + 1]), "f"(e[4 * u4 + 2]), "f"(e[4 * u4 + 3])
                     : "memory");
    while (mask) {
        const int u = __ffs(mask) - 1;
        mask &= mask - 1;
        float k;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(k) : "r"(stage + (uint32_t)((u >> 2) * 512 + (u & 3) * 4)));
        if (k < top.b4) top.push(k, cb + u);
    }
}

template <int NKB, int STAGES, int QT>
struct AsLayout {
    static constexpr uint32_t kA = QT * NKB * TC_TILE_BYTES;
    static constexpr uint32_t kB = TC_TILE_BYTES;  // one 128 x 64 centroid chunk per stage
    static constexpr uint32_t kStage = QT * 4 * 32 * 16 * 4;  // 16 staged keys per epilogue thread
    static constexpr uint32_t kCn = AS_CN_RING * 128 * 4;
    static constexpr uint32_t kBar = 8 * (2 * STAGES + 5 + 2 * AS_CN_RING) + 8;
    static constexpr uint32_t total = 1024 + kA + STAGES * kB + kStage + kCn + kBar;
};

template <int NKB, int STAGES, int QT>
__global__ void __launch_bounds__(64 + QT * 128, 1)
    assign_tc_kernel(const __grid_constant__ CUtensorMap vmap, const __grid_constant__ CUtensorMap cmap, int64_t n,
                     int64_t nptiles, int64_t nctiles, const float* __restrict__ cnk, float key_scale,
                     int32_t* __restrict__ best_idx, float2* __restrict__ best_keys, int2* __restrict__ alt_idx,
                     float2* __restrict__ alt_keys) {
    using Lay = AsLayout<NKB, STAGES, QT>;
    constexpr int NEPI = 4 * QT;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;
    uint8_t* sB = base + Lay::kA;
    float* sStage = reinterpret_cast<float*>(sB + STAGES * Lay::kB);
    float* sCn = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sStage) + Lay::kStage);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sCn) + Lay::kCn);
    uint64_t* empty = full + STAGES;
    uint64_t* afull = empty + STAGES;
    uint64_t* tfull = afull + 1;
    uint64_t* tempty = tfull + 2;
    uint64_t* cfull = tempty + 2;
    uint64_t* cempty = cfull + AS_CN_RING;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + AS_CN_RING);
    constexpr uint32_t kTmemCols = QT * 256;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t pt0 = (int64_t)blockIdx.x * QT;

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&vmap);
        tc::tma_prefetch(&cmap);
    }
    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s) {
                tc::mbar_init(&full[s], 1);
                tc::mbar_init(&empty[s], 1);
            }
            tc::mbar_init(afull, 1);
            for (int b = 0; b < 2; ++b) {
                tc::mbar_init(&tfull[b], 1);
                tc::mbar_init(&tempty[b], NEPI);
            }
            for (int c = 0; c < AS_CN_RING; ++c) {
                tc::mbar_init(&cfull[c], 1);
                tc::mbar_init(&cempty[c], NEPI);
            }
            tc::fence_mbar_init();
        }
        __syncwarp();
        tc::tmem_alloc(tmem_slot, kTmemCols);
    }
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            tc::mbar_expect_tx(afull, Lay::kA);
            for (int q = 0; q < QT; ++q)
                for (int kb = 0; kb < NKB; ++kb)
                    tc::tma_load_2d(sA + (q * NKB + kb) * TC_TILE_BYTES, &vmap, afull, kb * 64, (int)((pt0 + q) * 128));
            int64_t it = 0;
            for (int64_t t = 0; t < nctiles; ++t) {
                const int c = (int)(t % AS_CN_RING);
                mbar_wait_hw<true>(&cempty[c], (uint32_t)(((t / AS_CN_RING) & 1) ^ 1));
                tc::mbar_expect_tx(&cfull[c], 128 * 4);
                tc::bulk_g2s(sCn + c * 128, cnk + t * 128, 128 * 4, &cfull[c]);
                for (int kb = 0; kb < NKB; ++kb, ++it) {
                    const int s = (int)(it % STAGES);
                    mbar_wait_hw<true>(&empty[s], (uint32_t)(((it / STAGES) & 1) ^ 1));
                    tc::mbar_expect_tx(&full[s], Lay::kB);
                    tc::tma_load_2d(sB + s * Lay::kB, &cmap, &full[s], kb * 64, (int)(t * 128));
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_f16_f32(128, 128);
            mbar_wait_hw<true>(afull, 0);
            int64_t it = 0;
            for (int64_t t = 0; t < nctiles; ++t) {
                const int buf = (int)(t & 1);
                mbar_wait_hw<true>(&tempty[buf], (uint32_t)(((t >> 1) & 1) ^ 1));
                tc::fence_after();
#pragma unroll
                for (int kb = 0; kb < NKB; ++kb, ++it) {
                    const int s = (int)(it % STAGES);
                    mbar_wait_hw<true>(&full[s], (uint32_t)((it / STAGES) & 1));
                    tc::fence_after();
                    const uint64_t bd = tc::desc_k_sw128(sB + s * Lay::kB);
#pragma unroll
                    for (int q = 0; q < QT; ++q) {
                        const uint64_t ad = tc::desc_k_sw128(sA + (q * NKB + kb) * TC_TILE_BYTES);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc::umma_f16(tmem + buf * (QT * 128) + q * 128, ad + 2 * k, bd + 2 * k, idesc,
                                         (kb | k) != 0);
                    }
                    tc::umma_commit(&empty[s]);
                }
                tc::umma_commit(&tfull[buf]);
            }
        }
    } else {
        const int quad = warp & 3;
        const int qi = (warp - 2) >> 2;
        const int64_t row = (pt0 + qi) * 128 + quad * 32 + lane;
        const bool valid = pt0 + qi < nptiles && row < n;
        const uint32_t stage = tc::smem_u32(sStage + (size_t)(warp - 2) * 512) + (uint32_t)lane * 16;
        AsTop3 top;
        const float2 ks = make_float2(key_scale, key_scale);
        for (int64_t t = 0; t < nctiles; ++t) {
            const int buf = (int)(t & 1);
            const int cslot = (int)(t % AS_CN_RING);
            mbar_wait_hw<true>(&cfull[cslot], (uint32_t)((t / AS_CN_RING) & 1));
            mbar_wait_hw<true>(&tfull[buf], (uint32_t)((t >> 1) & 1));
            tc::fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * (QT * 128) + qi * 128);
            float v[128];
            tc::tmem_ld64(taddr, v);
            tc::tmem_ld64(taddr + 64, v + 64);
            tc::tmem_wait_ld();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[buf]);
            const uint32_t cn_s = tc::smem_u32(sCn + cslot * 128);
            float qm[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float m = INFINITY;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float4 cn4 = lds_f4(cn_s + (uint32_t)(16 * (4 * q + u)));
                    float* e = v + 16 * q + 4 * u;
                    const float2 k01 = ffma2(ks, make_float2(e[0], e[1]), make_float2(cn4.x, cn4.y));
                    const float2 k23 = ffma2(ks, make_float2(e[2], e[3]), make_float2(cn4.z, cn4.w));
                    e[0] = k01.x;
                    e[1] = k01.y;
                    e[2] = k23.x;
                    e[3] = k23.y;
                    m = fmin3(m, fmin3(k01.x, k01.y, k23.x), k23.y);
                }
                qm[q] = m;
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&cempty[cslot]);
            // padded centroid columns carry +inf norms, so they never win
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (!(valid && qm[q] < top.b4)) continue;
                as_walk_quarter(top, v + 16 * q, stage, (int32_t)(t * 128 + q * 16));
            }
        }
        if (valid) top.store(row, best_idx, best_keys, alt_idx, alt_keys);
    }
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, kTmemCols);
    }
}

// Wide embeddings (dp > 256, e.g. C3's d = k = 1000): a 128-row point tile
// no longer fits shared memory next to a centroid ring, so both operands
// stream through the ring in 64-column K chunks.  Stage = QT point chunks +
// one centroid chunk (QT+1 TMA boxes of 128 x 64 fp16); the MMA thread runs
// the K loop of a centroid tile into one of two TMEM accumulator sets and
// commits it to the epilogue, which is the same key / (best, second-best)
// pass as assign_tc_kernel.  The point chunks are re-read (from L2) once per
// centroid tile; QT point tiles share every centroid chunk.
template <int STAGES, int QT>
struct AsKlLayout {
    static constexpr uint32_t kStageBytes = (QT + 1) * TC_TILE_BYTES;
    static constexpr uint32_t kStage = QT * 4 * 32 * 16 * 4;
    static constexpr uint32_t kCn = AS_CN_RING * 128 * 4;
    static constexpr uint32_t kBar = 8 * (2 * STAGES + 4 + 2 * AS_CN_RING) + 8;
    static constexpr uint32_t total = 1024 + STAGES * kStageBytes + kStage + kCn + kBar;
};

template <int STAGES, int QT>
__global__ void __launch_bounds__(64 + QT * 128, 1)
    assign_tc_kl_kernel(const __grid_constant__ CUtensorMap vmap, const __grid_constant__ CUtensorMap cmap, int64_t n,
                        int64_t nptiles, int64_t nctiles, int nkb, const float* __restrict__ cnk, float key_scale,
                        int32_t* __restrict__ best_idx, float2* __restrict__ best_keys, int2* __restrict__ alt_idx,
                        float2* __restrict__ alt_keys) {
    using Lay = AsKlLayout<STAGES, QT>;
    constexpr int NEPI = 4 * QT;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sRing = base;
    float* sStage = reinterpret_cast<float*>(sRing + STAGES * Lay::kStageBytes);
    float* sCn = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sStage) + Lay::kStage);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sCn) + Lay::kCn);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* cfull = tempty + 2;
    uint64_t* cempty = cfull + AS_CN_RING;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + AS_CN_RING);
    constexpr uint32_t kTmemCols = QT * 256;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t pt0 = (int64_t)blockIdx.x * QT;
    const int nq = (int)(nptiles - pt0 < QT ? nptiles - pt0 : QT);  // point tiles this CTA owns

    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&vmap);
        tc::tma_prefetch(&cmap);
    }
    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s) {
                tc::mbar_init(&full[s], 1);
                tc::mbar_init(&empty[s], 1);
            }
            for (int b = 0; b < 2; ++b) {
                tc::mbar_init(&tfull[b], 1);
                tc::mbar_init(&tempty[b], NEPI);
            }
            for (int c = 0; c < AS_CN_RING; ++c) {
                tc::mbar_init(&cfull[c], 1);
                tc::mbar_init(&cempty[c], NEPI);
            }
            tc::fence_mbar_init();
        }
        __syncwarp();
        tc::tmem_alloc(tmem_slot, kTmemCols);
    }
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int64_t it = 0;
            for (int64_t t = 0; t < nctiles; ++t) {
                const int c = (int)(t % AS_CN_RING);
                mbar_wait_hw<true>(&cempty[c], (uint32_t)(((t / AS_CN_RING) & 1) ^ 1));
                tc::mbar_expect_tx(&cfull[c], 128 * 4);
                tc::bulk_g2s(sCn + c * 128, cnk + t * 128, 128 * 4, &cfull[c]);
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = (int)(it % STAGES);
                    mbar_wait_hw<true>(&empty[s], (uint32_t)(((it / STAGES) & 1) ^ 1));
                    uint8_t* st = sRing + s * Lay::kStageBytes;
                    tc::mbar_expect_tx(&full[s], (uint32_t)(nq + 1) * TC_TILE_BYTES);
                    for (int q = 0; q < nq; ++q)
                        tc::tma_load_2d(st + q * TC_TILE_BYTES, &vmap, &full[s], kb * 64, (int)((pt0 + q) * 128));
                    tc::tma_load_2d(st + QT * TC_TILE_BYTES, &cmap, &full[s], kb * 64, (int)(t * 128));
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_f16_f32(128, 128);
            int64_t it = 0;
            for (int64_t t = 0; t < nctiles; ++t) {
                const int buf = (int)(t & 1);
                mbar_wait_hw<true>(&tempty[buf], (uint32_t)(((t >> 1) & 1) ^ 1));
                tc::fence_after();
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const int s = (int)(it % STAGES);
                    mbar_wait_hw<true>(&full[s], (uint32_t)((it / STAGES) & 1));
                    tc::fence_after();
                    uint8_t* st = sRing + s * Lay::kStageBytes;
                    const uint64_t bd = tc::desc_k_sw128(st + QT * TC_TILE_BYTES);
#pragma unroll
                    for (int q = 0; q < QT; ++q) {
                        if (q >= nq) break;
                        const uint64_t ad = tc::desc_k_sw128(st + q * TC_TILE_BYTES);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc::umma_f16(tmem + buf * (QT * 128) + q * 128, ad + 2 * k, bd + 2 * k, idesc,
                                         (kb | k) != 0);
                    }
                    tc::umma_commit(&empty[s]);
                }
                tc::umma_commit(&tfull[buf]);
            }
        }
    } else {
        const int quad = warp & 3;
        const int qi = (warp - 2) >> 2;
        const int64_t row = (pt0 + qi) * 128 + quad * 32 + lane;
        const bool valid = qi < nq && row < n;
        const uint32_t stage = tc::smem_u32(sStage + (size_t)(warp - 2) * 512) + (uint32_t)lane * 16;
        AsTop3 top;
        const float2 ks = make_float2(key_scale, key_scale);
        for (int64_t t = 0; t < nctiles; ++t) {
            const int buf = (int)(t & 1);
            const int cslot = (int)(t % AS_CN_RING);
            mbar_wait_hw<true>(&cfull[cslot], (uint32_t)((t / AS_CN_RING) & 1));
            mbar_wait_hw<true>(&tfull[buf], (uint32_t)((t >> 1) & 1));
            tc::fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * (QT * 128) + qi * 128);
            float v[128];
            tc::tmem_ld64(taddr, v);
            tc::tmem_ld64(taddr + 64, v + 64);
            tc::tmem_wait_ld();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[buf]);
            const uint32_t cn_s = tc::smem_u32(sCn + cslot * 128);
            float qm[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float m = INFINITY;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float4 cn4 = lds_f4(cn_s + (uint32_t)(16 * (4 * q + u)));
                    float* e = v + 16 * q + 4 * u;
                    const float2 k01 = ffma2(ks, make_float2(e[0], e[1]), make_float2(cn4.x, cn4.y));
                    const float2 k23 = ffma2(ks, make_float2(e[2], e[3]), make_float2(cn4.z, cn4.w));
                    e[0] = k01.x;
                    e[1] = k01.y;
                    e[2] = k23.x;
                    e[3] = k23.y;
                    m = fmin3(m, fmin3(k01.x, k01.y, k23.x), k23.y);
                }
                qm[q] = m;
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&cempty[cslot]);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (!(valid && qm[q] < top.b4)) continue;
                as_walk_quarter(top, v + 16 * q, stage, (int32_t)(t * 128 + q * 16));
            }
        }
        if (valid) top.store(row, best_idx, best_keys, alt_idx, alt_keys);
    }
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, kTmemCols);
    }
}

}  // namespace sc
