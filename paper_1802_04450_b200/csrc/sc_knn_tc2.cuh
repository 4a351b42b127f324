// kNN candidate generation on the 5th-generation tensor cores, query-pair
// variant (d <= 128): one CTA per SM owns TWO query tiles (256 rows) and
// streams every candidate tile once for both of them.
//
//   warp 0      TMA producer: both query tiles once, candidate tiles through
//               a STAGES-deep ring (one B tile feeds two MMAs)
//   warp 1      TMEM allocation (512 columns) + single-thread tcgen05.mma
//               issuer: per candidate tile two M=128 x N=128 accumulators
//               (one per query tile) in one of two TMEM buffers
//   warps 2-9   epilogue, thread <-> query row: warp w reads TMEM lane
//               quarter w % 4 of query tile (w - 2) / 4
//
// Compared with the one-query-tile kernel (sc_knn_tc.cuh) this halves the
// candidate operand traffic and the producer / MMA warps per query row, gives
// every SM sub-partition two epilogue warps without register spills (1 CTA/SM,
// 320 threads), and waits on mbarriers with a hardware suspend hint instead of
// nanosleep spin loops (~40 % of the old kernel's issued instructions, ncu).
// The candidate tiles' column norms travel through their own ring, loaded by
// the producer STAGES tiles ahead (issuing them with the MMA put an L2 round
// trip on the accumulator hand-off), and the scan runs outward from the query
// pair so a row meets its locality region first from both sides.
//
// Measured at C2 (N=1M, d=64; SPECLUST_KNN_WAIT profiling modes): MMA + TMA
// alone 103 ms (1240 TFLOP/s algorithmic), the fast filter path (TMEM loads,
// packed f32x2 key FMAs, 3-input mins, one vote per 64 columns) alone 71 ms,
// both together 103 ms; the whole kernel ~270 ms, i.e. the per-row candidate
// list maintenance (~430 appends and ~8 warp compactions per row, fired in
// ~3 % of the 64-column halves) is what remains to be taken off the critical
// path.
#pragma once
#include <cuda_fp16.h>

#include "sc_knn_tc.cuh"
#include "sc_tc.cuh"

namespace sc {

constexpr int TC2_THREADS = 320;
constexpr int TC2_CN_RING = 8;  // column-norm ring (>= STAGES + 2 tiles in flight)

template <int NKB, int STAGES>
struct Tc2Layout {
    static constexpr uint32_t kA = 2 * NKB * TC_TILE_BYTES;  // two query tiles
    static constexpr uint32_t kB = NKB * TC_TILE_BYTES;
    static constexpr uint32_t kL = 256 * 64 * 4;  // 64 staged keys per epilogue thread (first half / quarters)
    static constexpr uint32_t kCn = TC2_CN_RING * 128 * 4;
    static constexpr uint32_t kBar = 8 * (2 * STAGES + 5 + 2 * TC2_CN_RING) + 8;
    static constexpr uint32_t total = 1024 + kA + STAGES * kB + kL + kCn + kBar;
};

// wait until the phase with `parity` completed; the thread is suspended in
// hardware (time hint ~1 ms) rather than spinning on issue slots
template <bool HINT = true>
__device__ __forceinline__ void mbar_wait_hw(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = tc::smem_u32(bar);
    uint32_t ok = 0;
    while (!ok) {
        if (HINT)
            asm volatile(
                "{\n\t.reg .pred P1;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
                "selp.b32 %0, 1, 0, P1;\n\t}"
                : "=r"(ok)
                : "r"(addr), "r"(parity), "r"(1000000u)
                : "memory");
        else
            asm volatile(
                "{\n\t.reg .pred P1;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                "selp.b32 %0, 1, 0, P1;\n\t}"
                : "=r"(ok)
                : "r"(addr), "r"(parity)
                : "memory");
    }
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
          "l"(*reinterpret_cast<uint64_t*>(&c)));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
    float4 r;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(addr));
    return r;
}
// Candidate tile of scan step t for the query pair at tile qt0: outward from
// the pair (qt0, qt0+1, qt0-1, qt0+2, qt0-2, ...), so that in the locality
// order a row meets its own region first, from both sides, and its threshold
// is near-final before the far tiles arrive.  Visits every tile once.
// |offset| <= ntiles / 2 + 1 and 0 <= qt0 < ntiles, so one conditional
// correction replaces the 64-bit modulo (which cost ~5 % of the kernel's
// issue slots when every epilogue thread evaluated it per tile).
__device__ __forceinline__ int64_t scan_tile(int64_t qt0, int64_t t, int64_t ntiles) {
    const int64_t off = (t & 1) ? ((t + 1) >> 1) : -(t >> 1);
    int64_t c = qt0 + off;
    if (c >= ntiles) c -= ntiles;
    if (c < 0) c += ntiles;
    return c;
}

// order-preserving map of a float key onto uint32 (total order, -0 < +0)
__device__ __forceinline__ uint32_t key_bits(float k) {
    const uint32_t u = __float_as_uint(k);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// keep the R smallest of a row's c_src list entries (global, c_src <= 32 *
// TC2_PER): warp radix select of the R-th smallest key on its
// order-preserving bits (ballot-count rounds over TC2_PER entries per lane,
// starting below the common prefix of the list's min and max), then one
// compaction pass that writes the entries below it and the first ties at it
// to Lg[0..R).  Returns the R-th key: every dropped entry is >= it.
// (Replaces a full bitonic sort per compaction: ~20 % of the kernel's stall
// samples in round 1.)
constexpr int TC2_PER = 4;                  // list entries per lane in a compaction
constexpr int TC2_LIST_MAX = 32 * TC2_PER;  // append capacity of the query-pair kernel
static __device__ __noinline__ float tc2_select_compact(float2* Lg, int c_src, int R, int lane) {
    __syncwarp();  // the owner lane's appends are visible to the warp
    float2 e[TC2_PER];
    uint32_t u[TC2_PER];
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
#pragma unroll
    for (int q = 0; q < TC2_PER; ++q) {
        const int i = lane + 32 * q;
        const bool in = i < c_src;
        e[q] = in ? Lg[i] : make_float2(INFINITY, __int_as_float(-1));
        u[q] = in ? key_bits(e[q].x) : 0xFFFFFFFFu;
        if (in) {
            lo = min(lo, u[q]);
            hi = max(hi, u[q]);
        }
    }
    // T = the (R-1)-th smallest (0-based): built bit by bit keeping
    // count(u < prefix) <= R - 1; T lies in [lo, hi], so the bits above their
    // highest differing bit are fixed
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    const int b0 = lo == hi ? -1 : 31 - __clz(lo ^ hi);
    uint32_t T = b0 < 0 ? lo : (b0 == 31 ? 0u : lo & ~((2u << b0) - 1u));
#pragma unroll 1
    for (int b = b0; b >= 0; --b) {
        const uint32_t cand = T | (1u << b);
        int c = 0;
#pragma unroll
        for (int q = 0; q < TC2_PER; ++q) c += u[q] < cand;
        if ((int)__reduce_add_sync(0xffffffffu, (unsigned)c) <= R - 1) T = cand;
    }
    // entries < T first, then ties == T until R are placed (index order)
    int below = 0;
#pragma unroll
    for (int q = 0; q < TC2_PER; ++q) below += u[q] < T;
    below = (int)__reduce_add_sync(0xffffffffu, (unsigned)below);
    __syncwarp();
    int pos_lt = 0, pos_eq = below;
    const unsigned lower = (1u << lane) - 1u;
#pragma unroll
    for (int q = 0; q < TC2_PER; ++q) {
        const bool lt = u[q] < T, eq = u[q] == T;
        const unsigned blt = __ballot_sync(0xffffffffu, lt), beq = __ballot_sync(0xffffffffu, eq);
        const int slt = pos_lt + __popc(blt & lower), seq = pos_eq + __popc(beq & lower);
        if (lt) Lg[slt] = e[q];
        if (eq && seq < R) Lg[seq] = e[q];
        pos_lt += __popc(blt);
        pos_eq += __popc(beq);
    }
    __syncwarp();
    const uint32_t tb = (T & 0x80000000u) ? (T & 0x7FFFFFFFu) : ~T;
    return __uint_as_float(tb);
}
__device__ __forceinline__ float fmin3(float a, float b, float c) { return fminf(a, fminf(b, c)); }

template <int NKB, int STAGES, int WMODE, bool HEAP>
__global__ void __launch_bounds__(TC2_THREADS, 1)
    knn_cand_tc2_kernel(const __grid_constant__ CUtensorMap xmap, int64_t n, int64_t ntiles, int64_t qtile0,
                        int64_t nq, const float* __restrict__ cnk, float key_scale, int cap, int R,
                        float2* __restrict__ lists, int* __restrict__ counts, float* __restrict__ taus,
                        long long* __restrict__ dbg = nullptr) {
    using Lay = Tc2Layout<NKB, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;
    uint8_t* sB = base + Lay::kA;
    float2* sL = reinterpret_cast<float2*>(sB + STAGES * Lay::kB);
    float* sCn = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sL) + Lay::kL);  // [TC2_CN_RING][128]
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sCn) + Lay::kCn);
    uint64_t* empty = full + STAGES;
    uint64_t* afull = empty + STAGES;
    uint64_t* tfull = afull + 1;   // [2]
    uint64_t* tempty = tfull + 2;  // [2]
    uint64_t* cfull = tempty + 2;                // [TC2_CN_RING]
    uint64_t* cempty = cfull + TC2_CN_RING;      // [TC2_CN_RING]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + TC2_CN_RING);
    // HEAP: per-row max-heaps of the R best candidates (256 x R float2) and a
    // 16-key staging slot per epilogue thread, after the barriers
    float2* sH = reinterpret_cast<float2*>(reinterpret_cast<uintptr_t>(tmem_slot + 4 + 15) & ~uintptr_t(15));
    float* sStage = reinterpret_cast<float*>(sH + (HEAP ? 256 * R : 0));

    // profiling: a negative cap keeps the list code compiled but never runs it
    const bool capneg = cap < 0;
    if (capneg) cap = -cap;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // query tiles qt0, qt0 + 1 (scan positions); list slots relative to qtile0
    const int64_t lq0 = (int64_t)blockIdx.x * 2;
    const int64_t qt0 = qtile0 + lq0;

    if (warp == 0 && lane == 0) tc::tma_prefetch(&xmap);
    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s) {
                tc::mbar_init(&full[s], 1);
                tc::mbar_init(&empty[s], 1);
            }
            tc::mbar_init(afull, 1);
            for (int b = 0; b < 2; ++b) {
                tc::mbar_init(&tfull[b], 1);   // MMA commit
                tc::mbar_init(&tempty[b], 8);  // the 8 epilogue warps
            }
            for (int c = 0; c < TC2_CN_RING; ++c) {
                tc::mbar_init(&cfull[c], 1);   // column-norm bulk copy (producer)
                tc::mbar_init(&cempty[c], 8);  // the 8 epilogue warps
            }
            tc::fence_mbar_init();
        }
        __syncwarp();
        tc::tmem_alloc(tmem_slot, 512);
    }
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            tc::mbar_expect_tx(afull, Lay::kA);
            for (int q = 0; q < 2; ++q)
                for (int kb = 0; kb < NKB; ++kb)
                    tc::tma_load_2d(sA + (q * NKB + kb) * TC_TILE_BYTES, &xmap, afull, kb * 64,
                                    (int)((qt0 + q) * 128));
            for (int64_t t = 0; t < ntiles; ++t) {
                const int s = (int)(t % STAGES);
                mbar_wait_hw<(WMODE & 1) != 0>(&empty[s], (uint32_t)(((t / STAGES) & 1) ^ 1));
                tc::mbar_expect_tx(&full[s], Lay::kB);
                const int64_t ct = scan_tile(qt0, t, ntiles);
                const int y = (int)(ct * 128);
                for (int kb = 0; kb < NKB; ++kb)
                    tc::tma_load_2d(sB + s * Lay::kB + kb * TC_TILE_BYTES, &xmap, &full[s], kb * 64, y);
                // the tile's column norms, far ahead of the epilogue that needs them
                const int c = (int)(t % TC2_CN_RING);
                mbar_wait_hw<(WMODE & 1) != 0>(&cempty[c], (uint32_t)(((t / TC2_CN_RING) & 1) ^ 1));
                tc::mbar_expect_tx(&cfull[c], 128 * 4);
                tc::bulk_g2s(sCn + c * 128, cnk + ct * 128, 128 * 4, &cfull[c]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_f16_f32(128, 128);
            mbar_wait_hw<(WMODE & 1) != 0>(afull, 0);
            for (int64_t t = 0; t < ntiles; ++t) {
                const int s = (int)(t % STAGES);
                const int buf = (int)(t & 1);
                mbar_wait_hw<(WMODE & 1) != 0>(&tempty[buf], (uint32_t)(((t >> 1) & 1) ^ 1));
                mbar_wait_hw<(WMODE & 1) != 0>(&full[s], (uint32_t)((t / STAGES) & 1));
                tc::fence_after();
                if (!(WMODE & 8))
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int kb = 0; kb < NKB; ++kb) {
                        const uint64_t ad = tc::desc_k_sw128(sA + (q * NKB + kb) * TC_TILE_BYTES);
                        const uint64_t bd = tc::desc_k_sw128(sB + s * Lay::kB + kb * TC_TILE_BYTES);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc::umma_f16(tmem + buf * 256 + q * 128, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                    }
                tc::umma_commit(&empty[s]);
                tc::umma_commit(&tfull[buf]);
            }
        }
    } else {
        const int quad = warp & 3;
        const int qi = (warp - 2) >> 2;
        const int lrow = qi * 128 + quad * 32 + lane;  // row within the pair
        const int64_t row = qt0 * 128 + lrow;
        const bool tile_ok = lq0 + qi < nq;
        const bool valid = tile_ok && row < n;
        const int64_t slot = lq0 * 128 + lrow;  // list slot of this row
        float2* L = lists + (valid ? slot : 0) * (int64_t)cap;
        float2* H = sH + (size_t)lrow * R;
        // per thread: 64 floats of staged first-half keys, then (HEAP: its
        // own slot) 16 floats of quarter staging for the append loop
        float* skeys = reinterpret_cast<float*>(sL) + ((size_t)(warp - 2) * 32 + lane) * 64;
        float* stage = HEAP ? sStage + ((size_t)(warp - 2) * 32 + lane) * 16 : skeys;
        int cnt = 0;
        float tau = INFINITY;
        long long dbg_c[3] = {0, 0, 0}, dbg_f[3] = {0, 0, 0};
        // max-heap on the key: sift `e` down from slot i
        auto sift_down = [&](int i, float2 e) {
            while (true) {
                const int l = 2 * i + 1;
                if (l >= R) break;
                int c = l;
                if (l + 1 < R && H[l + 1].x > H[l].x) c = l + 1;
                const float2 hc = H[c];
                if (hc.x <= e.x) break;
                H[i] = hc;
                i = c;
            }
            H[i] = e;
        };
        // keep the R smallest keys: fill, heapify once full, then replace the max
        auto heap_push = [&](float k, int64_t col) {
            const float2 e = make_float2(k, __int_as_float((int)col));
            if (cnt < R) {
                H[cnt++] = e;
                if (cnt == R) {
                    for (int i = R / 2 - 1; i >= 0; --i) sift_down(i, H[i]);
                    tau = H[0].x;
                }
            } else {
                sift_down(0, e);
                tau = H[0].x;
            }
        };
        const float2 ks = make_float2(key_scale, key_scale);
        for (int64_t t = 0; t < ntiles; ++t) {
            const int buf = (int)(t & 1);
            const int cslot = (int)(t % TC2_CN_RING);
            mbar_wait_hw<(WMODE & 2) != 0>(&cfull[cslot], (uint32_t)((t / TC2_CN_RING) & 1));
            mbar_wait_hw<(WMODE & 2) != 0>(&tfull[buf], (uint32_t)((t >> 1) & 1));
            tc::fence_after();
            const int64_t col0 = scan_tile(qt0, t, ntiles) * 128;
            const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * 256 + qi * 128);
            if (WMODE & 4) {
                tc::fence_before();
                __syncwarp();
                if (lane == 0) {
                    tc::mbar_arrive(&tempty[buf]);
                    tc::mbar_arrive(&cempty[cslot]);
                }
                continue;
            }
            // the accumulator in two 64-column halves through the same 64
            // registers: the first half's keys go to shared memory only when
            // its filter fires, so the tile loop needs half the registers
            // (with both halves live, 168 registers and spills)
            const uint32_t cn_s = tc::smem_u32(sCn + cslot * 128);
            float va[64];
            float qm[8];
            auto keys_half = [&](int hf) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float m = INFINITY;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float4 cn4 = lds_f4(cn_s + (uint32_t)(16 * (4 * (4 * hf + q) + u)));  // smem broadcast
                        float* e = va + 16 * q + 4 * u;
                        const float2 k01 = ffma2(ks, make_float2(e[0], e[1]), make_float2(cn4.x, cn4.y));
                        const float2 k23 = ffma2(ks, make_float2(e[2], e[3]), make_float2(cn4.z, cn4.w));
                        e[0] = k01.x;
                        e[1] = k01.y;
                        e[2] = k23.x;
                        e[3] = k23.y;
                        m = fmin3(m, fmin3(k01.x, k01.y, k23.x), k23.y);
                    }
                    qm[4 * hf + q] = m;
                }
            };
            tc::tmem_ld64(taddr, va);
            tc::tmem_wait_ld();
            keys_half(0);
            const float h0 = fminf(fminf(qm[0], qm[1]), fminf(qm[2], qm[3]));
            const bool fire0 = !capneg && !(WMODE & 16) && __any_sync(0xffffffffu, valid && h0 < tau);
            if (fire0) {
                float4* d4 = reinterpret_cast<float4*>(skeys);
#pragma unroll
                for (int u = 0; u < 16; ++u) d4[u] = make_float4(va[4 * u], va[4 * u + 1], va[4 * u + 2], va[4 * u + 3]);
            }
            tc::tmem_ld64(taddr + 64, va);
            tc::tmem_wait_ld();
            // the accumulator is in registers / shared memory: hand the TMEM
            // buffer back, so the MMA of tile t + 2 overlaps this tile's list work
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[buf]);
            keys_half(1);
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&cempty[cslot]);  // column norms consumed
            const float h1 = fminf(fminf(qm[4], qm[5]), fminf(qm[6], qm[7]));
            // rare path: append the passing keys of a 64-column half to the row's list
            auto slow = [&](const float* keys64, const float* qm4, int64_t cbase) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool pass = valid && qm4[q] < tau;
                    if (!__any_sync(0xffffffffu, pass)) continue;
                    unsigned want = __ballot_sync(0xffffffffu, pass && cnt > cap - 16);
                    while (want) {  // warp-cooperative compaction of lists about to overflow
                        __syncwarp();
                        const int src = __ffs(want) - 1;
                        want &= want - 1;
                        const int c_src = __shfl_sync(0xffffffffu, cnt, src);
                        const int64_t sslot = __shfl_sync(0xffffffffu, slot, src);
                        float2* Lg = lists + sslot * (int64_t)cap;
                        const float new_tau = tc2_select_compact(Lg, c_src, R, lane);
                        if (lane == src) {
                            cnt = R;
                            tau = new_tau;
                        }
                    }
                    if (pass) {
                        // passing keys as a bit mask, walked with ffs: one
                        // store per appended key instead of 16 predicated ones
                        const float* keys = keys64 + 16 * q;
                        const int64_t cb = cbase + q * 16;
                        unsigned msk = 0;
#pragma unroll
                        for (int u = 0; u < 16; ++u) msk |= (keys[u] < tau ? 1u : 0u) << u;
                        if (row >= cb && row < cb + 16) msk &= ~(1u << (int)(row - cb));
                        if (cb + 16 > n) msk &= n > cb ? (1u << (int)(n - cb)) - 1u : 0u;
                        if (msk) {
                            float4* st4 = reinterpret_cast<float4*>(stage);
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                st4[u] = make_float4(keys[4 * u], keys[4 * u + 1], keys[4 * u + 2], keys[4 * u + 3]);
                            while (msk) {
                                const int u = __ffs(msk) - 1;
                                msk &= msk - 1;
                                L[cnt++] = make_float2(stage[u], __int_as_float((int)(cb + u)));
                            }
                        }
                    }
                }
            };
            // heap variant: every row owns its heap, so lanes proceed
            // independently; the passing 16-key quarter is staged in shared
            // memory and walked by a rolled loop (small code, no register
            // indexing)
            auto slow_heap = [&](const float* keys64, const float* qm4, int64_t cbase) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (!(valid && qm4[q] < tau)) continue;
                    float4* st4 = reinterpret_cast<float4*>(stage);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        st4[u] = make_float4(keys64[16 * q + 4 * u], keys64[16 * q + 4 * u + 1],
                                             keys64[16 * q + 4 * u + 2], keys64[16 * q + 4 * u + 3]);
                    const int64_t cb = cbase + q * 16;
#pragma unroll 1
                    for (int u = 0; u < 16; ++u) {
                        const float k = stage[u];
                        const int64_t col = cb + u;
                        if (k < tau && col != row && col < n) heap_push(k, col);
                    }
                }
            };
            if (capneg) {
            } else if (HEAP) {
                if (fire0) slow_heap(skeys, qm, col0);
                if (!(WMODE & 16) && __any_sync(0xffffffffu, valid && h1 < tau)) slow_heap(va, qm + 4, col0 + 64);
            } else {
                const long long z0 = (WMODE & 64) ? clock64() : 0;
                int fired = 0;
                if (fire0) {
                    slow(skeys, qm, col0);
                    ++fired;
                }
                if (!(WMODE & 16) && __any_sync(0xffffffffu, valid && h1 < tau)) {
                    slow(va, qm + 4, col0 + 64);
                    ++fired;
                }
                if (WMODE & 64) {
                    const int bin = t < 16 ? 0 : t < 128 ? 1 : 2;
                    dbg_c[bin] += clock64() - z0;
                    dbg_f[bin] += fired;
                }
            }
        }
        if ((WMODE & 64) && lane == 0 && dbg) {
            for (int b = 0; b < 3; ++b) {
                atomicAdd(reinterpret_cast<unsigned long long*>(dbg + b), (unsigned long long)dbg_c[b]);
                atomicAdd(reinterpret_cast<unsigned long long*>(dbg + 3 + b), (unsigned long long)dbg_f[b]);
            }
        }
        if (!HEAP) {
            // the recheck sorts at most TC_LIST_P entries per row: longer lists
            // are compacted to R once more (tau tightens accordingly)
            unsigned want = __ballot_sync(0xffffffffu, valid && cnt > TC_LIST_P);
            while (want) {
                const int src = __ffs(want) - 1;
                want &= want - 1;
                const int c_src = __shfl_sync(0xffffffffu, cnt, src);
                const int64_t sslot = __shfl_sync(0xffffffffu, slot, src);
                const float new_tau = tc2_select_compact(lists + sslot * (int64_t)cap, c_src, R, lane);
                if (lane == src) {
                    cnt = R;
                    tau = new_tau;
                }
            }
        }
        if (valid) {
            if (HEAP)
                for (int e = 0; e < cnt; ++e) L[e] = H[e];
            counts[slot] = cnt;
            taus[slot] = tau;
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, 512);
    }
}

}  // namespace sc
