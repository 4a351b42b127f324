// Shared helpers for the speclust_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/speclust_b200.h"

namespace sc {

// B200: 2 dies x 74 SMs.  Used only to size grids (one or a few resident
// waves); no result depends on it -- the placement-sensitive SpMV measures
// the block -> SM placement itself (sc_sparse.cu, "placed"), and the
// occupancy-sized launches query the device's SM count.
constexpr int kNumSMs = 148;

// ---- error plumbing ---------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);

#define SC_CUDA(expr)                                          \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return ::sc::cuda_fail(_e, #expr); \
    } while (0)

// check the last launch; every wrapper calls this after its kernels
#define SC_LAUNCHED(n)                                                    \
    do {                                                                  \
        ::sc::count_launch(n);                                            \
        cudaError_t _e = cudaGetLastError();                              \
        if (_e != cudaSuccess) return ::sc::cuda_fail(_e, "kernel launch"); \
    } while (0)

inline cudaStream_t as_stream(sc_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- kernel timing ----------------------------------------------------------
// Scoped CUDA-event bracket around launches of a named kernel class; a no-op
// unless sc_profile_enable(1).  `work` = algorithmic bytes or flops.
struct ProfScope {
    int slot = -1;
    cudaStream_t stream = nullptr;
    ProfScope(const char* name, cudaStream_t s, double work);
    ~ProfScope();
};
// ProfScopes opened on this thread while a ProfMute lives are not recorded
// (an internal helper run accounted under its caller's kernel class)
struct ProfMute {
    ProfMute();
    ~ProfMute();
};

// ---- device memory owned by the library ---------------------------------------
// Scratch comes from the stream-ordered pool (cudaMallocAsync on the stream
// the calling entry point works on; the pool keeps freed memory, so repeated
// calls never go back to the driver and never synchronise the device).
// Entry points set the thread's working stream with StreamScope.
cudaStream_t& tl_stream();
void ensure_pool();
void trim_pool();
// Blocking device->host read of a small result (scalars, flags, counts)
// through a per-thread pinned staging buffer: the copy is a plain DMA and the
// stream synchronisation spins; a read into pageable memory takes the
// driver's staged path, whose completion wait sleeps and, on a virtualised
// host, wakes late (measured: 0.1-1 s stalls per pipeline run at C2).
cudaError_t d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t st);
struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(tl_stream()) { tl_stream() = s; }
    ~StreamScope() { tl_stream() = prev; }
};

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    bool owned = true;
    // use caller memory (not freed here)
    void borrow(T* ext, size_t count) {
        free();
        p = ext;
        n = count;
        owned = false;
    }
    int alloc(size_t count) {
        free();
        owned = true;
        n = count;
        if (count == 0) return SC_OK;
        ensure_pool();
        s = tl_stream();
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s);
        if (e == cudaErrorMemoryAllocation) {  // return the pool's cached blocks, then retry once
            (void)cudaGetLastError();
            trim_pool();
            e = cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s);
        }
        if (e != cudaSuccess) {
            p = nullptr;
            n = 0;
            (void)cudaGetLastError();
            return fail(SC_ERR_NO_MEMORY, "device allocation failed for " + std::to_string(count * sizeof(T)) +
                                              " bytes");
        }
        return SC_OK;
    }
    void free() {
        if (p && owned) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
        owned = true;
    }
    ~DevBuf() { free(); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t ceil_div_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

// Philox4x32-10 counter-based generator (device side), used for Lanczos start
// vectors, fresh directions and probe vectors.  Deterministic in (seed, stream,
// element index).
struct Philox {
    __device__ static uint4 round(uint4 c, uint2 k) {
        const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
        uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
        uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
        return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    __device__ static uint4 gen(uint4 c, uint2 k) {
#pragma unroll
        for (int i = 0; i < 10; ++i) {
            c = round(c, k);
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        return c;
    }
};

// standard normal for element `i` of stream `stream_id` under `seed`
__device__ __forceinline__ double philox_normal(uint64_t seed, uint64_t stream_id, uint64_t i) {
    uint4 c = make_uint4((uint32_t)i, (uint32_t)(i >> 32), (uint32_t)stream_id,
                         (uint32_t)(stream_id >> 32));
    uint2 k = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    uint4 r = Philox::gen(c, k);
    // two 53-bit uniforms in (0, 1]
    uint64_t a = ((uint64_t)r.x << 21) ^ ((uint64_t)r.y >> 11);
    uint64_t b = ((uint64_t)r.z << 21) ^ ((uint64_t)r.w >> 11);
    double u1 = ((double)(a & ((1ull << 53) - 1)) + 1.0) * (1.0 / 9007199254740992.0);
    double u2 = (double)(b & ((1ull << 53) - 1)) * (1.0 / 9007199254740992.0);
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// ---------------------------------------------------------------------------
// numpy's float64 sum-of-products order.  The reference computes squared
// norms, distances and k-means cross terms with np.einsum over contiguous
// rows (graph.py:92, kmeans.py:92-104), whose inner loop (this image's x86
// numpy build) runs on two-lane vectors: each block of 8 elements is folded
// last vector first (acc = p0 + (p1 + (p2 + (p3 + acc)))), the tail goes two
// lanes at a time with zero fill, the result is lane0 + lane1, and nothing is
// fused.  Reproducing it makes those values bit-identical to the reference
// (identified against numpy for d = 1..129; checked by the golden tests).
struct NpDot {
    double a0 = 0.0, a1 = 0.0;
    // products of elements c..c+7 of a full block (c % 8 == 0)
    __device__ __forceinline__ void block(double p0, double p1, double p2, double p3, double p4, double p5, double p6,
                                          double p7) {
        a0 = __dadd_rn(p0, __dadd_rn(p2, __dadd_rn(p4, __dadd_rn(p6, a0))));
        a1 = __dadd_rn(p1, __dadd_rn(p3, __dadd_rn(p5, __dadd_rn(p7, a1))));
    }
    __device__ __forceinline__ void pair(double pe, double po) {
        a0 = __dadd_rn(pe, a0);
        a1 = __dadd_rn(po, a1);
    }
    __device__ __forceinline__ void single(double pe) { a0 = __dadd_rn(pe, a0); }
    __device__ __forceinline__ double result() const { return __dadd_rn(a0, a1); }
};

// sum over l of f(l) (a product, computed unfused) for l in [c, end), in the
// order above; c % 8 == 0 and the span is either whole blocks or reaches d
template <class F>
__device__ __forceinline__ void np_dot_span(NpDot& s, int64_t c, int64_t end, F f) {
    for (; c + 8 <= end; c += 8) s.block(f(c), f(c + 1), f(c + 2), f(c + 3), f(c + 4), f(c + 5), f(c + 6), f(c + 7));
    for (; c + 2 <= end; c += 2) s.pair(f(c), f(c + 1));
    if (c < end) s.single(f(c));
}

// |a - b|^2 (np.einsum("ij,ij->i", diff, diff) with diff = a - b)
__device__ __forceinline__ double np_sqdist(const double* __restrict__ a, const double* __restrict__ b, int64_t d) {
    NpDot s;
    np_dot_span(s, 0, d, [&](int64_t l) {
        const double t = __dsub_rn(a[l], b[l]);
        return __dmul_rn(t, t);
    });
    return s.result();
}

// |a|^2 (np.einsum("ij,ij->i", v, v))
__device__ __forceinline__ double np_sqnorm(const double* __restrict__ a, int64_t d) {
    NpDot s;
    np_dot_span(s, 0, d, [&](int64_t l) { return __dmul_rn(a[l], a[l]); });
    return s.result();
}

// Warp-cooperative dot(a_t, b_t) in the einsum order for one row pair per
// lane (nullptr: none).  Each row is read with coalesced warp loads (two rows
// of 16 columns per load) into a shared-memory tile, 16 columns at a time,
// and every lane then folds its own pair from the tiles -- a lane-per-row
// loop would cost one L1 wavefront per lane per element.  stage: kPairStage
// doubles per warp.  Bit-identical to np_dot_span over __dmul_rn(a[l], b[l]).
constexpr int kPairW = 16;
constexpr int kPairLd = kPairW + 1;
constexpr int kPairStage = 2 * 32 * kPairLd + 64;
__device__ __forceinline__ double warp_pair_dot_np(const double* a, const double* b, int64_t d,
                                                   double* __restrict__ stage) {
    const int lane = threadIdx.x & 31, half = lane >> 4, cl = lane & 15;
    double* sa = stage;
    double* sb = stage + 32 * kPairLd;
    const double** pa = reinterpret_cast<const double**>(stage + 2 * 32 * kPairLd);
    const double** pb = pa + 32;
    __syncwarp();
    pa[lane] = a;
    pb[lane] = b;
    NpDot acc;
    for (int64_t c0 = 0; c0 < d; c0 += kPairW) {
        const int w = (int)(d - c0 < kPairW ? d - c0 : kPairW);
        __syncwarp();
#pragma unroll
        for (int r0 = 0; r0 < 32; r0 += 16) {
            double va[8], vb[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int r = r0 + 2 * q + half;
                const double* ra = pa[r];
                const double* rb = pb[r];
                const bool ok = ra && cl < w;
                va[q] = ok ? __ldg(ra + c0 + cl) : 0.0;
                vb[q] = ok ? __ldg(rb + c0 + cl) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int r = r0 + 2 * q + half;
                sa[r * kPairLd + cl] = va[q];
                sb[r * kPairLd + cl] = vb[q];
            }
        }
        __syncwarp();
        if (a) {
            const double* ra = sa + lane * kPairLd - c0;
            const double* rb = sb + lane * kPairLd - c0;
            np_dot_span(acc, c0, c0 + w, [&](int64_t l) { return __dmul_rn(ra[l], rb[l]); });
        }
    }
    return acc.result();
}

// numpy's pairwise summation of a contiguous float64 run (pairwise.c: blocks
// of 8 accumulators up to 128 elements, halving above)
inline __device__ double np_pairwise_sum_dev(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;  // numpy's short loop starts from +0.0
        for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_pairwise_sum_dev(a, n2), np_pairwise_sum_dev(a + n2, n - n2));
}

}  // namespace sc
