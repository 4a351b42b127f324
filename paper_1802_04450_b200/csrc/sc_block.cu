// Block Gram-Schmidt against the Krylov basis as tall-skinny fp64 GEMMs on
// the DMMA tensor path (mma.sync.m8n8k4.f64):
//
//   H = B[:, :nb]^T V      (block_tn: nb x c, split over row ranges, fixed-order reduce)
//   V -= B[:, :nb] H       (block_nn)
//
// with V = c (<= 40) consecutive basis columns.  This is the "flush" of the
// windowed reorthogonalisation in sc_lanczos.cu: the reference's CGS2 over the
// whole basis after every step (eigen.py:131-135, 163) reads the n x j basis
// four times per Lanczos vector; here every step orthogonalises against a
// short window of recent vectors and the window is orthogonalised against the
// older basis once per c vectors, reading it twice per block instead.
#include <algorithm>

#include "sc_block.cuh"

namespace sc {

namespace {

constexpr int BK_ROWS = 32;  // rows per staged chunk (tn) / basis columns per chunk (nn)
constexpr int BK_COLS = 64;  // basis columns per CTA (tn) / rows per CTA (nn)
constexpr int BK_MAXT = 5;   // N tiles of 8 (c <= 40)
constexpr int BK_STAGES = 3; // cp.async ring depth
// shared-memory strides (doubles): a column of 32 rows padded to 36 (tn), a
// basis column of 64 rows padded to 68 (nn) -- 16-byte aligned and
// conflict-free for the m8n8k4 fragment loads of a half warp
constexpr int TN_LDA = 36, NN_LDA = 68;

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}
// 16-byte async copy of `bytes` (0, 8 or 16) valid bytes; the rest of the
// 16 is zero-filled
__device__ __forceinline__ void cp16n(void* smem, const void* gmem, int bytes) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool pred) { cp16n(smem, gmem, pred ? 16 : 0); }
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int NT>
struct TnSmem {
    static constexpr int kA = BK_COLS * TN_LDA;     // [col][row]
    static constexpr int kV = NT * 8 * TN_LDA;      // [o][row]
    static constexpr int kStage = kA + kV;
    static constexpr size_t bytes = (size_t)BK_STAGES * kStage * sizeof(double);
};

// partial[g][col][o] = sum_{rows of split g} B[col*ld + r] * V[o*ld + r].
// CTA = 64 basis columns x one row split; 32-row chunks stream through a
// BK_STAGES-deep cp.async ring (16-byte copies; ld and the row splits are
// multiples of 2 rows so every copy is aligned), m8n8k4 DMMA per warp.
template <int NT>
__global__ void __launch_bounds__(256) block_tn_kernel(int64_t n, int64_t ld, int nb, const double* __restrict__ B,
                                                       const double* __restrict__ V, int c, int64_t rows_per_split,
                                                       double* __restrict__ part) {
    using L = TnSmem<NT>;
    extern __shared__ __align__(16) double tn_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col0 = blockIdx.x * BK_COLS;
    const int64_t r_begin = (int64_t)blockIdx.y * rows_per_split;
    const int64_t r_end = imin64(n, r_begin + rows_per_split);
    const int64_t nchunks = r_end > r_begin ? (r_end - r_begin + BK_ROWS - 1) / BK_ROWS : 0;
    auto load = [&](int64_t ch, int stage) {
        double* As = tn_smem + stage * L::kStage;
        double* Vs = As + L::kA;
        const int64_t r0 = r_begin + ch * BK_ROWS;
        // B: 64 columns x 16 pairs of rows
        for (int e = threadIdx.x; e < BK_COLS * 16; e += 256) {
            const int cc = e >> 4, pr = (e & 15) * 2;
            const int col = col0 + cc;
            const int64_t r = r0 + pr;
            // a last odd row (r_end = n odd) copies 8 bytes: the padding row
            // past n is never read
            const int bytes = (col < nb && r < r_end) ? (r + 1 < r_end ? 16 : 8) : 0;
            cp16n(As + cc * TN_LDA + pr, bytes ? B + (int64_t)col * ld + r : B, bytes);
        }
        for (int e = threadIdx.x; e < NT * 8 * 16; e += 256) {
            const int o = e >> 4, pr = (e & 15) * 2;
            const int64_t r = r0 + pr;
            const int bytes = (o < c && r < r_end) ? (r + 1 < r_end ? 16 : 8) : 0;
            cp16n(Vs + o * TN_LDA + pr, bytes ? V + (int64_t)o * ld + r : V, bytes);
        }
    };
    double acc[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < BK_STAGES - 1; ++s) {
        if (s < nchunks) load(s, s);
        cp_commit();
    }
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        cp_wait<BK_STAGES - 2>();
        __syncthreads();
        // refill the stage consumed in the previous iteration
        if (ch + BK_STAGES - 1 < nchunks) load(ch + BK_STAGES - 1, (int)((ch + BK_STAGES - 1) % BK_STAGES));
        cp_commit();
        const double* As = tn_smem + (ch % BK_STAGES) * L::kStage;
        const double* Vs = As + L::kA;
        const double* ap = As + (warp * 8 + (lane >> 2)) * TN_LDA + (lane & 3);
        const double* bp = Vs + (lane >> 2) * TN_LDA + (lane & 3);
#pragma unroll
        for (int k4 = 0; k4 < BK_ROWS; k4 += 4) {
            const double a = ap[k4];
#pragma unroll
            for (int t = 0; t < NT; ++t) dmma884(acc[t], a, bp[t * 8 * TN_LDA + k4]);
        }
    }
    cp_wait<0>();
    const int col = col0 + warp * 8 + (lane >> 2);
    if (col < nb) {
        double* p = part + ((int64_t)blockIdx.y * nb + col) * (NT * 8);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            p[t * 8 + 2 * (lane & 3)] = acc[t][0];
            p[t * 8 + 2 * (lane & 3) + 1] = acc[t][1];
        }
    }
}

// H[col][o] = sum_g part[g][col][o] (fixed order); *maxabs = max |H| (ordered bits)
// H[col][o] = sum over the nsplit row groups of part[g][col][o]: one warp per
// output element, lanes strided over the groups (4 loads in flight each),
// then the warp's xor tree -- a fixed order.  (One thread per element looping
// over all groups was a serial chain of L2 loads: 73 us per flush at C2.)
__global__ void block_reduce_kernel(int nsplit, int nb, int c, int ldp, const double* __restrict__ part,
                                    double* __restrict__ H, unsigned long long* __restrict__ maxabs) {
    const int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (e >= (int64_t)nb * c) return;
    const int col = (int)(e / c), o = (int)(e % c);
    const double* src = part + (int64_t)col * ldp + o;
    const int64_t gstride = (int64_t)nb * ldp;
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    int g = lane;
    for (; g + 96 < nsplit; g += 128)
#pragma unroll
        for (int u = 0; u < 4; ++u) t[u] += src[(int64_t)(g + 32 * u) * gstride];
    for (; g < nsplit; g += 32) t[0] += src[(int64_t)g * gstride];
    const double v = warp_sum((t[0] + t[1]) + (t[2] + t[3]));
    if (lane == 0) {
        H[(int64_t)col * c + o] = v;
        if (maxabs) atomicMax(maxabs, (unsigned long long)__double_as_longlong(fabs(v)));
    }
}

template <int NT>
struct NnSmem {
    static constexpr int kHs = NT * 8 + 4;           // H row stride (doubles)
    static constexpr int kA = BK_ROWS * NN_LDA;      // [basis col][row]
    static constexpr int kH = BK_ROWS * kHs;         // [basis col][o]
    static constexpr int kStage = kA + kH;
    static constexpr size_t bytes = (size_t)BK_STAGES * kStage * sizeof(double);
};

// V[o*ld + r] -= sum_col B[col*ld + r] * H[col][o] for the 64 rows of this CTA;
// 32 basis columns per chunk through the cp.async ring (B rows and the H
// chunk), m8n8k4 DMMA with the rows as M
template <int NT>
__global__ void __launch_bounds__(256) block_nn_kernel(int64_t n, int64_t ld, int nb, const double* __restrict__ B,
                                                       const double* __restrict__ H, int c, double* __restrict__ V) {
    using L = NnSmem<NT>;
    extern __shared__ __align__(16) double nn_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * BK_COLS;
    const int nchunks = (nb + BK_ROWS - 1) / BK_ROWS;
    const bool hvec = (c & 1) == 0;  // H rows 16-byte aligned: pairwise copies
    auto load = [&](int ch, int stage) {
        double* As = nn_smem + stage * L::kStage;
        double* Hs = As + L::kA;
        const int k0 = ch * BK_ROWS;
        for (int e = threadIdx.x; e < BK_ROWS * 32; e += 256) {
            const int kk = e >> 5, pr = (e & 31) * 2;
            const int k = k0 + kk;
            const int64_t r = row0 + pr;
            const bool ok = k < nb && r < n;
            cp16(As + kk * NN_LDA + pr, ok ? B + (int64_t)k * ld + r : B, ok);
        }
        if (hvec) {
            const int pairs = c / 2;
            for (int e = threadIdx.x; e < BK_ROWS * pairs; e += 256) {
                const int kk = e / pairs, o = (e % pairs) * 2;
                const int k = k0 + kk;
                cp16(Hs + kk * L::kHs + o, k < nb ? H + (int64_t)k * c + o : H, k < nb);
            }
        } else {
            for (int e = threadIdx.x; e < BK_ROWS * c; e += 256) {
                const int kk = e / c, o = e % c;
                const int k = k0 + kk;
                Hs[kk * L::kHs + o] = k < nb ? H[(int64_t)k * c + o] : 0.0;
            }
        }
    };
    // columns o >= c of the staged H chunk are never written by the loads:
    // zero them once in every stage
    for (int e = threadIdx.x; e < BK_STAGES * BK_ROWS * (NT * 8 - c); e += 256) {
        const int s = e / (BK_ROWS * (NT * 8 - c)), rem = e % (BK_ROWS * (NT * 8 - c));
        const int kk = rem / (NT * 8 - c), o = c + rem % (NT * 8 - c);
        nn_smem[s * L::kStage + L::kA + kk * L::kHs + o] = 0.0;
    }
    double acc[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < BK_STAGES - 1; ++s) {
        if (s < nchunks) load(s, s);
        cp_commit();
    }
    for (int ch = 0; ch < nchunks; ++ch) {
        cp_wait<BK_STAGES - 2>();
        __syncthreads();
        if (ch + BK_STAGES - 1 < nchunks) load(ch + BK_STAGES - 1, (ch + BK_STAGES - 1) % BK_STAGES);
        cp_commit();
        const double* As = nn_smem + (ch % BK_STAGES) * L::kStage;
        const double* Hs = As + L::kA;
        const double* ap = As + (lane & 3) * NN_LDA + warp * 8 + (lane >> 2);
        const double* bp = Hs + (lane & 3) * L::kHs + (lane >> 2);
#pragma unroll
        for (int k4 = 0; k4 < BK_ROWS; k4 += 4) {
            const double a = ap[k4 * NN_LDA];
#pragma unroll
            for (int t = 0; t < NT; ++t) dmma884(acc[t], a, bp[k4 * L::kHs + t * 8]);
        }
    }
    cp_wait<0>();
    const int64_t r = row0 + warp * 8 + (lane >> 2);
    if (r < n) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int o = t * 8 + 2 * (lane & 3) + i;
                if (o < c) V[(int64_t)o * ld + r] -= acc[t][i];
            }
        }
    }
}

int resident_ctas(const void* fn, size_t smem) {
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, 256, smem);
    int dev = 0, nsm = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return std::max(1, bps) * nsm;
}

template <int NT>
int launch_tn(int64_t n, int64_t ld, int nb, const double* B, const double* V, int c, int* nsplit, double* part,
              cudaStream_t st, bool query_only = false) {
    const size_t smem = TnSmem<NT>::bytes;
    static int slots = 0;
    if (!slots) {
        cudaFuncSetAttribute(block_tn_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        slots = resident_ctas((const void*)block_tn_kernel<NT>, smem);
    }
    // one wave: column tiles x row splits <= resident CTAs, splits of >= 2K rows
    const int cb = (nb + BK_COLS - 1) / BK_COLS;
    int64_t g = std::max<int64_t>(1, slots / cb);
    g = std::min<int64_t>(g, std::max<int64_t>(1, ceil_div(n, 2048)));
    const int64_t rps = ceil_div(ceil_div(n, g), BK_ROWS) * BK_ROWS;
    *nsplit = (int)ceil_div(n, rps);
    if (query_only) return SC_OK;
    dim3 grid((unsigned)cb, (unsigned)*nsplit);
    block_tn_kernel<NT><<<grid, 256, smem, st>>>(n, ld, nb, B, V, c, rps, part);
    return SC_OK;
}
template <int NT>
void launch_nn(int64_t n, int64_t ld, int nb, const double* B, const double* H, int c, double* V, cudaStream_t st) {
    const size_t smem = NnSmem<NT>::bytes;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(block_nn_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    block_nn_kernel<NT><<<(unsigned)ceil_div(n, BK_COLS), 256, smem, st>>>(n, ld, nb, B, H, c, V);
}

int tn_dispatch(int nt, int64_t n, int64_t ld, int nb, const double* B, const double* V, int c, int* nsplit,
                double* part, cudaStream_t st, bool query_only) {
    switch (nt) {
        case 1: return launch_tn<1>(n, ld, nb, B, V, c, nsplit, part, st, query_only);
        case 2: return launch_tn<2>(n, ld, nb, B, V, c, nsplit, part, st, query_only);
        case 3: return launch_tn<3>(n, ld, nb, B, V, c, nsplit, part, st, query_only);
        case 4: return launch_tn<4>(n, ld, nb, B, V, c, nsplit, part, st, query_only);
        default: return launch_tn<5>(n, ld, nb, B, V, c, nsplit, part, st, query_only);
    }
}

}  // namespace

int block_tn(int64_t n, int64_t ld, int nb, const double* B, const double* V, int c, double* H, double* part,
             unsigned long long* maxabs, cudaStream_t st) {
    if (c < 1 || c > BK_MAXT * 8) return fail(SC_ERR_VALUE, "block width must be in [1, 40]");
    if (nb <= 0) return SC_OK;
    if ((ld & 1) || (reinterpret_cast<uintptr_t>(B) & 15) || (reinterpret_cast<uintptr_t>(V) & 15))
        return fail(SC_ERR_VALUE, "block GEMMs need 16-byte aligned columns (even ld)");
    const int nt = (c + 7) / 8;
    int gs = 0;
    tn_dispatch(nt, n, ld, nb, B, V, c, &gs, part, st, false);
    const int64_t tot = (int64_t)nb * c;
    block_reduce_kernel<<<(unsigned)ceil_div(tot, 8), 256, 0, st>>>(gs, nb, c, nt * 8, part, H, maxabs);
    SC_LAUNCHED(2);
    return SC_OK;
}

int block_nn(int64_t n, int64_t ld, int nb, const double* B, const double* H, int c, double* V, cudaStream_t st) {
    if (c < 1 || c > BK_MAXT * 8) return fail(SC_ERR_VALUE, "block width must be in [1, 40]");
    if (nb <= 0) return SC_OK;
    if ((ld & 1) || (reinterpret_cast<uintptr_t>(B) & 15) || (reinterpret_cast<uintptr_t>(H) & 15))
        return fail(SC_ERR_VALUE, "block GEMMs need 16-byte aligned columns (even ld)");
    switch ((c + 7) / 8) {
        case 1: launch_nn<1>(n, ld, nb, B, H, c, V, st); break;
        case 2: launch_nn<2>(n, ld, nb, B, H, c, V, st); break;
        case 3: launch_nn<3>(n, ld, nb, B, H, c, V, st); break;
        case 4: launch_nn<4>(n, ld, nb, B, H, c, V, st); break;
        default: launch_nn<5>(n, ld, nb, B, H, c, V, st); break;
    }
    SC_LAUNCHED(1);
    return SC_OK;
}

size_t block_part_size(int64_t n, int nb, int c) {
    const int nt = (c + 7) / 8;
    int gs = 0;
    tn_dispatch(nt, n, 0, nb, nullptr, nullptr, c, &gs, nullptr, nullptr, true);
    return (size_t)gs * (size_t)nb * (size_t)(nt * 8);
}

}  // namespace sc

extern "C" {

int sc_block_tn_f64(int64_t n, int64_t ld, int64_t nb, const double* B, const double* V, int64_t c, double* H,
                    sc_stream_t stream) {
    cudaStream_t st = sc::as_stream(stream);
    sc::StreamScope scope(st);
    if (nb <= 0) return SC_OK;
    sc::DevBuf<double> part;
    if (int rc = part.alloc(sc::block_part_size(n, (int)nb, (int)c))) return rc;
    return sc::block_tn(n, ld, (int)nb, B, V, (int)c, H, part.p, nullptr, st);
}

int sc_block_nn_f64(int64_t n, int64_t ld, int64_t nb, const double* B, const double* H, int64_t c, double* V,
                    sc_stream_t stream) {
    cudaStream_t st = sc::as_stream(stream);
    sc::StreamScope scope(st);
    return sc::block_nn(n, ld, (int)nb, B, H, (int)c, V, st);
}

}  // extern "C"
