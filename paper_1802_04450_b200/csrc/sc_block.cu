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
#include "sc_block.cuh"

namespace sc {

namespace {

constexpr int BK_ROWS = 32;  // rows per staged chunk (tn) / columns per chunk (nn)
constexpr int BK_COLS = 64;  // basis columns per CTA (tn) / rows per CTA (nn)
constexpr int BK_MAXT = 5;   // N tiles of 8 (c <= 40)

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// partial[g][col][o] = sum_{rows of split g} B[col*ld + r] * V[o*ld + r]
template <int NT>
__global__ void __launch_bounds__(256) block_tn_kernel(int64_t n, int64_t ld, int nb, const double* __restrict__ B,
                                                       const double* __restrict__ V, int c, int64_t rows_per_split,
                                                       double* __restrict__ part) {
    __shared__ double As[BK_ROWS][BK_COLS + 1];
    __shared__ double Vs[BK_ROWS][NT * 8 + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col0 = blockIdx.x * BK_COLS;
    const int64_t r_begin = (int64_t)blockIdx.y * rows_per_split;
    const int64_t r_end = imin64(n, r_begin + rows_per_split);
    double acc[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
    const int lr = threadIdx.x & 31, lc = threadIdx.x >> 5;  // loader: row, column group
    for (int64_t r0 = r_begin; r0 < r_end; r0 += BK_ROWS) {
        const int64_t r = r0 + lr;
        const bool rok = r < r_end;
#pragma unroll
        for (int i = 0; i < BK_COLS / 8; ++i) {
            const int cc = lc + 8 * i;
            const int col = col0 + cc;
            As[lr][cc] = (rok && col < nb) ? __ldg(B + (int64_t)col * ld + r) : 0.0;
        }
        for (int o = lc; o < NT * 8; o += 8) Vs[lr][o] = (rok && o < c) ? __ldg(V + (int64_t)o * ld + r) : 0.0;
        __syncthreads();
#pragma unroll
        for (int k4 = 0; k4 < BK_ROWS; k4 += 4) {
            const double a = As[k4 + (lane & 3)][warp * 8 + (lane >> 2)];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const double b = Vs[k4 + (lane & 3)][t * 8 + (lane >> 2)];
                dmma884(acc[t], a, b);
            }
        }
        __syncthreads();
    }
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
__global__ void block_reduce_kernel(int nsplit, int nb, int c, int ldp, const double* __restrict__ part,
                                    double* __restrict__ H, unsigned long long* __restrict__ maxabs) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double v = 0.0;
    if (e < (int64_t)nb * c) {
        const int col = (int)(e / c), o = (int)(e % c);
        for (int g = 0; g < nsplit; ++g) v += part[((int64_t)g * nb + col) * ldp + o];
        H[(int64_t)col * c + o] = v;
    }
    if (maxabs) {
        double a = fabs(v);
        for (int s = 16; s > 0; s >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, s));
        if ((threadIdx.x & 31) == 0) atomicMax(maxabs, (unsigned long long)__double_as_longlong(a));
    }
}

// V[o*ld + r] -= sum_col B[col*ld + r] * H[col][o], rows of this CTA
template <int NT>
__global__ void __launch_bounds__(256) block_nn_kernel(int64_t n, int64_t ld, int nb, const double* __restrict__ B,
                                                       const double* __restrict__ H, int c, double* __restrict__ V) {
    __shared__ double As[BK_ROWS][BK_COLS + 1];  // [k = basis column][row]
    __shared__ double Hs[BK_ROWS][NT * 8 + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * BK_COLS;
    double acc[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
    const int lrow = threadIdx.x & 63, lk = threadIdx.x >> 6;  // loader: row, column group (4)
    for (int k0 = 0; k0 < nb; k0 += BK_ROWS) {
        const int64_t r = row0 + lrow;
#pragma unroll
        for (int i = 0; i < BK_ROWS / 4; ++i) {
            const int kk = lk + 4 * i;
            const int k = k0 + kk;
            As[kk][lrow] = (r < n && k < nb) ? __ldg(B + (int64_t)k * ld + r) : 0.0;
        }
        for (int e = threadIdx.x; e < BK_ROWS * NT * 8; e += 256) {
            const int kk = e / (NT * 8), o = e % (NT * 8);
            const int k = k0 + kk;
            Hs[kk][o] = (k < nb && o < c) ? H[(int64_t)k * c + o] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k4 = 0; k4 < BK_ROWS; k4 += 4) {
            const double a = As[k4 + (lane & 3)][warp * 8 + (lane >> 2)];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const double b = Hs[k4 + (lane & 3)][t * 8 + (lane >> 2)];
                dmma884(acc[t], a, b);
            }
        }
        __syncthreads();
    }
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

template <int NT>
void launch_tn(dim3 g, int64_t n, int64_t ld, int nb, const double* B, const double* V, int c, int64_t rps,
               double* part, cudaStream_t st) {
    block_tn_kernel<NT><<<g, 256, 0, st>>>(n, ld, nb, B, V, c, rps, part);
}
template <int NT>
void launch_nn(unsigned g, int64_t n, int64_t ld, int nb, const double* B, const double* H, int c, double* V,
               cudaStream_t st) {
    block_nn_kernel<NT><<<g, 256, 0, st>>>(n, ld, nb, B, H, c, V);
}

}  // namespace

int block_tn_splits(int64_t n, int nb) {
    const int64_t cb = ceil_div(nb, BK_COLS);
    // about four waves of 256-thread CTAs, each split at least 4K rows
    int64_t g = ceil_div(4 * 2 * kNumSMs, cb);
    g = std::max<int64_t>(1, std::min<int64_t>(g, ceil_div(n, 4096)));
    return (int)g;
}

int block_tn(int64_t n, int64_t ld, int nb, const double* B, const double* V, int c, double* H, double* part,
             unsigned long long* maxabs, cudaStream_t st) {
    if (c < 1 || c > BK_MAXT * 8) return fail(SC_ERR_VALUE, "block width must be in [1, 40]");
    if (nb <= 0) return SC_OK;
    const int nt = (c + 7) / 8;
    const int g = block_tn_splits(n, nb);
    const int64_t rps = ceil_div(ceil_div(n, g), BK_ROWS) * BK_ROWS;
    const int gs = (int)ceil_div(n, rps);
    dim3 grid((unsigned)ceil_div(nb, BK_COLS), (unsigned)gs);
    switch (nt) {
        case 1: launch_tn<1>(grid, n, ld, nb, B, V, c, rps, part, st); break;
        case 2: launch_tn<2>(grid, n, ld, nb, B, V, c, rps, part, st); break;
        case 3: launch_tn<3>(grid, n, ld, nb, B, V, c, rps, part, st); break;
        case 4: launch_tn<4>(grid, n, ld, nb, B, V, c, rps, part, st); break;
        default: launch_tn<5>(grid, n, ld, nb, B, V, c, rps, part, st); break;
    }
    const int64_t tot = (int64_t)nb * c;
    block_reduce_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(gs, nb, c, nt * 8, part, H, maxabs);
    SC_LAUNCHED(2);
    return SC_OK;
}

int block_nn(int64_t n, int64_t ld, int nb, const double* B, const double* H, int c, double* V, cudaStream_t st) {
    if (c < 1 || c > BK_MAXT * 8) return fail(SC_ERR_VALUE, "block width must be in [1, 40]");
    if (nb <= 0) return SC_OK;
    const int nt = (c + 7) / 8;
    const unsigned g = (unsigned)ceil_div(n, BK_COLS);
    switch (nt) {
        case 1: launch_nn<1>(g, n, ld, nb, B, H, c, V, st); break;
        case 2: launch_nn<2>(g, n, ld, nb, B, H, c, V, st); break;
        case 3: launch_nn<3>(g, n, ld, nb, B, H, c, V, st); break;
        case 4: launch_nn<4>(g, n, ld, nb, B, H, c, V, st); break;
        default: launch_nn<5>(g, n, ld, nb, B, H, c, V, st); break;
    }
    SC_LAUNCHED(1);
    return SC_OK;
}

size_t block_part_size(int64_t n, int nb, int c) {
    const int nt = (c + 7) / 8;
    return (size_t)block_tn_splits(n, nb) * (size_t)nb * (size_t)(nt * 8);
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
