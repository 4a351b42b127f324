// Internal launchers shared between translation units.
#pragma once
#include "sc_common.cuh"

namespace sc {

int spmv_launch(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                const double* vals, const double* x, double* y, bool deterministic,
                cudaStream_t st);
int degrees_launch(int64_t n, const int64_t* row_ptr, const double* vals, double* d,
                   cudaStream_t st);

// Bulk-staged SpMV plan for an operator applied many times (the Lanczos
// matvecs): the nonzeros are cut into chunks of ~SPMV_CH (whole rows; a chunk
// holds the rows whose first nonzero falls in its window), one persistent CTA
// per SM streams its contiguous run of chunks through a shared-memory ring
// with cp.async.bulk while consumer warps gather x and reduce rows.  Chunks
// that do not fit a stage (hub rows) are read straight from global memory.
constexpr int64_t SPMV_CH = 2048;
constexpr int SPMV_CAP = 3072, SPMV_RCAP = 192, SPMV_STAGES = 3, SPMV_THREADS = 512;
struct SpmvChunk {
    int64_t row_begin, row_end, p_begin, p_end;
    int64_t staged;
};
struct SpmvPlan {
    int64_t n = 0, nnz = 0, nch = 0;
    const int64_t* row_ptr = nullptr;
    const int32_t* col = nullptr;
    const double* vals = nullptr;
    DevBuf<SpmvChunk> chunks;
    int build(int64_t n_, const int64_t* row_ptr, const int32_t* col, const double* vals, cudaStream_t st);
    int apply(const double* x, double* y, cudaStream_t st) const;
};

// Sliced ELLPACK (SELL-32-sigma) copy of a CSR matrix for the eigensolver's
// SpMV: rows are sorted by length (descending, stable) inside windows of
// SELL_SIGMA consecutive rows, every 32 sorted rows form a slice stored
// column-major (entry j of the slice's 32 rows is contiguous), so a warp's
// loads are coalesced, each lane sums one row sequentially with several
// independent gathers in flight, and a block's rows are consecutive (in the
// kNN locality order their x gathers share L1 lines).
// Rows longer than `lcap` (kNN hubs) would stall their slice's warp: they are
// stored empty in the slices and summed by a warp-per-row kernel instead.
constexpr int SELL_SIGMA = 256;
struct SellMatrix {
    int64_t n = 0, nslices = 0, stored = 0, nlong = 0, lcap = 0;
    DevBuf<int32_t> lrows;      // nlong: the long rows
    const int64_t* row_ptr = nullptr;  // CSR kept for the long rows
    const int32_t* csr_col = nullptr;
    const double* csr_vals = nullptr;
    DevBuf<int64_t> slice_ptr;  // nslices + 1 (entries)
    DevBuf<int32_t> width;      // nslices
    DevBuf<int32_t> srow;       // nslices * 32: sorted position -> row (>= n: padding)
    DevBuf<int32_t> slen;       // nslices * 32: row length at that position
    DevBuf<int32_t> col;        // stored
    DevBuf<double> vals;        // stored
    int build(int64_t n_, const int64_t* row_ptr, const int32_t* col_in, const double* vals_in, cudaStream_t st);
    int spmv(const double* x, double* y, cudaStream_t st) const;
};

// Stable bucketing of n items by label in [0, k): members[] lists item
// indices grouped by label, ascending index within a label; start[k+1] are
// the group offsets.  Workspace is owned by the struct.
struct Bucketer {
    int64_t n = 0, k = 0, nblk = 0;
    DevBuf<int32_t> blkcount;   // nblk x k
    DevBuf<int64_t> blkoff;     // nblk x k
    DevBuf<int64_t> start;      // k + 1
    DevBuf<int32_t> members;    // n
    int init(int64_t n_, int64_t k_);
    int run(const int64_t* labels, cudaStream_t st);
};

// labels[i] = index of the nearest of the k rows of c (fp64 Gram-expansion
// distance tiles; ties -> lowest index)
int assign_nearest(int64_t n, int64_t d, const double* v, int64_t k, const double* c, int64_t* labels,
                   cudaStream_t st);

}  // namespace sc
