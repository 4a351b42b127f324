// Internal launchers shared between translation units.
#pragma once
#include "sc_common.cuh"

namespace sc {

int spmv_launch(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                const double* vals, const double* x, double* y, bool deterministic,
                cudaStream_t st);
int degrees_launch(int64_t n, const int64_t* row_ptr, const double* vals, double* d,
                   cudaStream_t st);

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
