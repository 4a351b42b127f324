#pragma once
#include "sc_common.cuh"

namespace sc {
int knn_graph_build(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq, int64_t* row_ptr,
                    int32_t* col, double* vals, int64_t* nnz_out, int64_t* stats, cudaStream_t st);
}  // namespace sc
