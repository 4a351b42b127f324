#pragma once
#include "sc_common.cuh"

namespace sc {
// H (nb x c, row-major) = B[:, :nb]^T V over n rows; B, V column-major with
// leading dimension ld.  part: block_part_size(n, nb, c) doubles of scratch;
// maxabs (dev, optional, zeroed by the caller) receives max |H| as ordered bits.
int block_tn(int64_t n, int64_t ld, int nb, const double* B, const double* V, int c, double* H, double* part,
             unsigned long long* maxabs, cudaStream_t st);
// V -= B[:, :nb] H
int block_nn(int64_t n, int64_t ld, int nb, const double* B, const double* H, int c, double* V, cudaStream_t st);
size_t block_part_size(int64_t n, int nb, int c);
}  // namespace sc
