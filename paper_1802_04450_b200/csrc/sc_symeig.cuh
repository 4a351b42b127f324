#pragma once
#include "sc_common.cuh"

namespace sc {
// Eigen-decomposition of the m x m symmetric matrix `a` (column-major,
// destroyed).  w_sorted[m] receives all eigenvalues in stable descending
// order, z_sorted (m x kout, column-major, ld m) the matching first kout
// eigenvectors.  z and w_raw are m*m and m scratch; *info (dev) != 0 on QL
// non-convergence.
int symeig_launch(int m, int kout, double* a, double* z, double* w_raw, double* w_sorted,
                  double* z_sorted, int* info, cudaStream_t st);
}  // namespace sc
