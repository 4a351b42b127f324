#pragma once
#include "sc_common.cuh"

namespace sc {
// Top-kout eigenpairs of the Lanczos projected matrix T (m x m, column-major,
// not modified) whose rows 0..p-1 are diag(theta) coupled only to row p and
// whose rows p..m-1 are tridiagonal (eigen.py:218-239; p = 0: tridiagonal).
// wsort[m]: all eigenvalues, descending; S (m x kout, ld m): the eigenvectors
// of the kout largest, in that order.  Arrowhead divide and conquer (sc_dc.cu).
int dc_symeig_launch(int m, int p, const double* T, int kout, double* wsort, double* S, cudaStream_t st);
}  // namespace sc
