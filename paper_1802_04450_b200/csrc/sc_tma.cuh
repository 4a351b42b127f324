// Tensor-map helpers shared by the tcgen05 kernels (kNN candidates, k-means
// assignment).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include "sc_common.cuh"

namespace sc {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
// 2-D map over a rows x dp fp16 row-major matrix: 64 x 128 boxes, 128-byte
// swizzle (the K-major UMMA operand layout of sc_tc.cuh)
int make_f16_tile_map(CUtensorMap* map, const __half* base, int64_t rows, int64_t dp);
}  // namespace sc
