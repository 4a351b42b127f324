// Streaming per-row candidate list shared by the kNN candidate kernels: an
// append buffer of `cap` (key, column) pairs owned by one thread; when full it
// is compacted in place to its R smallest keys and the threshold tau becomes
// the largest kept key, so every discarded or rejected column has key >= tau.
#pragma once
#include <cuda_runtime.h>

namespace sc {

__device__ __noinline__ static float list_compact(float2* L, int cap, int R) {
    int lo = 0, hi = cap - 1, target = R - 1;
    while (lo < hi) {
        float a = L[lo].x, b = L[(lo + hi) >> 1].x, c = L[hi].x;
        float pivot = fmaxf(fminf(a, b), fminf(fmaxf(a, b), c));  // median of three
        int i = lo, j = hi;
        while (i <= j) {
            while (L[i].x < pivot) ++i;
            while (L[j].x > pivot) --j;
            if (i <= j) {
                float2 t = L[i];
                L[i] = L[j];
                L[j] = t;
                ++i;
                --j;
            }
        }
        if (target <= j) hi = j;
        else if (target >= i) lo = i;
        else break;
    }
    float tau = -INFINITY;
    for (int q = 0; q < R; ++q) tau = fmaxf(tau, L[q].x);
    return tau;
}

}  // namespace sc
