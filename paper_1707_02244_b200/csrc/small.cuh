// Persistent single-cluster ISTA for small n (see small.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace clb {
// n in {2048, 4096, 8192} (and CLB_NO_SMALL unset)
bool small_ista_supported(int64_t n, int64_t m);
// Runs `iters` ISTA iterations in one launch on device arrays (c~ fp32, omega int32, y, x in/out,
// r and delta out: the state after the last iteration, as the multi-kernel step leaves it).
cudaError_t launch_small_ista(int64_t n, int64_t m, const float* hc, const int* omega, const float* y, float* x,
                              float* r, float* delta, float tau, float thr, int iters, cudaStream_t st);
}  // namespace clb
