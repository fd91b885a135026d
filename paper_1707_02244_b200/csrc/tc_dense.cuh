// Dense circulant product on the 5th-generation tensor cores (tcgen05; 3xTF32 or an fp16
// 2-term split, both fp32-grade).
//
//   out[i] = sum_j h[(i - j) mod n] u[j]        (the cADMM products, parallel.hpp:173-231)
//
// Blocking n into b = 256 turns the product into a sum over block offsets D of
// GEMMs between a Hankel tile of h and a row-shifted view of u ("Tensor-core
// products").
// Both operands are shared-memory descriptor views; the accumulator lives in TMEM.
// Output: split-K partials partial[s * n + i], summed by the same epilogues as the
// FFMA dense kernel (fixed split order: deterministic, a function of n only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace clb {

// Power-of-two n with at least one 128-block tile (n >= 2^15).
bool tc_dense_supported(int64_t n);
// Plan for the tensor-core kernel: tile = 128 * 256 outputs, splits over the block offsets.
ConvPlan make_tc_plan(int64_t n);
void tc_dense_init();
// Floats of per-product scratch the fp16 operand path needs (ConvPlan::tc_scratch).
size_t tc_scratch_floats();
// Launch errors (including a missing scratch buffer) are returned, not deferred.
cudaError_t launch_tc_dense(const ConvPlan& p, const float* h, const float* u, float* partial, cudaStream_t st);

}  // namespace clb
