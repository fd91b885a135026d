// Probe for the tcgen05 dense circulant product (csrc/tc_dense.cu): correctness on sampled
// outputs against an fp64 host sum, and CUDA-event timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1707_02244_b200/csrc \
//        -o tc_probe tc_probe.cu ../../paper_1707_02244_b200/csrc/tc_dense.cu
//   ./tc_probe [log2 n] [reps]
// Environment: CLB_TC_F16=0/1 (operand format; default fp16 for n >= 2^18), CLB_TC_SPLITS=S,
// CLB_TC_PAIR=0 (single CTAs instead of cta_group::2 pairs).
// Build flags used in the DESIGN experiments: -DTC_SPD=k (TF32 steps per drain; fp16 uses 2k).
// The tensor-flop column counts 3 tensor flops per algorithmic flop for either format.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "tc_dense.cuh"

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

int main(int argc, char** argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 20;
  const int reps = argc > 2 ? atoi(argv[2]) : 5;
  const int64_t n = int64_t(1) << lg;
  std::mt19937_64 rng(7);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> h(n), u(n);
  for (auto& v : h) v = nd(rng);
  for (auto& v : u) v = nd(rng);
  clb::ConvPlan p = clb::make_tc_plan(n);
  printf("n=2^%d tiles=%lld splits=%d units=%lld\n", lg, (long long)p.tiles, p.splits,
         (long long)(p.tiles * p.splits));
  float *dh, *du, *dp;
  CK(cudaMalloc(&dh, n * 4));
  CK(cudaMalloc(&du, n * 4));
  CK(cudaMalloc(&dp, n * 4 * p.splits));
  CK(cudaMemcpy(dh, h.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(du, u.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dp, 0, n * 4 * p.splits));
  CK(cudaMalloc(&p.tc_scratch, clb::tc_scratch_floats() * 4));
  CK(clb::launch_tc_dense(p, dh, du, dp, 0));
  CK(cudaDeviceSynchronize());
  std::vector<float> part(n * p.splits);
  CK(cudaMemcpy(part.data(), dp, n * 4 * p.splits, cudaMemcpyDeviceToHost));
  double max_rel = 0, max_abs = 0, ref_norm = 0;
  const int samples = 64;
  for (int t = 0; t < samples; ++t) {
    const int64_t i = (t < 8) ? t * 257 : (int64_t)(rng() % n);
    double ref = 0, mag = 0;
    for (int64_t j = 0; j < n; ++j) {
      const double a = (double)h[(i - j) & (n - 1)] * u[j];
      ref += a;
      mag += std::fabs(a);
    }
    double got = 0;
    for (int s = 0; s < p.splits; ++s) got += part[s * n + i];
    const double err = std::fabs(got - ref);
    max_abs = std::max(max_abs, err);
    max_rel = std::max(max_rel, err / mag);
    ref_norm = std::max(ref_norm, std::fabs(ref));
    if (t < 4) printf("  i=%lld ref=%.6f got=%.6f\n", (long long)i, ref, got);
  }
  printf("max |err| %.3e   max |err| / sum|terms| %.3e   (max |ref| %.3f)\n", max_abs, max_rel, ref_norm);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) CK(clb::launch_tc_dense(p, dh, du, dp, 0));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;
  const double useful = 2.0 * double(n) * double(n);
  printf("time %.3f ms   useful %.1f TFLOP/s   tensor (3xTF32) %.1f TFLOP/s\n", ms, useful / ms * 1e-9,
         3 * useful / ms * 1e-9);
  return 0;
}
