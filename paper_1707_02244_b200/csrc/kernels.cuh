// Device kernels of the direct (shift-indexed) circulant engine, sm_100a.
//
// Every circulant product of the reference hot path is expressed as one
// circular convolution
//     out[i] = sum_j h[(i - j) mod n] * u[j]
// with h a (possibly index-reversed) first row:
//   C^T v   (cpadmm primal,   parallel.hpp:178-191)  h = c
//   B beta  (cpadmm recovery, parallel.hpp:193-205)  h = b_rev, b_rev[k] = b[-k mod n]
//   C x     (cpadmm duals,    parallel.hpp:207-228)  h = c_rev
//   A^T r   (cpista gradient, parallel.hpp:258-276)  h = c,     u = P^T r (rows only)
//   (A x)_t (cpista residual, parallel.hpp:243-256)  h = c_rev, outputs only at rows omega
//
// Work decomposition (fixed by n and m only, never by the GPU count, so
// results are bitwise identical for any sharding):
//   tile  = kThreads * R consecutive register-owned indices (R per thread),
//   chunk = kChunk consecutive positions staged in shared memory,
//   split = a contiguous range of 32-position blocks (whole chunks at large n,
//           fractions of a chunk at small n); a unit (tile, split) is one CTA.
// Partial sums of the splits (or of the tiles, for the residual) are combined
// in ascending order by the epilogue kernels, which also apply the fused
// solver updates.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace clb {

// Kernel function attributes (max dynamic shared memory, cluster sizes) are set per device.
// True the first time it is called for the current device with this flag word; callers set the
// attributes then.  (A process may drive several devices through SolverConfig::device.)
inline bool first_use_on_device(std::atomic<uint64_t>& flags) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const uint64_t bit = uint64_t(1) << dev;
  return (flags.fetch_or(bit) & bit) == 0;
}

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;   // 128
constexpr int kP = 32;                  // positions per register window block
constexpr int kChunk = 1024;            // positions per shared-memory stage
// Split-count target (CTAs per product), a function of n only, so the decomposition and the
// results are independent of the GPU count.  Large n: 96 x 148 units -- smaller CTAs balance the
// waves (C3 step 37.3 -> 34.1 ms, cADMM products 40.8 -> 36.3 ms at n = 2^20; flat from 64 to
// 128 x 148) and leave 12 CTAs per SM when a product is sharded over 8 GPUs.  Below 2^19 the
// split-K partial traffic would dominate, so 8 x 148.
constexpr int kTargetUnits = 1184;
constexpr int kTargetUnitsLarge = 14208;
constexpr int64_t kUnitsLargeN = int64_t(1) << 19;
int64_t target_units(int64_t n);  // CLB_UNITS overrides (experiments)
constexpr int kEpiBlocks = 592;         // grid of the elementwise epilogues (fixed -> deterministic metrics)

// Register blocking of the dense kernel (indices owned per thread); the
// sparse kernels' R comes from the variant selected for n (grad_R(n), res_R(n)).
constexpr int kRDense = 64;
int grad_R(int64_t n);
int dense_R(int64_t n);  // R of the selected dense-product kernel (kRDense by default)
int res_R(int64_t n);

struct ConvPlan {
  int64_t n = 0;
  int64_t tile = 0;     // kThreads * R
  int64_t tiles = 0;    // ceil(n / tile)
  int64_t chunks = 0;   // ceil(n / kChunk)
  int splits = 1;       // S
  int64_t tile_lo = 0, tile_hi = 0;    // shard: tiles run by this rank
  int split_lo = 0, split_hi = 0;      // shard: splits run by this rank (residual)
  bool tc = false;                     // dense product on the tensor cores (tc_dense.cu)
  // tensor-core fp16 path: device scratch of tc_scratch_floats() floats for the operand scales,
  // owned by the caller (one per solver / product; never shared between streams)
  float* tc_scratch = nullptr;
};

ConvPlan make_plan(int64_t n, int R);
// Plan of the cADMM dense products: the tcgen05 kernel (tc_dense.cu) for power-of-two
// n >= 2^15 unless CLB_NO_TC=1, else the FFMA kernel.  Pure host logic.
ConvPlan make_dense_plan(int64_t n);
// ISTA's direct engine embeds both sparse products in dense tensor-core products for
// n >= 2^17 (where that beats the FFMA sparse kernels).  Pure host logic.
bool ista_uses_tc(int64_t n);
// [blo, bhi) in 32-position blocks covered by split `split` of a plan.
void split_block_range(const ConvPlan& p, int split, int64_t* blo, int64_t* bhi);

// Epilogue parameter block (device pointers; unused ones may be null).
struct EpiArgs {
  const float* partial = nullptr;  // [splits][n] (or [tiles][m] for the residual)
  int splits = 1;
  int64_t n = 0, lo = 0, hi = 0;   // element range [lo, hi) processed; n = partial stride
  // ISTA
  const float* y = nullptr;        // residual: r = y - sum
  float* r = nullptr;
  float* x = nullptr;
  float* delta = nullptr;
  float tau = 0.f, thr = 0.f;
  // cADMM
  const float *d = nullptr, *pty = nullptr;
  float *z = nullptr, *nu = nullptr, *mu = nullptr, *v = nullptr, *beta = nullptr;
  float rho = 0.f, sigma = 0.f, tau1 = 1.f, tau2 = 1.f;
  // check metrics
  const float* truth = nullptr;
  double* blk = nullptr;           // [kEpiBlocks][4]: sum d_iter^2, sum d_truth^2, nonfinite, unused
  int want_metrics = 0;
  int vec4 = 0;  // set by launch_admm_duals: the unchecked single-split form (the FFT engine) in 16-byte accesses
  // sharded solves with the peer-store transport: the vector this epilogue produces (r, x, beta or v) is
  // also stored, at the same indices, into every other rank's copy of it (device pointers on the same or a
  // peer-accessible GPU) -- the all-gather fused into the producing kernel
  static constexpr int kMaxPeers = 7;
  float* peer[kMaxPeers] = {};
  int npeer = 0;
};

// partial[split][i] for the plan's shard tiles (dense u).  plan from make_plan(n, kRDense).
cudaError_t launch_conv_dense(const ConvPlan& p, const float* h, const float* u, float* partial, cudaStream_t st);
// gradient: u = P^T r given as rows (omega32 sorted, rvals), rowstart[chunk].  plan R = kRGrad.
void launch_conv_rows(const ConvPlan& p, const float* h, const int* omega32, const float* rvals,
                      const int* rowstart, float* partial, cudaStream_t st);
// residual: partial[tile][t] = sum_{j in tile} h[omega[t]-j] x[j] for rows of the shard's splits.  R = kRRes.
void launch_conv_residual(const ConvPlan& p, int64_t m, const float* h, const float* x, const int* omega32,
                          const int* rowstart, float* partial, cudaStream_t st);

void launch_ista_residual_reduce(const EpiArgs& a, int64_t tiles, cudaStream_t st);
// r[t] = y[t] - sum_s partial[s][omega[t]] for t in [a.lo, a.hi) (dense-embedded residual)
void launch_ista_residual_gather(const EpiArgs& a, const int* omega, cudaStream_t st);
void launch_ista_update(const EpiArgs& a, cudaStream_t st);
void launch_admm_beta(const EpiArgs& a, cudaStream_t st);
void launch_admm_x(const EpiArgs& a, cudaStream_t st);
void launch_admm_duals(const EpiArgs& a, cudaStream_t st);
void launch_metrics_final(const double* blk, double* out4, cudaStream_t st);

void conv_kernels_init();

// matvec scheme benchmark: dense row-major copy of the circulant and a plain dense GEMV
void launch_materialize_circulant(const float* c, float* M, int64_t n, cudaStream_t st);
void launch_dense_gemv(const float* M, const float* x, float* out, int64_t n, cudaStream_t st);

// Persistent cooperative cADMM for n in {2048, 4096, 8192} (CLB_NO_SMALL unset): all unchecked iterations
// in one launch; partial holds n/32 x n floats.
bool coop_cadmm_supported(int64_t n);
cudaError_t launch_coop_cadmm(int64_t n, const float* hc, const float* hbr, const float* hcr, const float* d,
                              const float* pty, float* x, float* z, float* nu, float* mu, float* v, float* beta,
                              float* partial, float rho, float sigma, float tau1, float tau2, float thr, int iters,
                              cudaStream_t st);

// Persistent cooperative ISTA (same n); partial holds n/32 x n floats.
cudaError_t launch_coop_ista(int64_t n, int64_t m, const float* hc, const float* hcr, const int* omega,
                             const float* y, float* x, float* r, float* delta, float* partial, float tau, float thr,
                             int iters, cudaStream_t st);

// FFMA throughput microkernel (roofline denominator), returns TFLOP/s.
double ffma_peak_tflops(int device);

}  // namespace clb
