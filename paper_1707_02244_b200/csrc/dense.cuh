// Dense ADMM baseline on the GPU (the paper's PADMM; reference solvers.hpp:267-327,
// parallel.hpp:284-317): the explicit n x n inverse B = (A~^T A~ + rho I)^-1 built once in fp64
// on the device, then one fp32 mat-vec with the fused z/u update per iteration.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace clb {

constexpr int kDenseTile = 64;  // Gauss-Jordan block and GEMM tile

// Padded order of the fp64 working matrix: n rounded up to the tile (the pad is an identity block).
inline int64_t dense_pad(int64_t n) { return (n + kDenseTile - 1) / kDenseTile * kDenseTile; }

// G = A~^T A~ + rho I (np x np, row-major, identity pad), A~[t][j] = c~[(j - omega_t) mod n] generated
// on the fly from the normalized first row c~ (fp64) and the rows omega (int32, sorted).
void launch_dense_gram(const double* cn, const int* omega, int64_t n, int64_t m, double rho, double* G, int64_t np,
                       cudaStream_t st);
// aty[j] = sum_t A~[t][j] y~[t] (j < n), ascending t.
void launch_dense_aty(const double* cn, const int* omega, const double* yn, int64_t n, int64_t m, double* aty,
                      cudaStream_t st);
// In-place inverse of the SPD matrix G (np x np) by blocked Gauss-Jordan without pivoting (B = G^-1 has
// condition <= (1 + rho) / rho on the normalized operator, so no pivoting is needed); scratch holds
// dense_gj_scratch(np) doubles.  `pivot_min` receives the smallest pivot-block determinant proxy (the
// smallest diagonal pivot met, for the singularity check).
size_t dense_gj_scratch(int64_t np);
void launch_dense_invert(double* G, int64_t np, double* scratch, double* pivot_min, cudaStream_t st);
// B32[i][j] = (float) G[i][j] for i, j < n (row stride n)
void launch_dense_to_f32(const double* G, int64_t np, int64_t n, float* B32, cudaStream_t st);
void launch_f64_to_f32(const double* a, int64_t count, float* out, cudaStream_t st);

// One padmm iteration, phase 1 (primal and dual update, parallel.hpp:290-304):
//   x_i = sum_j B[i][j] rhs_j,  z_i = eta(x_i + u_i, thr),  u_i += x_i - z_i;
// with the run loop's check metrics (|z - z_prev|^2, |z - truth|^2, non-finite count) into blk
// ([kEpiBlocks][4]) when want_metrics.
struct PadmmArgs {
  const float* B = nullptr;
  const float* rhs = nullptr;
  float *x = nullptr, *z = nullptr, *u = nullptr;
  const float* truth = nullptr;
  double* blk = nullptr;
  int64_t n = 0;
  float thr = 0.f;
  int want_metrics = 0;
};
void launch_padmm_primal(const PadmmArgs& a, cudaStream_t st);
// phase 2 (parallel.hpp:306-314): rhs_i = aty_i + rho (z_i - u_i)
void launch_padmm_rhs(const float* aty, const float* z, const float* u, float rho, float* rhs, int64_t n,
                      cudaStream_t st);

}  // namespace clb
