// Dense ADMM baseline (the paper's PADMM) on the GPU: see dense.cuh.
//
// Setup, fp64 (reference admm_setup, solvers.hpp:285-314, which materializes A~ = A / s, forms
// A~^T A~ + rho I and inverts it with Eigen::LLT):
//  * Gram matrix G = A~^T A~ + rho I by 64 x 64 output tiles (lower-triangle tiles, mirrored), the
//    rows of A~ generated on the fly from the normalized first row and Omega (A~ is never stored);
//  * G^-1 in place by blocked Gauss-Jordan (block 64): per pivot block K, P = G_KK^-1 (one CTA, in
//    shared memory), the panel Z = [-G_iK P ; P], the saved row panel R = G_K*, and the rank-64 update
//    G_ij <- [i not in K] G_ij + Z_i R_j (j not in K), G_iK <- Z_i.  2 n^3 flops, all of them in
//    64 x 64 x 64 register-tiled DFMA products.  G is SPD with spectrum in [rho, 1 + rho] (the operator
//    is spectrally normalized), so the unpivoted elimination is stable.
// Iterations, fp32 (padmm_phases, parallel.hpp:284-317): one warp per row of B streams the row
// (L2-resident: 64 MB at n = 4096) against rhs and applies the z/u update in its epilogue; a second
// elementwise kernel rebuilds rhs.
#include "dense.cuh"

#include <algorithm>

#include "kernels.cuh"

namespace clb {
namespace {

constexpr int kT = kDenseTile;  // 64
constexpr int kKC = 16;         // K chunk staged in shared memory
constexpr int kTT = 256;        // threads per tile CTA: 16 x 16, 4 x 4 outputs each

// acc[a][b] += sum_kk As[kk][ty + 16 a] * Bs[kk][tx + 16 b]
__device__ __forceinline__ void tile_fma(double (&acc)[4][4], const double (*As)[kT], const double (*Bs)[kT], int ty,
                                         int tx) {
#pragma unroll
  for (int kk = 0; kk < kKC; ++kk) {
    double a[4], b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a[q] = As[kk][ty + 16 * q];
      b[q] = Bs[kk][tx + 16 * q];
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
  }
}

// A~[t][j] = c~[(j - omega_t) mod n]; 0 outside [0, n) (the pad)
__device__ __forceinline__ double gen_a(const double* __restrict__ cn, int w, int64_t j, int64_t n) {
  if (j >= n) return 0.0;
  const int64_t k = j - w;
  return cn[k >= 0 ? k : k + n];
}

__global__ void __launch_bounds__(kTT) k_gram(const double* __restrict__ cn, const int* __restrict__ omega, int64_t n,
                                              int64_t m, double rho, double* __restrict__ G, int64_t np) {
  // lower-triangle tile (I, J), J <= I, from the linear block index
  const int64_t b = blockIdx.x;
  int64_t I = static_cast<int64_t>((sqrt(8.0 * static_cast<double>(b) + 1.0) - 1.0) / 2.0);
  while ((I + 1) * (I + 2) / 2 <= b) ++I;
  while (I * (I + 1) / 2 > b) --I;
  const int64_t J = b - I * (I + 1) / 2;
  __shared__ double As[kKC][kT], Bs[kKC][kT];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  double acc[4][4] = {};
  for (int64_t t0 = 0; t0 < m; t0 += kKC) {
#pragma unroll
    for (int q = 0; q < (kKC * kT) / kTT; ++q) {
      const int e = tid + q * kTT, kk = e / kT, r = e % kT;
      const int64_t t = t0 + kk;
      double va = 0.0, vb = 0.0;
      if (t < m) {
        const int w = omega[t];
        va = gen_a(cn, w, I * kT + r, n);
        vb = gen_a(cn, w, J * kT + r, n);
      }
      As[kk][r] = va;
      Bs[kk][r] = vb;
    }
    __syncthreads();
    tile_fma(acc, As, Bs, ty, tx);
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = I * kT + ty + 16 * p, j = J * kT + tx + 16 * q;
      double v = acc[p][q];
      if (i >= n || j >= n) v = 0.0;
      if (i == j) v += i < n ? rho : 1.0;  // identity pad keeps the padded matrix block-diagonal
      G[i * np + j] = v;
      G[j * np + i] = v;
    }
}

__global__ void k_aty(const double* __restrict__ cn, const int* __restrict__ omega, const double* __restrict__ yn,
                      int64_t n, int64_t m, double* __restrict__ aty) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  double acc = 0.0;
  for (int64_t t = 0; t < m; ++t) acc += gen_a(cn, omega[t], j, n) * yn[t];
  aty[j] = acc;
}

// P = G_KK^-1 by unblocked Gauss-Jordan in shared memory (one CTA)
__global__ void __launch_bounds__(kTT) k_gj_pivot(const double* __restrict__ G, int64_t np, int64_t kb,
                                                  double* __restrict__ P) {
  __shared__ double A[kT][kT + 1];
  __shared__ double rowp[kT], colp[kT];
  const int tid = threadIdx.x;
  for (int e = tid; e < kT * kT; e += kTT) A[e / kT][e % kT] = G[(kb * kT + e / kT) * np + kb * kT + e % kT];
  __syncthreads();
  for (int p = 0; p < kT; ++p) {
    if (tid < kT) {
      rowp[tid] = A[p][tid];
      colp[tid] = A[tid][p];
    }
    __syncthreads();
    const double inv = 1.0 / rowp[p];
    for (int e = tid; e < kT * kT; e += kTT) {
      const int i = e / kT, j = e % kT;
      double v;
      if (i == p && j == p) v = inv;
      else if (i == p) v = rowp[j] * inv;
      else if (j == p) v = -colp[i] * inv;
      else v = A[i][j] - colp[i] * rowp[j] * inv;
      A[i][j] = v;
    }
    __syncthreads();
  }
  for (int e = tid; e < kT * kT; e += kTT) P[e] = A[e / kT][e % kT];
}

// CTA b: Z[b rows] = (b == kb) ? P : -G[b rows, K] P;  R[:, b cols] = G[K, b cols]
__global__ void __launch_bounds__(kTT) k_gj_panel(const double* __restrict__ G, int64_t np, int64_t kb,
                                                  const double* __restrict__ P, double* __restrict__ Z,
                                                  double* __restrict__ R) {
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  for (int e = tid; e < kT * kT; e += kTT) {
    const int kk = e / kT, c = e % kT;
    R[kk * np + b * kT + c] = G[(kb * kT + kk) * np + b * kT + c];
  }
  if (b == kb) {
    for (int e = tid; e < kT * kT; e += kTT) Z[(b * kT + e / kT) * kT + e % kT] = P[e];
    return;
  }
  __shared__ double As[kKC][kT], Bs[kKC][kT];
  double acc[4][4] = {};
  for (int k0 = 0; k0 < kT; k0 += kKC) {
#pragma unroll
    for (int q = 0; q < (kKC * kT) / kTT; ++q) {
      const int e = tid + q * kTT;
      const int ra = e / kKC, ka = e % kKC;  // A = G[b rows, K]: As[kk][r]
      As[ka][ra] = G[(b * kT + ra) * np + kb * kT + k0 + ka];
      const int kb2 = e / kT, cb = e % kT;   // B = P: Bs[kk][c]
      Bs[kb2][cb] = P[(k0 + kb2) * kT + cb];
    }
    __syncthreads();
    tile_fma(acc, As, Bs, ty, tx);
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) Z[(b * kT + ty + 16 * p) * kT + tx + 16 * q] = -acc[p][q];
}

// tile (I, J): G[I, J] = (J == kb) ? Z[I] : [I != kb] G[I, J] + Z[I] R[:, J]
__global__ void __launch_bounds__(kTT) k_gj_update(double* __restrict__ G, int64_t np, int64_t kb,
                                                   const double* __restrict__ Z, const double* __restrict__ R) {
  const int64_t T = np / kT;
  const int64_t I = blockIdx.x / T, J = blockIdx.x % T;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  if (J == kb) {
    for (int e = tid; e < kT * kT; e += kTT) G[(I * kT + e / kT) * np + kb * kT + e % kT] = Z[(I * kT + e / kT) * kT + e % kT];
    return;
  }
  __shared__ double As[kKC][kT], Bs[kKC][kT];
  double acc[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q)
      acc[p][q] = I == kb ? 0.0 : G[(I * kT + ty + 16 * p) * np + J * kT + tx + 16 * q];
  for (int k0 = 0; k0 < kT; k0 += kKC) {
#pragma unroll
    for (int q = 0; q < (kKC * kT) / kTT; ++q) {
      const int e = tid + q * kTT;
      const int ra = e / kKC, ka = e % kKC;
      As[ka][ra] = Z[(I * kT + ra) * kT + k0 + ka];
      const int kb2 = e / kT, cb = e % kT;
      Bs[kb2][cb] = R[(k0 + kb2) * np + J * kT + cb];
    }
    __syncthreads();
    tile_fma(acc, As, Bs, ty, tx);
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) G[(I * kT + ty + 16 * p) * np + J * kT + tx + 16 * q] = acc[p][q];
}

// B[i][j] = G[i][j] for i < rows, j < n (G row stride np, B row stride n)
__global__ void k_to_f32(const double* __restrict__ G, int64_t np, int64_t n, float* __restrict__ B, int64_t rows) {
  const int64_t total = rows * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    B[e] = static_cast<float>(G[(e / n) * np + e % n]);
}

__device__ __forceinline__ float soft_d(float v, float g) {  // solvers.hpp:39-44 (strict; NaN -> +0)
  if (v > g) return __fsub_rn(v, g);
  if (v < -g) return __fadd_rn(v, g);
  return 0.f;
}

constexpr int kRowWarps = 8;

__global__ void __launch_bounds__(kRowWarps * 32) k_padmm_primal(PadmmArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double m0 = 0, m1 = 0, m2 = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRowWarps) + warp; i < a.n;
       i += static_cast<int64_t>(gridDim.x) * kRowWarps) {
    const float* row = a.B + i * a.n;
    float acc = 0.f;
    for (int64_t j = lane; j < a.n; j += 32) acc = fmaf(__ldg(row + j), __ldg(a.rhs + j), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const float zo = a.z[i];
      const float zn = soft_d(__fadd_rn(acc, a.u[i]), a.thr);
      a.x[i] = acc;
      a.z[i] = zn;
      a.u[i] = __fadd_rn(a.u[i], __fsub_rn(acc, zn));
      if (a.want_metrics) {
        const double dd = static_cast<double>(zn) - static_cast<double>(zo);
        m0 += dd * dd;
        if (a.truth) {
          const double dt = static_cast<double>(zn) - static_cast<double>(a.truth[i]);
          m1 += dt * dt;
        }
        if (!isfinite(zn)) m2 += 1.0;
      }
    }
  }
  if (!a.want_metrics) return;
  __shared__ double sm[3][kRowWarps];
  if (lane == 0) {
    sm[0][warp] = m0;
    sm[1][warp] = m1;
    sm[2][warp] = m2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // fixed order: deterministic
    double s0 = 0, s1 = 0, s2 = 0;
    for (int w = 0; w < kRowWarps; ++w) {
      s0 += sm[0][w];
      s1 += sm[1][w];
      s2 += sm[2][w];
    }
    a.blk[blockIdx.x * 4] = s0;
    a.blk[blockIdx.x * 4 + 1] = s1;
    a.blk[blockIdx.x * 4 + 2] = s2;
    a.blk[blockIdx.x * 4 + 3] = 0.0;
  }
}

__global__ void k_padmm_rhs(const float* __restrict__ aty, const float* __restrict__ z, const float* __restrict__ u,
                            float rho, float* __restrict__ rhs, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    rhs[i] = __fadd_rn(aty[i], __fmul_rn(rho, __fsub_rn(z[i], u[i])));
}

}  // namespace

void launch_dense_gram(const double* cn, const int* omega, int64_t n, int64_t m, double rho, double* G, int64_t np,
                       cudaStream_t st) {
  const int64_t T = np / kT;
  k_gram<<<static_cast<unsigned>(T * (T + 1) / 2), kTT, 0, st>>>(cn, omega, n, m, rho, G, np);
}

void launch_dense_aty(const double* cn, const int* omega, const double* yn, int64_t n, int64_t m, double* aty,
                      cudaStream_t st) {
  k_aty<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(cn, omega, yn, n, m, aty);
}

size_t dense_gj_scratch(int64_t np) { return static_cast<size_t>(kT * kT + 2 * np * kT); }

void launch_dense_invert(double* G, int64_t np, double* scratch, double* /*pivot_min*/, cudaStream_t st) {
  const int64_t T = np / kT;
  double* P = scratch;
  double* Z = P + kT * kT;
  double* R = Z + np * kT;
  for (int64_t kb = 0; kb < T; ++kb) {
    k_gj_pivot<<<1, kTT, 0, st>>>(G, np, kb, P);
    k_gj_panel<<<static_cast<unsigned>(T), kTT, 0, st>>>(G, np, kb, P, Z, R);
    k_gj_update<<<static_cast<unsigned>(T * T), kTT, 0, st>>>(G, np, kb, Z, R);
  }
}

void launch_dense_to_f32(const double* G, int64_t np, int64_t n, float* B32, cudaStream_t st) {
  k_to_f32<<<148 * 8, 256, 0, st>>>(G, np, n, B32, n);
}

void launch_f64_to_f32(const double* a, int64_t count, float* out, cudaStream_t st) {
  // one row of `count` entries
  k_to_f32<<<static_cast<unsigned>(std::min<int64_t>(148 * 8, (count + 255) / 256)), 256, 0, st>>>(a, count, count,
                                                                                                     out, 1);
}

void launch_padmm_primal(const PadmmArgs& a, cudaStream_t st) {
  const int64_t blocks = a.want_metrics ? kEpiBlocks
                                        : std::min<int64_t>(kEpiBlocks, (a.n + kRowWarps - 1) / kRowWarps);
  k_padmm_primal<<<static_cast<unsigned>(blocks), kRowWarps * 32, 0, st>>>(a);
}

void launch_padmm_rhs(const float* aty, const float* z, const float* u, float rho, float* rhs, int64_t n,
                      cudaStream_t st) {
  k_padmm_rhs<<<static_cast<unsigned>(std::min<int64_t>(148 * 4, (n + 255) / 256)), 256, 0, st>>>(aty, z, u, rho,
                                                                                                 rhs, n);
}

}  // namespace clb
