// Direct shift-indexed circulant kernels for sm_100a (see kernels.cuh for the
// index algebra and the work decomposition).
//
// Register tiling.  A thread owns R consecutive indices.  For a block of
// kP = 32 consecutive positions it loads an (R + kP)-float window of the
// first row from shared memory ((R + kP) / 4 x LDS.128) and then
//   * dense / gradient kernels (outer-product form, one broadcast scalar
//     shared by R consecutive FFMAs):  acc[q] += w[q - s + kP] * u[s]
//   * residual kernel (dot form, rows are the outputs):
//       out[s] = sum_q w[s - q + R] * x[q]      x[q] register-resident
// Every register index is a compile-time constant.  The data-dependent row
// positions (omega is a random subset, density m/n) are handled by 32
// statically indexed bodies per block, each behind a warp-uniform bit test of
// the block's row mask: straight-line code, no jump table, no dynamic
// register indexing.
//
// Shared memory.  Lanes own windows R floats apart; a plain layout would put
// all 8 lanes of an LDS.128 phase in one bank group.  The staged row is padded
// by 4 floats every R elements (lane pitch R + 4 words), which spreads the 8
// lanes of every phase over 8 distinct bank groups.
#include <climits>
#include <cstdio>

#include "kernels.cuh"

namespace clb {

namespace {

constexpr int kBlocks = kChunk / kP;  // position blocks per chunk
static_assert(kChunk % 64 == 0 && kP == 32, "window phase logic assumes kP = 32");

template <int R>
struct Geo {
  static_assert(R == 32 || R == 64, "R must be 32 or 64");
  static constexpr int kTileR = kThreads * R;
  static constexpr int kSeg = kTileR + kChunk;
  __host__ __device__ static constexpr int pad(int e) { return e + 4 * (e / R); }
  static constexpr int kSegPhys = pad(kSeg) + 4;
  static constexpr int kPitch = R + 4;
};

// hs[pad(e)] = h[(base + e) mod n] for e in [0, kSeg).
template <int R>
__device__ __forceinline__ void stage_segment(float* __restrict__ hs, const float* __restrict__ h, int64_t n,
                                              int64_t base) {
  using G = Geo<R>;
  int64_t b = base % n;
  if (b < 0) b += n;
  if ((n & 3) == 0) {
    if (b + G::kSeg <= n) {  // no wrap inside the segment: plain coalesced copy
      const float* src = h + b;
      for (int e = threadIdx.x * 4; e < G::kSeg; e += kThreads * 4)
        *reinterpret_cast<float4*>(hs + G::pad(e)) = __ldg(reinterpret_cast<const float4*>(src + e));
    } else {
      for (int e = threadIdx.x * 4; e < G::kSeg; e += kThreads * 4) {
        int64_t src = b + e;
        if (src >= n) src %= n;
        *reinterpret_cast<float4*>(hs + G::pad(e)) = __ldg(reinterpret_cast<const float4*>(h + src));
      }
    }
  } else {
    for (int e = threadIdx.x; e < G::kSeg; e += kThreads) hs[G::pad(e)] = __ldg(h + (b + e) % n);
  }
}

// Lane window w[k] = seg[x + k], k in [0, R + kP), for x a multiple of 32.
template <int R, int PH>
__device__ __forceinline__ void load_window_ph(float (&w)[R + kP], const float* __restrict__ p) {
  using G = Geo<R>;
#pragma unroll
  for (int k = 0; k < R + kP; k += 4) {
    const float4 t = *reinterpret_cast<const float4*>(p + (G::pad(PH + k) - PH));
    w[k] = t.x;
    w[k + 1] = t.y;
    w[k + 2] = t.z;
    w[k + 3] = t.w;
  }
}
template <int R>
__device__ __forceinline__ void window_at(float (&w)[R + kP], const float* __restrict__ lane_base, int x) {
  const float* p = lane_base + (x / R) * (R + 4) + (x % R);
  if (R == 64 && (x & 32)) load_window_ph<R, 32 % R>(w, p);
  else load_window_ph<R, 0>(w, p);
}

// ---- outer-product body: acc[q] += w[q - S + kP] * r ----------------------
template <int R, int S>
__device__ __forceinline__ void grad_body(float (&acc)[R], const float (&w)[R + kP], float r) {
#pragma unroll
  for (int q = 0; q < R; ++q) acc[q] = fmaf(w[q - S + kP], r, acc[q]);
}

// ---- dot body: sum_q w[S - q + R] * x[q] ----------------------------------
template <int R, int S>
__device__ __forceinline__ float res_body(const float (&w)[R + kP], const float (&x)[R]) {
  float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
  for (int q = 0; q < R; q += 4) {
    p0 = fmaf(w[S - q + R], x[q], p0);
    p1 = fmaf(w[S - q - 1 + R], x[q + 1], p1);
    p2 = fmaf(w[S - q - 2 + R], x[q + 2], p2);
    p3 = fmaf(w[S - q - 3 + R], x[q + 3], p3);
  }
  return (p0 + p1) + (p2 + p3);
}

// ===========================================================================
// Dense circular convolution (cADMM products).  unit = (tile, split).
// ===========================================================================
template <int R>
__global__ void __launch_bounds__(kThreads, 2)
k_conv_dense(const float* __restrict__ h, const float* __restrict__ u, int64_t n, int64_t chunks, int splits,
             int64_t tile_lo, float* __restrict__ partial) {
  using G = Geo<R>;
  extern __shared__ float4 smem_f4[];
  float* hs = reinterpret_cast<float*>(smem_f4);
  float* us = hs + G::kSegPhys;
  const int64_t unit = blockIdx.x;
  const int64_t tile = tile_lo + unit / splits;
  const int split = static_cast<int>(unit % splits);
  const int64_t I0 = tile * G::kTileR;
  const int64_t c0 = split * chunks / splits, c1 = (split + 1) * chunks / splits;
  const int own = threadIdx.x;
  const float* lane_base = hs + own * G::kPitch;

  float acc[R];
#pragma unroll
  for (int q = 0; q < R; ++q) acc[q] = 0.f;

  for (int64_t ch = c0; ch < c1; ++ch) {
    const int64_t Jc = ch * kChunk;
    stage_segment<R>(hs, h, n, I0 - Jc - kChunk);
    for (int s = threadIdx.x; s < kChunk; s += kThreads) {
      const int64_t j = Jc + s;
      us[s] = j < n ? __ldg(u + j) : 0.f;
    }
    __syncthreads();
    for (int b = 0; b < kBlocks; ++b) {
      float w[R + kP];
      window_at<R>(w, lane_base, kChunk - (b + 1) * kP);
#pragma unroll
      for (int s4 = 0; s4 < kP; s4 += 4) {
        const float4 uu = *reinterpret_cast<const float4*>(us + b * kP + s4);
        const float uv[4] = {uu.x, uu.y, uu.z, uu.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
#pragma unroll
          for (int q = 0; q < R; ++q) acc[q] = fmaf(w[q - (s4 + e) + kP], uv[e], acc[q]);
        }
      }
    }
    __syncthreads();
  }
  const int64_t ib = I0 + own * R;
  float* out = partial + static_cast<int64_t>(split) * n;
#pragma unroll
  for (int q = 0; q < R; ++q)
    if (ib + q < n) out[ib + q] = acc[q];
}

// ===========================================================================
// Gradient A^T r: convolution with the sparse input P^T r, rows only.
// The staged chunk holds r scattered to its positions (zeros elsewhere) and
// a 32-bit row mask per 32-position block (a zero residual contributes
// exactly nothing, so value != 0 is the mask).
// ===========================================================================
template <int R, int S>
__device__ __forceinline__ void grad_pos(float (&acc)[R], const float (&w)[R + kP], uint32_t mask, float r) {
  if (mask & (1u << S)) grad_body<R, S>(acc, w, r);
}

template <int R, int G>
__device__ __forceinline__ void grad_group(float (&acc)[R], const float (&w)[R + kP], uint32_t mask,
                                           const float* __restrict__ rb) {
  if (mask & (0xFu << (4 * G))) {
    const float4 r4 = *reinterpret_cast<const float4*>(rb + 4 * G);
    grad_pos<R, 4 * G>(acc, w, mask, r4.x);
    grad_pos<R, 4 * G + 1>(acc, w, mask, r4.y);
    grad_pos<R, 4 * G + 2>(acc, w, mask, r4.z);
    grad_pos<R, 4 * G + 3>(acc, w, mask, r4.w);
  }
}

template <int R>
__global__ void __launch_bounds__(kThreads, 3)
k_conv_rows(const float* __restrict__ h, const int* __restrict__ omega, const float* __restrict__ rv,
            const int* __restrict__ rowstart, int64_t n, int64_t chunks, int splits, int64_t tile_lo,
            float* __restrict__ partial) {
  using Gm = Geo<R>;
  extern __shared__ float4 smem_f4[];
  float* hs = reinterpret_cast<float*>(smem_f4);
  float* rd = hs + Gm::kSegPhys;                                   // [kChunk] r scattered
  uint32_t* bmask = reinterpret_cast<uint32_t*>(rd + kChunk);      // [kBlocks]
  const int64_t unit = blockIdx.x;
  const int64_t tile = tile_lo + unit / splits;
  const int split = static_cast<int>(unit % splits);
  const int64_t I0 = tile * Gm::kTileR;
  const int64_t c0 = split * chunks / splits, c1 = (split + 1) * chunks / splits;
  const int own = threadIdx.x, warp = own >> 5, lane = own & 31;
  const float* lane_base = hs + own * Gm::kPitch;

  float acc[R];
#pragma unroll
  for (int q = 0; q < R; ++q) acc[q] = 0.f;

  for (int64_t ch = c0; ch < c1; ++ch) {
    const int64_t Jc = ch * kChunk;
    const int r0 = rowstart[ch], nr = rowstart[ch + 1] - r0;
    if (nr == 0) continue;  // uniform across the CTA
    stage_segment<R>(hs, h, n, I0 - Jc - kChunk);
    for (int s = threadIdx.x; s < kChunk; s += kThreads) rd[s] = 0.f;
    __syncthreads();
    for (int k = threadIdx.x; k < nr; k += kThreads) rd[omega[r0 + k] - static_cast<int>(Jc)] = __ldg(rv + r0 + k);
    __syncthreads();
    for (int b = warp; b < kBlocks; b += kWarps) {
      const uint32_t mk = __ballot_sync(0xffffffffu, rd[b * kP + lane] != 0.f);
      if (lane == 0) bmask[b] = mk;
    }
    __syncthreads();
    for (int b = 0; b < kBlocks; ++b) {
      const uint32_t mask = bmask[b];
      if (mask == 0u) continue;
      float w[R + kP];
      window_at<R>(w, lane_base, kChunk - (b + 1) * kP);
      const float* rb = rd + b * kP;
      grad_group<R, 0>(acc, w, mask, rb);
      grad_group<R, 1>(acc, w, mask, rb);
      grad_group<R, 2>(acc, w, mask, rb);
      grad_group<R, 3>(acc, w, mask, rb);
      grad_group<R, 4>(acc, w, mask, rb);
      grad_group<R, 5>(acc, w, mask, rb);
      grad_group<R, 6>(acc, w, mask, rb);
      grad_group<R, 7>(acc, w, mask, rb);
    }
    __syncthreads();
  }
  const int64_t ib = I0 + own * R;
  float* out = partial + static_cast<int64_t>(split) * n;
#pragma unroll
  for (int q = 0; q < R; ++q)
    if (ib + q < n) out[ib + q] = acc[q];
}

// ===========================================================================
// Residual (A x)_t: rows are the outputs, x is register-resident.
// unit = (input tile, split of position chunks); partial[tile][t].
// Per block the selected positions compute their lane-partial dots into
// statically indexed registers; one transpose-reduce across the warp then
// leaves lane L with the warp sum of position L, which it stores to the row's
// slot.  Warps are combined in fixed order at the end of the chunk.
// ===========================================================================
template <int R, int S>
__device__ __forceinline__ void res_pos(const float (&w)[R + kP], const float (&xr)[R], uint32_t mask,
                                        float (&out)[kP]) {
  if (mask & (1u << S)) out[S] = res_body<R, S>(w, xr);
  else out[S] = 0.f;
}

template <int R, int G>
__device__ __forceinline__ void res_group(const float (&w)[R + kP], const float (&xr)[R], uint32_t mask,
                                          float (&out)[kP]) {
  if (mask & (0xFu << (4 * G))) {
    res_pos<R, 4 * G>(w, xr, mask, out);
    res_pos<R, 4 * G + 1>(w, xr, mask, out);
    res_pos<R, 4 * G + 2>(w, xr, mask, out);
    res_pos<R, 4 * G + 3>(w, xr, mask, out);
  } else {
    out[4 * G] = out[4 * G + 1] = out[4 * G + 2] = out[4 * G + 3] = 0.f;
  }
}

// After the call lane L holds sum over the warp's lanes of v[L] in v[0].
__device__ __forceinline__ void transpose_reduce32(float (&v)[kP], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
}

template <int R>
__global__ void __launch_bounds__(kThreads, 3)
k_conv_residual(const float* __restrict__ h, const float* __restrict__ x, const int* __restrict__ omega,
                const int* __restrict__ rowstart, int64_t n, int64_t m, int64_t chunks, int splits,
                int split_lo, int split_cnt, float* __restrict__ partial) {
  using Gm = Geo<R>;
  extern __shared__ float4 smem_f4[];
  float* hs = reinterpret_cast<float*>(smem_f4);
  int* flag = reinterpret_cast<int*>(hs + Gm::kSegPhys);         // [kChunk]
  uint32_t* bmask = reinterpret_cast<uint32_t*>(flag + kChunk);  // [kBlocks]
  int* bbase = reinterpret_cast<int*>(bmask + kBlocks);          // [kBlocks]
  float* red = reinterpret_cast<float*>(bbase + kBlocks);        // [kWarps][kChunk]
  const int64_t unit = blockIdx.x;
  const int64_t tile = unit / split_cnt;
  const int split = split_lo + static_cast<int>(unit % split_cnt);
  const int64_t I0 = tile * Gm::kTileR;
  const int64_t c0 = split * chunks / splits, c1 = (split + 1) * chunks / splits;
  const int own = threadIdx.x, warp = own >> 5, lane = own & 31;
  const float* lane_base = hs + (kThreads - 1 - own) * Gm::kPitch;
  float* redw = red + warp * kChunk;

  float xr[R];
  const int64_t jb = I0 + own * R;
#pragma unroll
  for (int q = 0; q < R; ++q) xr[q] = (jb + q < n) ? __ldg(x + jb + q) : 0.f;

  for (int64_t ch = c0; ch < c1; ++ch) {
    const int64_t Jc = ch * kChunk;
    const int r0 = rowstart[ch], nr = rowstart[ch + 1] - r0;
    if (nr == 0) continue;
    stage_segment<R>(hs, h, n, Jc - I0 - Gm::kTileR);
    for (int s = threadIdx.x; s < kChunk; s += kThreads) flag[s] = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < nr; k += kThreads) flag[omega[r0 + k] - static_cast<int>(Jc)] = 1;
    __syncthreads();
    if (warp == 0) {  // masks + exclusive prefix of row counts per block
      int run = 0;
      for (int b = 0; b < kBlocks; ++b) {
        const uint32_t mk = __ballot_sync(0xffffffffu, flag[b * kP + lane] != 0);
        if (lane == 0) {
          bmask[b] = mk;
          bbase[b] = run;
        }
        run += __popc(mk);
      }
    }
    __syncthreads();
    for (int b = 0; b < kBlocks; ++b) {
      const uint32_t mask = bmask[b];
      if (mask == 0u) continue;
      float w[R + kP];
      window_at<R>(w, lane_base, b * kP);
      float out[kP];
      res_group<R, 0>(w, xr, mask, out);
      res_group<R, 1>(w, xr, mask, out);
      res_group<R, 2>(w, xr, mask, out);
      res_group<R, 3>(w, xr, mask, out);
      res_group<R, 4>(w, xr, mask, out);
      res_group<R, 5>(w, xr, mask, out);
      res_group<R, 6>(w, xr, mask, out);
      res_group<R, 7>(w, xr, mask, out);
      transpose_reduce32(out, lane);
      if (mask & (1u << lane)) redw[bbase[b] + __popc(mask & ((1u << lane) - 1u))] = out[0];
    }
    __syncthreads();
    float* outp = partial + tile * m + r0;
    for (int kk = threadIdx.x; kk < nr; kk += kThreads) {
      float s = red[kk];
#pragma unroll
      for (int wi = 1; wi < kWarps; ++wi) s += red[wi * kChunk + kk];
      outp[kk] = s;
    }
    __syncthreads();
  }
}

// ===========================================================================
// Elementwise epilogues (fixed grid kEpiBlocks -> deterministic metrics).
// ===========================================================================
__device__ __forceinline__ float soft(float v, float g) {  // solvers.hpp:39-44
  if (v > g) return v - g;
  if (v < -g) return v + g;
  return 0.f;
}

__device__ __forceinline__ void block_metrics(double a, double b, double c, double* out) {
  __shared__ double sh[3][kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[0][w] = a;
    sh[1][w] = b;
    sh[2][w] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0, s1 = 0, s2 = 0;
    for (int i = 0; i < kThreads / 32; ++i) {
      s0 += sh[0][i];
      s1 += sh[1][i];
      s2 += sh[2][i];
    }
    out[blockIdx.x * 4 + 0] = s0;
    out[blockIdx.x * 4 + 1] = s1;
    out[blockIdx.x * 4 + 2] = s2;
    out[blockIdx.x * 4 + 3] = 0.0;
  }
}

__device__ __forceinline__ float sum_partials(const float* __restrict__ p, int splits, int64_t stride, int64_t i) {
  float s = p[i];
  for (int k = 1; k < splits; ++k) s += p[k * stride + i];
  return s;
}

__global__ void __launch_bounds__(kThreads) k_residual_reduce(EpiArgs a, int64_t tiles) {
  // r[t] = y[t] - sum_tile partial[tile][t]   (cpista residual, parallel.hpp:252)
  for (int64_t t = a.lo + blockIdx.x * (int64_t)kThreads + threadIdx.x; t < a.hi;
       t += (int64_t)gridDim.x * kThreads) {
    const float s = sum_partials(a.partial, static_cast<int>(tiles), a.n, t);
    a.r[t] = a.y[t] - s;
  }
}

__global__ void __launch_bounds__(kThreads) k_ista_update(EpiArgs a) {
  // delta[i] = sum_s partial; x[i] = eta_g(x[i] + tau * delta[i])   (parallel.hpp:269-271)
  double m0 = 0, m1 = 0, m2 = 0;
  for (int64_t i = a.lo + blockIdx.x * (int64_t)kThreads + threadIdx.x; i < a.hi;
       i += (int64_t)gridDim.x * kThreads) {
    const float d = sum_partials(a.partial, a.splits, a.n, i);
    const float xo = a.x[i];
    const float xn = soft(__fadd_rn(xo, __fmul_rn(a.tau, d)), a.thr);
    a.delta[i] = d;
    a.x[i] = xn;
    if (a.want_metrics) {
      const double dd = (double)xn - (double)xo;
      m0 += dd * dd;
      if (a.truth) {
        const double dt = (double)xn - (double)a.truth[i];
        m1 += dt * dt;
      }
      if (!isfinite(xn)) m2 += 1.0;
    }
  }
  if (a.want_metrics) block_metrics(m0, m1, m2, a.blk);
}

__global__ void __launch_bounds__(kThreads) k_admm_beta(EpiArgs a) {
  // beta = rho * C^T v + sigma * (z - nu)   (parallel.hpp:186-187)
  for (int64_t i = a.lo + blockIdx.x * (int64_t)kThreads + threadIdx.x; i < a.hi;
       i += (int64_t)gridDim.x * kThreads) {
    const float s = sum_partials(a.partial, a.splits, a.n, i);
    a.beta[i] = __fadd_rn(__fmul_rn(a.rho, s), __fmul_rn(a.sigma, __fsub_rn(a.z[i], a.nu[i])));
  }
}

__global__ void __launch_bounds__(kThreads) k_admm_x(EpiArgs a) {
  for (int64_t i = a.lo + blockIdx.x * (int64_t)kThreads + threadIdx.x; i < a.hi;
       i += (int64_t)gridDim.x * kThreads)
    a.x[i] = sum_partials(a.partial, a.splits, a.n, i);
}

__global__ void __launch_bounds__(kThreads) k_admm_duals(EpiArgs a) {
  // parallel.hpp:215-221
  double m0 = 0, m1 = 0, m2 = 0;
  for (int64_t i = a.lo + blockIdx.x * (int64_t)kThreads + threadIdx.x; i < a.hi;
       i += (int64_t)gridDim.x * kThreads) {
    const float cx = sum_partials(a.partial, a.splits, a.n, i);
    const float xi = a.x[i], nui = a.nu[i], zo = a.z[i];
    const float vn = __fmul_rn(a.d[i], __fadd_rn(__fmul_rn(a.rho, __fsub_rn(cx, a.mu[i])), a.pty[i]));
    const float zn = soft(__fadd_rn(xi, nui), a.thr);
    const float mun = __fadd_rn(a.mu[i], __fmul_rn(a.tau1, __fsub_rn(vn, cx)));
    a.z[i] = zn;
    a.mu[i] = mun;
    a.nu[i] = __fadd_rn(nui, __fmul_rn(a.tau2, __fsub_rn(xi, zn)));
    a.v[i] = __fadd_rn(vn, mun);
    if (a.want_metrics) {
      const double dd = (double)zn - (double)zo;
      m0 += dd * dd;
      if (a.truth) {
        const double dt = (double)zn - (double)a.truth[i];
        m1 += dt * dt;
      }
      if (!isfinite(zn)) m2 += 1.0;
    }
  }
  if (a.want_metrics) block_metrics(m0, m1, m2, a.blk);
}

__global__ void k_metrics_final(const double* __restrict__ blk, double* __restrict__ out) {
  // fixed-order tree over the kEpiBlocks per-block partials
  __shared__ double sh[3][256];
  double s0 = 0, s1 = 0, s2 = 0;
  for (int i = threadIdx.x; i < kEpiBlocks; i += blockDim.x) {
    s0 += blk[i * 4];
    s1 += blk[i * 4 + 1];
    s2 += blk[i * 4 + 2];
  }
  sh[0][threadIdx.x] = s0;
  sh[1][threadIdx.x] = s1;
  sh[2][threadIdx.x] = s2;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + o];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + o];
      sh[2][threadIdx.x] += sh[2][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sh[0][0];
    out[1] = sh[1][0];
    out[2] = sh[2][0];
    out[3] = 0.0;
  }
}

// FP32 FFMA roofline microkernel: independent outer-product chains, one
// shared multiplier per 32 FFMAs (the shape of the gradient/dense kernels).
__global__ void __launch_bounds__(256) k_ffma_peak(float* out, int iters) {
  float acc[32], w[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    acc[q] = 0.f;
    w[q] = 1.0f + 1e-3f * (threadIdx.x + q);
  }
  float r = 1.0f + 1e-4f * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = fmaf(w[q], r, acc[q]);
    r *= 0.9999f;
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 32; ++q) s += acc[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int R>
constexpr size_t smem_dense() { return Geo<R>::kSegPhys * 4 + kChunk * 4; }
template <int R>
constexpr size_t smem_rows() { return Geo<R>::kSegPhys * 4 + kChunk * 4 + kBlocks * 4; }
template <int R>
constexpr size_t smem_res() { return Geo<R>::kSegPhys * 4 + kChunk * 4 + 2 * kBlocks * 4 + kWarps * kChunk * 4; }

}  // namespace

ConvPlan make_plan(int64_t n, int R) {
  ConvPlan p;
  p.n = n;
  p.tile = static_cast<int64_t>(kThreads) * R;
  p.tiles = (n + p.tile - 1) / p.tile;
  p.chunks = (n + kChunk - 1) / kChunk;
  int64_t s = (kTargetUnits + p.tiles - 1) / p.tiles;
  if (s < 1) s = 1;
  if (s > p.chunks) s = p.chunks;
  p.splits = static_cast<int>(s);
  p.tile_lo = 0;
  p.tile_hi = p.tiles;
  p.split_lo = 0;
  p.split_hi = p.splits;
  return p;
}

void conv_kernels_init() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_conv_dense<kRDense>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_dense<kRDense>());
  cudaFuncSetAttribute(k_conv_rows<kRGrad>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_rows<kRGrad>());
  cudaFuncSetAttribute(k_conv_residual<kRRes>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_res<kRRes>());
  done = true;
}

void launch_conv_dense(const ConvPlan& p, const float* h, const float* u, float* partial, cudaStream_t st) {
  const int64_t units = (p.tile_hi - p.tile_lo) * p.splits;
  if (units <= 0) return;
  k_conv_dense<kRDense><<<static_cast<unsigned>(units), kThreads, smem_dense<kRDense>(), st>>>(
      h, u, p.n, p.chunks, p.splits, p.tile_lo, partial);
}

void launch_conv_rows(const ConvPlan& p, const float* h, const int* omega32, const float* rvals, const int* rowstart,
                      float* partial, cudaStream_t st) {
  const int64_t units = (p.tile_hi - p.tile_lo) * p.splits;
  if (units <= 0) return;
  k_conv_rows<kRGrad><<<static_cast<unsigned>(units), kThreads, smem_rows<kRGrad>(), st>>>(
      h, omega32, rvals, rowstart, p.n, p.chunks, p.splits, p.tile_lo, partial);
}

void launch_conv_residual(const ConvPlan& p, int64_t m, const float* h, const float* x, const int* omega32,
                          const int* rowstart, float* partial, cudaStream_t st) {
  const int cnt = p.split_hi - p.split_lo;
  const int64_t units = p.tiles * cnt;
  if (units <= 0) return;
  k_conv_residual<kRRes><<<static_cast<unsigned>(units), kThreads, smem_res<kRRes>(), st>>>(
      h, x, omega32, rowstart, p.n, m, p.chunks, p.splits, p.split_lo, cnt, partial);
}

static unsigned epi_grid(int64_t len) {
  int64_t g = (len + kThreads - 1) / kThreads;
  if (g > kEpiBlocks) g = kEpiBlocks;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

void launch_ista_residual_reduce(const EpiArgs& a, int64_t tiles, cudaStream_t st) {
  k_residual_reduce<<<epi_grid(a.hi - a.lo), kThreads, 0, st>>>(a, tiles);
}
// Metric-producing epilogues always use the full fixed grid so the
// per-block partial layout (and hence the metric) does not depend on n.
void launch_ista_update(const EpiArgs& a, cudaStream_t st) {
  k_ista_update<<<a.want_metrics ? kEpiBlocks : epi_grid(a.hi - a.lo), kThreads, 0, st>>>(a);
}
void launch_admm_beta(const EpiArgs& a, cudaStream_t st) { k_admm_beta<<<epi_grid(a.hi - a.lo), kThreads, 0, st>>>(a); }
void launch_admm_x(const EpiArgs& a, cudaStream_t st) { k_admm_x<<<epi_grid(a.hi - a.lo), kThreads, 0, st>>>(a); }
void launch_admm_duals(const EpiArgs& a, cudaStream_t st) {
  k_admm_duals<<<a.want_metrics ? kEpiBlocks : epi_grid(a.hi - a.lo), kThreads, 0, st>>>(a);
}
void launch_metrics_final(const double* blk, double* out4, cudaStream_t st) {
  k_metrics_final<<<1, 256, 0, st>>>(blk, out4);
}

double ffma_peak_tflops(int device) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 4, threads = 256, iters = 20000;
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float) * blocks * threads) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_ffma_peak<<<blocks, threads>>>(out, iters / 10);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_ffma_peak<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * 32.0 * blocks * threads * static_cast<double>(iters);
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace clb
