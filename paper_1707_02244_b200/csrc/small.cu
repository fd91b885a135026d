// Persistent single-cluster ISTA for small problems (BASELINE config 1, n = 4096):
// the whole solve state lives in shared memory of one thread-block cluster and
// all requested iterations run in ONE launch.  At n = 4096
// an iteration is only 8.4 MFMA; the multi-kernel path spends ~50 us per
// iteration in launch and split-K latency.
//
// Cluster of CL = 8 CTAs x 256 threads (RG = RX: both thread windows share the padding period); CTA k owns positions / outputs
// [k n/CL, (k+1) n/CL).  Per iteration (cpista_phases, parallel.hpp:236-279):
//   residual: CTA k computes the complete dot of each of its rows (x is
//     replicated in every CTA; thread owns RX = n/256 consecutive x in
//     registers; 32-position blocks share one register window of c~; lane
//     partials are reduced in fixed order), r = y - A x, and stores r into
//     every CTA's dense P^T r copy through distributed shared memory.
//   cluster barrier.
//   gradient: CTA k computes delta for its outputs over all rows (warp w takes
//     blocks w, w+8, ...; lane owns RG = n/(32 CL) outputs), sums the 8 warps
//     in fixed order, x = eta(x + tau delta), and stores x into every CTA.
//   cluster barrier.
// No reduction crosses CTAs, so the result is deterministic; parity is the
// same tolerance contract as the multi-kernel path (tests/test_gpu_parity.py).
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdlib>

#include "small.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace clb {
namespace {

constexpr int kSt = 256;  // threads per CTA
constexpr int kSw = kSt / 32;

__device__ __forceinline__ float soft_s(float v, float g) {  // solvers.hpp:39-44
  if (v > g) return v - g;
  if (v < -g) return v + g;
  return 0.f;
}

// c2: c~[(e) mod n] for e in [0, 2n), padded by 4 floats every P elements (P = n/256:
// thread windows start P apart; the padding spreads LDS.128 phases over the banks).
template <int P>
__device__ __forceinline__ int padc(int e) { return e + 4 * (e / P); }

template <int N, int CL>
struct SG {
  static constexpr int NPC = N / CL;   // positions (residual) / outputs (gradient) per CTA
  static constexpr int RX = N / kSt;   // residual: x values per thread (= the padding period)
  static constexpr int RG = NPC / 32;  // gradient: outputs per lane
  static constexpr int NB = N / 32;    // 32-position blocks
  static constexpr int C2 = 2 * N + 4 * (2 * N / RX) + 64;  // padded c2 (+ slack for the window tail)
  // shared memory (floats): c2 | xs[N] | rd[N] | red[kSw][NPC] | lp[kSw][32][33] | ys[NPC] | rloc[NPC]
  static constexpr int OFF_XS = C2, OFF_RD = OFF_XS + N, OFF_RED = OFF_RD + N, OFF_LP = OFF_RED + kSw * NPC,
                       OFF_YS = OFF_LP + kSw * 32 * 33, OFF_RL = OFF_YS + NPC, OFF_MASK = OFF_RL + NPC,
                       OFF_BBASE = OFF_MASK + NB, TOTAL = OFF_BBASE + NB + 1;
};

template <int N, int CL>
size_t small_smem() { return static_cast<size_t>(SG<N, CL>::TOTAL) * 4; }

template <int L, int K>
__device__ __forceinline__ void ldw(float (&w)[L], const float* __restrict__ p) {
  const float4 t = *reinterpret_cast<const float4*>(p);
  w[K] = t.x;
  w[K + 1] = t.y;
  w[K + 2] = t.z;
  w[K + 3] = t.w;
}
// w[k] = c2[base + k], k in [0, L); base a multiple of P (window origin), padded layout.
template <int L, int P>
__device__ __forceinline__ void load_win(float (&w)[L], const float* __restrict__ c2, int base) {
  const float* b = c2 + padc<P>(base);
#pragma unroll
  for (int k = 0; k < L; k += 4) {
    const float4 t = *reinterpret_cast<const float4*>(b + k + 4 * (k / P));
    w[k] = t.x;
    w[k + 1] = t.y;
    w[k + 2] = t.z;
    w[k + 3] = t.w;
  }
}

// Sums the K (<= 32) rows of lane partials lp[lane * 33 + row] over the 32 lanes in fixed order.
__device__ __forceinline__ void reduce_lanes(const float* __restrict__ lp, float* __restrict__ out, int K, int lane) {
  for (int g = 0; g < K; g += 8) {
    const int k = g + (lane >> 2), part = lane & 3;
    float a0 = 0.f, a1 = 0.f;
    if (k < K) {
      const float* col = lp + (part * 8) * 33 + k;
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        a0 += col[i * 33];
        a1 += col[(i + 1) * 33];
      }
    }
    float s = a0 + a1;
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (k < K && part == 0) out[k] = s;
  }
}

template <int RX, int S>
__device__ __forceinline__ void res_row(const float (&w)[RX + 32], const float (&xr)[RX], float*& lpp) {
  float p0 = w[32 - S] * xr[0], p1 = w[33 - S] * xr[1];
#pragma unroll
  for (int q = 2; q < RX; q += 2) {
    p0 = fmaf(w[32 - S + q], xr[q], p0);
    p1 = fmaf(w[33 - S + q], xr[q + 1], p1);
  }
  *lpp++ = p0 + p1;
}
template <int RX, int S0>
__device__ __forceinline__ void res_quad(const float (&w)[RX + 32], const float (&xr)[RX], uint32_t mask, float*& lpp) {
  if ((mask >> S0) & 0xFu) {
    if ((mask >> S0) & 1u) res_row<RX, S0>(w, xr, lpp);
    if ((mask >> (S0 + 1)) & 1u) res_row<RX, S0 + 1>(w, xr, lpp);
    if ((mask >> (S0 + 2)) & 1u) res_row<RX, S0 + 2>(w, xr, lpp);
    if ((mask >> (S0 + 3)) & 1u) res_row<RX, S0 + 3>(w, xr, lpp);
  }
}

template <int RG, int S>
__device__ __forceinline__ void grad_row(float (&acc)[RG], const float (&w)[RG + 32], float r) {
#pragma unroll
  for (int q = 0; q < RG; ++q) acc[q] = fmaf(w[q - S + 32], r, acc[q]);
}
template <int RG, int S0>
__device__ __forceinline__ void grad_quad(float (&acc)[RG], const float (&w)[RG + 32], uint32_t mask,
                                          const float* __restrict__ rb) {
  if ((mask >> S0) & 0xFu) {
    const float4 r4 = *reinterpret_cast<const float4*>(rb + S0);
    if ((mask >> S0) & 1u) grad_row<RG, S0>(acc, w, r4.x);
    if ((mask >> (S0 + 1)) & 1u) grad_row<RG, S0 + 1>(acc, w, r4.y);
    if ((mask >> (S0 + 2)) & 1u) grad_row<RG, S0 + 2>(acc, w, r4.z);
    if ((mask >> (S0 + 3)) & 1u) grad_row<RG, S0 + 3>(acc, w, r4.w);
  }
}

template <int N, int CL>
__global__ void __launch_bounds__(kSt, 1)
k_small_ista(const float* __restrict__ hc, const int* __restrict__ omega, const float* __restrict__ y,
             float* __restrict__ x, float* __restrict__ r, float* __restrict__ delta, int m, float tau, float thr,
             int iters) {
  using G = SG<N, CL>;
  constexpr int RX = G::RX, RG = G::RG, NPC = G::NPC, NB = G::NB;
  extern __shared__ float4 smem_f4[];
  float* sm = reinterpret_cast<float*>(smem_f4);
  float* c2 = sm;
  float* xs = sm + G::OFF_XS;
  float* rd = sm + G::OFF_RD;
  float* red = sm + G::OFF_RED;
  float* lp = sm + G::OFF_LP;
  float* ys = sm + G::OFF_YS;
  float* rloc = sm + G::OFF_RL;
  uint32_t* bmask = reinterpret_cast<uint32_t*>(sm + G::OFF_MASK);
  int* bbase = reinterpret_cast<int*>(sm + G::OFF_BBASE);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- prologue: operator row (padded, wrapped), x, row masks, row ranges ----
  for (int e = tid; e < 2 * N; e += kSt) c2[padc<RX>(e)] = __ldg(hc + (e < N ? e : e - N));
  for (int e = tid; e < N; e += kSt) {
    xs[e] = x[e];
    rd[e] = 0.f;
  }
  for (int e = tid; e < NB; e += kSt) bmask[e] = 0u;
  __syncthreads();
  for (int t = tid; t < m; t += kSt) atomicOr(&bmask[omega[t] >> 5], 1u << (omega[t] & 31));
  __syncthreads();
  if (warp == 0) {  // exclusive prefix of row counts per block
    int run = 0;
    for (int b0 = 0; b0 < NB; b0 += 32) {
      const int b = b0 + lane;
      const int c = b < NB ? __popc(bmask[b]) : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (b < NB) bbase[b] = run + incl - c;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) bbase[NB] = run;
  }
  __syncthreads();
  const int blo = rank * (NPC / 32), bhi = blo + NPC / 32;  // this CTA's residual blocks
  const int t_lo = bbase[blo], t_hi = bbase[bhi];
  for (int t = t_lo + tid; t < t_hi; t += kSt) ys[t - t_lo] = y[t];
  __syncthreads();
  cluster.sync();  // every CTA initialised before any remote store

  float* lp_lane = lp + warp * 32 * 33 + lane * 33;
  float* lpw = lp + warp * 32 * 33;
  float* redw = red + warp * NPC;
  const int O0 = rank * NPC;

  for (int it = 0; it < iters; ++it) {
    // ---- residual: rows of this CTA's blocks -------------------------------------
    float xr[RX];
    {
      const float* xp = xs + tid * RX;
#pragma unroll
      for (int q = 0; q < RX; q += 4) {
        const float4 t = *reinterpret_cast<const float4*>(xp + q);
        xr[q] = t.x;
        xr[q + 1] = t.y;
        xr[q + 2] = t.z;
        xr[q + 3] = t.w;
      }
    }
    for (int b = blo; b < bhi; ++b) {
      const uint32_t mask = __reduce_or_sync(0xffffffffu, bmask[b]);  // uniform: no divergence bookkeeping
      if (!mask) continue;
      float w[RX + 32];
      load_win<RX + 32, RX>(w, c2, tid * RX - 32 * b + N - 32);
      float* lpp = lp_lane;
      res_quad<RX, 0>(w, xr, mask, lpp);
      res_quad<RX, 4>(w, xr, mask, lpp);
      res_quad<RX, 8>(w, xr, mask, lpp);
      res_quad<RX, 12>(w, xr, mask, lpp);
      res_quad<RX, 16>(w, xr, mask, lpp);
      res_quad<RX, 20>(w, xr, mask, lpp);
      res_quad<RX, 24>(w, xr, mask, lpp);
      res_quad<RX, 28>(w, xr, mask, lpp);
      __syncwarp();
      reduce_lanes(lpw, redw + (bbase[b] - t_lo), __popc(mask), lane);
      __syncwarp();
    }
    __syncthreads();
    for (int tl = tid; tl < t_hi - t_lo; tl += kSt) {
      float s = red[tl];
#pragma unroll
      for (int wi = 1; wi < kSw; ++wi) s += red[wi * NPC + tl];
      const float rv = ys[tl] - s;  // cpista residual, parallel.hpp:252
      rloc[tl] = rv;
      const int pos = __ldg(omega + t_lo + tl);
#pragma unroll
      for (int k = 0; k < CL; ++k) cluster.map_shared_rank(rd, k)[pos] = rv;
    }
    cluster.sync();

    // ---- gradient: this CTA's outputs over all rows ----------------------------
    float acc[RG];
#pragma unroll
    for (int q = 0; q < RG; ++q) acc[q] = 0.f;
    for (int b = warp; b < NB; b += kSw) {
      const uint32_t mask = __reduce_or_sync(0xffffffffu, bmask[b]);  // uniform: no divergence bookkeeping
      if (!mask) continue;
      float w[RG + 32];
      load_win<RG + 32, RX>(w, c2, O0 + lane * RG - 32 * b + N - 32);
      const float* rb = rd + 32 * b;
      grad_quad<RG, 0>(acc, w, mask, rb);
      grad_quad<RG, 4>(acc, w, mask, rb);
      grad_quad<RG, 8>(acc, w, mask, rb);
      grad_quad<RG, 12>(acc, w, mask, rb);
      grad_quad<RG, 16>(acc, w, mask, rb);
      grad_quad<RG, 20>(acc, w, mask, rb);
      grad_quad<RG, 24>(acc, w, mask, rb);
      grad_quad<RG, 28>(acc, w, mask, rb);
    }
#pragma unroll
    for (int q = 0; q < RG; ++q) redw[q * 32 + lane] = acc[q];  // output lane*RG + q, conflict-free layout
    __syncthreads();
    for (int o = tid; o < NPC; o += kSt) {
      const int slot = (o % RG) * 32 + o / RG;
      float d = red[slot];
#pragma unroll
      for (int wi = 1; wi < kSw; ++wi) d += red[wi * NPC + slot];
      const int i = O0 + o;
      const float xn = soft_s(__fadd_rn(xs[i], __fmul_rn(tau, d)), thr);  // parallel.hpp:269-271
      if (it == iters - 1) delta[i] = d;
#pragma unroll
      for (int k = 0; k < CL; ++k) cluster.map_shared_rank(xs, k)[i] = xn;
    }
    cluster.sync();
  }
  // ---- epilogue: state back to global ---------------------------------------------
  for (int o = tid; o < NPC; o += kSt) x[O0 + o] = xs[O0 + o];
  for (int tl = tid; tl < t_hi - t_lo; tl += kSt) r[t_lo + tl] = rloc[tl];
}

template <int N, int CL>
cudaError_t launch_t(const float* hc, const int* omega, const float* y, float* x, float* r, float* delta, int m,
                     float tau, float thr, int iters, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  const size_t smem = small_smem<N, CL>();
  if (first_use_on_device(attr)) {
    cudaFuncSetAttribute(k_small_ista<N, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (CL > 8) cudaFuncSetAttribute(k_small_ista<N, CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(kSt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_small_ista<N, CL>, hc, omega, y, x, r, delta, m, tau, thr, iters);
}

}  // namespace

bool small_ista_supported(int64_t n, int64_t m) {
  const char* off = std::getenv("CLB_NO_SMALL");
  if (off && off[0] == '1') return false;
  return (n == 2048 || n == 4096 || n == 8192) && m >= 1 && m <= n;
}

cudaError_t launch_small_ista(int64_t n, int64_t m, const float* hc, const int* omega, const float* y, float* x,
                              float* r, float* delta, float tau, float thr, int iters, cudaStream_t st) {
  const int mm = static_cast<int>(m);
  switch (n) {
    case 2048: return launch_t<2048, 8>(hc, omega, y, x, r, delta, mm, tau, thr, iters, st);
    case 4096: return launch_t<4096, 8>(hc, omega, y, x, r, delta, mm, tau, thr, iters, st);
    case 8192: return launch_t<8192, 8>(hc, omega, y, x, r, delta, mm, tau, thr, iters, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace clb
