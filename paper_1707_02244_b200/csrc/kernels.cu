// Direct shift-indexed circulant kernels for sm_100a (see kernels.cuh for the
// index algebra and the work decomposition).
//
// Register tiling.  A thread owns R consecutive indices.  For a block of PB
// consecutive positions it loads an (R + PB)-float window of the first row
// from shared memory ((R + PB) / 4 x LDS.128) and then
//   * dense / gradient kernels (outer-product form, one broadcast scalar
//     shared by R consecutive FFMAs):  acc[q] += w[q - s + PB] * u[s]
//   * residual kernel (dot form, rows are the outputs):
//       out[s] = sum_q w[s - q + R] * x[q]      x[q] register-resident
// Every register index is a compile-time constant.  The data-dependent row
// positions (omega is a random subset, density m/n) are handled by PB
// statically indexed bodies per block, each behind a warp-uniform bit test of
// the block's row mask (straight-line code; a jump table per row was measured
// 1.3-1.5x slower: indirect branches are expensive on sm_100a).
//
// Shared memory.  Lanes own windows R floats apart; a plain layout would put
// all 8 lanes of an LDS.128 phase in one bank group.  The staged row is padded
// by 4 floats every R elements (lane pitch R + 4 words), which spreads the 8
// lanes of every phase over 8 distinct bank groups.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "kernels.cuh"
#include "tc_dense.cuh"

namespace cg = cooperative_groups;

namespace clb {

namespace {

// Block range [blo, bhi) (32-position blocks) of split `split`: whole chunks
// when there are at least as many chunks as splits (large n), otherwise
// fractions of a chunk (small n needs more CTAs than it has chunks).
__host__ __device__ __forceinline__ void split_blocks(int64_t chunks, int splits, int split, int64_t* blo,
                                                      int64_t* bhi) {
  constexpr int64_t kB = kChunk / 32;
  if (splits <= chunks) {
    *blo = split * chunks / splits * kB;
    *bhi = (split + 1) * chunks / splits * kB;
  } else {
    *blo = split * (chunks * kB) / splits;
    *bhi = (split + 1) * (chunks * kB) / splits;
  }
}

#ifndef CLB_RES_CHAINS
#define CLB_RES_CHAINS 4
#endif
constexpr int kResChains = CLB_RES_CHAINS;  // dot-form chains in the residual

__device__ int g_force_dense = 0;  // timing experiment: treat every position as a row

template <int R>
struct Geo {
  static_assert(R == 16 || R == 32 || R == 64, "R must be 16, 32 or 64");
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

// Lane window w[k] = seg[x + k], k in [0, R + PB), x a multiple of PB whose
// phase x mod R is PH (compile time), p = lane window origin for that phase.
template <int R, int PB, int PH>
__device__ __forceinline__ void load_window_ph(float (&w)[R + PB], const float* __restrict__ p) {
  using G = Geo<R>;
#pragma unroll
  for (int k = 0; k < R + PB; k += 4) {
    const float4 t = *reinterpret_cast<const float4*>(p + (G::pad(PH + k) - PH));
    w[k] = t.x;
    w[k + 1] = t.y;
    w[k + 2] = t.z;
    w[k + 3] = t.w;
  }
}
template <int R, int PB>
__device__ __forceinline__ void window_at(float (&w)[R + PB], const float* __restrict__ lane_base, int x) {
  const float* p = lane_base + (x / R) * (R + 4) + (x % R);
  const int ph = x % R;
  if (PB >= R) { load_window_ph<R, PB, 0>(w, p); return; }
  if (R / PB == 2) {
    if (ph) load_window_ph<R, PB, (R / 2) % R>(w, p);
    else load_window_ph<R, PB, 0>(w, p);
  } else {  // R / PB == 4
    switch (ph / PB) {
      case 1: load_window_ph<R, PB, (PB) % R>(w, p); break;
      case 2: load_window_ph<R, PB, (2 * PB) % R>(w, p); break;
      case 3: load_window_ph<R, PB, (3 * PB) % R>(w, p); break;
      default: load_window_ph<R, PB, 0>(w, p); break;
    }
  }
}

// ===========================================================================
// Dense circular convolution (cADMM products).  unit = (tile, split).
// ===========================================================================
template <int R>
__global__ void __launch_bounds__(kThreads, 2)
k_conv_dense(const float* __restrict__ h, const float* __restrict__ u, int64_t n, int64_t chunks, int splits,
             int64_t tile_lo, float* __restrict__ partial) {
  constexpr int PB = 32;
  using G = Geo<R>;
  extern __shared__ float4 smem_f4[];
  float* hs = reinterpret_cast<float*>(smem_f4);
  float* us = hs + G::kSegPhys;
  const int64_t unit = blockIdx.x;
  const int64_t tile = tile_lo + unit / splits;
  const int split = static_cast<int>(unit % splits);
  const int64_t I0 = tile * G::kTileR;
  int64_t blo, bhi;
  split_blocks(chunks, splits, split, &blo, &bhi);
  const int own = threadIdx.x;
  const float* lane_base = hs + own * G::kPitch;

  float acc[R];
#pragma unroll
  for (int q = 0; q < R; ++q) acc[q] = 0.f;

  for (int64_t ch = blo / (kChunk / 32); ch * (kChunk / 32) < bhi; ++ch) {
    const int64_t Jc = ch * kChunk;
    stage_segment<R>(hs, h, n, I0 - Jc - kChunk);
    for (int s = threadIdx.x; s < kChunk; s += kThreads) {
      const int64_t j = Jc + s;
      us[s] = j < n ? __ldg(u + j) : 0.f;
    }
    __syncthreads();
    const int64_t bsub = 32 / (PB), cb = ch * (kChunk / 32);
    const int b0 = static_cast<int>((blo > cb ? blo - cb : 0) * bsub);
    const int b1 = static_cast<int>((bhi - cb < kChunk / 32 ? bhi - cb : kChunk / 32) * bsub);
    for (int b = 0; b < kChunk / PB; ++b) {
      if (b < b0 || b >= b1) continue;  // split covers part of the chunk (small n)
      float w[R + PB];
      window_at<R, PB>(w, lane_base, kChunk - (b + 1) * PB);
#pragma unroll
      for (int s4 = 0; s4 < PB; s4 += 4) {
        const float4 uu = *reinterpret_cast<const float4*>(us + b * PB + s4);
        const float uv[4] = {uu.x, uu.y, uu.z, uu.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
#pragma unroll
          for (int q = 0; q < R; ++q) acc[q] = fmaf(w[q - (s4 + e) + PB], uv[e], acc[q]);
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
// Gradient A^T r (padded R = 32 layout; the small-n kernel): convolution with
// the sparse input P^T r, rows only.  The staged chunk holds r scattered to its
// positions (zeros elsewhere) and a row mask per PB-position block (a zero
// residual contributes exactly nothing, so value != 0 is the mask).
// ===========================================================================
// 32-lane ballot of a flag array into PB-bit masks, one per block.
template <int PB>
__device__ __forceinline__ uint32_t block_mask(uint32_t ballot32, int sub) {
  return PB == 32 ? ballot32 : (ballot32 >> (sub * PB)) & ((1u << PB) - 1u);
}

// Out-of-line layout of the 32 position bodies (R = 32, PB = 32): the common
// case (position not a row) falls through its test; a row costs a jump to its
// body and a jump back.
#define CLB_T(S) if (mask & (1u << S)) goto body##S; ret##S:
#define CLB_B(S)                                                        \
  body##S : {                                                           \
    const float r = rb[S];                                              \
    _Pragma("unroll") for (int q = 0; q < R; ++q) acc[q] = fmaf(w[q - S + PB], r, acc[q]); \
  }                                                                     \
  goto ret##S;
#define S_COMP(S) S_COMP_##S

#define S_COMP_0 x
#define S_COMP_1 y
#define S_COMP_2 z
#define S_COMP_3 w
#define S_COMP_4 x
#define S_COMP_5 y
#define S_COMP_6 z
#define S_COMP_7 w
#define S_COMP_8 x
#define S_COMP_9 y
#define S_COMP_10 z
#define S_COMP_11 w
#define S_COMP_12 x
#define S_COMP_13 y
#define S_COMP_14 z
#define S_COMP_15 w
#define S_COMP_16 x
#define S_COMP_17 y
#define S_COMP_18 z
#define S_COMP_19 w
#define S_COMP_20 x
#define S_COMP_21 y
#define S_COMP_22 z
#define S_COMP_23 w
#define S_COMP_24 x
#define S_COMP_25 y
#define S_COMP_26 z
#define S_COMP_27 w
#define S_COMP_28 x
#define S_COMP_29 y
#define S_COMP_30 z
#define S_COMP_31 w
#define CLB_ALL16(M) M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15)
#define CLB_ALL32(M) CLB_ALL16(M) \
  M(16) M(17) M(18) M(19) M(20) M(21) M(22) M(23) M(24) M(25) M(26) M(27) M(28) M(29) M(30) M(31)

template <int R>
__device__ __forceinline__ void ool_block32(float (&acc)[R], const float (&w)[R + 32], uint32_t mask,
                                            const float* __restrict__ rb) {
  constexpr int PB = 32;
  CLB_ALL32(CLB_T)
  return;
  CLB_ALL32(CLB_B)
}
template <int R>
__device__ __forceinline__ void ool_block16(float (&acc)[R], const float (&w)[R + 16], uint32_t mask,
                                            const float* __restrict__ rb) {
  constexpr int PB = 16;
  CLB_ALL16(CLB_T)
  return;
  CLB_ALL16(CLB_B)
}

template <int MINB, int R = 32, int PB = 32>
__global__ void __launch_bounds__(kThreads, MINB)
k_conv_rows_ool(const float* __restrict__ h, const int* __restrict__ omega, const float* __restrict__ rv,
                const int* __restrict__ rowstart, int64_t n, int64_t chunks, int splits, int64_t tile_lo,
                float* __restrict__ partial) {
  static_assert(PB == 32 || PB == 16, "PB must be 16 or 32");
  using Gm = Geo<R>;
  extern __shared__ float4 smem_f4[];
  float* hs = reinterpret_cast<float*>(smem_f4);
  float* rd = hs + Gm::kSegPhys;
  uint32_t* bmask = reinterpret_cast<uint32_t*>(rd + kChunk);
  const int64_t unit = blockIdx.x;
  const int64_t tile = tile_lo + unit / splits;
  const int split = static_cast<int>(unit % splits);
  const int64_t I0 = tile * Gm::kTileR;
  int64_t blo, bhi;
  split_blocks(chunks, splits, split, &blo, &bhi);
  const int own = threadIdx.x, warp = own >> 5, lane = own & 31;
  const float* lane_base = hs + own * Gm::kPitch;

  float acc[R];
#pragma unroll
  for (int q = 0; q < R; ++q) acc[q] = 0.f;

  for (int64_t ch = blo / (kChunk / 32); ch * (kChunk / 32) < bhi; ++ch) {
    const int64_t Jc = ch * kChunk;
    const int r0 = rowstart[ch], nr = rowstart[ch + 1] - r0;
    if (nr == 0) continue;
    stage_segment<R>(hs, h, n, I0 - Jc - kChunk);
    for (int s = threadIdx.x; s < kChunk; s += kThreads) rd[s] = 0.f;
    __syncthreads();
    for (int k = threadIdx.x; k < nr; k += kThreads) rd[omega[r0 + k] - static_cast<int>(Jc)] = __ldg(rv + r0 + k);
    __syncthreads();
    for (int b32 = warp; b32 < kChunk / 32; b32 += kWarps) {
      const uint32_t mk = g_force_dense == 1 ? 0xffffffffu : g_force_dense == 2 ? 0x11111111u : g_force_dense == 3 ? 0x000000ffu : __ballot_sync(0xffffffffu, rd[b32 * 32 + lane] != 0.f);
      if (lane == 0)
        for (int sub = 0; sub < 32 / PB; ++sub) bmask[b32 * (32 / PB) + sub] = block_mask<PB>(mk, sub);
    }
    __syncthreads();
    const int64_t bsub = 32 / (PB), cb = ch * (kChunk / 32);
    const int b0 = static_cast<int>((blo > cb ? blo - cb : 0) * bsub);
    const int b1 = static_cast<int>((bhi - cb < kChunk / 32 ? bhi - cb : kChunk / 32) * bsub);
    for (int b = 0; b < kChunk / PB; ++b) {
      if (b < b0 || b >= b1) continue;  // split covers part of the chunk (small n)
      const uint32_t mask = bmask[b];
      if (mask == 0u) continue;
      float w[R + PB];
      window_at<R, PB>(w, lane_base, kChunk - (b + 1) * PB);
      const float* rb = rd + b * PB;
      if constexpr (PB == 32) ool_block32<R>(acc, w, mask, rb);
      else ool_block16<R>(acc, w, mask, rb);
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
// leaves lane L with the warp sum of position L mod PB, which it stores to
// the row's slot.  Warps are combined in fixed order at the end of a chunk.
// ===========================================================================
template <int R, int PB, int S>
__device__ __forceinline__ void res_pos(const float (&w)[R + PB], const float (&xr)[R], uint32_t mask,
                                        float*& lpp) {
  if (mask & (1u << S)) {
    // CH independent chains: the dot form has no shared operand, so its FFMA rate is
    // latency-bound with few chains (microbench: 4 chains 45 TF, 8 chains 69 TF).
    float p[kResChains];
#pragma unroll
    for (int c = 0; c < kResChains; ++c) p[c] = w[S - c + R] * xr[c];
#pragma unroll
    for (int q = kResChains; q < R; ++q) p[q % kResChains] = fmaf(w[S - q + R], xr[q], p[q % kResChains]);
    // fixed-order pairwise fold of the chains (any chain count)
#pragma unroll
    for (int width = kResChains; width > 1; width = (width + 1) / 2)
#pragma unroll
      for (int c = 0; c < width / 2; ++c) p[c] += p[c + (width + 1) / 2];
    *lpp++ = p[0];  // lane-major slot list: lp[lane * 33 + slot]
  }
}

template <int R, int PB, int G>
__device__ __forceinline__ void res_group(const float (&w)[R + PB], const float (&xr)[R], uint32_t mask,
                                          float*& lpp) {
  if (G * 4 < PB && (mask & (0xFu << (4 * G)))) {
    res_pos<R, PB, 4 * G>(w, xr, mask, lpp);
    res_pos<R, PB, 4 * G + 1>(w, xr, mask, lpp);
    res_pos<R, PB, 4 * G + 2>(w, xr, mask, lpp);
    res_pos<R, PB, 4 * G + 3>(w, xr, mask, lpp);
  }
}

// Sums the K (<= 32) rows of lane partials lp[lane * 33 + row] over the 32
// lanes: 4 lanes per row, 8 rows per round, fixed order.  Row sums go to
// redw[base + row].  Conflict-free: bank = (8 part + i + row) mod 32.
__device__ __forceinline__ void reduce_lane_partials(const float* __restrict__ lp, float* __restrict__ redw,
                                                     int base, int K, int lane) {
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
    float sacc = a0 + a1;
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
    if (k < K && part == 0) redw[base + k] = sacc;
  }
}

template <int R, int PB, int MINB = (R <= 32 ? 3 : 2)>
__global__ void __launch_bounds__(kThreads, MINB)
k_conv_residual(const float* __restrict__ h, const float* __restrict__ x, const int* __restrict__ omega,
                const int* __restrict__ rowstart, int64_t n, int64_t m, int64_t chunks, int splits,
                int split_lo, int split_cnt, float* __restrict__ partial) {
  constexpr int NB = kChunk / PB;
  using Gm = Geo<R>;
  extern __shared__ float4 smem_f4[];
  float* hs = reinterpret_cast<float*>(smem_f4);
  uint32_t* bmask = reinterpret_cast<uint32_t*>(hs + Gm::kSegPhys);  // [NB]
  int* bbase = reinterpret_cast<int*>(bmask + NB);                    // [NB]
  float* red = reinterpret_cast<float*>(bbase + NB);                  // [kWarps][kChunk]
  int* flag = reinterpret_cast<int*>(red);  // [kChunk] row flags, dead before red is written
  float* lanep = red + kWarps * kChunk;     // [kWarps][32 lanes][33]
  const int64_t unit = blockIdx.x;
  const int64_t tile = unit / split_cnt;
  const int split = split_lo + static_cast<int>(unit % split_cnt);
  const int64_t I0 = tile * Gm::kTileR;
  int64_t blo, bhi;
  split_blocks(chunks, splits, split, &blo, &bhi);
  const int own = threadIdx.x, warp = own >> 5, lane = own & 31;
  const float* lane_base = hs + (kThreads - 1 - own) * Gm::kPitch;
  float* redw = red + warp * kChunk;
  float* lp = lanep + warp * 32 * 33;
  float* const lp_lane = lp + lane * 33;

  float xr[R];
  const int64_t jb = I0 + own * R;
#pragma unroll
  for (int q = 0; q < R; ++q) xr[q] = (jb + q < n) ? __ldg(x + jb + q) : 0.f;

  for (int64_t ch = blo / (kChunk / 32); ch * (kChunk / 32) < bhi; ++ch) {
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
      for (int b32 = 0; b32 < kChunk / 32; ++b32) {
        const uint32_t mk = g_force_dense ? 0xffffffffu : __ballot_sync(0xffffffffu, flag[b32 * 32 + lane] != 0);
        if (lane == 0) {
          for (int sub = 0; sub < 32 / PB; ++sub) {
            const uint32_t bm = block_mask<PB>(mk, sub);
            bmask[b32 * (32 / PB) + sub] = bm;
            bbase[b32 * (32 / PB) + sub] = run;
            run += __popc(bm);
          }
        }
        run = __shfl_sync(0xffffffffu, run, 0);
      }
    }
    __syncthreads();
    const int64_t bsub = 32 / (PB), cb = ch * (kChunk / 32);
    const int b0 = static_cast<int>((blo > cb ? blo - cb : 0) * bsub);
    const int b1 = static_cast<int>((bhi - cb < kChunk / 32 ? bhi - cb : kChunk / 32) * bsub);
    for (int b = 0; b < kChunk / PB; ++b) {
      if (b < b0 || b >= b1) continue;  // split covers part of the chunk (small n)
      const uint32_t mask = __reduce_or_sync(0xffffffffu, bmask[b]);  // REDUX: uniform register -> uniform branches
      if (mask == 0u) continue;
      float w[R + PB];
      window_at<R, PB>(w, lane_base, b * PB);
      float* lpp = lp_lane;
      res_group<R, PB, 0>(w, xr, mask, lpp);
      res_group<R, PB, 1>(w, xr, mask, lpp);
      res_group<R, PB, 2>(w, xr, mask, lpp);
      res_group<R, PB, 3>(w, xr, mask, lpp);
      res_group<R, PB, 4>(w, xr, mask, lpp);
      res_group<R, PB, 5>(w, xr, mask, lpp);
      res_group<R, PB, 6>(w, xr, mask, lpp);
      res_group<R, PB, 7>(w, xr, mask, lpp);
      __syncwarp();
      reduce_lane_partials(lp, redw, bbase[b], __popc(mask), lane);
      __syncwarp();
    }
    __syncthreads();
    float* outp = partial + tile * m + r0;
    const int k_lo = b0 < NB ? bbase[b0] : nr;
    const int k_hi = b1 < NB ? bbase[b1] : nr;
    for (int kk = k_lo + threadIdx.x; kk < k_hi; kk += kThreads) {
      float s = red[kk];
#pragma unroll
      for (int wi = 1; wi < kWarps; ++wi) s += red[wi * kChunk + kk];
      outp[kk] = s;
    }
    __syncthreads();
  }
}

// ===========================================================================
// Streamed-window sparse kernels.
//
// Layout: the staged row is NOT padded.  Lanes own R consecutive indices with
// R = 4 (mod 8), so the window origins of the 8 lanes of an LDS.128 phase are
// R/4 (odd) 16-byte units apart and land in 8 distinct bank groups; every
// window address is then lane_base + compile-time offset.
//
// Streaming: the 32 positions of a block are processed in 8 groups of 4.  A
// position needs R window floats; consecutive groups need windows 4 floats
// apart, so each group issues ONE LDS.128 for the next group (prefetch) and
// the compiler retires the 4 floats the group no longer needs: about R + 8
// window registers are live instead of R + 32, which pays for the larger R
// (fewer (warp, block) visits per row -> less per-block skeleton per FMA).
// The row values of the next group are prefetched the same way, so no body
// waits on a shared-memory load.
// ===========================================================================
template <int R, int NT = kThreads>
struct GeoU {
  static_assert(R % 8 == 4, "unpadded layout needs R = 4 mod 8 (conflict-free LDS.128 phases)");
  static constexpr int kTileR = NT * R;
  static constexpr int kSeg = kTileR + kChunk;
  static constexpr int kSegPhys = kSeg + 4;
};

// hs[e] = h[(base + e) mod n] for e in [0, kSeg).
template <int kSeg, int NT = kThreads>
__device__ __forceinline__ void stage_plain(float* __restrict__ hs, const float* __restrict__ h, int64_t n,
                                            int64_t base) {
  int64_t b = base % n;
  if (b < 0) b += n;
  if ((n & 3) == 0) {
    if (b + kSeg <= n) {
      const float4* src = reinterpret_cast<const float4*>(h + b);
      for (int e = threadIdx.x; e < kSeg / 4; e += NT) reinterpret_cast<float4*>(hs)[e] = __ldg(src + e);
    } else {
      for (int e = threadIdx.x * 4; e < kSeg; e += NT * 4) {
        int64_t s = b + e;
        if (s >= n) s %= n;
        *reinterpret_cast<float4*>(hs + e) = __ldg(reinterpret_cast<const float4*>(h + s));
      }
    }
  } else {
    for (int e = threadIdx.x; e < kSeg; e += NT) hs[e] = __ldg(h + (b + e) % n);
  }
}

template <int N, int K>
__device__ __forceinline__ void ld4(float (&w)[N], const float* __restrict__ p) {
  const float4 t = *reinterpret_cast<const float4*>(p + K);
  w[K] = t.x;
  w[K + 1] = t.y;
  w[K + 2] = t.z;
  w[K + 3] = t.w;
}

// Gradient block: acc[q] += w[q - s + 32] * r[s] for the rows s of the block,
// ascending s (the reference's ascending-row order).  w[k] = wp[k].
// Row test of position s.  PAIR: positions are first tested in pairs, so an
// empty pair (9/16 of pairs at density 1/4) costs one taken branch over two
// bodies instead of two (a taken branch over a body lands on code that was
// never fetched: an instruction-cache miss).
__device__ __forceinline__ bool row_at(uint32_t mask, int s) { return (mask >> s) & 1u; }
template <bool PAIR>
__device__ __forceinline__ bool pair_live(uint32_t mask, int s) { return !PAIR || ((mask >> s) & 3u); }

template <int R, int G, bool PAIR>
__device__ __forceinline__ void grad_group_s(float (&acc)[R], float (&w)[R + 32], uint32_t mask,
                                             const float* __restrict__ wp, const float* __restrict__ rb,
                                             float4& r4) {
  float4 rn;
  if constexpr (G < 7) {
    rn = *reinterpret_cast<const float4*>(rb + 4 * (G + 1));
    ld4<R + 32, 24 - 4 * G>(w, wp);
  }
  const float rr[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
  for (int e2 = 0; e2 < 4; e2 += 2) {
    if (pair_live<PAIR>(mask, 4 * G + e2)) {
#pragma unroll
      for (int e = e2; e < e2 + 2; ++e) {
        const int s = 4 * G + e;
        if (row_at(mask, s)) {
#pragma unroll
          for (int q = 0; q < R; ++q) acc[q] = fmaf(w[q - s + 32], rr[e], acc[q]);
        }
      }
    }
  }
  if constexpr (G < 7) r4 = rn;
}

template <int R, bool PAIR>
__device__ __forceinline__ void grad_block_s(float (&acc)[R], const float* __restrict__ wp,
                                             const float* __restrict__ rb, uint32_t mask) {
  float w[R + 32];
#pragma unroll
  for (int k = 28; k < R + 32; k += 4) {
    const float4 t = *reinterpret_cast<const float4*>(wp + k);
    w[k] = t.x;
    w[k + 1] = t.y;
    w[k + 2] = t.z;
    w[k + 3] = t.w;
  }
  float4 r4 = *reinterpret_cast<const float4*>(rb);
  grad_group_s<R, 0, PAIR>(acc, w, mask, wp, rb, r4);
  grad_group_s<R, 1, PAIR>(acc, w, mask, wp, rb, r4);
  grad_group_s<R, 2, PAIR>(acc, w, mask, wp, rb, r4);
  grad_group_s<R, 3, PAIR>(acc, w, mask, wp, rb, r4);
  grad_group_s<R, 4, PAIR>(acc, w, mask, wp, rb, r4);
  grad_group_s<R, 5, PAIR>(acc, w, mask, wp, rb, r4);
  grad_group_s<R, 6, PAIR>(acc, w, mask, wp, rb, r4);
  grad_group_s<R, 7, PAIR>(acc, w, mask, wp, rb, r4);
}

template <int R, int MINB, bool PAIR = false, int NT = kThreads>
__global__ void __launch_bounds__(NT, MINB)
k_grad_s(const float* __restrict__ h, const int* __restrict__ omega, const float* __restrict__ rv,
         const int* __restrict__ rowstart, int64_t n, int64_t chunks, int splits, int64_t tile_lo,
         float* __restrict__ partial) {
  constexpr int PB = 32;
  using G = GeoU<R, NT>;
  extern __shared__ float4 smem_f4[];
  float* hs = reinterpret_cast<float*>(smem_f4);
  float* rd = hs + G::kSegPhys;
  uint32_t* bmask = reinterpret_cast<uint32_t*>(rd + kChunk);
  const int64_t unit = blockIdx.x;
  const int64_t tile = tile_lo + unit / splits;
  const int split = static_cast<int>(unit % splits);
  const int64_t I0 = tile * G::kTileR;
  int64_t blo, bhi;
  split_blocks(chunks, splits, split, &blo, &bhi);
  const int own = threadIdx.x, warp = own >> 5, lane = own & 31;

  float acc[R];
#pragma unroll
  for (int q = 0; q < R; ++q) acc[q] = 0.f;

  for (int64_t ch = blo / (kChunk / 32); ch * (kChunk / 32) < bhi; ++ch) {
    const int64_t Jc = ch * kChunk;
    const int r0 = rowstart[ch], nr = rowstart[ch + 1] - r0;
    if (nr == 0) continue;
    stage_plain<G::kSeg, NT>(hs, h, n, I0 - Jc - kChunk);
    for (int s = threadIdx.x; s < kChunk; s += NT) rd[s] = 0.f;
    __syncthreads();
    for (int k = threadIdx.x; k < nr; k += NT) rd[omega[r0 + k] - static_cast<int>(Jc)] = __ldg(rv + r0 + k);
    __syncthreads();
    for (int b32 = warp; b32 < kChunk / 32; b32 += NT / 32) {
      const uint32_t mk = g_force_dense ? 0xffffffffu : __ballot_sync(0xffffffffu, rd[b32 * 32 + lane] != 0.f);
      if (lane == 0) bmask[b32] = mk;
    }
    __syncthreads();
    const int64_t cb = ch * (kChunk / 32);
    const int b0 = static_cast<int>(blo > cb ? blo - cb : 0);
    const int b1 = static_cast<int>(bhi - cb < kChunk / 32 ? bhi - cb : kChunk / 32);
    const float* wl = hs + own * R + kChunk - PB;
    for (int b = b0; b < b1; ++b) {
      const uint32_t mask = __reduce_or_sync(0xffffffffu, bmask[b]);
      if (mask == 0u) continue;
      grad_block_s<R, PAIR>(acc, wl - b * PB, rd + b * PB, mask);
    }
    __syncthreads();
  }
  const int64_t ib = I0 + own * R;
  float* out = partial + static_cast<int64_t>(split) * n;
#pragma unroll
  for (int q = 0; q < R; ++q)
    if (ib + q < n) out[ib + q] = acc[q];
}

// Residual block (dot form, x register-resident): row s computes
// sum_q w[s - q + R] x[q]; position s needs w[s+1 .. s+R], so the window
// moves up by 4 per group.
template <int R, int S, int CH>
__device__ __forceinline__ void res_row_s(const float (&w)[R + 32], const float (&xr)[R], float*& lpp) {
  float p[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) p[c] = w[S - c + R] * xr[c];
#pragma unroll
  for (int q = CH; q < R; ++q) p[q % CH] = fmaf(w[S - q + R], xr[q], p[q % CH]);
#pragma unroll
  for (int width = CH; width > 1; width = (width + 1) / 2)
#pragma unroll
    for (int c = 0; c < width / 2; ++c) p[c] += p[c + (width + 1) / 2];
  *lpp++ = p[0];
}

template <int R, int G, bool PAIR, int CH>
__device__ __forceinline__ void res_group_s(float (&w)[R + 32], const float (&xr)[R], uint32_t mask,
                                            const float* __restrict__ wp, float*& lpp) {
  if constexpr (G < 7) ld4<R + 32, R + 4 + 4 * G>(w, wp);
  if (pair_live<PAIR>(mask, 4 * G)) {
    if (row_at(mask, 4 * G)) res_row_s<R, 4 * G, CH>(w, xr, lpp);
    if (row_at(mask, 4 * G + 1)) res_row_s<R, 4 * G + 1, CH>(w, xr, lpp);
  }
  if (pair_live<PAIR>(mask, 4 * G + 2)) {
    if (row_at(mask, 4 * G + 2)) res_row_s<R, 4 * G + 2, CH>(w, xr, lpp);
    if (row_at(mask, 4 * G + 3)) res_row_s<R, 4 * G + 3, CH>(w, xr, lpp);
  }
}

template <int R, bool PAIR, int CH>
__device__ __forceinline__ void res_block_s(const float* __restrict__ wp, const float (&xr)[R], uint32_t mask,
                                            float*& lpp) {
  float w[R + 32];
#pragma unroll
  for (int k = 0; k < R + 4; k += 4) {
    const float4 t = *reinterpret_cast<const float4*>(wp + k);
    w[k] = t.x;
    w[k + 1] = t.y;
    w[k + 2] = t.z;
    w[k + 3] = t.w;
  }
  res_group_s<R, 0, PAIR, CH>(w, xr, mask, wp, lpp);
  res_group_s<R, 1, PAIR, CH>(w, xr, mask, wp, lpp);
  res_group_s<R, 2, PAIR, CH>(w, xr, mask, wp, lpp);
  res_group_s<R, 3, PAIR, CH>(w, xr, mask, wp, lpp);
  res_group_s<R, 4, PAIR, CH>(w, xr, mask, wp, lpp);
  res_group_s<R, 5, PAIR, CH>(w, xr, mask, wp, lpp);
  res_group_s<R, 6, PAIR, CH>(w, xr, mask, wp, lpp);
  res_group_s<R, 7, PAIR, CH>(w, xr, mask, wp, lpp);
}

template <int R, int MINB, bool PAIR = false, int CH = kResChains>
__global__ void __launch_bounds__(kThreads, MINB)
k_res_s(const float* __restrict__ h, const float* __restrict__ x, const int* __restrict__ omega,
        const int* __restrict__ rowstart, int64_t n, int64_t m, int64_t chunks, int splits, int split_lo,
        int split_cnt, float* __restrict__ partial) {
  constexpr int PB = 32, NB = kChunk / PB;
  using G = GeoU<R>;
  extern __shared__ float4 smem_f4[];
  float* hs = reinterpret_cast<float*>(smem_f4);
  uint32_t* bmask = reinterpret_cast<uint32_t*>(hs + G::kSegPhys);  // [NB]
  int* bbase = reinterpret_cast<int*>(bmask + NB);                   // [NB]
  float* red = reinterpret_cast<float*>(bbase + NB);                 // [kWarps][kChunk]
  int* flag = reinterpret_cast<int*>(red);  // [kChunk] row flags, dead before red is written
  float* lanep = red + kWarps * kChunk;     // [kWarps][32 lanes][33]
  const int64_t unit = blockIdx.x;
  const int64_t tile = unit / split_cnt;
  const int split = split_lo + static_cast<int>(unit % split_cnt);
  const int64_t I0 = tile * G::kTileR;
  int64_t blo, bhi;
  split_blocks(chunks, splits, split, &blo, &bhi);
  const int own = threadIdx.x, warp = own >> 5, lane = own & 31;
  const float* lane_base = hs + (kThreads - 1 - own) * R;
  float* redw = red + warp * kChunk;
  float* lp = lanep + warp * 32 * 33;
  float* const lp_lane = lp + lane * 33;

  float xr[R];
  const int64_t jb = I0 + own * R;
#pragma unroll
  for (int q = 0; q < R; ++q) xr[q] = (jb + q < n) ? __ldg(x + jb + q) : 0.f;

  for (int64_t ch = blo / (kChunk / 32); ch * (kChunk / 32) < bhi; ++ch) {
    const int64_t Jc = ch * kChunk;
    const int r0 = rowstart[ch], nr = rowstart[ch + 1] - r0;
    if (nr == 0) continue;
    stage_plain<G::kSeg>(hs, h, n, Jc - I0 - G::kTileR);
    for (int s = threadIdx.x; s < kChunk; s += kThreads) flag[s] = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < nr; k += kThreads) flag[omega[r0 + k] - static_cast<int>(Jc)] = 1;
    __syncthreads();
    if (warp == 0) {  // masks + exclusive prefix of row counts per block
      int run = 0;
      for (int b32 = 0; b32 < NB; ++b32) {
        const uint32_t mk = g_force_dense ? 0xffffffffu : __ballot_sync(0xffffffffu, flag[b32 * 32 + lane] != 0);
        if (lane == 0) {
          bmask[b32] = mk;
          bbase[b32] = run;
        }
        run += __popc(mk);
      }
    }
    __syncthreads();
    const int64_t cb = ch * (kChunk / 32);
    const int b0 = static_cast<int>(blo > cb ? blo - cb : 0);
    const int b1 = static_cast<int>(bhi - cb < kChunk / 32 ? bhi - cb : kChunk / 32);
    for (int b = b0; b < b1; ++b) {
      const uint32_t mask = __reduce_or_sync(0xffffffffu, bmask[b]);
      if (mask == 0u) continue;
      float* lpp = lp_lane;
      res_block_s<R, PAIR, CH>(lane_base + b * PB, xr, mask, lpp);
      __syncwarp();
      reduce_lane_partials(lp, redw, bbase[b], __popc(mask), lane);
      __syncwarp();
    }
    __syncthreads();
    float* outp = partial + tile * m + r0;
    const int k_lo = b0 < NB ? bbase[b0] : nr;
    const int k_hi = b1 < NB ? bbase[b1] : nr;
    for (int kk = k_lo + threadIdx.x; kk < k_hi; kk += kThreads) {
      float s = red[kk];
#pragma unroll
      for (int wi = 1; wi < kWarps; ++wi) s += red[wi * kChunk + kk];
      outp[kk] = s;
    }
    __syncthreads();
  }
}

// ===========================================================================
// Persistent cooperative cADMM for small n (config 2: n = 4096).
// One launch runs all unchecked iterations; CTA b owns position block b (the
// 32 inputs of each product it multiplies in, with the three operator rows'
// segments staged once in shared memory) and outputs [32 b, 32 b + 32) for the
// fused updates.  Per iteration (cpadmm_phases, parallel.hpp:173-231):
//   C^T v -> beta -> B beta -> x -> C x -> duals, a grid barrier after each
// product (split-K partials) and each update.  The tile is the whole problem
// (128 threads x R = n); partials are summed in ascending block order.
// ===========================================================================
template <int R>
__device__ __forceinline__ void coop_product(float (&acc)[R], const float* __restrict__ lane_base,
                                             const float* __restrict__ us) {
  constexpr int PB = 32;
#pragma unroll
  for (int q = 0; q < R; ++q) acc[q] = 0.f;
  float w[R + PB];
  window_at<R, PB>(w, lane_base, 0);
#pragma unroll
  for (int s4 = 0; s4 < PB; s4 += 4) {
    const float4 uu = *reinterpret_cast<const float4*>(us + s4);
    const float uv[4] = {uu.x, uu.y, uu.z, uu.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
#pragma unroll
      for (int q = 0; q < R; ++q) acc[q] = fmaf(w[q - (s4 + e) + PB], uv[e], acc[q]);
    }
  }
}

struct CoopArgs {
  const float *hc, *hbr, *hcr, *d, *pty;
  float *x, *z, *nu, *mu, *v, *beta, *partial;
  int64_t n;
  float rho, sigma, tau1, tau2, thr;
  int iters;
};

template <int R>
__global__ void __launch_bounds__(kThreads, 1) k_coop_cadmm(CoopArgs a) {
  using G = Geo<R>;
  constexpr int PB = 32;
  constexpr int SEG = G::pad(G::kTileR + PB) + 4;  // one block's segment (logical kTileR + 32)
  extern __shared__ float4 smem_f4[];
  float* s_c = reinterpret_cast<float*>(smem_f4);
  float* s_b = s_c + SEG;
  float* s_r = s_b + SEG;
  float* us = s_r + SEG;          // [32]
  float* red = us + PB;           // [4][32]
  cg::grid_group grid = cg::this_grid();
  const int64_t n = a.n;
  const int b = blockIdx.x, own = threadIdx.x;
  const int64_t Jb = static_cast<int64_t>(b) * PB;
  // segments hs[pad(e)] = h[(-Jb - 32 + e) mod n], e < kTileR + 32 (I0 = 0: one tile)
  for (int e = threadIdx.x; e < G::kTileR + PB; e += kThreads) {
    int64_t k = (e - Jb - PB) % n;
    if (k < 0) k += n;
    s_c[G::pad(e)] = a.hc[k];
    s_b[G::pad(e)] = a.hbr[k];
    s_r[G::pad(e)] = a.hcr[k];
  }
  __syncthreads();
  const int ib = own * R;
  float acc[R];
  const int o = own & 31, part = own >> 5;
  const int64_t i_out = Jb + o;  // this thread's output in the update phases (parts combined by thread o)
  auto sum_partials = [&](void) -> float {  // fixed order: 4 parts of 32 blocks, ascending
    const int nb = static_cast<int>(gridDim.x);
    const int k0 = part * ((nb + 3) / 4), k1 = min(nb, k0 + (nb + 3) / 4);
    float sacc = 0.f;
    for (int k = k0; k < k1; ++k) sacc += a.partial[static_cast<int64_t>(k) * n + i_out];
    red[part * 32 + o] = sacc;
    __syncthreads();
    const float tot = (red[o] + red[32 + o]) + (red[64 + o] + red[96 + o]);
    __syncthreads();
    return tot;
  };
  auto product = [&](const float* seg, const float* u) {
    if (threadIdx.x < PB) us[threadIdx.x] = u[Jb + threadIdx.x];
    __syncthreads();
    coop_product<R>(acc, seg + own * G::kPitch, us);
    float* out = a.partial + static_cast<int64_t>(b) * n;
#pragma unroll
    for (int q = 0; q < R; ++q) out[ib + q] = acc[q];
    __syncthreads();
  };
  for (int it = 0; it < a.iters; ++it) {
    product(s_c, a.v);  // C^T v
    grid.sync();
    {
      const float sct = sum_partials();
      if (part == 0)  // parallel.hpp:186-187
        a.beta[i_out] = __fadd_rn(__fmul_rn(a.rho, sct), __fmul_rn(a.sigma, __fsub_rn(a.z[i_out], a.nu[i_out])));
    }
    grid.sync();
    product(s_b, a.beta);  // B beta
    grid.sync();
    {
      const float xs = sum_partials();
      if (part == 0) a.x[i_out] = xs;
    }
    grid.sync();
    product(s_r, a.x);  // C x
    grid.sync();
    {
      const float cx = sum_partials();
      if (part == 0) {  // parallel.hpp:215-221
        const float xi = a.x[i_out], nui = a.nu[i_out];
        const float vn = __fmul_rn(a.d[i_out], __fadd_rn(__fmul_rn(a.rho, __fsub_rn(cx, a.mu[i_out])), a.pty[i_out]));
        const float sv = __fadd_rn(xi, nui);
        const float zn = sv > a.thr ? sv - a.thr : (sv < -a.thr ? sv + a.thr : 0.f);
        const float mun = __fadd_rn(a.mu[i_out], __fmul_rn(a.tau1, __fsub_rn(vn, cx)));
        a.z[i_out] = zn;
        a.mu[i_out] = mun;
        a.nu[i_out] = __fadd_rn(nui, __fmul_rn(a.tau2, __fsub_rn(xi, zn)));
        a.v[i_out] = __fadd_rn(vn, mun);
      }
    }
    grid.sync();
  }
}

// Persistent cooperative ISTA for small n (config 1): CTA b owns position block
// b.  Per iteration (cpista_phases, parallel.hpp:236-279) it computes the
// residual of block b's rows (x in registers, lane partials reduced in fixed
// order), keeps those r values in shared memory, multiplies them into a split-K
// partial of the gradient for all n outputs, and -- after one grid barrier --
// sums the partials of outputs [32 b, 32 b + 32) and applies the threshold.
// Only x crosses CTAs (a second barrier), so two barriers per iteration.
struct CoopIstaArgs {
  const float *hc, *hcr, *y;
  const int* omega;
  float *x, *r, *delta, *partial;
  int64_t n, m;
  float tau, thr;
  int iters;
};

template <int R>
__global__ void __launch_bounds__(kThreads, 1) k_coop_ista(CoopIstaArgs a) {
  using G = Geo<R>;
  constexpr int PB = 32;
  constexpr int SEG = G::pad(G::kTileR + PB) + 4;
  extern __shared__ float4 smem_f4[];
  float* s_g = reinterpret_cast<float*>(smem_f4);  // gradient segment: h = c~, base -Jb - 32
  float* s_r = s_g + SEG;                             // residual segment: h = c~_rev, base Jb - kTileR
  float* rd = s_r + SEG;                              // [32] r at the block's positions (0 elsewhere)
  float* red = rd + PB;                               // [kWarps][32] per-warp row sums; update parts
  float* lanep = red + kWarps * PB;                   // [kWarps][32][33]
  int* meta = reinterpret_cast<int*>(lanep + kWarps * 32 * 33);  // [0] mask, [1] first row, [2] rows
  cg::grid_group grid = cg::this_grid();
  const int64_t n = a.n;
  const int b = blockIdx.x, own = threadIdx.x, warp = own >> 5, lane = own & 31;
  const int64_t Jb = static_cast<int64_t>(b) * PB;
  for (int e = threadIdx.x; e < G::kTileR + PB; e += kThreads) {
    int64_t kg = (e - Jb - PB) % n;
    if (kg < 0) kg += n;
    int64_t kr = (Jb - G::kTileR + e) % n;
    if (kr < 0) kr += n;
    s_g[G::pad(e)] = a.hc[kg];
    s_r[G::pad(e)] = a.hcr[kr];
  }
  if (threadIdx.x == 0) {  // this block's rows: omega is sorted, so they are one contiguous run
    int64_t lo = 0, hi = a.m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (a.omega[mid] < Jb) lo = mid + 1;
      else hi = mid;
    }
    uint32_t mask = 0u;
    int64_t t = lo;
    while (t < a.m && a.omega[t] < Jb + PB) mask |= 1u << (a.omega[t++] - Jb);
    meta[0] = static_cast<int>(mask);
    meta[1] = static_cast<int>(lo);
    meta[2] = static_cast<int>(t - lo);
  }
  __syncthreads();
  const uint32_t mask = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(meta[0]));
  const int t0 = meta[1], nrow = meta[2];
  const int o = own & 31, part = own >> 5;
  const int64_t i_out = Jb + o;
  float* lp = lanep + warp * 32 * 33;
  float* const lp_lane = lp + lane * 33;
  for (int it = 0; it < a.iters; ++it) {
    // residual rows of block b: r_t = y_t - sum_j c~[(j - omega_t) mod n] x_j
    float xr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) xr[q] = a.x[own * R + q];
    if (mask) {
      float w[R + PB];
      window_at<R, PB>(w, s_r + (kThreads - 1 - own) * G::kPitch, 0);
      float* lpp = lp_lane;
      res_group<R, PB, 0>(w, xr, mask, lpp);
      res_group<R, PB, 1>(w, xr, mask, lpp);
      res_group<R, PB, 2>(w, xr, mask, lpp);
      res_group<R, PB, 3>(w, xr, mask, lpp);
      res_group<R, PB, 4>(w, xr, mask, lpp);
      res_group<R, PB, 5>(w, xr, mask, lpp);
      res_group<R, PB, 6>(w, xr, mask, lpp);
      res_group<R, PB, 7>(w, xr, mask, lpp);
      __syncwarp();
      reduce_lane_partials(lp, red + warp * PB, 0, nrow, lane);
    }
    __syncthreads();
    if (threadIdx.x < PB) rd[threadIdx.x] = 0.f;
    __syncthreads();
    if (threadIdx.x < nrow) {  // fixed-order warp sum; the block's r values stay in shared memory
      const float sres = (red[threadIdx.x] + red[PB + threadIdx.x]) + (red[2 * PB + threadIdx.x] + red[3 * PB + threadIdx.x]);
      const float rv = a.y[t0 + threadIdx.x] - sres;  // parallel.hpp:252
      const int pos = a.omega[t0 + threadIdx.x];
      rd[pos - Jb] = rv;
      if (it == a.iters - 1) a.r[t0 + threadIdx.x] = rv;
    }
    __syncthreads();
    // gradient partial of block b for all outputs: acc[q] += c~[(i - omega_t) mod n] r_t
    float acc[R];
#pragma unroll
    for (int q = 0; q < R; ++q) acc[q] = 0.f;
    if (mask) {
      float w[R + PB];
      window_at<R, PB>(w, s_g + own * G::kPitch, 0);
      ool_block32<R>(acc, w, mask, rd);
    }
    float* outp = a.partial + static_cast<int64_t>(b) * n + own * R;
#pragma unroll
    for (int q = 0; q < R; ++q) outp[q] = acc[q];
    grid.sync();
    // update of outputs [32 b, 32 b + 32): delta = sum of the block partials (fixed order), x = eta(x + tau delta)
    {
      const int nb = static_cast<int>(gridDim.x);
      const int k0 = part * ((nb + 3) / 4), k1 = min(nb, k0 + (nb + 3) / 4);
      float sacc = 0.f;
      for (int k = k0; k < k1; ++k) sacc += a.partial[static_cast<int64_t>(k) * n + i_out];
      red[part * 32 + o] = sacc;
      __syncthreads();
      if (part == 0) {
        const float d = (red[o] + red[32 + o]) + (red[64 + o] + red[96 + o]);
        const float xn = __fadd_rn(a.x[i_out], __fmul_rn(a.tau, d));  // parallel.hpp:269-271
        a.x[i_out] = xn > a.thr ? xn - a.thr : (xn < -a.thr ? xn + a.thr : 0.f);
        if (it == a.iters - 1) a.delta[i_out] = d;
      }
    }
    grid.sync();
  }
}

template <int R>
constexpr size_t coop_ista_smem() {
  return (2 * (Geo<R>::pad(Geo<R>::kTileR + 32) + 4) + 32 + kWarps * 32 + kWarps * 32 * 33 + 4) * 4;
}

template <int R>
constexpr size_t coop_smem() { return (3 * (Geo<R>::pad(Geo<R>::kTileR + 32) + 4) + 32 + 128) * 4; }

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

// the fused all-gather of the peer-store transport (EpiArgs::peer): the same value at the same index on
// every other rank (NVLink stores when the ranks sit on different GPUs)
__device__ __forceinline__ void to_peers(const EpiArgs& a, int64_t i, float v) {
  for (int p = 0; p < a.npeer; ++p) a.peer[p][i] = v;
}
// after a thread's last peer store: visible system-wide (another process's or GPU's reads) before the
// rank's phase flag is raised by the next kernel
__device__ __forceinline__ void peers_fence(const EpiArgs& a) {
  if (a.npeer) __threadfence_system();
}

__device__ __forceinline__ float sum_partials(const float* __restrict__ p, int splits, int64_t stride, int64_t i) {
  float s = p[i];
  for (int k = 1; k < splits; ++k) s += p[k * stride + i];
  return s;
}
// the same ascending sum with the loads of 8 splits issued together ahead of their adds: for the residual's
// gather at the rows Omega (scattered 4-byte loads, latency-bound: 0.031 vs 0.042 ms at C3); the contiguous
// epilogues keep the plain loop (batched: 0.17 vs 0.105 ms for the ISTA update)
__device__ __forceinline__ float sum_partials_batched(const float* __restrict__ p, int splits, int64_t stride,
                                                      int64_t i) {
  float s = p[i];
  int k = 1;
  for (; k + 8 <= splits; k += 8) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldcs(p + (k + q) * stride + i);
#pragma unroll
    for (int q = 0; q < 8; ++q) s += v[q];
  }
  for (; k < splits; ++k) s += __ldcs(p + k * stride + i);
  return s;
}

__global__ void __launch_bounds__(kThreads) k_residual_reduce(EpiArgs a, int64_t tiles) {
  // r[t] = y[t] - sum_tile partial[tile][t]   (cpista residual, parallel.hpp:252)
  for (int64_t t = a.lo + blockIdx.x * (int64_t)kThreads + threadIdx.x; t < a.hi;
       t += (int64_t)gridDim.x * kThreads) {
    const float s = sum_partials(a.partial, static_cast<int>(tiles), a.n, t);
    const float rv = a.y[t] - s;
    a.r[t] = rv;
    to_peers(a, t, rv);
  }
  peers_fence(a);
}

__global__ void __launch_bounds__(kThreads) k_residual_gather(EpiArgs a, const int* __restrict__ omega) {
  // r[t] = y[t] - (C x)[omega[t]], C x from the dense product's split partials (a.n = n)
  for (int64_t t = a.lo + blockIdx.x * (int64_t)kThreads + threadIdx.x; t < a.hi;
       t += (int64_t)gridDim.x * kThreads) {
    const float s = sum_partials_batched(a.partial, a.splits, a.n, omega[t]);
    const float rv = a.y[t] - s;
    a.r[t] = rv;
    to_peers(a, t, rv);
  }
  peers_fence(a);
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
    to_peers(a, i, xn);
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
  peers_fence(a);
  if (a.want_metrics) block_metrics(m0, m1, m2, a.blk);
}

__global__ void __launch_bounds__(kThreads) k_admm_beta(EpiArgs a) {
  // beta = rho * C^T v + sigma * (z - nu)   (parallel.hpp:186-187)
  for (int64_t i = a.lo + blockIdx.x * (int64_t)kThreads + threadIdx.x; i < a.hi;
       i += (int64_t)gridDim.x * kThreads) {
    const float s = sum_partials(a.partial, a.splits, a.n, i);
    const float b = __fadd_rn(__fmul_rn(a.rho, s), __fmul_rn(a.sigma, __fsub_rn(a.z[i], a.nu[i])));
    a.beta[i] = b;
    to_peers(a, i, b);
  }
  peers_fence(a);
}

__global__ void __launch_bounds__(kThreads) k_admm_x(EpiArgs a) {
  for (int64_t i = a.lo + blockIdx.x * (int64_t)kThreads + threadIdx.x; i < a.hi;
       i += (int64_t)gridDim.x * kThreads) {
    const float xv = sum_partials(a.partial, a.splits, a.n, i);
    a.x[i] = xv;
    to_peers(a, i, xv);
  }
  peers_fence(a);
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__global__ void __launch_bounds__(kThreads) k_admm_duals(EpiArgs a) {
  // parallel.hpp:215-221
  if (a.vec4) {
    // the FFT engine's unchecked iterations (one split, no metrics, no peers): 4 consecutive entries per thread,
    // every input loaded before any store, z not read (its old value only feeds the metrics); the per-entry
    // arithmetic is the scalar loop's below, bit for bit
    for (int64_t i = a.lo + 4 * (blockIdx.x * (int64_t)kThreads + threadIdx.x); i < a.hi;
         i += 4 * (int64_t)gridDim.x * kThreads) {
      const float4 cx4 = ld4(a.partial + i), x4 = ld4(a.x + i), nu4 = ld4(a.nu + i), mu4 = ld4(a.mu + i);
      const float4 d4 = ld4(a.d + i), py4 = ld4(a.pty + i);
      const float cxa[4] = {cx4.x, cx4.y, cx4.z, cx4.w}, xa[4] = {x4.x, x4.y, x4.z, x4.w};
      const float nua[4] = {nu4.x, nu4.y, nu4.z, nu4.w}, mua[4] = {mu4.x, mu4.y, mu4.z, mu4.w};
      const float da[4] = {d4.x, d4.y, d4.z, d4.w}, pya[4] = {py4.x, py4.y, py4.z, py4.w};
      float zr[4], mur[4], nur[4], vr[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float cx = cxa[q], xi = xa[q], nui = nua[q];
        const float vn = __fmul_rn(da[q], __fadd_rn(__fmul_rn(a.rho, __fsub_rn(cx, mua[q])), pya[q]));
        zr[q] = soft(__fadd_rn(xi, nui), a.thr);
        mur[q] = __fadd_rn(mua[q], __fmul_rn(a.tau1, __fsub_rn(vn, cx)));
        nur[q] = __fadd_rn(nui, __fmul_rn(a.tau2, __fsub_rn(xi, zr[q])));
        vr[q] = __fadd_rn(vn, mur[q]);
      }
      st4(a.z + i, make_float4(zr[0], zr[1], zr[2], zr[3]));
      st4(a.mu + i, make_float4(mur[0], mur[1], mur[2], mur[3]));
      st4(a.nu + i, make_float4(nur[0], nur[1], nur[2], nur[3]));
      st4(a.v + i, make_float4(vr[0], vr[1], vr[2], vr[3]));
    }
    return;
  }
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
    const float vv = __fadd_rn(vn, mun);
    a.v[i] = vv;
    to_peers(a, i, vv);
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
  peers_fence(a);
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

// ---- matvec scheme benchmark (parallel.hpp:318-406, paper Fig. 5) -------------
// The "reference" scheme streams a dense row-major copy of the circulant
// (n^2 + n unique fetches); the circulant scheme is the direct engine's dense
// product (2n unique fetches).  M[i][j] = c[(j - i) mod n]  (circ_entry).
__global__ void k_materialize_circulant(const float* __restrict__ c, float* __restrict__ M, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    int64_t k = j - i;
    if (k < 0) k += n;
    M[e] = c[k];
  }
}
// out[i] = sum_j M[i][j] x[j]: one warp per row, coalesced float4 streaming, fixed-order warp tree.
__global__ void __launch_bounds__(256) k_dense_gemv(const float* __restrict__ M, const float* __restrict__ x,
                                                    float* __restrict__ out, int64_t n) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* mr = M + row * n;
  float acc = 0.f;
  if ((n & 3) == 0) {
    const float4* m4 = reinterpret_cast<const float4*>(mr);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t j = lane; j < n / 4; j += 32) {
      const float4 a = __ldcs(m4 + j), b = __ldg(x4 + j);
      acc = fmaf(a.x, b.x, acc);
      acc = fmaf(a.y, b.y, acc);
      acc = fmaf(a.z, b.z, acc);
      acc = fmaf(a.w, b.w, acc);
    }
  } else {
    for (int64_t j = lane; j < n; j += 32) acc = fmaf(__ldcs(mr + j), __ldg(x + j), acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[row] = acc;
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
template <int R, int PB>
constexpr size_t smem_rows() { return Geo<R>::kSegPhys * 4 + kChunk * 4 + (kChunk / PB) * 4; }
template <int R, int NT = kThreads>
constexpr size_t smem_grad_s() { return (GeoU<R, NT>::kSegPhys + kChunk + kChunk / 32) * 4; }
template <int R>
constexpr size_t smem_res_s() {
  return (GeoU<R>::kSegPhys + 2 * (kChunk / 32) + kWarps * kChunk + kWarps * 32 * 33) * 4;
}
template <int R, int PB>
constexpr size_t smem_res() {
  return Geo<R>::kSegPhys * 4 + 2 * (kChunk / PB) * 4 + kWarps * kChunk * 4 + kWarps * 32 * 33 * 4;
}

// Kernel variant table (CLB_GRAD / CLB_RES / CLB_DENSE select an entry; the entries are the defaults,
// the measured best on B200 -- the rejected variants of DESIGN.md §3 are no longer compiled in).
struct GradVariant {
  int R, PB;
  void (*fn)(const float*, const int*, const float*, const int*, int64_t, int64_t, int, int64_t, float*);
  size_t smem;
  int nt = kThreads;  // threads per CTA
};
struct ResVariant {
  int R, PB;
  void (*fn)(const float*, const float*, const int*, const int*, int64_t, int64_t, int64_t, int, int, int, float*);
  size_t smem;
};
const GradVariant kGrad[] = {
    {32, 32, k_conv_rows_ool<4>, smem_rows<32, 32>()},            // 0: small-n default (padded R = 32; C3: 17.2 ms)
    {44, 32, k_grad_s<44, 4, true>, smem_grad_s<44>()},           // 1: large-n default (streamed, pair tests)
};
const ResVariant kRes[] = {
    {32, 32, k_conv_residual<32, 32, 4>, smem_res<32, 32>()},     // 0: small-n default (padded R = 32, 4 CTAs/SM)
    {52, 32, k_res_s<52, 3, true, 2>, smem_res_s<52>()},          // 1: large-n default (streamed, pair tests, 2 chains)
};
struct DenseVariant {
  int R;
  void (*fn)(const float*, const float*, int64_t, int64_t, int, int64_t, float*);
  size_t smem;
};
const DenseVariant kDense[] = {
    {64, k_conv_dense<64>, smem_dense<64>()},   // 0: padded R = 64 (default for n > 4096)
    {32, k_conv_dense<32>, smem_dense<32>()},   // 1: R = 32: a 4096-index tile (default for 2048 < n <= 4096)
    {16, k_conv_dense<16>, smem_dense<16>()},   // 2: R = 16: a 2048-index tile (default for n <= 2048)
};
int g_dense = -1;  // -1: choose by n (a tile no longer than n: no idle threads at small n)
static int dense_index(int64_t n) {
  if (g_dense >= 0) return g_dense;
  return n <= 2048 ? 2 : n <= 4096 ? 1 : 0;
}

// Defaults (measured best on B200, tools/variants.py): the streamed-window
// kernels with pair tests at large n; the R = 32 padded kernels at small n,
// where a 4096-index tile already covers the whole problem.
constexpr int64_t kLargeN = int64_t(1) << 17;
constexpr int kGradLarge = 1, kGradSmall = 0, kResLarge = 1, kResSmall = 0;
int g_grad = -1, g_res = -1;  // -1: choose by n

}  // namespace

// Variant selection is pure host logic (no CUDA calls): shard ranges can be
// computed on a machine without a GPU.
static void select_variants() {
  static bool done = false;
  if (done) return;
  done = true;
  if (const char* v = getenv("CLB_GRAD")) g_grad = atoi(v) % (int)(sizeof(kGrad) / sizeof(kGrad[0]));
  if (const char* v = getenv("CLB_RES")) g_res = atoi(v) % (int)(sizeof(kRes) / sizeof(kRes[0]));
  if (const char* v = getenv("CLB_DENSE")) g_dense = atoi(v) % (int)(sizeof(kDense) / sizeof(kDense[0]));
}
static const GradVariant& grad_variant(int64_t n) {
  select_variants();
  return kGrad[g_grad >= 0 ? g_grad : (n >= kLargeN ? kGradLarge : kGradSmall)];
}
static const ResVariant& res_variant(int64_t n) {
  select_variants();
  return kRes[g_res >= 0 ? g_res : (n >= kLargeN ? kResLarge : kResSmall)];
}
int dense_R(int64_t n) {
  select_variants();
  return kDense[dense_index(n)].R;
}
// plan "R" = indices per 128 threads (the tile is kThreads * R)
int grad_R(int64_t n) { return grad_variant(n).R * grad_variant(n).nt / kThreads; }
int res_R(int64_t n) { return res_variant(n).R; }

void split_block_range(const ConvPlan& p, int split, int64_t* blo, int64_t* bhi) {
  split_blocks(p.chunks, p.splits, split, blo, bhi);
}

int64_t target_units(int64_t n) {
  static const int64_t forced = [] {
    const char* v = getenv("CLB_UNITS");
    return v ? static_cast<int64_t>(atoll(v)) : int64_t(0);
  }();
  if (forced > 0) return forced;
  return n >= kUnitsLargeN ? kTargetUnitsLarge : kTargetUnits;
}

ConvPlan make_plan(int64_t n, int R) {
  ConvPlan p;
  p.n = n;
  p.tile = static_cast<int64_t>(kThreads) * R;
  p.tiles = (n + p.tile - 1) / p.tile;
  p.chunks = (n + kChunk - 1) / kChunk;
  const int64_t units = target_units(n);
  int64_t s = (units + p.tiles - 1) / p.tiles;
  // a multiple of 8 splits: the residual is sharded by splits, so 2, 4 and 8 ranks get equal chunk
  // counts (a function of n only, like everything in the plan)
  if (s >= 8) s = (s + 7) / 8 * 8;
  const int64_t blocks32 = p.chunks * (kChunk / 32);  // splits are ranges of 32-position blocks
  if (s < 1) s = 1;
  if (s > blocks32) s = blocks32;
  p.splits = static_cast<int>(s);
  p.tile_lo = 0;
  p.tile_hi = p.tiles;
  p.split_lo = 0;
  p.split_hi = p.splits;
  return p;
}

void conv_kernels_init() {
  tc_dense_init();
  static std::atomic<uint64_t> devs{0};
  if (!first_use_on_device(devs)) return;
  if (const char* v = getenv("CLB_FORCE_DENSE")) {
    const int one = atoi(v);
    cudaMemcpyToSymbol(g_force_dense, &one, sizeof(int));
  }
  select_variants();
  for (const auto& d : kDense)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(d.fn), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem);
  for (const auto& g : kGrad)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(g.fn), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
  for (const auto& r : kRes)
    cudaFuncSetAttribute(reinterpret_cast<const void*>(r.fn), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)r.smem);
}

ConvPlan make_dense_plan(int64_t n) {
  const char* v = getenv("CLB_NO_TC");  // read per call (setup time): tests switch it per solver
  const bool no_tc = v && atoi(v) != 0;
  if (!no_tc && tc_dense_supported(n)) {
    ConvPlan p = make_tc_plan(n);
    p.tc = true;
    return p;
  }
  return make_plan(n, dense_R(n));
}

bool ista_uses_tc(int64_t n) { return n >= (int64_t(1) << 17) && make_dense_plan(n).tc; }

cudaError_t launch_conv_dense(const ConvPlan& p, const float* h, const float* u, float* partial, cudaStream_t st) {
  if (p.tc) return launch_tc_dense(p, h, u, partial, st);
  const int64_t units = (p.tile_hi - p.tile_lo) * p.splits;
  if (units <= 0) return cudaSuccess;
  select_variants();
  const DenseVariant& d = kDense[dense_index(p.n)];
  d.fn<<<static_cast<unsigned>(units), kThreads, d.smem, st>>>(h, u, p.n, p.chunks, p.splits, p.tile_lo, partial);
  return cudaGetLastError();
}

void launch_conv_rows(const ConvPlan& p, const float* h, const int* omega32, const float* rvals, const int* rowstart,
                      float* partial, cudaStream_t st) {
  const int64_t units = (p.tile_hi - p.tile_lo) * p.splits;
  if (units <= 0) return;
  const GradVariant& g = grad_variant(p.n);
  g.fn<<<static_cast<unsigned>(units), g.nt, g.smem, st>>>(h, omega32, rvals, rowstart, p.n, p.chunks, p.splits,
                                                              p.tile_lo, partial);
}

void launch_conv_residual(const ConvPlan& p, int64_t m, const float* h, const float* x, const int* omega32,
                          const int* rowstart, float* partial, cudaStream_t st) {
  const int cnt = p.split_hi - p.split_lo;
  const int64_t units = p.tiles * cnt;
  if (units <= 0) return;
  const ResVariant& r = res_variant(p.n);
  r.fn<<<static_cast<unsigned>(units), kThreads, r.smem, st>>>(h, x, omega32, rowstart, p.n, m, p.chunks, p.splits,
                                                              p.split_lo, cnt, partial);
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
void launch_ista_residual_gather(const EpiArgs& a, const int* omega, cudaStream_t st) {
  k_residual_gather<<<epi_grid(a.hi - a.lo), kThreads, 0, st>>>(a, omega);
}
void launch_ista_update(const EpiArgs& a, cudaStream_t st) {
  k_ista_update<<<a.want_metrics ? kEpiBlocks : epi_grid(a.hi - a.lo), kThreads, 0, st>>>(a);
}
void launch_admm_beta(const EpiArgs& a, cudaStream_t st) { k_admm_beta<<<epi_grid(a.hi - a.lo), kThreads, 0, st>>>(a); }
void launch_admm_x(const EpiArgs& a, cudaStream_t st) { k_admm_x<<<epi_grid(a.hi - a.lo), kThreads, 0, st>>>(a); }
void launch_admm_duals(const EpiArgs& a, cudaStream_t st) {
  EpiArgs b = a;
  const auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  b.vec4 = a.splits == 1 && !a.want_metrics && a.npeer == 0 && a.lo % 4 == 0 && a.hi % 4 == 0 && al(a.partial) &&
           al(a.x) && al(a.nu) && al(a.mu) && al(a.d) && al(a.pty) && al(a.z) && al(a.v);
  k_admm_duals<<<a.want_metrics ? kEpiBlocks : epi_grid(a.hi - a.lo), kThreads, 0, st>>>(b);
}
void launch_materialize_circulant(const float* c, float* M, int64_t n, cudaStream_t st) {
  k_materialize_circulant<<<148 * 16, 256, 0, st>>>(c, M, n);
}
void launch_dense_gemv(const float* M, const float* x, float* out, int64_t n, cudaStream_t st) {
  k_dense_gemv<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, st>>>(M, x, out, n);
}
void launch_metrics_final(const double* blk, double* out4, cudaStream_t st) {
  k_metrics_final<<<1, 256, 0, st>>>(blk, out4);
}

bool coop_cadmm_supported(int64_t n) {
  const char* v = getenv("CLB_NO_SMALL");
  return !(v && v[0] == '1') && (n == 2048 || n == 4096 || n == 8192);
}
cudaError_t launch_coop_cadmm(int64_t n, const float* hc, const float* hbr, const float* hcr, const float* d,
                              const float* pty, float* x, float* z, float* nu, float* mu, float* v, float* beta,
                              float* partial, float rho, float sigma, float tau1, float tau2, float thr, int iters,
                              cudaStream_t st) {
  CoopArgs a{hc, hbr, hcr, d, pty, x, z, nu, mu, v, beta, partial, n, rho, sigma, tau1, tau2, thr, iters};
  void* args[] = {&a};
  const dim3 grid(static_cast<unsigned>(n / 32)), block(kThreads);
  switch (n) {
#define CLB_COOP(N, R)                                                                                      \
  case N: {                                                                                                 \
    static std::atomic<uint64_t> attr{0};                                                                   \
    if (first_use_on_device(attr)) {                                                                        \
      cudaFuncSetAttribute(k_coop_cadmm<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coop_smem<R>()); \
    }                                                                                                       \
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_coop_cadmm<R>), grid, block, args,   \
                                       coop_smem<R>(), st);                                                 \
  }
    CLB_COOP(2048, 16)
    CLB_COOP(4096, 32)
    CLB_COOP(8192, 64)
#undef CLB_COOP
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_coop_ista(int64_t n, int64_t m, const float* hc, const float* hcr, const int* omega,
                             const float* y, float* x, float* r, float* delta, float* partial, float tau, float thr,
                             int iters, cudaStream_t st) {
  CoopIstaArgs a{hc, hcr, y, omega, x, r, delta, partial, n, m, tau, thr, iters};
  void* args[] = {&a};
  const dim3 grid(static_cast<unsigned>(n / 32)), block(kThreads);
  switch (n) {
#define CLB_COOPI(N, R)                                                                                     \
  case N: {                                                                                                 \
    static std::atomic<uint64_t> attr{0};                                                                   \
    if (first_use_on_device(attr)) {                                                                        \
      cudaFuncSetAttribute(k_coop_ista<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)coop_ista_smem<R>()); \
    }                                                                                                       \
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_coop_ista<R>), grid, block, args,    \
                                       coop_ista_smem<R>(), st);                                            \
  }
    CLB_COOPI(2048, 16)
    CLB_COOPI(4096, 32)
    CLB_COOPI(8192, 64)
#undef CLB_COOPI
    default:
      return cudaErrorInvalidValue;
  }
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
