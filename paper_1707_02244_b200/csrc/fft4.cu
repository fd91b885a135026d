// Four-step FFT engine for the circulant products (the reference's default
// `use_fft=true` path, circulant.hpp:236-274), power-of-two 2^14 <= n <= 2^24.
//
// n = N1 * N2, natural index j = n1 * N2 + n2, spectral index k = k1 + N1 * k2.
// One product y = idft(H . dft(u)) is three kernels and three passes over n
// complex values (the Stockham engine of fft.cu needs ~4 log16(n) passes plus
// the pointwise ones):
//   cols_fwd : per column n2, DIF FFT over n1 (in shared memory) -> T[p][n2],
//              p = a digit-reversed k1 (no reordering: convolution does not
//              care about the spectral order as long as H uses the same one);
//              the input is real (x, v, beta, or P^T r kept dense).
//   rows     : per row p, twiddle w_n^{n2 k1}, DIF FFT over n2, multiply by
//              H~[p][q] (H permuted to the same order), DIT inverse FFT over
//              n2 (natural order again), twiddle w_n^{-n2 k1}; in place.
//   cols_inv : per column, DIT inverse FFT over p -> natural n1, real part
//              times 1/n, written as the product (or gathered at the rows).
// DIF forward + DIT inverse = no bit reversal anywhere.  Every stage is an
// in-place radix-16 (then 8/4/2) butterfly on shared memory with a twiddle
// table; global loads and stores are coalesced row segments.
//
// Real plans (the default): the product's input and output are real, so the
// engine transforms the length-N = n/2 complex sequence z[j] = u[2j] + i u[2j+1]
// (half the bytes of every pass).  The rows kernel holds each row together with
// its mirror row (the row of the spectral indices N - k) and, between the
// forward and the inverse row FFTs, turns Z into the real spectrum U, multiplies
// by H and packs Y back into the spectrum of y[2j] + i y[2j+1]:
//   U[k] = E + W^k O, U[k+N] = E - W^k O,  E = (Z[k] + Z*[N-k]) / 2,  O = (Z[k] - Z*[N-k]) / 2i
//   Z'[k] = (Y[k] + Y[k+N]) / 2 + i W^-k (Y[k] - Y[k+N]) / 2,   W = e^{-2 pi i / n},
// with H[k+N] = conj(H[N-k]) (h real): the engine stores H[k] for k < N only,
// and H[0], H[N] (both real) packed into entry 0.
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cmath>
#include <vector>

#include "fft4.cuh"
#include "kernels.cuh"

namespace clb {
namespace {

constexpr int kThr = 256;
constexpr int kElems = 4096;  // complex values per CTA (32 KB of shared memory + padding)

__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulf_conj(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

__device__ constexpr float kC16[16] = {1.0f, 0.92387953251128674f, 0.70710678118654757f, 0.38268343236508978f, 0.0f,
                                       -0.38268343236508978f, -0.70710678118654757f, -0.92387953251128674f, -1.0f,
                                       -0.92387953251128674f, -0.70710678118654757f, -0.38268343236508978f, -0.0f,
                                       0.38268343236508978f, 0.70710678118654757f, 0.92387953251128674f};
__device__ constexpr float kS16[16] = {0.0f, 0.38268343236508978f, 0.70710678118654757f, 0.92387953251128674f, 1.0f,
                                       0.92387953251128674f, 0.70710678118654757f, 0.38268343236508978f, 0.0f,
                                       -0.38268343236508978f, -0.70710678118654757f, -0.92387953251128674f, -1.0f,
                                       -0.92387953251128674f, -0.70710678118654757f, -0.38268343236508978f};

// Radix-R DFT in registers, natural order in and out, sign SG.
template <int R, int SG>
__device__ __forceinline__ void dftr(float2 (&v)[R]) {
  float2 t[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    int r = 0;
#pragma unroll
    for (int b = 1, j = i; b < R; b <<= 1, j >>= 1) r = (r << 1) | (j & 1);
    t[r] = v[i];
  }
#pragma unroll
  for (int half = 1; half < R; half <<= 1) {
#pragma unroll
    for (int base = 0; base < R; base += 2 * half) {
#pragma unroll
      for (int k = 0; k < half; ++k) {
        const int e = k * (16 / (2 * half));
        const float2 u = t[base + k], bb = t[base + k + half];
        // w = e^{SG 2 pi i e / 16}; the trivial factors (e = 0: 1, e = 4: SG i) as moves and negations
        // (e is a constant after unrolling, so the branches fold)
        const float2 x = e == 0 ? bb
                         : e == 4 ? make_float2(-SG * bb.y, SG * bb.x)
                                  : cmulf(bb, make_float2(kC16[e], SG * kS16[e]));
        t[base + k] = make_float2(u.x + x.x, u.y + x.y);
        t[base + k + half] = make_float2(u.x - x.x, u.y - x.y);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = t[i];
}

// Shared-memory layout: element i of sequence s at buf[s * sstride + pad(i)],
// one complex of padding every 16 (the last DIF / first DIT stage reads 16
// consecutive elements per thread; unpadded, all lanes would hit one bank).
__host__ __device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }
// Radix schedule of a length-N transform: the remainder radix 2^(log2 N mod 4) first
// (a large stride, conflict-free), then radix 16 down to the last stage.
template <int N, int L>
struct Radix {
  static constexpr int value = (L == N && (ilog2(N) % 4) != 0) ? (1 << (ilog2(N) % 4)) : 16;
};

// One in-place stage on nseq sequences of length N in shared memory; sub-length L = R * M.
//   DIF (SG = -1): V = DFT_R(v_r at j + rM); V_q *= w_L^{jq}; store at j + qM.
//   DIT (SG = +1): v_q = x(j + qM) * w_L^{-jq}; V = IDFT_R(v); store V_r at j + rM.
// tw[k] = e^{-2 pi i k / N}.
template <int N, int L, int SG, int NSEQ, int NT = kThr>
__device__ __forceinline__ void stage(float2* buf, int sstride, const float2* __restrict__ tw) {
  constexpr int R = Radix<N, L>::value;
  constexpr int M = L / R;
  constexpr int per_seq = N / R;
  constexpr int total = NSEQ * per_seq;
  constexpr int twstep = N / L;
  for (int idx = threadIdx.x; idx < total; idx += NT) {
    const int s = idx / per_seq, rem = idx - s * per_seq;
    const int blk = rem / M, j = rem - blk * M;
    float2* p = buf + s * sstride;
    const int i0 = blk * L + j;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = p[pad16(i0 + r * M)];
    if (SG < 0) {
      dftr<R, -1>(v);
      if (M > 1) {
#pragma unroll
        for (int q = 1; q < R; ++q) v[q] = cmulf(v[q], __ldg(tw + j * q * twstep));
      }
    } else {
      if (M > 1) {
#pragma unroll
        for (int q = 1; q < R; ++q) v[q] = cmulf_conj(v[q], __ldg(tw + j * q * twstep));
      }
      dftr<R, +1>(v);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) p[pad16(i0 + r * M)] = v[r];
  }
}

// Forward DIF over all stages (natural in, digit-reversed out).
template <int N, int L, int NSEQ, int NT = kThr>
__device__ __forceinline__ void dif_from(float2* buf, int sstride, const float2* tw) {
  stage<N, L, -1, NSEQ, NT>(buf, sstride, tw);
  __syncthreads();
  constexpr int next = L / Radix<N, L>::value;
  if constexpr (next > 1) dif_from<N, next, NSEQ, NT>(buf, sstride, tw);
}
// Inverse DIT: the DIF stages undone in reverse order (digit-reversed in, natural out; scale N).
template <int N, int L, int NSEQ, int NT = kThr>
__device__ __forceinline__ void dit_from(float2* buf, int sstride, const float2* tw) {
  constexpr int next = L / Radix<N, L>::value;
  if constexpr (next > 1) dit_from<N, next, NSEQ, NT>(buf, sstride, tw);
  stage<N, L, +1, NSEQ, NT>(buf, sstride, tw);
  __syncthreads();
}

// position p of a DIF output of length N holds frequency rev(p) (same radix schedule)
__host__ __device__ __forceinline__ int digit_rev(int p, int N) {
  int k = 0, mult = 1, lg = 0;
  while ((1 << lg) < N) ++lg;
  for (int L = N; L > 1;) {
    const int R = (L == N && (lg % 4) != 0) ? (1 << (lg % 4)) : 16;
    L /= R;
    const int q = p / L;
    p -= q * L;
    k += q * mult;
    mult *= R;
  }
  return k;
}

// inverse of digit_rev: the DIF output position holding frequency k
__host__ __device__ __forceinline__ int digit_pos(int k, int N) {
  int lg = 0;
  while ((1 << lg) < N) ++lg;
  int p = 0;
  for (int L = N; L > 1;) {
    const int R = (L == N && (lg % 4) != 0) ? (1 << (lg % 4)) : 16;
    L /= R;
    p += (k % R) * L;
    k /= R;
  }
  return p;
}

// ---- kernels -----------------------------------------------------------------
// Columns per CTA and the column pitch: pitch = (16 / B) mod 16 (complex) keeps
// the coalesced row-segment loads (B columns x 4 rows per half-warp) conflict-free.
// 2048-long columns (two-level plans at N >= 2^22): 8 columns = 64-byte row segments, 139 KB of shared memory
__host__ __device__ constexpr int cols_per_cta(int N1) { return N1 <= 1024 ? kElems / N1 : N1 == 2048 ? 8 : 4; }
// FINE (L2-resident sizes): half the columns / row units per CTA -- twice the CTAs in flight for the
// latency-bound passes -- and 512 threads per CTA (half the serial work per thread in every stage)
constexpr int kThrFine = 512;
// FINE = 1: the halved tiles at 256 threads; FINE = 2: the halved tiles at 512 threads
__host__ __device__ constexpr int threads_of(int fine) { return fine == 2 ? kThrFine : kThr; }
__host__ __device__ constexpr int cols_b(int N1, int fine) {
  return fine && cols_per_cta(N1) > 1 ? cols_per_cta(N1) / 2 : cols_per_cta(N1);
}
__host__ __device__ constexpr int col_pitch_b(int N1, int B) { return N1 + N1 / 16 + (B <= 16 ? 16 / B : 1); }
__host__ __device__ constexpr int col_pitch(int N1) { return col_pitch_b(N1, cols_per_cta(N1)); }
__host__ __device__ constexpr int row_count(int N2) { return N2 >= kElems ? 1 : kElems / N2; }
__host__ __device__ constexpr int row_pitch(int N2) { return N2 + N2 / 16 + 1; }

// w_n^idx = e^{-2 pi i idx / n} = twB[idx >> 12] * twA[idx & 4095]
__device__ __forceinline__ float2 tw_n(const float2* __restrict__ twA, const float2* __restrict__ twB, int idx) {
  return cmulf(__ldg(twB + (idx >> 12)), __ldg(twA + (idx & 4095)));
}
// the same e^{-2 pi i idx / N} (N = 2^lg, idx < N) computed in registers (sincospif, ~1 ulp): no load latency
__device__ __forceinline__ float2 tw_calc(int idx, int lg) {
  float s, c;
  sincospif(-ldexpf(static_cast<float>(idx), 1 - lg), &s, &c);
  return make_float2(c, s);
}

// Column-tile load (B consecutive elements of each of the N1 rows, stride N2) into shared memory: every
// global load of the thread is issued before its first shared store, so a tile costs one memory latency
// instead of a batch plus a serialized tail (ncu at 2^24: the tail loads held 12% of k_mid's stall samples,
// and the load->store pairs ~25% of k_cols_inv_fwd's).  ld(j) returns element j of the row-major input.
template <int N1, int B, int P, int NT, class Ld>
__device__ __forceinline__ void tile_in(float2* sm, int c0, int N2, Ld ld) {
  constexpr int cnt = B * N1;
  if constexpr (cnt % NT == 0 && NT % B == 0 && cnt / NT <= 16) {
    constexpr int per = cnt / NT, rstep = NT / B;
    const int w = threadIdx.x % B, i0 = threadIdx.x / B;
    const int64_t j0 = static_cast<int64_t>(i0) * N2 + c0 + w, js = static_cast<int64_t>(rstep) * N2;
    float2 v[per];
#pragma unroll
    for (int k = 0; k < per; ++k) v[k] = ld(j0 + k * js);
#pragma unroll
    for (int k = 0; k < per; ++k) sm[w * P + pad16(i0 + k * rstep)] = v[k];
  } else {
#pragma unroll
    for (int e = threadIdx.x; e < cnt; e += NT) {
      const int i = e / B, w = e - i * B;
      sm[w * P + pad16(i)] = ld(static_cast<int64_t>(i) * N2 + c0 + w);
    }
  }
}

// Columns forward: input real u[j] (j = n1 N2 + n2).
// REAL: the input is read as N complex values z[j] = (u[2j], u[2j+1]) (the real plans); else as the real
// parts of n complex values.
template <int N1, bool REAL, int FINE = 0>
__global__ void __launch_bounds__(threads_of(FINE), N1 <= 256 ? 4 : 1) k_cols_fwd(const float* __restrict__ u, float2* __restrict__ T, int N2,
                                                   const float2* __restrict__ tw1) {
  extern __shared__ float2 sm[];
  constexpr int B = cols_b(N1, FINE), P = col_pitch_b(N1, B), cnt = B * N1;
  const int c0 = blockIdx.x * B;
  tile_in<N1, B, P, threads_of(FINE)>(sm, c0, N2, [u](int64_t j) {
    return REAL ? __ldg(reinterpret_cast<const float2*>(u) + j) : make_float2(__ldg(u + j), 0.f);
  });
  __syncthreads();
  dif_from<N1, N1, B, threads_of(FINE)>(sm, P, tw1);
#pragma unroll
  for (int e = threadIdx.x; e < cnt; e += threads_of(FINE)) {
    const int i = e / B, w = e - i * B;
    T[static_cast<int64_t>(i) * N2 + c0 + w] = sm[w * P + pad16(i)];
  }
}

// Rows: row_count(N2) rows per CTA, in place on T.
// Row r's twiddle is w_n^{mult * n2 * digit_rev(r mod rowmod, rowmod)}: the four-step twiddle
// w_n^{n2 k1} (rowmod = N1, mult = 1), or, for the inner four-step of a three-level plan,
// w_{N2}^{n3 k2a} = w_n^{N1 n3 k2a} (rowmod = A, mult = N1).
template <int N2>
__global__ void __launch_bounds__(kThr, N2 <= 256 ? 4 : 1)
k_rows(float2* __restrict__ T, const float2* __restrict__ H, int conj_h, int rowmod, int mult,
       const float2* __restrict__ tw2, const float2* __restrict__ twA, const float2* __restrict__ twB) {
  extern __shared__ float2 sm[];
  constexpr int rows = row_count(N2), P = row_pitch(N2), cnt = rows * N2;
  constexpr int per = (cnt + kThr - 1) / kThr;
  // Short rows (the three-level plan's contiguous B-point rows): a register-lean form -- the twiddle is
  // recomputed for the store and the spectrum fetched after the forward stages -- so four CTAs fit per SM
  // and their load / compute / store phases overlap.  Longer rows keep both in registers across the stages.
  constexpr bool kLean = N2 <= 256;
  __shared__ int k1s[rows];
  const int p0 = blockIdx.x * rows;
  if (threadIdx.x < rows) k1s[threadIdx.x] = mult * digit_rev((p0 + threadIdx.x) % rowmod, rowmod);
  __syncthreads();
  float2 tw[kLean ? 1 : per];  // w_n^{n2 k1} of this thread's elements (reused for the inverse twiddle)
#pragma unroll
  for (int k = 0; k < per; ++k) {
    const int e = threadIdx.x + k * kThr;
    if (e < cnt) {
      const int rr = e / N2, n2 = e - rr * N2;
      const float2 w = tw_n(twA, twB, n2 * k1s[rr]);
      if constexpr (!kLean) tw[k] = w;
      sm[rr * P + pad16(n2)] = cmulf(T[static_cast<int64_t>(p0) * N2 + e], w);
    }
  }
  // long rows: the spectrum is fetched before the forward stages (its latency hides behind them)
  float2 hv[kLean ? 1 : per];
  if constexpr (!kLean) {
#pragma unroll
    for (int k = 0; k < per; ++k) {
      const int e = threadIdx.x + k * kThr;
      if (e < cnt) hv[k] = __ldg(H + static_cast<int64_t>(p0) * N2 + e);
    }
  }
  __syncthreads();
  dif_from<N2, N2, rows>(sm, P, tw2);
#pragma unroll
  for (int k = 0; k < per; ++k) {
    const int e = threadIdx.x + k * kThr;
    if (e < cnt) {
      const int rr = e / N2, q = e - rr * N2;
      const float2 h = kLean ? __ldg(H + static_cast<int64_t>(p0) * N2 + e) : hv[kLean ? 0 : k];
      float2& a = sm[rr * P + pad16(q)];
      a = conj_h ? cmulf_conj(a, h) : cmulf(a, h);
    }
  }
  __syncthreads();
  dit_from<N2, N2, rows>(sm, P, tw2);
#pragma unroll
  for (int k = 0; k < per; ++k) {
    const int e = threadIdx.x + k * kThr;
    if (e < cnt) {
      const int rr = e / N2, n2 = e - rr * N2;
      const float2 w = kLean ? tw_n(twA, twB, n2 * k1s[rr]) : tw[kLean ? 0 : k];
      T[static_cast<int64_t>(p0) * N2 + e] = cmulf_conj(sm[rr * P + pad16(n2)], w);
    }
  }
}


// Real plans: the rows kernel on row pairs.  Position q of row R holds the spectral index
// k = kb + kmul digit_rev(q, N2), kb = digit_rev(R / A, N1) + N1 digit_rev(R mod A, A) (A = 1 for two-level
// plans), kmul = N1 A; the mirror indices N - k all lie in the row of kb' = (kmul - kb) mod kmul.  Unit
// u in [0, kmul / 2] is the row pair (kb = u, kb' = kmul - u); kb = 0 and kmul / 2 are their own mirrors.
// The four-step twiddle of row R is w^{mult n2 digit_rev(R mod rowmod, rowmod)}, as in k_rows.  H holds
// H[k] (k < N) in the same positions, entry k = 0 = (H[0], H[N]).
__host__ __device__ constexpr int units_per_cta(int N2, int fine = 0) {
  return N2 >= 2048 ? 1 : fine && N2 == 1024 ? 1 : (fine ? 1024 : 2048) / N2;
}

// Z'[k] from Z[k], Z[N-k] (zk, zb), H[k], H[k+N] and W^k; the factor 1/4 is folded into the inverse scale.
__device__ __forceinline__ float2 r2c_mul(float2 zk, float2 zb, float2 hk, float2 hkn, float2 w) {
  const float2 e = make_float2(zk.x + zb.x, zk.y - zb.y);  // 2 E
  const float2 d = make_float2(zk.x - zb.x, zk.y + zb.y);  // Z[k] - conj(Z[N-k])
  const float2 o = make_float2(d.y, -d.x);                 // 2 O = d / i
  const float2 wo = cmulf(w, o);
  const float2 yk = cmulf(hk, make_float2(e.x + wo.x, e.y + wo.y));    // 2 Y[k]
  const float2 ykn = cmulf(hkn, make_float2(e.x - wo.x, e.y - wo.y));  // 2 Y[k+N]
  const float2 dd = cmulf_conj(make_float2(yk.x - ykn.x, yk.y - ykn.y), w);  // W^-k (Y[k] - Y[k+N])
  return make_float2(yk.x + ykn.x - dd.y, yk.y + ykn.y + dd.x);          // 4 Z'[k]
}

// H2[u N2 + q] = (H at (row of kb = u, q), H at the mirror position): one 16-byte load per index pair.
// t2[q] = W^{kmul digit_rev(q)}, so W^k = W^{kb} t2[q]; W^{N-k} = -conj(W^k).
template <int N2, int FINE = 0>
__global__ void __launch_bounds__(threads_of(FINE), N2 <= 256 ? 4 : 1)
k_rows_r2c(float2* __restrict__ T, const float4* __restrict__ H2, int conj_h, int N1, int A, int rowmod, int mult,
           const float2* __restrict__ tw2, const float2* __restrict__ twA, const float2* __restrict__ twB,
           const float2* __restrict__ twCA, const float2* __restrict__ twCB, const float2* __restrict__ t2) {
  extern __shared__ float2 sm[];
  constexpr int upc = units_per_cta(N2, FINE), slots = 2 * upc, P = row_pitch(N2), cnt = slots * N2;
  const int kmul = N1 * A;
  const int lgN = 31 - __clz(kmul * N2);
  // the four-step twiddle w^{n2 k1} of slot s.  Rows of 256+ points: two per-slot shared tables, n2 = h LO + l,
  // w^{h LO k1} w^{l k1} (slots x (LO + HI) sincospif per CTA instead of two per element, no load latency:
  // ISTA 2^20 0.079 vs 0.083 ms, cADMM 2^22 0.283 vs 0.288).  The three-level plans' 64/128-point rows:
  // sincospif per element (the tables' build and barrier in front of the loads lost: 2^24 0.983 vs 0.961).
  // Up to 16 elements per thread: the tables are built while the row loads are in flight (the loads go to
  // registers first, the table build follows, then the twiddled stores).
  constexpr bool kLate = cnt / threads_of(FINE) <= 16 && cnt % threads_of(FINE) == 0;
  constexpr int LO = 1 << ((ilog2(N2) + 1) / 2), HI = N2 / LO;
  __shared__ float2 tw_lo[slots][LO], tw_hi[slots][HI];
  __shared__ int rows_s[slots], k1s[slots], kbs[slots];
  __shared__ float2 wrow[upc];
  const auto twiddle = [&](int s, int n2) { return cmulf(tw_hi[s][n2 / LO], tw_lo[s][n2 % LO]); };
  const auto build_tables = [&] {
    for (int e = threadIdx.x; e < slots * (LO + HI); e += threads_of(FINE)) {
      const int s = e / (LO + HI), j = e - s * (LO + HI);
      if (j < LO) tw_lo[s][j] = tw_calc(j * k1s[s], lgN);  // j k1 < N (n2 k1 < N for every plan)
      else tw_hi[s][j - LO] = tw_calc((j - LO) * LO * k1s[s], lgN);
    }
  };
  if (threadIdx.x < slots) {
    const int u = blockIdx.x * upc + (threadIdx.x >> 1);
    const int kb = (threadIdx.x & 1) ? (kmul - u) & (kmul - 1) : u;
    const bool live = u <= kmul / 2 && !((threadIdx.x & 1) && kb == u);  // the mirror slot of a self unit idles
    const int R = live ? digit_pos(kb % N1, N1) * A + digit_pos(kb / N1, A) : -1;
    rows_s[threadIdx.x] = R;
    k1s[threadIdx.x] = R >= 0 ? mult * digit_rev(R % rowmod, rowmod) : 0;
    kbs[threadIdx.x] = kb;
    if (!(threadIdx.x & 1)) wrow[threadIdx.x >> 1] = tw_n(twCA, twCB, kb);  // W^{kb}
  }
  {  // L2 prefetch of this CTA's spectrum pairs (contiguous, units [u0, u0 + upc) within [0, kmul / 2]): the
     // spectral step's loads then hit L2 instead of serializing DRAM latency per loop trip
    const int u0 = blockIdx.x * upc, units = min(upc, kmul / 2 + 1 - u0);
    const float4* hb = H2 + static_cast<int64_t>(u0) * N2;
    for (int l = threadIdx.x; l < units * N2 / 8; l += threads_of(FINE))  // 8 float4 per 128-byte line
      asm volatile("prefetch.global.L2 [%0];" ::"l"(hb + 8 * l));
  }
  __syncthreads();
  if constexpr (kLate) {
    constexpr int per = cnt / threads_of(FINE);
    static_assert(cnt % threads_of(FINE) == 0, "whole rows per thread pass");
    float2 v[per];
#pragma unroll
    for (int k = 0; k < per; ++k) {
      const int e = threadIdx.x + k * threads_of(FINE), s = e / N2, n2 = e - s * N2, R = rows_s[s];
      v[k] = R >= 0 ? T[static_cast<int64_t>(R) * N2 + n2] : make_float2(0.f, 0.f);
    }
    build_tables();
    __syncthreads();
#pragma unroll
    for (int k = 0; k < per; ++k) {
      const int e = threadIdx.x + k * threads_of(FINE), s = e / N2, n2 = e - s * N2;
      if (rows_s[s] >= 0) sm[s * P + pad16(n2)] = cmulf(v[k], twiddle(s, n2));
    }
  } else {
    build_tables();
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += threads_of(FINE)) {
      const int s = e / N2, n2 = e - s * N2, R = rows_s[s];
      if (R >= 0) sm[s * P + pad16(n2)] = cmulf(T[static_cast<int64_t>(R) * N2 + n2], twiddle(s, n2));
    }
  }
  __syncthreads();
  dif_from<N2, N2, slots, threads_of(FINE)>(sm, P, tw2);
  // spectral step: the thread of (slot 2u, q) handles k and its mirror N - k, at (2u + 1, qb) -- or at (2u, qb)
  // when the row is its own mirror (kb = 0 or kmul / 2), and then only q <= qb works.  Mirror position:
  // kb != 0: digit complement qb = N2 - 1 - q; kb = 0: the position of (N2 - k2) mod N2.
  for (int e = threadIdx.x; e < upc * N2; e += threads_of(FINE)) {
    const int ul = e / N2, q = e - ul * N2, sa = 2 * ul;
    if (rows_s[sa] < 0) continue;
    const bool self = rows_s[sa + 1] < 0;
    const int kbA = kbs[sa];
    const int qb = kbA != 0 ? N2 - 1 - q : digit_pos((N2 - digit_rev(q, N2)) & (N2 - 1), N2);
    if (self && qb < q) continue;
    const int sb = self ? sa : sa + 1;
    const float4 hh = __ldg(H2 + static_cast<int64_t>(blockIdx.x * upc + ul) * N2 + q);
    const float sgn = conj_h ? -1.f : 1.f;
    const float2 hk = make_float2(hh.x, sgn * hh.y), hb = make_float2(hh.z, sgn * hh.w);
    const float2 w = cmulf(wrow[ul], __ldg(t2 + q));  // W^k
    const float2 zk = sm[sa * P + pad16(q)];
    if (kbA == 0 && q == 0) {  // k = 0: H[0], H[N] real, packed (conj_h leaves them)
      sm[sa * P] = r2c_mul(zk, zk, make_float2(hh.x, 0.f), make_float2(hh.y, 0.f), w);
      continue;
    }
    const float2 zb = sm[sb * P + pad16(qb)];
    sm[sa * P + pad16(q)] = r2c_mul(zk, zb, hk, make_float2(hb.x, -hb.y), w);  // H[k+N] = conj H[N-k]
    if (qb != q || sb != sa)
      sm[sb * P + pad16(qb)] = r2c_mul(zb, zk, hb, make_float2(hk.x, -hk.y), make_float2(-w.x, w.y));
  }
  __syncthreads();
  dit_from<N2, N2, slots, threads_of(FINE)>(sm, P, tw2);
  for (int e = threadIdx.x; e < cnt; e += threads_of(FINE)) {
    const int s = e / N2, n2 = e - s * N2, R = rows_s[s];
    if (R >= 0)
      T[static_cast<int64_t>(R) * N2 + n2] = cmulf_conj(sm[s * P + pad16(n2)], twiddle(s, n2));
  }
}

// Three-level plans: the A-point transforms of the row length N2 = A * B, along the stride-B axis of each
// row p (element n2 = n2a B + n3), C = cols_per_cta(A) consecutive n3 per CTA (128-byte segments).
//   FWD: x w_n^{n2 k1} (the outer four-step twiddle, k1 = digit_rev(p)), DIF over n2a, in place;
//   INV: DIT over the digit-reversed axis back to natural n2a, x conj(w_n^{n2 k1}), in place.
template <int A, bool FWD>
__global__ void __launch_bounds__(kThr, 4) k_mid(float2* __restrict__ T, int N1, int N2, int B,
                                              const float2* __restrict__ twM, const float2* __restrict__ twA,
                                              const float2* __restrict__ twB) {
  extern __shared__ float2 sm[];
  constexpr int C = cols_per_cta(A), P = col_pitch(A), cnt = C * A;
  const int per_row = B / C;
  const int p = blockIdx.x / per_row, n30 = (blockIdx.x - p * per_row) * C;
  const int k1 = digit_rev(p, N1);
  const int lgN = 31 - __clz(N1 * N2);
  float2* row = T + static_cast<int64_t>(p) * N2;
  // the four-step twiddle w^{n2 k1} in registers: a thread's elements step n2 by (kThr / C) B, so after one
  // sincospif for its first element each next twiddle is one complex multiply by the step's (~1e-7 relative
  // after the 15 steps, against two table loads or one sincospif per element)
  static_assert(kThr % C == 0, "a thread keeps its column");
  const int n2_0 = (threadIdx.x / C) * B + n30 + threadIdx.x % C;
  const int64_t step = static_cast<int64_t>(kThr / C) * B * k1 % (static_cast<int64_t>(N1) * N2);
  const float2 w_step = tw_calc(static_cast<int>(step), lgN);
  float2 w_e = tw_calc(n2_0 * k1, lgN);
  {  // all loads first (see tile_in), then the twiddle progression and the stores in the same order
    constexpr int per = cnt / kThr, rstep = kThr / C;
    static_assert(cnt % kThr == 0 && per <= 16, "one register batch per thread");
    const int w = threadIdx.x % C, i0 = threadIdx.x / C;
    float2 v[per];
#pragma unroll
    for (int k = 0; k < per; ++k) v[k] = row[(i0 + k * rstep) * B + n30 + w];
#pragma unroll
    for (int k = 0; k < per; ++k) {
      sm[w * P + pad16(i0 + k * rstep)] = FWD ? cmulf(v[k], w_e) : v[k];
      if (FWD) w_e = cmulf(w_e, w_step);
    }
  }
  __syncthreads();
  if constexpr (FWD) dif_from<A, A, C>(sm, P, twM);
  else dit_from<A, A, C>(sm, P, twM);
#pragma unroll
  for (int e = threadIdx.x; e < cnt; e += kThr) {
    const int i = e / C, w = e - i * C, n2 = i * B + n30 + w;
    const float2 v = sm[w * P + pad16(i)];
    row[n2] = FWD ? v : cmulf_conj(v, w_e);
    if (!FWD) w_e = cmulf(w_e, w_step);
  }
}

// Columns inverse, with the consumer of the product fused into the write-out:
//   Fft4Out::kProduct  out[j] = Re / n
//   Fft4Out::kRows     out[rowid[j]] = Re / n at the rows
//   Fft4Out::kResidual r[t] = y[t] - Re / n and u[j] = r[t] at the rows (P^T r kept dense)
//   Fft4Out::kIstaStep delta[j] = Re / n, x[j] = eta(x[j] + tau delta[j])  (unchecked iterations)
//   Fft4Out::kBeta     beta[j] = rho Re / n + sigma (z[j] - nu[j])
// Writes output j of the product (value v) as o.mode says; returns the vector the mode produces at j (the
// next product's input when k_cols_inv_fwd chains two products): the product, beta, the new x, or P^T r.
__device__ __forceinline__ float emit_out(const Fft4Out& o, int64_t j, float v) {
  if (j >= o.n_valid) return 0.f;  // the padded engine's convolution tail: zero input
  if (o.mode == Fft4Out::kProduct) {
    o.out[j] = v;
    return v;
  } else if (o.mode == Fft4Out::kBeta) {  // parallel.hpp:186-187
    const float b = __fadd_rn(__fmul_rn(o.rho, v), __fmul_rn(o.sigma, __fsub_rn(o.z[j], o.nu[j])));
    o.out[j] = b;
    return b;
  } else if (o.mode == Fft4Out::kIstaStep) {
    const float xo = o.x[j];
    const float xn = __fadd_rn(xo, __fmul_rn(o.tau, v));  // parallel.hpp:269-271
    const float xs = xn > o.thr ? xn - o.thr : (xn < -o.thr ? xn + o.thr : 0.f);
    o.x[j] = xs;
    o.out[j] = v;
    return xs;
  } else {
    const int t = __ldg(o.rowid + j);
    if (t >= 0) {
      if (o.mode == Fft4Out::kRows) {
        o.out[t] = v;
      } else {  // kResidual: cpista residual, parallel.hpp:252
        const float rv = __ldg(o.y + t) - v;
        o.out[t] = rv;
        o.u[j] = rv;
        return rv;
      }
    }
    return 0.f;
  }
}
// The consumer's inputs at output j (z and nu for beta, x for the ISTA update, the row t and y[t] for the
// residual), loaded ahead of any of the thread's stores: the batched emit loop below issues every load of a
// tile first (the stores through o's pointers would otherwise keep each later load behind them -- one or two
// dependent memory latencies per output; C3's inverse column passes were 16-22 us at 16% issue).
struct EmitIn {
  float a = 0.f, b = 0.f;
  int t = -1;
};
__device__ __forceinline__ void emit_load1(const Fft4Out& o, int64_t j, EmitIn& in) {
  if (j >= o.n_valid) return;
  if (o.mode == Fft4Out::kBeta) {
    in.a = o.z[j];
    in.b = o.nu[j];
  } else if (o.mode == Fft4Out::kIstaStep) {
    in.a = o.x[j];
  } else if (o.mode != Fft4Out::kProduct) {
    in.t = __ldg(o.rowid + j);
  }
}
__device__ __forceinline__ void emit_load2(const Fft4Out& o, EmitIn& in) {  // y[t] after the row ids landed
  if (o.mode == Fft4Out::kResidual && in.t >= 0) in.a = __ldg(o.y + in.t);
}
// emit_out with the inputs already loaded: the same arithmetic, bit for bit
__device__ __forceinline__ float emit_with(const Fft4Out& o, int64_t j, float v, const EmitIn& in) {
  if (j >= o.n_valid) return 0.f;
  if (o.mode == Fft4Out::kProduct) {
    o.out[j] = v;
    return v;
  } else if (o.mode == Fft4Out::kBeta) {  // parallel.hpp:186-187
    const float b = __fadd_rn(__fmul_rn(o.rho, v), __fmul_rn(o.sigma, __fsub_rn(in.a, in.b)));
    o.out[j] = b;
    return b;
  } else if (o.mode == Fft4Out::kIstaStep) {
    const float xn = __fadd_rn(in.a, __fmul_rn(o.tau, v));  // parallel.hpp:269-271
    const float xs = xn > o.thr ? xn - o.thr : (xn < -o.thr ? xn + o.thr : 0.f);
    o.x[j] = xs;
    o.out[j] = v;
    return xs;
  } else if (in.t >= 0) {
    if (o.mode == Fft4Out::kRows) {
      o.out[in.t] = v;
    } else {  // kResidual: cpista residual, parallel.hpp:252
      const float rv = in.a - v;
      o.out[in.t] = rv;
      o.u[j] = rv;
      return rv;
    }
  }
  return 0.f;
}
// The inverse passes' write-out of a B-column tile from shared memory through the consumer `o`; with CHAIN the
// values the consumer produces go back into the tile (the next product's input).  Batched as tile_in.
template <int N1, int B, int P, int NT, bool REAL, bool CHAIN>
__device__ __forceinline__ void emit_tile(float2* sm, const Fft4Out& o, int c0, int N2, float inv_n) {
  constexpr int cnt = B * N1;
  constexpr bool kBatch = cnt % NT == 0 && NT % B == 0 && cnt / NT <= 16;
  // chunks of CH elements per thread: the whole tile at <= 8 per thread; 4 at a time for the DRAM-resident
  // plans' 16 (their 64-register cap), where beta's z/nu (already L2-prefetched) measured faster unbatched
  // (cADMM 2^24 0.852 vs 0.860 ms) and the ISTA update batched (ISTA 2^24 0.486 vs 0.531 ms)
  if (kBatch && (cnt / NT <= 8 || o.mode != Fft4Out::kBeta)) {
    constexpr int per = kBatch ? cnt / NT : 1, rstep = NT / B, f = REAL ? 2 : 1, CH = per <= 8 ? per : 4;
    const int w = threadIdx.x % B, i0 = threadIdx.x / B;
#pragma unroll
    for (int k0 = 0; k0 < per; k0 += CH) {
      EmitIn in[CH][f];
#pragma unroll
      for (int k = 0; k < CH; ++k)
#pragma unroll
        for (int q = 0; q < f; ++q)
          emit_load1(o, (static_cast<int64_t>(i0 + (k0 + k) * rstep) * N2 + c0 + w) * f + q, in[k][q]);
#pragma unroll
      for (int k = 0; k < CH; ++k)
#pragma unroll
        for (int q = 0; q < f; ++q) emit_load2(o, in[k][q]);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int i = i0 + (k0 + k) * rstep;
        const int64_t j = static_cast<int64_t>(i) * N2 + c0 + w;
        float2& sv = sm[w * P + pad16(i)];
        if (REAL) {
          const float a = emit_with(o, 2 * j, sv.x * inv_n, in[k][0]);
          const float b = emit_with(o, 2 * j + 1, sv.y * inv_n, in[k][f - 1]);
          if (CHAIN) sv = make_float2(a, b);
        } else {
          const float a = emit_with(o, j, sv.x * inv_n, in[k][0]);
          if (CHAIN) sv = make_float2(a, 0.f);
        }
      }
    }
  } else {
#pragma unroll
    for (int e = threadIdx.x; e < cnt; e += NT) {
      const int i = e / B, w = e - i * B;
      const int64_t j = static_cast<int64_t>(i) * N2 + c0 + w;
      float2& sv = sm[w * P + pad16(i)];
      if (REAL) {
        const float a = emit_out(o, 2 * j, sv.x * inv_n), b = emit_out(o, 2 * j + 1, sv.y * inv_n);
        if (CHAIN) sv = make_float2(a, b);
      } else {
        const float a = emit_out(o, j, sv.x * inv_n);
        if (CHAIN) sv = make_float2(a, 0.f);
      }
    }
  }
}
// Before the inverse stages: L2 prefetch of the lines the consumer will read at this CTA's outputs (z and nu
// for beta, x for the ISTA update), so the emit loop's loads hit L2 instead of waiting on DRAM.  Row i of the
// tile covers outputs [(i N2 + c0) f, + B f) with f = 2 for real plans: B f floats, one or two 128-byte lines.
template <int B, bool REAL>
__device__ __forceinline__ void prefetch_consumer(const Fft4Out& o, int N1, int N2, int c0, int nthreads) {
  const float* a = o.mode == Fft4Out::kBeta ? o.z : o.mode == Fft4Out::kIstaStep ? o.x : nullptr;
  if (!a) return;
  const float* b = o.mode == Fft4Out::kBeta ? o.nu : nullptr;
  constexpr int f = REAL ? 2 : 1, lines = (B * f * 4 + 127) / 128;
  for (int e = threadIdx.x; e < N1 * lines; e += nthreads) {
    const int i = e / lines, l = e - i * lines;
    const int64_t j = (static_cast<int64_t>(i) * N2 + c0) * f + l * 32;
    if (j >= o.n_valid) continue;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a + j));
    if (b) asm volatile("prefetch.global.L2 [%0];" ::"l"(b + j));
  }
}
// REAL: element j of the inverse holds y[2j] + i y[2j+1]; else Re = y[j].
template <int N1, bool REAL, int FINE = 0>
__global__ void __launch_bounds__(threads_of(FINE), N1 <= 256 ? 4 : 1) k_cols_inv(const float2* __restrict__ T, Fft4Out o, int N2,
                                                   const float2* __restrict__ tw1, float inv_n) {
  extern __shared__ float2 sm[];
  constexpr int B = cols_b(N1, FINE), P = col_pitch_b(N1, B), cnt = B * N1;
  const int c0 = blockIdx.x * B;
  tile_in<N1, B, P, threads_of(FINE)>(sm, c0, N2, [T](int64_t j) { return T[j]; });
  __syncthreads();
  if (FINE == 0) prefetch_consumer<B, REAL>(o, N1, N2, c0, threads_of(FINE));  // DRAM-resident plans
  dit_from<N1, N1, B, threads_of(FINE)>(sm, P, tw1);
  emit_tile<N1, B, P, threads_of(FINE), REAL, false>(sm, o, c0, N2, inv_n);
}

// Two chained products: the inverse columns of the first with its consumer (`o`), then -- on the vector that
// consumer produced, still in shared memory -- the forward columns of the next product, in place on T.
// Every CTA owns whole columns, so the next product's column FFT needs nothing from other CTAs (ISTA: the
// residual's P^T r feeds the gradient; cADMM: beta feeds B beta, and x = B beta feeds C x).
template <int N1, bool REAL, int FINE = 0>
__global__ void __launch_bounds__(threads_of(FINE), N1 <= 256 ? 4 : 1) k_cols_inv_fwd(float2* __restrict__ T, Fft4Out o, int N2,
                                                       const float2* __restrict__ tw1, float inv_n) {
  extern __shared__ float2 sm[];
  constexpr int B = cols_b(N1, FINE), P = col_pitch_b(N1, B), cnt = B * N1;
  const int c0 = blockIdx.x * B;
  tile_in<N1, B, P, threads_of(FINE)>(sm, c0, N2, [T](int64_t j) { return T[j]; });
  __syncthreads();
  if (FINE == 0) prefetch_consumer<B, REAL>(o, N1, N2, c0, threads_of(FINE));  // DRAM-resident plans
  dit_from<N1, N1, B, threads_of(FINE)>(sm, P, tw1);
  emit_tile<N1, B, P, threads_of(FINE), REAL, true>(sm, o, c0, N2, inv_n);
  __syncthreads();
  dif_from<N1, N1, B, threads_of(FINE)>(sm, P, tw1);
#pragma unroll
  for (int e = threadIdx.x; e < cnt; e += threads_of(FINE)) {
    const int i = e / B, w = e - i * B;
    T[static_cast<int64_t>(i) * N2 + c0 + w] = sm[w * P + pad16(i)];
  }
}

// H~[p N2 + q] = spec[rev1(p) + N1 rev2(q)] / s  (fp64 spectrum -> permuted fp32); three levels (A > 0):
// q = q2a B + q3 holds k2 = rev_A(q2a) + A rev_B(q3)
// real: entry k = 0 holds (H[0], H[N]) (both real)
// Real plans: H2[u N2r + q] for units u in [0, kmul / 2] of row length N2r (see k_rows_r2c); entry k = 0
// holds (H[0], H[N]).
__global__ void k_perm_spectrum_pairs(const double2* __restrict__ spec, double s, float4* __restrict__ out, int N1,
                                      int A, int N2r) {
  const int kmul = N1 * A, N = kmul * N2r;
  const int64_t total = static_cast<int64_t>(kmul / 2 + 1) * N2r;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int u = static_cast<int>(e / N2r), q = static_cast<int>(e - static_cast<int64_t>(u) * N2r);
    const int k = u + kmul * digit_rev(q, N2r);
    const int kb = (N - k) & (N - 1);
    const double2 a = spec[k], b = spec[kb];
    out[e] = k == 0 ? make_float4(static_cast<float>(a.x / s), static_cast<float>(spec[N].x / s), 0.f, 0.f)
                    : make_float4(static_cast<float>(a.x / s), static_cast<float>(a.y / s),
                                  static_cast<float>(b.x / s), static_cast<float>(b.y / s));
  }
}
__global__ void k_perm_spectrum(const double2* __restrict__ spec, double s, float2* __restrict__ out, int N1, int N2,
                                int A, int B, int real) {
  const int64_t n = static_cast<int64_t>(N1) * N2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int p = static_cast<int>(e / N2), q = static_cast<int>(e - static_cast<int64_t>(p) * N2);
    const int64_t k2 = A > 0 ? digit_rev(q / B, A) + static_cast<int64_t>(A) * digit_rev(q % B, B) : digit_rev(q, N2);
    const int64_t k = digit_rev(p, N1) + static_cast<int64_t>(N1) * k2;
    const double2 v = spec[k];
    out[e] = (real && k == 0) ? make_float2(static_cast<float>(v.x / s), static_cast<float>(spec[n].x / s))
                              : make_float2(static_cast<float>(v.x / s), static_cast<float>(v.y / s));
  }
}

__global__ void k_scatter_real(const float* __restrict__ r, const int* __restrict__ omega, float* __restrict__ u,
                               int64_t m) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    u[omega[t]] = r[t];
}


// ---- one-CTA FFT-engine ISTA for small n -------------------------------------
// Config 1 (n = 4096) on the FFT engine: the whole iteration in one CTA's shared
// memory, all unchecked iterations in one launch.  A length-n DIF FFT, the
// spectral multiply in the DIF output order (H permuted to match), a DIT inverse
// FFT -- per product, twice per iteration (circulant.hpp:236-274):
//   r = y - P C x,   delta = C^T P^T r,   x = eta(x + tau delta).
template <int N>
__global__ void __launch_bounds__(kThr, 1)
k_small_fft_ista(const float2* __restrict__ Hp, const float2* __restrict__ tw, const int* __restrict__ omega,
                 const float* __restrict__ y, float* __restrict__ x, float* __restrict__ r, float* __restrict__ delta,
                 int m, float tau, float thr, int iters) {
  extern __shared__ float4 smem_f4[];
  float2* A = reinterpret_cast<float2*>(smem_f4);          // padded N complex
  float* xs = reinterpret_cast<float*>(A + pad16(N) + 4);  // N
  float* rs = xs + N;                                      // m (<= N)
  const float inv_n = 1.0f / static_cast<float>(N);
  for (int i = threadIdx.x; i < N; i += kThr) xs[i] = x[i];
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    // residual: A = x -> DIF -> * conj(H) -> DIT -> r = y - Re(A[omega]) / n
    for (int i = threadIdx.x; i < N; i += kThr) A[pad16(i)] = make_float2(xs[i], 0.f);
    __syncthreads();
    dif_from<N, N, 1>(A, 0, tw);
    for (int i = threadIdx.x; i < N; i += kThr) A[pad16(i)] = cmulf_conj(A[pad16(i)], __ldg(Hp + i));
    __syncthreads();
    dit_from<N, N, 1>(A, 0, tw);
    for (int t = threadIdx.x; t < m; t += kThr) rs[t] = __ldg(y + t) - A[pad16(__ldg(omega + t))].x * inv_n;
    __syncthreads();
    // gradient: A = P^T r -> DIF -> * H -> DIT -> delta = Re(A) / n; x update
    for (int i = threadIdx.x; i < N; i += kThr) A[pad16(i)] = make_float2(0.f, 0.f);
    __syncthreads();
    for (int t = threadIdx.x; t < m; t += kThr) A[pad16(__ldg(omega + t))] = make_float2(rs[t], 0.f);
    __syncthreads();
    dif_from<N, N, 1>(A, 0, tw);
    for (int i = threadIdx.x; i < N; i += kThr) A[pad16(i)] = cmulf(A[pad16(i)], __ldg(Hp + i));
    __syncthreads();
    dit_from<N, N, 1>(A, 0, tw);
    for (int i = threadIdx.x; i < N; i += kThr) {
      const float d = A[pad16(i)].x * inv_n;
      const float v = __fadd_rn(xs[i], __fmul_rn(tau, d));  // parallel.hpp:269-271
      xs[i] = v > thr ? v - thr : (v < -thr ? v + thr : 0.f);
      if (it == iters - 1) delta[i] = d;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < N; i += kThr) x[i] = xs[i];
  for (int t = threadIdx.x; t < m; t += kThr) r[t] = rs[t];
}

// One-CTA FFT-engine cADMM (config 2) in the same style (cpadmm_phases, parallel.hpp:173-231):
//   beta = rho C^T v + sigma (z - nu);  x = B beta;  cx = C x;  the D/z/mu/nu/v updates.
template <int N>
__global__ void __launch_bounds__(kThr, 1)
k_small_fft_cadmm(const float2* __restrict__ Hc, const float2* __restrict__ Hb, const float2* __restrict__ tw,
                  const float* __restrict__ d, const float* __restrict__ pty, float* __restrict__ xg,
                  float* __restrict__ zg, float* __restrict__ nug, float* __restrict__ mug, float* __restrict__ vg,
                  float* __restrict__ betag, float rho, float sigma, float tau1, float tau2, float thr, int iters) {
  extern __shared__ float4 smem_f4[];
  float2* A = reinterpret_cast<float2*>(smem_f4);
  float* xs = reinterpret_cast<float*>(A + pad16(N) + 4);
  float* zs = xs + N;
  float* nus = zs + N;
  float* mus = nus + N;
  float* vs = mus + N;
  const float inv_n = 1.0f / static_cast<float>(N);
  for (int i = threadIdx.x; i < N; i += kThr) {
    xs[i] = xg[i];
    zs[i] = zg[i];
    nus[i] = nug[i];
    mus[i] = mug[i];
    vs[i] = vg[i];
  }
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    const bool last = it == iters - 1;
    // beta = rho C^T v + sigma (z - nu)
    for (int i = threadIdx.x; i < N; i += kThr) A[pad16(i)] = make_float2(vs[i], 0.f);
    __syncthreads();
    dif_from<N, N, 1>(A, 0, tw);
    for (int i = threadIdx.x; i < N; i += kThr) A[pad16(i)] = cmulf(A[pad16(i)], __ldg(Hc + i));
    __syncthreads();
    dit_from<N, N, 1>(A, 0, tw);
    for (int i = threadIdx.x; i < N; i += kThr) {
      const float sct = A[pad16(i)].x * inv_n;
      const float b = __fadd_rn(__fmul_rn(rho, sct), __fmul_rn(sigma, __fsub_rn(zs[i], nus[i])));
      A[pad16(i)] = make_float2(b, 0.f);
      if (last) betag[i] = b;
    }
    __syncthreads();
    // x = B beta
    dif_from<N, N, 1>(A, 0, tw);
    for (int i = threadIdx.x; i < N; i += kThr) A[pad16(i)] = cmulf_conj(A[pad16(i)], __ldg(Hb + i));
    __syncthreads();
    dit_from<N, N, 1>(A, 0, tw);
    for (int i = threadIdx.x; i < N; i += kThr) {
      const float xv = A[pad16(i)].x * inv_n;
      xs[i] = xv;
      A[pad16(i)] = make_float2(xv, 0.f);
    }
    __syncthreads();
    // cx = C x; duals
    dif_from<N, N, 1>(A, 0, tw);
    for (int i = threadIdx.x; i < N; i += kThr) A[pad16(i)] = cmulf_conj(A[pad16(i)], __ldg(Hc + i));
    __syncthreads();
    dit_from<N, N, 1>(A, 0, tw);
    for (int i = threadIdx.x; i < N; i += kThr) {
      const float cx = A[pad16(i)].x * inv_n;
      const float xi = xs[i], nui = nus[i];
      const float vn = __fmul_rn(__ldg(d + i), __fadd_rn(__fmul_rn(rho, __fsub_rn(cx, mus[i])), __ldg(pty + i)));
      const float sv = __fadd_rn(xi, nui);
      const float zn = sv > thr ? sv - thr : (sv < -thr ? sv + thr : 0.f);
      const float mun = __fadd_rn(mus[i], __fmul_rn(tau1, __fsub_rn(vn, cx)));
      zs[i] = zn;
      mus[i] = mun;
      nus[i] = __fadd_rn(nui, __fmul_rn(tau2, __fsub_rn(xi, zn)));
      vs[i] = __fadd_rn(vn, mun);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < N; i += kThr) {
    xg[i] = xs[i];
    zg[i] = zs[i];
    nug[i] = nus[i];
    mug[i] = mus[i];
    vg[i] = vs[i];
  }
}
template <int N>
size_t small_fft_cadmm_smem() { return (static_cast<size_t>(pad16(N) + 4) * 2 + 5 * N) * sizeof(float); }

// Hp[p] = H[digit_rev(p, N)] (fp32 natural-order spectrum -> the DIF output order)
__global__ void k_perm_small(const float2* __restrict__ H, float2* __restrict__ Hp, int N) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) Hp[p] = H[digit_rev(p, N)];
}

template <int N>
size_t small_fft_smem() { return (static_cast<size_t>(pad16(N) + 4) * 2 + 2 * N) * sizeof(float); }

}  // namespace

// the three-level plan from n = 2^22 up (arrays no longer L2-resident); CLB_FFT_TWO_LEVEL=1 forces two
constexpr int kThreeLevelLog = 22;

bool fft4_supported(int64_t n) { return n >= (int64_t(1) << 14) && n <= (int64_t(1) << 24) && (n & (n - 1)) == 0; }

// Real plans for n >= 2^18 (half the bytes per pass; cADMM per iteration at 2^24 / 2^22 / 2^20: 1.10 / 0.33 /
// 0.119 ms against 1.82 / 0.48 / 0.174 for the complex plans; ISTA at 2^18 / 2^19: 0.075 vs 0.085 ms); below,
// the complex plans' finer row split keeps more CTAs in flight (2^17: 0.097 vs 0.134 ms).  CLB_FFT_C2C=0/1
// forces either.
Fft4Plan fft4_plan(int64_t n) {
  Fft4Plan p;
  p.n = n;
  int Ln = 0;
  while ((int64_t(1) << Ln) < n) ++Ln;
  const char* c2c = std::getenv("CLB_FFT_C2C");
  p.real = (c2c && *c2c) ? c2c[0] == '0' : Ln >= 18;
  p.N = p.real ? n / 2 : n;
  int L = 0;
  while ((int64_t(1) << L) < p.N) ++L;
  // three levels from n = 2^22 (N1 = 256 columns: 128-byte row segments in every pass)
  if (Ln >= kThreeLevelLog && !std::getenv("CLB_FFT_TWO_LEVEL")) {  // 256 x A x B, A in {128, 256}
    p.N1 = 256;
    p.N2 = static_cast<int>(p.N >> 8);
    p.A = p.N2 >= (1 << 15) ? 256 : 128;
    p.B = p.N2 / p.A;
    return p;
  }
  int l1 = L / 2;
  if (l1 > 11) l1 = 11;
  p.N1 = 1 << l1;
  p.N2 = static_cast<int>(p.N >> l1);
  return p;
}

void fft4_twiddles(const Fft4Plan& p, std::vector<float2>* tw1, std::vector<float2>* tw2, std::vector<float2>* twA,
                   std::vector<float2>* twB) {
  auto table = [](std::vector<float2>& t, int count, double step) {
    t.resize(static_cast<size_t>(count));
    for (int k = 0; k < count; ++k) {
      const double a = -2.0 * M_PI * k * step;
      t[static_cast<size_t>(k)] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
    }
  };
  table(*tw1, p.N1, 1.0 / p.N1);
  if (p.three()) {  // the A-point table, then the B-point table
    std::vector<float2> ta, tb;
    table(ta, p.A, 1.0 / p.A);
    table(tb, p.B, 1.0 / p.B);
    tw2->assign(ta.begin(), ta.end());
    tw2->insert(tw2->end(), tb.begin(), tb.end());
  } else {
    table(*tw2, p.N2, 1.0 / p.N2);
  }
  const double NN = static_cast<double>(p.N);
  table(*twA, 4096, 1.0 / NN);                                              // e^{-2 pi i a / N}
  table(*twB, static_cast<int>(std::max<int64_t>(1, p.N / 4096)), 4096.0 / NN);  // e^{-2 pi i 4096 b / N}
  if (p.real) {  // W^k = e^{-2 pi i k / n} for the real-spectrum unpacking
    const double nn = static_cast<double>(p.n);
    std::vector<float2> ca, cb;
    table(ca, 4096, 1.0 / nn);
    table(cb, static_cast<int>(std::max<int64_t>(1, p.n / 4096)), 4096.0 / nn);
    twA->insert(twA->end(), ca.begin(), ca.end());
    twB->insert(twB->end(), cb.begin(), cb.end());
    // t2[q] = W^{kmul digit_rev(q)} = e^{-2 pi i digit_rev(q) / (2 N2r)} over the spectral row length N2r
    const int N2r = p.three() ? p.B : p.N2;
    for (int q = 0; q < N2r; ++q) {
      const double a = -2.0 * M_PI * digit_rev(q, N2r) / (2.0 * N2r);
      twA->push_back(make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a))));
    }
  }
}
// offsets of the e^{-2 pi i idx / n} factors appended to twA / twB (then t2 after twA's 8192 entries)
static int64_t twB_len(const Fft4Plan& p) { return std::max<int64_t>(1, p.N / 4096); }

// FINE launches for the L2-resident real plans (N <= 2^19: ISTA at n = 2^20 0.091 vs 0.111 ms per iteration;
// no gain at N = 2^20); CLB_FFT_FINE=0/1 forces either
static int fft4_fine(const Fft4Plan& p) {
  static const int env = [] {
    const char* v = std::getenv("CLB_FFT_FINE");
    return (v && *v) ? atoi(v) : -1;
  }();
  if (!p.real) return 0;
  if (env >= 0) return env;
  return p.N <= (int64_t(1) << 18) ? 2 : p.N <= (int64_t(1) << 19) ? 1 : 0;
}
template <int N>
static size_t cols_smem_t(int fine = 0) {
  return static_cast<size_t>(cols_b(N, fine)) * col_pitch_b(N, cols_b(N, fine)) * sizeof(float2);
}
template <int N>
static size_t rows_smem_t() { return static_cast<size_t>(row_count(N)) * row_pitch(N) * sizeof(float2); }
template <int N>
static size_t rows_r2c_smem_t(int fine = 0) {
  return static_cast<size_t>(2 * units_per_cta(N, fine)) * row_pitch(N) * sizeof(float2);
}

#define CLB_FFT4_SIZES(X) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)

void fft4_init_attributes() {
  static std::atomic<uint64_t> devs{0};
  if (!first_use_on_device(devs)) return;
  // columns are at most 2048 long (fft4_plan); longer column kernels are never launched
#define CLB_ATTR(N)                                                                                             \
  if (N <= 2048) {                                                                                              \
    cudaFuncSetAttribute(k_cols_fwd<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem_t<N>()); \
    cudaFuncSetAttribute(k_cols_inv<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem_t<N>()); \
    cudaFuncSetAttribute(k_cols_fwd<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem_t<N>());  \
    cudaFuncSetAttribute(k_cols_inv<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem_t<N>());  \
    cudaFuncSetAttribute(k_cols_fwd<N, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                         (int)cols_smem_t<N>(1));                                                                \
    cudaFuncSetAttribute(k_cols_fwd<N, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                         (int)cols_smem_t<N>(2));                                                                \
    cudaFuncSetAttribute(k_cols_inv_fwd<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,                  \
                         (int)cols_smem_t<N>());                                                                 \
    cudaFuncSetAttribute(k_cols_inv_fwd<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,                   \
                         (int)cols_smem_t<N>());                                                                 \
    cudaFuncSetAttribute(k_cols_inv_fwd<N, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,                \
                         (int)cols_smem_t<N>(1));                                                                \
    cudaFuncSetAttribute(k_cols_inv_fwd<N, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,                \
                         (int)cols_smem_t<N>(2));                                                                \
    cudaFuncSetAttribute(k_cols_inv<N, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                         (int)cols_smem_t<N>(1));                                                                \
    cudaFuncSetAttribute(k_cols_inv<N, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                         (int)cols_smem_t<N>(2));                                                                \
  }                                                                                                             \
  cudaFuncSetAttribute(k_rows<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_smem_t<N>());         \
  cudaFuncSetAttribute(k_rows_r2c<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows_r2c_smem_t<N>());   \
  cudaFuncSetAttribute(k_rows_r2c<N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,                          \
                       (int)rows_r2c_smem_t<N>(1));                                                            \
  cudaFuncSetAttribute(k_rows_r2c<N, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,                          \
                       (int)rows_r2c_smem_t<N>(2));
  CLB_FFT4_SIZES(CLB_ATTR)
#undef CLB_ATTR
  cudaFuncSetAttribute(k_mid<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem_t<128>());
  cudaFuncSetAttribute(k_mid<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem_t<128>());
  cudaFuncSetAttribute(k_mid<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem_t<256>());
  cudaFuncSetAttribute(k_mid<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols_smem_t<256>());
}

void launch_fft4_cols_fwd(const Fft4Plan& p, const float* u, float2* T, const float2* tw1, cudaStream_t st) {
  switch (p.N1) {
#define CLB_CASE(N)                                                                                        \
  case N:                                                                                                  \
    if (fft4_fine(p) == 2)                                                                                 \
      k_cols_fwd<N, true, 2><<<p.N2 / cols_b(N, 2), threads_of(2), cols_smem_t<N>(2), st>>>(u, T, p.N2, tw1); \
    else if (fft4_fine(p) == 1)                                                                            \
      k_cols_fwd<N, true, 1><<<p.N2 / cols_b(N, 1), threads_of(1), cols_smem_t<N>(1), st>>>(u, T, p.N2, tw1); \
    else if (p.real) k_cols_fwd<N, true><<<p.N2 / cols_per_cta(N), kThr, cols_smem_t<N>(), st>>>(u, T, p.N2, tw1); \
    else k_cols_fwd<N, false><<<p.N2 / cols_per_cta(N), kThr, cols_smem_t<N>(), st>>>(u, T, p.N2, tw1);      \
    break;
    CLB_FFT4_SIZES(CLB_CASE)
#undef CLB_CASE
  }
}
template <int A>
static void launch_mid(const Fft4Plan& p, float2* T, bool fwd, const float2* twM, const float2* twA,
                       const float2* twB, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(p.N1 * (p.B / cols_per_cta(A)));
  if (fwd) k_mid<A, true><<<grid, kThr, cols_smem_t<A>(), st>>>(T, p.N1, p.N2, p.B, twM, twA, twB);
  else k_mid<A, false><<<grid, kThr, cols_smem_t<A>(), st>>>(T, p.N1, p.N2, p.B, twM, twA, twB);
}
template <int N>
static void launch_rows_r2c_fine(const Fft4Plan& p, float2* T, const float2* H, bool conj_h, int A, int rowmod, int mult,
                                 const float2* twR, const float2* twA, const float2* twB, const float2* twCA,
                                 const float2* twCB, cudaStream_t st) {
  const int kmul = p.N1 * A;
  const float4* H2 = reinterpret_cast<const float4*>(H);
  if (fft4_fine(p) == 2)
    k_rows_r2c<N, 2><<<(kmul / 2 + units_per_cta(N, 2)) / units_per_cta(N, 2), threads_of(2), rows_r2c_smem_t<N>(2),
                       st>>>(T, H2, conj_h ? 1 : 0, p.N1, A, rowmod, mult, twR, twA, twB, twCA, twCB, twA + 8192);
  else
    k_rows_r2c<N, 1><<<(kmul / 2 + units_per_cta(N, 1)) / units_per_cta(N, 1), threads_of(1), rows_r2c_smem_t<N>(1),
                       st>>>(T, H2, conj_h ? 1 : 0, p.N1, A, rowmod, mult, twR, twA, twB, twCA, twCB, twA + 8192);
}
void launch_fft4_rows(const Fft4Plan& p, float2* T, const float2* H, bool conj_h, const float2* tw2,
                      const float2* twA, const float2* twB, cudaStream_t st) {
  // rows of length R, `count` of them; row r's twiddle exponent mult * n2 * digit_rev(r mod rowmod)
  const int R = p.three() ? p.B : p.N2;
  const int count = static_cast<int>(p.N / R), rowmod = p.three() ? p.A : p.N1, mult = p.three() ? p.N1 : 1;
  const float2* twR = p.three() ? tw2 + p.A : tw2;
  const int A = p.three() ? p.A : 1, kmul = p.N1 * A;
  const float2 *twCA = twA + 4096, *twCB = twB + twB_len(p);
  if (p.three()) {
    if (p.A == 256) launch_mid<256>(p, T, true, tw2, twA, twB, st);
    else launch_mid<128>(p, T, true, tw2, twA, twB, st);
  }
  switch (R) {
#define CLB_CASE(N)                                                                                            \
  case N:                                                                                                      \
    if (fft4_fine(p))                                                                                          \
      launch_rows_r2c_fine<N>(p, T, H, conj_h, A, rowmod, mult, twR, twA, twB, twCA, twCB, st);                \
    else if (p.real)                                                                                           \
      k_rows_r2c<N><<<(kmul / 2 + units_per_cta(N)) / units_per_cta(N), kThr, rows_r2c_smem_t<N>(), st>>>(     \
          T, reinterpret_cast<const float4*>(H), conj_h ? 1 : 0, p.N1, A, rowmod, mult, twR, twA, twB, twCA,   \
          twCB, twA + 8192);                                                                                   \
    else                                                                                                       \
      k_rows<N><<<count / row_count(N), kThr, rows_smem_t<N>(), st>>>(T, H, conj_h ? 1 : 0, rowmod, mult, twR, \
                                                                        twA, twB);                             \
    break;
    CLB_FFT4_SIZES(CLB_CASE)
#undef CLB_CASE
  }
  if (p.three()) {
    if (p.A == 256) launch_mid<256>(p, T, false, tw2, twA, twB, st);
    else launch_mid<128>(p, T, false, tw2, twA, twB, st);
  }
}
void launch_fft4_cols_inv(const Fft4Plan& p, const float2* T, const Fft4Out& o, const float2* tw1,
                          cudaStream_t st) {
  // real plans: 1 / N for the length-N inverse times the 1/4 of the spectral step (k_rows_r2c)
  const float inv_n = p.real ? 1.0f / (4.0f * static_cast<float>(p.N)) : 1.0f / static_cast<float>(p.n);
  switch (p.N1) {
#define CLB_CASE(N)                                                                                        \
  case N:                                                                                                  \
    if (fft4_fine(p) == 2)                                                                                 \
      k_cols_inv<N, true, 2><<<p.N2 / cols_b(N, 2), threads_of(2), cols_smem_t<N>(2), st>>>(T, o, p.N2, tw1, inv_n); \
    else if (fft4_fine(p) == 1)                                                                            \
      k_cols_inv<N, true, 1><<<p.N2 / cols_b(N, 1), threads_of(1), cols_smem_t<N>(1), st>>>(T, o, p.N2, tw1, inv_n); \
    else if (p.real) k_cols_inv<N, true><<<p.N2 / cols_per_cta(N), kThr, cols_smem_t<N>(), st>>>(T, o, p.N2, tw1, inv_n); \
    else k_cols_inv<N, false><<<p.N2 / cols_per_cta(N), kThr, cols_smem_t<N>(), st>>>(T, o, p.N2, tw1, inv_n);      \
    break;
    CLB_FFT4_SIZES(CLB_CASE)
#undef CLB_CASE
  }
}
void launch_fft4_cols_inv_fwd(const Fft4Plan& p, float2* T, const Fft4Out& o, const float2* tw1, cudaStream_t st) {
  const float inv_n = p.real ? 1.0f / (4.0f * static_cast<float>(p.N)) : 1.0f / static_cast<float>(p.n);
  switch (p.N1) {
#define CLB_CASE(N)                                                                                          \
  case N:                                                                                                    \
    if (fft4_fine(p) == 2)                                                                                   \
      k_cols_inv_fwd<N, true, 2><<<p.N2 / cols_b(N, 2), threads_of(2), cols_smem_t<N>(2), st>>>(T, o, p.N2, tw1, inv_n); \
    else if (fft4_fine(p) == 1)                                                                              \
      k_cols_inv_fwd<N, true, 1><<<p.N2 / cols_b(N, 1), threads_of(1), cols_smem_t<N>(1), st>>>(T, o, p.N2, tw1, inv_n); \
    else if (p.real)                                                                                         \
      k_cols_inv_fwd<N, true><<<p.N2 / cols_per_cta(N), kThr, cols_smem_t<N>(), st>>>(T, o, p.N2, tw1, inv_n);   \
    else                                                                                                     \
      k_cols_inv_fwd<N, false><<<p.N2 / cols_per_cta(N), kThr, cols_smem_t<N>(), st>>>(T, o, p.N2, tw1, inv_n);  \
    break;
    CLB_FFT4_SIZES(CLB_CASE)
#undef CLB_CASE
  }
}
void launch_fft4_perm_spectrum(const Fft4Plan& p, const double2* spec, double s, float2* out, cudaStream_t st) {
  if (p.real)
    k_perm_spectrum_pairs<<<148 * 8, 256, 0, st>>>(spec, s, reinterpret_cast<float4*>(out), p.N1,
                                                   p.three() ? p.A : 1, p.three() ? p.B : p.N2);
  else
    k_perm_spectrum<<<148 * 8, 256, 0, st>>>(spec, s, out, p.N1, p.N2, p.A, p.B, 0);
}
bool small_fft_supported(int64_t n) {
  const char* v = std::getenv("CLB_NO_SMALL");
  return !(v && v[0] == '1') && (n == 1024 || n == 2048 || n == 4096 || n == 8192);
}
void launch_small_fft_perm(const float2* H, float2* Hp, int64_t n, cudaStream_t st) {
  k_perm_small<<<8, 256, 0, st>>>(H, Hp, static_cast<int>(n));
}
cudaError_t launch_small_fft_ista(int64_t n, int64_t m, const float2* Hp, const float2* tw, const int* omega,
                                  const float* y, float* x, float* r, float* delta, float tau, float thr, int iters,
                                  cudaStream_t st) {
  switch (n) {
#define CLB_SMALL_CASE(N)                                                                                   \
  case N: {                                                                                                 \
    static std::atomic<uint64_t> attr{0};                                                                   \
    if (first_use_on_device(attr)) {                                                                        \
      cudaFuncSetAttribute(k_small_fft_ista<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,                \
                           static_cast<int>(small_fft_smem<N>()));                                          \
    }                                                                                                       \
    k_small_fft_ista<N><<<1, kThr, small_fft_smem<N>(), st>>>(Hp, tw, omega, y, x, r, delta,                \
                                                               static_cast<int>(m), tau, thr, iters);       \
    return cudaGetLastError();                                                                              \
  }
    CLB_SMALL_CASE(1024)
    CLB_SMALL_CASE(2048)
    CLB_SMALL_CASE(4096)
    CLB_SMALL_CASE(8192)
#undef CLB_SMALL_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

bool small_fft_cadmm_supported(int64_t n) { return small_fft_supported(n) && n <= 4096; }
cudaError_t launch_small_fft_cadmm(int64_t n, const float2* Hc, const float2* Hb, const float2* tw, const float* d,
                                   const float* pty, float* x, float* z, float* nu, float* mu, float* v, float* beta,
                                   float rho, float sigma, float tau1, float tau2, float thr, int iters,
                                   cudaStream_t st) {
  switch (n) {
#define CLB_SMALL_CASE(N)                                                                                   \
  case N: {                                                                                                 \
    static std::atomic<uint64_t> attr{0};                                                                   \
    if (first_use_on_device(attr)) {                                                                        \
      cudaFuncSetAttribute(k_small_fft_cadmm<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,               \
                           static_cast<int>(small_fft_cadmm_smem<N>()));                                    \
    }                                                                                                       \
    k_small_fft_cadmm<N><<<1, kThr, small_fft_cadmm_smem<N>(), st>>>(Hc, Hb, tw, d, pty, x, z, nu, mu, v,    \
                                                                     beta, rho, sigma, tau1, tau2, thr, iters); \
    return cudaGetLastError();                                                                              \
  }
    CLB_SMALL_CASE(1024)
    CLB_SMALL_CASE(2048)
    CLB_SMALL_CASE(4096)
#undef CLB_SMALL_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

void launch_scatter_real(const float* r, const int* omega, float* u, int64_t m, cudaStream_t st) {
  if (m > 0) k_scatter_real<<<148 * 4, 256, 0, st>>>(r, omega, u, m);
}

}  // namespace clb

namespace clb {
namespace {
__global__ void k_rowid(const int* __restrict__ omega, int* __restrict__ rowid, int64_t m) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    rowid[omega[t]] = static_cast<int>(t);
}
}  // namespace
void launch_rowid(const int* omega, int* rowid, int64_t n, int64_t m, cudaStream_t st) {
  cudaMemsetAsync(rowid, 0xff, sizeof(int) * n, st);  // -1: not a row
  if (m > 0) k_rowid<<<148 * 4, 256, 0, st>>>(omega, rowid, m);
}
}  // namespace clb
