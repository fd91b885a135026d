// On-device FFT engine: the reference's default
// `use_fft=true` path (circulant.hpp:236-274, solvers.hpp:154-165) on sm_100a.
//
// Hand-written Stockham autosort FFT over fp32 complex (float2), power-of-two
// n.  One kernel per radix-R pass, R in {16, 8, 4, 2}; each thread loads R
// elements strided by n/R (coalesced across threads), applies the pass
// twiddles, runs a register radix-R butterfly and writes R outputs strided by
// Ns (the first pass, Ns = 1, writes each thread's R outputs contiguously).
// HBM/L2-bound: every pass reads and writes n complex values once.  The forward transform uses
// e^{-2 pi i jk/n}; the inverse uses +, without the 1/n (folded into the
// pointwise kernels, like idft in fft.hpp:59-69).
#include <cstdint>

#include "fft.cuh"

namespace clb {
namespace {

__device__ constexpr float kCos16[16] = {1.000000000f, 0.923879533f, 0.707106781f, 0.382683432f, 0.000000000f, -0.382683432f, -0.707106781f, -0.923879533f, -1.000000000f, -0.923879533f, -0.707106781f, -0.382683432f, -0.000000000f, 0.382683432f, 0.707106781f, 0.923879533f};
__device__ constexpr float kSin16[16] = {0.000000000f, 0.382683432f, 0.707106781f, 0.923879533f, 1.000000000f, 0.923879533f, 0.707106781f, 0.382683432f, 0.000000000f, -0.382683432f, -0.707106781f, -0.923879533f, -1.000000000f, -0.923879533f, -0.707106781f, -0.382683432f};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// In-register radix-R DFT (R = 2^k), natural order in and out, sign SG (-1 fwd).
template <int R, int SG>
__device__ __forceinline__ void dft_reg(float2 (&v)[R]) {
  // iterative radix-2 DIT on R registers with bit-reversal via static index math
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
        // e^{SG 2 pi i k / (2 half)} from the 16-point table (compile-time index)
        const int e = k * (16 / (2 * half));
        const float2 w = make_float2(kCos16[e], SG * kSin16[e]);
        const float2 u = t[base + k];
        const float2 x = cmul(t[base + k + half], w);
        t[base + k] = cadd(u, x);
        t[base + k + half] = csub(u, x);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = t[i];
}

// One Stockham pass: Ns = product of radices already applied.
template <int R, int SG>
__global__ void __launch_bounds__(256) k_fft_pass(const float2* __restrict__ in, float2* __restrict__ out, int64_t n,
                                                  int64_t Ns) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = n / R;
  if (j >= stride) return;
  const int64_t jm = j % Ns;
  float2 v[R];
  const float inv = 2.0f / (float)(Ns * R);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float2 a = in[j + r * stride];
    if (r > 0 && Ns > 1) {
      // angle 2 pi r jm / (Ns R): r*jm < Ns R <= 2^24 is exact in fp32
      float s, c;
      sincospif((float)(r * jm) * inv, &s, &c);
      a = cmul(a, make_float2(c, SG * s));
    }
    v[r] = a;
  }
  dft_reg<R, SG>(v);
  const int64_t idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
  for (int r = 0; r < R; ++r) out[idxD + r * Ns] = v[r];
}

template <int SG>
void launch_pass(int R, const float2* in, float2* out, int64_t n, int64_t Ns, cudaStream_t st) {
  const int64_t threads = n / R;
  const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
  switch (R) {
    case 16: k_fft_pass<16, SG><<<grid, 256, 0, st>>>(in, out, n, Ns); break;
    case 8: k_fft_pass<8, SG><<<grid, 256, 0, st>>>(in, out, n, Ns); break;
    case 4: k_fft_pass<4, SG><<<grid, 256, 0, st>>>(in, out, n, Ns); break;
    default: k_fft_pass<2, SG><<<grid, 256, 0, st>>>(in, out, n, Ns); break;
  }
}

}  // namespace

int fft_passes(int64_t n) {
  int lg = 0;
  while ((int64_t(1) << lg) < n) ++lg;
  int passes = 0;
  while (lg > 0) {
    lg -= lg >= 4 ? 4 : lg;
    ++passes;
  }
  return passes;
}

const float2* fft_run(float2* a, float2* b, int64_t n, bool inverse, cudaStream_t st) {
  int lg = 0;
  while ((int64_t(1) << lg) < n) ++lg;
  float2* src = a;
  float2* dst = b;
  int64_t Ns = 1;
  while (lg > 0) {
    const int k = lg >= 4 ? 4 : lg;
    const int R = 1 << k;
    if (inverse) launch_pass<+1>(R, src, dst, n, Ns, st);
    else launch_pass<-1>(R, src, dst, n, Ns, st);
    Ns *= R;
    lg -= k;
    float2* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

// ---- pointwise kernels of the FFT engine ------------------------------------
namespace {
constexpr int kPw = 256;
inline unsigned pw_grid(int64_t len) {
  int64_t g = (len + kPw - 1) / kPw;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}
#define CLB_GRID_LOOP(i, len) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (len); i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_real_to_complex(const float* __restrict__ x, float2* __restrict__ X, int64_t n) {
  CLB_GRID_LOOP(i, n) X[i] = make_float2(x[i], 0.f);
}
__global__ void k_zero_c(float2* __restrict__ X, int64_t n) {
  CLB_GRID_LOOP(i, n) X[i] = make_float2(0.f, 0.f);
}
__global__ void k_scatter_rows(const float* __restrict__ r, const int* __restrict__ omega, float2* __restrict__ X,
                               int64_t m) {
  CLB_GRID_LOOP(t, m) X[omega[t]] = make_float2(r[t], 0.f);
}
// X[k] *= H[k] (conj_h: conj(H[k]))
__global__ void k_spec_mul(float2* __restrict__ X, const float2* __restrict__ H, int conj_h, int64_t n) {
  CLB_GRID_LOOP(k, n) {
    const float2 h = H[k];
    const float hy = conj_h ? -h.y : h.y;
    const float2 a = X[k];
    X[k] = make_float2(a.x * h.x - a.y * hy, a.x * hy + a.y * h.x);
  }
}
// out[i] = Re(Y[i]) / n   (idft_real, fft.hpp:74-89, without the residue check)
__global__ void k_extract_real(const float2* __restrict__ Y, float* __restrict__ out, float inv_n, int64_t n) {
  CLB_GRID_LOOP(i, n) out[i] = Y[i].x * inv_n;
}
// out[t] = Re(Y[omega[t]]) / n   (mask.apply of the full product, circulant.hpp:160-167)
__global__ void k_gather_real(const float2* __restrict__ Y, const int* __restrict__ omega, float* __restrict__ out,
                              float inv_n, int64_t m) {
  CLB_GRID_LOOP(t, m) out[t] = Y[omega[t]].x * inv_n;
}
}  // namespace

void launch_real_to_complex(const float* x, float2* X, int64_t n, cudaStream_t st) {
  k_real_to_complex<<<pw_grid(n), kPw, 0, st>>>(x, X, n);
}
void launch_embed_rows(const float* r, const int* omega, float2* X, int64_t n, int64_t m, cudaStream_t st) {
  k_zero_c<<<pw_grid(n), kPw, 0, st>>>(X, n);
  k_scatter_rows<<<pw_grid(m), kPw, 0, st>>>(r, omega, X, m);
}
void launch_spec_mul(float2* X, const float2* H, bool conj_h, int64_t n, cudaStream_t st) {
  k_spec_mul<<<pw_grid(n), kPw, 0, st>>>(X, H, conj_h ? 1 : 0, n);
}
void launch_extract_real(const float2* Y, float* out, int64_t n, cudaStream_t st) {
  k_extract_real<<<pw_grid(n), kPw, 0, st>>>(Y, out, 1.0f / static_cast<float>(n), n);
}
void launch_gather_real(const float2* Y, const int* omega, float* out, int64_t n, int64_t m, cudaStream_t st) {
  k_gather_real<<<pw_grid(m), kPw, 0, st>>>(Y, omega, out, 1.0f / static_cast<float>(n), m);
}

}  // namespace clb
