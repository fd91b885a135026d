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

// 16-point twiddle table (fp64 constants; the fp32 engine uses them rounded).
__device__ constexpr double kCos16[16] = {1.0, 0.92387953251128674, 0.70710678118654757, 0.38268343236508978, 0.0,
                                          -0.38268343236508978, -0.70710678118654757, -0.92387953251128674, -1.0,
                                          -0.92387953251128674, -0.70710678118654757, -0.38268343236508978, -0.0,
                                          0.38268343236508978, 0.70710678118654757, 0.92387953251128674};
__device__ constexpr double kSin16[16] = {0.0, 0.38268343236508978, 0.70710678118654757, 0.92387953251128674, 1.0,
                                          0.92387953251128674, 0.70710678118654757, 0.38268343236508978, 0.0,
                                          -0.38268343236508978, -0.70710678118654757, -0.92387953251128674, -1.0,
                                          -0.92387953251128674, -0.70710678118654757, -0.38268343236508978};

// fp32 (the FFT engine) and fp64 (the setup transforms) share one pass kernel.
template <typename T>
struct Cx;
template <>
struct Cx<float> {
  using V = float2;
  static __device__ __forceinline__ V mk(float a, float b) { return make_float2(a, b); }
  static __device__ __forceinline__ void sincospi_(float x, float* s, float* c) { sincospif(x, s, c); }
};
template <>
struct Cx<double> {
  using V = double2;
  static __device__ __forceinline__ V mk(double a, double b) { return make_double2(a, b); }
  static __device__ __forceinline__ void sincospi_(double x, double* s, double* c) { sincospi(x, s, c); }
};

template <typename V>
__device__ __forceinline__ V cmul(V a, V b) { return V{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
template <typename V>
__device__ __forceinline__ V cadd(V a, V b) { return V{a.x + b.x, a.y + b.y}; }
template <typename V>
__device__ __forceinline__ V csub(V a, V b) { return V{a.x - b.x, a.y - b.y}; }

// In-register radix-R DFT (R = 2^k), natural order in and out, sign SG (-1 fwd).
template <int R, int SG, typename T>
__device__ __forceinline__ void dft_reg(typename Cx<T>::V (&v)[R]) {
  using V = typename Cx<T>::V;
  // iterative radix-2 DIT on R registers with bit-reversal via static index math
  V t[R];
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
        const V w = Cx<T>::mk(static_cast<T>(kCos16[e]), static_cast<T>(SG * kSin16[e]));
        const V u = t[base + k];
        const V x = cmul(t[base + k + half], w);
        t[base + k] = cadd(u, x);
        t[base + k + half] = csub(u, x);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = t[i];
}

// One Stockham pass: Ns = product of radices already applied.
template <int R, int SG, typename T>
__global__ void __launch_bounds__(256) k_fft_pass(const typename Cx<T>::V* __restrict__ in,
                                                  typename Cx<T>::V* __restrict__ out, int64_t n, int64_t Ns) {
  using V = typename Cx<T>::V;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = n / R;
  if (j >= stride) return;
  const int64_t jm = j % Ns;
  V v[R];
  const T inv = T(2) / (T)(Ns * R);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    V a = in[j + r * stride];
    if (r > 0 && Ns > 1) {
      // angle 2 pi r jm / (Ns R): r*jm < Ns R is exact (2^24 in fp32, 2^53 in fp64)
      T s, c;
      Cx<T>::sincospi_((T)(r * jm) * inv, &s, &c);
      a = cmul(a, Cx<T>::mk(c, SG * s));
    }
    v[r] = a;
  }
  dft_reg<R, SG, T>(v);
  const int64_t idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
  for (int r = 0; r < R; ++r) out[idxD + r * Ns] = v[r];
}

template <int SG, typename T>
void launch_pass(int R, const typename Cx<T>::V* in, typename Cx<T>::V* out, int64_t n, int64_t Ns,
                 cudaStream_t st) {
  const int64_t threads = n / R;
  const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
  switch (R) {
    case 16: k_fft_pass<16, SG, T><<<grid, 256, 0, st>>>(in, out, n, Ns); break;
    case 8: k_fft_pass<8, SG, T><<<grid, 256, 0, st>>>(in, out, n, Ns); break;
    case 4: k_fft_pass<4, SG, T><<<grid, 256, 0, st>>>(in, out, n, Ns); break;
    default: k_fft_pass<2, SG, T><<<grid, 256, 0, st>>>(in, out, n, Ns); break;
  }
}

template <typename T>
const typename Cx<T>::V* fft_run_t(typename Cx<T>::V* a, typename Cx<T>::V* b, int64_t n, bool inverse,
                                   cudaStream_t st) {
  using V = typename Cx<T>::V;
  int lg = 0;
  while ((int64_t(1) << lg) < n) ++lg;
  V* src = a;
  V* dst = b;
  int64_t Ns = 1;
  while (lg > 0) {
    const int k = lg >= 4 ? 4 : lg;
    const int R = 1 << k;
    if (inverse) launch_pass<+1, T>(R, src, dst, n, Ns, st);
    else launch_pass<-1, T>(R, src, dst, n, Ns, st);
    Ns *= R;
    lg -= k;
    V* t = src;
    src = dst;
    dst = t;
  }
  return src;
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
  return fft_run_t<float>(a, b, n, inverse, st);
}
const double2* fft64_run(double2* a, double2* b, int64_t n, bool inverse, cudaStream_t st) {
  return fft_run_t<double>(a, b, n, inverse, st);
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

// ---- fp64 setup transforms on the device (power-of-two n) -------------------
// spectral_norm (circulant.hpp:347-351), regularized_gram_inverse
// (circulant.hpp:297-320, with its 1e-14 floor and the idft_real residue
// check of fft.hpp:74-89) and the fp32 operator rows, computed where they are
// used instead of on the host (the host fp64 FFT took ~0.1 s per transform at
// n = 2^20; these take well under a millisecond).
namespace {
// max over non-negative doubles: their IEEE bit patterns order like the values
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* a, double v) {
  atomicMax(a, static_cast<unsigned long long>(__double_as_longlong(v)));
}
__device__ __forceinline__ void atomic_min_nonneg(unsigned long long* a, double v) {
  atomicMin(a, static_cast<unsigned long long>(__double_as_longlong(v)));
}
__global__ void k_real_to_complex64(const double* __restrict__ x, double2* __restrict__ X, int64_t n) {
  CLB_GRID_LOOP(i, n) X[i] = make_double2(x[i], 0.0);
}
__global__ void k_absmax64(const double2* __restrict__ X, int64_t n, unsigned long long* out) {
  double mx = 0.0;
  CLB_GRID_LOOP(k, n) mx = fmax(mx, hypot(X[k].x, X[k].y));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, mx);
}
// B[k] = 1 / (rho |X_k / s|^2 + sigma) (real); bhat (optional) its fp32 copy;
// mind = min denominator (the reference's invertibility floor).
__global__ void k_gram_spectrum(const double2* __restrict__ X, double s, double rho, double sigma,
                                double2* __restrict__ B, float2* __restrict__ bhat, unsigned long long* mind,
                                int64_t n) {
  double mn = 1e300;
  CLB_GRID_LOOP(k, n) {
    const double re = X[k].x / s, im = X[k].y / s;
    const double den = rho * (re * re + im * im) + sigma;
    mn = fmin(mn, den);
    const double v = 1.0 / den;
    B[k] = make_double2(v, 0.0);
    if (bhat) bhat[k] = make_float2(static_cast<float>(v), 0.f);
  }
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) atomic_min_nonneg(mind, mn);
}
// out[i] = Re(Y[i]) / n; max |re| and max |im| (after the 1/n) for the residue check.
__global__ void k_real_part64(const double2* __restrict__ Y, double inv_n, double* __restrict__ out,
                              unsigned long long* mre, unsigned long long* mim, int64_t n) {
  double a = 0.0, b = 0.0;
  CLB_GRID_LOOP(i, n) {
    const double re = Y[i].x * inv_n, im = Y[i].y * inv_n;
    out[i] = re;
    a = fmax(a, fabs(re));
    b = fmax(b, fabs(im));
  }
  for (int o = 16; o > 0; o >>= 1) {
    a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(mre, a);
    atomic_max_nonneg(mim, b);
  }
}
// out[i] = (float)(x[i] / s); rev[i] = out[(n - i) mod n] (either may be null)
__global__ void k_rows_f32(const double* __restrict__ x, double s, float* __restrict__ out, float* __restrict__ rev,
                           int64_t n) {
  CLB_GRID_LOOP(i, n) {
    const float v = static_cast<float>(x[i] / s);
    if (out) out[i] = v;
    if (rev) rev[i == 0 ? 0 : n - i] = v;
  }
}
// Y[k] = (conj_x ? conj(X[k]) : X[k]) * Y[k]
__global__ void k_cmul64(const double2* __restrict__ X, double2* __restrict__ Y, int conj_x, int64_t n) {
  CLB_GRID_LOOP(k, n) {
    const double2 a = X[k], b = Y[k];
    const double ay = conj_x ? -a.y : a.y;
    Y[k] = make_double2(a.x * b.x - ay * b.y, a.x * b.y + ay * b.x);
  }
}
// spectrum of x / s in fp32 (the FFT engine's operator spectrum)
__global__ void k_spectrum_f32(const double2* __restrict__ X, double s, float2* __restrict__ out, int64_t n) {
  CLB_GRID_LOOP(k, n) out[k] = make_float2(static_cast<float>(X[k].x / s), static_cast<float>(X[k].y / s));
}
}  // namespace

void launch_real_to_complex64(const double* x, double2* X, int64_t n, cudaStream_t st) {
  k_real_to_complex64<<<pw_grid(n), kPw, 0, st>>>(x, X, n);
}
void launch_absmax64(const double2* X, int64_t n, unsigned long long* out, cudaStream_t st) {
  k_absmax64<<<pw_grid(n), kPw, 0, st>>>(X, n, out);
}
void launch_gram_spectrum(const double2* X, double s, double rho, double sigma, double2* B, float2* bhat,
                          unsigned long long* mind, int64_t n, cudaStream_t st) {
  k_gram_spectrum<<<pw_grid(n), kPw, 0, st>>>(X, s, rho, sigma, B, bhat, mind, n);
}
void launch_real_part64(const double2* Y, double* out, unsigned long long* mre, unsigned long long* mim, int64_t n,
                        cudaStream_t st) {
  k_real_part64<<<pw_grid(n), kPw, 0, st>>>(Y, 1.0 / static_cast<double>(n), out, mre, mim, n);
}
void launch_rows_f32(const double* x, double s, float* out, float* rev, int64_t n, cudaStream_t st) {
  k_rows_f32<<<pw_grid(n), kPw, 0, st>>>(x, s, out, rev, n);
}
void launch_cmul64(const double2* X, double2* Y, bool conj_x, int64_t n, cudaStream_t st) {
  k_cmul64<<<pw_grid(n), kPw, 0, st>>>(X, Y, conj_x ? 1 : 0, n);
}
void launch_spectrum_f32(const double2* X, double s, float2* out, int64_t n, cudaStream_t st) {
  k_spectrum_f32<<<pw_grid(n), kPw, 0, st>>>(X, s, out, n);
}

}  // namespace clb
