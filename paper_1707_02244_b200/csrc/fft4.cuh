// Four-step FFT engine (fp32 complex, power-of-two 2^14 <= n <= 2^24); see fft4.cu.
#pragma once
#include <climits>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace clb {
struct Fft4Plan {
  int64_t n = 0;       // length of the (real) product
  int64_t N = 0;       // transform length: n / 2 complex values for real plans (the default), else n
  bool real = false;   // real plans: z[j] = u[2j] + i u[2j+1], the spectrum unpacked pairwise in the rows kernel
  int N1 = 0, N2 = 0;  // N = N1 * N2; columns of length N1, rows of length N2
  // n >= 2^22: three levels, N1 = 256 and the length-N2 row transforms themselves four-step, N2 = A * B
  // (A along a stride-B axis, B contiguous), so every pass moves 128-byte row segments
  int A = 0, B = 0;
  bool three() const { return A > 0; }
};
bool fft4_supported(int64_t n);
Fft4Plan fft4_plan(int64_t n);
// twiddle tables (host, fp64-accurate fp32): e^{-2 pi i k / N1}, e^{-2 pi i k / N2} (three levels: the
// A-point table followed by the B-point table), and the two factors of
// e^{-2 pi i idx / N} = twB[idx >> 12] * twA[idx & 4095]; real plans append to twA / twB the factors of
// e^{-2 pi i idx / n} (4096 and n / 4096 entries)
void fft4_twiddles(const Fft4Plan& p, std::vector<float2>* tw1, std::vector<float2>* tw2, std::vector<float2>* twA,
                   std::vector<float2>* twB);
void fft4_init_attributes();
// u real (n) -> T (N complex): column DIF FFTs (spectral order permuted)
void launch_fft4_cols_fwd(const Fft4Plan& p, const float* u, float2* T, const float2* tw1, cudaStream_t st);
// in place: twiddle, row DIF FFT, times H~ (or conj), row DIT inverse FFT, inverse twiddle (three levels:
// the length-N2 row transforms as A-point passes over a stride-B axis around B-point contiguous rows)
void launch_fft4_rows(const Fft4Plan& p, float2* T, const float2* H, bool conj_h, const float2* tw2,
                      const float2* twA, const float2* twB, cudaStream_t st);
// What the inverse column pass does with Re(y)/n (see k_cols_inv).
struct Fft4Out {
  enum Mode { kProduct = 0, kRows = 1, kResidual = 2, kIstaStep = 3, kBeta = 4 } mode = kProduct;
  float* out = nullptr;         // product (n), rows (m), residual r (m), or delta (n)
  const int* rowid = nullptr;   // position -> row (kRows, kResidual)
  const float* y = nullptr;     // kResidual
  float* u = nullptr;           // kResidual: dense P^T r
  float* x = nullptr;           // kIstaStep
  float tau = 0.f, thr = 0.f;   // kIstaStep
  const float* z = nullptr;     // kBeta: out = rho * Re/n + sigma (z - nu)
  const float* nu = nullptr;
  float rho = 0.f, sigma = 0.f;
  int64_t n_valid = INT64_MAX;  // outputs j >= n_valid (the padded engine's convolution tail) are not written
};
// T -> column DIT inverse FFTs, then `o`.
void launch_fft4_cols_inv(const Fft4Plan& p, const float2* T, const Fft4Out& o, const float2* tw1, cudaStream_t st);
// T -> column DIT inverse FFTs, then `o`, then -- on the vector `o` produces (the residual's P^T r, beta, or
// the product itself) -- the next product's column DIF FFTs, in place on T (two chained products, one pass).
void launch_fft4_cols_inv_fwd(const Fft4Plan& p, float2* T, const Fft4Out& o, const float2* tw1, cudaStream_t st);
// natural-order fp64 spectrum (n entries) / s -> the engine's permuted fp32 order (N entries; real plans pack
// H[0] and H[n / 2] into entry 0)
void launch_fft4_perm_spectrum(const Fft4Plan& p, const double2* spec, double s, float2* out, cudaStream_t st);
// rowid[j] = t for j = omega[t], -1 elsewhere
void launch_rowid(const int* omega, int* rowid, int64_t n, int64_t m, cudaStream_t st);
// u[omega[t]] = r[t]
void launch_scatter_real(const float* r, const int* omega, float* u, int64_t m, cudaStream_t st);
// One-CTA FFT-engine ISTA for n in {1024, 2048, 4096, 8192} (CLB_NO_SMALL unset): all unchecked
// iterations in one launch.  Hp = the operator spectrum in the DIF output order (launch_small_fft_perm),
// tw = e^{-2 pi i k / n}, k < n.
bool small_fft_supported(int64_t n);
void launch_small_fft_perm(const float2* H, float2* Hp, int64_t n, cudaStream_t st);
cudaError_t launch_small_fft_ista(int64_t n, int64_t m, const float2* Hp, const float2* tw, const int* omega,
                                  const float* y, float* x, float* r, float* delta, float tau, float thr, int iters,
                                  cudaStream_t st);
// One-CTA FFT-engine cADMM for n in {1024, 2048, 4096}; Hc, Hb in the DIF output order.
bool small_fft_cadmm_supported(int64_t n);
cudaError_t launch_small_fft_cadmm(int64_t n, const float2* Hc, const float2* Hb, const float2* tw, const float* d,
                                   const float* pty, float* x, float* z, float* nu, float* mu, float* v, float* beta,
                                   float rho, float sigma, float tau1, float tau2, float thr, int iters,
                                   cudaStream_t st);
}  // namespace clb
