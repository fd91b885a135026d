// Device FFT (fp32 complex, power-of-two n) for the FFT engine; see fft.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace clb {
bool is_pow2(int64_t n);
int fft_passes(int64_t n);
// Unnormalized DFT of a (length n) using b as ping-pong scratch; returns the
// buffer (a or b) holding the result.  inverse: sign +1.
const float2* fft_run(float2* a, float2* b, int64_t n, bool inverse, cudaStream_t st);
// fp64 variant (setup transforms).
const double2* fft64_run(double2* a, double2* b, int64_t n, bool inverse, cudaStream_t st);
// Pointwise kernels of the FFT engine.
void launch_real_to_complex(const float* x, float2* X, int64_t n, cudaStream_t st);
void launch_embed_rows(const float* r, const int* omega, float2* X, int64_t n, int64_t m, cudaStream_t st);
void launch_spec_mul(float2* X, const float2* H, bool conj_h, int64_t n, cudaStream_t st);
void launch_extract_real(const float2* Y, float* out, int64_t n, cudaStream_t st);
void launch_gather_real(const float2* Y, const int* omega, float* out, int64_t n, int64_t m, cudaStream_t st);
// fp64 setup kernels (device-side spectral norm / Gram inverse / operator rows).
void launch_real_to_complex64(const double* x, double2* X, int64_t n, cudaStream_t st);
void launch_absmax64(const double2* X, int64_t n, unsigned long long* out, cudaStream_t st);
void launch_gram_spectrum(const double2* X, double s, double rho, double sigma, double2* B, float2* bhat,
                          unsigned long long* mind, int64_t n, cudaStream_t st);
void launch_real_part64(const double2* Y, double* out, unsigned long long* mre, unsigned long long* mim, int64_t n,
                        cudaStream_t st);
void launch_rows_f32(const double* x, double s, float* out, float* rev, int64_t n, cudaStream_t st);
void launch_spectrum_f32(const double2* X, double s, float2* out, int64_t n, cudaStream_t st);
// Y = conj?(X) * Y (fp64 complex, pointwise)
void launch_cmul64(const double2* X, double2* Y, bool conj_x, int64_t n, cudaStream_t st);
}  // namespace clb
