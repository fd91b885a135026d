// fp64 setup transforms of the circlasso_b200 library.
//
// These run once per solve on the host, exactly where the paper places the
// Gram inversion ("the inversion is done on the CPU via
// FFT"); the per-iteration hot path never touches them.  The DFT is an
// iterative radix-2 transform for powers of two and Bluestein's chirp-z
// algorithm (over a power-of-two transform) for every other length.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <sstream>

#include "host_common.hpp"

namespace clb {

namespace {
thread_local std::string g_error;

constexpr double kPi = 3.14159265358979323846;

bool power_of_two(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

// Cache of twiddle tables keyed by (n, direction): setup transforms for one
// solve reuse the same lengths several times.
struct Twiddles {
  int64_t n = 0;
  bool inverse = false;
  std::vector<cplx> w;
};
thread_local Twiddles g_tw[2];

const std::vector<cplx>& twiddles(int64_t n, bool inverse) {
  Twiddles& t = g_tw[inverse ? 1 : 0];
  if (t.n != n) {
    t.n = n;
    t.inverse = inverse;
    t.w.resize(static_cast<size_t>(std::max<int64_t>(1, n / 2)));
    const double sgn = inverse ? 1.0 : -1.0;
    for (int64_t k = 0; k < n / 2; ++k) {
      const double a = sgn * 2.0 * kPi * static_cast<double>(k) / static_cast<double>(n);
      t.w[static_cast<size_t>(k)] = cplx(std::cos(a), std::sin(a));
    }
  }
  return t.w;
}

void radix2(std::vector<cplx>& a, bool inverse) {
  const int64_t n = static_cast<int64_t>(a.size());
  int lg = 0;
  while ((int64_t(1) << lg) < n) ++lg;
  for (int64_t i = 0; i < n; ++i) {  // bit-reversal permutation
    int64_t r = 0;
    for (int b = 0; b < lg; ++b) r |= ((i >> b) & 1) << (lg - 1 - b);
    if (i < r) std::swap(a[static_cast<size_t>(i)], a[static_cast<size_t>(r)]);
  }
  const std::vector<cplx>& w = twiddles(n, inverse);
  for (int64_t half = 1; half < n; half <<= 1) {
    const int64_t stride = n / (2 * half);
    for (int64_t base = 0; base < n; base += 2 * half) {
      cplx* lo = a.data() + base;
      cplx* hi = lo + half;
      for (int64_t k = 0; k < half; ++k) {
        const cplx t = hi[k] * w[static_cast<size_t>(k * stride)];
        hi[k] = lo[k] - t;
        lo[k] += t;
      }
    }
  }
}

void bluestein(std::vector<cplx>& a, bool inverse) {
  const int64_t n = static_cast<int64_t>(a.size());
  const double sgn = inverse ? 1.0 : -1.0;
  std::vector<cplx> chirp(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) {
    const int64_t q = (j * j) % (2 * n);  // exact angle reduction
    const double ang = sgn * kPi * static_cast<double>(q) / static_cast<double>(n);
    chirp[static_cast<size_t>(j)] = cplx(std::cos(ang), std::sin(ang));
  }
  int64_t len = 1;
  while (len < 2 * n - 1) len <<= 1;
  std::vector<cplx> f(static_cast<size_t>(len)), g(static_cast<size_t>(len));
  for (int64_t j = 0; j < n; ++j) f[static_cast<size_t>(j)] = a[static_cast<size_t>(j)] * chirp[static_cast<size_t>(j)];
  g[0] = std::conj(chirp[0]);
  for (int64_t j = 1; j < n; ++j)
    g[static_cast<size_t>(j)] = g[static_cast<size_t>(len - j)] = std::conj(chirp[static_cast<size_t>(j)]);
  radix2(f, false);
  radix2(g, false);
  for (int64_t i = 0; i < len; ++i) f[static_cast<size_t>(i)] *= g[static_cast<size_t>(i)];
  radix2(f, true);
  const double scale = 1.0 / static_cast<double>(len);
  for (int64_t k = 0; k < n; ++k)
    a[static_cast<size_t>(k)] = f[static_cast<size_t>(k)] * scale * chirp[static_cast<size_t>(k)];
}
}  // namespace

void set_error(const std::string& msg) { g_error = msg; }
const std::string& last_error() { return g_error; }

void dft_inplace(std::vector<cplx>& a, bool inverse) {
  if (a.size() <= 1) return;
  if (power_of_two(static_cast<int64_t>(a.size()))) radix2(a, inverse);
  else bluestein(a, inverse);
}

std::vector<cplx> dft_real(const double* x, int64_t n) {
  std::vector<cplx> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[static_cast<size_t>(i)] = cplx(x[i], 0.0);
  dft_inplace(out, false);
  return out;
}

void idft_real_checked(std::vector<cplx> f, double* out, double rel_tol) {
  const int64_t n = static_cast<int64_t>(f.size());
  if (n == 0) return;
  dft_inplace(f, true);
  const double inv = 1.0 / static_cast<double>(n);
  double scale = 0.0, residue = 0.0;
  for (auto& v : f) {
    v *= inv;
    scale = std::max(scale, std::abs(v.real()));
    residue = std::max(residue, std::abs(v.imag()));
  }
  if (scale < 1.0) scale = 1.0;
  if (residue > rel_tol * scale) {
    std::ostringstream msg;
    msg << "inverse DFT of a real-valued quantity has imaginary residue " << residue << " (relative tolerance "
        << rel_tol << ")";
    raise(CL_ECONSIST, msg.str());
  }
  for (int64_t i = 0; i < n; ++i) out[i] = f[static_cast<size_t>(i)].real();
}

double spectral_norm(const double* c, int64_t n) {
  if (n < 1) raise(CL_EPARAM, "spectral_norm: empty operator");
  const std::vector<cplx> s = dft_real(c, n);
  double mx = 0.0;
  for (const cplx& v : s) mx = std::max(mx, std::abs(v));
  return mx;
}

void regularized_gram_inverse(const double* c, int64_t n, double rho, double sigma, double* b) {
  if (rho < 0.0 || sigma < 0.0 || (rho == 0.0 && sigma == 0.0))
    raise(CL_EPARAM,
          "regularized_gram_inverse: rho and sigma must be nonnegative with at least one strictly positive");
  std::vector<cplx> s = dft_real(c, n);
  for (int64_t k = 0; k < n; ++k) {
    const double denom = rho * std::norm(s[static_cast<size_t>(k)]) + sigma;
    if (denom < 1e-14) {
      std::ostringstream msg;
      msg << "regularized_gram_inverse: eigenvalue " << k << " of (rho C^T C + sigma I) is " << denom
          << ", below the invertibility floor 1e-14";
      raise(CL_ESINGULAR, msg.str());
    }
    s[static_cast<size_t>(k)] = cplx(1.0 / denom, 0.0);
  }
  idft_real_checked(std::move(s), b);
}

void mask_gram_inverse(const int64_t* omega, int64_t m, int64_t n, double rho, double* d) {
  if (!(rho > 0.0)) raise(CL_EPARAM, "mask_gram_inverse: rho must be positive");
  std::fill(d, d + n, 1.0 / rho);
  for (int64_t t = 0; t < m; ++t) d[omega[t]] = 1.0 / (1.0 + rho);
}

static bool is_identity_row(const double* r, int64_t n) {  // deblur.hpp:41-46
  if (n < 1 || r[0] != 1.0) return false;
  for (int64_t i = 1; i < n; ++i)
    if (r[i] != 0.0) return false;
  return true;
}

void compose_rows(const double* c, const double* b, int64_t n, double* out) {
  if (is_identity_row(b, n)) { std::copy(c, c + n, out); return; }
  if (is_identity_row(c, n)) { std::copy(b, b + n, out); return; }
  std::vector<cplx> sc = dft_real(c, n), sb = dft_real(b, n);
  for (int64_t k = 0; k < n; ++k) sc[static_cast<size_t>(k)] *= sb[static_cast<size_t>(k)];
  idft_real_checked(std::move(sc), out);
}

void measure(const double* c, const int64_t* omega, int64_t n, int64_t m, const double* x, double* y) {
  if (n == 0) return;
  std::vector<cplx> sc = dft_real(c, n), sx = dft_real(x, n);
  for (int64_t k = 0; k < n; ++k) sx[static_cast<size_t>(k)] *= std::conj(sc[static_cast<size_t>(k)]);
  std::vector<double> cx(static_cast<size_t>(n));
  idft_real_checked(std::move(sx), cx.data());
  for (int64_t t = 0; t < m; ++t) y[t] = cx[static_cast<size_t>(omega[t])];
}

void check_mask(const int64_t* omega, int64_t m, int64_t n) {
  if (n < 0) raise(CL_EPARAM, "SubsamplingMask: negative dimension");
  int64_t prev = -1;
  for (int64_t t = 0; t < m; ++t) {
    if (omega[t] <= prev || omega[t] >= n)
      raise(CL_EPARAM, "SubsamplingMask: indices must be strictly increasing and within [0, n)");
    prev = omega[t];
  }
}

}  // namespace clb
