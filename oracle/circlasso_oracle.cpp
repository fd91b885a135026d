// circlasso_oracle.cpp — TEST INFRASTRUCTURE ONLY (the parity checker).
//
// A CPU restatement of the reference `circlasso` hot path (arxiv 1707.02244),
// used ONLY by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// `--impl reference` leg.  The product (paper_1707_02244_b200/, the CUDA
// C-ABI library) never links, imports or calls this file.
//
// Parity pinning.  The reference itself cannot be built here: it is a
// header-only C++20 library on Eigen >= 3.3 (incl. unsupported/Eigen/FFT),
// and neither Eigen nor the vendored CLI11/doctest exist in this image
// (/root/reference/proj/CMakeLists.txt:12-20).  This restatement is pinned
// instead against (a) every known-answer test the reference's own suite
// holds for this path (tests/golden/kats.json, each entry citing its
// reference test file:line) and (b) the C++-standard known answer of
// std::mt19937_64 ([rand.predef]: 10000th output of a default-seeded engine
// is 9981545732273789042), which fixes the RNG stream bit for bit.
//
// Third-party arithmetic boundary: the reference's FFT is Eigen::FFT's
// kissfft backend (Eigen 3.3+, unpinned version).  Its results are only ever
// pinned to tolerance by the reference tests (tests/fft_test.cpp:47-57 at
// 1e-10, tests/parallel_test.cpp:210-213 at 1e-12), so any correct DFT is
// within the reference's own contract.  Here: iterative radix-2 for powers of
// two, Bluestein (chirp-z over a power of two) otherwise.
//
// Rounding.  The reference build sets no -march (x86-64 baseline, no FMA), so
// every a*b+c rounds twice.  This file must be compiled with
// -ffp-contract=off (oracle/Makefile) to reproduce that.
//
// Every function cites the reference file:line it restates.  Paths are
// relative to /root/reference/proj/include/circlasso/ unless noted.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using cd = std::complex<double>;

// Status codes: identical numbering to include/circlasso_b200.h (cl_status).
enum Status {
  OK = 0, EDIM = 1, EPARAM = 2, ESINGULAR = 3, EDIVERGE = 4, ECAPACITY = 5,
  EFORMAT = 6, ECONSIST = 7, EPHASE = 8
};

thread_local std::string g_err;
static int fail(int code, const std::string& msg) { g_err = msg; return code; }

// ---------------------------------------------------------------------------
// RNG — sensing.hpp:35-113
// ---------------------------------------------------------------------------
static inline uint64_t splitmix64(uint64_t x) {  // sensing.hpp:35-40
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
static inline uint64_t derive_seed(uint64_t seed, uint64_t tag) {  // :42-44
  return splitmix64(seed ^ splitmix64(tag));
}
constexpr uint64_t kSignalStream = 0x7369676e616cULL;  // :47 "signal"
constexpr uint64_t kRowStream = 0x726f77ULL;           // :48 "row"
constexpr uint64_t kMaskStream = 0x6d61736bULL;        // :49 "mask"

struct Rng {  // SeededRng, sensing.hpp:56-95
  std::mt19937_64 e;
  double spare = 0.0;
  bool has_spare = false;
  explicit Rng(uint64_t s) : e(s) {}
  double uniform() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }  // :61-63
  double normal() {  // :67-79 Box-Muller with cached spare
    if (has_spare) { has_spare = false; return spare; }
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    spare = radius * std::sin(angle);
    has_spare = true;
    return radius * std::cos(angle);
  }
  uint64_t uniform_below(uint64_t bound) {  // :82-89 (bound > 0 checked by caller)
    const uint64_t limit = ~uint64_t(0) - (~uint64_t(0) % bound);
    uint64_t draw = e();
    while (draw >= limit) draw = e();
    return draw % bound;
  }
};

// Partial Fisher-Yates k-subset of [0, n), sorted — sensing.hpp:100-113
static std::vector<int64_t> sample_subset(int64_t n, int64_t k, Rng& rng) {
  std::vector<int64_t> pool(static_cast<size_t>(n));
  std::iota(pool.begin(), pool.end(), int64_t(0));
  for (int64_t i = 0; i < k; ++i) {
    const int64_t j = i + static_cast<int64_t>(rng.uniform_below(static_cast<uint64_t>(n - i)));
    std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
  }
  pool.resize(static_cast<size_t>(k));
  std::sort(pool.begin(), pool.end());
  return pool;
}

// ---------------------------------------------------------------------------
// FFT — fft.hpp:46-89 semantics (full complex spectrum of real input; inverse
// includes 1/n; idft_real residue check).
// ---------------------------------------------------------------------------
static bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

static void fft_pow2(std::vector<cd>& a, bool inverse) {
  const size_t n = a.size();
  for (size_t i = 1, j = 0; i < n; ++i) {  // bit reversal
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  std::vector<cd> tw(n / 2 > 0 ? n / 2 : 1);
  const double sgn = inverse ? 1.0 : -1.0;
  for (size_t k = 0; k < n / 2; ++k) {
    const double ang = sgn * 2.0 * 3.14159265358979323846 * static_cast<double>(k) / static_cast<double>(n);
    tw[k] = cd(std::cos(ang), std::sin(ang));
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t half = len >> 1, step = n / len;
    for (size_t i = 0; i < n; i += len)
      for (size_t k = 0; k < half; ++k) {
        const cd u = a[i + k];
        const cd v = a[i + k + half] * tw[k * step];
        a[i + k] = u + v;
        a[i + k + half] = u - v;
      }
  }
}

// Unnormalized DFT (sign -1 forward, +1 inverse) of arbitrary length.
static void dft_any(std::vector<cd>& a, bool inverse) {
  const int64_t n = static_cast<int64_t>(a.size());
  if (n <= 1) return;
  if (is_pow2(n)) { fft_pow2(a, inverse); return; }
  // Bluestein: X_k = conj(w_k) * sum_j (x_j conj(w_j)) w_{k-j}, w_j = e^{i pi j^2/n}
  const double sgn = inverse ? 1.0 : -1.0;
  std::vector<cd> w(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) {
    const int64_t jj = (j * j) % (2 * n);
    const double ang = sgn * 3.14159265358979323846 * static_cast<double>(jj) / static_cast<double>(n);
    w[static_cast<size_t>(j)] = cd(std::cos(ang), std::sin(ang));
  }
  int64_t m = 1;
  while (m < 2 * n - 1) m <<= 1;
  std::vector<cd> A(static_cast<size_t>(m)), B(static_cast<size_t>(m));
  for (int64_t j = 0; j < n; ++j) A[static_cast<size_t>(j)] = a[static_cast<size_t>(j)] * w[static_cast<size_t>(j)];
  B[0] = std::conj(w[0]);
  for (int64_t j = 1; j < n; ++j) B[static_cast<size_t>(j)] = B[static_cast<size_t>(m - j)] = std::conj(w[static_cast<size_t>(j)]);
  fft_pow2(A, false);
  fft_pow2(B, false);
  for (int64_t i = 0; i < m; ++i) A[static_cast<size_t>(i)] *= B[static_cast<size_t>(i)];
  fft_pow2(A, true);
  const double inv_m = 1.0 / static_cast<double>(m);
  for (int64_t k = 0; k < n; ++k) a[static_cast<size_t>(k)] = A[static_cast<size_t>(k)] * inv_m * w[static_cast<size_t>(k)];
}

static std::vector<cd> dft(const double* x, int64_t n) {  // fft.hpp:46-56
  std::vector<cd> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[static_cast<size_t>(i)] = cd(x[i], 0.0);
  dft_any(out, false);
  return out;
}

static std::vector<cd> idft(std::vector<cd> f) {  // fft.hpp:59-69 (includes 1/n)
  const int64_t n = static_cast<int64_t>(f.size());
  if (n <= 1) return f;
  dft_any(f, true);
  const double inv = 1.0 / static_cast<double>(n);
  for (auto& v : f) v *= inv;
  return f;
}

// fft.hpp:74-89: imaginary residue above rel_tol*max(1, |re|_inf) -> ConsistencyError
static int idft_real(const std::vector<cd>& f, double* out, double rel_tol = 1e-10) {
  const std::vector<cd> t = idft(f);
  if (t.empty()) return OK;
  double scale = 0.0, residue = 0.0;
  for (const cd& v : t) { scale = std::max(scale, std::abs(v.real())); residue = std::max(residue, std::abs(v.imag())); }
  if (scale < 1.0) scale = 1.0;
  if (residue > rel_tol * scale)
    return fail(ECONSIST, "inverse DFT of a real-valued quantity has imaginary residue " + std::to_string(residue));
  for (size_t i = 0; i < t.size(); ++i) out[i] = t[i].real();
  return OK;
}

// ---------------------------------------------------------------------------
// Operators — circulant.hpp:214-351
// ---------------------------------------------------------------------------
static double spectral_norm(const double* c, int64_t n) {  // circulant.hpp:347-351
  const std::vector<cd> s = dft(c, n);
  double mx = 0.0;
  for (const cd& v : s) mx = std::max(mx, std::abs(v));
  return mx;
}

// circulant.hpp:297-320: b = idft(1 / (rho |c_k|^2 + sigma)), floor 1e-14
static int regularized_gram_inverse(const double* c, int64_t n, double rho, double sigma, double* b) {
  if (rho < 0.0 || sigma < 0.0 || (rho == 0.0 && sigma == 0.0))
    return fail(EPARAM, "regularized_gram_inverse: rho and sigma must be nonnegative with at least one strictly positive");
  const std::vector<cd> s = dft(c, n);
  std::vector<cd> inv(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) {
    const double denom = rho * std::norm(s[static_cast<size_t>(k)]) + sigma;
    if (denom < 1e-14)
      return fail(ESINGULAR, "regularized_gram_inverse: eigenvalue " + std::to_string(k) + " below the invertibility floor 1e-14");
    inv[static_cast<size_t>(k)] = cd(1.0 / denom, 0.0);
  }
  return idft_real(inv, b);
}

// circulant.hpp:324-333
static int mask_gram_inverse(const int64_t* omega, int64_t m, int64_t n, double rho, double* d) {
  if (!(rho > 0.0)) return fail(EPARAM, "mask_gram_inverse: rho must be positive");
  for (int64_t i = 0; i < n; ++i) d[i] = 1.0 / rho;
  for (int64_t t = 0; t < m; ++t) d[omega[t]] = 1.0 / (1.0 + rho);
  return OK;
}

// circulant.hpp:337-343: first row of C*B = idft(c_hat . b_hat)
static int circ_compose(const double* c, const double* b, int64_t n, double* out) {
  std::vector<cd> sc = dft(c, n), sb = dft(b, n);
  for (int64_t k = 0; k < n; ++k) sc[static_cast<size_t>(k)] *= sb[static_cast<size_t>(k)];
  return idft_real(sc, out);
}

// circulant.hpp:216-232: y[i] = sum_j c[(j-i) mod n] x[j], ascending j
static void circ_matvec_naive(const double* c, const double* x, int64_t n, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) acc += c[j >= i ? j - i : j - i + n] * x[j];
    y[i] = acc;
  }
}
// circulant.hpp:248-264: y[i] = sum_j c[(i-j) mod n] x[j]
static void circ_transpose_matvec_naive(const double* c, const double* x, int64_t n, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) acc += c[i >= j ? i - j : i - j + n] * x[j];
    y[i] = acc;
  }
}
// circulant.hpp:236-244 (transpose=false: conj(c_hat) . x_hat) and :267-274
static int circ_matvec_fft(const std::vector<cd>& chat, const double* x, int64_t n, bool transpose, double* y) {
  if (n == 0) return OK;
  std::vector<cd> xh = dft(x, n);
  for (int64_t k = 0; k < n; ++k)
    xh[static_cast<size_t>(k)] *= transpose ? chat[static_cast<size_t>(k)] : std::conj(chat[static_cast<size_t>(k)]);
  return idft_real(xh, y);
}

// solvers.hpp:39-44 (strict; NaN -> 0)
static inline double soft(double v, double g) {
  if (v > g) return v - g;
  if (v < -g) return v + g;
  return 0.0;
}

// ---------------------------------------------------------------------------
// Fork/join over contiguous output chunks — parallel.hpp:64-126.  Each output
// is computed by exactly one thread with a self-contained ascending loop, so
// results are bitwise independent of the thread count (parallel.hpp:4-8).
// ---------------------------------------------------------------------------
template <typename F>
static void parallel_for(int64_t total, int threads, F body) {
  if (total <= 0) return;
  const int workers = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, total)));
  if (workers == 1) { body(int64_t(0), total); return; }
  std::vector<std::thread> pool;
  const int64_t chunk = (total + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const int64_t b = w * chunk, e = std::min(b + chunk, total);
    if (b >= e) break;
    pool.emplace_back([=] { body(b, e); });
  }
  for (auto& t : pool) t.join();
}

// ---------------------------------------------------------------------------
// ISTA — solvers.hpp:208-263 (state/setup/step), phases parallel.hpp:236-279
// ---------------------------------------------------------------------------
struct Ista {
  int64_t n = 0, m = 0;
  std::vector<double> c;     // normalized first row c/s
  std::vector<int64_t> omega;
  std::vector<double> y;     // normalized measurements y/s
  double tau = 0.0, threshold = 0.0, s = 1.0;
  std::vector<double> x, r, delta;
  std::vector<cd> chat;      // spectrum of c (FFT engine only)
  long t = 0;
};

struct Cadmm {  // solvers.hpp:337-357
  int64_t n = 0, m = 0;
  std::vector<double> c, b, d, pty;
  std::vector<int64_t> omega;
  double rho = 0, sigma = 0, tau1 = 1, tau2 = 1, threshold = 0, s = 1.0;
  std::vector<double> x, z, nu, mu, v, beta;
  std::vector<cd> chat, bhat;
  long t = 0;
};

// solvers.hpp:170-183
static int normalization(const double* c, int64_t n, const double* y, int64_t m, double* s_out) {
  for (int64_t i = 0; i < m; ++i)
    if (!std::isfinite(y[i])) return fail(EDIVERGE, "solver: measurements contain non-finite entries");
  if (n < 1) return fail(EPARAM, "spectral_norm: empty operator");
  const double s = spectral_norm(c, n);
  if (s > 0.0) { *s_out = s; return OK; }
  double mx = 0.0;
  for (int64_t i = 0; i < m; ++i) mx = std::max(mx, std::abs(y[i]));
  if (m == 0 || mx == 0.0) { *s_out = 1.0; return OK; }
  return fail(ESINGULAR, "solver: sensing operator is zero but measurements are not");
}

static int check_mask(const int64_t* omega, int64_t m, int64_t n) {  // circulant.hpp:134-146
  int64_t prev = -1;
  for (int64_t t = 0; t < m; ++t) {
    if (omega[t] <= prev || omega[t] >= n)
      return fail(EPARAM, "SubsamplingMask: indices must be strictly increasing and within [0, n)");
    prev = omega[t];
  }
  return OK;
}

// ista_setup solvers.hpp:222-249
static int ista_setup(Ista& st, int64_t n, int64_t m, const double* c, const int64_t* omega, const double* y,
                      double alpha, double tau_cfg, int proximal) {
  if (int rc = check_mask(omega, m, n)) return rc;
  double tau = tau_cfg;
  if (tau == 0.0) tau = 0.9;
  if (!(tau > 0.0) || !(tau < 1.0))
    return fail(EPARAM, "ista_setup: tau must lie in (0, |A|^-2); on the normalized operator the admissible range is (0, 1)");
  if (!(alpha > 0.0)) return fail(EPARAM, "ista_setup: alpha must be > 0");
  double s = 1.0;
  if (int rc = normalization(c, n, y, m, &s)) return rc;
  st.n = n; st.m = m; st.s = s;
  st.c.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) st.c[static_cast<size_t>(i)] = c[i] / s;
  st.omega.assign(omega, omega + m);
  st.y.resize(static_cast<size_t>(m));
  for (int64_t i = 0; i < m; ++i) st.y[static_cast<size_t>(i)] = y[i] / s;
  st.tau = tau;
  st.threshold = proximal ? tau * alpha : alpha;
  st.x.assign(static_cast<size_t>(n), 0.0);
  st.r.assign(static_cast<size_t>(m), 0.0);
  st.delta.assign(static_cast<size_t>(n), 0.0);
  st.t = 0;
  return OK;
}

// cpista_phases: residual phase parallel.hpp:243-256, gradient phase :258-276.
// The inner loops are split at the wrap point instead of branching per
// element (circ_entry :161-166); the accumulation order is unchanged.
// rows_hi / outs_hi < m / n restrict the phases to a leading sample of their
// outputs (timing only: bench.py's CPU baseline); phase_s receives the wall
// time of each phase.
static void ista_step_phases(Ista& st, int threads, int64_t rows_hi = -1, int64_t outs_hi = -1,
                             double* phase_s = nullptr) {
  const int64_t n = st.n, m = st.m;
  const double* c = st.c.data();
  const double* x = st.x.data();
  const auto t0 = std::chrono::steady_clock::now();
  parallel_for(rows_hi < 0 ? m : rows_hi, threads, [&](int64_t b, int64_t e) {
    for (int64_t t = b; t < e; ++t) {
      const int64_t w = st.omega[static_cast<size_t>(t)];
      double acc = 0.0;
      for (int64_t j = 0; j < w; ++j) acc += c[j - w + n] * x[j];
      for (int64_t j = w; j < n; ++j) acc += c[j - w] * x[j];
      st.r[static_cast<size_t>(t)] = st.y[static_cast<size_t>(t)] - acc;
    }
  });
  const auto t1 = std::chrono::steady_clock::now();
  const double* r = st.r.data();
  const int64_t* om = st.omega.data();
  parallel_for(outs_hi < 0 ? n : outs_hi, threads, [&](int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) {
      double acc = 0.0;
      for (int64_t t = 0; t < m; ++t) {
        const int64_t w = om[t];
        acc += c[i >= w ? i - w : i - w + n] * r[t];
      }
      st.delta[static_cast<size_t>(i)] = acc;
      st.x[static_cast<size_t>(i)] = soft(st.x[static_cast<size_t>(i)] + st.tau * acc, st.threshold);
    }
  });
  if (phase_s) {
    const auto t2 = std::chrono::steady_clock::now();
    phase_s[0] = std::chrono::duration<double>(t1 - t0).count();
    phase_s[1] = std::chrono::duration<double>(t2 - t1).count();
  }
  ++st.t;
}

// ista_step with use_fft=true: solvers.hpp:252-263 over circulant.hpp:236-274
static int ista_step_fft(Ista& st) {
  const int64_t n = st.n, m = st.m;
  if (st.chat.empty() && n > 0) st.chat = dft(st.c.data(), n);
  std::vector<double> cx(static_cast<size_t>(n)), emb(static_cast<size_t>(n), 0.0);
  if (int rc = circ_matvec_fft(st.chat, st.x.data(), n, false, cx.data())) return rc;
  for (int64_t t = 0; t < m; ++t) st.r[static_cast<size_t>(t)] = st.y[static_cast<size_t>(t)] - cx[static_cast<size_t>(st.omega[static_cast<size_t>(t)])];
  for (int64_t t = 0; t < m; ++t) emb[static_cast<size_t>(st.omega[static_cast<size_t>(t)])] = st.r[static_cast<size_t>(t)];
  if (int rc = circ_matvec_fft(st.chat, emb.data(), n, true, st.delta.data())) return rc;
  for (int64_t i = 0; i < n; ++i)
    st.x[static_cast<size_t>(i)] = soft(st.x[static_cast<size_t>(i)] + st.tau * st.delta[static_cast<size_t>(i)], st.threshold);
  ++st.t;
  return OK;
}

// cadmm_setup solvers.hpp:359-395
static int cadmm_setup(Cadmm& st, int64_t n, int64_t m, const double* c, const int64_t* omega, const double* y,
                       double alpha, double rho, double sigma, double tau1, double tau2) {
  if (int rc = check_mask(omega, m, n)) return rc;
  if (!(rho > 0.0) || !(sigma > 0.0)) return fail(EPARAM, "cadmm_setup: rho and sigma must be > 0");
  if (!(alpha > 0.0)) return fail(EPARAM, "cadmm_setup: alpha must be > 0");
  constexpr double kGolden = 1.6180339887498949;
  if (!(tau1 > 0.0) || tau1 >= kGolden || !(tau2 > 0.0) || tau2 >= kGolden)
    return fail(EPARAM, "cadmm_setup: tau1 and tau2 must lie in (0, (sqrt(5)+1)/2)");
  double s = 1.0;
  if (int rc = normalization(c, n, y, m, &s)) return rc;
  st.n = n; st.m = m; st.s = s;
  st.c.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) st.c[static_cast<size_t>(i)] = c[i] / s;
  st.omega.assign(omega, omega + m);
  st.b.resize(static_cast<size_t>(n));
  if (int rc = regularized_gram_inverse(st.c.data(), n, rho, sigma, st.b.data())) return rc;
  st.d.resize(static_cast<size_t>(n));
  if (int rc = mask_gram_inverse(omega, m, n, rho, st.d.data())) return rc;
  st.pty.assign(static_cast<size_t>(n), 0.0);
  for (int64_t t = 0; t < m; ++t) st.pty[static_cast<size_t>(omega[t])] = y[t] / s;
  st.rho = rho; st.sigma = sigma; st.tau1 = tau1; st.tau2 = tau2;
  st.threshold = alpha / sigma;
  for (auto* v : {&st.x, &st.z, &st.nu, &st.mu, &st.v, &st.beta}) v->assign(static_cast<size_t>(n), 0.0);
  st.t = 0;
  return OK;
}

// cpadmm_phases parallel.hpp:173-231 (primal :178-191, recovery :193-205, duals :207-228)
static void cadmm_step_phases(Cadmm& st, int threads, int64_t outs_hi = -1, double* phase_s = nullptr) {
  const int64_t n = st.n;
  const int64_t nh = outs_hi < 0 ? n : outs_hi;
  const double* c = st.c.data();
  const double* b = st.b.data();
  const auto t0 = std::chrono::steady_clock::now();
  parallel_for(nh, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {  // acc += c[(i-j) mod n] * v[j]   (circ_entry(row, j, i))
      double acc = 0.0;
      for (int64_t j = 0; j <= i; ++j) acc += c[i - j] * st.v[static_cast<size_t>(j)];
      for (int64_t j = i + 1; j < n; ++j) acc += c[i - j + n] * st.v[static_cast<size_t>(j)];
      st.beta[static_cast<size_t>(i)] = st.rho * acc + st.sigma * (st.z[static_cast<size_t>(i)] - st.nu[static_cast<size_t>(i)]);
    }
  });
  const auto t1 = std::chrono::steady_clock::now();
  parallel_for(nh, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {  // acc += b[(j-i) mod n] * beta[j]
      double acc = 0.0;
      for (int64_t j = 0; j < i; ++j) acc += b[j - i + n] * st.beta[static_cast<size_t>(j)];
      for (int64_t j = i; j < n; ++j) acc += b[j - i] * st.beta[static_cast<size_t>(j)];
      st.x[static_cast<size_t>(i)] = acc;
    }
  });
  const auto t2 = std::chrono::steady_clock::now();
  parallel_for(nh, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      double cx = 0.0;
      for (int64_t j = 0; j < i; ++j) cx += c[j - i + n] * st.x[static_cast<size_t>(j)];
      for (int64_t j = i; j < n; ++j) cx += c[j - i] * st.x[static_cast<size_t>(j)];
      const size_t k = static_cast<size_t>(i);
      const double v_new = st.d[k] * (st.rho * (cx - st.mu[k]) + st.pty[k]);
      st.z[k] = soft(st.x[k] + st.nu[k], st.threshold);
      st.mu[k] += st.tau1 * (v_new - cx);
      st.nu[k] += st.tau2 * (st.x[k] - st.z[k]);
      st.v[k] = v_new + st.mu[k];
    }
  });
  if (phase_s) {
    const auto t3 = std::chrono::steady_clock::now();
    phase_s[0] = std::chrono::duration<double>(t1 - t0).count();
    phase_s[1] = std::chrono::duration<double>(t2 - t1).count();
    phase_s[2] = std::chrono::duration<double>(t3 - t2).count();
  }
  ++st.t;
}

// cadmm_step with use_fft=true: solvers.hpp:399-415
static int cadmm_step_fft(Cadmm& st) {
  const int64_t n = st.n;
  if (st.chat.empty() && n > 0) st.chat = dft(st.c.data(), n);
  if (st.bhat.empty() && n > 0) st.bhat = dft(st.b.data(), n);
  std::vector<double> ctv(static_cast<size_t>(n)), cx(static_cast<size_t>(n));
  if (int rc = circ_matvec_fft(st.chat, st.v.data(), n, true, ctv.data())) return rc;
  for (int64_t i = 0; i < n; ++i) {
    const size_t k = static_cast<size_t>(i);
    st.beta[k] = st.rho * ctv[k] + st.sigma * (st.z[k] - st.nu[k]);
  }
  if (int rc = circ_matvec_fft(st.bhat, st.beta.data(), n, false, st.x.data())) return rc;
  if (int rc = circ_matvec_fft(st.chat, st.x.data(), n, false, cx.data())) return rc;
  for (int64_t i = 0; i < n; ++i) {
    const size_t k = static_cast<size_t>(i);
    st.v[k] = st.d[k] * (st.rho * (cx[k] - st.mu[k]) + st.pty[k]);
  }
  for (int64_t i = 0; i < n; ++i) {
    const size_t k = static_cast<size_t>(i);
    st.z[k] = soft(st.x[k] + st.nu[k], st.threshold);
  }
  for (int64_t i = 0; i < n; ++i) { const size_t k = static_cast<size_t>(i); st.mu[k] += st.tau1 * (st.v[k] - cx[k]); }
  for (int64_t i = 0; i < n; ++i) { const size_t k = static_cast<size_t>(i); st.nu[k] += st.tau2 * (st.x[k] - st.z[k]); }
  for (int64_t i = 0; i < n; ++i) { const size_t k = static_cast<size_t>(i); st.v[k] += st.mu[k]; }
  ++st.t;
  return OK;
}

// ---------------------------------------------------------------------------
// Dense ADMM — solvers.hpp:267-327 (AdmmState, admm_setup, admm_step), phases
// parallel.hpp:284-317 (padmm_phases), run solvers.hpp:497-514.  The paper's
// dense baseline: (A^T A + rho I)^-1 stored as an explicit n x n matrix.
// ---------------------------------------------------------------------------
struct Admm {
  int64_t n = 0, m = 0;
  std::vector<double> B;    // n x n row-major, (A~^T A~ + rho I)^-1
  std::vector<double> aty;  // A~^T y~
  double rho = 0, threshold = 0, s = 1.0;
  std::vector<double> x, z, u, rhs;
  long t = 0;
};

// admm_setup solvers.hpp:285-314.  The reference factors the Gram matrix with
// Eigen::LLT and solves against the identity; restated as a plain Cholesky
// (lower L, G = L L^T) and one forward + back substitution per column.
static int admm_setup(Admm& st, int64_t n, int64_t m, const double* c, const int64_t* omega, const double* y,
                      double alpha, double rho, int64_t dense_cap, int threads) {
  if (int rc = check_mask(omega, m, n)) return rc;
  if (n > dense_cap)  // (no iostreams in this library: it is loaded into processes with other libstdc++ users)
    return fail(ECAPACITY, "admm_setup: n = " + std::to_string(n) + " exceeds the dense cap " + std::to_string(dense_cap));
  if (!(rho > 0.0)) return fail(EPARAM, "admm_setup: rho must be > 0");
  if (!(alpha > 0.0)) return fail(EPARAM, "admm_setup: alpha must be > 0");
  double s = 1.0;
  if (int rc = normalization(c, n, y, m, &s)) return rc;
  const size_t N = static_cast<size_t>(n);
  // A~ = dense_materialize(A) / s (circulant.hpp:382-394): A~[t][j] = c[(j - omega_t) mod n] / s
  std::vector<double> ad(static_cast<size_t>(m) * N);
  for (int64_t t = 0; t < m; ++t)
    for (int64_t j = 0; j < n; ++j) {
      const int64_t w = omega[t];
      ad[static_cast<size_t>(t) * N + static_cast<size_t>(j)] = c[j >= w ? j - w : j - w + n] / s;
    }
  // gram = A~^T A~ + rho I
  std::vector<double> g(N * N);
  parallel_for(n, threads, [&](int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i)
      for (int64_t j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int64_t t = 0; t < m; ++t)
          acc += ad[static_cast<size_t>(t) * N + static_cast<size_t>(i)] * ad[static_cast<size_t>(t) * N + static_cast<size_t>(j)];
        g[static_cast<size_t>(i) * N + static_cast<size_t>(j)] = acc + (i == j ? rho : 0.0);
      }
  });
  // Cholesky, lower triangle in place
  for (int64_t k = 0; k < n; ++k) {
    double d = g[static_cast<size_t>(k) * N + static_cast<size_t>(k)];
    for (int64_t p = 0; p < k; ++p) d -= g[static_cast<size_t>(k) * N + static_cast<size_t>(p)] * g[static_cast<size_t>(k) * N + static_cast<size_t>(p)];
    if (!(d > 0.0)) return fail(ESINGULAR, "admm_setup: Gram matrix is not positive definite");
    const double lkk = std::sqrt(d);
    g[static_cast<size_t>(k) * N + static_cast<size_t>(k)] = lkk;
    parallel_for(n - k - 1, threads, [&](int64_t b, int64_t e) {
      for (int64_t i = k + 1 + b; i < k + 1 + e; ++i) {
        double acc = g[static_cast<size_t>(i) * N + static_cast<size_t>(k)];
        for (int64_t p = 0; p < k; ++p) acc -= g[static_cast<size_t>(i) * N + static_cast<size_t>(p)] * g[static_cast<size_t>(k) * N + static_cast<size_t>(p)];
        g[static_cast<size_t>(i) * N + static_cast<size_t>(k)] = acc / lkk;
      }
    });
  }
  // B = (L L^T)^-1 I, column by column
  st.B.assign(N * N, 0.0);
  parallel_for(n, threads, [&](int64_t b, int64_t e) {
    std::vector<double> w(N);
    for (int64_t col = b; col < e; ++col) {
      for (int64_t i = 0; i < n; ++i) {  // L w = e_col
        double acc = i == col ? 1.0 : 0.0;
        for (int64_t p = 0; p < i; ++p) acc -= g[static_cast<size_t>(i) * N + static_cast<size_t>(p)] * w[static_cast<size_t>(p)];
        w[static_cast<size_t>(i)] = acc / g[static_cast<size_t>(i) * N + static_cast<size_t>(i)];
      }
      for (int64_t i = n - 1; i >= 0; --i) {  // L^T b = w
        double acc = w[static_cast<size_t>(i)];
        for (int64_t p = i + 1; p < n; ++p) acc -= g[static_cast<size_t>(p) * N + static_cast<size_t>(i)] * w[static_cast<size_t>(p)];
        w[static_cast<size_t>(i)] = acc / g[static_cast<size_t>(i) * N + static_cast<size_t>(i)];
      }
      for (int64_t i = 0; i < n; ++i) st.B[static_cast<size_t>(i) * N + static_cast<size_t>(col)] = w[static_cast<size_t>(i)];
    }
  });
  st.aty.assign(N, 0.0);  // A~^T (y / s)
  for (int64_t j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int64_t t = 0; t < m; ++t) acc += ad[static_cast<size_t>(t) * N + static_cast<size_t>(j)] * (y[t] / s);
    st.aty[static_cast<size_t>(j)] = acc;
  }
  st.n = n; st.m = m; st.s = s; st.rho = rho;
  st.threshold = alpha / rho;
  st.x.assign(N, 0.0);
  st.z.assign(N, 0.0);
  st.u.assign(N, 0.0);
  st.rhs = st.aty;
  st.t = 0;
  return OK;
}

// padmm_phases (parallel.hpp:284-317) == admm_step (solvers.hpp:318-327):
// primal x_i = sum_j B(i, j) rhs_j ascending, z_i = eta(x_i + u_i), u_i += x_i - z_i;
// then rhs_i = A~^T y~_i + rho (z_i - u_i)
static void admm_step_phases(Admm& st, int threads) {
  const int64_t n = st.n;
  const size_t N = static_cast<size_t>(n);
  parallel_for(n, threads, [&](int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) {
      const size_t k = static_cast<size_t>(i);
      double acc = 0.0;
      for (int64_t j = 0; j < n; ++j) acc += st.B[k * N + static_cast<size_t>(j)] * st.rhs[static_cast<size_t>(j)];
      st.x[k] = acc;
      st.z[k] = soft(acc + st.u[k], st.threshold);
      st.u[k] += acc - st.z[k];
    }
  });
  for (int64_t i = 0; i < n; ++i) {
    const size_t k = static_cast<size_t>(i);
    st.rhs[k] = st.aty[k] + st.rho * (st.z[k] - st.u[k]);
  }
  ++st.t;
}

}  // namespace orc

// ===========================================================================
// extern "C" surface for tests/ (ctypes).  Engines: 0 = phases (direct,
// threaded; bitwise equal to the reference's naive steps), 1 = FFT (the
// reference default, use_fft=true).
// ===========================================================================
using namespace orc;

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

uint64_t orc_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t orc_derive_seed(uint64_t s, uint64_t tag) { return derive_seed(s, tag); }

// Raw mt19937_64 draws (KAT pinning of the engine).
void orc_mt19937_64(uint64_t seed, int64_t count, uint64_t* out) {
  std::mt19937_64 e(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = e();
}
// SeededRng draws: kind 0 uniform, 1 normal, 2 uniform_below(bound)
int orc_rng_draws(uint64_t seed, int kind, uint64_t bound, int64_t count, double* out) {
  if (kind == 2 && bound == 0) return fail(EPARAM, "SeededRng::uniform_below: bound must be > 0");
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i)
    out[i] = kind == 0 ? r.uniform() : kind == 1 ? r.normal() : static_cast<double>(r.uniform_below(bound));
  return OK;
}

// gen_sparse_signal sensing.hpp:129-145
int orc_gen_sparse_signal(int64_t n, int64_t k, uint64_t seed, double* values, int64_t* support) {
  if (n < 0 || k < 0 || k > n) return fail(EPARAM, "gen_sparse_signal: need 0 <= k <= n");
  Rng rng(derive_seed(seed, kSignalStream));
  std::vector<int64_t> sup = sample_subset(n, k, rng);
  for (int64_t i = 0; i < n; ++i) values[i] = 0.0;
  for (size_t i = 0; i < sup.size(); ++i) { support[i] = sup[i]; values[sup[i]] = rng.normal(); }
  return OK;
}

// gen_circulant_sensing sensing.hpp:149-168
int orc_gen_circulant_sensing(int64_t n, int64_t m, uint64_t seed, double* row, int64_t* omega) {
  if (m < 1 || m > n) return fail(EPARAM, "gen_circulant_sensing: need 1 <= m <= n");
  Rng rr(derive_seed(seed, kRowStream));
  for (int64_t i = 0; i < n; ++i) row[i] = rr.normal();
  Rng mr(derive_seed(seed, kMaskStream));
  std::vector<int64_t> om = sample_subset(n, m, mr);
  std::copy(om.begin(), om.end(), omega);
  return OK;
}

// measure sensing.hpp:171-176 -> partial_matvec circulant.hpp:277-282 (FFT path)
int orc_measure(int64_t n, int64_t m, const double* row, const int64_t* omega, const double* x, double* y) {
  std::vector<cd> chat = dft(row, n);
  std::vector<double> cx(static_cast<size_t>(n));
  if (int rc = circ_matvec_fft(chat, x, n, false, cx.data())) return rc;
  for (int64_t t = 0; t < m; ++t) y[t] = cx[static_cast<size_t>(omega[t])];
  return OK;
}

// make_problem sensing.hpp:198-207
int orc_make_problem(int64_t n, int64_t m, int64_t k, uint64_t seed, double* row, int64_t* omega,
                     double* xtrue, int64_t* support, double* y) {
  if (int rc = orc_gen_sparse_signal(n, k, seed, xtrue, support)) return rc;
  if (int rc = orc_gen_circulant_sensing(n, m, seed, row, omega)) return rc;
  return orc_measure(n, m, row, omega, xtrue, y);
}

// gen_star_field deblur.hpp:69-86
int orc_gen_star_field(int64_t width, int64_t height, double density, uint64_t seed, double* pixels) {
  if (width < 1 || height < 1) return fail(EPARAM, "gen_star_field: dimensions must be positive");
  if (!(density >= 0.0) || !(density <= 1.0)) return fail(EPARAM, "gen_star_field: density must lie in [0, 1]");
  const int64_t n = width * height;
  const auto k = static_cast<int64_t>(density * static_cast<double>(n));
  Rng rng(derive_seed(seed, kSignalStream));
  for (int64_t i = 0; i < n; ++i) pixels[i] = 0.0;
  for (int64_t idx : sample_subset(n, k, rng)) pixels[idx] = 0.3 + 0.7 * rng.uniform();
  return OK;
}

// blur_matrix deblur.hpp:26-36
int orc_blur_row(int64_t n, int64_t L, double* row) {
  if (L < 1 || L > n) return fail(EPARAM, "blur_matrix: need 1 <= L <= n");
  for (int64_t i = 0; i < n; ++i) row[i] = i < L ? 1.0 / static_cast<double>(L) : 0.0;
  return OK;
}

int orc_dft(int64_t n, const double* x, double* re, double* im) {
  std::vector<cd> f = dft(x, n);
  for (int64_t k = 0; k < n; ++k) { re[k] = f[static_cast<size_t>(k)].real(); im[k] = f[static_cast<size_t>(k)].imag(); }
  return OK;
}
int orc_idft(int64_t n, const double* re, const double* im, double* ore, double* oim) {
  std::vector<cd> f(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) f[static_cast<size_t>(k)] = cd(re[k], im[k]);
  f = idft(f);
  for (int64_t k = 0; k < n; ++k) { ore[k] = f[static_cast<size_t>(k)].real(); oim[k] = f[static_cast<size_t>(k)].imag(); }
  return OK;
}
int orc_idft_real(int64_t n, const double* re, const double* im, double rel_tol, double* out) {
  std::vector<cd> f(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) f[static_cast<size_t>(k)] = cd(re[k], im[k]);
  return idft_real(f, out, rel_tol);
}
int orc_spectral_norm(int64_t n, const double* c, double* out) {
  if (n < 1) return fail(EPARAM, "spectral_norm: empty operator");
  *out = spectral_norm(c, n);
  return OK;
}
int orc_regularized_gram_inverse(int64_t n, const double* c, double rho, double sigma, double* b) {
  return regularized_gram_inverse(c, n, rho, sigma, b);
}
int orc_mask_gram_inverse(int64_t n, int64_t m, const int64_t* omega, double rho, double* d) {
  if (int rc = check_mask(omega, m, n)) return rc;
  return mask_gram_inverse(omega, m, n, rho, d);
}
int orc_circ_compose(int64_t n, const double* c, const double* b, double* out) { return circ_compose(c, b, n, out); }
int orc_circ_matvec(int64_t n, const double* c, const double* x, int transpose, int use_fft, double* y) {
  if (use_fft) return circ_matvec_fft(dft(c, n), x, n, transpose != 0, y);
  if (transpose) circ_transpose_matvec_naive(c, x, n, y); else circ_matvec_naive(c, x, n, y);
  return OK;
}
double orc_soft_threshold(double v, double g) { return soft(v, g); }

// ---- ISTA handle ----------------------------------------------------------
void* orc_ista_setup(int64_t n, int64_t m, const double* c, const int64_t* omega, const double* y,
                     double alpha, double tau, int proximal, int* status) {
  auto* st = new Ista();
  const int rc = ista_setup(*st, n, m, c, omega, y, alpha, tau, proximal);
  *status = rc;
  if (rc) { delete st; return nullptr; }
  return st;
}
int orc_ista_step(void* h, int64_t iters, int engine, int threads) {
  auto* st = static_cast<Ista*>(h);
  for (int64_t k = 0; k < iters; ++k) {
    if (engine == 1) { if (int rc = ista_step_fft(*st)) return rc; }
    else ista_step_phases(*st, threads);
  }
  return OK;
}
// Timing sample of the phase engine (bench CPU baseline): the residual phase
// over rows [0, rows), the gradient phase over outputs [0, outs).
int orc_ista_phase_sample(void* h, int64_t rows, int64_t outs, int threads, double* phase_s) {
  auto* st = static_cast<Ista*>(h);
  if (rows < 0 || rows > st->m || outs < 0 || outs > st->n) return fail(EPARAM, "orc_ista_phase_sample: bad range");
  ista_step_phases(*st, threads, rows, outs, phase_s);
  return OK;
}
// which: 0 x, 1 r, 2 delta, 3 c~, 4 y~
int orc_ista_get(void* h, int which, double* out) {
  auto* st = static_cast<Ista*>(h);
  const std::vector<double>* v = which == 0 ? &st->x : which == 1 ? &st->r : which == 2 ? &st->delta : which == 3 ? &st->c : &st->y;
  std::copy(v->begin(), v->end(), out);
  return OK;
}
void orc_ista_scalars(void* h, double* tau, double* threshold, double* s) {
  auto* st = static_cast<Ista*>(h);
  *tau = st->tau; *threshold = st->threshold; *s = st->s;
}
void orc_ista_free(void* h) { delete static_cast<Ista*>(h); }

// ---- cADMM handle ---------------------------------------------------------
void* orc_cadmm_setup(int64_t n, int64_t m, const double* c, const int64_t* omega, const double* y,
                      double alpha, double rho, double sigma, double tau1, double tau2, int* status) {
  auto* st = new Cadmm();
  const int rc = cadmm_setup(*st, n, m, c, omega, y, alpha, rho, sigma, tau1, tau2);
  *status = rc;
  if (rc) { delete st; return nullptr; }
  return st;
}
int orc_cadmm_step(void* h, int64_t iters, int engine, int threads) {
  auto* st = static_cast<Cadmm*>(h);
  for (int64_t k = 0; k < iters; ++k) {
    if (engine == 1) { if (int rc = cadmm_step_fft(*st)) return rc; }
    else cadmm_step_phases(*st, threads);
  }
  return OK;
}
// Timing sample: the three phases over outputs [0, outs).
int orc_cadmm_phase_sample(void* h, int64_t outs, int threads, double* phase_s) {
  auto* st = static_cast<Cadmm*>(h);
  if (outs < 0 || outs > st->n) return fail(EPARAM, "orc_cadmm_phase_sample: bad range");
  cadmm_step_phases(*st, threads, outs, phase_s);
  return OK;
}
// which: 0 x, 1 z, 2 nu, 3 mu, 4 v, 5 beta, 6 c~, 7 b, 8 d, 9 pty
int orc_cadmm_get(void* h, int which, double* out) {
  auto* st = static_cast<Cadmm*>(h);
  const std::vector<double>* tab[] = {&st->x, &st->z, &st->nu, &st->mu, &st->v, &st->beta, &st->c, &st->b, &st->d, &st->pty};
  if (which < 0 || which > 9) return fail(EPARAM, "orc_cadmm_get: bad field");
  std::copy(tab[which]->begin(), tab[which]->end(), out);
  return OK;
}
void orc_cadmm_scalars(void* h, double* threshold, double* s) {
  auto* st = static_cast<Cadmm*>(h);
  *threshold = st->threshold; *s = st->s;
}
void orc_cadmm_free(void* h) { delete static_cast<Cadmm*>(h); }

// ---- dense ADMM handle (solvers.hpp:267-327) --------------------------------
void* orc_admm_setup(int64_t n, int64_t m, const double* c, const int64_t* omega, const double* y, double alpha,
                     double rho, int64_t dense_cap, int threads, int* status) {
  auto* st = new Admm();
  const int rc = admm_setup(*st, n, m, c, omega, y, alpha, rho, dense_cap, threads);
  *status = rc;
  if (rc) { delete st; return nullptr; }
  return st;
}
int orc_admm_step(void* h, int64_t iters, int threads) {
  auto* st = static_cast<Admm*>(h);
  for (int64_t k = 0; k < iters; ++k) admm_step_phases(*st, threads);
  return OK;
}
// which: 0 x, 1 z, 2 u, 3 rhs, 4 aty, 5 B (n * n, row-major)
int orc_admm_get(void* h, int which, double* out) {
  auto* st = static_cast<Admm*>(h);
  const std::vector<double>* tab[] = {&st->x, &st->z, &st->u, &st->rhs, &st->aty, &st->B};
  if (which < 0 || which > 5) return fail(EPARAM, "orc_admm_get: bad field");
  std::copy(tab[which]->begin(), tab[which]->end(), out);
  return OK;
}
void orc_admm_scalars(void* h, double* threshold, double* s) {
  auto* st = static_cast<Admm*>(h);
  *threshold = st->threshold; *s = st->s;
}
void orc_admm_free(void* h) { delete static_cast<Admm*>(h); }

// ---- run_loop solvers.hpp:426-472 over either handle ----------------------
// kind 0 = ISTA (iterate x), 1 = cADMM (iterate z, solvers.hpp:528), 2 = dense ADMM (iterate z, :508).
// trace arrays (capacity trace_cap) receive (iteration, value) per check.
// Returns status; fills iterations, reached_target, final_metric, trace_len.
int orc_run_loop(void* h, int kind, const double* truth, int64_t max_iter, double target, int64_t check_every,
                 int engine, int threads, int64_t* iterations, int* reached, double* final_metric,
                 int64_t* trace_it, double* trace_val, int64_t trace_cap, int64_t* trace_len) {
  if (max_iter < 0) return fail(EPARAM, "solver: max_iter must be >= 0");
  if (check_every < 1) return fail(EPARAM, "solver: check_every must be >= 1");
  std::vector<double>* it = kind == 0 ? &static_cast<Ista*>(h)->x
                          : kind == 1 ? &static_cast<Cadmm*>(h)->z : &static_cast<Admm*>(h)->z;
  const int64_t n = static_cast<int64_t>(it->size());
  const bool has_target = !std::isnan(target);
  const double inv_sqrt_n = n > 0 ? 1.0 / std::sqrt(static_cast<double>(n)) : 1.0;
  std::vector<double> prev;
  int64_t t = 0, tl = 0;
  *reached = 0;
  *final_metric = std::numeric_limits<double>::quiet_NaN();
  while (t < max_iter) {
    prev = *it;
    const int rc = kind == 0 ? orc_ista_step(h, 1, engine, threads)
                 : kind == 1 ? orc_cadmm_step(h, 1, engine, threads) : orc_admm_step(h, 1, threads);
    if (rc) return rc;
    ++t;
    if (t % check_every != 0 && t != max_iter) continue;
    for (double v : *it)
      if (!std::isfinite(v))
        return fail(EDIVERGE, kind == 0   ? "ista_run: iterate became non-finite"
                              : kind == 1 ? "cadmm_run: iterate became non-finite"
                                          : "admm_dense_run: iterate became non-finite");
    double value = 0.0;
    if (truth) {
      for (int64_t i = 0; i < n; ++i) { const double d = (*it)[static_cast<size_t>(i)] - truth[i]; value += d * d; }
      value = n > 0 ? value / static_cast<double>(n) : 0.0;
    } else {
      for (int64_t i = 0; i < n; ++i) { const double d = (*it)[static_cast<size_t>(i)] - prev[static_cast<size_t>(i)]; value += d * d; }
      value = std::sqrt(value) * inv_sqrt_n;
    }
    if (tl < trace_cap) { trace_it[tl] = t; trace_val[tl] = value; }
    ++tl;
    *final_metric = value;
    if (has_target && value <= target) { *reached = 1; break; }
  }
  *iterations = t;
  *trace_len = tl;
  return OK;
}

}  // extern "C"
