// Seeded problem generation (reference sensing.hpp:29-207, deblur.hpp:26-86).
//
// Bit-exact with the reference: every draw is a fixed transform of raw
// std::mt19937_64 output (pinned by the C++ standard), seeds are derived by
// SplitMix64 from (seed, stream tag), and subsets come from a partial
// Fisher-Yates shuffle followed by a sort.  Generation runs on the host; it
// produces the synthetic (c, omega, x*, y) inputs the solver consumes.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>

#include "host_common.hpp"

namespace clb {
namespace {

uint64_t mix64(uint64_t z) {  // sensing.hpp:35-40
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

enum : uint64_t {                    // sensing.hpp:47-49
  kTagSignal = 0x7369676e616cULL,    // "signal"
  kTagRow = 0x726f77ULL,             // "row"
  kTagMask = 0x6d61736bULL,          // "mask"
};

uint64_t stream_seed(uint64_t seed, uint64_t tag) { return mix64(seed ^ mix64(tag)); }  // :42-44

class Stream {  // SeededRng sensing.hpp:56-95
 public:
  explicit Stream(uint64_t seed) : mt_(seed) {}
  double unit() { return static_cast<double>(mt_() >> 11) * 0x1.0p-53; }
  double gauss() {
    if (cached_) {
      cached_ = false;
      return cache_;
    }
    const double u1 = 1.0 - unit();
    const double u2 = unit();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * 3.14159265358979323846 * u2;
    cache_ = rad * std::sin(th);
    cached_ = true;
    return rad * std::cos(th);
  }
  uint64_t below(uint64_t bound) {
    const uint64_t limit = ~uint64_t(0) - (~uint64_t(0) % bound);
    uint64_t v;
    do v = mt_(); while (v >= limit);
    return v % bound;
  }

 private:
  std::mt19937_64 mt_;
  double cache_ = 0.0;
  bool cached_ = false;
};

// sensing.hpp:100-113
std::vector<int64_t> sorted_subset(int64_t n, int64_t k, Stream& s) {
  std::vector<int64_t> pool(static_cast<size_t>(n));
  std::iota(pool.begin(), pool.end(), int64_t(0));
  for (int64_t i = 0; i < k; ++i) {
    const int64_t j = i + static_cast<int64_t>(s.below(static_cast<uint64_t>(n - i)));
    std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
  }
  pool.resize(static_cast<size_t>(k));
  std::sort(pool.begin(), pool.end());
  return pool;
}

}  // namespace

void gen_sparse_signal(int64_t n, int64_t k, uint64_t seed, double* values, int64_t* support) {
  if (n < 0 || k < 0 || k > n) raise(CL_EPARAM, "gen_sparse_signal: need 0 <= k <= n");
  Stream s(stream_seed(seed, kTagSignal));
  const std::vector<int64_t> sup = sorted_subset(n, k, s);
  std::fill(values, values + n, 0.0);
  for (size_t i = 0; i < sup.size(); ++i) {
    support[i] = sup[i];
    values[sup[i]] = s.gauss();
  }
}

// matvec_scheme_bench inputs (parallel.hpp:343-348): n row draws then n x draws of one "row" stream.
void scheme_bench_inputs(int64_t n, uint64_t seed, double* row, double* x) {
  Stream rng(stream_seed(seed, kTagRow));
  for (int64_t i = 0; i < n; ++i) row[i] = rng.gauss();
  for (int64_t i = 0; i < n; ++i) x[i] = rng.gauss();
}

void gen_circulant_sensing(int64_t n, int64_t m, uint64_t seed, double* c, int64_t* omega) {
  if (m < 1 || m > n) raise(CL_EPARAM, "gen_circulant_sensing: need 1 <= m <= n");
  Stream rs(stream_seed(seed, kTagRow));
  for (int64_t i = 0; i < n; ++i) c[i] = rs.gauss();
  Stream ms(stream_seed(seed, kTagMask));
  const std::vector<int64_t> om = sorted_subset(n, m, ms);
  std::copy(om.begin(), om.end(), omega);
}

void gen_star_field(int64_t width, int64_t height, double density, uint64_t seed, double* px) {
  if (width < 1 || height < 1) raise(CL_EPARAM, "gen_star_field: dimensions must be positive");
  if (!(density >= 0.0) || !(density <= 1.0)) raise(CL_EPARAM, "gen_star_field: density must lie in [0, 1]");
  const int64_t n = width * height;
  const auto k = static_cast<int64_t>(density * static_cast<double>(n));
  Stream s(stream_seed(seed, kTagSignal));
  std::fill(px, px + n, 0.0);
  for (int64_t idx : sorted_subset(n, k, s)) px[idx] = 0.3 + 0.7 * s.unit();
}

void blur_row(int64_t n, int64_t L, double* row) {
  if (L < 1 || L > n) raise(CL_EPARAM, "blur_matrix: need 1 <= L <= n");
  for (int64_t i = 0; i < n; ++i) row[i] = i < L ? 1.0 / static_cast<double>(L) : 0.0;
}

}  // namespace clb
