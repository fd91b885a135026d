// circlasso_b200.hpp — C++ drop-in adapter over the C-ABI (circlasso_b200.h).
//
// Mirrors the reference circlasso solver API (header-only C++20 library,
// /root/reference/proj/include/circlasso/) with the same names, argument
// meaning and error behaviour, so a reference user swaps
//     #include "circlasso/circlasso.hpp"   ->   #include "circlasso_b200.hpp"
//     circlasso::ista_run(...)             ->   circlasso_b200::ista_run(...)
// and links libcirclasso_b200.so.  Vectors are std::vector<double> (the
// reference's Eigen::VectorXd); when Eigen is available, Eigen overloads are
// provided too.  Every solve runs on the GPU; there is no CPU fallback.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "circlasso_b200.h"

namespace circlasso_b200 {

using Vector = std::vector<double>;
using Index = std::int64_t;

// ---- errors.hpp:12-72 -------------------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class DimensionError : public Error { using Error::Error; };
class ParameterError : public Error { using Error::Error; };
class SingularityError : public Error { using Error::Error; };
class DivergenceError : public Error { using Error::Error; };
class CapacityError : public Error { using Error::Error; };
class FormatError : public Error { using Error::Error; };
class ConsistencyError : public Error { using Error::Error; };
class PhaseError : public Error { using Error::Error; };
class CudaError : public Error { using Error::Error; };
class CommError : public Error { using Error::Error; };

inline void check(cl_status st) {
  if (st == CL_OK) return;
  const std::string msg = cl_last_error();
  switch (st) {
    case CL_EDIM: throw DimensionError(msg);
    case CL_EPARAM: throw ParameterError(msg);
    case CL_ESINGULAR: throw SingularityError(msg);
    case CL_EDIVERGE: throw DivergenceError(msg);
    case CL_ECAPACITY: throw CapacityError(msg);
    case CL_EFORMAT: throw FormatError(msg);
    case CL_ECONSIST: throw ConsistencyError(msg);
    case CL_EPHASE: throw PhaseError(msg);
    case CL_ECOMM: throw CommError(msg);
    default: throw CudaError(msg);
  }
}

namespace detail {
inline void check_same_size(Index a, Index b, const char* op) {  // fft.hpp:27-33
  if (a != b) throw DimensionError(std::string(op) + ": dimension mismatch, " + std::to_string(a) + " vs " +
                                   std::to_string(b));
}
}  // namespace detail

// ---- solvers.hpp:83, 112-150 --------------------------------------------------
enum class ThresholdPairing { kLiteral, kProximal };
enum class StopMetric { kMseVsTruth, kIterateChange };

struct SolverConfig {
  double alpha = 1e-4;
  double tau = 0.0;
  double rho = 0.1;
  double sigma = 0.1;
  double tau1 = 1.0;
  double tau2 = 1.0;
  long max_iter = 100000;
  double target_mse = std::numeric_limits<double>::quiet_NaN();
  int check_every = 10;
  ThresholdPairing pairing = ThresholdPairing::kLiteral;
  bool use_fft = false;  // true: on-device FFT engine (any n); false: direct sm_100a kernels
  Index dense_cap = 4096;  // circulant.hpp:31 kDenseCap: largest n of the dense ADMM
  int device = 0;       // new: CUDA device of the solve

  cl_config c() const {
    cl_config k;
    cl_config_default(&k);
    k.alpha = alpha;
    k.tau = tau;
    k.rho = rho;
    k.sigma = sigma;
    k.tau1 = tau1;
    k.tau2 = tau2;
    k.max_iter = max_iter;
    k.target_mse = target_mse;
    k.check_every = check_every;
    k.pairing = pairing == ThresholdPairing::kLiteral ? CL_PAIRING_LITERAL : CL_PAIRING_PROXIMAL;
    k.engine = use_fft ? CL_ENGINE_FFT : CL_ENGINE_DIRECT;
    k.dense_cap = dense_cap;
    return k;
  }
};

struct TracePoint {
  long iteration;
  double value;
  double elapsed_seconds;
};

struct RecoveryReport {
  Vector final_x;
  long iterations = 0;
  std::vector<TracePoint> mse_trace;
  double setup_seconds = 0.0;
  double total_seconds = 0.0;
  std::uint64_t footprint_bytes = 0;
  StopMetric metric = StopMetric::kIterateChange;
  bool reached_target = false;
  double final_metric = std::numeric_limits<double>::quiet_NaN();
};

// ---- circulant.hpp operators ----------------------------------------------------
class CirculantMatrix {
 public:
  CirculantMatrix() = default;
  explicit CirculantMatrix(Vector first_row) : row_(std::move(first_row)) {}
  static CirculantMatrix Identity(Index n) {
    Vector r(static_cast<size_t>(n), 0.0);
    if (n > 0) r[0] = 1.0;
    return CirculantMatrix(std::move(r));
  }
  Index n() const { return static_cast<Index>(row_.size()); }
  const Vector& first_row() const { return row_; }
  Index stored_scalars() const { return n(); }

 private:
  Vector row_;
};

class SubsamplingMask {
 public:
  SubsamplingMask() = default;
  SubsamplingMask(std::vector<Index> omega, Index n) : omega_(std::move(omega)), n_(n) {
    if (n_ < 0) throw ParameterError("SubsamplingMask: negative dimension");
    Index prev = -1;
    for (Index idx : omega_) {
      if (idx <= prev || idx >= n_)
        throw ParameterError("SubsamplingMask: indices must be strictly increasing and within [0, n)");
      prev = idx;
    }
  }
  static SubsamplingMask Full(Index n) {
    std::vector<Index> all(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) all[static_cast<size_t>(i)] = i;
    return SubsamplingMask(std::move(all), n);
  }
  Index m() const { return static_cast<Index>(omega_.size()); }
  Index n() const { return n_; }
  const std::vector<Index>& omega() const { return omega_; }
  Vector apply(const Vector& x) const {
    detail::check_same_size(static_cast<Index>(x.size()), n_, "SubsamplingMask::apply");
    Vector out(omega_.size());
    for (size_t i = 0; i < omega_.size(); ++i) out[i] = x[static_cast<size_t>(omega_[i])];
    return out;
  }
  Vector embed(const Vector& y) const {
    detail::check_same_size(static_cast<Index>(y.size()), m(), "SubsamplingMask::embed");
    Vector out(static_cast<size_t>(n_), 0.0);
    for (size_t i = 0; i < omega_.size(); ++i) out[static_cast<size_t>(omega_[i])] = y[i];
    return out;
  }

 private:
  std::vector<Index> omega_;
  Index n_ = 0;
};

class PartialCirculantOperator {
 public:
  PartialCirculantOperator() = default;
  PartialCirculantOperator(CirculantMatrix c, SubsamplingMask mask) : c_(std::move(c)), mask_(std::move(mask)) {
    detail::check_same_size(c_.n(), mask_.n(), "PartialCirculantOperator");
  }
  Index n() const { return c_.n(); }
  Index m() const { return mask_.m(); }
  const CirculantMatrix& circulant() const { return c_; }
  const SubsamplingMask& mask() const { return mask_; }

 private:
  CirculantMatrix c_;
  SubsamplingMask mask_;
};

inline double spectral_norm(const CirculantMatrix& C) {
  double s = 0;
  check(cl_spectral_norm(C.n(), C.first_row().data(), &s));
  return s;
}
inline CirculantMatrix regularized_gram_inverse(const CirculantMatrix& C, double rho, double sigma) {
  Vector b(static_cast<size_t>(C.n()));
  check(cl_regularized_gram_inverse(C.n(), C.first_row().data(), rho, sigma, b.data()));
  return CirculantMatrix(std::move(b));
}
inline Vector mask_gram_inverse(const SubsamplingMask& P, double rho) {
  Vector d(static_cast<size_t>(P.n()));
  check(cl_mask_gram_inverse(P.n(), P.m(), P.omega().data(), rho, d.data()));
  return d;
}
inline Vector circ_matvec(const CirculantMatrix& M, const Vector& x, int device = 0) {
  detail::check_same_size(static_cast<Index>(x.size()), M.n(), "circ_matvec");
  Vector out(x.size());
  check(cl_circ_matvec(device, M.n(), M.first_row().data(), x.data(), 0, out.data()));
  return out;
}
inline Vector circ_transpose_matvec(const CirculantMatrix& M, const Vector& x, int device = 0) {
  detail::check_same_size(static_cast<Index>(x.size()), M.n(), "circ_transpose_matvec");
  Vector out(x.size());
  check(cl_circ_matvec(device, M.n(), M.first_row().data(), x.data(), 1, out.data()));
  return out;
}
inline Vector partial_matvec(const PartialCirculantOperator& A, const Vector& x, int device = 0) {
  detail::check_same_size(static_cast<Index>(x.size()), A.n(), "partial_matvec");
  Vector out(static_cast<size_t>(A.m()));
  check(cl_partial_matvec(device, A.n(), A.m(), A.circulant().first_row().data(), A.mask().omega().data(), x.data(),
                          out.data()));
  return out;
}
inline Vector partial_transpose_matvec(const PartialCirculantOperator& A, const Vector& y, int device = 0) {
  detail::check_same_size(static_cast<Index>(y.size()), A.m(), "partial_transpose_matvec");
  Vector out(static_cast<size_t>(A.n()));
  check(cl_partial_transpose_matvec(device, A.n(), A.m(), A.circulant().first_row().data(),
                                    A.mask().omega().data(), y.data(), out.data()));
  return out;
}

// ---- sensing.hpp generation -------------------------------------------------------
struct SparseSignal {
  Vector values;
  std::vector<Index> support;
  Index n() const { return static_cast<Index>(values.size()); }
  Index k() const { return static_cast<Index>(support.size()); }
};
struct SensingProblem {
  SparseSignal signal;
  PartialCirculantOperator op;
  Vector measurements;
  std::uint64_t seed = 0;
  Index n() const { return op.n(); }
  Index m() const { return op.m(); }
  Index k() const { return signal.k(); }
};
inline SparseSignal gen_sparse_signal(Index n, Index k, std::uint64_t seed) {
  SparseSignal s;
  s.values.resize(static_cast<size_t>(n < 0 ? 0 : n));
  s.support.resize(static_cast<size_t>(k < 0 ? 0 : k));
  check(cl_gen_sparse_signal(n, k, seed, s.values.data(), s.support.data()));
  return s;
}
inline PartialCirculantOperator gen_circulant_sensing(Index n, Index m, std::uint64_t seed) {
  Vector row(static_cast<size_t>(n < 0 ? 0 : n));
  std::vector<Index> om(static_cast<size_t>(m < 0 ? 0 : m));
  check(cl_gen_circulant_sensing(n, m, seed, row.data(), om.data()));
  return PartialCirculantOperator(CirculantMatrix(std::move(row)), SubsamplingMask(std::move(om), n));
}
inline Vector measure(const PartialCirculantOperator& A, const Vector& x) {
  detail::check_same_size(static_cast<Index>(x.size()), A.n(), "measure");
  Vector y(static_cast<size_t>(A.m()));
  check(cl_measure(A.n(), A.m(), A.circulant().first_row().data(), A.mask().omega().data(), x.data(), y.data()));
  return y;
}
inline SensingProblem make_problem(Index n, Index m, Index k, std::uint64_t seed) {
  SensingProblem p;
  p.signal = gen_sparse_signal(n, k, seed);
  p.op = gen_circulant_sensing(n, m, seed);
  p.measurements = measure(p.op, p.signal.values);
  p.seed = seed;
  return p;
}

// ---- solver states (IstaState / CadmmState on the GPU) ---------------------------
class DeviceState {
 public:
  DeviceState(int kind, const PartialCirculantOperator& A, const Vector& y, const SolverConfig& cfg) {
    detail::check_same_size(static_cast<Index>(y.size()), A.m(),
                            kind == CL_KIND_ISTA ? "ista_setup" : kind == CL_KIND_CADMM ? "cadmm_setup" : "admm_setup");
    cl_solver* s = nullptr;
    const cl_config c = cfg.c();
    check(cl_solver_create(kind, A.n(), A.m(), A.circulant().first_row().data(), A.mask().omega().data(), y.data(),
                           &c, cfg.device, &s));
    h_.reset(s);
    n_ = A.n();
    m_ = A.m();
  }
  cl_solver* handle() const { return h_.get(); }
  void step(long iters = 1) { check(cl_solver_step(h_.get(), iters)); }
  Vector get(const char* field) const {
    const std::string f(field);
    Vector out(static_cast<size_t>((f == "r" || f == "y") ? m_ : f == "B" ? n_ * n_ : n_));
    check(cl_solver_get(h_.get(), field, out.data()));
    return out;
  }
  long t() const {
    int64_t tt = 0;
    check(cl_solver_info(h_.get(), nullptr, nullptr, &tt, nullptr, nullptr));
    return static_cast<long>(tt);
  }

 private:
  struct Del {
    void operator()(cl_solver* s) const { cl_solver_destroy(s); }
  };
  std::unique_ptr<cl_solver, Del> h_;
  Index n_ = 0, m_ = 0;
};
struct IstaState : DeviceState {
  IstaState(const PartialCirculantOperator& A, const Vector& y, const SolverConfig& cfg)
      : DeviceState(CL_KIND_ISTA, A, y, cfg) {}
};
struct CadmmState : DeviceState {
  CadmmState(const PartialCirculantOperator& A, const Vector& y, const SolverConfig& cfg)
      : DeviceState(CL_KIND_CADMM, A, y, cfg) {}
};
inline IstaState ista_setup(const PartialCirculantOperator& A, const Vector& y, const SolverConfig& cfg) {
  return IstaState(A, y, cfg);
}
inline void ista_step(IstaState& s, bool /*use_fft*/ = true) { s.step(1); }
inline CadmmState cadmm_setup(const PartialCirculantOperator& A, const Vector& y, const SolverConfig& cfg) {
  return CadmmState(A, y, cfg);
}
inline void cadmm_step(CadmmState& s, bool /*use_fft*/ = true) { s.step(1); }
// Dense ADMM (solvers.hpp:267-327): B = (A~^T A~ + rho I)^-1 built in fp64 on the GPU; get("B") is n x n.
struct AdmmState : DeviceState {
  AdmmState(const PartialCirculantOperator& A, const Vector& y, const SolverConfig& cfg)
      : DeviceState(CL_KIND_ADMM, A, y, cfg) {}
};
inline AdmmState admm_setup(const PartialCirculantOperator& A, const Vector& y, const SolverConfig& cfg) {
  return AdmmState(A, y, cfg);
}
inline void admm_step(AdmmState& s) { s.step(1); }

namespace detail {
template <typename RunFn>
inline RecoveryReport run_with(RunFn run_fn, const SolverConfig& cfg, Index n) {
  const long cap = cfg.max_iter >= 0 ? cfg.max_iter / (cfg.check_every > 0 ? cfg.check_every : 1) + 2 : 0;
  std::vector<int64_t> it(static_cast<size_t>(cap > 0 ? cap : 1));
  std::vector<double> val(it.size()), sec(it.size());
  RecoveryReport rep;
  rep.final_x.resize(static_cast<size_t>(n));
  cl_report r{};
  check(run_fn(&r, rep.final_x.data(), it.data(), val.data(), sec.data(), static_cast<int64_t>(cap)));
  rep.iterations = static_cast<long>(r.iterations);
  rep.setup_seconds = r.setup_seconds;
  rep.total_seconds = r.total_seconds;
  rep.footprint_bytes = r.footprint_bytes;
  rep.metric = r.metric == CL_METRIC_MSE_VS_TRUTH ? StopMetric::kMseVsTruth : StopMetric::kIterateChange;
  rep.reached_target = r.reached_target != 0;
  rep.final_metric = r.final_metric;
  for (int64_t i = 0; i < r.trace_len && i < cap; ++i)
    rep.mse_trace.push_back({static_cast<long>(it[static_cast<size_t>(i)]), val[static_cast<size_t>(i)],
                             sec[static_cast<size_t>(i)]});
  return rep;
}
inline RecoveryReport run(DeviceState& st, const Vector* truth, const SolverConfig& cfg, Index n) {
  if (truth) {
    check_same_size(static_cast<Index>(truth->size()), n, "truth");
    check(cl_solver_set_truth(st.handle(), truth->data()));
  }
  return run_with(
      [&](cl_report* r, double* fx, int64_t* it, double* val, double* sec, int64_t cap) {
        return cl_solver_run(st.handle(), r, fx, it, val, sec, cap);
      },
      cfg, n);
}
}  // namespace detail

// solvers.hpp:479-495
inline RecoveryReport ista_run(const Vector& y, const PartialCirculantOperator& A, const SolverConfig& cfg,
                               const Vector* truth = nullptr) {
  IstaState st(A, y, cfg);
  return detail::run(st, truth, cfg, A.n());
}
// solvers.hpp:518-534
inline RecoveryReport cadmm_run(const Vector& y, const PartialCirculantOperator& A, const SolverConfig& cfg,
                                const Vector* truth = nullptr) {
  CadmmState st(A, y, cfg);
  return detail::run(st, truth, cfg, A.n());
}

// solvers.hpp:497-514
inline RecoveryReport admm_dense_run(const Vector& y, const PartialCirculantOperator& A, const SolverConfig& cfg,
                                     const Vector* truth = nullptr) {
  AdmmState st(A, y, cfg);
  return detail::run(st, truth, cfg, A.n());
}

// ---- sharded solve from one process (cl_group_*) -----------------------
// Rank r on devices[r]; after each phase the ranks exchange their slices inside the library: NCCL
// (ncclCommInitAll over the listed GPUs) or peer copies (Transport::kCopy; devices may repeat).  The
// iterate equals the unsharded solve's bitwise.  One process per GPU instead: cl_comm_init_rank +
// cl_solver_attach_comm on a DeviceState's handle.
enum class Transport { kNccl = CL_TRANSPORT_NCCL, kCopy = CL_TRANSPORT_COPY };
class ShardedSolve {
 public:
  ShardedSolve(int kind, const PartialCirculantOperator& A, const Vector& y, const SolverConfig& cfg,
               const std::vector<int>& devices, Transport transport = Transport::kNccl)
      : cfg_(cfg), n_(A.n()), m_(A.m()) {
    detail::check_same_size(static_cast<Index>(y.size()), A.m(), kind == CL_KIND_ISTA ? "ista_setup" : "cadmm_setup");
    cl_group* g = nullptr;
    const cl_config c = cfg.c();
    check(cl_group_create(kind, A.n(), A.m(), A.circulant().first_row().data(), A.mask().omega().data(), y.data(), &c,
                          devices.data(), static_cast<int>(devices.size()), static_cast<int>(transport), &g));
    g_.reset(g);
  }
  void step(long iters = 1) { check(cl_group_step(g_.get(), iters)); }
  Vector get(const char* field) const {
    const std::string f(field);
    Vector out(static_cast<size_t>((f == "r" || f == "y") ? m_ : n_));
    check(cl_group_get(g_.get(), field, out.data()));
    return out;
  }
  int world() const {
    int w = 0;
    check(cl_group_info(g_.get(), &w, nullptr, nullptr));
    return w;
  }
  RecoveryReport run(const Vector* truth = nullptr) {
    if (truth) {
      detail::check_same_size(static_cast<Index>(truth->size()), n_, "truth");
      check(cl_group_set_truth(g_.get(), truth->data()));
    }
    return detail::run_with(
        [&](cl_report* r, double* fx, int64_t* it, double* val, double* sec, int64_t cap) {
          return cl_group_run(g_.get(), r, fx, it, val, sec, cap);
        },
        cfg_, n_);
  }

 private:
  struct Del {
    void operator()(cl_group* g) const { cl_group_destroy(g); }
  };
  std::unique_ptr<cl_group, Del> g_;
  SolverConfig cfg_;
  Index n_ = 0, m_ = 0;
};

// ---- artifact formats (io.hpp) ---------------------------------------------------
inline void write_vector(const Vector& v, const std::string& path) {  // io.hpp:80-87
  check(cl_write_vector(path.c_str(), v.data(), static_cast<int64_t>(v.size())));
}
inline Vector read_vector(const std::string& path) {  // io.hpp:89-97
  int64_t n = 0;
  check(cl_read_vector(path.c_str(), nullptr, 0, &n));
  Vector v(static_cast<size_t>(n));
  check(cl_read_vector(path.c_str(), v.data(), n, &n));
  return v;
}
inline void write_operator(const PartialCirculantOperator& A, const std::string& path) {  // io.hpp:99-112
  const std::vector<Index>& om = A.mask().omega();
  std::vector<int64_t> o(om.begin(), om.end());
  check(cl_write_operator(path.c_str(), A.n(), A.m(), A.circulant().first_row().data(), o.data()));
}
inline PartialCirculantOperator read_operator(const std::string& path) {  // io.hpp:114-131
  int64_t n = 0, m = 0;
  check(cl_read_operator(path.c_str(), nullptr, 0, nullptr, 0, &n, &m));
  Vector row(static_cast<size_t>(n));
  std::vector<int64_t> om(static_cast<size_t>(m));
  check(cl_read_operator(path.c_str(), row.data(), n, om.data(), m, &n, &m));
  return PartialCirculantOperator(CirculantMatrix(std::move(row)),
                                  SubsamplingMask(std::vector<Index>(om.begin(), om.end()), n));
}

struct BenchRow {  // io.hpp:133-153
  std::string algorithm;
  Index n = 0, m = 0, k = 0;
  std::uint64_t seed = 0;
  long iterations = 0;
  double setup_seconds = 0.0, total_seconds = 0.0, final_mse = 0.0;
  std::uint64_t footprint_bytes = 0;
  std::string status = "ok";
  cl_bench_row c() const {
    return cl_bench_row{algorithm.c_str(), n, m, k, seed, iterations, setup_seconds, total_seconds, final_mse,
                        footprint_bytes, status.c_str()};
  }
  double iterations_per_second() const {
    const cl_bench_row r = c();
    return cl_bench_iters_per_second(&r);
  }
};
inline constexpr const char* kBenchCsvHeader =
    "algorithm,n,m,k,seed,iterations,setup_s,total_s,final_mse,footprint_bytes,iters_per_s,status";
inline void write_bench_header(std::ostream& out) { out << kBenchCsvHeader << "\n"; }  // io.hpp:157-159
inline void write_bench_row(std::ostream& out, const BenchRow& row) {                 // io.hpp:161-168
  const cl_bench_row r = row.c();
  int64_t len = 0;
  check(cl_bench_csv_row(&r, nullptr, 0, &len));
  std::string text(static_cast<size_t>(len) + 1, '\0');
  check(cl_bench_csv_row(&r, text.data(), len + 1, &len));
  text.resize(static_cast<size_t>(len));
  out << text << "\n";
}

}  // namespace circlasso_b200
