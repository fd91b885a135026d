// Drop-in check of include/circlasso_b200.hpp: reference-style C++ code
// (mirroring /root/reference/proj/tests/solvers_test.cpp) against the C-ABI.
// Usage: adapter_test cpu | gpu | c4     (exit code 0 = pass; c4: the sharded config-4 solve)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "circlasso_b200.hpp"

namespace cl = circlasso_b200;

static int failures = 0;
#define CHECK(c)                                                    \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                   \
    }                                                               \
  } while (0)
template <typename E, typename F>
static bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void cpu_checks() {
  const cl::SensingProblem<double> a = cl::make_problem<double>(128, 64, 12, 9), b = cl::make_problem(128, 64, 12, 9);
  CHECK(a.signal.values == b.signal.values && a.op.mask().omega() == b.op.mask().omega());
  CHECK(a.measurements == b.measurements && a.k() == 12);
  CHECK(cl::gen_sparse_signal<double>(4096, 409, 1).k() == 409);
  CHECK(std::abs(cl::spectral_norm(cl::CirculantMatrix<double>::Identity(6)) - 1.0) < 1e-12);
  const cl::Vector<double> d = cl::mask_gram_inverse(cl::SubsamplingMask({0, 3}, 5), 0.25).diag();
  CHECK(std::abs(d[0] - 0.8) < 1e-15 && std::abs(d[1] - 4.0) < 1e-15);
  CHECK(throws<cl::SingularityError>([] { cl::regularized_gram_inverse(cl::CirculantMatrix<double>({1.0, 1.0}), 1.0, 0.0); }));
  CHECK(throws<cl::ParameterError>([] { cl::SubsamplingMask({4, 1}, 8); }));
  const cl::SensingProblem<double> p = cl::make_problem(32, 16, 3, 13);
  cl::SolverConfig bad;
  bad.tau = 1.5;
  CHECK(throws<cl::ParameterError>([&] { cl::ista_run(p.measurements, p.op, bad); }));
  cl::SolverConfig cfg;
  cl::Vector<double> y = p.measurements;
  y[3] = std::nan("");
  CHECK(throws<cl::DivergenceError>([&] { cl::ista_run(y, p.op, cfg); }));
  CHECK(throws<cl::DimensionError>([&] { cl::ista_run(cl::Vector<double>(15, 0.0), p.op, cfg); }));
  // dense ADMM: the size check, then the dense cap (solvers.hpp:288-296), before any device work
  CHECK(throws<cl::DimensionError>([&] { cl::admm_dense_run(cl::Vector<double>(15, 0.0), p.op, cfg); }));
  cl::SolverConfig capped;
  capped.dense_cap = 16;
  CHECK(throws<cl::CapacityError>([&] { cl::admm_dense_run(p.measurements, p.op, capped); }));
  // artifact formats (io.hpp), the same names as the reference
  {
    const cl::PartialCirculantOperator<double> A = cl::gen_circulant_sensing(64, 24, 99);
    cl::write_operator(A, "/tmp/clb_adapter_op.bin");
    const cl::PartialCirculantOperator<double> back = cl::read_operator("/tmp/clb_adapter_op.bin");
    CHECK(back.n() == 64 && back.m() == 24 && back.circulant().first_row() == A.circulant().first_row() &&
          back.mask().omega() == A.mask().omega());
    cl::write_vector(A.circulant().first_row(), "/tmp/clb_adapter_vec.bin");
    CHECK(cl::read_vector("/tmp/clb_adapter_vec.bin") == A.circulant().first_row());
    bool threw = false;
    try {
      cl::read_vector("/tmp/clb_adapter_missing.bin");
    } catch (const cl::FormatError&) {
      threw = true;
    }
    CHECK(threw);
    cl::BenchRow row;
    row.algorithm = "cadmm";
    row.iterations = 1180;
    row.setup_seconds = 0.25;
    row.total_seconds = 1.5;
    CHECK(std::abs(row.iterations_per_second() - 944.0) < 1e-9);
  }
}

static void gpu_checks() {
  // solvers_test.cpp:213-243 report bookkeeping
  const cl::SensingProblem<double> p = cl::make_problem(256, 128, 25, 17);
  cl::SolverConfig cfg;
  cfg.target_mse = 1e-4;
  cfg.max_iter = 20000;
  const cl::RecoveryReport<double> rep = cl::cadmm_run(p.measurements, p.op, cfg, &p.signal.values);
  CHECK(rep.reached_target && rep.metric == cl::StopMetric::kMseVsTruth && rep.final_metric <= 1e-4);
  CHECK(!rep.mse_trace.empty() && rep.mse_trace.back().value == rep.final_metric);
  CHECK(rep.setup_seconds <= rep.total_seconds && rep.footprint_bytes == 10 * 256 * 4);
  // ista_step advances t; literal == proximal (solvers_test.cpp:260-275)
  cl::IstaState<double> st = cl::ista_setup(p.op, p.measurements, cl::SolverConfig{});
  cl::ista_step(st);
  cl::ista_step(st);
  CHECK(st.t == 2);
  cl::SolverConfig lit, prox;
  lit.tau = prox.tau = 0.5;
  lit.alpha = 5e-4;
  prox.alpha = 1e-3;
  prox.pairing = cl::ThresholdPairing::kProximal;
  lit.max_iter = prox.max_iter = 200;
  CHECK(cl::ista_run(p.measurements, p.op, lit).final_x == cl::ista_run(p.measurements, p.op, prox).final_x);
  // dense ADMM baseline (solvers.hpp:497-514): same recovery as cADMM, dense footprint
  {
    cl::SolverConfig dc;
    dc.target_mse = 1e-4;
    dc.max_iter = 20000;
    const cl::RecoveryReport<double> dr = cl::admm_dense_run(p.measurements, p.op, dc, &p.signal.values);
    CHECK(dr.reached_target && dr.final_metric <= 1e-4);
    CHECK(dr.footprint_bytes == (256ull * 256 + 4 * 256 + 128) * 4);
    cl::AdmmState<double> ast = cl::admm_setup(p.op, p.measurements, cl::SolverConfig{});
    cl::admm_step(ast);
    CHECK(ast.t == 1 && ast.B().size() == 256u * 256u && ast.z.size() == 256u);
  }
  // reference-style state use (solvers_test.cpp:303-323): ista_step refreshes state.x; the per-call
  // use_fft picks the engine of each step (FFT by default, like the reference), the iterate carries over
  {
    cl::IstaState<double> a = cl::ista_setup(p.op, p.measurements, cl::SolverConfig{});
    cl::IstaState<double> b = cl::ista_setup(p.op, p.measurements, cl::SolverConfig{});
    for (int i = 0; i < 4; ++i) {
      cl::ista_step(a, false);
      cl::ista_step(b, i % 2 == 0);  // FFT, direct, FFT, direct
    }
    CHECK(a.t == 4 && b.t == 4 && a.x.size() == 256u && a.r.size() == 128u);
    double num = 0, den = 0;
    for (size_t i = 0; i < a.x.size(); ++i) {
      num += (a.x[i] - b.x[i]) * (a.x[i] - b.x[i]);
      den += a.x[i] * a.x[i];
    }
    CHECK(den > 0 && std::sqrt(num / den) < 1e-5);
    CHECK(std::abs(a.tau - 0.9) < 1e-15 && a.threshold == 1e-4 && a.y.size() == 128u);
    cl::CadmmState<double> c = cl::cadmm_setup(p.op, p.measurements, cl::SolverConfig{});
    cl::cadmm_step(c);
    cl::cadmm_step(c, false);
    CHECK(c.t == 2 && c.z.size() == 256u && c.B.n() == 256 && c.D.n() == 256 && c.threshold == 1e-4 / 0.1);
  }
  // Scalar = float instantiates the same API (the device computes in fp32 either way)
  {
    const cl::SensingProblem<float> pf = cl::make_problem<float>(256, 128, 25, 17);
    cl::SolverConfig fc;
    fc.max_iter = 50;
    const cl::RecoveryReport<float> rf = cl::ista_run(pf.measurements, pf.op, fc);
    CHECK(rf.iterations == 50 && rf.final_x.size() == 256u);
  }
  // device products vs the fp64 measure
  const cl::Vector<double> ax = cl::partial_matvec(p.op, p.signal.values);
  double err = 0, nrm = 0;
  for (size_t i = 0; i < ax.size(); ++i) {
    err += (ax[i] - p.measurements[i]) * (ax[i] - p.measurements[i]);
    nrm += p.measurements[i] * p.measurements[i];
  }
  CHECK(std::sqrt(err / nrm) < 5e-5);
}

// BASELINE config 4 through the C-ABI in one process: cADMM n = 2^24, m = 2^22, k = 2^16, sharded over
// the listed ranks (the library's exchange), against the unsharded solve -- bitwise.
static void sharded_c4_checks(int world, cl::Transport transport) {
  const cl::SensingProblem<double> p = cl::make_problem(1 << 24, 1 << 22, 1 << 16, 1);
  cl::SolverConfig cfg;
  cfg.max_iter = 2;
  cfg.check_every = 2;
  const cl::RecoveryReport<double> solo = cl::cadmm_run(p.measurements, p.op, cfg, &p.signal.values);
  cl::ShardedSolve<double> sh(CL_KIND_CADMM, p.op, p.measurements, cfg, std::vector<int>(static_cast<size_t>(world), 0),
                      transport);
  CHECK(sh.world() == world);
  const cl::RecoveryReport<double> rep = sh.run(&p.signal.values);
  CHECK(rep.iterations == 2 && solo.iterations == 2);
  CHECK(rep.final_x == solo.final_x);
  CHECK(std::abs(rep.final_metric - solo.final_metric) <= 1e-12 * std::abs(solo.final_metric));
  std::printf("sharded C4 cADMM, %d rank(s) (%s): 2 iterations, z bitwise equal to the unsharded solve, MSE %.6e\n",
              world, transport == cl::Transport::kNccl ? "NCCL" : "peer copies", rep.final_metric);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_checks();
  if (mode == "gpu") gpu_checks();
  if (mode == "c4") {
    sharded_c4_checks(1, cl::Transport::kNccl);
    sharded_c4_checks(2, cl::Transport::kCopy);
  }
  std::printf("adapter_test %s: %s\n", mode.c_str(), failures ? "FAIL" : "PASS");
  return failures ? 1 : 0;
}
