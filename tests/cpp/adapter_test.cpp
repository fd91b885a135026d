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

// parallel_test.cpp:29-108: the host executor's contract (every item once; parallelism >= 1; a throwing item
// surfaces as the lowest-id PhaseError; overlapping declared writes are rejected)
static void phase_checks() {
  for (const int parallelism : {1, 3, 16}) {
    std::vector<int> hits(10, 0);
    cl::KernelPhase phase;
    phase.name = "counting";
    phase.work_items = 10;
    phase.body = [&hits](cl::Index i) { ++hits[static_cast<size_t>(i)]; };
    cl::run_phase(phase, parallelism);
    for (const int h : hits) CHECK(h == 1);
  }
  cl::KernelPhase empty;
  empty.name = "empty";
  empty.body = [](cl::Index) { throw std::runtime_error("never"); };
  cl::run_phase(empty, 4);
  cl::KernelPhase one;
  one.name = "one";
  one.work_items = 1;
  one.body = [](cl::Index) {};
  CHECK(throws<cl::ParameterError>([&] { cl::run_phase(one, 0); }));
  cl::KernelPhase faulty;
  faulty.name = "faulty kernel";
  faulty.work_items = 30;
  faulty.body = [](cl::Index i) {
    if (i == 5 || i == 17) throw std::runtime_error("boom");
  };
  for (const int parallelism : {1, 4}) {
    bool caught = false;
    try {
      cl::run_phase(faulty, parallelism);
    } catch (const cl::PhaseError& e) {
      caught = e.global_id() == 5 && std::string(e.what()).find("faulty kernel") != std::string::npos &&
               std::string(e.what()).find("boom") != std::string::npos;
    }
    CHECK(caught);
  }
  std::vector<double> buffer(8, 0.0);
  cl::KernelPhase overlapping;
  overlapping.name = "overlapping";
  overlapping.work_items = 4;
  overlapping.body = [](cl::Index) {};
  overlapping.writes = [&buffer](cl::Index i) {
    return std::vector<cl::WriteAddress>{{buffer.data(), i == 1 ? 3 : i}};
  };
  CHECK(throws<cl::ConsistencyError>([&] { cl::check_disjoint_writes(overlapping); }));
  CHECK(cl::hardware_parallelism() >= 1);
}

// the factory phases on the device: run_pipeline(cpista_phases) / cpadmm_phases / padmm_phases advance the state
// exactly like *_step (the same kernels in the same order: bitwise), parallel_test.cpp:75-96,143-165
static void device_phase_checks() {
  const cl::SensingProblem<double> p = cl::make_problem(1 << 14, 1 << 12, 64, 41);  // not a persistent-kernel size
  cl::SolverConfig cfg;
  cl::IstaState<double> a = cl::ista_setup(p.op, p.measurements, cfg), b = cl::ista_setup(p.op, p.measurements, cfg);
  int checked = 0;
  const std::vector<cl::KernelPhase> ph = cl::cpista_phases(a);
  for (const cl::KernelPhase& k : ph) {
    cl::check_disjoint_writes(k);
    ++checked;
  }
  for (int it = 0; it < 3; ++it) {
    cl::run_pipeline(ph, cl::hardware_parallelism());
    cl::ista_step(b, false);
  }
  CHECK(a.t == 3 && b.t == 3 && a.x == b.x && a.r == b.r && a.delta == b.delta);
  cl::CadmmState<double> c = cl::cadmm_setup(p.op, p.measurements, cfg), d = cl::cadmm_setup(p.op, p.measurements, cfg);
  const std::vector<cl::KernelPhase> pc = cl::cpadmm_phases(c);
  checked += static_cast<int>(pc.size());
  for (int it = 0; it < 3; ++it) {
    cl::run_pipeline(pc, 4);
    cl::cadmm_step(d, false);
  }
  CHECK(c.t == 3 && d.t == 3 && c.z == d.z && c.x == d.x && c.v == d.v);
  const cl::SensingProblem<double> q = cl::make_problem(256, 128, 8, 42);
  cl::AdmmState<double> e = cl::admm_setup(q.op, q.measurements, cfg), f = cl::admm_setup(q.op, q.measurements, cfg);
  const std::vector<cl::KernelPhase> pa = cl::padmm_phases(e);
  checked += static_cast<int>(pa.size());
  for (int it = 0; it < 3; ++it) {
    cl::run_pipeline(pa, 2);
    cl::admm_step(f);
  }
  CHECK(e.t == 3 && f.t == 3 && e.z == f.z && e.u == f.u);
  CHECK(checked == 7);
}

static void gpu_checks() {
  device_phase_checks();
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
  phase_checks();
  if (mode == "gpu") gpu_checks();
  if (mode == "c4") {
    sharded_c4_checks(1, cl::Transport::kNccl);
    sharded_c4_checks(2, cl::Transport::kCopy);
  }
  std::printf("adapter_test %s: %s\n", mode.c_str(), failures ? "FAIL" : "PASS");
  return failures ? 1 : 0;
}
