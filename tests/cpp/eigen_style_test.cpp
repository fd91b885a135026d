// Reference-style code (the shapes of /root/reference/proj/tests/solvers_test.cpp and sensing_test.cpp:
// Vector<double>::Zero, the comma initializer, templated types with <double>, state members) compiled
// against include/circlasso_b200.hpp's Eigen branch.  Built with -I tests/cpp/eigen_stub (a test double of
// the few Eigen members used; see its header) because Eigen is not installed here.
// Usage: eigen_style_test cpu | gpu
#include <cmath>
#include <cstdio>
#include <string>

#include "circlasso_b200.hpp"

#ifndef CIRCLASSO_B200_EIGEN
#error "the adapter did not take its Eigen branch"
#endif

using circlasso_b200::CirculantMatrix;
using circlasso_b200::PartialCirculantOperator;
using circlasso_b200::RecoveryReport;
using circlasso_b200::SensingProblem;
using circlasso_b200::SolverConfig;
using circlasso_b200::SubsamplingMask;
using circlasso_b200::Vector;

static int failures = 0;
#define CHECK(c)                                                                  \
  do {                                                                            \
    if (!(c)) {                                                                   \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);   \
      ++failures;                                                                 \
    }                                                                             \
  } while (0)

static PartialCirculantOperator<double> identity_operator(Eigen::Index n) {  // solvers_test.cpp:34-37
  return PartialCirculantOperator<double>(CirculantMatrix<double>::Identity(n), SubsamplingMask::Full(n));
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  {  // solvers_test.cpp:48-56
    Vector<double> x(3);
    x << 2.0, -0.5, -3.0;
    const Vector<double> y = circlasso_b200::soft_threshold(x, 1.0);
    CHECK(y[0] == 1.0 && y[1] == 0.0 && y[2] == -2.0);
  }
  {  // sensing_test.cpp:69-81: the same seed gives the same problem
    const SensingProblem<double> a = circlasso_b200::make_problem<double>(128, 64, 12, 9);
    const SensingProblem<double> b = circlasso_b200::make_problem<double>(128, 64, 12, 9);
    CHECK((a.measurements - b.measurements).norm() == 0.0 && a.k() == 12);
    CHECK(std::abs(circlasso_b200::spectral_norm(identity_operator(6).circulant()) - 1.0) < 1e-12);
  }
  if (mode == "gpu") {
    {  // solvers_test.cpp:123-135: identity operator, proximal pairing -> eta_alpha(y)
      const Eigen::Index n = 32;
      Vector<double> y = Vector<double>::Zero(n);
      for (Eigen::Index i = 0; i < n; ++i) y[i] = 0.5 * std::sin(0.7 * static_cast<double>(i));
      SolverConfig cfg;
      cfg.alpha = 0.3;
      cfg.pairing = circlasso_b200::ThresholdPairing::kProximal;
      cfg.max_iter = 400;
      const RecoveryReport<double> rep = circlasso_b200::ista_run(y, identity_operator(n), cfg);
      const Vector<double> want = circlasso_b200::soft_threshold(y, 0.3);
      CHECK((rep.final_x - want).norm() <= 1e-6);
    }
    {  // solvers_test.cpp:303-323 style: the state's members after ista_step
      const SensingProblem<double> p = circlasso_b200::make_problem<double>(256, 128, 25, 17);
      circlasso_b200::IstaState<double> state = circlasso_b200::ista_setup(p.op, p.measurements, SolverConfig{});
      const double weight = SolverConfig{}.alpha / state.tau;
      circlasso_b200::ista_step(state);
      CHECK(state.t == 1 && state.x.size() == 256 && weight > 0 && (state.x - state.x).norm() == 0.0);
      const RecoveryReport<double> r = circlasso_b200::cadmm_run(p.measurements, p.op, SolverConfig{},
                                                                 &p.signal.values);
      CHECK(r.final_x.size() == 256 && r.iterations > 0);
    }
  }
  std::printf("eigen_style_test %s: %s\n", mode.c_str(), failures ? "FAIL" : "PASS");
  return failures ? 1 : 0;
}
