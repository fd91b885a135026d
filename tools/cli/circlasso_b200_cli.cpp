// circlasso_b200_cli — the reference's command-line front end (tools/circlasso_cli.cpp) over the B200
// engine: problem generation, recovery runs, benchmark sweeps, matvec scheme timing and compressed
// deblurring, with the reference's subcommands, options, output text, files and exit codes
// (0 success, 1 usage or I/O failure, 2 numerical failure or an unreached recovery target).
//
// Every solve runs on the GPU through include/circlasso_b200.hpp.  --engine selects the product engine
// (cli:48,60,221): `cuda` (default) = the direct shift-indexed sm_100a kernels; `cuda-fft` = the
// on-device FFT engine; the reference's CPU engine names map onto them (`naive` -> cuda, `fft` -> cuda-fft),
// and `phases` runs the solver's device kernel phases through run_pipeline (cli:111-184).  New: `--device D`, and `--devices 0,1,...` shards an ISTA / cADMM recover over
// those GPUs with the library's NCCL exchange.  The reference's CLI11 parser is not in this image; the
// option syntax (`--name value`, repeatable `--n` / `--solver`, flags) is parsed here.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "circlasso_b200.hpp"

namespace {

using namespace circlasso_b200;

constexpr int kExitOk = 0;
constexpr int kExitUsage = 1;
constexpr int kExitNumerical = 2;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --name value options (repeatable ones keep every value), --flag switches
struct Args {
  std::map<std::string, std::vector<std::string>> opt;
  std::map<std::string, bool> flag;
  bool has(const std::string& k) const { return opt.count(k) > 0; }
  std::string str(const std::string& k, const std::string& def) const {
    return has(k) ? opt.at(k).back() : def;
  }
  double num(const std::string& k, double def) const {
    if (!has(k)) return def;
    const std::string& v = opt.at(k).back();
    char* end = nullptr;
    const double d = std::strtod(v.c_str(), &end);
    if (end == v.c_str() || *end != '\0') throw UsageError(k + ": '" + v + "' is not a number");
    return d;
  }
  long integer(const std::string& k, long def) const {
    if (!has(k)) return def;
    const std::string& v = opt.at(k).back();
    char* end = nullptr;
    const long d = std::strtol(v.c_str(), &end, 10);
    if (end == v.c_str() || *end != '\0') throw UsageError(k + ": '" + v + "' is not an integer");
    return d;
  }
};

Args parse(int argc, char** argv, const std::vector<std::string>& valued, const std::vector<std::string>& flags) {
  Args a;
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    bool known = false;
    for (const auto& f : flags)
      if (k == f) {
        a.flag[k] = true;
        known = true;
      }
    if (known) continue;
    for (const auto& v : valued)
      if (k == v) known = true;
    if (!known) throw UsageError("unknown option " + k);
    if (i + 1 >= argc) throw UsageError(k + " needs a value");
    a.opt[k].push_back(argv[++i]);
  }
  return a;
}

const std::vector<std::string> kSolverOpts = {"--alpha", "--tau", "--rho", "--sigma", "--tau1", "--tau2",
                                              "--max-iter", "--target-mse", "--check-every", "--pairing",
                                              "--engine", "--device"};

// SolverFlags (cli:45-86)
SolverConfig solver_config(const Args& a, SolverConfig cfg) {
  cfg.alpha = a.num("--alpha", cfg.alpha);
  cfg.tau = a.num("--tau", cfg.tau);
  cfg.rho = a.num("--rho", cfg.rho);
  cfg.sigma = a.num("--sigma", cfg.sigma);
  cfg.tau1 = a.num("--tau1", cfg.tau1);
  cfg.tau2 = a.num("--tau2", cfg.tau2);
  cfg.max_iter = a.integer("--max-iter", cfg.max_iter);
  cfg.target_mse = a.num("--target-mse", cfg.target_mse);
  cfg.check_every = static_cast<int>(a.integer("--check-every", cfg.check_every));
  const std::string pairing = a.str("--pairing", "literal");
  if (pairing == "literal") cfg.pairing = ThresholdPairing::kLiteral;
  else if (pairing == "proximal") cfg.pairing = ThresholdPairing::kProximal;
  else throw ParameterError("--pairing must be literal or proximal");
  const std::string engine = a.str("--engine", "cuda");
  if (engine == "cuda" || engine == "naive" || engine == "phases") cfg.use_fft = false;
  else if (engine == "cuda-fft" || engine == "fft") cfg.use_fft = true;
  else throw ParameterError("--engine must be cuda, cuda-fft, naive, phases or fft");
  cfg.device = static_cast<int>(a.integer("--device", 0));
  return cfg;
}

std::uint64_t nonzero_count(const Vector<double>& x) {
  std::uint64_t c = 0;
  for (double v : x)
    if (v != 0.0) ++c;
  return c;
}

void print_report(const std::string& algorithm, Index n, Index m, const RecoveryReport<double>& report) {  // cli:90-107
  std::cout << algorithm << ": n=" << n << " m=" << m << " iterations=" << report.iterations
            << " setup_s=" << report.setup_seconds << " total_s=" << report.total_seconds << "\n";
  std::cout << (report.metric == StopMetric::kMseVsTruth ? "  final mse vs truth: " : "  final iterate change: ")
            << report.final_metric << (report.reached_target ? " (target reached)" : " (target not reached)") << "\n";
  std::cout << "  footprint_bytes=" << report.footprint_bytes << "\n";
}

std::vector<int> device_list(const std::string& s) {
  std::vector<int> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    char* end = nullptr;
    const long d = std::strtol(tok.c_str(), &end, 10);
    if (tok.empty() || *end != '\0' || d < 0) throw UsageError("--devices must look like 0,1,2,3");
    out.push_back(static_cast<int>(d));
  }
  return out;
}

int cmd_gen(const Args& a) {  // cli:186-199
  if (!a.has("--n") || !a.has("--out")) throw UsageError("gen: --n and --out are required");
  const Index n = a.integer("--n", 1024);
  Index k = a.integer("--k", -1), m = a.integer("--m", -1);
  const std::uint64_t seed = static_cast<std::uint64_t>(a.integer("--seed", 1));
  const std::string out = a.str("--out", "");
  if (k < 0) k = n / 10;
  if (m < 0) m = n / 2;
  const SensingProblem<double> problem = make_problem<double>(n, m, k, seed);
  write_vector(problem.signal.values, out + ".signal.bin");
  write_operator(problem.op, out + ".operator.bin");
  write_vector(problem.measurements, out + ".measurements.bin");
  std::cout << "gen: n=" << n << " m=" << m << " k=" << k << " seed=" << seed << "\n";
  std::cout << "  wrote " << out << ".signal.bin, " << out << ".operator.bin, " << out << ".measurements.bin\n";
  return kExitOk;
}

// --engine phases (cli:111-184): the solver advanced through its kernel phases with run_pipeline, the stop rule
// checked between pipeline runs on the state's host members (refreshed by the last phase of each iteration)
template <typename State>
RecoveryReport<double> run_phases_loop(State& st, std::vector<KernelPhase> phases, const Vector<double>& iterate,
                                       const SolverConfig& cfg, const Vector<double>* truth, int parallelism,
                                       FootprintKind kind, Index n, Index m, double setup_s) {
  RecoveryReport<double> rep;
  rep.metric = truth ? StopMetric::kMseVsTruth : StopMetric::kIterateChange;
  rep.setup_seconds = setup_s;
  const auto t0 = std::chrono::steady_clock::now();
  const auto since = [&t0] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  long t = 0;
  while (t < cfg.max_iter) {
    const Vector<double> before = iterate;
    run_pipeline(phases, parallelism);
    ++t;
    if (t % cfg.check_every != 0 && t != cfg.max_iter) continue;
    double change = 0.0;
    for (Index i = 0; i < static_cast<Index>(iterate.size()); ++i) {
      if (!std::isfinite(iterate[i])) throw DivergenceError("phase run: iterate became non-finite");
      change += (iterate[i] - before[i]) * (iterate[i] - before[i]);
    }
    const double value = truth ? mse(iterate, *truth) : std::sqrt(change / std::max<double>(1, iterate.size()));
    rep.mse_trace.push_back({t, value, since()});
    rep.final_metric = value;
    if (!std::isnan(cfg.target_mse) && value <= cfg.target_mse) {
      rep.reached_target = true;
      break;
    }
  }
  (void)st;
  rep.iterations = t;
  rep.final_x = iterate;
  rep.total_seconds = since() + setup_s;
  rep.footprint_bytes = analytic_footprint(kind, static_cast<std::uint64_t>(n), static_cast<std::uint64_t>(m),
                                           sizeof(double));
  return rep;
}

RecoveryReport<double> run_with_phases(const std::string& solver, const Vector<double>& y,
                                       const PartialCirculantOperator<double>& A, const SolverConfig& cfg,
                                       const Vector<double>* truth, int parallelism) {
  const auto t0 = std::chrono::steady_clock::now();
  const auto setup_s = [&t0] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  if (solver == "ista") {
    IstaState<double> st = ista_setup(A, y, cfg);
    return run_phases_loop(st, cpista_phases(st), st.x, cfg, truth, parallelism, FootprintKind::kCpista, A.n(),
                           A.m(), setup_s());
  }
  if (solver == "admm") {
    AdmmState<double> st = admm_setup(A, y, cfg);
    return run_phases_loop(st, padmm_phases(st), st.z, cfg, truth, parallelism, FootprintKind::kDenseAdmm, A.n(),
                           A.m(), setup_s());
  }
  if (solver != "cadmm") throw ParameterError("--solver must be ista, admm, or cadmm");
  CadmmState<double> st = cadmm_setup(A, y, cfg);
  return run_phases_loop(st, cpadmm_phases(st), st.z, cfg, truth, parallelism, FootprintKind::kCpadmm, A.n(), A.m(),
                         setup_s());
}

int cmd_recover(const Args& a) {  // cli:201-261
  if (!a.has("--problem")) throw UsageError("recover: --problem is required");
  const std::string problem = a.str("--problem", "");
  const std::string solver = a.str("--solver", "cadmm");
  const SolverConfig cfg = solver_config(a, SolverConfig{});
  const PartialCirculantOperator<double> A = read_operator(problem + ".operator.bin");
  const Vector<double> y = read_vector(problem + ".measurements.bin");
  Vector<double> truth;
  bool has_truth = false;
  if (!a.flag.count("--ignore-truth")) {
    std::ifstream probe(problem + ".signal.bin", std::ios::binary);
    if (probe.good()) {
      truth = read_vector(problem + ".signal.bin");
      has_truth = true;
    }
  }
  const Vector<double>* truth_ptr = has_truth ? &truth : nullptr;
  RecoveryReport<double> report;
  if (a.has("--devices") && solver != "admm") {  // sharded over the listed GPUs, the library's NCCL exchange
    if (solver != "ista" && solver != "cadmm") throw ParameterError("--solver must be ista, admm, or cadmm");
    ShardedSolve<double> sh(solver == "ista" ? CL_KIND_ISTA : CL_KIND_CADMM, A, y, cfg, device_list(a.str("--devices", "")));
    report = sh.run(truth_ptr);
  } else if (a.str("--engine", "cuda") == "phases") {  // the kernel-phase executor (cli:221-223)
    const long threads = a.integer("--threads", hardware_parallelism());
    report = run_with_phases(solver, y, A, cfg, truth_ptr, static_cast<int>(threads));
  } else if (solver == "ista") {
    report = ista_run(y, A, cfg, truth_ptr);
  } else if (solver == "admm") {
    report = admm_dense_run(y, A, cfg, truth_ptr);
  } else if (solver == "cadmm") {
    report = cadmm_run(y, A, cfg, truth_ptr);
  } else {
    throw ParameterError("--solver must be ista, admm, or cadmm");
  }
  print_report(solver, A.n(), A.m(), report);
  const std::string out_x = a.str("--out-x", "");
  if (!out_x.empty()) write_vector(report.final_x, out_x);
  const std::string out_csv = a.str("--out", "");
  if (!out_csv.empty()) {
    BenchRow row;
    row.algorithm = solver;
    row.n = A.n();
    row.m = A.m();
    row.k = has_truth ? static_cast<Index>(nonzero_count(truth)) : 0;
    row.seed = 0;
    row.iterations = report.iterations;
    row.setup_seconds = report.setup_seconds;
    row.total_seconds = report.total_seconds;
    row.final_mse = report.final_metric;
    row.footprint_bytes = report.footprint_bytes;
    row.status = report.reached_target || std::isnan(cfg.target_mse) ? "ok" : "max_iter";
    std::ofstream out(out_csv);
    if (!out) throw FormatError("cannot open '" + out_csv + "' for writing");
    write_bench_header(out);
    write_bench_row(out, row);
  }
  if (!std::isnan(cfg.target_mse) && !report.reached_target) return kExitNumerical;
  return kExitOk;
}

int cmd_bench(const Args& a) {  // cli:263-333 (protocol problems m = n/2, k = n/10)
  if (!a.has("--n")) throw UsageError("bench: --n is required");
  SolverConfig base;
  base.target_mse = 1e-4;
  const SolverConfig cfg = solver_config(a, base);
  std::vector<std::string> solvers = a.has("--solver") ? a.opt.at("--solver")
                                                       : std::vector<std::string>{"ista", "admm", "cadmm"};
  const long seeds = a.integer("--seeds", 3);
  const std::string out_path = a.str("--out", "");
  std::ofstream file;
  if (!out_path.empty()) {
    file.open(out_path);
    if (!file) throw FormatError("cannot open '" + out_path + "' for writing");
  }
  std::ostream& out = out_path.empty() ? std::cout : file;
  write_bench_header(out);
  for (const std::string& ns : a.opt.at("--n")) {
    const Index n = std::strtol(ns.c_str(), nullptr, 10);
    const Index m = n / 2, k = n / 10;
    for (long seed = 1; seed <= seeds; ++seed) {
      const SensingProblem<double> problem = make_problem<double>(n, m, k, static_cast<std::uint64_t>(seed));
      for (const std::string& solver : solvers) {
        BenchRow row;
        row.algorithm = solver;
        row.n = n;
        row.m = m;
        row.k = k;
        row.seed = static_cast<std::uint64_t>(seed);
        if (solver == "admm" && n > cfg.dense_cap) {
          row.status = "skipped";
          row.footprint_bytes = analytic_footprint(FootprintKind::kDenseAdmm, static_cast<std::uint64_t>(n),
                                                   static_cast<std::uint64_t>(m), sizeof(double));
          write_bench_row(out, row);
          continue;
        }
        try {
          RecoveryReport<double> report;
          if (solver == "ista") report = ista_run(problem.measurements, problem.op, cfg, &problem.signal.values);
          else if (solver == "admm")
            report = admm_dense_run(problem.measurements, problem.op, cfg, &problem.signal.values);
          else if (solver == "cadmm")
            report = cadmm_run(problem.measurements, problem.op, cfg, &problem.signal.values);
          else throw ParameterError("--solver must be ista, admm, or cadmm");
          row.iterations = report.iterations;
          row.setup_seconds = report.setup_seconds;
          row.total_seconds = report.total_seconds;
          row.final_mse = report.final_metric;
          row.footprint_bytes = report.footprint_bytes;
          row.status = report.reached_target || std::isnan(cfg.target_mse) ? "ok" : "max_iter";
        } catch (const DivergenceError&) {
          row.status = "diverged";
        } catch (const Error& e) {
          row.status = "error";
          std::cerr << "bench: " << solver << " n=" << n << " seed=" << seed << ": " << e.what() << "\n";
        }
        write_bench_row(out, row);
        std::cerr << "bench: " << solver << " n=" << n << " seed=" << seed << " status=" << row.status
                  << " iters=" << row.iterations << " mse=" << row.final_mse << "\n";
      }
    }
  }
  return kExitOk;
}

int cmd_matvec_bench(const Args& a) {  // cli:335-379 (parallel.hpp:318-406 schemes on the GPU)
  if (!a.has("--n")) throw UsageError("matvec-bench: --n is required");
  const int repeats = static_cast<int>(a.integer("--repeats", 5));
  const std::uint64_t seed = static_cast<std::uint64_t>(a.integer("--seed", 1));
  const int device = static_cast<int>(a.integer("--device", 0));
  const std::string out_path = a.str("--out", "");
  std::ofstream file;
  if (!out_path.empty()) {
    file.open(out_path);
    if (!file) throw FormatError("cannot open '" + out_path + "' for writing");
  }
  std::ostream& out = out_path.empty() ? std::cout : file;
  write_bench_header(out);
  for (const std::string& ns : a.opt.at("--n")) {
    const Index n = std::strtol(ns.c_str(), nullptr, 10);
    for (int scheme : {0, 1}) {
      BenchRow row;
      row.algorithm = scheme == 0 ? "matvec-circulant" : "matvec-reference";
      row.n = n;
      row.m = n;
      row.k = 0;
      row.seed = seed;
      if (scheme == 1 && n > kDenseCap) {
        row.status = "skipped";
        write_bench_row(out, row);
        continue;
      }
      double min_s = 0, mean_s = 0, checksum = 0;
      uint64_t unique = 0, vec = 0;
      check(cl_matvec_scheme_bench(device, n, scheme, repeats, seed, kDenseCap, &min_s, &mean_s, &unique, &vec,
                                   &checksum));
      row.iterations = repeats;
      row.setup_seconds = 0.0;
      row.total_seconds = mean_s * repeats;
      row.final_mse = 0.0;
      row.footprint_bytes = unique * sizeof(double);
      write_bench_row(out, row);
      std::cerr << "matvec-bench: " << row.algorithm << " n=" << n << " min_s=" << min_s << " mean_s=" << mean_s
                << " unique_fetches=" << unique << " vector_fetches=" << vec << "\n";
    }
  }
  return kExitOk;
}

int cmd_deblur(const Args& a) {  // cli:381-435
  SolverConfig base;
  base.alpha = 1e-2;
  base.target_mse = 1e-6;  // iterate-change target; truth never steers
  const SolverConfig cfg = solver_config(a, base);
  const std::string image_path = a.str("--image", "");
  const std::string star_field = a.str("--star-field", "64x64");
  const double density = a.num("--density", 0.1);
  const Index L = a.integer("--L", 5);
  const Index m_abs = a.integer("--m", -1);
  const double m_ratio = a.num("--m-ratio", 0.5);
  const std::uint64_t seed = static_cast<std::uint64_t>(a.integer("--seed", 1));
  const std::string out = a.str("--out", "deblur");
  GrayImage<double> truth;
  if (!image_path.empty()) {
    truth = read_pgm(image_path);
  } else {
    long width = 0, height = 0;
    if (std::sscanf(star_field.c_str(), "%ldx%ld", &width, &height) != 2 || width < 1 || height < 1)
      throw ParameterError("--star-field must look like 64x64, got '" + star_field + "'");
    truth = gen_star_field<double>(width, height, density, seed);
  }
  const Index n = truth.size();
  Index m = m_abs;
  if (m < 0) m = static_cast<Index>(m_ratio * static_cast<double>(n));
  if (m < 1 || m > n) throw ParameterError("deblur: subsample count must satisfy 1 <= m <= n");
  const DeblurResult<double> result = run_deblur_experiment(truth, L, m, cfg, seed);
  const CirculantMatrix<double> B = blur_matrix<double>(n, L);
  const Vector<double> blurred = circ_matvec(B, truth.pixels, cfg.device);
  write_pgm(make_image(truth.width, truth.height, blurred), out + ".blurred.pgm");
  write_pgm(result.recovered, out + ".recovered.pgm");
  if (image_path.empty()) write_pgm(truth, out + ".truth.pgm");
  write_pgm(make_image(truth.width, truth.height, result.error_map), out + ".errmap.pgm");
  std::ofstream stats(out + ".stats.csv");
  if (!stats) throw FormatError("cannot open '" + out + ".stats.csv' for writing");
  stats << "width,height,n,m,L,alpha,seed,iterations,total_s,mse,normalized_mse,error_map_mean,status\n";
  stats << truth.width << ',' << truth.height << ',' << n << ',' << m << ',' << L << ',' << cfg.alpha << ','
        << seed << ',' << result.report.iterations << ',' << result.report.total_seconds << ','
        << result.mse_vs_truth << ',' << result.normalized_mse << ',' << result.error_map_mean << ','
        << (result.report.reached_target ? "ok" : "max_iter") << "\n";
  print_report("deblur (cadmm)", n, m, result.report);
  std::cout << "  mse_vs_truth=" << result.mse_vs_truth << " normalized_mse=" << result.normalized_mse
            << " error_map_mean=" << result.error_map_mean << "\n";
  std::cout << "  wrote " << out << ".{recovered,blurred,errmap}.pgm and " << out << ".stats.csv\n";
  if (!std::isnan(cfg.target_mse) && !result.report.reached_target) return kExitNumerical;
  return kExitOk;
}

const char* kUsage =
    "circulant compressed-sensing recovery toolkit (B200)\n"
    "usage: circlasso_b200_cli <gen|recover|bench|matvec-bench|deblur> [options]\n"
    "  gen          --n N --out PREFIX [--k K] [--m M] [--seed S]\n"
    "  recover      --problem PREFIX [--solver ista|admm|cadmm] [--ignore-truth] [--out CSV] [--out-x FILE]\n"
    "               [--devices 0,1,...] SOLVER FLAGS\n"
    "  bench        --n N [--n N ...] [--solver S ...] [--seeds K] [--out CSV] SOLVER FLAGS\n"
    "  matvec-bench --n N [--n N ...] [--repeats R] [--seed S] [--out CSV] [--device D]\n"
    "  deblur       [--image PGM | --star-field WxH] [--density D] [--L L] [--m M | --m-ratio R] [--seed S]\n"
    "               [--out PREFIX] SOLVER FLAGS\n"
    "  SOLVER FLAGS --alpha --tau --rho --sigma --tau1 --tau2 --max-iter --target-mse --check-every\n"
    "               --pairing literal|proximal --engine cuda|cuda-fft (naive, phases -> cuda; fft -> cuda-fft)\n"
    "               --device D\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
    std::cout << kUsage;
    return argc < 2 ? kExitUsage : kExitOk;
  }
  const std::string cmd = argv[1];
  auto with = [](std::vector<std::string> a, const std::vector<std::string>& b) {
    a.insert(a.end(), b.begin(), b.end());
    return a;
  };
  try {
    if (cmd == "gen") return cmd_gen(parse(argc, argv, {"--n", "--k", "--m", "--seed", "--out"}, {}));
    if (cmd == "recover")
      return cmd_recover(parse(argc, argv, with({"--problem", "--solver", "--out", "--out-x", "--threads", "--devices"},
                                                kSolverOpts),
                               {"--ignore-truth"}));
    if (cmd == "bench")
      return cmd_bench(parse(argc, argv, with({"--n", "--solver", "--seeds", "--out"}, kSolverOpts), {}));
    if (cmd == "matvec-bench")
      return cmd_matvec_bench(parse(argc, argv, {"--n", "--repeats", "--seed", "--out", "--device"}, {}));
    if (cmd == "deblur")
      return cmd_deblur(parse(argc, argv,
                              with({"--image", "--star-field", "--density", "--L", "--m", "--m-ratio", "--seed",
                                    "--out"},
                                   kSolverOpts),
                              {}));
    throw UsageError("unknown subcommand '" + cmd + "'");
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n" << kUsage;
    return kExitUsage;
  } catch (const DivergenceError& e) {
    std::cerr << "numerical failure: " << e.what() << "\n";
    return kExitNumerical;
  } catch (const SingularityError& e) {
    std::cerr << "numerical failure: " << e.what() << "\n";
    return kExitNumerical;
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
}
