/* circlasso_b200.h — C-ABI of the B200-native circulant LASSO engine.
 *
 * Drop-in boundary for the reference `circlasso` solver path (arxiv
 * 1707.02244).  The reference is a header-only C++20 library with no FFI;
 * each entry point below names the reference interface it replaces
 * (paths relative to /root/reference/proj/include/circlasso/).  A C++
 * adapter with the reference's own names and signatures
 * (circlasso_b200::ista_run, cadmm_run, SolverConfig, RecoveryReport, ...)
 * sits on top of this header in include/circlasso_b200.hpp; the Python
 * package paper_1707_02244_b200 binds the same symbols with ctypes.
 *
 * Conventions: plain pointers and sizes; host arrays are fp64 / int64 like
 * the reference (Eigen::VectorXd, std::vector<Eigen::Index>); the device
 * iterates in fp32.  No exception crosses the boundary: every call returns a
 * cl_status whose numbering mirrors the reference's exception hierarchy
 * (errors.hpp:12-72) and sets a thread-local message (cl_last_error).
 * A handle is not thread-safe, like the reference's solver states.
 */
#ifndef CIRCLASSO_B200_H_
#define CIRCLASSO_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CL_ABI_VERSION 3

/* errors.hpp:18-72 — one code per exception type, plus device failures. */
typedef enum cl_status {
  CL_OK = 0,
  CL_EDIM = 1,       /* DimensionError      errors.hpp:19-22 */
  CL_EPARAM = 2,     /* ParameterError      errors.hpp:25-28 */
  CL_ESINGULAR = 3,  /* SingularityError    errors.hpp:31-34 */
  CL_EDIVERGE = 4,   /* DivergenceError     errors.hpp:38-41 */
  CL_ECAPACITY = 5,  /* CapacityError       errors.hpp:44-47 */
  CL_EFORMAT = 6,    /* FormatError         errors.hpp:50-53 */
  CL_ECONSIST = 7,   /* ConsistencyError    errors.hpp:57-60 */
  CL_EPHASE = 8,     /* PhaseError          errors.hpp:63-72 */
  CL_ECUDA = 9,      /* CUDA runtime / launch failure (new) */
  CL_ECOMM = 10      /* collective failure in a sharded solve (new) */
} cl_status;

typedef enum cl_pairing { CL_PAIRING_LITERAL = 0, CL_PAIRING_PROXIMAL = 1 } cl_pairing; /* solvers.hpp:83 */
/* ISTA (solvers.hpp:208-263), circulant ADMM (:337-415) and the dense ADMM
 * baseline with its explicit n x n inverse (:267-327, the paper's PADMM). */
typedef enum cl_kind { CL_KIND_ISTA = 0, CL_KIND_CADMM = 1, CL_KIND_ADMM = 2 } cl_kind;
typedef enum cl_metric { CL_METRIC_MSE_VS_TRUTH = 0, CL_METRIC_ITERATE_CHANGE = 1 } cl_metric; /* solvers.hpp:130 */
/* Product engine (SolverConfig::use_fft, solvers.hpp:123): the direct
 * shift-indexed kernels (the paper's OpenCL scheme, north star) or the
 * on-device FFT (the reference's default; any n: non-power-of-two n runs as a
 * linear convolution in the next power of two >= 2n-1). */
typedef enum cl_engine { CL_ENGINE_DIRECT = 0, CL_ENGINE_FFT = 1 } cl_engine;

/* SolverConfig, solvers.hpp:112-125 (use_fft -> engine). */
typedef struct cl_config {
  double alpha;       /* l1 weight, default 1e-4 */
  double tau;         /* ISTA step, 0 = automatic 0.9 */
  double rho;         /* ADMM penalty, default 0.1 */
  double sigma;       /* cADMM z-split penalty, default 0.1 */
  double tau1;        /* dual step (v), default 1 */
  double tau2;        /* dual step (z), default 1 */
  int64_t max_iter;   /* default 100000 */
  double target_mse;  /* NaN = never stop early */
  int32_t check_every;/* default 10 */
  int32_t pairing;    /* cl_pairing, default literal */
  int32_t engine;     /* cl_engine, default CL_ENGINE_DIRECT */
  int64_t dense_cap;  /* largest n of the dense ADMM (CL_ECAPACITY above), default 4096 (circulant.hpp:31) */
} cl_config;

/* RecoveryReport, solvers.hpp:139-150 (final_x and the trace are returned
 * through caller-owned arrays). */
typedef struct cl_report {
  int64_t iterations;
  double setup_seconds;
  double total_seconds;
  uint64_t footprint_bytes;
  int32_t metric;          /* cl_metric */
  int32_t reached_target;
  double final_metric;
  int64_t trace_len;       /* number of check points (may exceed trace_cap) */
} cl_report;

typedef struct cl_solver cl_solver;

/* ---- library ------------------------------------------------------------ */
int cl_abi_version(void);
const char* cl_last_error(void);
void cl_config_default(cl_config* cfg);                 /* SolverConfig{} */
/* Number of CUDA devices visible; CL_ECUDA if the driver/runtime is absent. */
cl_status cl_device_count(int* count);

/* ---- problem generation (sensing.hpp, host, bit-exact) ------------------- */
/* make_problem sensing.hpp:198-207: c[n], omega[m] (sorted), x_true[n],
 * support[k] (sorted), y[m] = P C x_true (fp64, FFT-evaluated). */
cl_status cl_make_problem(int64_t n, int64_t m, int64_t k, uint64_t seed, double* c, int64_t* omega,
                          double* x_true, int64_t* support, double* y);
/* gen_sparse_signal sensing.hpp:129-145 */
cl_status cl_gen_sparse_signal(int64_t n, int64_t k, uint64_t seed, double* values, int64_t* support);
/* gen_circulant_sensing sensing.hpp:149-168 */
cl_status cl_gen_circulant_sensing(int64_t n, int64_t m, uint64_t seed, double* c, int64_t* omega);
/* measure sensing.hpp:171-182 (y = P C x, fp64) */
cl_status cl_measure(int64_t n, int64_t m, const double* c, const int64_t* omega, const double* x, double* y);
/* gen_star_field deblur.hpp:69-86 */
cl_status cl_gen_star_field(int64_t width, int64_t height, double density, uint64_t seed, double* pixels);
/* blur_matrix deblur.hpp:26-36 (first row) */
cl_status cl_blur_row(int64_t n, int64_t L, double* row);
/* compose_sensing deblur.hpp:53-64 first-row part (identity short-circuit
 * + circ_compose circulant.hpp:337-343) */
cl_status cl_compose_rows(int64_t n, const double* c, const double* b, double* out);

/* ---- setup operators (circulant.hpp, fp64) ------------------------------- */
cl_status cl_spectral_norm(int64_t n, const double* c, double* out);                 /* :347-351 */
cl_status cl_regularized_gram_inverse(int64_t n, const double* c, double rho, double sigma,
                                      double* b);                                   /* :297-320 */
cl_status cl_mask_gram_inverse(int64_t n, int64_t m, const int64_t* omega, double rho,
                               double* d);                                          /* :324-333 */

/* ---- device products (circulant.hpp:214-291, direct sm_100a kernels) ----
 * out = C x (transpose=0, rule C(i,j)=c[(j-i) mod n]) or C^T x; partial
 * forms gather/scatter through omega.  fp32 on device, host fp64 in/out. */
cl_status cl_circ_matvec(int device, int64_t n, const double* c, const double* x, int transpose,
                         double* out);                                              /* :216-274 */
cl_status cl_partial_matvec(int device, int64_t n, int64_t m, const double* c, const int64_t* omega,
                            const double* x, double* out_m);                        /* :277-282 */
cl_status cl_partial_transpose_matvec(int device, int64_t n, int64_t m, const double* c,
                                      const int64_t* omega, const double* r_m,
                                      double* out_n);                               /* :286-291 */

/* ---- solver handles (IstaState/CadmmState + *_setup, solvers.hpp) ------- */
/* ista_setup solvers.hpp:222-249 / cadmm_setup :359-395 / admm_setup
 * :285-314 (kind CL_KIND_ADMM: G = A~^T A~ + rho I and its inverse B built in
 * fp64 on the device; n <= cfg->dense_cap).  Validates exactly where the
 * reference throws; uploads the normalized operator to `device`. */
cl_status cl_solver_create(int kind, int64_t n, int64_t m, const double* c, const int64_t* omega,
                           const double* y, const cl_config* cfg, int device, cl_solver** out);
void cl_solver_destroy(cl_solver* s);
/* Optional ground truth: switches the check metric to MSE (run_loop :437). */
cl_status cl_solver_set_truth(cl_solver* s, const double* truth_n);
/* ista_step / cadmm_step x iters (solvers.hpp:252-263, 399-415), enqueued on
 * the solver's stream; asynchronous. */
cl_status cl_solver_step(cl_solver* s, int64_t iters);
/* One step that also computes the check metric (MSE vs truth if set, else
 * |x_t - x_{t-1}|/sqrt(n)) and the non-finite flag; synchronous. */
cl_status cl_solver_step_checked(cl_solver* s, double* metric, int* nonfinite);
/* run_loop solvers.hpp:426-472 + ista_run/cadmm_run :479-534: full solve
 * with the reference's check cadence and stopping rule.  final_x (n, may be
 * NULL) receives x (ISTA) or z (cADMM, dense ADMM); trace arrays may be NULL:
 * per check point the iteration, the metric and the seconds since the
 * iterations started (TracePoint, solvers.hpp:134-137). */
cl_status cl_solver_run(cl_solver* s, cl_report* rep, double* final_x, int64_t* trace_iter,
                        double* trace_value, double* trace_seconds, int64_t trace_cap);
/* Device -> host copy of a state vector by name:
 * ISTA: "x","r","delta","c","y"; cADMM: "x","z","nu","mu","v","beta","c","b","d","pty";
 * dense ADMM: "x","z","u","rhs","aty" (n each) and "B" (n * n, row-major). */
cl_status cl_solver_get(cl_solver* s, const char* field, double* out);
/* Host -> device (tests, warm state). Same names. */
cl_status cl_solver_set(cl_solver* s, const char* field, const double* in);
cl_status cl_solver_info(cl_solver* s, int64_t* n, int64_t* m, int64_t* t, double* scale,
                         double* threshold);
cl_status cl_solver_synchronize(cl_solver* s);
/* Elapsed device time (ms) of the last cl_solver_step call, CUDA events on
 * the solver's stream (for benchmarking). */
cl_status cl_solver_last_step_ms(cl_solver* s, double* ms);
/* Per-kernel device time of the last step (ms), by phase:
 * ISTA: [residual, residual_reduce, gradient, update]; cADMM: [ctv, beta,
 * bbeta, x, cx, duals]; dense ADMM: [primal, rhs].  `count` in/out. */
cl_status cl_solver_phase_ms(cl_solver* s, double* ms, int* count);
/* Per-phase event timing: 0 off (default), 1 eager launches, 2 event nodes
 * captured inside the step's CUDA graph (phase times of the replayed step). */
cl_status cl_solver_profile(cl_solver* s, int mode);
/* Mode 2 only: the per-phase times (ms) of each of the last graph replays,
 * oldest first, ms[k * nphase + i]; up to 256 replays are kept, so a timed
 * loop of back-to-back cl_solver_step(s, 1) calls needs no host
 * synchronization to be timed phase by phase.  ms = NULL queries *steps. */
cl_status cl_solver_phase_history(cl_solver* s, double* ms, int64_t max_steps, int64_t* steps, int* nphase);

/* ---- sharded solve (one process per GPU; row/output-range sharding) -----
 * The caller owns the collective: between phases it all-gathers the
 * per-shard slices this library exposes (e.g. torch.distributed NCCL on the
 * stream returned by cl_solver_stream).  Shard g of G owns outputs
 * [g*n/G, (g+1)*n/G) (rounded to the kernel tile) and the matching ISTA rows.
 * Results are bitwise identical for every G: no reduction crosses shards. */
cl_status cl_solver_shard(cl_solver* s, int rank, int world);
cl_status cl_solver_stream(cl_solver* s, void** cuda_stream);
/* Phase-level stepping for sharded solves: phase ids as in cl_solver_phase_ms;
 * ISTA: 0 = residual (local rows), 1 = gradient+update (local outputs);
 * cADMM: 0 = beta, 1 = x, 2 = duals; dense ADMM (unsharded; padmm_phases,
 * parallel.hpp:284-317): 0 = primal and dual update, 1 = right-hand side. */
cl_status cl_solver_run_phase(cl_solver* s, int phase);
/* Pure host helper (no device needed): the output range [out_lo, out_hi) and,
 * for ISTA, the residual row range [row_lo, row_hi) owned by shard `rank`. */
cl_status cl_shard_ranges(int kind, int64_t n, int64_t m, const int64_t* omega, int rank, int world,
                          int64_t* out_lo, int64_t* out_hi, int64_t* row_lo, int64_t* row_hi);
/* Device pointer + [begin,end) element range of the vector a phase produced,
 * and the full vector length, for the caller's all-gather. */
cl_status cl_solver_phase_output(cl_solver* s, int phase, void** dev_ptr, int64_t* begin,
                                 int64_t* end, int64_t* total);

/* ---- library-owned collectives (NCCL over NVLink) -------------
 * The sharded solve with the exchange inside the library: after each phase
 * every rank receives the other ranks' slices of the produced vector in place
 * (one ncclBroadcast per owner, grouped), on the solver's stream; the check
 * metrics are summed with one ncclAllReduce.  NCCL (libnccl.so.2) is loaded
 * at run time; without it these calls fail with CL_ECOMM.
 *
 * One process per GPU: rank 0 calls cl_comm_unique_id and hands the 128
 * bytes to the others (any channel); every rank calls cl_comm_init_rank, then
 * cl_solver_attach_comm on its solver.  From then on cl_solver_step /
 * cl_solver_step_checked / cl_solver_run run the sharded iteration and
 * return the same iterate on every rank, bitwise equal to the unsharded
 * solve.  The communicator must outlive the solver's use of it. */
typedef struct cl_comm cl_comm;
cl_status cl_comm_unique_id(unsigned char* id /* [128] */);                       /* ncclGetUniqueId */
cl_status cl_comm_init_rank(const unsigned char* id, int world, int rank, int device, cl_comm** out);
void cl_comm_destroy(cl_comm* c);
cl_status cl_solver_attach_comm(cl_solver* s, cl_comm* c);

/* One process per GPU without NCCL: CUDA IPC peer stores.  Each rank calls
 * cl_solver_peer_export(s, rank, world, blob) (shards the solver and makes
 * its exchange vectors IPC-exportable), the caller hands every rank's
 * CL_PEER_BLOB_BYTES-byte blob to every rank in rank order (any channel), and
 * each rank calls cl_solver_peer_attach(s, blobs).  From then on
 * cl_solver_step / _step_checked / cl_solver_run run the sharded iteration:
 * each phase's epilogue kernel stores its slice into every rank's copy of
 * the vector (NVLink peer stores), and the ranks order their phases through
 * system-scope flags -- no separate all-gather, no NCCL.  At most 8 ranks;
 * destroying the solvers is collective (a final barrier). */
#define CL_PEER_BLOB_BYTES 512
cl_status cl_solver_peer_export(cl_solver* s, int rank, int world, unsigned char* blob);
cl_status cl_solver_peer_attach(cl_solver* s, const unsigned char* blobs /* world x CL_PEER_BLOB_BYTES */);

/* One process driving several GPUs (or several shards of one GPU): a group of
 * `ndev` solvers, rank r on devices[r].  Transport CL_TRANSPORT_NCCL builds
 * the communicators with ncclCommInitAll and issues every rank's exchange in
 * one NCCL group; CL_TRANSPORT_COPY exchanges slices with peer copies ordered
 * by events (devices may repeat: the 2/4/8-rank data plane on one GPU);
 * CL_TRANSPORT_PEER fuses the exchange into the kernels that produce each
 * slice (their stores go to every rank's copy; peer access over NVLink, at
 * most 8 ranks), leaving only event ordering between the phases.  The
 * run loop, stopping rule and report are those of cl_solver_run; get()
 * assembles a vector from the ranks' slices.  ISTA and cADMM (direct
 * engine). */
typedef enum cl_transport { CL_TRANSPORT_NCCL = 0, CL_TRANSPORT_COPY = 1, CL_TRANSPORT_PEER = 2 } cl_transport;
typedef struct cl_group cl_group;
cl_status cl_group_create(int kind, int64_t n, int64_t m, const double* c, const int64_t* omega, const double* y,
                          const cl_config* cfg, const int* devices, int ndev, int transport, cl_group** out);
void cl_group_destroy(cl_group* g);
cl_status cl_group_set_truth(cl_group* g, const double* truth_n);
cl_status cl_group_step(cl_group* g, int64_t iters);
cl_status cl_group_run(cl_group* g, cl_report* rep, double* final_x, int64_t* trace_iter, double* trace_value,
                       double* trace_seconds, int64_t trace_cap);
cl_status cl_group_get(cl_group* g, const char* field, double* out);
cl_status cl_group_synchronize(cl_group* g);
cl_status cl_group_info(cl_group* g, int* world, int64_t* t, int* transport);

/* ---- artifact formats (io.hpp:1-170) -------------------------------------
 * Vectors: magic "CIRCVEC1", u64 length, little-endian f64 data.
 * Operators: magic "CIRCOPR1", u64 n, u64 m, f64 first row[n], u64 omega[m].
 * Errors are CL_EFORMAT with the reference's messages ("cannot open", "bad
 * magic", "truncated ...", "m exceeds n").  Readers report the stored sizes
 * in *len / *n, *m; a NULL or too-small output buffer only queries them. */
cl_status cl_write_vector(const char* path, const double* v, int64_t n);          /* io.hpp:80-87 */
cl_status cl_read_vector(const char* path, double* out, int64_t cap, int64_t* len); /* io.hpp:89-97 */
cl_status cl_write_operator(const char* path, int64_t n, int64_t m, const double* row,
                            const int64_t* omega);                                   /* io.hpp:99-112 */
cl_status cl_read_operator(const char* path, double* row, int64_t cap_n, int64_t* omega, int64_t cap_m,
                           int64_t* n, int64_t* m);                                  /* io.hpp:114-131 */
/* Binary PGM images (image.hpp:56-153): read P5 with maxval 1..255 into
 * [0, 1] intensities (row-major; a NULL or too-small buffer only reports the
 * size); write P5/255 with the intensities clamped to [0, 1] and rounded to 8
 * bits.  CL_EFORMAT with the reference's messages. */
cl_status cl_write_pgm(const char* path, int64_t width, int64_t height, const double* pixels);
cl_status cl_read_pgm(const char* path, double* pixels, int64_t cap, int64_t* width, int64_t* height);
/* One benchmark run in the reference's pinned CSV schema (io.hpp:133-170). */
typedef struct cl_bench_row {
  const char* algorithm;
  int64_t n, m, k;
  uint64_t seed;
  int64_t iterations;
  double setup_seconds, total_seconds, final_mse;
  uint64_t footprint_bytes;
  const char* status;
} cl_bench_row;
/* iterations / (total - setup), 0 without active time or iterations (io.hpp:148-152) */
double cl_bench_iters_per_second(const cl_bench_row* row);
/* The header line / one row, without the newline, formatted exactly as the
 * reference's std::ostream writer; *len = the text length (buf may be NULL). */
cl_status cl_bench_csv_header(char* buf, int64_t cap, int64_t* len);
cl_status cl_bench_csv_row(const cl_bench_row* row, char* buf, int64_t cap, int64_t* len);

/* ---- matvec scheme benchmark (parallel.hpp:318-406; the paper's Fig. 5) ---
 * `repeats` timed products (CUDA events) of the same seeded Gaussian circulant
 * and input: scheme 0 = the direct circulant engine (2n unique fetches),
 * scheme 1 = a dense row-major copy streamed by a plain GEMV (n^2 + n unique
 * fetches; CL_ECAPACITY above dense_cap, the reference's kDenseCap = 4096 by
 * default; B200's 180 GB allow fp32 copies up to n = 2^17).  fp32 on device. */
cl_status cl_matvec_scheme_bench(int device, int64_t n, int scheme, int repeats, uint64_t seed, int64_t dense_cap,
                                 double* min_s, double* mean_s, uint64_t* unique_fetches, uint64_t* vector_fetches,
                                 double* checksum);

/* ---- roofline helper ----------------------------------------------------- */
/* FP32 FFMA peak microbenchmark on `device` (TFLOP/s), the roofline
 * denominator for the direct engine. */
cl_status cl_ffma_peak(int device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* CIRCLASSO_B200_H_ */
