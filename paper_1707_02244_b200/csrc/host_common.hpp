// Host-side shared declarations of the circlasso_b200 library: status
// plumbing and the fp64 setup transforms (spectral norm, Gram inverse,
// composition, measurement) that run once per solve.
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/circlasso_b200.h"

namespace clb {

// Thread-local error message behind cl_last_error().
void set_error(const std::string& msg);
const std::string& last_error();

// Internal exception carrying a cl_status; caught at the C-ABI boundary
// (the reference throws its typed exceptions at the same places).
struct Failure {
  cl_status code;
  std::string msg;
};
[[noreturn]] inline void raise(cl_status code, const std::string& msg) { throw Failure{code, msg}; }

// ---- fp64 DFT (setup path; fft.hpp:46-89 semantics) ----------------------
using cplx = std::complex<double>;
// In-place unnormalized DFT of any length (sign -1 forward / +1 inverse).
void dft_inplace(std::vector<cplx>& a, bool inverse);
// Full spectrum of a real vector (fft.hpp:46-56).
std::vector<cplx> dft_real(const double* x, int64_t n);
// Inverse with 1/n and the imaginary-residue consistency check
// (fft.hpp:74-89, rel_tol 1e-10 of max(1, |re|_inf)); raises CL_ECONSIST.
void idft_real_checked(std::vector<cplx> f, double* out, double rel_tol = 1e-10);

// circulant.hpp:347-351
double spectral_norm(const double* c, int64_t n);
// circulant.hpp:297-320
void regularized_gram_inverse(const double* c, int64_t n, double rho, double sigma, double* b);
// circulant.hpp:324-333
void mask_gram_inverse(const int64_t* omega, int64_t m, int64_t n, double rho, double* d);
// circulant.hpp:337-343 with the identity short-circuit of deblur.hpp:53-64
void compose_rows(const double* c, const double* b, int64_t n, double* out);
// circulant.hpp:277-282 (y = P C x through the DFT, fp64)
void measure(const double* c, const int64_t* omega, int64_t n, int64_t m, const double* x, double* y);
// circulant.hpp:134-146
void check_mask(const int64_t* omega, int64_t m, int64_t n);

// matvec_scheme_bench inputs (parallel.hpp:343-348)
void scheme_bench_inputs(int64_t n, uint64_t seed, double* row, double* x);

// ---- artifact formats (io.hpp; io.cpp) ------------------------------------
void write_vector_file(const std::string& path, const double* v, int64_t n);
std::vector<double> read_vector_file(const std::string& path);
void write_operator_file(const std::string& path, int64_t n, int64_t m, const double* row, const int64_t* omega);
void read_operator_file(const std::string& path, std::vector<double>* row, std::vector<int64_t>* omega);
double bench_iters_per_second(const cl_bench_row& r);
void read_pgm_file(const std::string& path, std::vector<double>* px, int64_t* width, int64_t* height);
void write_pgm_file(const std::string& path, int64_t width, int64_t height, const double* px);
std::string bench_csv_header();
std::string bench_csv_row(const cl_bench_row& r);

}  // namespace clb
