// Host orchestration of the QDWHpartial algorithms on device views (DMat).
// Each function restates the control flow of the reference driver it cites;
// every O(n^2)/O(n^3) step is a device kernel, the host only handles scalars
// (Halley weights, the diag(R) scan, counts) and launches.
#pragma once
#include <array>
#include <vector>

#include "internal.hpp"
#include "scalars.hpp"

namespace qdwhg {


struct StageClock {
  explicit StageClock(Ctx& c);
  ~StageClock();
  void mark(int stage);  // everything since the previous mark is charged to `stage`
  void finish(double* stage_seconds, double* total);
  Ctx& ctx;
  std::vector<cudaEvent_t> ev;
  std::vector<int> owner;
};

// polar.cpp:82-128.  Xout may alias X.
void qdwh_chol_step(Ctx& ctx, const DMat& X, const WeightStep& w, const DMat& Xout,
                    bool symmetric = false);
// polar.cpp:53-80.  Xout may alias X.
void qdwh_qr_step(Ctx& ctx, const DMat& X, const WeightStep& w, const DMat& Xout);

struct FixedIterResult {
  double ell = 0;
  std::vector<double> trace;
  size_t iters_qr = 0, iters_chol = 0;
};
// polar.cpp:179-215, in place on X.  qr_first: FixedVariant::QrFirst.
FixedIterResult run_fixed_iterations(Ctx& ctx, const DMat& X, double ell0, size_t iters,
                                     bool qr_first, bool known_symmetric = false);

struct PolarOut {
  double alpha = 0;
  size_t iters_qr = 0, iters_chol = 0;
  std::vector<double> trace;
  double flops = 0;
};
struct PolarCfg {
  double ell0 = 1e-15;
  size_t max_iters = 60;
  double conv_eps = 2.220446049250313e-16;
  double chol_switch_c = 100.0;
  int force_variant = 0;  // 0 Auto, 1 QrOnly, 2 CholeskyOnly
};
// polar.cpp:130-177.  Up (m x n) and H (n x n, optional: H.base == nullptr to skip).
PolarOut polar_decompose(Ctx& ctx, const DMat& A, const PolarCfg& cfg, const DMat& Up,
                         const DMat& H);
// Full-spectrum drivers (fullsolve.cpp:76-103): all eigenpairs (ascending) by QDWH
// spectral divide-and-conquer down to base_size (returns the depth); all singular
// triplets (descending) via the polar factor.
int64_t eig_full(Ctx& ctx, const DMat& A, int64_t base_size, std::vector<double>& vals, const DMat& Vout);
void svd_full(Ctx& ctx, const DMat& A, int64_t base_size, const DMat& U, std::vector<double>& sigma,
              const DMat& V);
// metrics.cpp:58-100 (accuracy_report) on the device.
struct AccuracyOut {
  double orth_left = 0, orth_right = 0, value_err = 0, resid_right = 0, resid_left = 0;
  bool has_value_err = false;
  int64_t n = 0, k = 0;
};
AccuracyOut accuracy_report(Ctx& ctx, const DMat& A, const DMat& U, const std::vector<double>& sigma,
                            const DMat& V, const double* delta, bool paper_pairing);
// Lower bound of sigma_min(A) / ||A||_2 for the polar's l0 (QR of A, R^-1 power iteration).
double polar_ell0_estimate(Ctx& ctx, const DMat& A);
double ell0_lower_bound(Ctx& ctx, const DMat& R, double alpha);

// svd_dense (kernels.cpp:217-330) restated for the device as polar + EIG
// (fullsolve.cpp:82-103): U (m x n), sigma descending (host), V (n x n).
// Returns the number k of singular vectors formed (those with sigma > cut).
int64_t svd_polar(Ctx& ctx, const DMat& A, const DMat& U, std::vector<double>& sigma, const DMat& V,
                  double cut = -1.0, double ell0 = 1e-15);

struct EigOut {
  std::vector<double> lambda;  // ascending
  DMat V;                      // n x k, in the arena
  double mu = 0, shift = 0, tol = 0.01;
  size_t rank_index = 0, subspace_size = 0, iters_qr = 0, iters_chol = 0, borderline = 0;
  bool no_savings = false, randomized = false;
  int subspace_path = 0;  // 0 Householder QR of B, 1 Cholesky-QR extraction
  std::vector<double> trace;
  double flops = 0;
};
// partial.cpp:40-99 (Alg. 1).
EigOut partial_eig(Ctx& ctx, const DMat& A, double s, size_t iters, bool randomize, double tol,
                   uint64_t seed, StageClock* clk);

struct SvdOut {
  std::vector<double> sigma;  // descending
  DMat U, V;                  // m x k, n x k in the arena
  double alpha = 0, threshold = 0, tol = 0.01;
  size_t rank_index = 0, subspace_size = 0, iters_qr = 0, iters_chol = 0;
  bool no_savings = false, randomized = false;
  std::vector<double> trace;
  double flops = 0;
};
// partial.cpp:101-158 (Alg. 2).  If s_abs > 0 the threshold is s = s_abs/alpha.
SvdOut partial_svd(Ctx& ctx, const DMat& A, double s, double s_abs, double tol, bool randomize,
                   uint64_t seed, StageClock* clk);

}  // namespace qdwhg
