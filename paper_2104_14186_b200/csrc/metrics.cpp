// Accuracy metrics of a computed (partial) decomposition A ~ U diag(sigma) V^T on
// the device (the reference's metrics.cpp:10-100, Eq. 5-7 of the paper):
//   orth = ||I - U^T U||_F / n   (historical 1/n scaling, metrics.hpp:9-10)
//   resid_right = max_i ||A v_i - sigma_i u_i||_2,  resid_left = max_i ||A^T u_i - sigma_i v_i||_2
//   (paper pairing: max ||A u_i - sigma_i v_i|| and max ||A v_i - sigma_i u_i||, square A)
//   value_err = ||sigma - delta||_F / ||delta||_F (host, when delta is given).
// Every O(mnk) product is a DMMA GEMM; the per-pair norms are the diagonal of
// R^T R for the residual block R.
#include <algorithm>
#include <cmath>
#include <vector>

#include "drivers.hpp"
#include "internal.hpp"

namespace qdwhg {

namespace {

double gram_defect(Ctx& ctx, const DMat& U) {
  const int64_t k = U.cols;
  const Arena::Mark mark = ctx.arena->mark();
  DMat G = ctx.arena->alloc(k, k);
  GemmExtra lo;
  lo.out = OutMode::LowerMirror;
  gemm(ctx, Op::T, Op::N, 1.0, U, U, 0.0, G, lo);
  axpby_identity(ctx, G, 1.0, -1.0, G);  // U^T U - I
  const double f = std::sqrt(mat_stats(ctx, G, false).fro2);
  ctx.arena->release_to(mark);
  return f;
}

// max_j || op(A) X(:, j) - sigma_j Y(:, j) ||_2
double max_pair_residual(Ctx& ctx, const DMat& A, const DMat& X, const std::vector<double>& sigma,
                         const DMat& Y, bool transpose_a) {
  const int64_t k = (int64_t)sigma.size();
  const int64_t rows = transpose_a ? A.cols : A.rows;
  const Arena::Mark mark = ctx.arena->mark();
  DMat R = ctx.arena->alloc(rows, k), D = ctx.arena->alloc(k, k), N = ctx.arena->alloc(k, k);
  std::vector<double> hd((size_t)k * k, 0.0);
  for (int64_t i = 0; i < k; ++i) hd[i + (size_t)i * k] = sigma[i];
  copy_from_host(ctx, hd.data(), k, D);
  gemm(ctx, transpose_a ? Op::T : Op::N, Op::N, 1.0, A, X, 0.0, R);
  gemm(ctx, Op::N, Op::N, -1.0, Y, D, 1.0, R);
  GemmExtra lo;
  lo.out = OutMode::Lower;
  gemm(ctx, Op::T, Op::N, 1.0, R, R, 0.0, N, lo);
  std::vector<double> d;
  diag_to_host(ctx, N, d);
  ctx.arena->release_to(mark);
  double worst = 0.0;
  for (double x : d) worst = std::max(worst, std::sqrt(std::max(x, 0.0)));
  return worst;
}

}  // namespace

AccuracyOut accuracy_report(Ctx& ctx, const DMat& A, const DMat& U, const std::vector<double>& sigma,
                            const DMat& V, const double* delta, bool paper_pairing) {
  const int64_t k = (int64_t)sigma.size();
  if (U.cols != k || V.cols != k)
    throw InvalidArgument("accuracy_report: sigma length must match U and V columns");
  if (U.rows != A.rows || V.rows != A.cols)
    throw InvalidArgument("accuracy_report: factor shapes do not conform with A");
  if (paper_pairing && A.rows != A.cols)
    throw InvalidArgument("accuracy_report: paper pairing needs a square A");
  AccuracyOut r;
  r.n = A.cols;
  r.k = k;
  const double nd = (double)std::max<int64_t>(r.n, 1);
  if (k > 0) {
    r.orth_left = gram_defect(ctx, U) / nd;
    r.orth_right = gram_defect(ctx, V) / nd;
  }
  if (delta) {
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < k; ++i) {
      const double d = sigma[i] - delta[i];
      num += d * d;
      den += delta[i] * delta[i];
    }
    r.has_value_err = true;
    r.value_err = den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
  }
  if (k > 0) {
    if (paper_pairing) {
      r.resid_left = max_pair_residual(ctx, A, U, sigma, V, false);
      r.resid_right = max_pair_residual(ctx, A, V, sigma, U, false);
    } else {
      r.resid_right = max_pair_residual(ctx, A, V, sigma, U, false);
      r.resid_left = max_pair_residual(ctx, A, U, sigma, V, true);
    }
  }
  return r;
}

}  // namespace qdwhg
