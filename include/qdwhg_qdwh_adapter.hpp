// qdwhg_qdwh_adapter.hpp — header-only drop-in for the reference's qdwh:: driver
// entry points, implemented on libqdwhg (include/qdwhg.h).
//
// A reference user replaces
//     #include "qdwh/partial.hpp"   ...   qdwh::qdwh_partial_eig(a, plan, ...)
// by
//     #include "qdwhg_qdwh_adapter.hpp" ...   qdwhg::qdwh_partial_eig(a, plan, ...)
// with the same argument lists, result structs and exceptions as
//   qdwh::qdwh_partial_eig  partial.hpp:55-57
//   qdwh::qdwh_partial_svd  partial.hpp:85-86
//   qdwh::polar_decompose   polar.hpp:60
//   qdwh::qdwh_eig_full / qdwh_svd_full   fullsolve.hpp:21-24
//   qdwh::accuracy_report   metrics.hpp:25-28
// The reference's own types (qdwh::DenseMatrix, ShiftPlan, PartialEigResult, ...)
// are used unchanged; link with -lqdwhg (paper_2104_14186_b200/lib/libqdwhg.so).
#pragma once

#include <memory>
#include <optional>
#include <vector>
#include <stdexcept>
#include <string>

#include "qdwh/fullsolve.hpp"
#include "qdwh/metrics.hpp"
#include "qdwh/partial.hpp"
#include "qdwh/polar.hpp"
#include "qdwhg.h"

namespace qdwhg {

inline void throw_status(qdwhg_status st, const qdwhg_handle* h) {
  const std::string msg = h ? qdwhg_last_error(h) : "qdwhg error";
  switch (st) {
    case QDWHG_OK: return;
    case QDWHG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case QDWHG_NOT_POSITIVE_DEFINITE: throw qdwh::NotPositiveDefinite(msg);
    case QDWHG_NOT_CONVERGED: throw qdwh::NotConverged(msg);
    default: throw std::runtime_error(msg);
  }
}

// One handle per thread (a handle is single-threaded, like a reference call).
inline qdwhg_handle* thread_handle() {
  struct Holder {
    qdwhg_handle* h = nullptr;
    ~Holder() { qdwhg_destroy(h); }
  };
  thread_local Holder holder;
  if (!holder.h) {
    qdwhg_options o{-1, 0, 0, 0};
    throw_status(qdwhg_create(&holder.h, &o), nullptr);
  }
  return holder.h;
}

inline qdwh::PartialEigResult qdwh_partial_eig(const qdwh::DenseMatrix& a,
                                               const qdwh::ShiftPlan& plan,
                                               bool use_randomization = false, double tol = 0.01,
                                               qdwh::Seed seed = {}) {
  qdwhg_handle* h = thread_handle();
  const int64_t n = static_cast<int64_t>(a.rows());
  if (a.cols() != a.rows()) throw std::invalid_argument("qdwh_partial_eig: matrix not square");
  std::vector<double> lam(n);
  qdwh::DenseMatrix v(n, n);
  qdwhg_eig_info info{};
  throw_status(qdwhg_partial_eig(h, n, a.data(), n, (int64_t)plan.qdwh_iters, use_randomization,
                                 tol, seed.value, lam.data(), v.data(), n, n, &info),
               h);
  qdwh::PartialEigResult r;
  r.lambda_minus.assign(lam.begin(), lam.begin() + info.k);
  r.v = qdwh::column_block(v, 0, static_cast<size_t>(info.k));
  r.subspace_size = static_cast<size_t>(info.subspace_size);
  r.mu = info.mu;
  r.shift = info.shift;
  r.rank_index = static_cast<size_t>(info.rank_index);
  r.diagnostics.ell_trace.assign(info.ell_trace, info.ell_trace + info.n_trace);
  r.diagnostics.tol = info.tol;
  r.diagnostics.iters_qr = static_cast<size_t>(info.iters_qr);
  r.diagnostics.iters_chol = static_cast<size_t>(info.iters_chol);
  r.diagnostics.borderline = static_cast<size_t>(info.borderline);
  r.diagnostics.no_savings = info.no_savings != 0;
  r.diagnostics.randomized = info.randomized != 0;
  return r;
}

inline qdwh::PartialSvdResult qdwh_partial_svd(const qdwh::DenseMatrix& a, double s,
                                               double tol = 0.01, bool use_randomization = false,
                                               qdwh::Seed seed = {}) {
  qdwhg_handle* h = thread_handle();
  const int64_t m = static_cast<int64_t>(a.rows()), n = static_cast<int64_t>(a.cols());
  std::vector<double> sig(n);
  qdwh::DenseMatrix u(m, n), v(n, n);
  qdwhg_svd_info info{};
  throw_status(qdwhg_partial_svd(h, m, n, a.data(), m, s, tol, use_randomization, seed.value,
                                 sig.data(), u.data(), m, v.data(), n, n, &info),
               h);
  qdwh::PartialSvdResult r;
  r.sigma1.assign(sig.begin(), sig.begin() + info.k);
  r.u1 = qdwh::column_block(u, 0, static_cast<size_t>(info.k));
  r.v1 = qdwh::column_block(v, 0, static_cast<size_t>(info.k));
  r.subspace_size = static_cast<size_t>(info.subspace_size);
  r.alpha = info.alpha;
  r.threshold = info.threshold;
  r.diagnostics.ell_trace.assign(info.ell_trace, info.ell_trace + info.n_trace);
  r.diagnostics.tol = info.tol;
  r.diagnostics.iters_qr = static_cast<size_t>(info.iters_qr);
  r.diagnostics.iters_chol = static_cast<size_t>(info.iters_chol);
  r.diagnostics.rank_index = static_cast<size_t>(info.rank_index);
  r.diagnostics.no_savings = info.no_savings != 0;
  r.diagnostics.randomized = info.randomized != 0;
  return r;
}

inline qdwh::PolarResult polar_decompose(const qdwh::DenseMatrix& a,
                                         const qdwh::PolarConfig& cfg = {}) {
  qdwhg_handle* h = thread_handle();
  const int64_t m = static_cast<int64_t>(a.rows()), n = static_cast<int64_t>(a.cols());
  qdwhg_polar_config c{cfg.ell0, (int64_t)cfg.max_iters, cfg.conv_eps, cfg.chol_switch_c,
                       cfg.force_variant == qdwh::PolarVariant::QrOnly         ? 1
                       : cfg.force_variant == qdwh::PolarVariant::CholeskyOnly ? 2
                                                                               : 0,
                       0};
  qdwh::PolarResult r;
  r.up = qdwh::DenseMatrix(m, n);
  r.h = qdwh::DenseMatrix(n, n);
  qdwhg_polar_info info{};
  throw_status(qdwhg_polar(h, m, n, a.data(), m, &c, r.up.data(), m, r.h.data(), n, &info), h);
  r.alpha = info.alpha;
  r.iters_qr = static_cast<size_t>(info.iters_qr);
  r.iters_chol = static_cast<size_t>(info.iters_chol);
  r.ell_trace.assign(info.ell_trace, info.ell_trace + info.n_trace);
  r.converged = info.converged != 0;
  return r;
}

inline qdwh::EigResult qdwh_eig_full(const qdwh::DenseMatrix& a, std::size_t base_size = 32) {
  qdwhg_handle* h = thread_handle();
  const int64_t n = static_cast<int64_t>(a.rows());
  if (a.cols() != a.rows()) throw std::invalid_argument("qdwh_eig_full: matrix not square");
  qdwh::EigResult r;
  r.lambda.resize(n);
  r.v = qdwh::DenseMatrix(n, n);
  int64_t depth = 0;
  throw_status(qdwhg_eig_full(h, n, a.data(), n, static_cast<int64_t>(base_size), r.lambda.data(),
                              r.v.data(), n, &depth),
               h);
  r.depth = static_cast<std::size_t>(depth);
  return r;
}

inline qdwh::SvdResult qdwh_svd_full(const qdwh::DenseMatrix& a, std::size_t base_size = 32) {
  qdwhg_handle* h = thread_handle();
  const int64_t m = static_cast<int64_t>(a.rows()), n = static_cast<int64_t>(a.cols());
  qdwh::SvdResult r;
  r.u = qdwh::DenseMatrix(m, n);
  r.sigma.resize(n);
  r.v = qdwh::DenseMatrix(n, n);
  throw_status(qdwhg_svd_full(h, m, n, a.data(), m, static_cast<int64_t>(base_size), r.u.data(), m,
                              r.sigma.data(), r.v.data(), n),
               h);
  return r;
}

inline qdwh::AccuracyReport accuracy_report(const qdwh::DenseMatrix& a, const qdwh::DenseMatrix& u,
                                            const std::vector<double>& sigma, const qdwh::DenseMatrix& v,
                                            const std::optional<std::vector<double>>& delta = std::nullopt,
                                            bool paper_pairing = false) {
  qdwhg_handle* h = thread_handle();
  if (delta && delta->size() != sigma.size())
    throw std::invalid_argument("accuracy_report: delta length differs from sigma");
  qdwhg_accuracy out{};
  throw_status(qdwhg_accuracy_report(h, static_cast<int64_t>(a.rows()), static_cast<int64_t>(a.cols()),
                                     a.data(), static_cast<int64_t>(a.rows()),
                                     static_cast<int64_t>(sigma.size()), u.data(),
                                     static_cast<int64_t>(u.rows()), sigma.data(), v.data(),
                                     static_cast<int64_t>(v.rows()), delta ? delta->data() : nullptr,
                                     paper_pairing ? 1 : 0, &out),
               h);
  qdwh::AccuracyReport r;
  r.orth_left = out.orth_left;
  r.orth_right = out.orth_right;
  if (out.has_value_err) r.value_err = out.value_err;
  r.resid_right = out.resid_right;
  r.resid_left = out.resid_left;
  r.n = static_cast<std::size_t>(out.n);
  r.k = static_cast<std::size_t>(out.k);
  return r;
}

}  // namespace qdwhg
