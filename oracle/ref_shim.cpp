// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference implementation compiled from
// /root/reference/proj/core/src/*.cpp (see oracle/Makefile).  It lets the
// Python tests, the golden-vector generator (tests/golden/make_golden.py) and
// bench.py's reference/cpu_baseline legs call the reference's own code path:
//   qdwh::qdwh_partial_eig   (partial.hpp:55-57, partial.cpp:40-99)
//   qdwh::qdwh_partial_svd   (partial.hpp:85-86, partial.cpp:101-158)
//   qdwh::polar_decompose    (polar.hpp:60,      polar.cpp:130-177)
//   qdwh::qdwh_eig_full / qdwh_svd_full (fullsolve.hpp:21-24), qdwh::accuracy_report
//   (metrics.hpp:25-28)
// plus the kernels/scalars the parity tests pin one by one.
// Status codes mirror include/qdwhg.h: 0 ok, 1 invalid_argument,
// 2 NotPositiveDefinite, 3 NotConverged, 8 other.
#include <cstdint>
#include <cstring>
#include <limits>
#include <optional>
#include <vector>
#include <stdexcept>
#include <string>

#include "qdwh/fullsolve.hpp"
#include "qdwh/kernels.hpp"
#include "qdwh/matgen.hpp"
#include "qdwh/metrics.hpp"
#include "qdwh/partial.hpp"
#include "qdwh/polar.hpp"

using namespace qdwh;

namespace {
thread_local std::string g_err;

DenseMatrix load(const double* a, int64_t m, int64_t n) {
  DenseMatrix x(static_cast<size_t>(m), static_cast<size_t>(n));
  if (m * n > 0) std::memcpy(x.data(), a, sizeof(double) * m * n);
  return x;
}
void store(const DenseMatrix& x, double* out) {
  if (out && x.rows() * x.cols() > 0) std::memcpy(out, x.data(), sizeof(double) * x.rows() * x.cols());
}
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const NotPositiveDefinite& e) {
    g_err = e.what();
    return 2;
  } catch (const NotConverged& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 8;
  }
}
}  // namespace

extern "C" {

// info layout (doubles): [0]=mu|alpha [1]=shift|threshold [2]=rank_index [3]=subspace_size
// [4]=k [5]=iters_qr [6]=iters_chol [7]=borderline [8]=no_savings [9]=randomized
// [10]=n_trace [11..11+n_trace) = ell_trace (max 48 entries)
enum { INFO_LEN = 64 };

const char* ref_last_error() { return g_err.c_str(); }

int ref_partial_eig(int64_t n, const double* a, int64_t iters, int randomize, double tol,
                    uint64_t seed, double* lambda, double* v, int64_t kcap, double* info) {
  return guard([&] {
    const ShiftPlan plan = choose_shift(static_cast<size_t>(iters));
    PartialEigResult r = qdwh_partial_eig(load(a, n, n), plan, randomize != 0, tol, Seed{seed});
    std::memset(info, 0, sizeof(double) * INFO_LEN);
    info[0] = r.mu;
    info[1] = r.shift;
    info[2] = static_cast<double>(r.rank_index);
    info[3] = static_cast<double>(r.subspace_size);
    info[4] = static_cast<double>(r.count());
    info[5] = static_cast<double>(r.diagnostics.iters_qr);
    info[6] = static_cast<double>(r.diagnostics.iters_chol);
    info[7] = static_cast<double>(r.diagnostics.borderline);
    info[8] = r.diagnostics.no_savings;
    info[9] = r.diagnostics.randomized;
    const size_t nt = std::min<size_t>(r.diagnostics.ell_trace.size(), 48);
    info[10] = static_cast<double>(nt);
    for (size_t i = 0; i < nt; ++i) info[11 + i] = r.diagnostics.ell_trace[i];
    if (static_cast<int64_t>(r.count()) > kcap) throw std::runtime_error("k exceeds kcap");
    for (size_t i = 0; i < r.count(); ++i) lambda[i] = r.lambda_minus[i];
    store(r.v, v);
  });
}

int ref_partial_svd(int64_t m, int64_t n, const double* a, double s, double tol, int randomize,
                    uint64_t seed, double* sigma, double* u, double* v, int64_t kcap,
                    double* info) {
  return guard([&] {
    PartialSvdResult r = qdwh_partial_svd(load(a, m, n), s, tol, randomize != 0, Seed{seed});
    std::memset(info, 0, sizeof(double) * INFO_LEN);
    info[0] = r.alpha;
    info[1] = r.threshold;
    info[2] = static_cast<double>(r.diagnostics.rank_index);
    info[3] = static_cast<double>(r.subspace_size);
    info[4] = static_cast<double>(r.count());
    info[5] = static_cast<double>(r.diagnostics.iters_qr);
    info[6] = static_cast<double>(r.diagnostics.iters_chol);
    info[8] = r.diagnostics.no_savings;
    info[9] = r.diagnostics.randomized;
    const size_t nt = std::min<size_t>(r.diagnostics.ell_trace.size(), 48);
    info[10] = static_cast<double>(nt);
    for (size_t i = 0; i < nt; ++i) info[11 + i] = r.diagnostics.ell_trace[i];
    if (static_cast<int64_t>(r.count()) > kcap) throw std::runtime_error("k exceeds kcap");
    for (size_t i = 0; i < r.count(); ++i) sigma[i] = r.sigma1[i];
    store(r.u1, u);
    store(r.v1, v);
  });
}

// variant: 0 Auto, 1 QrOnly, 2 CholeskyOnly.  info: [0]=alpha [5]=iters_qr [6]=iters_chol
// [10]=n_trace [11..] trace
int ref_polar(int64_t m, int64_t n, const double* a, double ell0, int64_t max_iters,
              double chol_switch_c, int variant, double* up, double* h, double* info) {
  return guard([&] {
    PolarConfig cfg;
    cfg.ell0 = ell0;
    cfg.max_iters = static_cast<size_t>(max_iters);
    cfg.chol_switch_c = chol_switch_c;
    cfg.force_variant = variant == 1   ? PolarVariant::QrOnly
                        : variant == 2 ? PolarVariant::CholeskyOnly
                                       : PolarVariant::Auto;
    PolarResult r = polar_decompose(load(a, m, n), cfg);
    std::memset(info, 0, sizeof(double) * INFO_LEN);
    info[0] = r.alpha;
    info[5] = static_cast<double>(r.iters_qr);
    info[6] = static_cast<double>(r.iters_chol);
    const size_t nt = std::min<size_t>(r.ell_trace.size(), 48);
    info[10] = static_cast<double>(nt);
    for (size_t i = 0; i < nt; ++i) info[11 + i] = r.ell_trace[i];
    store(r.up, up);
    store(r.h, h);
  });
}

int ref_halley_weights(double ell, double* out5) {
  return guard([&] {
    const WeightStep w = halley_weights(ell);
    out5[0] = w.a;
    out5[1] = w.b;
    out5[2] = w.c;
    out5[3] = w.ell_in;
    out5[4] = w.ell_out;
  });
}

int ref_iterations_to_converge(double ell0, double eps, int64_t max_iters, int64_t* out) {
  return guard([&] { *out = static_cast<int64_t>(iterations_to_converge(ell0, eps, max_iters)); });
}

int ref_gaussian_matrix(int64_t m, int64_t n, uint64_t seed, double* out) {
  return guard([&] { store(gaussian_matrix(m, n, Seed{seed}), out); });
}

int ref_qr_factor(int64_t m, int64_t n, const double* a, double* q, double* r) {
  return guard([&] {
    QrFactors f = qr_factor(load(a, m, n));
    store(f.q, q);
    store(f.r, r);
  });
}

int ref_cholesky(int64_t n, const double* z, double* w) {
  return guard([&] { store(cholesky(load(z, n, n)), w); });
}

int ref_sym_eig_dense(int64_t n, const double* s, double* values, double* vectors) {
  return guard([&] {
    SymEig e = sym_eig_dense(load(s, n, n));
    for (int64_t i = 0; i < n; ++i) values[i] = e.values[i];
    store(e.vectors, vectors);
  });
}

int ref_svd_dense(int64_t m, int64_t n, const double* a, double* u, double* sigma, double* v) {
  return guard([&] {
    Svd s = svd_dense(load(a, m, n));
    for (size_t i = 0; i < s.sigma.size(); ++i) sigma[i] = s.sigma[i];
    store(s.u, u);
    store(s.v, v);
  });
}

int ref_two_norm_estimate(int64_t m, int64_t n, const double* a, double* out) {
  return guard([&] { *out = two_norm_estimate(load(a, m, n)); });
}

int ref_lanczos_min_bound(int64_t n, const double* a, int64_t steps, double* out) {
  return guard([&] { *out = lanczos_min_bound(load(a, n, n), static_cast<size_t>(steps)); });
}

int ref_qdwh_chol_step(int64_t m, int64_t n, const double* x, double ell, double* out) {
  return guard([&] { store(qdwh_chol_step(load(x, m, n), halley_weights(ell)), out); });
}

int ref_qdwh_qr_step(int64_t m, int64_t n, const double* x, double ell, double* out) {
  return guard([&] { store(qdwh_qr_step(load(x, m, n), halley_weights(ell)), out); });
}

// variant: 0 QrFirst, 1 CholeskyOnly
int ref_run_fixed_iterations(int64_t m, int64_t n, const double* x0, double ell0, int64_t iters,
                             int variant, double* out, double* info) {
  return guard([&] {
    FixedIterResult r = run_fixed_iterations(
        load(x0, m, n), ell0, static_cast<size_t>(iters),
        variant == 0 ? FixedVariant::QrFirst : FixedVariant::CholeskyOnly);
    std::memset(info, 0, sizeof(double) * INFO_LEN);
    info[0] = r.ell;
    info[5] = static_cast<double>(r.iters_qr);
    info[6] = static_cast<double>(r.iters_chol);
    const size_t nt = std::min<size_t>(r.ell_trace.size(), 48);
    info[10] = static_cast<double>(nt);
    for (size_t i = 0; i < nt; ++i) info[11 + i] = r.ell_trace[i];
    store(r.x, out);
  });
}

int ref_gen_sym_eig_test(int64_t n, int64_t k, uint64_t seed, double* a, double* d) {
  return guard([&] {
    SymEigTestMatrix g = gen_sym_eig_test(n, k, Seed{seed});
    store(g.a, a);
    for (int64_t i = 0; i < n; ++i) d[i] = g.d[i];
  });
}

int ref_gen_svd_test(int64_t n, uint64_t seed, double* a, double* d) {
  return guard([&] {
    SvdTestMatrix g = gen_svd_test(n, Seed{seed});
    store(g.a, a);
    for (int64_t i = 0; i < n; ++i) d[i] = g.d[i];
  });
}

int ref_eig_full(int64_t n, const double* a, int64_t base, double* lambda, double* v, int64_t* depth) {
  return guard([&] {
    EigResult r = qdwh_eig_full(load(a, n, n), static_cast<size_t>(base));
    for (int64_t i = 0; i < n; ++i) lambda[i] = r.lambda[i];
    store(r.v, v);
    *depth = static_cast<int64_t>(r.depth);
  });
}

int ref_svd_full(int64_t m, int64_t n, const double* a, int64_t base, double* u, double* sigma, double* v) {
  return guard([&] {
    SvdResult r = qdwh_svd_full(load(a, m, n), static_cast<size_t>(base));
    for (int64_t i = 0; i < n; ++i) sigma[i] = r.sigma[i];
    store(r.u, u);
    store(r.v, v);
  });
}

// out: [0] orth_left [1] orth_right [2] value_err (NaN if none) [3] resid_right [4] resid_left
int ref_accuracy_report(int64_t m, int64_t n, const double* a, int64_t k, const double* u,
                        const double* sigma, const double* v, const double* delta, int paper,
                        double* out) {
  return guard([&] {
    std::vector<double> sg(sigma, sigma + k);
    std::optional<std::vector<double>> dl;
    if (delta) dl = std::vector<double>(delta, delta + k);
    AccuracyReport r = accuracy_report(load(a, m, n), load(u, m, k), sg, load(v, n, k), dl, paper != 0);
    out[0] = r.orth_left;
    out[1] = r.orth_right;
    out[2] = r.value_err ? *r.value_err : std::numeric_limits<double>::quiet_NaN();
    out[3] = r.resid_right;
    out[4] = r.resid_left;
  });
}

}  // extern "C"
