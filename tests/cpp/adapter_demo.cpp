// Drop-in demo: the same call site through the reference (qdwh::) and through
// libqdwhg via include/qdwhg_qdwh_adapter.hpp (qdwhg::).  Built against the
// untouched reference headers by tests/test_integration.py; run on a GPU box.
#include <cmath>
#include <cstdio>

#include "qdwh/matgen.hpp"
#include "qdwhg_qdwh_adapter.hpp"

int main() {
  const qdwh::SymEigTestMatrix gen = qdwh::gen_sym_eig_test(256, 26, qdwh::Seed{1});
  const qdwh::ShiftPlan plan = qdwh::choose_shift(3);
  const qdwh::PartialEigResult ref = qdwh::qdwh_partial_eig(gen.a, plan);
  const qdwh::PartialEigResult gpu = qdwhg::qdwh_partial_eig(gen.a, plan);
  if (ref.count() != gpu.count()) {
    std::printf("FAIL count %zu vs %zu\n", ref.count(), gpu.count());
    return 1;
  }
  double worst = 0.0;
  for (size_t i = 0; i < ref.count(); ++i)
    worst = std::fmax(worst, std::fabs(ref.lambda_minus[i] - gpu.lambda_minus[i]) /
                                 std::fabs(ref.lambda_minus[i]));
  const qdwh::SvdTestMatrix sg = qdwh::gen_svd_test(128, qdwh::Seed{2});
  const qdwh::PartialSvdResult rs = qdwh::qdwh_partial_svd(sg.a, 0.01);
  const qdwh::PartialSvdResult gs = qdwhg::qdwh_partial_svd(sg.a, 0.01);
  if (rs.count() != gs.count()) {
    std::printf("FAIL svd count %zu vs %zu\n", rs.count(), gs.count());
    return 1;
  }
  for (size_t i = 0; i < rs.count(); ++i)
    worst = std::fmax(worst, std::fabs(rs.sigma1[i] - gs.sigma1[i]) / rs.sigma1[i]);
  // full-spectrum driver and the Eq. 5-7 report (fullsolve.hpp, metrics.hpp)
  const qdwh::EigResult rf = qdwh::qdwh_eig_full(gen.a, 32);
  const qdwh::EigResult gf = qdwhg::qdwh_eig_full(gen.a, 32);
  for (size_t i = 0; i < rf.lambda.size(); ++i)
    worst = std::fmax(worst, std::fabs(rf.lambda[i] - gf.lambda[i]) / std::fmax(1.0, std::fabs(rf.lambda[i])));
  const qdwh::AccuracyReport ra = qdwh::accuracy_report(sg.a, rs.u1, rs.sigma1, rs.v1);
  const qdwh::AccuracyReport ga = qdwhg::accuracy_report(sg.a, rs.u1, rs.sigma1, rs.v1);
  const double scale = std::fmax(ra.resid_right, 1e-300);
  if (std::fabs(ra.resid_right - ga.resid_right) > 1e-6 * scale + 1e-15 || ra.k != ga.k) {
    std::printf("FAIL accuracy_report %.3e vs %.3e\n", ra.resid_right, ga.resid_right);
    return 1;
  }
  bool threw = false;
  try {
    qdwhg::qdwh_partial_svd(sg.a, 1.5);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  std::printf("%s max_rel_err=%.3e eig_k=%zu svd_k=%zu invalid_argument=%d\n",
              (worst < 1e-10 && threw) ? "OK" : "FAIL", worst, gpu.count(), gs.count(), (int)threw);
  return (worst < 1e-10 && threw) ? 0 : 1;
}
