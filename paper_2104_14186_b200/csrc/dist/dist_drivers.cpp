// Distributed QDWHpartial drivers (partial.cpp:40-158) and their Krylov bounds
// (kernels.cpp:332-439) on the 2D block-cyclic grid.  Control flow, constants,
// seeds and edge cases restate the reference like the single-GPU drivers
// (drivers.cpp); every matrix operation is a distributed building block
// (dist_core.cpp).  Decisions that steer control flow (mu, the deficiency index,
// counts) are computed identically on every rank and additionally broadcast
// from rank 0, so the ranks can never diverge.
#include <algorithm>
#include <cmath>

#include "dist.hpp"

namespace qdwhg {
namespace dist {

namespace {
constexpr double kEps = 2.220446049250313e-16;

// host scalars broadcast from world rank 0 (device round trip for NCCL)
void bcast_host(Ctx& c, std::vector<double>& v) {
  if (v.empty()) return;
  Engine& e = *c.eng;
  const EMark mk = e.mark();
  double* d = e.alloc_vec(v.size());
  e.from_host(v.data(), (int64_t)v.size(), (int64_t)v.size(), 1, d, (int64_t)v.size());
  c.comm->bcast(d, v.size(), 0, Team::World);
  ++c.collectives;
  e.to_host(d, (int64_t)v.size(), (int64_t)v.size(), 1, v.data(), (int64_t)v.size());
  e.release(mk);
}

std::vector<double> unit_start(int64_t n, uint64_t seed) {
  std::vector<double> v = host_gaussian(n, seed);
  double s = 0.0;
  for (double x : v) s += x * x;
  const double nv = std::sqrt(s);
  for (double& x : v) x /= nv;
  return v;
}
}  // namespace

double lanczos_min_bound(Ctx& c, const DistMat& A, int steps, double fro) {
  // kernels.cpp:362-439: two-pass full reorthogonalisation, breakdown tolerance
  // n u max(1, ||A||_F), mu = theta_min - beta_last |s_last|, x1.1 if negative
  Engine& e = *c.eng;
  const int64_t n = A.n;
  const int m = (int)std::min<int64_t>(steps, n);
  const EMark mk = e.mark();
  int64_t ldq;
  double* Qm = e.alloc(n, m + 1, &ldq);
  double* w = e.alloc_vec((size_t)n);
  double* h = e.alloc_vec((size_t)m + 1);
  const std::vector<double> q0 = unit_start(n, 0x6c616e637aull);  // kernels.cpp:379
  e.from_host(q0.data(), n, n, 1, Qm, ldq);
  const double breakdown_tol = (double)n * kEps * std::max(1.0, fro);
  std::vector<double> alpha, beta;
  double beta_last = 0.0;
  for (int j = 0; j < m; ++j) {
    double* qj = Qm + (int64_t)j * ldq;
    pgemv(c, A, false, qj, w);
    alpha.push_back(e.dot(qj, w, n));
    for (int pass = 0; pass < 2; ++pass) {  // w -= Q (Q^T w), Q = q_0..q_j
      e.gemm(true, false, j + 1, 1, n, 1.0, Qm, ldq, w, n, 0.0, h, j + 1);
      e.gemm(false, false, n, 1, j + 1, -1.0, Qm, ldq, h, j + 1, 1.0, w, n);
    }
    const double bj = std::sqrt(e.dot(w, w, n));
    beta_last = bj;
    if (j + 1 == m || bj <= breakdown_tol) {
      if (bj <= breakdown_tol) beta_last = 0.0;
      break;
    }
    beta.push_back(bj);
    e.axpby(w, n, Qm + (int64_t)(j + 1) * ldq, ldq, n, 1, 1.0 / bj, 0.0);
  }
  double theta = 0.0, s_last = 0.0;
  e.tridiag_lowest(alpha, beta, &theta, &s_last);
  double mu = theta - beta_last * std::abs(s_last);
  if (mu < 0.0) mu *= 1.1;
  e.release(mk);
  std::vector<double> hv{mu};
  bcast_host(c, hv);
  return hv[0];
}

double two_norm_estimate(Ctx& c, const DistMat& A) {
  // kernels.cpp:332-360: power iteration on A^T A from the seeded start
  Engine& e = *c.eng;
  const int64_t m = A.m, n = A.n;
  const EMark mk = e.mark();
  double* v = e.alloc_vec((size_t)n);
  double* y = e.alloc_vec((size_t)m);
  double* z = e.alloc_vec((size_t)n);
  const std::vector<double> v0 = unit_start(n, 0x6e6f726d32ull);  // kernels.cpp:336
  e.from_host(v0.data(), n, n, 1, v, n);
  double est = 0.0;
  for (int it = 0; it < 100; ++it) {
    pgemv(c, A, false, v, y);
    const double ny = std::sqrt(e.dot(y, y, m));
    if (ny == 0.0) {
      std::vector<double> ax(n, 0.0);
      ax[it % n] = 1.0;
      e.from_host(ax.data(), n, n, 1, v, n);
      continue;
    }
    pgemv(c, A, true, y, z);
    const double nz = std::sqrt(e.dot(z, z, n));
    const double prev = est;
    est = ny;
    if (nz == 0.0) break;
    e.axpby(z, n, v, n, n, 1, 1.0 / nz, 0.0);
    if (it > 0 && std::abs(est - prev) < 1e-3 * est) break;
  }
  e.release(mk);
  std::vector<double> hv{1.05 * est};
  bcast_host(c, hv);
  return hv[0];
}

namespace {
// X <- (b/c) X + (a - b/c) X Z^-1, Z = I + c X^T X (polar.cpp:82-128).
// Symmetric X (EIG path): Z^-1 = W^-1 W^-T (LAUUM) and the lower triangle of
// G = X Z^-1 (symmetric) in one GEMM, mirrored; otherwise Y = X W^-1 and
// X+ = (b/c) X + coef Y W^-T (the update fused as beta).
void chol_step(Ctx& c, DistMat& X, DistMat& Xn, const WeightStep& w, bool symmetric, const DistMat& Z,
               const DistMat& Winv, const DistMat& Mw) {
  const double bc = w.b / w.c, coef = w.a - bc;
  Structure lo;
  lo.c_lower = true;
  pgemm(c, true, false, w.c, whole(X), whole(X), 0.0, whole(Z), lo);
  axpby_identity(c, nullptr, 0.0, Z, 1.0, 1.0);
  chol_inv(c, Z, Winv);
  if (symmetric) {
    Structure lau;  // M = W^-1 W^-T: lower tiles, k >= max(i, j) = i
    lau.a_upper = true;
    lau.b_lower = true;
    lau.c_lower = true;
    pgemm(c, false, true, 1.0, whole(Winv), whole(Winv), 0.0, whole(Mw), lau);
    mirror_lower(c, Mw);
    axpby_identity(c, &X, bc, Xn, 0.0, 0.0);
    pgemm(c, false, false, coef, whole(X), whole(Mw), 1.0, whole(Xn), lo);
    mirror_lower(c, Xn);
    std::swap(X, Xn);
  } else {
    Structure bu;
    bu.b_upper = true;  // W^-1 upper
    pgemm(c, false, false, 1.0, whole(X), whole(Winv), 0.0, whole(Xn), bu);
    Structure bl;
    bl.b_lower = true;  // W^-T lower
    pgemm(c, false, true, coef, whole(Xn), whole(Winv), bc, whole(X), bl);
  }
}

size_t deficiency_index(Ctx& c, const std::vector<double>& rdiag, double tol) {
  // partial.cpp:32-38 on the replicated |R_ii|; rank 0's answer is authoritative
  std::vector<double> v{0.0};
  for (size_t i = 0; i < rdiag.size(); ++i)
    if (std::abs(rdiag[i]) < tol) {
      v[0] = (double)(i + 1);
      break;
    }
  bcast_host(c, v);
  return (size_t)v[0];
}

// root: ell x k block W replicated to all ranks, then V = Q2 W by rows
// (row-team reduction), gathered to the root as a dense n x k matrix.
double* form_vectors(Ctx& c, const DistMat& Q2, double* Wroot, int64_t ldw_root, int64_t k, int64_t* vld_out) {
  Engine& e = *c.eng;
  const Grid& g = c.g;
  const int64_t n = Q2.m, ell = Q2.n, nb = g.nb;
  const int me = g.world_rank(g.p, g.q);
  int64_t ldw;
  double* W = e.alloc(ell, k, &ldw);
  if (me == 0) e.copy_tiles({TileCopy{Wroot, ldw_root, W, ldw, (int32_t)ell, (int32_t)k, 0}});
  // (contiguous broadcast: ldw-padded columns)
  c.comm->bcast(W, (size_t)(ldw * k), 0, Team::World);
  ++c.collectives;
  // rows of W for my local Q2 columns
  int64_t ldwl;
  double* Wl = e.alloc(std::max<int64_t>(Q2.lc, 1), k, &ldwl);
  std::vector<TileCopy> tc;
  for (int64_t J = g.q; J < Q2.nt(); J += g.Q)
    tc.push_back(TileCopy{W + J * nb, ldw, Wl + Q2.lcol(J), ldwl, (int32_t)Q2.tile_cols(J), (int32_t)k, 0});
  if (!tc.empty()) e.copy_tiles(tc);
  int64_t ldv;
  double* Vl = e.alloc(std::max<int64_t>(Q2.lr, 1), k, &ldv);
  if (Q2.lr > 0) {
    if (Q2.lc > 0) e.gemm(false, false, Q2.lr, k, Q2.lc, 1.0, Q2.a, Q2.ld, Wl, ldwl, 0.0, Vl, ldv);
    else e.fill(Vl, ldv, Q2.lr, k, 0.0);
    c.comm->allreduce(Vl, (size_t)(ldv * k), RedOp::Sum, Team::Row);
    ++c.collectives;
  }
  // gather the rows to the root (process column 0 sends its packed rows)
  double* V = nullptr;
  if (me == 0) V = e.alloc(n, k, vld_out);
  double* sb = nullptr;
  if (g.q == 0 && me != 0 && Q2.lr > 0) {
    sb = e.alloc_vec((size_t)(Q2.lr * k));
    e.copy_tiles({TileCopy{Vl, ldv, sb, Q2.lr, (int32_t)Q2.lr, (int32_t)k, 0}});
  }
  std::vector<double*> rb(g.P, nullptr);
  std::vector<int64_t> rlen(g.P, 0);
  c.comm->group_begin();
  if (sb) c.comm->send(sb, (size_t)(Q2.lr * k), 0);
  if (me == 0)
    for (int pr = 1; pr < g.P; ++pr) {
      rlen[pr] = numroc(n, nb, pr, g.P);
      if (rlen[pr] == 0) continue;
      rb[pr] = e.alloc_vec((size_t)(rlen[pr] * k));
      c.comm->recv(rb[pr], (size_t)(rlen[pr] * k), g.world_rank(pr, 0));
    }
  c.comm->group_end();
  ++c.collectives;
  if (me == 0) {
    tc.clear();
    for (int64_t I = 0; I < Q2.mt(); ++I) {
      const int pr = (int)(I % g.P);
      const double* src = pr == 0 ? Vl + (I / g.P) * nb : rb[pr] + (I / g.P) * nb;
      tc.push_back(TileCopy{src, pr == 0 ? ldv : rlen[pr], V + I * nb, *vld_out, (int32_t)Q2.tile_rows(I),
                            (int32_t)k, 0});
    }
    e.copy_tiles(tc);
  }
  return V;
}

void stage(double* acc, int s, const std::function<double()>& clock, double& t) {
  if (!clock) return;
  const double now = clock();
  acc[s] += now - t;
  t = now;
}
}  // namespace

EigResult partial_eig(Ctx& c, const DistMat& A, double s, size_t iters, bool randomize, double tol,
                      uint64_t seed, const std::function<double()>& clock) {
  // partial.cpp:40-99
  Engine& e = *c.eng;
  const Grid& g = c.g;
  const int64_t n = A.m;
  if (A.n != n) throw InvalidArgument("qdwh_partial_eig: matrix not square");
  double t = clock ? clock() : 0.0;
  double st[3];
  stats(c, A, true, st);
  if (st[2] > 0) throw InvalidArgument("qdwh_partial_eig: non-finite entry");
  const double fro = std::sqrt(st[0]);
  if (st[1] > 1e3 * (double)n * kEps * std::max(1.0, fro))
    throw InvalidArgument("qdwh_partial_eig: input not symmetric within tolerance");
  EigResult out;
  out.mu = lanczos_min_bound(c, A, 30, fro);
  stage(out.stage_seconds, 0, clock, t);
  if (out.mu >= 0.0) return out;  // partial.cpp:52
  const double scale = std::abs(out.mu);
  // As = sym(A)/|mu| (transpose exchange), X = (1-s) As - s I   (partial.cpp:54-59)
  DistMat As = make_dist(e, g, n, n);
  transpose_into(c, A, As);
  axpby_identity(c, &A, 0.5 / scale, As, 0.5 / scale, 0.0);
  DistMat X = make_dist(e, g, n, n), Xn = make_dist(e, g, n, n);
  axpby_identity(c, &As, 1.0 - s, X, 0.0, -s);
  {
    const EMark mk = e.mark();
    DistMat Z = make_dist(e, g, n, n), Wi = make_dist(e, g, n, n), Mw = make_dist(e, g, n, n);
    double ell = s;
    out.trace.push_back(ell);
    for (size_t k = 0; k < iters; ++k) {  // polar.cpp:179-215, Cholesky-only, symmetric
      const WeightStep w = halley_weights(ell);
      chol_step(c, X, Xn, w, true, Z, Wi, Mw);
      ++out.iters_chol;
      ell = w.ell_out;
      out.trace.push_back(ell);
    }
    e.release(mk);
  }
  stage(out.stage_seconds, 1, clock, t);
  // B = (X + I)/2 (partial.cpp:67-69), optionally B Omega (partial.cpp:70)
  axpby_identity(c, nullptr, 0.0, X, 0.5, 0.5);
  const DistMat* B = &X;
  DistMat BO;
  if (randomize) {
    DistMat Om = make_dist(e, g, n, n);
    for (int64_t I = 0; I < Om.mt(); ++I)
      for (int64_t J = 0; J < Om.nt(); ++J)
        if (Om.owns_row(I) && Om.owns_col(J))
          e.gaussian(Om.tile(I, J), Om.ld, Om.tile_rows(I), Om.tile_cols(J), seed, I * g.nb, J * g.nb, n);
    BO = make_dist(e, g, n, n);
    pgemm(c, false, false, 1.0, whole(X), whole(Om), 0.0, whole(BO));
    B = &BO;
  }
  QrDist qr;
  pgeqrf(c, *B, qr);
  const double nd = (double)n;
  out.flops = (double)out.iters_chol * (10.0 / 3.0) * nd * nd * nd + 4.0 / 3.0 * nd * nd * nd +
              (randomize ? 2 * nd * nd * nd : 0.0);
  const size_t ind = deficiency_index(c, qr.rdiag, tol);
  stage(out.stage_seconds, 2, clock, t);
  if (ind == 0) return out;  // partial.cpp:72-73
  out.rank_index = ind;
  const int64_t ell = n - (int64_t)ind + 1;
  out.subspace_size = ell;
  out.no_savings = ell > n / 2;
  DistMat Q2 = make_dist(e, g, n, ell);
  porgqr_cols(c, qr, (int64_t)ind - 1, Q2);
  stage(out.stage_seconds, 3, clock, t);
  // Rayleigh-Ritz (partial.cpp:80-81): AQ = As Q2, S = Q2^T AQ gathered to rank 0
  DistMat AQ = make_dist(e, g, n, ell);
  pgemm(c, false, false, 1.0, whole(As), whole(Q2), 0.0, whole(AQ));
  DistMat S = make_dist(e, g, ell, ell);
  pgemm(c, true, false, 1.0, whole(Q2), whole(AQ), 0.0, whole(S));
  const int me = g.world_rank(g.p, g.q);
  int64_t lds = 0, ldw = 0;
  double* Sd = me == 0 ? e.alloc(ell, ell, &lds) : nullptr;
  gather(c, S, Sd, lds, 0);
  stage(out.stage_seconds, 4, clock, t);
  std::vector<double> vals;
  double* Wd = nullptr;
  int64_t sel0 = 0;
  std::vector<double> hk{0.0};
  if (me == 0) {
    e.mirror_lower(Sd, lds, ell);  // exactly symmetric (lower triangle kept)
    Wd = e.alloc(ell, ell, &ldw);
    e.syev_range(Sd, lds, ell, vals, Wd, ldw, -INFINITY, 0.0, &sel0);
    int64_t k = 0;
    while (k < ell && vals[k] < 0.0) ++k;
    hk[0] = (double)k;
  }
  bcast_host(c, hk);
  const int64_t k = (int64_t)hk[0];
  if (me != 0) vals.assign((size_t)ell, 0.0);
  bcast_host(c, vals);
  stage(out.stage_seconds, 5, clock, t);
  const double l = (double)ell;
  out.flops += 2 * nd * nd * l - 2 * l * l * l / 3 + 2 * nd * nd * l + 2 * nd * l * l + 9 * l * l * l;
  if (k == 0) return out;  // partial.cpp:89-90
  double max_abs_ritz = 0.0;
  for (double v : vals) max_abs_ritz = std::max(max_abs_ritz, std::abs(v));
  const double floor = -nd * kEps * max_abs_ritz;
  out.lambda.resize((size_t)k);
  for (int64_t i = 0; i < k; ++i) {
    out.lambda[(size_t)i] = scale * vals[(size_t)i];
    if (vals[(size_t)i] >= floor) ++out.borderline;
  }
  out.V = form_vectors(c, Q2, Wd, ldw, k, &out.vld);
  out.flops += 2 * nd * l * (double)k;
  stage(out.stage_seconds, 6, clock, t);
  return out;
}

SvdResult partial_svd(Ctx& c, const DistMat& A, double s, double s_abs, double tol, bool randomize,
                      uint64_t seed, const std::function<double()>& clock) {
  // partial.cpp:101-158
  Engine& e = *c.eng;
  const Grid& g = c.g;
  const int64_t m = A.m, n = A.n;
  double t = clock ? clock() : 0.0;
  double st[3];
  stats(c, A, false, st);
  if (st[2] > 0) throw InvalidArgument("qdwh_partial_svd: non-finite entry");
  if (st[0] == 0.0) throw InvalidArgument("two_norm_estimate: zero matrix");
  if (m < n) throw InvalidArgument("qdwh_partial_svd: requires rows >= cols");
  SvdResult out;
  out.alpha = two_norm_estimate(c, A);
  if (s_abs > 0.0) s = s_abs / out.alpha;
  if (!(s > 0.0) || s >= 1.0) throw InvalidArgument("qdwh_partial_svd: threshold s must be in (0, 1)");
  out.threshold = s;
  stage(out.stage_seconds, 0, clock, t);
  DistMat X = make_dist(e, g, m, n);
  axpby_identity(c, &A, 1.0 / out.alpha, X, 0.0, 0.0);
  const size_t iters = iterations_to_converge(s, 5.0 * kEps);
  if (iters > 0 && s < 1e-3)
    throw InvalidArgument(
        "distributed qdwh_partial_svd: the QR-based first step (s < 1e-3) runs on one GPU only");
  out.trace.push_back(s);
  {
    const EMark mk = e.mark();
    DistMat Xn = make_dist(e, g, m, n);
    DistMat Z = make_dist(e, g, n, n), Wi = make_dist(e, g, n, n);
    double ell = s;
    for (size_t k = 0; k < iters; ++k) {
      const WeightStep w = halley_weights(ell);
      chol_step(c, X, Xn, w, false, Z, Wi, Z);
      ++out.iters_chol;
      ell = w.ell_out;
      out.trace.push_back(ell);
    }
    e.release(mk);
  }
  stage(out.stage_seconds, 1, clock, t);
  // M = I - sym(X^T X) (partial.cpp:134-136): lower tiles, mirrored
  DistMat Mm = make_dist(e, g, n, n);
  Structure lo;
  lo.c_lower = true;
  pgemm(c, true, false, -1.0, whole(X), whole(X), 0.0, whole(Mm), lo);
  axpby_identity(c, nullptr, 0.0, Mm, 1.0, 1.0);
  mirror_lower(c, Mm);
  const DistMat* B = &Mm;
  DistMat BO;
  if (randomize) {
    DistMat Om = make_dist(e, g, n, n);
    for (int64_t I = 0; I < Om.mt(); ++I)
      for (int64_t J = 0; J < Om.nt(); ++J)
        if (Om.owns_row(I) && Om.owns_col(J))
          e.gaussian(Om.tile(I, J), Om.ld, Om.tile_rows(I), Om.tile_cols(J), seed, I * g.nb, J * g.nb, n);
    BO = make_dist(e, g, n, n);
    pgemm(c, false, false, 1.0, whole(Mm), whole(Om), 0.0, whole(BO));
    B = &BO;
  }
  QrDist qr;
  pgeqrf(c, *B, qr);
  const size_t ind = deficiency_index(c, qr.rdiag, tol);
  stage(out.stage_seconds, 2, clock, t);
  const double md = (double)m, nd = (double)n;
  out.flops = (double)out.iters_chol * (3 * md * nd * nd + nd * nd * nd / 3) + md * nd * nd +
              4.0 / 3.0 * nd * nd * nd + (randomize ? 2 * nd * nd * nd : 0.0);
  if (ind == 0) return out;
  out.rank_index = ind;
  const int64_t ell = n - (int64_t)ind + 1;
  out.subspace_size = ell;
  out.no_savings = ell > n / 2;
  DistMat Q2 = make_dist(e, g, n, ell);
  porgqr_cols(c, qr, (int64_t)ind - 1, Q2);
  stage(out.stage_seconds, 3, clock, t);
  // Y = A Q2 (unscaled A, partial.cpp:147), gathered to rank 0 for the R-SVD
  DistMat Y = make_dist(e, g, m, ell);
  pgemm(c, false, false, 1.0, whole(A), whole(Q2), 0.0, whole(Y));
  const int me = g.world_rank(g.p, g.q);
  int64_t ldy = 0;
  double* Yd = me == 0 ? e.alloc(m, ell, &ldy) : nullptr;
  gather(c, Y, Yd, ldy, 0);
  stage(out.stage_seconds, 4, clock, t);
  const double cutoff = s * out.alpha;
  std::vector<double> sig;
  std::vector<double> hk{0.0};
  int64_t ldvs = 0;
  double* Vs = nullptr;
  if (me == 0) {
    out.U = e.alloc(m, ell, &out.uld);
    Vs = e.alloc(ell, ell, &ldvs);
    e.svd_polar(Yd, ldy, m, ell, out.U, out.uld, sig, Vs, ldvs, cutoff);
    int64_t k = 0;
    while (k < (int64_t)sig.size() && sig[(size_t)k] > cutoff) ++k;
    hk[0] = (double)k;
  }
  bcast_host(c, hk);
  const int64_t k = (int64_t)hk[0];
  sig.resize((size_t)k);
  bcast_host(c, sig);
  stage(out.stage_seconds, 5, clock, t);
  const double l = (double)ell;
  out.flops += 2 * nd * nd * l - 2 * l * l * l / 3 + 2 * md * nd * l + 6 * md * l * l + 20 * l * l * l;
  if (k == 0) return out;
  out.sigma = sig;
  out.V = form_vectors(c, Q2, Vs, ldvs, k, &out.vld);
  out.flops += 2 * nd * l * (double)k;
  stage(out.stage_seconds, 6, clock, t);
  return out;
}

}  // namespace dist
}  // namespace qdwhg
