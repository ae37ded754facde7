// QDWH iteration, polar decomposition and the QDWHpartial drivers on device
// views.  Control flow, constants, seeds and edge cases restate the reference
// (file:line cited per function); all matrix work runs in our sm_100a kernels.
#include "drivers.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <sstream>
#include <cstdlib>

namespace qdwhg {

constexpr double kEps = 2.220446049250313e-16;
extern const int kJacobiMaxN;
void syev_jacobi(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout);
void permute_cols(Ctx& ctx, const DMat& V, const std::vector<int>& order, const DMat& Vout);

// ----------------------------------------------------------------- stage clock
StageClock::StageClock(Ctx& c) : ctx(c) {
  cudaEvent_t e;
  QDWHG_CUDA(cudaEventCreate(&e));
  QDWHG_CUDA(cudaEventRecord(e, ctx.stream));
  ev.push_back(e);
  owner.push_back(-1);
}
StageClock::~StageClock() {
  for (auto e : ev) cudaEventDestroy(e);
}
void StageClock::mark(int stage) {
  cudaEvent_t e;
  QDWHG_CUDA(cudaEventCreate(&e));
  QDWHG_CUDA(cudaEventRecord(e, ctx.stream));
  ev.push_back(e);
  owner.push_back(stage);
}
void StageClock::finish(double* stage_seconds, double* total) {
  QDWHG_CUDA(cudaEventSynchronize(ev.back()));
  for (size_t i = 1; i < ev.size(); ++i) {
    float ms = 0.f;
    QDWHG_CUDA(cudaEventElapsedTime(&ms, ev[i - 1], ev[i]));
    if (stage_seconds && owner[i] >= 0 && owner[i] < 8) stage_seconds[owner[i]] += ms * 1e-3;
  }
  if (total) {
    float ms = 0.f;
    QDWHG_CUDA(cudaEventElapsedTime(&ms, ev.front(), ev.back()));
    *total = ms * 1e-3;
  }
}

// ----------------------------------------------------------------- QDWH steps
void qdwh_chol_step(Ctx& ctx, const DMat& X, const WeightStep& w, const DMat& Xout,
                    bool symmetric) {
  // polar.cpp:82-128:  Z = I + c sym(X^T X);  W = chol(Z);  X+ = (b/c) X + (a - b/c) X W^-1 W^-T
  // symmetric: X is symmetric, so is G = X Z^-1 (a function of X): only its lower
  // triangle is computed and mirrored (1/3 fewer TRMM flops, X+ exactly symmetric)
  const int64_t m = X.rows, n = X.cols;
  const Arena::Mark mark = ctx.arena->mark();
  DMat Z = ctx.arena->alloc(n, n);
  DMat Winv = ctx.arena->alloc(n, n);
  DMat Y = ctx.arena->alloc(m, n);
  const double bc = w.b / w.c;
  const double coef = w.a - bc;
  static const bool no_lauum = getenv("QDWHG_CHOL_NO_LAUUM") != nullptr;
  const bool sym = symmetric && m == n && !no_lauum;
  static const bool no_overlap = getenv("QDWHG_CHOL_NO_OVERLAP") != nullptr;
  static const bool stable_env = getenv("QDWHG_CHOL_STABLE") != nullptr;
  const int64_t n1 = ((n / 2 + 127) / 128) * 128;
  // (only for mid-size n — measured per step: -0.3 ms at 3072, -0.1 ms at 4096,
  // neutral at 4546, +3.5 ms at 6144, where the capped side launches run well
  // below the GEMM rate and the chain is a small share)
  if (!no_overlap && !stable_env && ctx.side != nullptr && n >= 2048 && n <= 5120 && n1 < n &&
      !chol_dag_applicable(n)) {
    // Overlapped schedule: the latency-bound recursive Cholesky-and-inverse
    // chain runs on the main stream while independent GEMM work runs on the
    // side stream in launches of <= 64 128x128 tiles (so the chain's small
    // kernels always find free SMs):
    //   side: Z22 = I + c X2^T X2   (main: Z11, Z21, left half of the recursion)
    //   side: Y1  = X1 W11^-1        (main: W12, Z22 update, right half, W^-1_12, Y2)
    // Outputs are disjoint; events order the hand-offs; side GEMMs take no
    // arena scratch (split_k = 1).
    const int64_t n2 = n - n1;
    const DMat X1 = X.sub(0, 0, m, n1), X2 = X.sub(0, n1, m, n2);
    cudaStream_t main_stream = ctx.stream;
    auto on_side = [&](cudaEvent_t done, auto&& body) {
      QDWHG_CUDA(cudaEventRecord(ctx.ev_main, main_stream));
      ctx.stream = ctx.side;
      QDWHG_CUDA(cudaStreamWaitEvent(ctx.side, ctx.ev_main, 0));
      body();
      QDWHG_CUDA(cudaEventRecord(done, ctx.side));
      ctx.stream = main_stream;
    };
    GemmExtra sx;
    sx.split_k = 1;
    sx.force_bm = 128;
    // W^-1's strictly lower part is never written by the chain's leaves
    // (kDiagUpperOnly) but is read as zeros by the main-stream GEMMs of the left
    // half of the recursion (W11^-T, W^-1 operands): zeroed on the main stream,
    // before anything reads it (the arena hands back stale data otherwise)
    zero_strict_lower(ctx, Winv);
    on_side(ctx.ev_side, [&] {
      // Z22 lower in <= 64-tile pieces: two lower diagonal quarters + one full block
      const int64_t h1 = ((n2 / 2 + 127) / 128) * 128, h2 = n2 - h1;
      GemmExtra lo = sx;
      lo.out = OutMode::Lower;
      lo.diag_add = 1.0;
      const DMat Xa = X2.col_block(0, h1), Xb = X2.col_block(h1, h2);
      gemm(ctx, Op::T, Op::N, w.c, Xa, Xa, 0.0, Z.sub(n1, n1, h1, h1), lo);
      const int64_t rows_per = std::max<int64_t>(128, (64 / ((h1 + 127) / 128)) * 128);
      for (int64_t r0 = 0; r0 < h2; r0 += rows_per) {
        const int64_t rr = std::min(rows_per, h2 - r0);
        gemm(ctx, Op::T, Op::N, w.c, Xb.col_block(r0, rr), Xa, 0.0, Z.sub(n1 + h1 + r0, n1, rr, h1), sx);
      }
      gemm(ctx, Op::T, Op::N, w.c, Xb, Xb, 0.0, Z.sub(n1 + h1, n1 + h1, h2, h2), lo);
    });
    bool y1_pending = false;
    try {
      GemmExtra s11;
      s11.out = OutMode::Lower;
      s11.diag_add = 1.0;
      gemm(ctx, Op::T, Op::N, w.c, X1, X1, 0.0, Z.sub(0, 0, n1, n1), s11);
      gemm(ctx, Op::T, Op::N, w.c, X2, X1, 0.0, Z.sub(n1, 0, n2, n1));
      potrf_fast_split(
          ctx, Z, Winv, n1,
          [&] { QDWHG_CUDA(cudaStreamWaitEvent(main_stream, ctx.ev_side, 0)); },
          [&] {
            if (sym) return;  // symmetric: Z^-1 by LAUUM below, no Y = X W^-1
            on_side(ctx.ev_side2, [&] {
              // Y1 = X1 W11^-1 by row pieces of <= 64 tiles
              GemmExtra t1 = sx;
              t1.krange = KRange::BUpper;
              const int64_t rows_per = std::max<int64_t>(128, (64 / ((n1 + 127) / 128)) * 128);
              for (int64_t r0 = 0; r0 < m; r0 += rows_per) {
                const int64_t rr = std::min(rows_per, m - r0);
                gemm(ctx, Op::N, Op::N, 1.0, X1.sub(r0, 0, rr, n1), Winv.sub(0, 0, n1, n1), 0.0,
                     Y.sub(r0, 0, rr, n1), t1);
              }
            });
            y1_pending = true;
          },
          /*winv_lower_zeroed=*/true);
    } catch (...) {
      ctx.stream = main_stream;
      QDWHG_CUDA(cudaStreamSynchronize(ctx.side));
      ctx.arena->release_to(mark);
      throw;
    }
    if (!sym) {
      // Y2 = X1 W^-1_12 + X2 W^-1_22
      gemm(ctx, Op::N, Op::N, 1.0, X1, Winv.sub(0, n1, n1, n2), 0.0, Y.sub(0, n1, m, n2));
      GemmExtra t1b;
      t1b.krange = KRange::BUpper;
      gemm(ctx, Op::N, Op::N, 1.0, X2, Winv.sub(n1, n1, n2, n2), 1.0, Y.sub(0, n1, m, n2), t1b);
    }
    if (y1_pending) QDWHG_CUDA(cudaStreamWaitEvent(main_stream, ctx.ev_side2, 0));
  } else {
    GemmExtra syrk;
    syrk.out = OutMode::Lower;  // POTRF reads the lower triangle only
    syrk.diag_add = 1.0;
    syrk.fine_tail = true;
    gemm(ctx, Op::T, Op::N, w.c, X, X, 0.0, Z, syrk);
    try {
      // kappa(Z) <= 1 + c: the fast recursive Cholesky-and-inverse is accurate here
      potrf_upper_and_inverse(ctx, Z, Winv, false, stable_env);
    } catch (...) {
      ctx.arena->release_to(mark);
      throw;
    }
    if (!sym) {
      GemmExtra t1;
      t1.krange = KRange::BUpper;  // W^-1 upper
      gemm(ctx, Op::N, Op::N, 1.0, X, Winv, 0.0, Y, t1);
    }
  }
  // W^-T materialised (one transpose pass) so the next product runs in the
  // faster K-major-B layout instead of reading W^-1 transposed tile by tile
  DMat WinvT = Z;  // Z is dead after the factorisation
  transpose(ctx, Winv, WinvT);
  if (sym) {
    // Symmetric X: G = X Z^-1 is symmetric.  Z^-1 = W^-1 W^-T (LAUUM: lower
    // tiles, K from the tile row, mirrored; n^3/3) then G's lower triangle by one
    // GEMM (n^3) — 4/3 n^3 instead of the two TRMMs' 5/3 n^3.  X is an operand,
    // so the result goes through Y (copied back when Xout aliases X).
    DMat Zi = ctx.arena->alloc(n, n);
    GemmExtra lu;
    lu.krange = KRange::AUpper;  // W^-1(i, k) != 0 for k >= i
    lu.out = OutMode::LowerMirror;
    gemm(ctx, Op::N, Op::N, 1.0, Winv, WinvT, 0.0, Zi, lu);
    GemmExtra g;
    g.cin = &X;  // fused weight update (b/c) X + (a - b/c) G
    g.out = OutMode::LowerMirror;
    g.fine_tail = true;
    const bool alias = Xout.base == X.base && Xout.r0 == X.r0 && Xout.c0 == X.c0;
    const DMat dst = alias ? Y : Xout;
    gemm(ctx, Op::N, Op::N, coef, X, Zi, bc, dst, g);
    if (alias) copy(ctx, Y, Xout);
  } else {
    GemmExtra t2;
    t2.krange = KRange::BLower;  // W^-T lower
    t2.cin = &X;                 // fused weight update (b/c) X + (a - b/c) G
    gemm(ctx, Op::N, Op::N, coef, Y, WinvT, bc, Xout, t2);
  }
  ctx.arena->release_to(mark);
}

void qdwh_qr_step(Ctx& ctx, const DMat& X, const WeightStep& w, const DMat& Xout) {
  // polar.cpp:53-80: QR of [sqrt(c) X; I], X+ = (b/c) X + ((a - b/c)/sqrt(c)) Q1 Q2^T
  const int64_t m = X.rows, n = X.cols;
  const double sc = std::sqrt(w.c);
  const Arena::Mark mark = ctx.arena->mark();
  DMat S = ctx.arena->alloc(m + n, n);
  axpby_identity(ctx, X, sc, 0.0, S.sub(0, 0, m, n));
  fill(ctx, S.sub(m, 0, n, n), 0.0, 1.0);
  QrWork qw;
  geqrf(ctx, S, qw, /*top_rows=*/m);  // the identity block: row-limited panels and updates
  DMat Q = ctx.arena->alloc(m + n, n);
  orgqr_cols(ctx, qw, m + n, n, 0, Q);
  const double bc = w.b / w.c;
  const double coef = (w.a - bc) / sc;
  GemmExtra e;
  e.cin = &X;
  gemm(ctx, Op::N, Op::T, coef, Q.sub(0, 0, m, n), Q.sub(m, 0, n, n), bc, Xout, e);
  ctx.arena->release_to(mark);
}

static bool is_symmetric(Ctx& ctx, const DMat& X) {
  if (X.rows != X.cols) return false;
  const MatStats st = mat_stats(ctx, X, true);
  return st.asym <= 1e3 * (double)X.rows * kEps * std::max(1.0, std::sqrt(st.fro2));
}

FixedIterResult run_fixed_iterations(Ctx& ctx, const DMat& X, double ell0, size_t iters,
                                     bool qr_first, bool known_symmetric) {
  // polar.cpp:179-215
  if (!(ell0 > 0.0) || ell0 > 1.0)
    throw InvalidArgument("run_fixed_iterations: ell0 must be in (0, 1]");
  if (iters < 1) throw InvalidArgument("run_fixed_iterations: iters must be >= 1");
  // (polar.cpp:186-195; the EIG driver's iterate is exactly symmetric by construction)
  const bool symmetric = known_symmetric || is_symmetric(ctx, X);
  FixedIterResult r;
  r.ell = ell0;
  r.trace.push_back(ell0);
  // Fixed trip count, no fallback (polar.cpp:206-207): one pivot check after the
  // last step instead of a host round trip per step; symmetric Cholesky steps
  // ping-pong between X and a second buffer (their mirrored epilogue cannot write
  // in place)
  const Arena::Mark mark = ctx.arena->mark();
  DMat cur = X;
  DMat spare;
  const bool pingpong = symmetric && X.rows == X.cols && !qr_first;
  if (pingpong) spare = ctx.arena->alloc(X.rows, X.cols);
  QDWHG_CUDA(cudaMemsetAsync(ctx.dflag, 0, sizeof(int), ctx.stream));
  ctx.defer_pivot_check = true;
  try {
    for (size_t k = 0; k < iters; ++k) {
      const WeightStep w = halley_weights(r.ell);
      if (qr_first && k == 0) {
        qdwh_qr_step(ctx, cur, w, cur);
        ++r.iters_qr;
        if (symmetric) symmetrize_scale(ctx, cur, 1.0, 0.0, cur);
      } else if (pingpong) {
        const DMat nxt = (cur.base == X.base) ? spare : X;
        qdwh_chol_step(ctx, cur, w, nxt, true);  // symmetric output by construction
        cur = nxt;
        ++r.iters_chol;
      } else {
        qdwh_chol_step(ctx, cur, w, cur, symmetric);
        ++r.iters_chol;
      }
      r.ell = w.ell_out;
      r.trace.push_back(r.ell);
    }
  } catch (...) {
    ctx.defer_pivot_check = false;
    ctx.arena->release_to(mark);
    throw;
  }
  ctx.defer_pivot_check = false;
  if (cur.base != X.base) copy(ctx, cur, X);
  ctx.arena->release_to(mark);
  int hflag = 0;
  QDWHG_CUDA(cudaMemcpyAsync(&hflag, ctx.dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  if (hflag) throw NotPositiveDefinite("cholesky: pivot is not positive");
  return r;
}

PolarOut polar_decompose(Ctx& ctx, const DMat& A, const PolarCfg& cfg, const DMat& Up,
                         const DMat& H) {
  // polar.cpp:130-177
  const int64_t m = A.rows, n = A.cols;
  if (m < n) throw InvalidArgument("polar_decompose: requires rows >= cols");
  if (!(cfg.ell0 > 0.0) || cfg.ell0 > 1.0)
    throw InvalidArgument("polar_decompose: ell0 must be in (0, 1]");
  PolarOut out;
  out.alpha = two_norm_estimate(ctx, A);
  axpby_identity(ctx, A, 1.0 / out.alpha, 0.0, Up);
  double ell = cfg.ell0 / 1.10;
  out.trace.push_back(ell);
  const double stop = 5.0 * cfg.conv_eps;
  const double md = (double)m, nd = (double)n;
  while (std::abs(ell - 1.0) >= stop) {
    if (out.iters_qr + out.iters_chol >= cfg.max_iters) {
      std::ostringstream msg;
      msg << "polar_decompose: no convergence after " << cfg.max_iters << " iterations (ell = " << ell
          << ")";
      throw NotConverged(msg.str());
    }
    const WeightStep w = halley_weights(ell);
    bool use_chol = w.c <= cfg.chol_switch_c;
    if (cfg.force_variant == 1) use_chol = false;
    if (cfg.force_variant == 2) use_chol = true;
    if (use_chol) {
      try {
        qdwh_chol_step(ctx, Up, w, Up);
        ++out.iters_chol;
        out.flops += 3 * md * nd * nd + nd * nd * nd / 3;
      } catch (const NotPositiveDefinite&) {
        if (cfg.force_variant == 2) throw;
        qdwh_qr_step(ctx, Up, w, Up);
        ++out.iters_qr;
        out.flops += 6 * md * nd * nd + 8.0 / 3.0 * nd * nd * nd;
      }
    } else {
      qdwh_qr_step(ctx, Up, w, Up);
      ++out.iters_qr;
      out.flops += 6 * md * nd * nd + 8.0 / 3.0 * nd * nd * nd;
    }
    ell = w.ell_out;
    out.trace.push_back(ell);
  }
  if (H.base) {
    // H = sym(Up^T A)  (polar.cpp:175)
    gemm(ctx, Op::T, Op::N, 1.0, Up, A, 0.0, H);
    symmetrize_scale(ctx, H, 1.0, 0.0, H);
    out.flops += 2 * md * nd * nd;
  }
  return out;
}

// ----------------------------------------------------------------- dense EIG / SVD
static double device_trace(Ctx& ctx, const DMat& A) {
  std::vector<double> d;
  diag_to_host(ctx, A, d);
  double t = 0.0;
  for (double x : d) t += x;
  return t;
}

// Spectral divide-and-conquer (fullsolve.cpp:22-72 strategy) for blocks larger
// than the single-CTA Jacobi: polar of A - sigma I gives the spectral projector
// C = (I - Up)/2 onto eigenvalues below sigma; a randomized QR of C splits the
// space; recurse on the two Rayleigh quotients.
static void syev_dc(Ctx& ctx, const DMat& A, std::vector<double>& vals, const DMat& Vout,
                    int depth) {
  const int64_t n = A.rows;
  if (n <= kJacobiMaxN) {
    syev_jacobi(ctx, A, vals, Vout);
    return;
  }
  const Arena::Mark mark = ctx.arena->mark();
  const double sigma0 = device_trace(ctx, A) / (double)n;
  DMat Sh = ctx.arena->alloc(n, n);
  const MatStats st = mat_stats(ctx, A, false);
  const double fro = std::sqrt(st.fro2);
  // candidate split points: the mean, then points between mean and the Gershgorin-free
  // Frobenius bound if the mean splits nothing off
  const double spread = fro / std::sqrt((double)n);
  const double cand[5] = {sigma0, sigma0 + 0.5 * spread, sigma0 - 0.5 * spread,
                          sigma0 + 0.25 * spread, sigma0 - 0.25 * spread};
  DMat Up = ctx.arena->alloc(n, n);
  int64_t k = 0;
  double sigma = sigma0;
  for (int attempt = 0; attempt < 5; ++attempt) {
    sigma = cand[attempt];
    axpby_identity(ctx, A, 1.0, -sigma, Sh);
    const MatStats ss = mat_stats(ctx, Sh, false);
    if (std::sqrt(ss.fro2) <= 10.0 * (double)n * kEps * std::max(1.0, std::abs(sigma))) {
      // constant-diagonal block (fullsolve.cpp:31-38)
      vals.assign(n, sigma);
      fill(ctx, Vout, 0.0, 1.0);
      ctx.arena->release_to(mark);
      return;
    }
    PolarCfg cfg;
    cfg.ell0 = 1e-15;
    DMat none;
    polar_decompose(ctx, Sh, cfg, Up, none);
    // C = sym((I - Up)/2), k = round(trace C); an eigenvalue a few l0 from the
    // shift leaves trace(C) visibly off an integer (see eig_full_rec): next candidate
    symmetrize_scale(ctx, Up, -0.5, 0.5, Up);
    const double tr = device_trace(ctx, Up);
    k = std::llround(tr);
    if (k > 0 && k < n && std::abs(tr - (double)k) < std::max(2e-13, 16.0 * (double)n * kEps)) break;
    k = 0;
  }
  if (k <= 0 || k >= n) throw NotConverged("syev: spectral divide-and-conquer found no split");
  DMat Om = ctx.arena->alloc(n, n);
  gaussian_fill(ctx, Om, 0x73706c6974ull + (uint64_t)depth);  // kSplitSeed, fullsolve.cpp:14
  DMat CO = ctx.arena->alloc(n, n);
  gemm(ctx, Op::N, Op::N, 1.0, Up, Om, 0.0, CO);
  QrWork qw;
  geqrf(ctx, CO, qw);
  DMat Q = ctx.arena->alloc(n, n);
  orgqr_cols(ctx, qw, n, n, 0, Q);
  const DMat Vlo = Q.sub(0, 0, n, k), Vhi = Q.sub(0, k, n, n - k);
  DMat T = ctx.arena->alloc(n, n);
  std::vector<double> vlo, vhi;
  DMat Alo = ctx.arena->alloc(k, k), Ahi = ctx.arena->alloc(n - k, n - k);
  {
    gemm(ctx, Op::N, Op::N, 1.0, A, Vlo, 0.0, T.sub(0, 0, n, k));
    gemm(ctx, Op::T, Op::N, 1.0, Vlo, T.sub(0, 0, n, k), 0.0, Alo);
    symmetrize_scale(ctx, Alo, 1.0, 0.0, Alo);
    gemm(ctx, Op::N, Op::N, 1.0, A, Vhi, 0.0, T.sub(0, 0, n, n - k));
    gemm(ctx, Op::T, Op::N, 1.0, Vhi, T.sub(0, 0, n, n - k), 0.0, Ahi);
    symmetrize_scale(ctx, Ahi, 1.0, 0.0, Ahi);
  }
  DMat Wlo = ctx.arena->alloc(k, k), Whi = ctx.arena->alloc(n - k, n - k);
  syev_dc(ctx, Alo, vlo, Wlo, depth + 1);
  syev_dc(ctx, Ahi, vhi, Whi, depth + 1);
  gemm(ctx, Op::N, Op::N, 1.0, Vlo, Wlo, 0.0, Vout.sub(0, 0, n, k));
  gemm(ctx, Op::N, Op::N, 1.0, Vhi, Whi, 0.0, Vout.sub(0, k, n, n - k));
  vals = vlo;
  vals.insert(vals.end(), vhi.begin(), vhi.end());
  ctx.arena->release_to(mark);
}

bool syev_tridiag(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout, double vlo,
                  double vhi, int64_t* sel0);

// ----------------------------------------------------------------- full-spectrum drivers
// qdwh_eig_full (fullsolve.cpp:22-80): shift by the trace mean, split with the
// spectral projector C = (I - Up)/2 of the QDWH polar factor, a QR of C Omega
// (the reference's fixed split seed at every depth) for the two invariant
// subspaces, Rayleigh-Ritz on each, recursion down to base_size and a dense
// finish (the device eigensolver) on the leaves; no split (k = 0 or n) also
// finishes densely.  Every O(n^3) step is a DMMA GEMM / QDWH iteration.
static int64_t eig_full_rec(Ctx& ctx, const DMat& A, int64_t base, std::vector<double>& vals,
                            const DMat& Vout) {
  const int64_t n = A.rows;
  if (n <= base) {
    syev(ctx, A, vals, Vout);
    return 0;
  }
  const Arena::Mark mark = ctx.arena->mark();
  const double sigma0 = device_trace(ctx, A) / (double)n;
  DMat Sh = ctx.arena->alloc(n, n);
  DMat Up = ctx.arena->alloc(n, n);
  // the reference's shift is the trace mean; when it lands on an eigenvalue
  // (trace(C) not an integer: that direction is split between the two subspaces,
  // which are then not invariant) the next candidate is tried — points between
  // the mean and the Frobenius spread, as in syev_dc
  const double spread = std::sqrt(mat_stats(ctx, A, false).fro2 / (double)n);
  const double cand[5] = {sigma0, sigma0 + 0.01 * spread, sigma0 - 0.01 * spread, sigma0 + 0.1 * spread,
                          sigma0 - 0.1 * spread};
  int64_t k = 0;
  for (int attempt = 0; attempt < 5; ++attempt) {
    const double sigma = cand[attempt];
    axpby_identity(ctx, A, 1.0, -sigma, Sh);
    if (attempt == 0 && std::sqrt(mat_stats(ctx, Sh, false).fro2) <=
                            10.0 * (double)n * kEps * std::max(1.0, std::abs(sigma))) {
      // constant-diagonal block: the shift exhausted the spectrum (fullsolve.cpp:31-38)
      vals.assign(n, sigma);
      fill(ctx, Vout, 0.0, 1.0);
      ctx.arena->release_to(mark);
      return 0;
    }
    PolarCfg cfg;
    cfg.ell0 = 1e-15;  // fullsolve.cpp:40: no condition estimate, the safe bound
    DMat none;
    polar_decompose(ctx, Sh, cfg, Up, none);
    symmetrize_scale(ctx, Up, -0.5, 0.5, Up);  // C = sym((I - Up)/2)
    const double tr = device_trace(ctx, Up);
    k = std::llround(tr);
    // a clean split leaves trace(C) an integer to rounding (~n u); an eigenvalue
    // within ~l0 ||A|| of the shift is only partly mapped by QDWH (C keeps a
    // fractional eigenvalue: 0.046 measured on a singular shift, but 1e-7 .. 1e-9
    // when the distance is a few l0: measured 7e-9 at n = 99 with the trace mean on
    // an eigenvalue of a uniform grid — a looser test lets such a split through and
    // its two subspaces are then invariant only to that accuracy; clean splits
    // measure |trace - k| <= 1e-13 up to n = 777, a split accepted at 7e-11 cost
    // 0.8 of the residual gate)
    if (std::abs(tr - (double)k) < std::max(2e-13, 16.0 * (double)n * kEps)) break;
    k = -1;  // ambiguous: an eigenvalue at the shift
  }
  if (k <= 0 || k >= n) {
    ctx.arena->release_to(mark);
    syev(ctx, A, vals, Vout);
    return 0;
  }
  DMat Om = ctx.arena->alloc(n, n);
  gaussian_fill(ctx, Om, 0x73706c6974ull);  // kSplitSeed (fullsolve.cpp:14)
  DMat CO = ctx.arena->alloc(n, n);
  gemm(ctx, Op::N, Op::N, 1.0, Up, Om, 0.0, CO);
  QrWork qw;
  geqrf(ctx, CO, qw);
  DMat Q = ctx.arena->alloc(n, n);
  orgqr_cols(ctx, qw, n, n, 0, Q);
  const DMat Vlo = Q.sub(0, 0, n, k), Vhi = Q.sub(0, k, n, n - k);
  DMat T = ctx.arena->alloc(n, std::max(k, n - k));
  DMat Alo = ctx.arena->alloc(k, k), Ahi = ctx.arena->alloc(n - k, n - k);
  GemmExtra rr;  // Rayleigh quotients V^T (A V): lower tiles, mirrored (exactly symmetric)
  rr.out = OutMode::LowerMirror;
  gemm(ctx, Op::N, Op::N, 1.0, A, Vlo, 0.0, T.sub(0, 0, n, k));
  gemm(ctx, Op::T, Op::N, 1.0, Vlo, T.sub(0, 0, n, k), 0.0, Alo, rr);
  gemm(ctx, Op::N, Op::N, 1.0, A, Vhi, 0.0, T.sub(0, 0, n, n - k));
  gemm(ctx, Op::T, Op::N, 1.0, Vhi, T.sub(0, 0, n, n - k), 0.0, Ahi, rr);
  DMat Wlo = ctx.arena->alloc(k, k), Whi = ctx.arena->alloc(n - k, n - k);
  std::vector<double> vlo, vhi;
  const int64_t dlo = eig_full_rec(ctx, Alo, base, vlo, Wlo);
  const int64_t dhi = eig_full_rec(ctx, Ahi, base, vhi, Whi);
  gemm(ctx, Op::N, Op::N, 1.0, Vlo, Wlo, 0.0, Vout.sub(0, 0, n, k));
  gemm(ctx, Op::N, Op::N, 1.0, Vhi, Whi, 0.0, Vout.sub(0, k, n, n - k));
  vals = vlo;
  vals.insert(vals.end(), vhi.begin(), vhi.end());
  ctx.arena->release_to(mark);
  return 1 + std::max(dlo, dhi);
}

int64_t eig_full(Ctx& ctx, const DMat& A, int64_t base_size, std::vector<double>& vals, const DMat& Vout) {
  const int64_t n = A.rows;
  const Arena::Mark mark = ctx.arena->mark();
  DMat S = ctx.arena->alloc(n, n);
  symmetrize_scale(ctx, A, 1.0, 0.0, S);  // fullsolve.cpp:78: symmetrize(a)
  const int64_t depth = eig_full_rec(ctx, S, std::max<int64_t>(base_size, 2), vals, Vout);
  ctx.arena->release_to(mark);
  return depth;
}

// qdwh_svd_full (fullsolve.cpp:82-103): A = Up H, H = V diag(sigma) V^T by
// eig_full, U = Up V; descending order, negative rounding-level values clamped.
void svd_full(Ctx& ctx, const DMat& A, int64_t base_size, const DMat& U, std::vector<double>& sigma,
              const DMat& V) {
  const int64_t m = A.rows, n = A.cols;
  const Arena::Mark mark = ctx.arena->mark();
  DMat Up = ctx.arena->alloc(m, n), H = ctx.arena->alloc(n, n), W = ctx.arena->alloc(n, n);
  PolarCfg cfg;  // polar.hpp defaults (ell0 = 1e-15)
  polar_decompose(ctx, A, cfg, Up, H);
  std::vector<double> lam;
  eig_full(ctx, H, base_size, lam, W);
  sigma.resize(n);
  std::vector<int> order(n);
  for (int64_t j = 0; j < n; ++j) {
    sigma[j] = std::max(lam[n - 1 - j], 0.0);
    order[j] = (int)(n - 1 - j);
  }
  permute_cols(ctx, W, order, V);
  gemm(ctx, Op::N, Op::N, 1.0, Up, V, 0.0, U);
  ctx.arena->release_to(mark);
}

void syev(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout) {
  int64_t i0;
  syev_range(ctx, S, vals, Vout, -INFINITY, INFINITY, &i0);
}

int64_t syev_range(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout, double vlo,
                   double vhi, int64_t* sel0) {
  // Jacobi (n <= 16) / tridiagonal + bisection + inverse iteration (faster and
  // better orthogonality above: measured with the one-CTA small tridiagonal path
  // 0.32 vs 0.48 ms at n = 30, 0.42 ms at n = 49, 1.2 ms at n = 132, wall time
  // through the C ABI); the QDWH spectral divide-and-conquer remains the
  // fallback for tight clusters.  Only the eigenvectors of the eigenvalues in
  // (vlo, vhi) are formed (the tridiagonal path skips the others entirely).
  static const bool force_dc = getenv("QDWHG_SYEV_DC") != nullptr;
  static const int jac_max =
      getenv("QDWHG_JACOBI_MAX") ? std::min(atoi(getenv("QDWHG_JACOBI_MAX")), kJacobiMaxN) : 16;
  const int64_t n = S.rows;
  if (n > jac_max && !force_dc) {
    if (syev_tridiag(ctx, S, vals, Vout, vlo, vhi, sel0)) {
      int64_t c = 0;
      for (double v : vals) c += (v > vlo && v < vhi);
      return c;
    }
  }
  const Arena::Mark mark = ctx.arena->mark();
  DMat Wall = ctx.arena->alloc(n, n);
  syev_dc(ctx, S, vals, Wall, 0);
  int64_t i0 = 0, i1 = 0;
  while (i0 < n && !(vals[i0] > vlo)) ++i0;
  i1 = i0;
  while (i1 < n && vals[i1] < vhi) ++i1;
  if (i1 > i0) copy(ctx, Wall.sub(0, i0, n, i1 - i0), Vout.sub(0, 0, n, i1 - i0));
  ctx.arena->release_to(mark);
  *sel0 = i0;
  return i1 - i0;
}

// A lower bound of sigma_min(R) / alpha for an upper-triangular R (the QDWH l0,
// polar.hpp:35 leaves it to the caller with a 1e-15 default): from R^-1 (one
// triangular inverse, ~n^3/3 flops) sigma_min(R) = 1 / ||R^-1||_2, estimated by
// the power iteration with a 2x safety margin and floored by the guaranteed
// 1 / ||R^-1||_F.  Falls back to 1e-15 when R is singular to working precision.
double ell0_lower_bound(Ctx& ctx, const DMat& R, double alpha) {
  const int64_t n = R.rows;
  double l0 = 1e-15;
  const Arena::Mark m2 = ctx.arena->mark();
  DMat Ri = ctx.arena->alloc(n, n);
  if (trtri_upper(ctx, R, Ri)) {
    const MatStats st = mat_stats(ctx, Ri, false);
    if (st.nonfinite == 0 && st.fro2 > 0) {
      const double inv2 = two_norm_estimate(ctx, Ri);  // ~||R^-1||_2 (x1.05)
      const double lb = std::max(1.0 / (std::sqrt(st.fro2) * alpha), 1.0 / (2.0 * inv2 * alpha));
      if (std::isfinite(lb) && lb > l0) l0 = std::min(1.0, lb);
    }
  }
  ctx.arena->release_to(m2);
  return l0;
}

// l0 for polar_decompose(A) when the caller has none: the R factor of a
// Householder QR of A (sigma(R) = sigma(A)), then ell0_lower_bound against the
// polar's own alpha.
double polar_ell0_estimate(Ctx& ctx, const DMat& A) {
  const int64_t m = A.rows, n = A.cols;
  const Arena::Mark mark = ctx.arena->mark();
  DMat Aw = ctx.arena->alloc(m, n);
  copy(ctx, A, Aw);
  QrWork qw;
  geqrf(ctx, Aw, qw);
  DMat R = ctx.arena->alloc(n, n);
  copy(ctx, Aw.sub(0, 0, n, n), R);  // upper triangle (zeros below from the panels)
  const double l0 = ell0_lower_bound(ctx, R, two_norm_estimate(ctx, A));
  ctx.arena->release_to(mark);
  return l0;
}

int64_t svd_polar(Ctx& ctx, const DMat& A, const DMat& U, std::vector<double>& sigma, const DMat& V,
                  double cut, double ell0) {
  // fullsolve.cpp:82-103: A = Up H, H = W diag W^T, U = Up W, descending order.
  // Tall A (m > n) is first reduced to its n x n triangular factor (A = Q R), so
  // every QDWH iteration runs on n x n instead of m x n; U = Q U_R.
  // All n singular values are returned; singular vectors only for sigma > cut
  // (their count is returned): U(:, 0:k), V(:, 0:k).
  const int64_t m = A.rows, n = A.cols;
  if (m > n) {
    const Arena::Mark mark = ctx.arena->mark();
    // Householder (not CholeskyQR2: A Q2 can be ill-conditioned and R's accuracy
    // sets the small singular values' relative accuracy)
    DMat R = ctx.arena->alloc(n, n);
    DMat Aw = ctx.arena->alloc(m, n);
    copy(ctx, A, Aw);
    QrWork qw;
    geqrf(ctx, Aw, qw);
    copy(ctx, Aw.sub(0, 0, n, n), R);  // upper triangle (zeros below from the panels)
    // l0 for the polar of R: a lower bound of sigma_min(R / alpha) (saves QDWH
    // iterations, the QR-based ones above all: iterations_to_converge gives
    // 1e-15 -> 2 QR + 4 Cholesky steps, 1e-4 -> 1 QR + 3 Cholesky steps)
    const double l0 = ell0_lower_bound(ctx, R, two_norm_estimate(ctx, R));
    const int64_t k = svd_polar(ctx, R, U.sub(0, 0, n, n), sigma, V, cut, l0);
    // U = Q [U_R; 0]: the reflectors applied to U_R directly (no explicit Q,
    // no m x n x k GEMM)
    if (k > 0) {
      fill(ctx, U.sub(n, 0, m - n, k), 0.0, 0.0);
      ormqr_left(ctx, qw, m, n, U.sub(0, 0, m, k));
    }
    ctx.arena->release_to(mark);
    return k;
  }
  const Arena::Mark mark = ctx.arena->mark();
  DMat Up = ctx.arena->alloc(m, n);
  DMat H = ctx.arena->alloc(n, n);
  PolarCfg cfg;
  cfg.ell0 = ell0;
  polar_decompose(ctx, A, cfg, Up, H);
  std::vector<double> vals;
  DMat W = ctx.arena->alloc(n, n);
  int64_t i0 = 0;
  const int64_t k = syev_range(ctx, H, vals, W, cut, INFINITY, &i0);  // ascending, top-k block
  sigma.resize(n);
  for (int64_t j = 0; j < n; ++j) sigma[j] = std::max(0.0, vals[n - 1 - j]);
  if (k > 0) {
    // descending: V(:, j) = W(:, k-1-j)
    std::vector<int> order(k);
    for (int64_t j = 0; j < k; ++j) order[j] = (int)(k - 1 - j);
    permute_cols(ctx, W.sub(0, 0, n, k), order, V.sub(0, 0, n, k));
    gemm(ctx, Op::N, Op::N, 1.0, Up, V.sub(0, 0, n, k), 0.0, U.sub(0, 0, m, k));
  }
  ctx.arena->release_to(mark);
  return k;
}

static void check_finite(Ctx& ctx, const DMat& A, const char* who, MatStats* out = nullptr,
                         bool asym = false) {
  if (A.rows == 0 || A.cols == 0) throw InvalidArgument(std::string(who) + ": empty matrix");
  const MatStats st = mat_stats(ctx, A, asym);
  if (st.nonfinite > 0) throw InvalidArgument(std::string(who) + ": non-finite entry");
  if (out) *out = st;
}

// Subspace extraction for a SMALL subspace (partial.cpp:71-79 semantics, Cholesky
// QR instead of Householder): the R factor of the unpivoted QR of B is the
// Cholesky factor of B^T B, so
//   ind = first i with |W_ii| < tol,  W = chol(B^T B + delta I)
// (delta = 4 n u ||B||^2 only keeps the rank-deficient tail positive definite; it
// moves the |R_ii| >= tol pivots by ~delta / R_ii), and Q2 is an orthonormal basis
// of span(B1)^perp, B1 = B(:, 0:ind-1) — the subspace spanned by Q(:, ind-1:n)
// of the Householder QR — from a projected Gaussian block with exactly l columns
//   Y = (I - B1 G11^{-1} B1^T)^3 Omega,  G11^{-1} = W11^{-1} W11^{-T}
// (three passes: the delta-shifted projector leaves ~delta/sigma_min(B1)^2 per
// pass), Q2 = CholQR2(Y).  Everything is GEMM-shaped plus the Cholesky-and-inverse
// (the tile DAG): ~1.7 n^3 instead of the latency-bound panel chain of GEQRF.
// Used when l is small (trace(I - B) <= n/16, n/6 for n <= 2048); returns false
// to fall back.
static bool subspace_cholqr(Ctx& ctx, const DMat& B, double tol, size_t& ind, DMat& Q2out,
                            const DMat& Q2buf) {
  static const bool off = getenv("QDWHG_SUBSPACE_HOUSEHOLDER") != nullptr;
  const int64_t n = B.rows;
  if (off || B.cols != n || n < 1024) return false;
  // the delta shift below floors every |W_ii| at ~sqrt(delta): a tol that close
  // to it cannot be resolved by this path (the reference's Householder R can)
  const double delta = 32.0 * std::sqrt((double)n) * kEps;
  if (!(tol > 10.0 * std::sqrt(delta))) return false;
  // l estimate from trace(B): small subspaces (the projection costs ~8 n^2 l per
  // pass); up to n/6 where the Householder QR is latency-bound (n <= 2048, cfg1)
  const double lmax = (n <= 2048) ? (double)n / 6.0 : (double)n / 16.0;
  if ((double)n - device_trace(ctx, B) > lmax) return false;
  const Arena::Mark mark = ctx.arena->mark();
  DMat G = ctx.arena->alloc(n, n);
  DMat Winv = ctx.arena->alloc(n, n);
  GemmExtra syrk;
  syrk.out = OutMode::Lower;
  // ||B||_2 <= 1 (B = (X + I)/2, |eig(X)| <= 1): delta a few times the rounding
  // noise of the Gram's entries keeps the deficient tail positive definite
  syrk.diag_add = delta;
  syrk.fine_tail = true;
  gemm(ctx, Op::T, Op::N, 1.0, B, B, 0.0, G, syrk);
  try {
    potrf_upper_and_inverse(ctx, G, Winv, /*want_w=*/false, /*stable=*/false);
  } catch (const NotPositiveDefinite&) {
    ctx.arena->release_to(mark);
    return false;
  }
  // |R_ii| = W_ii = 1 / (W^{-1})_ii (triangular inverse: no need to write W out);
  // detect_deficiency_index, partial.cpp:32-38
  ind = (size_t)first_deficient(ctx, Winv, tol, /*reciprocal=*/true);
  if (ind == 0) {
    // no deficient pivot: confirmed on the reference's Householder path (as for k == 0)
    ctx.arena->release_to(mark);
    return false;
  }
  const int64_t ell = n - (int64_t)ind + 1, k1 = (int64_t)ind - 1;
  if (ell > Q2buf.cols || k1 < 1) {
    ctx.arena->release_to(mark);
    return false;
  }
  // exactly l columns: span(B1)^perp has dimension l, so the projection of l
  // Gaussian columns spans it (no oversampling, hence no r x r eigensolve to
  // drop rounding-level directions); CholQR2 orthonormalises
  Q2out = Q2buf.col_block(0, ell);
  DMat Y = Q2out;
  gaussian_fill(ctx, Y, 0x7375627370ull);  // fixed stream ("subsp")
  DMat T1 = ctx.arena->alloc(k1, ell), T2 = ctx.arena->alloc(k1, ell);
  const DMat B1 = B.col_block(0, k1), W11i = Winv.sub(0, 0, k1, k1);
  // Richardson passes of the least-squares projection: each leaves ~delta /
  // sigma_min(B1)^2 (+ u kappa(B1)^2) of what is left in span(B1); three passes,
  // and the caller checks the Ritz residuals of the result (falls back otherwise)
  static const int npass = getenv("QDWHG_SUBSPACE_PASSES") ? std::max(1, atoi(getenv("QDWHG_SUBSPACE_PASSES"))) : 3;
  for (int pass = 0; pass < npass; ++pass) {
    GemmExtra sk;  // l-column blocks against n x n: the two-per-SM 64-tile plan
    sk.skinny = true;
    gemm(ctx, Op::T, Op::N, 1.0, B1, Y, 0.0, T1, sk);       // B1^T Y
    GemmExtra lo = sk;
    lo.krange = KRange::ALower;                              // W11^{-T} lower
    gemm(ctx, Op::T, Op::N, 1.0, W11i, T1, 0.0, T2, lo);
    GemmExtra up = sk;
    up.krange = KRange::AUpper;                              // W11^{-1} upper
    gemm(ctx, Op::N, Op::N, 1.0, W11i, T2, 0.0, T1, up);
    gemm(ctx, Op::N, Op::N, -1.0, B1, T1, 1.0, Y, sk);       // Y -= B1 G11^{-1} B1^T Y
  }
  // CholQR2: Q2 <- Q2 F^{-1}, F = chol(Q2^T Q2), twice (kappa(Y) of a projected
  // Gaussian block is O(sqrt(l)): the second pass reaches rounding-level
  // orthogonality).  kappa(F) = kappa(Y)^2 is small, so the fast Cholesky-and-
  // inverse is accurate here (the stable panel variant cost 0.15 ms per pass at l = 132)
  DMat F = ctx.arena->alloc(ell, ell), Fi = ctx.arena->alloc(ell, ell), Qt = ctx.arena->alloc(n, ell);
  for (int pass = 0; pass < 2; ++pass) {
    GemmExtra fl;
    fl.out = OutMode::Lower;
    gemm(ctx, Op::T, Op::N, 1.0, Q2out, Q2out, 0.0, F, fl);
    try {
      potrf_upper_and_inverse(ctx, F, Fi, false, /*stable=*/false);
    } catch (const NotPositiveDefinite&) {
      ctx.arena->release_to(mark);
      return false;
    }
    copy(ctx, Q2out, Qt);
    GemmExtra bu;
    bu.krange = KRange::BUpper;
    bu.skinny = true;
    gemm(ctx, Op::N, Op::N, 1.0, Qt, Fi, 0.0, Q2out, bu);
  }
  ctx.arena->release_to(mark);
  return true;
}

EigOut partial_eig(Ctx& ctx, const DMat& A, double s, size_t iters, bool randomize, double tol,
                   uint64_t seed, StageClock* clk) {
  // partial.cpp:40-99
  const int64_t n = A.rows;
  if (A.cols != n) throw InvalidArgument("qdwh_partial_eig: matrix not square");
  MatStats st;
  check_finite(ctx, A, "qdwh_partial_eig", &st, true);
  if (st.asym > 1e3 * (double)n * kEps * std::max(1.0, std::sqrt(st.fro2)))
    throw InvalidArgument("qdwh_partial_eig: input not symmetric within tolerance");
  EigOut out;
  out.shift = s;
  out.tol = tol;
  out.randomized = randomize;
  out.mu = lanczos_min_bound(ctx, A, 30, &st);
  if (clk) clk->mark(0);
  if (out.mu >= 0.0) return out;  // partial.cpp:52
  const double scale = std::abs(out.mu);
  DMat As = ctx.arena->alloc(n, n);
  DMat X = ctx.arena->alloc(n, n);
  // As = sym(A)/|mu| and X = (1-s) As - s I (partial.cpp:54-59) from one read of A
  symmetrize_scale2(ctx, A, 1.0 / scale, 0.0, As, 1.0 - s, -s, X);
  // X = (1-s) sym(A)/|mu| - s I is exactly symmetric (symmetrize_scale above)
  FixedIterResult it = run_fixed_iterations(ctx, X, s, iters, false, true);
  out.trace = it.trace;
  out.iters_qr = it.iters_qr;
  out.iters_chol = it.iters_chol;
  if (clk) clk->mark(1);
  // B = (r(A~) + I)/2 (partial.cpp:67-69)
  axpby_identity(ctx, X, 0.5, 0.5, X);
  DMat B = X;
  if (randomize) {
    DMat Om = ctx.arena->alloc(n, n);
    gaussian_fill(ctx, Om, seed);
    B = ctx.arena->alloc(n, n);
    gemm(ctx, Op::N, Op::N, 1.0, X, Om, 0.0, B);
  }
  // small subspace: Cholesky-QR extraction first (same ind, same span), verified by
  // the Ritz residuals of the result; otherwise (or if that check fails) the
  // reference's Householder QR + trailing-column Q formation
  const Arena::Mark sub_mark = ctx.arena->mark();
  const double nd = (double)n;
  const double as_fro = std::sqrt(st.fro2) / scale;
  for (int attempt = 0; attempt < 2; ++attempt) {
    ctx.arena->release_to(sub_mark);
    out.rank_index = 0;
    out.subspace_size = 0;
    out.no_savings = false;
    out.borderline = 0;
    out.subspace_path = 0;
    out.lambda.clear();
    out.V = DMat{};
    size_t ind = 0;
    DMat Q2;
    const DMat Q2buf =
        (randomize || attempt > 0) ? DMat{} : ctx.arena->alloc(n, std::max<int64_t>(1, n <= 2048 ? n / 4 : n / 8));
    const bool chq = !randomize && attempt == 0 && subspace_cholqr(ctx, B, tol, ind, Q2, Q2buf);
    out.subspace_path = chq ? 1 : 0;
    QrWork qw;
    if (!chq) {
      geqrf(ctx, B, qw);
      ind = (size_t)first_deficient(ctx, B, tol);  // detect_deficiency_index, partial.cpp:32-38
    }
    if (clk) clk->mark(2);
    out.flops = it.iters_chol * (10.0 / 3.0) * nd * nd * nd + 4.0 / 3.0 * nd * nd * nd +
                (randomize ? 2 * nd * nd * nd : 0.0);
    if (ind == 0) return out;
    out.rank_index = ind;
    const int64_t ell = n - (int64_t)ind + 1;
    out.subspace_size = ell;
    out.no_savings = ell > n / 2;
    if (!chq) {
      Q2 = ctx.arena->alloc(n, ell);
      orgqr_cols(ctx, qw, n, n, (int64_t)ind - 1, Q2);
    }
    if (clk) clk->mark(3);
    DMat AQ = ctx.arena->alloc(n, ell);
    GemmExtra sk;  // n x l products: the two-per-SM 64-tile plan when the model picks 64 tiles
    sk.skinny = true;
    gemm(ctx, Op::N, Op::N, 1.0, As, Q2, 0.0, AQ, sk);
    DMat S = ctx.arena->alloc(ell, ell);
    GemmExtra rr;  // S = Q2^T (A Q2) is symmetric: lower tiles, mirrored (exactly symmetric)
    rr.out = OutMode::LowerMirror;
    gemm(ctx, Op::T, Op::N, 1.0, Q2, AQ, 0.0, S, rr);
    if (clk) clk->mark(4);
    std::vector<double> vals;
    DMat W = ctx.arena->alloc(ell, ell);
    int64_t sel0 = 0;
    syev_range(ctx, S, vals, W, -INFINITY, 0.0, &sel0);  // vectors for the negative Ritz values only
    if (clk) clk->mark(5);
    double max_abs_ritz = 0.0;
    for (double v : vals) max_abs_ritz = std::max(max_abs_ritz, std::abs(v));
    const double floor = -nd * kEps * max_abs_ritz;
    int64_t k = 0;
    while (k < ell && vals[k] < 0.0) ++k;
    const double l = (double)ell;
    out.flops += 2 * nd * nd * l - 2 * l * l * l / 3 + 2 * nd * nd * l + 2 * nd * l * l + 9 * l * l * l;
    if (k == 0) {
      if (chq) continue;  // confirm an empty result on the reference path
      return out;
    }
    out.lambda.resize(k);
    for (int64_t i = 0; i < k; ++i) {
      out.lambda[i] = scale * vals[i];
      if (vals[i] >= floor) ++out.borderline;
    }
    out.V = ctx.arena->alloc(n, k);
    gemm(ctx, Op::N, Op::N, 1.0, Q2, W.sub(0, 0, ell, k), 0.0, out.V, sk);
    out.flops += 2 * nd * l * (double)k;
    if (chq) {
      // Ritz residual ||As V - V Lambda||_F against 1e-13 sqrt(n) ||As||_F (10x inside
      // the north-star gate): a subspace that lost accuracy is redone by Householder
      const Arena::Mark rm = ctx.arena->mark();
      DMat R = ctx.arena->alloc(n, k), D = ctx.arena->alloc(k, k);
      std::vector<double> hd((size_t)k * k, 0.0);
      for (int64_t i = 0; i < k; ++i) hd[i + (size_t)i * k] = vals[i];
      copy_from_host(ctx, hd.data(), k, D);
      // As V = (As Q2) W_k: the n x l product is already there (AQ), no n^2 k GEMM
      gemm(ctx, Op::N, Op::N, 1.0, AQ, W.sub(0, 0, ell, k), 0.0, R);
      gemm(ctx, Op::N, Op::N, -1.0, out.V, D, 1.0, R);
      const double res = std::sqrt(mat_stats(ctx, R, false).fro2);
      ctx.arena->release_to(rm);
      if (!(res <= 1e-13 * std::sqrt(nd) * as_fro)) continue;
    }
    break;
  }
  if (clk) clk->mark(6);
  return out;
}

SvdOut partial_svd(Ctx& ctx, const DMat& A, double s, double s_abs, double tol, bool randomize,
                   uint64_t seed, StageClock* clk) {
  // partial.cpp:101-158
  const int64_t m = A.rows, n = A.cols;
  check_finite(ctx, A, "qdwh_partial_svd");
  if (m < n) throw InvalidArgument("qdwh_partial_svd: requires rows >= cols");
  SvdOut out;
  out.tol = tol;
  out.randomized = randomize;
  out.alpha = two_norm_estimate(ctx, A);
  if (s_abs > 0.0) s = s_abs / out.alpha;
  if (!(s > 0.0) || s >= 1.0)
    throw InvalidArgument("qdwh_partial_svd: threshold s must be in (0, 1)");
  out.threshold = s;
  if (clk) clk->mark(0);
  DMat X = ctx.arena->alloc(m, n);
  axpby_identity(ctx, A, 1.0 / out.alpha, 0.0, X);
  const size_t iters = iterations_to_converge(s, 5.0 * kEps);
  if (iters > 0) {
    FixedIterResult it = run_fixed_iterations(ctx, X, s, iters, s < 1e-3);
    out.trace = it.trace;
    out.iters_qr = it.iters_qr;
    out.iters_chol = it.iters_chol;
  } else {
    out.trace.push_back(s);
  }
  if (clk) clk->mark(1);
  // M = I - sym(X^T X) (partial.cpp:134-136)
  DMat M = ctx.arena->alloc(n, n);
  GemmExtra syrk;
  syrk.out = OutMode::LowerMirror;
  syrk.diag_add = 1.0;
  gemm(ctx, Op::T, Op::N, -1.0, X, X, 0.0, M, syrk);
  DMat B = M;
  if (randomize) {
    DMat Om = ctx.arena->alloc(n, n);
    gaussian_fill(ctx, Om, seed);
    B = ctx.arena->alloc(n, n);
    gemm(ctx, Op::N, Op::N, 1.0, M, Om, 0.0, B);
  }
  QrWork qw;
  geqrf(ctx, B, qw);
  const size_t ind = (size_t)first_deficient(ctx, B, tol);  // partial.cpp:32-38
  if (clk) clk->mark(2);
  const double md = (double)m, nd = (double)n;
  out.flops = out.iters_qr * (6 * md * nd * nd + 8.0 / 3.0 * nd * nd * nd) +
              out.iters_chol * (3 * md * nd * nd + nd * nd * nd / 3) + md * nd * nd +
              4.0 / 3.0 * nd * nd * nd + (randomize ? 2 * nd * nd * nd : 0.0);
  if (ind == 0) return out;
  out.rank_index = ind;
  const int64_t ell = n - (int64_t)ind + 1;
  out.subspace_size = ell;
  out.no_savings = ell > n / 2;
  DMat Q2 = ctx.arena->alloc(n, ell);
  orgqr_cols(ctx, qw, n, n, (int64_t)ind - 1, Q2);
  if (clk) clk->mark(3);
  DMat Y = ctx.arena->alloc(m, ell);
  gemm(ctx, Op::N, Op::N, 1.0, A, Q2, 0.0, Y);  // unscaled A (partial.cpp:147)
  if (clk) clk->mark(4);
  DMat Us = ctx.arena->alloc(m, ell), Vs = ctx.arena->alloc(ell, ell);
  std::vector<double> sig;
  const double cutoff = s * out.alpha;
  svd_polar(ctx, Y, Us, sig, Vs, cutoff);  // vectors only for sigma > cutoff (partial.cpp:151)
  if (clk) clk->mark(5);
  int64_t k = 0;
  while (k < (int64_t)sig.size() && sig[k] > cutoff) ++k;
  const double l = (double)ell;
  out.flops += 2 * nd * nd * l - 2 * l * l * l / 3 + 2 * md * nd * l + 6 * md * l * l + 20 * l * l * l;
  if (k == 0) return out;
  out.sigma.assign(sig.begin(), sig.begin() + k);
  out.U = Us.sub(0, 0, m, k);
  out.V = ctx.arena->alloc(n, k);
  gemm(ctx, Op::N, Op::N, 1.0, Q2, Vs.sub(0, 0, ell, k), 0.0, out.V);
  out.flops += 2 * nd * l * (double)k;
  if (clk) clk->mark(6);
  return out;
}

}  // namespace qdwhg
