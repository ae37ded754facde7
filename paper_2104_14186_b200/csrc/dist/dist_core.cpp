// Distributed building blocks on the 2D block-cyclic layout (see dist.hpp):
// SUMMA-style GEMM with grouped panel broadcasts, the recursive
// Cholesky-and-inverse, Householder QR with world-broadcast panels, trailing-
// column Q formation, tile transposes and replicated-vector GEMV.
// CUDA-free: everything goes through Engine (local compute) and Comm.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "dist.hpp"

namespace qdwhg {
namespace dist {

int64_t numroc(int64_t n, int64_t nb, int iproc, int nprocs) {
  const int64_t nblocks = n / nb;
  int64_t num = (nblocks / nprocs) * nb;
  const int64_t extra = nblocks % nprocs;
  if (iproc < extra) num += nb;
  else if (iproc == extra) num += n % nb;
  return num;
}

DistMat make_dist(Engine& e, const Grid& g, int64_t m, int64_t n) {
  DistMat d;
  d.m = m;
  d.n = n;
  d.g = &g;
  d.lr = numroc(m, g.nb, g.p, g.P);
  d.lc = numroc(n, g.nb, g.q, g.Q);
  d.a = e.alloc(std::max<int64_t>(d.lr, 1), std::max<int64_t>(d.lc, 1), &d.ld);
  return d;
}

namespace {

// Tiles t in [t0, t0 + nt) with t % np == ip: first/last global tile, count and
// the local element range [l0, l0 + len) they occupy (contiguous locally).
struct LRange {
  int64_t first = -1, last = -1, cnt = 0, l0 = 0, len = 0;
  bool empty() const { return cnt == 0; }
  // local element offset of global tile t (owned) within the range
  int64_t off(int64_t t, int np, int64_t nb) const { return (t / np - first / np) * nb; }
};

LRange lrange(int64_t t0, int64_t nt, int ip, int np, int64_t nb, int64_t total) {
  LRange r;
  if (nt <= 0) return r;
  const int64_t first = t0 + (((ip - t0 % np) % np) + np) % np;
  if (first >= t0 + nt) return r;
  r.first = first;
  r.last = first + ((t0 + nt - 1 - first) / np) * np;
  r.cnt = (r.last - r.first) / np + 1;
  r.l0 = (first / np) * nb;
  r.len = (r.last / np) * nb + std::min<int64_t>(nb, total - r.last * nb) - r.l0;
  return r;
}

int64_t tile_len(int64_t t, int64_t nb, int64_t total) { return std::min<int64_t>(nb, total - t * nb); }

// The whole tile-aligned view replicated on every rank: one world broadcast per
// owner (P*Q in one group); tile(I, J) addresses the staged copy (global tiles).
struct FullView {
  const View* v = nullptr;
  std::vector<double*> stage;  // [p * Q + q]
  std::vector<LRange> rr, cr;  // per process row / column
  int P = 1, Q = 1;
  int64_t nb = 0;
  const double* tile(int64_t I, int64_t J, int64_t* ld) const {
    const int pr = (int)(I % P), pc = (int)(J % Q);
    *ld = rr[pr].len;
    return stage[pr * Q + pc] + rr[pr].off(I, P, nb) + cr[pc].off(J, Q, nb) * rr[pr].len;
  }
};

void fetch_full(Ctx& c, const View& v, FullView& f) {
  const Grid& g = c.g;
  const DistMat& M = *v.M;
  f.v = &v;
  f.P = g.P;
  f.Q = g.Q;
  f.nb = g.nb;
  f.rr.resize(g.P);
  f.cr.resize(g.Q);
  f.stage.assign((size_t)g.P * g.Q, nullptr);
  for (int pr = 0; pr < g.P; ++pr) f.rr[pr] = lrange(v.i0, v.mt, pr, g.P, g.nb, M.m);
  for (int pc = 0; pc < g.Q; ++pc) f.cr[pc] = lrange(v.j0, v.nt, pc, g.Q, g.nb, M.n);
  // pack my own block first (the root's send buffer)
  for (int pr = 0; pr < g.P; ++pr)
    for (int pc = 0; pc < g.Q; ++pc) {
      if (f.rr[pr].empty() || f.cr[pc].empty()) continue;
      int64_t ldd;
      f.stage[pr * g.Q + pc] = c.eng->alloc(f.rr[pr].len, f.cr[pc].len, &ldd);
      (void)ldd;
      if (pr == g.p && pc == g.q)
        c.eng->copy_tiles({TileCopy{M.a + f.rr[pr].l0 + f.cr[pc].l0 * M.ld, M.ld, f.stage[pr * g.Q + pc],
                                    f.rr[pr].len, (int32_t)f.rr[pr].len, (int32_t)f.cr[pc].len, 0}});
    }
  c.comm->group_begin();
  for (int pr = 0; pr < g.P; ++pr)
    for (int pc = 0; pc < g.Q; ++pc) {
      if (f.rr[pr].empty() || f.cr[pc].empty()) continue;
      c.comm->bcast(f.stage[pr * g.Q + pc], (size_t)(f.rr[pr].len * f.cr[pc].len), g.world_rank(pr, pc),
                    Team::World);
      ++c.collectives;
    }
  c.comm->group_end();
}

bool same_view(const View& a, const View& b) {
  return a.M == b.M && a.i0 == b.i0 && a.j0 == b.j0 && a.mt == b.mt && a.nt == b.nt;
}

// One local GEMM over tile-aligned pieces of the fetched operands.
struct LocalOps {
  bool ta, tb;
  const double *A, *B;
  int64_t lda, ldb;
  double* C;
  int64_t ldc;
  // A piece for local rows [r0, r0+rn) and K range [k0, k0+kn)
  const double* a_at(int64_t r0, int64_t k0) const { return ta ? A + k0 + r0 * lda : A + r0 + k0 * lda; }
  const double* b_at(int64_t k0, int64_t c0) const { return tb ? B + c0 + k0 * ldb : B + k0 + c0 * ldb; }
};

}  // namespace

void pgemm(Ctx& c, bool ta, bool tb, double alpha, const View& A, const View& B, double beta,
           const View& C, const Structure& st) {
  const Grid& g = c.g;
  const int64_t nb = g.nb;
  const int64_t M = C.mt, N = C.nt;
  const int64_t K = ta ? A.mt : A.nt;
  if ((ta ? A.nt : A.mt) != M || (tb ? B.mt : B.nt) != N || (tb ? B.nt : B.mt) != K)
    throw InvalidArgument("pgemm: tile shapes do not conform");
  const DistMat& Am = *A.M;
  const DistMat& Bm = *B.M;
  const DistMat& Cm = *C.M;
  // k-tile widths and element offsets (the k order is the view order on both sides)
  std::vector<int64_t> kw(K), koff(K + 1, 0);
  for (int64_t kt = 0; kt < K; ++kt) {
    kw[kt] = ta ? tile_len(A.i0 + kt, nb, Am.m) : tile_len(A.j0 + kt, nb, Am.n);
    const int64_t wb = tb ? tile_len(B.j0 + kt, nb, Bm.n) : tile_len(B.i0 + kt, nb, Bm.m);
    if (wb != kw[kt]) throw InvalidArgument("pgemm: inner tile widths differ");
    koff[kt + 1] = koff[kt] + kw[kt];
  }
  const int64_t Kel = koff[K];
  const LRange rC = lrange(C.i0, M, g.p, g.P, nb, Cm.m);
  const LRange cC = lrange(C.j0, N, g.q, g.Q, nb, Cm.n);
  const EMark mk = c.eng->mark();
  Engine& e = *c.eng;

  // ---- operand A: op(A) rows of my C rows, all K
  int64_t ldA = 0, ldB = 0;
  double* Abuf = nullptr;
  double* Bbuf = nullptr;
  if (!rC.empty() && Kel > 0) Abuf = ta ? e.alloc(Kel, rC.len, &ldA) : e.alloc(rC.len, Kel, &ldA);
  if (!cC.empty() && Kel > 0) Bbuf = tb ? e.alloc(cC.len, Kel, &ldB) : e.alloc(Kel, cC.len, &ldB);
  const bool a_aligned = !ta && ((A.i0 - C.i0) % g.P + g.P) % g.P == 0;
  const bool b_aligned = !tb && ((B.j0 - C.j0) % g.Q + g.Q) % g.Q == 0;
  FullView fa, fb;
  std::vector<TileCopy> place;
  if (K > 0 && a_aligned) {
    // my process row holds the rows: one row-team broadcast per process column
    const LRange rA = lrange(A.i0, M, g.p, g.P, nb, Am.m);
    if (rA.len != rC.len) throw InvalidArgument("pgemm: aligned A rows differ from C rows");
    std::vector<double*> stg(g.Q, nullptr);
    std::vector<LRange> crA(g.Q);
    for (int pc = 0; pc < g.Q; ++pc) {
      crA[pc] = lrange(A.j0, K, pc, g.Q, nb, Am.n);
      if (rA.empty() || crA[pc].empty()) continue;
      int64_t ld;
      stg[pc] = e.alloc(rA.len, crA[pc].len, &ld);
      if (pc == g.q)
        e.copy_tiles({TileCopy{Am.a + rA.l0 + crA[pc].l0 * Am.ld, Am.ld, stg[pc], rA.len, (int32_t)rA.len,
                               (int32_t)crA[pc].len, 0}});
    }
    c.comm->group_begin();
    for (int pc = 0; pc < g.Q; ++pc) {
      if (!stg[pc]) continue;
      c.comm->bcast(stg[pc], (size_t)(rA.len * crA[pc].len), g.world_rank(g.p, pc), Team::Row);
      ++c.collectives;
    }
    c.comm->group_end();
    if (Abuf)
      for (int64_t kt = 0; kt < K; ++kt) {
        const int pc = (int)((A.j0 + kt) % g.Q);
        place.push_back(TileCopy{stg[pc] + crA[pc].off(A.j0 + kt, g.Q, nb) * rA.len, rA.len,
                                 Abuf + koff[kt] * ldA, ldA, (int32_t)rA.len, (int32_t)kw[kt], 0});
      }
  } else if (K > 0) {
    fetch_full(c, A, fa);
    if (Abuf)
      for (int64_t I = rC.first; I >= 0 && I <= rC.last; I += g.P) {
        const int64_t i = I - C.i0;  // view-relative row tile
        const int64_t ro = rC.off(I, g.P, nb);
        for (int64_t kt = 0; kt < K; ++kt) {
          int64_t lds;
          if (!ta) {
            const double* s = fa.tile(A.i0 + i, A.j0 + kt, &lds);
            place.push_back(TileCopy{s, lds, Abuf + ro + koff[kt] * ldA, ldA,
                                     (int32_t)tile_len(A.i0 + i, nb, Am.m), (int32_t)kw[kt], 0});
          } else {
            const double* s = fa.tile(A.i0 + kt, A.j0 + i, &lds);
            place.push_back(TileCopy{s, lds, Abuf + koff[kt] + ro * ldA, ldA, (int32_t)kw[kt],
                                     (int32_t)tile_len(A.j0 + i, nb, Am.n), 0});
          }
        }
      }
  }
  // ---- operand B: op(B) columns of my C columns, all K
  if (K > 0 && b_aligned) {
    const LRange cB = lrange(B.j0, N, g.q, g.Q, nb, Bm.n);
    if (cB.len != cC.len) throw InvalidArgument("pgemm: aligned B columns differ from C columns");
    std::vector<double*> stg(g.P, nullptr);
    std::vector<LRange> rB(g.P);
    for (int pr = 0; pr < g.P; ++pr) {
      rB[pr] = lrange(B.i0, K, pr, g.P, nb, Bm.m);
      if (cB.empty() || rB[pr].empty()) continue;
      int64_t ld;
      stg[pr] = e.alloc(rB[pr].len, cB.len, &ld);
      if (pr == g.p)
        e.copy_tiles({TileCopy{Bm.a + rB[pr].l0 + cB.l0 * Bm.ld, Bm.ld, stg[pr], rB[pr].len,
                               (int32_t)rB[pr].len, (int32_t)cB.len, 0}});
    }
    c.comm->group_begin();
    for (int pr = 0; pr < g.P; ++pr) {
      if (!stg[pr]) continue;
      c.comm->bcast(stg[pr], (size_t)(rB[pr].len * cB.len), g.world_rank(pr, g.q), Team::Col);
      ++c.collectives;
    }
    c.comm->group_end();
    if (Bbuf)
      for (int64_t kt = 0; kt < K; ++kt) {
        const int pr = (int)((B.i0 + kt) % g.P);
        place.push_back(TileCopy{stg[pr] + rB[pr].off(B.i0 + kt, g.P, nb), rB[pr].len, Bbuf + koff[kt], ldB,
                                 (int32_t)kw[kt], (int32_t)cB.len, 0});
      }
  } else if (K > 0) {
    const bool reuse = !a_aligned && same_view(A, B);
    if (!reuse) fetch_full(c, B, fb);
    const FullView& f = reuse ? fa : fb;
    if (Bbuf)
      for (int64_t J = cC.first; J >= 0 && J <= cC.last; J += g.Q) {
        const int64_t j = J - C.j0;
        const int64_t co = cC.off(J, g.Q, nb);
        for (int64_t kt = 0; kt < K; ++kt) {
          int64_t lds;
          if (!tb) {
            const double* s = f.tile(B.i0 + kt, B.j0 + j, &lds);
            place.push_back(TileCopy{s, lds, Bbuf + koff[kt] + co * ldB, ldB, (int32_t)kw[kt],
                                     (int32_t)tile_len(B.j0 + j, nb, Bm.n), 0});
          } else {
            const double* s = f.tile(B.i0 + j, B.j0 + kt, &lds);
            place.push_back(TileCopy{s, lds, Bbuf + co + koff[kt] * ldB, ldB,
                                     (int32_t)tile_len(B.i0 + j, nb, Bm.m), (int32_t)kw[kt], 0});
          }
        }
      }
  }
  if (!place.empty()) e.copy_tiles(place);

  // ---- local products
  if (!rC.empty() && !cC.empty()) {
    double* Cl = Cm.a + rC.l0 + cC.l0 * Cm.ld;
    LocalOps lo{ta, tb, Abuf, Bbuf, ldA, ldB, Cl, Cm.ld};
    const bool structured = st.a_upper || st.a_lower || st.b_upper || st.b_lower || st.c_lower;
    auto krange = [&](int64_t i, int64_t j, int64_t* klo, int64_t* khi) {
      *klo = 0;
      *khi = K;
      if (st.a_upper) *klo = std::max(*klo, i);
      if (st.a_lower) *khi = std::min(*khi, i + 1);
      if (st.b_upper) *khi = std::min(*khi, j + 1);
      if (st.b_lower) *klo = std::max(*klo, j);
    };
    auto run = [&](int64_t ro, int64_t rn, int64_t co, int64_t cn, int64_t klo, int64_t khi) {
      double* Cp = Cl + ro + co * Cm.ld;
      if (khi <= klo || Kel == 0) {
        if (beta == 0.0) e.fill(Cp, Cm.ld, rn, cn, 0.0);
        else if (beta != 1.0) e.axpby(nullptr, 0, Cp, Cm.ld, rn, cn, 0.0, beta);
        return;
      }
      e.gemm(ta, tb, rn, cn, koff[khi] - koff[klo], alpha, lo.a_at(ro, koff[klo]), ldA,
             lo.b_at(koff[klo], co), ldB, beta, Cp, Cm.ld);
      ++c.gemms;
    };
    if (!structured) {
      run(0, rC.len, 0, cC.len, 0, K);
    } else {
      // my tiles (view-relative i, j) with their k ranges; pick the grouping
      // (per tile row, per tile column, or per tile) with the fewest launches
      const bool by_row_ok = !(st.b_upper || st.b_lower) || (st.c_lower && st.b_lower && st.a_upper);
      const bool by_col_ok = !(st.a_upper || st.a_lower);
      if (by_col_ok) {
        for (int64_t J = cC.first; J <= cC.last; J += g.Q) {
          const int64_t j = J - C.j0, co = cC.off(J, g.Q, nb), cn = tile_len(J, nb, Cm.n);
          int64_t I0 = rC.first;
          if (st.c_lower) {
            while (I0 <= rC.last && I0 - C.i0 < j) I0 += g.P;
            if (I0 > rC.last) continue;
          }
          int64_t klo, khi;
          krange(I0 - C.i0, j, &klo, &khi);
          const int64_t ro = rC.off(I0, g.P, nb);
          run(ro, rC.len - ro, co, cn, klo, khi);
        }
      } else if (by_row_ok) {
        for (int64_t I = rC.first; I <= rC.last; I += g.P) {
          const int64_t i = I - C.i0, ro = rC.off(I, g.P, nb), rn = tile_len(I, nb, Cm.m);
          int64_t J1 = cC.last;
          if (st.c_lower) {
            while (J1 >= cC.first && J1 - C.j0 > i) J1 -= g.Q;
            if (J1 < cC.first) continue;
          }
          int64_t klo, khi;
          krange(i, J1 - C.j0, &klo, &khi);
          const int64_t cn = cC.off(J1, g.Q, nb) + tile_len(J1, nb, Cm.n);
          run(ro, rn, 0, cn, klo, khi);
        }
      } else {
        for (int64_t J = cC.first; J <= cC.last; J += g.Q)
          for (int64_t I = rC.first; I <= rC.last; I += g.P) {
            const int64_t i = I - C.i0, j = J - C.j0;
            if (st.c_lower && i < j) continue;
            int64_t klo, khi;
            krange(i, j, &klo, &khi);
            run(rC.off(I, g.P, nb), tile_len(I, nb, Cm.m), cC.off(J, g.Q, nb), tile_len(J, nb, Cm.n), klo,
                khi);
          }
      }
    }
  }
  e.release(mk);
}

// ------------------------------------------------------------------ tile exchange
// For every owned tile (I, J) selected by `want`, the transposed tile goes to the
// owner of (J, I), which applies `store` to it there.  One grouped send/recv per
// peer (tiles packed back to back), diagonal tiles handled locally.
namespace {
template <typename Sel>
void transpose_exchange(Ctx& c, const DistMat& X, const DistMat& Y, Sel want, bool diag_mirror) {
  const Grid& g = c.g;
  Engine& e = *c.eng;
  const int me = g.world_rank(g.p, g.q);
  const int nr = g.P * g.Q;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> out(nr), in(nr);
  for (int64_t I = 0; I < X.mt(); ++I)
    for (int64_t J = 0; J < X.nt(); ++J) {
      if (!want(I, J)) continue;
      const int src = g.world_rank((int)(I % g.P), (int)(J % g.Q));
      const int dst = g.world_rank((int)(J % g.P), (int)(I % g.Q));
      if (src == me && dst == me) continue;
      if (src == me) out[dst].push_back({I, J});
      if (dst == me) in[src].push_back({I, J});
    }
  const EMark mk = e.mark();
  std::vector<double*> sb(nr, nullptr), rb(nr, nullptr);
  std::vector<size_t> sc(nr, 0), rc(nr, 0);
  std::vector<TileCopy> pack, unpack;
  for (int r = 0; r < nr; ++r) {
    for (auto& t : out[r]) sc[r] += (size_t)(X.tile_rows(t.first) * X.tile_cols(t.second));
    for (auto& t : in[r]) rc[r] += (size_t)(X.tile_rows(t.first) * X.tile_cols(t.second));
    if (sc[r]) sb[r] = e.alloc_vec(sc[r]);
    if (rc[r]) rb[r] = e.alloc_vec(rc[r]);
    size_t o = 0;
    for (auto& t : out[r]) {  // packed transposed: (cols x rows) per tile
      const int64_t tr = X.tile_rows(t.first), tc = X.tile_cols(t.second);
      pack.push_back(TileCopy{X.tile(t.first, t.second), X.ld, sb[r] + o, tc, (int32_t)tr, (int32_t)tc, 1});
      o += (size_t)(tr * tc);
    }
    o = 0;
    for (auto& t : in[r]) {  // lands as tile (J, I) of Y
      const int64_t tr = X.tile_rows(t.first), tc = X.tile_cols(t.second);
      unpack.push_back(TileCopy{rb[r] + o, tc, Y.tile(t.second, t.first), Y.ld, (int32_t)tc, (int32_t)tr, 0});
      o += (size_t)(tr * tc);
    }
  }
  // local tiles (owner of (I, J) also owns (J, I))
  std::vector<TileCopy> local;
  for (int64_t I = 0; I < X.mt(); ++I)
    for (int64_t J = 0; J < X.nt(); ++J) {
      if (!want(I, J)) continue;
      const int src = g.world_rank((int)(I % g.P), (int)(J % g.Q));
      const int dst = g.world_rank((int)(J % g.P), (int)(I % g.Q));
      if (src != me || dst != me) continue;
      if (I == J && diag_mirror) {
        if (X.a != Y.a) e.copy_tiles({TileCopy{X.tile(I, I), X.ld, Y.tile(I, I), Y.ld, (int32_t)X.tile_rows(I),
                                               (int32_t)X.tile_cols(I), 0}});
        e.mirror_lower(Y.tile(I, I), Y.ld, X.tile_rows(I));
        continue;
      }
      local.push_back(TileCopy{X.tile(I, J), X.ld, Y.tile(J, I), Y.ld, (int32_t)X.tile_rows(I),
                               (int32_t)X.tile_cols(J), 1});
    }
  if (!pack.empty()) e.copy_tiles(pack);
  c.comm->group_begin();
  for (int r = 0; r < nr; ++r) {
    if (sc[r]) c.comm->send(sb[r], sc[r], r);
    if (rc[r]) c.comm->recv(rb[r], rc[r], r);
  }
  c.comm->group_end();
  ++c.collectives;
  if (!local.empty()) e.copy_tiles(local);
  if (!unpack.empty()) e.copy_tiles(unpack);
  e.release(mk);
}
}  // namespace

void transpose_into(Ctx& c, const DistMat& X, const DistMat& Y);

void mirror_lower(Ctx& c, const DistMat& X) {
  transpose_exchange(c, X, X, [](int64_t I, int64_t J) { return I >= J; }, true);
}

void transpose_into(Ctx& c, const DistMat& X, const DistMat& Y) {
  transpose_exchange(c, X, Y, [](int64_t, int64_t) { return true; }, false);
}

void axpby_identity(Ctx& c, const DistMat* X, double a, const DistMat& Y, double b, double d) {
  Engine& e = *c.eng;
  if (Y.lr > 0 && Y.lc > 0) e.axpby(X ? X->a : nullptr, X ? X->ld : 0, Y.a, Y.ld, Y.lr, Y.lc, a, b);
  if (d != 0.0)
    for (int64_t I = 0; I < std::min(Y.mt(), Y.nt()); ++I)
      if (Y.owns_row(I) && Y.owns_col(I))
        e.add_diag(Y.tile(I, I), Y.ld, std::min(Y.tile_rows(I), Y.tile_cols(I)), d);
}

void stats(Ctx& c, const DistMat& X, bool want_asym, double out[3]) {
  Engine& e = *c.eng;
  double loc[3] = {0, 0, 0};  // sum of squares, max |x|, non-finite count
  if (X.lr > 0 && X.lc > 0) e.stats(X.a, X.ld, X.lr, X.lc, loc, false);
  double asym = 0.0;
  if (want_asym) {
    // max |x_ij - x_ji| through a distributed transpose
    const EMark mk = e.mark();
    DistMat T = make_dist(e, c.g, X.n, X.m);
    transpose_into(c, X, T);
    if (X.lr > 0 && X.lc > 0) {
      e.axpby(X.a, X.ld, T.a, T.ld, X.lr, X.lc, 1.0, -1.0);
      double t3[3];
      e.stats(T.a, T.ld, X.lr, X.lc, t3, false);
      asym = t3[1];
    }
    e.release(mk);
  }
  const EMark mk = e.mark();
  double* buf = e.alloc_vec(4);
  double h[4] = {loc[0], loc[2], asym, 0.0};
  e.from_host(h, 4, 4, 1, buf, 4);
  c.comm->allreduce(buf, 2, RedOp::Sum, Team::World);
  c.comm->allreduce(buf + 2, 1, RedOp::Max, Team::World);
  c.collectives += 2;
  e.to_host(buf, 4, 4, 1, h, 4);
  e.release(mk);
  out[0] = h[0];  // ||X||_F^2
  out[1] = h[2];  // max |x_ij - x_ji|
  out[2] = h[1];  // non-finite entries
}

// ------------------------------------------------------------------ gather / scatter
void gather(Ctx& c, const DistMat& X, double* dst, int64_t ldd, int root) {
  const Grid& g = c.g;
  Engine& e = *c.eng;
  const int me = g.world_rank(g.p, g.q);
  const int64_t nb = g.nb;
  const EMark mk = e.mark();
  std::vector<TileCopy> place;
  if (root < 0) {
    // everyone gets everything: the full view broadcast, then placement
    View v = whole(X);
    FullView f;
    fetch_full(c, v, f);
    for (int64_t I = 0; I < X.mt(); ++I)
      for (int64_t J = 0; J < X.nt(); ++J) {
        int64_t lds;
        const double* s = f.tile(I, J, &lds);
        place.push_back(TileCopy{s, lds, dst + I * nb + J * nb * ldd, ldd, (int32_t)X.tile_rows(I),
                                 (int32_t)X.tile_cols(J), 0});
      }
    e.copy_tiles(place);
    e.release(mk);
    return;
  }
  // to the root: one send per rank of its whole local array
  std::vector<double*> rb(g.P * g.Q, nullptr);
  double* sb = nullptr;
  if (me != root && X.lr > 0 && X.lc > 0) {
    sb = e.alloc_vec((size_t)(X.lr * X.lc));
    e.copy_tiles({TileCopy{X.a, X.ld, sb, X.lr, (int32_t)X.lr, (int32_t)X.lc, 0}});
  }
  c.comm->group_begin();
  if (sb) c.comm->send(sb, (size_t)(X.lr * X.lc), root);
  if (me == root)
    for (int pr = 0; pr < g.P; ++pr)
      for (int pc = 0; pc < g.Q; ++pc) {
        const int r = g.world_rank(pr, pc);
        const int64_t lr = numroc(X.m, nb, pr, g.P), lc = numroc(X.n, nb, pc, g.Q);
        if (r == root || lr == 0 || lc == 0) continue;
        rb[r] = e.alloc_vec((size_t)(lr * lc));
        c.comm->recv(rb[r], (size_t)(lr * lc), r);
      }
  c.comm->group_end();
  ++c.collectives;
  if (me == root) {
    for (int64_t I = 0; I < X.mt(); ++I)
      for (int64_t J = 0; J < X.nt(); ++J) {
        const int pr = (int)(I % g.P), pc = (int)(J % g.Q);
        const int r = g.world_rank(pr, pc);
        const int64_t lr = numroc(X.m, nb, pr, g.P);
        const double* src;
        int64_t lds;
        if (r == root) {
          src = X.tile(I, J);
          lds = X.ld;
        } else {
          src = rb[r] + (I / g.P) * nb + (J / g.Q) * nb * lr;
          lds = lr;
        }
        place.push_back(TileCopy{src, lds, dst + I * nb + J * nb * ldd, ldd, (int32_t)X.tile_rows(I),
                                 (int32_t)X.tile_cols(J), 0});
      }
    e.copy_tiles(place);
  }
  e.release(mk);
}

void scatter_from_full(Ctx& c, const double* full, int64_t ldf, bool host, const DistMat& X) {
  Engine& e = *c.eng;
  const int64_t nb = c.g.nb;
  if (host) {
    for (int64_t I = 0; I < X.mt(); ++I) {
      if (!X.owns_row(I)) continue;
      for (int64_t J = 0; J < X.nt(); ++J) {
        if (!X.owns_col(J)) continue;
        e.from_host(full + I * nb + J * nb * ldf, ldf, X.tile_rows(I), X.tile_cols(J), X.tile(I, J), X.ld);
      }
    }
    return;
  }
  std::vector<TileCopy> tc;
  for (int64_t I = 0; I < X.mt(); ++I) {
    if (!X.owns_row(I)) continue;
    for (int64_t J = 0; J < X.nt(); ++J) {
      if (!X.owns_col(J)) continue;
      tc.push_back(TileCopy{full + I * nb + J * nb * ldf, ldf, X.tile(I, J), X.ld, (int32_t)X.tile_rows(I),
                            (int32_t)X.tile_cols(J), 0});
    }
  }
  if (!tc.empty()) e.copy_tiles(tc);
}

// ------------------------------------------------------------------ Cholesky-and-inverse
namespace {
struct CholWork {
  const DistMat *Z, *Winv;
  DistMat W12, T1;
  bool failed = false;
};

void chol_rec(Ctx& c, CholWork& w, int64_t t0, int64_t T) {
  const DistMat& Z = *w.Z;
  const DistMat& Wi = *w.Winv;
  if (T == 1) {
    // leaf: one tile on its owner, the single-GPU Cholesky-and-inverse
    if (Z.owns_row(t0) && Z.owns_col(t0)) {
      try {
        c.eng->chol_inv(Z.tile(t0, t0), Z.ld, Z.tile_rows(t0), Wi.tile(t0, t0), Wi.ld);
      } catch (const NotPositiveDefinite&) {
        w.failed = true;
      }
    }
    return;
  }
  const int64_t h = (T + 1) / 2, h2 = T - h;
  chol_rec(c, w, t0, h);
  // W12 = W11^-T Z12 = Winv11^T Z21^T   (Winv11^T lower)
  Structure s1;
  s1.a_lower = true;
  pgemm(c, true, true, 1.0, View{&Wi, t0, t0, h, h}, View{&Z, t0 + h, t0, h2, h}, 0.0,
        View{&w.W12, t0, t0 + h, h, h2}, s1);
  // Z22 -= W12^T W12 (lower tiles)
  Structure s2;
  s2.c_lower = true;
  const View w12{&w.W12, t0, t0 + h, h, h2};
  pgemm(c, true, false, -1.0, w12, w12, 1.0, View{&Z, t0 + h, t0 + h, h2, h2}, s2);
  chol_rec(c, w, t0 + h, h2);
  // Winv12 = -Winv11 W12 Winv22
  Structure s3;
  s3.b_upper = true;
  pgemm(c, false, false, 1.0, w12, View{&Wi, t0 + h, t0 + h, h2, h2}, 0.0, View{&w.T1, t0, t0 + h, h, h2},
        s3);
  Structure s4;
  s4.a_upper = true;
  pgemm(c, false, false, -1.0, View{&Wi, t0, t0, h, h}, View{&w.T1, t0, t0 + h, h, h2}, 0.0,
        View{&Wi, t0, t0 + h, h, h2}, s4);
}
}  // namespace

void chol_inv(Ctx& c, const DistMat& Z, const DistMat& Winv) {
  Engine& e = *c.eng;
  const EMark mk = e.mark();
  CholWork w;
  w.Z = &Z;
  w.Winv = &Winv;
  w.W12 = make_dist(e, c.g, Z.m, Z.n);
  w.T1 = make_dist(e, c.g, Z.m, Z.n);
  if (Winv.lr > 0 && Winv.lc > 0) e.fill(Winv.a, Winv.ld, Winv.lr, Winv.lc, 0.0);
  chol_rec(c, w, 0, Z.mt());
  // every rank learns whether any leaf failed (no rank throws alone)
  double* f = e.alloc_vec(1);
  double hf = w.failed ? 1.0 : 0.0;
  e.from_host(&hf, 1, 1, 1, f, 1);
  c.comm->allreduce(f, 1, RedOp::Max, Team::World);
  ++c.collectives;
  e.to_host(f, 1, 1, 1, &hf, 1);
  e.release(mk);
  if (hf != 0.0) throw NotPositiveDefinite("cholesky: pivot is not positive");
}

// ------------------------------------------------------------------ QR
void pgeqrf(Ctx& c, const DistMat& X, QrDist& qr) {
  const Grid& g = c.g;
  Engine& e = *c.eng;
  const int64_t nb = g.nb, m = X.m, n = X.n;
  if (m < n) throw InvalidArgument("pgeqrf: requires rows >= cols");
  qr.m = m;
  qr.n = n;
  qr.rdiag.clear();
  qr.V.clear();
  qr.T.clear();
  int64_t vld;
  double* Vall = e.alloc(std::max<int64_t>(X.lr, 1), std::max<int64_t>(n, 1), &vld);  // my rows, all panels
  qr.vld = vld;
  const int64_t NT = X.nt();
  for (int64_t J = 0; J < NT; ++J) {
    const int64_t w = X.tile_cols(J);
    const int64_t mrows = m - J * nb;
    int64_t ldt;
    double* T = e.alloc(nb, nb, &ldt);
    (void)ldt;
    qr.T.push_back(T);
    qr.V.push_back(Vall + J * nb * vld);
    const EMark mk = e.mark();
    // the panel (tiles I >= J of column J), replicated on every rank
    int64_t ldp;
    double* Pn = e.alloc(mrows, w, &ldp);
    const int pc = (int)(J % g.Q);
    std::vector<double*> stg(g.P, nullptr);
    std::vector<LRange> rr(g.P);
    for (int pr = 0; pr < g.P; ++pr) {
      rr[pr] = lrange(J, X.mt() - J, pr, g.P, nb, m);
      if (rr[pr].empty()) continue;
      stg[pr] = e.alloc_vec((size_t)(rr[pr].len * w));
      if (pr == g.p && pc == g.q)
        e.copy_tiles({TileCopy{X.a + rr[pr].l0 + X.lcol(J) * X.ld, X.ld, stg[pr], rr[pr].len,
                               (int32_t)rr[pr].len, (int32_t)w, 0}});
    }
    c.comm->group_begin();
    for (int pr = 0; pr < g.P; ++pr)
      if (stg[pr]) c.comm->bcast(stg[pr], (size_t)(rr[pr].len * w), g.world_rank(pr, pc), Team::World);
    c.comm->group_end();
    ++c.collectives;
    std::vector<TileCopy> place;
    for (int64_t I = J; I < X.mt(); ++I) {
      const int pr = (int)(I % g.P);
      place.push_back(TileCopy{stg[pr] + rr[pr].off(I, g.P, nb), rr[pr].len, Pn + (I - J) * nb, ldp,
                               (int32_t)X.tile_rows(I), (int32_t)w, 0});
    }
    e.copy_tiles(place);
    std::vector<double> rd;
    e.qr_panel(Pn, ldp, mrows, w, T, nb, rd);  // identical on every rank
    qr.rdiag.insert(qr.rdiag.end(), rd.begin(), rd.end());
    // my rows of V (tiles I >= J) into the per-rank store; zero above
    const LRange mine = lrange(J, X.mt() - J, g.p, g.P, nb, m);
    double* Vj = qr.V.back();
    if (X.lr > 0) e.fill(Vj, vld, X.lr, w, 0.0);
    std::vector<TileCopy> vs;
    for (int64_t I = mine.first; I >= 0 && I <= mine.last; I += g.P)
      vs.push_back(TileCopy{Pn + (I - J) * nb, ldp, Vj + X.lrow(I), vld, (int32_t)X.tile_rows(I), (int32_t)w, 0});
    if (!vs.empty()) e.copy_tiles(vs);
    // trailing update of my columns J' > J:  C -= V T^T (V^T C)
    const LRange cols = lrange(J + 1, NT - J - 1, g.q, g.Q, nb, n);
    if (!cols.empty()) {
      const int64_t r0 = mine.empty() ? X.lr : mine.l0;
      const int64_t rn = X.lr - r0;
      double* Cl = X.a + r0 + cols.l0 * X.ld;
      int64_t ldw;
      double* W = e.alloc(w, cols.len, &ldw);
      double* W2 = e.alloc(w, cols.len, &ldw);
      if (rn > 0) e.gemm(true, false, w, cols.len, rn, 1.0, Vj + r0, vld, Cl, X.ld, 0.0, W, ldw);
      else e.fill(W, ldw, w, cols.len, 0.0);
      // sum over the process column (contiguous: ldw-padded rows included)
      c.comm->allreduce(W, (size_t)(ldw * cols.len), RedOp::Sum, Team::Col);
      ++c.collectives;
      e.gemm(true, false, w, cols.len, w, 1.0, T, nb, W, ldw, 0.0, W2, ldw);
      if (rn > 0) e.gemm(false, false, rn, cols.len, w, -1.0, Vj + r0, vld, W2, ldw, 1.0, Cl, X.ld);
    }
    // (ranks without trailing columns: their whole process column has none, so
    // the column team's reduction above is skipped consistently)
    e.release(mk);
  }
}

void porgqr_cols(Ctx& c, const QrDist& qr, int64_t c0, const DistMat& Q2) {
  const Grid& g = c.g;
  Engine& e = *c.eng;
  const int64_t nb = g.nb, m = qr.m;
  // E = [0; I] rows c0 .. c0 + ell - 1
  if (Q2.lr > 0 && Q2.lc > 0) e.fill(Q2.a, Q2.ld, Q2.lr, Q2.lc, 0.0);
  for (int64_t J2 = 0; J2 < Q2.nt(); ++J2) {
    if (!Q2.owns_col(J2)) continue;
    const int64_t j0 = J2 * nb, j1 = j0 + Q2.tile_cols(J2);
    for (int64_t j = j0; j < j1;) {
      const int64_t r = c0 + j, I = r / nb;
      const int64_t run = std::min(j1 - j, (I + 1) * nb - r);
      if (Q2.owns_row(I))
        e.add_diag(Q2.a + Q2.lrow(I) + (r - I * nb) + (Q2.lcol(J2) + (j - j0)) * Q2.ld, Q2.ld, run, 1.0);
      j += run;
    }
  }
  const int64_t NP = (int64_t)qr.V.size();
  for (int64_t J = NP - 1; J >= 0; --J) {
    const int64_t w = std::min<int64_t>(nb, qr.n - J * nb);
    const LRange mine = lrange(J, (m + nb - 1) / nb - J, g.p, g.P, nb, m);
    const int64_t r0 = mine.empty() ? Q2.lr : mine.l0;
    const int64_t rn = Q2.lr - r0;
    if (Q2.lc == 0) continue;  // the whole process column has no Q2 columns
    const EMark mk = e.mark();
    int64_t ldw;
    double* W = e.alloc(w, Q2.lc, &ldw);
    double* W2 = e.alloc(w, Q2.lc, &ldw);
    double* Cl = Q2.a + r0;
    if (rn > 0) e.gemm(true, false, w, Q2.lc, rn, 1.0, qr.V[J] + r0, qr.vld, Cl, Q2.ld, 0.0, W, ldw);
    else e.fill(W, ldw, w, Q2.lc, 0.0);
    c.comm->allreduce(W, (size_t)(ldw * Q2.lc), RedOp::Sum, Team::Col);
    ++c.collectives;
    e.gemm(false, false, w, Q2.lc, w, 1.0, qr.T[J], nb, W, ldw, 0.0, W2, ldw);
    if (rn > 0) e.gemm(false, false, rn, Q2.lc, w, -1.0, qr.V[J] + r0, qr.vld, W2, ldw, 1.0, Cl, Q2.ld);
    e.release(mk);
  }
}

// ------------------------------------------------------------------ replicated-vector GEMV
void pgemv(Ctx& c, const DistMat& A, bool trans, const double* x, double* y) {
  const Grid& g = c.g;
  Engine& e = *c.eng;
  const int64_t nb = g.nb;
  const EMark mk = e.mark();
  // x entries of my local columns (rows for trans), y partial of my rows (cols)
  const int64_t nin = trans ? A.lr : A.lc, nout = trans ? A.lc : A.lr;
  const int64_t tin = trans ? A.mt() : A.nt(), tout = trans ? A.nt() : A.mt();
  const int np_in = trans ? g.P : g.Q, ip_in = trans ? g.p : g.q;
  const int np_out = trans ? g.Q : g.P;
  double* xl = e.alloc_vec((size_t)std::max<int64_t>(nin, 1));
  double* yl = e.alloc_vec((size_t)std::max<int64_t>(nout, 1));
  std::vector<TileCopy> tc;
  for (int64_t t = ip_in; t < tin; t += np_in) {
    const int64_t len = trans ? A.tile_rows(t) : A.tile_cols(t);
    tc.push_back(TileCopy{x + t * nb, 1, xl + (t / np_in) * nb, 1, (int32_t)len, 1, 0});
  }
  if (!tc.empty()) e.copy_tiles(tc);
  if (nout > 0) {
    if (nin > 0) e.gemm(trans, false, nout, 1, nin, 1.0, A.a, A.ld, xl, std::max<int64_t>(nin, 1), 0.0, yl,
                        std::max<int64_t>(nout, 1));
    else e.fill(yl, std::max<int64_t>(nout, 1), nout, 1, 0.0);
  }
  if (nout > 0) c.comm->allreduce(yl, (size_t)nout, RedOp::Sum, trans ? Team::Col : Team::Row);
  // replicate: one world broadcast per process row (column) of its piece
  std::vector<double*> stg(np_out, nullptr);
  std::vector<int64_t> len(np_out);
  const int64_t total = trans ? A.n : A.m;
  for (int r = 0; r < np_out; ++r) {
    len[r] = numroc(total, nb, r, np_out);
    if (len[r] == 0) continue;
    const bool mine = trans ? (r == g.q) : (r == g.p);
    stg[r] = mine ? yl : e.alloc_vec((size_t)len[r]);
  }
  c.comm->group_begin();
  for (int r = 0; r < np_out; ++r) {
    if (!stg[r]) continue;
    const int root = trans ? g.world_rank(0, r) : g.world_rank(r, 0);
    c.comm->bcast(stg[r], (size_t)len[r], root, Team::World);
  }
  c.comm->group_end();
  c.collectives += 2;
  tc.clear();
  for (int64_t t = 0; t < tout; ++t) {
    const int r = (int)(t % np_out);
    const int64_t l = trans ? A.tile_cols(t) : A.tile_rows(t);
    tc.push_back(TileCopy{stg[r] + (t / np_out) * nb, 1, y + t * nb, 1, (int32_t)l, 1, 0});
  }
  e.copy_tiles(tc);
  e.release(mk);
}

}  // namespace dist
}  // namespace qdwhg
