// dist::Engine on one B200: the rank's local compute through libqdwhg's own
// sm_100a kernels (DMMA GEMM engine, recursive Cholesky-and-inverse, register
// panel QR, tridiagonal / polar-based Rayleigh-Ritz solvers, tiles.cu copies).
// Workspace comes from the rank handle's arena (stack discipline); every call is
// asynchronous on the handle's stream except the host reads (dot, stats, QR
// diagonal, eigen/singular values).
#include <cmath>
#include <cstdio>

#include "../drivers.hpp"
#include "../internal.hpp"
#include "dist.hpp"

namespace qdwhg {
namespace dist {

namespace {

DMat view(const double* p, int64_t ld, int64_t rows, int64_t cols) {
  DMat d;
  d.base = const_cast<double*>(p);
  // a single column's stride is never stepped: pad it so TMA sees a 16-byte
  // multiple (vectors are packed with ld = length)
  d.ld = cols == 1 ? std::max<int64_t>(ld, round_ld(rows)) : ld;
  d.rows = rows;
  d.cols = cols;
  return d;
}

class CudaEngine : public Engine {
 public:
  explicit CudaEngine(qdwhg::Ctx& ctx) : c_(ctx) {}

  double* alloc(int64_t rows, int64_t cols, int64_t* ld) override {
    DMat d = c_.arena->alloc(std::max<int64_t>(rows, 1), std::max<int64_t>(cols, 1));
    *ld = d.ld;
    if (poison()) qdwhg::fill(c_, view(d.base, d.ld, d.ld, d.cols), NAN, 0.0);
    return d.base;
  }
  double* alloc_vec(size_t count) override {
    double* p = static_cast<double*>(c_.arena->alloc_bytes(sizeof(double) * std::max<size_t>(count, 1)));
    if (poison()) qdwhg::fill(c_, view(p, (int64_t)count, (int64_t)count, 1), NAN, 0.0);
    return p;
  }
  // QDWHG_DIST_POISON: every workspace allocation starts as NaN (debug: a read of
  // memory the driver never wrote shows up as a non-finite result)
  static bool poison() {
    static const bool on = getenv("QDWHG_DIST_POISON") != nullptr;
    return on;
  }
  EMark mark() override {
    const Arena::Mark m = c_.arena->mark();
    return EMark{m.chunk, m.off};
  }
  void release(EMark m) override { c_.arena->release_to(Arena::Mark{m.a, m.b}); }

  void gemm(bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
            const double* B, int64_t ldb, double beta, double* C, int64_t ldc) override {
    if (m <= 0 || n <= 0) return;
    if (k <= 0) {
      if (beta == 0.0) fill(C, ldc, m, n, 0.0);
      else qdwhg::axpby(c_, nullptr, 0, C, ldc, m, n, 0.0, beta);
      return;
    }
    const DMat Av = ta ? view(A, lda, k, m) : view(A, lda, m, k);
    const DMat Bv = tb ? view(B, ldb, n, k) : view(B, ldb, k, n);
    static const bool verify = getenv("QDWHG_DIST_VERIFY") != nullptr;
    std::vector<double> ha, hb, hc;
    if (verify) {
      ha = host(A, lda, ta ? k : m, ta ? m : k);
      hb = host(B, ldb, tb ? n : k, tb ? k : n);
      hc = host(C, ldc, m, n);
    }
    qdwhg::gemm(c_, ta ? Op::T : Op::N, tb ? Op::T : Op::N, alpha, Av, Bv, beta, view(C, ldc, m, n));
    if (verify) {
      const std::vector<double> got = host(C, ldc, m, n);
      double err = 0, scale = 1e-300;
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
          double acc = 0;
          for (int64_t p = 0; p < k; ++p)
            acc += (ta ? ha[p + i * k] : ha[i + p * m]) * (tb ? hb[j + p * n] : hb[p + j * k]);
          const double want = alpha * acc + (beta == 0.0 ? 0.0 : beta * hc[i + j * m]);
          err = std::max(err, std::abs(got[i + j * m] - want));
          scale = std::max(scale, std::abs(want));
        }
      if (!(err <= 1e-11 * scale * std::max<int64_t>(k, 1)))
        fprintf(stderr, "DIST_VERIFY gemm mismatch ta=%d tb=%d m=%ld n=%ld k=%ld lda=%ld ldb=%ld ldc=%ld "
                        "alpha=%g beta=%g A=%p B=%p C=%p err=%.3e scale=%.3e\n",
                (int)ta, (int)tb, (long)m, (long)n, (long)k, (long)lda, (long)ldb, (long)ldc, alpha, beta,
                (const void*)A, (const void*)B, (void*)C, err, scale);
    }
  }
  std::vector<double> host(const double* p, int64_t ld, int64_t rows, int64_t cols) {
    std::vector<double> h((size_t)(rows * cols));
    QDWHG_CUDA(cudaMemcpy2DAsync(h.data(), rows * 8, p, ld * 8, rows * 8, cols, cudaMemcpyDefault, c_.stream));
    QDWHG_CUDA(cudaStreamSynchronize(c_.stream));
    return h;
  }
  void copy_tiles(const std::vector<TileCopy>& list) override {
    std::vector<TileDesc> d;
    d.reserve(list.size());
    for (const TileCopy& t : list)
      if (t.rows > 0 && t.cols > 0) d.push_back(TileDesc{t.src, t.lds, t.dst, t.ldd, t.rows, t.cols, t.trans});
    if (!d.empty()) qdwhg::copy_tiles(c_, d);
  }
  void axpby(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t rows, int64_t cols, double a,
             double b) override {
    qdwhg::axpby(c_, X, ldx, Y, ldy, rows, cols, a, b);
  }
  void fill(double* Y, int64_t ldy, int64_t rows, int64_t cols, double v) override {
    if (rows > 0 && cols > 0) qdwhg::fill(c_, view(Y, ldy, rows, cols), v, 0.0);
  }
  void add_diag(double* Y, int64_t ldy, int64_t len, double v) override { qdwhg::add_diag(c_, Y, ldy, len, v); }
  void mirror_lower(double* Y, int64_t ldy, int64_t n) override {
    if (n > 0) mirror_lower_to_upper(c_, view(Y, ldy, n, n));
  }
  void gaussian(double* Y, int64_t ldy, int64_t rows, int64_t cols, uint64_t seed, int64_t gr0, int64_t gc0,
                int64_t gm) override {
    gaussian_fill_at(c_, Y, ldy, rows, cols, seed, gr0, gc0, gm);
  }
  void stats(const double* X, int64_t ldx, int64_t rows, int64_t cols, double out[3], bool) override {
    const MatStats st = mat_stats(c_, view(X, ldx, rows, cols), false);
    out[0] = st.fro2;
    out[1] = st.maxabs;
    out[2] = st.nonfinite;
  }
  double dot(const double* x, const double* y, int64_t n) override {
    double* d = c_.dscratch + 64;
    qdwhg::gemm(c_, Op::T, Op::N, 1.0, view(x, n, n, 1), view(y, n, n, 1), 0.0, view(d, 1, 1, 1));
    QDWHG_CUDA(cudaMemcpyAsync(c_.hscratch + 64, d, sizeof(double), cudaMemcpyDeviceToHost, c_.stream));
    QDWHG_CUDA(cudaStreamSynchronize(c_.stream));
    return c_.hscratch[64];
  }
  void to_host(const double* src, int64_t lds, int64_t rows, int64_t cols, double* h, int64_t ldh) override {
    if (rows <= 0 || cols <= 0) return;
    QDWHG_CUDA(cudaMemcpy2DAsync(h, ldh * 8, src, lds * 8, rows * 8, cols, cudaMemcpyDefault, c_.stream));
    QDWHG_CUDA(cudaStreamSynchronize(c_.stream));
  }
  void from_host(const double* h, int64_t ldh, int64_t rows, int64_t cols, double* dst, int64_t ldd) override {
    if (rows <= 0 || cols <= 0) return;
    QDWHG_CUDA(cudaMemcpy2DAsync(dst, ldd * 8, h, ldh * 8, rows * 8, cols, cudaMemcpyDefault, c_.stream));
    // pageable sources are staged before the call returns; pinned ones must stay
    // valid until the copy runs: callers pass host vectors that outlive the sync
    // of the next host read, or pinned buffers they keep
    QDWHG_CUDA(cudaStreamSynchronize(c_.stream));
  }
  void chol_inv(const double* Z, int64_t ldz, int64_t n, double* Winv, int64_t ldw) override {
    potrf_upper_and_inverse(c_, view(Z, ldz, n, n), view(Winv, ldw, n, n), false, false);
  }
  void qr_panel(double* Pn, int64_t ldp, int64_t m, int64_t w, double* T, int64_t ldt,
                std::vector<double>& rdiag) override {
    const bool det = c_.deterministic;
    c_.deterministic = true;  // every rank factors the same panel: identical bits
    const Arena::Mark mk = c_.arena->mark();
    try {
      const DMat P = view(Pn, ldp, m, w);
      QrWork qw;
      geqrf(c_, P, qw);
      diag_to_host(c_, P, rdiag);
      for (double& x : rdiag) x = std::abs(x);
      copy(c_, qw.V.sub(0, 0, m, w), P);
      zero_strict_upper(c_, P);  // explicit zeros above the unit diagonal in every column
      // compact-WY T of the whole panel by merging the outer-block T's:
      //   T = [T1, -T1 (V1^T V2) T2; 0, T2]
      const int64_t nbo = qw.nb;
      const DMat Tv = view(T, ldt, w, w);
      fill(T, ldt, w, w, 0.0);
      for (int64_t b0 = 0; b0 < w; b0 += nbo) {
        const int64_t bs = std::min<int64_t>(nbo, w - b0);
        copy(c_, qw.T.sub(0, b0, bs, bs), Tv.sub(b0, b0, bs, bs));
        if (b0 == 0) continue;
        DMat G = c_.arena->alloc(b0, bs), X1 = c_.arena->alloc(b0, bs);
        qdwhg::gemm(c_, Op::T, Op::N, 1.0, P.sub(0, 0, m, b0), P.sub(0, b0, m, bs), 0.0, G);
        qdwhg::gemm(c_, Op::N, Op::N, 1.0, Tv.sub(0, 0, b0, b0), G, 0.0, X1);
        qdwhg::gemm(c_, Op::N, Op::N, -1.0, X1, Tv.sub(b0, b0, bs, bs), 0.0, Tv.sub(0, b0, b0, bs));
      }
    } catch (...) {
      c_.deterministic = det;
      c_.arena->release_to(mk);
      throw;
    }
    c_.deterministic = det;
    c_.arena->release_to(mk);
  }
  int64_t syev_range(double* S, int64_t lds, int64_t n, std::vector<double>& vals, double* V, int64_t ldv,
                     double vlo, double vhi, int64_t* sel0) override {
    return qdwhg::syev_range(c_, view(S, lds, n, n), vals, view(V, ldv, n, n), vlo, vhi, sel0);
  }
  int64_t svd_polar(const double* A, int64_t lda, int64_t m, int64_t n, double* U, int64_t ldu,
                    std::vector<double>& sigma, double* V, int64_t ldv, double cut) override {
    return qdwhg::svd_polar(c_, view(A, lda, m, n), view(U, ldu, m, n), sigma, view(V, ldv, n, n), cut);
  }
  void tridiag_lowest(const std::vector<double>& d, const std::vector<double>& e, double* theta,
                      double* zlast) override {
    qdwhg::tridiag_lowest(c_, d, e, theta, zlast);
  }
  void sync() override { QDWHG_CUDA(cudaStreamSynchronize(c_.stream)); }
  void* stream() override { return c_.stream; }

 private:
  qdwhg::Ctx& c_;
};

}  // namespace

Engine* make_cuda_engine(qdwhg::Ctx& ctx) { return new CudaEngine(ctx); }

}  // namespace dist
}  // namespace qdwhg
