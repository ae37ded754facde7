// TEST INFRASTRUCTURE ONLY — the distributed QDWHpartial orchestration
// (paper_2104_14186_b200/csrc/dist/*.cpp, compiled unchanged) on a plain host
// Engine with emulated ranks (threads + the loopback communicator), so the
// CPU test suite can run the 2D block-cyclic algorithms at world size 2 and 4
// without a GPU.  Never linked into libqdwhg and never on the product path:
// the product's Engine is engine_cuda.cpp over the sm_100a kernels.
//
// Built by tests/cpp/Makefile into tests/cpp/libqdwhg_disthost.so; driven from
// tests/test_dist_host.py through ctypes (dh_* entry points below).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../paper_2104_14186_b200/csrc/dist/dist.hpp"

using namespace qdwhg;
using namespace qdwhg::dist;

namespace {

int64_t round_ld(int64_t r) { return ((std::max<int64_t>(r, 1) + 31) / 32) * 32; }

class HostEngine : public Engine {
 public:
  double* alloc(int64_t rows, int64_t cols, int64_t* ld) override {
    *ld = round_ld(rows);
    return push((size_t)(*ld) * (size_t)std::max<int64_t>(cols, 1));
  }
  double* alloc_vec(size_t count) override { return push(std::max<size_t>(count, 1)); }
  EMark mark() override { return EMark{bufs_.size(), 0}; }
  void release(EMark m) override { bufs_.resize(m.a); }

  void gemm(bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
            const double* B, int64_t ldb, double beta, double* C, int64_t ldc) override {
    std::vector<double> acc((size_t)m);
    for (int64_t j = 0; j < n; ++j) {
      std::fill(acc.begin(), acc.end(), 0.0);
      for (int64_t p = 0; p < k; ++p) {
        const double b = tb ? B[j + p * ldb] : B[p + j * ldb];
        if (b == 0.0) continue;
        for (int64_t i = 0; i < m; ++i) acc[i] += (ta ? A[p + i * lda] : A[i + p * lda]) * b;
      }
      for (int64_t i = 0; i < m; ++i) {
        double& c = C[i + j * ldc];
        c = beta == 0.0 ? alpha * acc[i] : alpha * acc[i] + beta * c;
      }
    }
  }
  void copy_tiles(const std::vector<TileCopy>& list) override {
    for (const TileCopy& t : list)
      for (int64_t j = 0; j < t.cols; ++j)
        for (int64_t i = 0; i < t.rows; ++i) {
          const double v = t.src[i + j * t.lds];
          if (t.trans) t.dst[j + i * t.ldd] = v;
          else t.dst[i + j * t.ldd] = v;
        }
  }
  void axpby(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t rows, int64_t cols, double a,
             double b) override {
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < rows; ++i) {
        const double xv = X ? a * X[i + j * ldx] : 0.0;
        double& y = Y[i + j * ldy];
        y = b == 0.0 ? xv : b * y + xv;
      }
  }
  void fill(double* Y, int64_t ldy, int64_t rows, int64_t cols, double v) override {
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < rows; ++i) Y[i + j * ldy] = v;
  }
  void add_diag(double* Y, int64_t ldy, int64_t len, double v) override {
    for (int64_t i = 0; i < len; ++i) Y[i + i * ldy] += v;
  }
  void mirror_lower(double* Y, int64_t ldy, int64_t n) override {
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < j; ++i) Y[i + j * ldy] = Y[j + i * ldy];
  }
  void gaussian(double* Y, int64_t ldy, int64_t rows, int64_t cols, uint64_t seed, int64_t gr0, int64_t gc0,
                int64_t gm) override {
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < rows; ++i) {
        const uint64_t g = (uint64_t)((gr0 + i) + (gc0 + j) * gm);
        auto h = [&](uint64_t c) {
          uint64_t z = seed + (c + 1) * 0x9E3779B97F4A7C15ull;
          z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
          z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
          return z ^ (z >> 31);
        };
        const double u1 = (double)((h(2 * g) >> 11) + 1) * 0x1.0p-53;
        const double u2 = (double)((h(2 * g + 1) >> 11) + 1) * 0x1.0p-53;
        Y[i + j * ldy] = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
      }
  }
  void stats(const double* X, int64_t ldx, int64_t rows, int64_t cols, double out[3], bool) override {
    double s = 0, mx = 0, nf = 0;
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < rows; ++i) {
        const double v = X[i + j * ldx];
        if (!std::isfinite(v)) {
          nf += 1;
          continue;
        }
        s += v * v;
        mx = std::max(mx, std::abs(v));
      }
    out[0] = s;
    out[1] = mx;
    out[2] = nf;
  }
  double dot(const double* x, const double* y, int64_t n) override {
    double s = 0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
  }
  void to_host(const double* src, int64_t lds, int64_t rows, int64_t cols, double* h, int64_t ldh) override {
    for (int64_t j = 0; j < cols; ++j) std::memcpy(h + j * ldh, src + j * lds, sizeof(double) * rows);
  }
  void from_host(const double* h, int64_t ldh, int64_t rows, int64_t cols, double* dst, int64_t ldd) override {
    for (int64_t j = 0; j < cols; ++j) std::memcpy(dst + j * ldd, h + j * ldh, sizeof(double) * rows);
  }
  void chol_inv(const double* Z, int64_t ldz, int64_t n, double* Winv, int64_t ldw) override {
    // L (lower) with Z = L L^T from Z's lower triangle; W = L^T, W^-1 = L^-T
    std::vector<double> L((size_t)n * n, 0.0), Li((size_t)n * n, 0.0);
    for (int64_t j = 0; j < n; ++j) {
      double d = Z[j + j * ldz];
      for (int64_t k = 0; k < j; ++k) d -= L[j + k * n] * L[j + k * n];
      if (!(d > 0.0)) throw NotPositiveDefinite("cholesky: pivot is not positive");
      L[j + j * n] = std::sqrt(d);
      for (int64_t i = j + 1; i < n; ++i) {
        double s = Z[i + j * ldz];
        for (int64_t k = 0; k < j; ++k) s -= L[i + k * n] * L[j + k * n];
        L[i + j * n] = s / L[j + j * n];
      }
    }
    for (int64_t j = 0; j < n; ++j) {  // L^-1 column j
      Li[j + j * n] = 1.0 / L[j + j * n];
      for (int64_t i = j + 1; i < n; ++i) {
        double s = 0.0;
        for (int64_t k = j; k < i; ++k) s += L[i + k * n] * Li[k + j * n];
        Li[i + j * n] = -s / L[i + i * n];
      }
    }
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) Winv[i + j * ldw] = i <= j ? Li[j + i * n] : 0.0;
  }
  void qr_panel(double* Pn, int64_t ldp, int64_t m, int64_t w, double* T, int64_t ldt,
                std::vector<double>& rdiag) override {
    // kernels.cpp:41-80 convention (v0 += sign ||x||, R_jj = -sign ||x||,
    // p = min(m - 1, w) reflectors), stored LAPACK-style: unit v, tau scaled
    const int64_t p = std::min<int64_t>(m - 1, w);
    std::vector<double> taus((size_t)w, 0.0);
    rdiag.assign((size_t)w, 0.0);
    for (int64_t j = 0; j < w; ++j) {
      if (j >= p) {
        rdiag[j] = std::abs(Pn[j + j * ldp]);
        for (int64_t i = 0; i < m; ++i) Pn[i + j * ldp] = i == j ? 1.0 : 0.0;
        continue;
      }
      double nx = 0.0;
      for (int64_t i = j; i < m; ++i) nx += Pn[i + j * ldp] * Pn[i + j * ldp];
      nx = std::sqrt(nx);
      if (nx > 0.0) {
        const double x0 = Pn[j + j * ldp];
        const double sign = x0 >= 0.0 ? 1.0 : -1.0;
        const double v0 = x0 + sign * nx;
        // unit-normalised v (v_j = 1), tau = 2 v0^2 / (v^T v)
        double vv = 1.0;
        for (int64_t i = j + 1; i < m; ++i) {
          Pn[i + j * ldp] /= v0;
          vv += Pn[i + j * ldp] * Pn[i + j * ldp];
        }
        const double tau = 2.0 / vv;
        taus[j] = tau;
        for (int64_t c = j + 1; c < w; ++c) {
          double s = Pn[j + c * ldp];
          for (int64_t i = j + 1; i < m; ++i) s += Pn[i + j * ldp] * Pn[i + c * ldp];
          s *= tau;
          Pn[j + c * ldp] -= s;
          for (int64_t i = j + 1; i < m; ++i) Pn[i + c * ldp] -= s * Pn[i + j * ldp];
        }
        rdiag[j] = nx;
      } else {
        for (int64_t i = j + 1; i < m; ++i) Pn[i + j * ldp] = 0.0;
        rdiag[j] = 0.0;
      }
      Pn[j + j * ldp] = 1.0;
      for (int64_t i = 0; i < j; ++i) Pn[i + j * ldp] = 0.0;
    }
    // T (forward, columnwise): T(0:j, j) = -tau_j T(0:j, 0:j) V(:, 0:j)^T v_j
    for (int64_t j = 0; j < w; ++j)
      for (int64_t i = 0; i < w; ++i) T[i + j * ldt] = 0.0;
    for (int64_t j = 0; j < w; ++j) {
      T[j + j * ldt] = taus[j];
      if (taus[j] == 0.0) continue;
      std::vector<double> g((size_t)j, 0.0);
      for (int64_t c = 0; c < j; ++c)
        for (int64_t i = 0; i < m; ++i) g[c] += Pn[i + c * ldp] * Pn[i + j * ldp];
      for (int64_t r = 0; r < j; ++r) {
        double s = 0.0;
        for (int64_t c = r; c < j; ++c) s += T[r + c * ldt] * g[c];
        T[r + j * ldt] = -taus[j] * s;
      }
    }
  }
  static void jacobi(std::vector<double>& S, int64_t n, std::vector<double>& V) {
    V.assign((size_t)n * n, 0.0);
    for (int64_t i = 0; i < n; ++i) V[i + i * n] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0.0, tot = 0.0;
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) {
          tot += S[i + j * n] * S[i + j * n];
          if (i != j) off += S[i + j * n] * S[i + j * n];
        }
      if (off <= 1e-30 * std::max(tot, 1e-300)) break;
      for (int64_t p = 0; p < n - 1; ++p)
        for (int64_t q = p + 1; q < n; ++q) {
          const double apq = S[p + q * n];
          if (apq == 0.0) continue;
          const double th = (S[q + q * n] - S[p + p * n]) / (2.0 * apq);
          const double t = (th >= 0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(th * th + 1.0));
          const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
          for (int64_t k = 0; k < n; ++k) {
            const double a = S[k + p * n], b = S[k + q * n];
            S[k + p * n] = c * a - s * b;
            S[k + q * n] = s * a + c * b;
          }
          for (int64_t k = 0; k < n; ++k) {
            const double a = S[p + k * n], b = S[q + k * n];
            S[p + k * n] = c * a - s * b;
            S[q + k * n] = s * a + c * b;
          }
          for (int64_t k = 0; k < n; ++k) {
            const double a = V[k + p * n], b = V[k + q * n];
            V[k + p * n] = c * a - s * b;
            V[k + q * n] = s * a + c * b;
          }
        }
    }
  }
  int64_t syev_range(double* S, int64_t lds, int64_t n, std::vector<double>& vals, double* V, int64_t ldv,
                     double vlo, double vhi, int64_t* sel0) override {
    std::vector<double> A((size_t)n * n), W;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) A[i + j * n] = S[i + j * lds];
    jacobi(A, n, W);
    std::vector<int64_t> order((size_t)n);
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return A[a + a * n] < A[b + b * n]; });
    vals.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) vals[i] = A[order[i] + order[i] * n];
    int64_t i0 = 0;
    while (i0 < n && !(vals[i0] > vlo)) ++i0;
    int64_t i1 = i0;
    while (i1 < n && vals[i1] < vhi) ++i1;
    for (int64_t c = i0; c < i1; ++c)
      for (int64_t r = 0; r < n; ++r) V[r + (c - i0) * ldv] = W[r + order[c] * n];
    *sel0 = i0;
    return i1 - i0;
  }
  int64_t svd_polar(const double* A, int64_t lda, int64_t m, int64_t n, double* U, int64_t ldu,
                    std::vector<double>& sigma, double* V, int64_t ldv, double cut) override {
    // eig(A^T A) on the host test engine: V, sigma = sqrt(eig), U = A V / sigma
    std::vector<double> G((size_t)n * n, 0.0), W;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t r = 0; r < m; ++r) s += A[r + i * lda] * A[r + j * lda];
        G[i + j * n] = s;
      }
    jacobi(G, n, W);
    std::vector<int64_t> order((size_t)n);
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return G[a + a * n] > G[b + b * n]; });
    sigma.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) sigma[i] = std::sqrt(std::max(0.0, G[order[i] + order[i] * n]));
    int64_t k = 0;
    while (k < n && sigma[k] > cut) ++k;
    for (int64_t c = 0; c < k; ++c) {
      for (int64_t r = 0; r < n; ++r) V[r + c * ldv] = W[r + order[c] * n];
      for (int64_t r = 0; r < m; ++r) {
        double s = 0.0;
        for (int64_t q = 0; q < n; ++q) s += A[r + q * lda] * V[q + c * ldv];
        U[r + c * ldu] = s / sigma[c];
      }
    }
    return k;
  }
  void tridiag_lowest(const std::vector<double>& d, const std::vector<double>& e, double* theta,
                      double* zlast) override {
    const int64_t n = (int64_t)d.size();
    std::vector<double> A((size_t)n * n, 0.0), W;
    for (int64_t i = 0; i < n; ++i) {
      A[i + i * n] = d[i];
      if (i + 1 < n) A[i + (i + 1) * n] = A[(i + 1) + i * n] = e[i];
    }
    jacobi(A, n, W);
    int64_t best = 0;
    for (int64_t i = 1; i < n; ++i)
      if (A[i + i * n] < A[best + best * n]) best = i;
    *theta = A[best + best * n];
    *zlast = W[(n - 1) + best * n];
  }
  void sync() override {}
  void* stream() override { return nullptr; }

 private:
  double* push(size_t count) {
    bufs_.emplace_back(new double[count]());
    if (getenv("QDWHG_DIST_POISON"))
      for (size_t i = 0; i < count; ++i) bufs_.back()[i] = NAN;
    return bufs_.back().get();
  }
  std::vector<std::unique_ptr<double[]>> bufs_;
};

struct Run {
  std::string err;
};

// one rank of a multi-process run: the comm is the caller's (callbacks)
template <class Body>
int run_one(int P, int Q, int nb, int rank, const CommCallbacks* cb, char* err, int errlen, Body body) {
  try {
    HostEngine e;
    Grid g;
    g.P = P;
    g.Q = Q;
    g.p = rank / Q;
    g.q = rank % Q;
    g.nb = nb;
    std::unique_ptr<Comm> comm(callback_comm_create(*cb, rank, P * Q, g, [] {}));
    Ctx c;
    c.g = g;
    c.comm = comm.get();
    c.eng = &e;
    body(c, rank);
  } catch (const std::exception& ex) {
    if (err && errlen > 0) std::snprintf(err, (size_t)errlen, "rank %d: %s", rank, ex.what());
    return 1;
  }
  return 0;
}

template <class Body>
int run_ranks(int P, int Q, int nb, char* err, int errlen, Body body) {
  const int nr = P * Q;
  LoopbackWorld* w = loopback_world_create(nr);
  std::vector<std::string> errs((size_t)nr);
  std::vector<std::thread> th;
  for (int r = 0; r < nr; ++r)
    th.emplace_back([&, r] {
      try {
        HostEngine e;
        Grid g;
        g.P = P;
        g.Q = Q;
        g.p = r / Q;
        g.q = r % Q;
        g.nb = nb;
        std::unique_ptr<Comm> comm(loopback_comm_create(
            w, r, g, [](void* d, const void* s, size_t b) { std::memcpy(d, s, b); }, [] {}));
        Ctx c;
        c.g = g;
        c.comm = comm.get();
        c.eng = &e;
        body(c, r);
      } catch (const std::exception& ex) {
        errs[(size_t)r] = ex.what();
      }
    });
  for (auto& t : th) t.join();
  loopback_world_destroy(w);
  for (int r = 0; r < nr; ++r)
    if (!errs[(size_t)r].empty()) {
      if (err && errlen > 0) std::snprintf(err, (size_t)errlen, "rank %d: %s", r, errs[(size_t)r].c_str());
      return 1;
    }
  return 0;
}

}  // namespace

extern "C" {

// C = alpha op(A) op(B) + beta C on whole matrices (full host inputs), with the
// structure flags bit0 a_upper, bit1 a_lower, bit2 b_upper, bit3 b_lower, bit4
// c_lower; the result is gathered to Cout (m x n, ldc)
int dh_pgemm(int P, int Q, int nb, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
             const double* A, int64_t lda, const double* B, int64_t ldb, double beta, const double* C0,
             double* Cout, int64_t ldc, int flags, char* err, int errlen) {
  return run_ranks(P, Q, nb, err, errlen, [&](Ctx& c, int r) {
    DistMat Am = make_dist(*c.eng, c.g, ta ? k : m, ta ? m : k);
    DistMat Bm = make_dist(*c.eng, c.g, tb ? n : k, tb ? k : n);
    DistMat Cm = make_dist(*c.eng, c.g, m, n);
    scatter_from_full(c, A, lda, true, Am);
    scatter_from_full(c, B, ldb, true, Bm);
    scatter_from_full(c, C0, ldc, true, Cm);
    Structure st;
    st.a_upper = flags & 1;
    st.a_lower = flags & 2;
    st.b_upper = flags & 4;
    st.b_lower = flags & 8;
    st.c_lower = flags & 16;
    pgemm(c, ta, tb, alpha, whole(Am), whole(Bm), beta, whole(Cm), st);
    gather(c, Cm, r == 0 ? Cout : nullptr, ldc, 0);
  });
}

// W^{-1} of Z = W^T W (lower of Z read) gathered to Winv (n x n)
int dh_chol_inv(int P, int Q, int nb, int64_t n, const double* Z, int64_t ldz, double* Winv, int64_t ldw,
                char* err, int errlen) {
  return run_ranks(P, Q, nb, err, errlen, [&](Ctx& c, int r) {
    DistMat Zm = make_dist(*c.eng, c.g, n, n), Wm = make_dist(*c.eng, c.g, n, n);
    scatter_from_full(c, Z, ldz, true, Zm);
    chol_inv(c, Zm, Wm);
    gather(c, Wm, r == 0 ? Winv : nullptr, ldw, 0);
  });
}

// |diag R| (n values) and Q(:, c0 : c0 + ell) of the Householder QR of X (m x n)
int dh_qr(int P, int Q, int nb, int64_t m, int64_t n, const double* X, int64_t ldx, int64_t c0, int64_t ell,
          double* rdiag, double* Q2, int64_t ldq, char* err, int errlen) {
  return run_ranks(P, Q, nb, err, errlen, [&](Ctx& c, int r) {
    DistMat Xm = make_dist(*c.eng, c.g, m, n);
    scatter_from_full(c, X, ldx, true, Xm);
    QrDist qr;
    pgeqrf(c, Xm, qr);
    DistMat Qm = make_dist(*c.eng, c.g, m, ell);
    porgqr_cols(c, qr, c0, Qm);
    gather(c, Qm, r == 0 ? Q2 : nullptr, ldq, 0);
    if (r == 0) std::memcpy(rdiag, qr.rdiag.data(), sizeof(double) * (size_t)n);
  });
}

// partial.cpp:40-99 (LARGEST map) as ONE rank of a multi-process run whose
// communicator is the caller's callbacks (the CPU gloo test)
int dh_partial_eig_rank(int P, int Q, int nb, int rank, const CommCallbacks* cb, int64_t n, const double* A,
                        int64_t lda, double cshift, int64_t kreq, double* lambda, double* V, int64_t ldv,
                        int64_t* k_out, int64_t* ell_out, double* mu_out, char* err, int errlen) {
  return run_one(P, Q, nb, rank, cb, err, errlen, [&](Ctx& c, int r) {
    DistMat Am = make_dist(*c.eng, c.g, n, n), Bm = make_dist(*c.eng, c.g, n, n);
    scatter_from_full(c, A, lda, true, Am);
    axpby_identity(c, &Am, -1.0, Bm, 0.0, cshift);
    EigResult res = partial_eig(c, Bm, choose_shift(3), 3, false, 0.01, 0);
    int64_t k = (int64_t)res.lambda.size();
    if (kreq > 0) k = std::min(k, kreq);
    *k_out = k;
    *ell_out = (int64_t)res.subspace_size;
    *mu_out = res.mu;
    for (int64_t i = 0; i < k; ++i) lambda[i] = cshift - res.lambda[(size_t)i];
    if (r == 0)
      for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < n; ++i) V[i + j * ldv] = res.V[i + j * res.vld];
  });
}

// partial.cpp:40-99 through the LARGEST request map (B = c I - A); rank 0's
// results: k values of A (largest first), V (n x k), ell, mu
int dh_partial_eig(int P, int Q, int nb, int64_t n, const double* A, int64_t lda, double cshift,
                   int64_t kreq, int randomize, uint64_t seed, double* lambda, double* V, int64_t ldv,
                   int64_t* k_out, int64_t* ell_out, double* mu_out, char* err, int errlen) {
  return run_ranks(P, Q, nb, err, errlen, [&](Ctx& c, int r) {
    DistMat Am = make_dist(*c.eng, c.g, n, n), Bm = make_dist(*c.eng, c.g, n, n);
    scatter_from_full(c, A, lda, true, Am);
    axpby_identity(c, &Am, -1.0, Bm, 0.0, cshift);
    EigResult res = partial_eig(c, Bm, choose_shift(3), 3, randomize != 0, 0.01, seed);
    if (r != 0) return;
    int64_t k = (int64_t)res.lambda.size();
    if (kreq > 0) k = std::min(k, kreq);
    *k_out = k;
    *ell_out = (int64_t)res.subspace_size;
    *mu_out = res.mu;
    for (int64_t i = 0; i < k; ++i) lambda[i] = cshift - res.lambda[(size_t)i];
    for (int64_t j = 0; j < k; ++j)
      for (int64_t i = 0; i < n; ++i) V[i + j * ldv] = res.V[i + j * res.vld];
  });
}

// partial.cpp:101-158 with an absolute cut; rank 0's results
int dh_partial_svd(int P, int Q, int nb, int64_t m, int64_t n, const double* A, int64_t lda, double cut,
                   int64_t kreq, int randomize, uint64_t seed, double* sigma, double* U, int64_t ldu, double* V,
                   int64_t ldv, int64_t* k_out, int64_t* ell_out, double* alpha_out, char* err, int errlen) {
  return run_ranks(P, Q, nb, err, errlen, [&](Ctx& c, int r) {
    DistMat Am = make_dist(*c.eng, c.g, m, n);
    scatter_from_full(c, A, lda, true, Am);
    SvdResult res = partial_svd(c, Am, 0.0, cut, 0.01, randomize != 0, seed);
    if (r != 0) return;
    int64_t k = (int64_t)res.sigma.size();
    if (kreq > 0) k = std::min(k, kreq);
    *k_out = k;
    *ell_out = (int64_t)res.subspace_size;
    *alpha_out = res.alpha;
    for (int64_t i = 0; i < k; ++i) sigma[i] = res.sigma[(size_t)i];
    for (int64_t j = 0; j < k; ++j) {
      for (int64_t i = 0; i < m; ++i) U[i + j * ldu] = res.U[i + j * res.uld];
      for (int64_t i = 0; i < n; ++i) V[i + j * ldv] = res.V[i + j * res.vld];
    }
  });
}

}  // extern "C"
