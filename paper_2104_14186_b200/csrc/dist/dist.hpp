// Distributed QDWHpartial on a P x Q process grid with 2D block-cyclic tiles
// (2D block-cyclic data distribution, Q >= P; Alg. 3,
// pdgemm / pdpotrf / pdgeqrf / pdorgqr building blocks).
//
// SPMD: every rank (one per GPU, or one host thread per emulated rank) runs the
// same driver on its local tiles.  The orchestration here is CUDA-free and
// talks to two interfaces:
//   Comm   — broadcasts of panels / diagonal blocks within the grid's row, column
//            or world teams, scalar / short-vector all-reductions, and grouped
//            point-to-point tile exchanges (transposes, gathers to the root).
//            NCCL over NVLink in libqdwhg (comm_nccl.cpp); an in-process loopback
//            for emulated ranks (comm_loopback.cpp).
//   Engine — the rank's local compute on its local arrays: the DMMA GEMM engine,
//            batched tile copies, the single-GPU Cholesky-and-inverse and panel
//            QR, and the gathered Rayleigh-Ritz solvers (engine_cuda.cpp), or a
//            plain host implementation for the CPU multi-rank tests.
//
// Layout (ScaLAPACK-style, zero source offsets): global tile (I, J) (nb x nb,
// the last row/column of tiles possibly partial) lives on rank (I % P, J % Q)
// at local tile (I / P, J / Q); each rank stores its tiles as ONE column-major
// local array (lrows x lcols, ld a multiple of 32), so the tiles of a tile-aligned
// sub-view owned by a rank form one contiguous local block.
#pragma once
#include <cstddef>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "../errors.hpp"
#include "../scalars.hpp"

namespace qdwhg {
namespace dist {

enum class Team { World, Row, Col };
enum class RedOp { Sum, Max, Min };

class Comm {
 public:
  virtual ~Comm() {}
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // Collectives over a team of the grid; `root` is the root's WORLD rank.
  // Calls between group_begin/group_end are issued as one group (NCCL group
  // semantics: they may complete in any order, all before group_end returns
  // their work to the stream).
  virtual void group_begin() = 0;
  virtual void group_end() = 0;
  virtual void bcast(double* buf, size_t count, int root, Team team) = 0;
  virtual void allreduce(double* buf, size_t count, RedOp op, Team team) = 0;
  virtual void send(const double* buf, size_t count, int peer) = 0;
  virtual void recv(double* buf, size_t count, int peer) = 0;
  // team geometry (set by the grid)
  int P = 1, Q = 1;
};

struct TileCopy {
  const double* src;
  int64_t lds;
  double* dst;
  int64_t ldd;
  int32_t rows, cols;  // of src
  int32_t trans;       // dst (cols x rows) = src^T
};

struct EMark {
  size_t a = 0, b = 0;
};

class Engine {
 public:
  virtual ~Engine() {}
  // workspace (stack discipline)
  virtual double* alloc(int64_t rows, int64_t cols, int64_t* ld) = 0;
  virtual double* alloc_vec(size_t count) = 0;
  virtual EMark mark() = 0;
  virtual void release(EMark m) = 0;
  // C = alpha op(A) op(B) + beta C   (column-major, M x N x K of the op shapes)
  virtual void gemm(bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                    int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) = 0;
  virtual void copy_tiles(const std::vector<TileCopy>& list) = 0;
  // Y = a X + b Y (rows x cols); X may be null (then Y = b Y)
  virtual void axpby(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t rows, int64_t cols,
                     double a, double b) = 0;
  virtual void fill(double* Y, int64_t ldy, int64_t rows, int64_t cols, double v) = 0;
  // Y(i, i) += v for i < len
  virtual void add_diag(double* Y, int64_t ldy, int64_t len, double v) = 0;
  // upper <- lower of a square block
  virtual void mirror_lower(double* Y, int64_t ldy, int64_t n) = 0;
  // counter-based N(0,1) (kernels.cpp:441-447): element (i, j) of the block is
  // the global entry (gr0 + i, gc0 + j) of a gm-row matrix
  virtual void gaussian(double* Y, int64_t ldy, int64_t rows, int64_t cols, uint64_t seed,
                        int64_t gr0, int64_t gc0, int64_t gm) = 0;
  // sum of squares, max |x_ij - x_ji| (square, want_asym), non-finite count
  virtual void stats(const double* X, int64_t ldx, int64_t rows, int64_t cols, double out[3],
                     bool want_asym) = 0;
  virtual double dot(const double* x, const double* y, int64_t n) = 0;
  virtual void to_host(const double* src, int64_t lds, int64_t rows, int64_t cols, double* h,
                       int64_t ldh) = 0;
  virtual void from_host(const double* h, int64_t ldh, int64_t rows, int64_t cols, double* dst,
                         int64_t ldd) = 0;
  // single-rank dense kernels
  // W^{-1} (upper, zeros below) of Z = W^T W reading Z's lower triangle (kappa(Z)
  // small: the QDWH Cholesky steps); throws NotPositiveDefinite
  virtual void chol_inv(const double* Z, int64_t ldz, int64_t n, double* Winv, int64_t ldw) = 0;
  // in place Householder QR of an m x w panel (reference convention,
  // kernels.cpp:41-80; bitwise reproducible): V unit lower with explicit 1/0 in P,
  // compact-WY T (w x w upper) so that H_0..H_{w-1} = I - V T V^T, |diag R| to rdiag
  virtual void qr_panel(double* Pn, int64_t ldp, int64_t m, int64_t w, double* T, int64_t ldt,
                        std::vector<double>& rdiag) = 0;
  // ascending eigenvalues of the symmetric S (all), vectors for those in (vlo, vhi)
  virtual int64_t syev_range(double* S, int64_t lds, int64_t n, std::vector<double>& vals, double* V,
                             int64_t ldv, double vlo, double vhi, int64_t* sel0) = 0;
  // descending singular values (all), U (m x k) / V (n x k) for sigma > cut; returns k
  virtual int64_t svd_polar(const double* A, int64_t lda, int64_t m, int64_t n, double* U, int64_t ldu,
                            std::vector<double>& sigma, double* V, int64_t ldv, double cut) = 0;
  virtual void tridiag_lowest(const std::vector<double>& d, const std::vector<double>& e, double* theta,
                              double* zlast) = 0;
  virtual void sync() = 0;
  virtual void* stream() = 0;  // the stream collectives are ordered on (null on host)
};

struct Grid {
  int P = 1, Q = 1, p = 0, q = 0, nb = 512;
  int world_rank(int pr, int pc) const { return pr * Q + pc; }
};

// local length of a block-cyclic dimension (ScaLAPACK numroc, source 0)
int64_t numroc(int64_t n, int64_t nb, int iproc, int nprocs);

struct DistMat {
  int64_t m = 0, n = 0;
  const Grid* g = nullptr;
  int64_t lr = 0, lc = 0;  // local rows / cols
  double* a = nullptr;
  int64_t ld = 1;
  int64_t mt() const { return (m + g->nb - 1) / g->nb; }
  int64_t nt() const { return (n + g->nb - 1) / g->nb; }
  int64_t tile_rows(int64_t I) const { return std::min<int64_t>(g->nb, m - I * g->nb); }
  int64_t tile_cols(int64_t J) const { return std::min<int64_t>(g->nb, n - J * g->nb); }
  // local row offset of global tile row I (caller owns it) / col offset of J
  int64_t lrow(int64_t I) const { return (I / g->P) * g->nb; }
  int64_t lcol(int64_t J) const { return (J / g->Q) * g->nb; }
  bool owns_row(int64_t I) const { return I % g->P == g->p; }
  bool owns_col(int64_t J) const { return J % g->Q == g->q; }
  double* tile(int64_t I, int64_t J) const { return a + lrow(I) + lcol(J) * ld; }
};

DistMat make_dist(Engine& e, const Grid& g, int64_t m, int64_t n);

// Tile-aligned sub-view: tiles [i0, i0 + mt) x [j0, j0 + nt) of M.
struct View {
  const DistMat* M;
  int64_t i0, j0, mt, nt;
};
inline View whole(const DistMat& M) { return View{&M, 0, 0, M.mt(), M.nt()}; }

// Zero structure of the operands (view-relative tile indices) and the output
// mask of a distributed GEMM; zero tiles are skipped, not multiplied.
struct Structure {
  bool a_upper = false;  // op(A)(I, k) = 0 for I > k
  bool a_lower = false;  // op(A)(I, k) = 0 for I < k
  bool b_upper = false;  // op(B)(k, J) = 0 for k > J
  bool b_lower = false;  // op(B)(k, J) = 0 for k < J
  bool c_lower = false;  // only tiles I >= J of C are computed (C square, on the diagonal)
};

struct Ctx {
  Grid g;
  Comm* comm = nullptr;
  Engine* eng = nullptr;
  uint64_t collectives = 0;  // issued (for accounting)
  uint64_t gemms = 0;
};

// C = alpha op(A) op(B) + beta C over tile-aligned views (SUMMA with whole-operand
// panel fetches: one grouped broadcast per operand, then local DMMA GEMMs).
void pgemm(Ctx& c, bool ta, bool tb, double alpha, const View& A, const View& B, double beta,
           const View& C, const Structure& st = {});
// Square DistMat: upper <- lower (tile exchange with the transposed owner).
void mirror_lower(Ctx& c, const DistMat& X);
// Y = X^T (Y n x m on the same grid; tile exchange)
void transpose_into(Ctx& c, const DistMat& X, const DistMat& Y);
// Y = a X + b Y + d I over the whole matrices (same shape/grid).
void axpby_identity(Ctx& c, const DistMat* X, double a, const DistMat& Y, double b, double d);
// sum of squares, max |x_ij - x_ji|, non-finite count over all ranks (replicated)
void stats(Ctx& c, const DistMat& X, bool want_asym, double out[3]);
// W^{-1} of Z = W^T W (lower triangle of Z read; Z used as workspace): recursive
// Cholesky-and-inverse over tile-aligned halves, leaf = one tile on its owner.
void chol_inv(Ctx& c, const DistMat& Z, const DistMat& Winv);
// Replicated dense copy of a DistMat on every rank (for small blocks) / on root.
void gather(Ctx& c, const DistMat& X, double* dst, int64_t ldd, int root /* -1: all */);
// Scatter a full matrix (host or engine buffer on every rank) into local tiles.
void scatter_from_full(Ctx& c, const double* full, int64_t ldf, bool host, const DistMat& X);

struct QrDist {
  std::vector<double*> V;        // per panel: V rows for my local rows (lr x w), ld vld
  int64_t vld = 0;
  std::vector<double*> T;        // per panel: w x w (replicated), ld nb
  std::vector<double> rdiag;     // |R_ii|, replicated
  int64_t m = 0, n = 0;
};
// Householder QR of the square/tall X (destroyed); panels gathered to every rank
// of the grid (world broadcasts), factored redundantly and bitwise identically.
void pgeqrf(Ctx& c, const DistMat& X, QrDist& qr);
// Q(:, c0 : c0 + ell) of the geqrf into Q2 (m x ell DistMat).
void porgqr_cols(Ctx& c, const QrDist& qr, int64_t c0, const DistMat& Q2);

// Replicated vectors: y = A x (A m x n distributed, x length n, y length m).
void pgemv(Ctx& c, const DistMat& A, bool trans, const double* x, double* y);

double lanczos_min_bound(Ctx& c, const DistMat& A, int steps, double fro);
double two_norm_estimate(Ctx& c, const DistMat& A);

struct EigResult {
  std::vector<double> lambda;  // ascending (of the input B)
  double* V = nullptr;         // root: n x k dense (engine buffer), ld vld
  int64_t vld = 0;
  double mu = 0;
  size_t rank_index = 0, subspace_size = 0, iters_chol = 0, borderline = 0;
  bool no_savings = false;
  std::vector<double> trace;
  double flops = 0;
  double stage_seconds[8] = {0};
};
// partial.cpp:40-99 (Alg. 1) on the distributed A (n x n).
EigResult partial_eig(Ctx& c, const DistMat& A, double s, size_t iters, bool randomize, double tol,
                      uint64_t seed, const std::function<double()>& clock = nullptr);

struct SvdResult {
  std::vector<double> sigma;  // descending
  double* U = nullptr;        // root: m x k dense, ld uld
  double* V = nullptr;        // root: n x k dense, ld vld
  int64_t uld = 0, vld = 0;
  double alpha = 0, threshold = 0;
  size_t rank_index = 0, subspace_size = 0, iters_qr = 0, iters_chol = 0;
  bool no_savings = false;
  std::vector<double> trace;
  double flops = 0;
  double stage_seconds[8] = {0};
};
// partial.cpp:101-158 (Alg. 2), Cholesky-based steps (s >= 1e-3).
SvdResult partial_svd(Ctx& c, const DistMat& A, double s, double s_abs, double tol, bool randomize,
                      uint64_t seed, const std::function<double()>& clock = nullptr);

// Communicator over caller callbacks (same layout as qdwhg_comm_callbacks).
// team: 0 world, 1 row, 2 column; op: 0 sum, 1 max, 2 min.  Received data and
// reduced results must be in place when the callback returns, except inside a
// group_begin/group_end bracket, where they must be in place at group_end.
struct CommCallbacks {
  void* ctx;
  int (*bcast)(void* ctx, double* buf, size_t count, int root, int team);
  int (*allreduce)(void* ctx, double* buf, size_t count, int op, int team);
  int (*send)(void* ctx, const double* buf, size_t count, int peer);
  int (*recv)(void* ctx, double* buf, size_t count, int peer);
  int (*group_begin)(void* ctx);
  int (*group_end)(void* ctx);
};
Comm* callback_comm_create(const CommCallbacks& cb, int rank, int world, const Grid& g,
                           std::function<void()> sync);

// In-process loopback world for emulated ranks (threads of one process).
class LoopbackWorld;
LoopbackWorld* loopback_world_create(int nranks);
void loopback_world_destroy(LoopbackWorld* w);
// copy_fn(dst, src, bytes): the engine's buffer copy (device or host memcpy,
// synchronous); `sync` flushes the calling rank's queued work before a rendezvous
Comm* loopback_comm_create(LoopbackWorld* w, int rank, const Grid& g,
                           std::function<void(void*, const void*, size_t)> copy_fn,
                           std::function<void()> sync);

}  // namespace dist
}  // namespace qdwhg
