// Internal host-side interfaces of libqdwhg (not exported).
//
// Every matrix the device code touches is a column-major FP64 view into a
// 256-byte aligned allocation whose leading dimension is a multiple of 32
// doubles (TMA needs 16-byte strides; 256 B keeps every column start
// sector-aligned).  Views carry the parent base pointer plus a (r0, c0)
// offset so the TMA descriptor can be encoded on the aligned base and the
// offset applied in tensor coordinates.
#pragma once
#include <cuda_runtime.h>

#include "errors.hpp"

#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <cstdlib>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

namespace qdwhg {


#define QDWHG_CUDA(expr)                                                                   \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      throw ::qdwhg::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @ " + \
                               __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

// Column-major view: element (i, j) of the view is base[(r0 + i) + (c0 + j) * ld].
struct DMat {
  double* base = nullptr;
  int64_t ld = 0;
  int64_t r0 = 0, c0 = 0;
  int64_t rows = 0, cols = 0;

  double* ptr() const { return base + r0 + c0 * ld; }
  DMat sub(int64_t i, int64_t j, int64_t m, int64_t n) const {
    DMat s = *this;
    s.r0 += i;
    s.c0 += j;
    s.rows = m;
    s.cols = n;
    return s;
  }
  DMat col_block(int64_t j, int64_t n) const { return sub(0, j, rows, n); }
};

inline int64_t round_ld(int64_t rows) { return ((rows + 31) / 32) * 32; }

// Device arena owned by a handle: bump allocation over a list of cudaMalloc'd
// chunks that persist across calls (no cudaMalloc in steady state).  Marks
// rewind; stream order makes reuse after rewind safe (one stream per handle).
class Arena {
 public:
  struct Mark {
    size_t chunk = 0, off = 0;
  };
  ~Arena();
  void* alloc_bytes(size_t bytes);
  DMat alloc(int64_t rows, int64_t cols);
  void reset() { cur_ = Mark{}; }
  Mark mark() const { return cur_; }
  void release_to(Mark m) { cur_ = m; }
  size_t reserved() const;
  size_t high_water() const { return high_; }
  void reserve(size_t bytes);

 private:
  struct Chunk {
    char* base;
    size_t cap;
  };
  std::vector<Chunk> chunks_;
  Mark cur_;
  size_t high_ = 0;
};

// Kernel attributes are per device: set once per (device, kernel, attribute,
// value) under a mutex, so a second handle on another GPU (or another thread)
// gets its own setting.
void func_attr(const void* kern, cudaFuncAttribute attr, int value);
template <typename... KArgs>
void func_attr(void (*kern)(KArgs...), cudaFuncAttribute attr, int value) {
  func_attr(reinterpret_cast<const void*>(kern), attr, value);
}

// Per-device cached probe result (slot < 8): probe() runs once per device.
int per_device_cached(int slot, int (*probe)());

enum class Op { N, T };
// Which part of the K range can contribute for an output tile (triangular
// operands store explicit zeros; skipping them is the TRMM saving).
enum class KRange { Full, BUpper, BLower, AUpper, ALower };
// Lower: only the lower triangle of a square C is written; LowerMirror also mirrors it.
enum class OutMode { Full, LowerMirror, Lower };

struct DagCache;  // chol_dag.cu: per-handle task list + counters

struct Ctx {
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;        // look-ahead stream (handle-owned, lowest priority)
  cudaStream_t hi = nullptr;          // critical-path stream (handle-owned, highest priority)
  cudaEvent_t ev_main = nullptr, ev_side = nullptr, ev_side2 = nullptr;  // cross-stream ordering
  Arena* arena = nullptr;
  int num_sms = 148;
  int panel_max_ctas = 0;  // GEQRF grid-panel CTA cap while a side stream runs (0 = none)
  // run_fixed_iterations: the factorisations leave the sticky pivot flag for ONE
  // check after the last step (no host round trip per Cholesky step)
  bool defer_pivot_check = false;
  // bitwise reproducible mode: grid-path QR panels reduce through per-CTA slots
  // in a fixed order instead of FP64 atomics (qdwhg_set_deterministic)
  bool deterministic = false;
  double* dscratch = nullptr;   // small device scratch (>= 64 KiB)
  double* hscratch = nullptr;   // pinned host mirror of dscratch
  int* dflag = nullptr;         // device status flag
  std::shared_ptr<DagCache> dag;  // tile-DAG Cholesky state (chol_dag.cu)
  uint64_t gemm_launches = 0;   // our kernels launched (for bench accounting)
  uint64_t other_launches = 0;
  void count(int n = 1) { other_launches += n; }
  // Live GEMM profiling: CUDA events around every DMMA GEMM launch on the
  // launching stream (qdwhg_profile / qdwhg_get_kernel_stats).
  bool profile = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<double> ev_flops;  // algorithmic flops of launch i (events 2i, 2i+1)
  std::vector<std::string> ev_tag;  // per-launch shape tag (QDWHG_PROFILE_LOG)
  std::vector<int> ev_kind;          // 0 GEMM engine, 1 tile-DAG Cholesky
  size_t ev_used = 0;
  double gemm_ms = 0.0, gemm_flops = 0.0, gemm_busy_ms = 0.0;
  uint64_t gemm_timed = 0;
  double dag_ms = 0.0, dag_flops = 0.0;
  uint64_t dag_timed = 0;
  void prof_begin(double flops, const std::string& tag = std::string(), int kind = 0);
  void prof_end();
  void prof_collect();
};

// Launch with programmatic stream serialisation (the kernel must call
// griddep_wait() before touching global memory); QDWHG_NO_PDL disables it.
template <typename... KArgs, typename... Args>
void launch_pdl(const Ctx& ctx, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                Args&&... args) {
  static const bool pdl = getenv("QDWHG_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx.stream;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &at;
  cfg.numAttrs = pdl ? 1 : 0;
  QDWHG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// ------------------------------------------------------------------ gemm.cu
// C = alpha * op(A) * op(B) + beta * Cin (+ diag_add on the diagonal of C).
// Cin defaults to C itself.  M x N x K are the op() shapes.
struct GemmExtra {
  KRange krange = KRange::Full;
  OutMode out = OutMode::Full;
  const DMat* cin = nullptr;
  double diag_add = 0.0;
  int split_k = 0;  // 0 = automatic
  int force_bm = 0;  // 0 = automatic; 128 / 64 / 32 pins the tile size
  // skinny products (an l-column block against n x n): 64-tile CTAs with a 6-stage
  // ring, two per SM, and the split-K model that goes with it (measured on cfg2's
  // projection GEMMs: 12-14 -> 18-19 TF).  Opt-in per call site: the default plan
  // also shapes the bench inputs' bytes (tests/golden/fullsize), so it stays as is.
  bool skinny = false;
  // wave-balanced tail: take the model's cheapest split factor outright instead of the
  // first one that improves on the previous by 3 % (n = 4096 lower-triangle launches:
  // 84 tail tiles split 7 ways, four waves of K/7, instead of 3 ways, two waves of K/3:
  // cfg2 -0.4 ms).  Opt-in per call site like `skinny`.
  bool fine_tail = false;
  // Batched launch: item b uses A/B/C shifted by b * (step_r rows, step_c cols)
  // of their stored matrices (items must tile exactly; no split-K).
  int batch = 1;
  int64_t a_step_r = 0, a_step_c = 0, b_step_r = 0, b_step_c = 0, c_step_r = 0, c_step_c = 0;
};
void gemm(Ctx& ctx, Op ta, Op tb, double alpha, const DMat& A, const DMat& B, double beta,
          const DMat& C, const GemmExtra& ex = {});

// ------------------------------------------------------------------ blas1.cu
void fill(Ctx& ctx, const DMat& X, double v, double diag);
// Y = a*X + b*I (Y may alias X)
void axpby_identity(Ctx& ctx, const DMat& X, double a, double diag, const DMat& Y);
// Y = a * (X + X^T)/2 + diag*I  (square; Y must not alias X unless in place-safe mode)
void symmetrize_scale(Ctx& ctx, const DMat& X, double a, double diag, const DMat& Y);
// Y = a (X + X^T)/2 + diag I and Y2 = a2 Y + diag2 I in one pass (Y, Y2 distinct from X)
void symmetrize_scale2(Ctx& ctx, const DMat& X, double a, double diag, const DMat& Y, double a2,
                       double diag2, const DMat& Y2);
void copy(Ctx& ctx, const DMat& X, const DMat& Y);
// Y = X^T (Y must not alias X)
void transpose(Ctx& ctx, const DMat& X, const DMat& Y);
void copy_from_host(Ctx& ctx, const double* h, int64_t ldh, const DMat& Y);
void copy_to_host(Ctx& ctx, const DMat& X, double* h, int64_t ldh);
// Reductions (results land in ctx.hscratch after sync): frobenius^2, max |x_ij - x_ji|,
// nonfinite count.
struct MatStats {
  double fro2 = 0, asym = 0, nonfinite = 0, maxabs = 0;
};
MatStats mat_stats(Ctx& ctx, const DMat& X, bool want_asym);
void gaussian_fill(Ctx& ctx, const DMat& X, uint64_t seed);
void mirror_lower_to_upper(Ctx& ctx, const DMat& X);
void zero_strict_lower(Ctx& ctx, const DMat& X);

// ------------------------------------------------------------------ tiles.cu
// (local-array kernels of the distributed driver)
struct TileDesc {
  const double* src;
  int64_t lds;
  double* dst;
  int64_t ldd;
  int32_t rows, cols;  // of src
  int32_t trans;       // dst (cols x rows) = src^T
};
void copy_tiles(Ctx& ctx, const std::vector<TileDesc>& list);
// Y = a X + b Y (X may be null: Y = b Y; b == 0: Y is not read)
void axpby(Ctx& ctx, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t m, int64_t n, double a,
           double b);
void add_diag(Ctx& ctx, double* Y, int64_t ld, int64_t len, double v);
void zero_strict_upper(Ctx& ctx, const DMat& X);
// entries (gr0 + i, gc0 + j) of the gm-row matrix of gaussian_fill's stream
void gaussian_fill_at(Ctx& ctx, double* X, int64_t ld, int64_t m, int64_t n, uint64_t seed, int64_t gr0,
                      int64_t gc0, int64_t gm);

// ------------------------------------------------------------------ potrf.cu
// Z = W^T W with W upper; only the lower triangle of Z is read (it is used as
// workspace).  Winv (n x n) receives W^{-1} (upper, explicit zeros below); with
// want_w, Z is overwritten by W (upper, zeros below).  Throws NotPositiveDefinite.
// stable = true: right-looking factorisation with triangular-solve panels
// (backward stable for any SPD input); stable = false: recursive variant that
// multiplies by explicit inverses of half blocks (errors ~ u*kappa(W)^2, used
// only for the QDWH Cholesky steps where kappa(Z) <= 1 + c).
void potrf_upper_and_inverse(Ctx& ctx, const DMat& Z, const DMat& Winv, bool want_w = false,
                             bool stable = true);

// ------------------------------------------------------------------ chol_dag.cu
// Tile-DAG Cholesky-and-inverse (n = 128 T, 2 <= T <= QDWHG_CHOL_DAG_TMAX): one
// persistent kernel.  Winv receives W^{-1} (upper; its strict lower must be zero
// already); all of Z is workspace (lower tiles: L, diagonal tiles: L_kk^{-1},
// upper tiles: partial sums of the inverse).  Pivot failures set ctx.dflag.
bool chol_dag_applicable(int64_t n);
void chol_dag(Ctx& ctx, const DMat& Z, const DMat& Winv);

// R^{-1} (upper, explicit zeros below) of an upper-triangular R; false if a
// diagonal entry is zero / non-finite.
bool trtri_upper(Ctx& ctx, const DMat& R, const DMat& Rinv);

// Top-level split of the fast variant with overlap hooks (see potrf.cu).
void potrf_fast_split(Ctx& ctx, const DMat& Z, const DMat& Winv, int64_t n1,
                      const std::function<void()>& z22_ready,
                      const std::function<void()>& left_done, bool winv_lower_zeroed = false);

// ------------------------------------------------------------------ geqrf.cu
struct QrWork {
  DMat V;               // m x n: unit-lower Householder vectors (explicit 1 / 0)
  DMat T;               // nb x n: compact-WY T factors per panel, packed
  std::vector<double> taus;
  int nb = 64;
  int64_t top_rows = 0;  // > 0: structured [T; upper-triangular] stack (geqrf's top_rows)
};
// In place Householder QR of A (m x n, m >= n): R in the upper triangle of A,
// reflectors in work.V / work.T.  Reference convention (kernels.cpp:41-80):
// p = min(m-1, n) reflectors, R_jj = -sign(x0) ||x||.
void geqrf(Ctx& ctx, const DMat& A, QrWork& work, int64_t top_rows = 0);
// Q(:, c0 : c0+ncols) of the m x m Q = H_0 H_1 ... H_{p-1} into Qout (m x ncols).
void orgqr_cols(Ctx& ctx, const QrWork& work, int64_t m, int64_t p, int64_t c0, const DMat& Qout);
// C <- Q C (C is m x ncols, Q = H_0 ... H_{p-1} of an m x n geqrf).
void ormqr_left(Ctx& ctx, const QrWork& work, int64_t m, int64_t n, const DMat& C);
// diag(R) to host (n values).
void diag_to_host(Ctx& ctx, const DMat& R, std::vector<double>& d);
// detect_deficiency_index on the device: first i (1-based) with |R_ii| < tol
// (reciprocal: with |1 / R_ii| < tol), 0 when none.
int64_t first_deficient(Ctx& ctx, const DMat& R, double tol, bool reciprocal = false);

// ------------------------------------------------------------------ syevj.cu
// Symmetric eigendecomposition of S (n x n, device).  Ascending values to host
// `vals`, vectors into Vout (n x n).  Jacobi for small n, QDWH spectral
// divide-and-conquer above the Jacobi cutoff.
void syev(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout);
// All eigenvalues (ascending) into vals; eigenvectors only for the eigenvalues
// in (vlo, vhi) — a contiguous index range starting at *sel0 — into
// Vout(:, 0:count).  Returns count.
int64_t syev_range(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout, double vlo,
                   double vhi, int64_t* sel0);

// Lowest eigenvalue of the symmetric tridiagonal (d, e) (host arrays, n <= 64)
// and the last component of its unit eigenvector, on the device: warp
// multisection on the Sturm count + inverse iteration (syevd.cu kernels).
void tridiag_lowest(Ctx& ctx, const std::vector<double>& d, const std::vector<double>& e,
                    double* theta, double* z_last);

// ------------------------------------------------------------------ krylov.cu
double two_norm_estimate(Ctx& ctx, const DMat& A);
// pre: the caller's mat_stats(A, true) of the same A (skips the second pass)
double lanczos_min_bound(Ctx& ctx, const DMat& A, int steps, const MatStats* pre = nullptr);

}  // namespace qdwhg
