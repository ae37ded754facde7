// Cholesky factor W (Z = W^T W, upper) and its inverse for the Cholesky-based
// QDWH step (polar.cpp:82-128; reference kernel kernels.cpp:124-146).
//
// B200 shape:
//   * blocked right-looking POTRF, block nb (64/128): the nb x nb diagonal block
//     is factored AND inverted by one CTA entirely in shared memory
//     (potrf_diag_kernel); the row panel W_k,rest = W_kk^-T Z_k,rest and the
//     trailing SYRK Z_rest -= W_k,rest^T W_k,rest are DMMA GEMMs.
//   * TRTRI by recursive halving on top of the diagonal-block inverses:
//     W^-1 = [W11^-1, -W11^-1 W12 W22^-1; 0, W22^-1], two triangular-skipping
//     GEMMs per level.  The two triangular solves of polar.cpp:95-121 then
//     become two TRMMs with W^-1 (same 2mn^2 flops, fully parallel).
// A non-positive pivot raises the device flag; the host turns it into
// NotPositiveDefinite, matching kernels.cpp:136-138.
#include <cstdlib>
#include <functional>

#include "common.cuh"
#include "internal.hpp"
#ifdef QDWHG_DIAG_TRACE  // tools/bench_src/diag_bench: per-phase clock64 marks
namespace qdwhg {
namespace {
__device__ long long g_diag_trace[64];
}
}  // namespace qdwhg
#define DIAG_MARK(i) \
  if (threadIdx.x == 0) g_diag_trace[i] = clock64()
#define QDWHG_LEAF_MARK(i) DIAG_MARK(i)
#define QDWHG_LEAF_MARK_T(i, t) \
  if (threadIdx.x == (t)) g_diag_trace[i] = clock64()
#else
#define DIAG_MARK(i)
#endif
#include "potrf_leaf.cuh"

namespace qdwhg {

namespace {

using leaf::kDiagThreads;
using leaf::kLDA;
using leaf::kLDT;
using leaf::kSB;

// Factor the nb x nb diagonal block (nb <= 128, reads the lower triangle of Z)
// -> W_kk = L^T (upper, to W) and W_kk^{-1} = L^{-T} (upper, to Winv), one CTA,
// all in shared memory (L in place, strict upper kept zero), blocked by 32:
//   load:    cp.async of the lower triangle (all loads in flight at once);
//   per 32-column step kb:
//     warp 0 factors the 32x32 diagonal block (rows in registers, columns broadcast via smem);
//     panel rows below: forward substitution, one row per thread, the row in
//       registers (no multiplication by an explicit inverse: u*kappa accuracy);
//     trailing lower triangle: rank-32 update on DMMA m8n8k4 tiles;
//   W = L^T written out (unless kDiagNoW);
//   D_kb^{-1} of the four diagonal blocks in parallel (one warp each, in place);
//   L^{-1} in place by recursive doubling (32 -> 64 -> 128):
//     L^{-1}_QP = -Q^{-1} (L_QP P^{-1}), both products on DMMA tiles, all pairs
//     of a level at once (2 levels x 2 products instead of 3 x 2 block columns);
//   Winv = L^{-T} written out (upper triangle only with kDiagUpperOnly).
// The block is padded to a multiple of 32 with an identity (chol([Z 0;0 I]) = [L 0;0 I]).
// launch flags
constexpr int kDiagInvertOnly = 1;  // input is an upper R: only R^{-1}
constexpr int kDiagNoW = 2;         // W = L^T is not wanted (not written)
constexpr int kDiagUpperOnly = 4;   // outputs pre-zeroed: write the upper triangles only

__global__ void __launch_bounds__(kDiagThreads, 1)
    potrf_diag_kernel(const double* Z, int64_t ldz, double* W, int64_t ldw, double* Winv,
                      int64_t ldwi, int nb, int* flag, int flags) {
  extern __shared__ double sm[];
  double* A = sm;                    // 128 x kLDA, column-major, lower = L (then L^{-1})
  double* T = A + 128 * kLDA;        // 64 columns x kLDT
  double* Sinv = T + 64 * kLDT;      // 128: 1 / L_ii
  __shared__ int bad_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nbp = ((nb + kSB - 1) / kSB) * kSB;
  if (tid == 0) bad_s = 0;
  DIAG_MARK(20);
  griddep_wait();

  if (flags & kDiagInvertOnly) {
    // Z holds an upper-triangular R: L = R^T is loaded (transposed reads), the
    // factorisation is skipped, and only L^{-1} (-> Winv = R^{-1}) is formed
    for (int c = warp; c < nbp; c += kDiagThreads / 32) {
      double* col = A + c * kLDA;
      for (int r = lane; r < nbp; r += 32)
        col[r] = (r >= c && r < nb && c < nb) ? Z[c + (int64_t)r * ldz] : (r == c ? 1.0 : 0.0);
    }
    __syncthreads();
    if (tid < nbp) {
      const double d = A[tid * kLDA + tid];
      if (!(d != 0.0) || !isfinite(d)) bad_s = 1;
      Sinv[tid] = 1.0 / d;
    }
    __syncthreads();
  } else {
  // ---- load: lower triangle by cp.async, identity padding, zero strict upper
  for (int c = warp; c < nbp; c += kDiagThreads / 32) {
    double* col = A + c * kLDA;
    for (int r = lane; r < nbp; r += 32) {
      if (r >= c && r < nb && c < nb)
        cp_async8(col + r, Z + r + (int64_t)c * ldz);
      else
        col[r] = (r == c) ? 1.0 : 0.0;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  DIAG_MARK(0);

  leaf::factor(A, Sinv, nbp, &bad_s);
  // ---- W = L^T (upper) with explicit zeros below
  if (!(flags & kDiagNoW)) {
    const int rend = (flags & kDiagUpperOnly) ? 0 : nb;
    for (int c = warp; c < nb; c += kDiagThreads / 32) {
      double* wc = W + (int64_t)c * ldw;
#pragma unroll 4
      for (int r = lane; r < max(c + 1, rend); r += 32) wc[r] = (r <= c) ? A[r * kLDA + c] : 0.0;
    }
  }
  DIAG_MARK(13);
  }  // !invert_only
  if (tid == 0 && bad_s) atomicExch(flag, 1);

  leaf::invert(A, T, Sinv, nbp);
  DIAG_MARK(15);

  // PDL: the dependent GEMM's launch and prologue overlap the write-out below
  griddep_launch_dependents();
  // ---- Winv = L^{-T} (upper) with explicit zeros below.  Winv(r, c) = A[r * kLDA + c]:
  // 8 lanes per column (4 columns per warp instruction), so the transposed shared
  // reads hit 16 distinct bank pairs (kLDA = 132) instead of 4 with a lane per row
  {
    const int rend = (flags & kDiagUpperOnly) ? 0 : nb;
    const int j = lane >> 3, rr = lane & 7;
    for (int c0 = 4 * warp; c0 < nb; c0 += 4 * (kDiagThreads / 32)) {
      const int c = c0 + j;
      const int rmax = max(c0 + 4, rend);  // warp-uniform trip count
      double* wc = Winv + (int64_t)c * ldwi;
#pragma unroll 4
      for (int r = rr; r < rmax; r += 8)
        if (c < nb && r < max(c + 1, rend)) wc[r] = (r <= c) ? A[r * kLDA + c] : 0.0;
    }
  }
  DIAG_MARK(16);
}

// The 128 x 128 leaf of the fast path when W itself is not wanted: the fused,
// pipelined factor-and-invert (potrf_leaf.cuh: factor_invert_fused).
__global__ void __launch_bounds__(kDiagThreads, 1)
    potrf_diag_fused_kernel(const double* Z, int64_t ldz, double* Winv, int64_t ldwi, int* flag, int flags) {
  extern __shared__ double sm[];
  double* A = sm;
  double* S = A + 128 * kLDA;
  __shared__ int bad_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int nb = 128;
  if (tid == 0) bad_s = 0;
  DIAG_MARK(20);
  griddep_wait();
  for (int c = warp; c < nb; c += kDiagThreads / 32) {
    double* col = A + c * kLDA;
    for (int r = lane; r < nb; r += 32) {
      if (r >= c)
        cp_async8(col + r, Z + r + (int64_t)c * ldz);
      else
        col[r] = 0.0;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  DIAG_MARK(0);
  leaf::factor_invert_fused(A, S, &bad_s);
  DIAG_MARK(15);
  if (tid == 0 && bad_s) atomicExch(flag, 1);
  griddep_launch_dependents();
  {
    const int rend = (flags & kDiagUpperOnly) ? 0 : nb;
    const int j = lane >> 3, rr = lane & 7;
    for (int c0 = 4 * warp; c0 < nb; c0 += 4 * (kDiagThreads / 32)) {
      const int c = c0 + j;
      const int rmax = max(c0 + 4, rend);  // warp-uniform trip count
      double* wc = Winv + (int64_t)c * ldwi;
#pragma unroll 4
      for (int r = rr; r < rmax; r += 8)
        if (r < max(c + 1, rend)) wc[r] = (r <= c) ? A[r * kLDA + c] : 0.0;
    }
  }
  DIAG_MARK(16);
}

void launch_diag_fused(Ctx& ctx, const DMat& Zkk, const DMat& Wikk, int flags) {
  const size_t fsmem = (size_t)leaf::kFusedSmemDoubles * 8;
  func_attr(potrf_diag_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
  launch_pdl(ctx, potrf_diag_fused_kernel, dim3(1), dim3(kDiagThreads), fsmem, Zkk.ptr(), Zkk.ld,
             Wikk.ptr(), Wikk.ld, ctx.dflag, flags);
  ctx.count();
}

void launch_diag(Ctx& ctx, const DMat& Zkk, const DMat& Wkk, const DMat& Wikk, int flags = 0) {
  static const bool no_fused = getenv("QDWHG_LEAF_NO_FUSED") != nullptr;
  if (Zkk.rows == 128 && (flags & kDiagNoW) && !(flags & kDiagInvertOnly) && !no_fused) {
    launch_diag_fused(ctx, Zkk, Wikk, flags);
    return;
  }
  const size_t smem = (size_t)(128 * kLDA + 64 * kLDT + 128) * 8;
  func_attr(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(ctx, potrf_diag_kernel, dim3(1), dim3(kDiagThreads), smem, Zkk.ptr(), Zkk.ld, Wkk.ptr(),
             Wkk.ld, Wikk.ptr(), Wikk.ld, (int)Zkk.rows, ctx.dflag, flags);
  ctx.count();
}

// W's off-diagonal blocks: from W itself (upper) or, with lower, transposed from
// the L = W^T stored in the lower triangle of the same matrix (chol_dag output).
DMat w_offdiag(const DMat& W, int64_t r0, int64_t c0, int64_t m, int64_t n, bool lower) {
  return lower ? W.sub(c0, r0, n, m) : W.sub(r0, c0, m, n);
}

void trtri_rec(Ctx& ctx, const DMat& W, const DMat& Winv, int64_t r0, int64_t n, int nb,
               bool lower = false) {
  if (n <= nb) return;
  int64_t n1 = ((n / 2 + nb - 1) / nb) * nb;
  if (n1 >= n) n1 = n - nb;
  const int64_t n2 = n - n1;
  trtri_rec(ctx, W, Winv, r0, n1, nb, lower);
  trtri_rec(ctx, W, Winv, r0 + n1, n2, nb, lower);
  const Arena::Mark mark = ctx.arena->mark();
  DMat T = ctx.arena->alloc(n1, n2);
  GemmExtra e1;
  e1.krange = KRange::BUpper;  // B = W22^-1 upper
  gemm(ctx, lower ? Op::T : Op::N, Op::N, 1.0, w_offdiag(W, r0, r0 + n1, n1, n2, lower),
       Winv.sub(r0 + n1, r0 + n1, n2, n2), 0.0, T, e1);
  GemmExtra e2;
  e2.krange = KRange::AUpper;  // A = W11^-1 upper
  gemm(ctx, Op::N, Op::N, -1.0, Winv.sub(r0, r0, n1, n1), T, 0.0, Winv.sub(r0, r0 + n1, n1, n2),
       e2);
  ctx.arena->release_to(mark);
}

// Same recursion, level by level for n = nb * 2^L: all merges of one level are
// independent, so each level is two batched GEMM launches instead of 2 * pairs.
void trtri_levels(Ctx& ctx, const DMat& W, const DMat& Winv, int64_t n, int nb, bool lower = false) {
  for (int64_t h = nb; h < n; h *= 2) {
    const int64_t pairs = n / (2 * h);
    const Arena::Mark mark = ctx.arena->mark();
    DMat T = ctx.arena->alloc(h, h * pairs);  // T_p = T(:, p*h : (p+1)*h)
    GemmExtra e1;
    e1.krange = KRange::BUpper;  // W22^-1 upper
    e1.batch = (int)pairs;
    e1.a_step_r = e1.a_step_c = 2 * h;
    e1.b_step_r = e1.b_step_c = 2 * h;
    e1.c_step_c = h;
    gemm(ctx, lower ? Op::T : Op::N, Op::N, 1.0, w_offdiag(W, 0, h, h, h, lower), Winv.sub(h, h, h, h),
         0.0, T.sub(0, 0, h, h), e1);
    GemmExtra e2;
    e2.krange = KRange::AUpper;  // W11^-1 upper
    e2.batch = (int)pairs;
    e2.a_step_r = e2.a_step_c = 2 * h;
    e2.b_step_c = h;
    e2.c_step_r = e2.c_step_c = 2 * h;
    gemm(ctx, Op::N, Op::N, -1.0, Winv.sub(0, 0, h, h), T.sub(0, 0, h, h), 0.0,
         Winv.sub(0, h, h, h), e2);
    ctx.arena->release_to(mark);
  }
}

// Panel of the stable POTRF: X = W_kk^{-T} Z_k,rest with Z_k,rest read as the
// transpose of the lower block Zr = Z(rest, k) (b x ncols result into X).
// W_kk^T is lower: forward substitution per column, 64 columns per CTA,
// W_kk and the solution tile in shared memory.
__global__ void __launch_bounds__(64) panel_trsm_kernel(const double* Wkk, int64_t ldw,
                                                         const double* Zr, int64_t ldz, double* X,
                                                         int64_t ldx, int b, int ncols) {
  extern __shared__ double smt[];
  double* Ws = smt;              // b x (b+1), Ws[c*(b+1) + r] = W_kk(r, c)
  double* Xs = Ws + b * (b + 1);  // b x 65, Xs[i*65 + col]
  const int tid = threadIdx.x;
  const int j = blockIdx.x * 64 + tid;
  for (int idx = tid; idx < b * b; idx += 64) {
    const int r = idx % b, c = idx / b;
    Ws[c * (b + 1) + r] = Wkk[r + (int64_t)c * ldw];
  }
  __syncthreads();
  if (j < ncols) {
    for (int i = 0; i < b; ++i) {
      double s = Zr[j + (int64_t)i * ldz];  // Z(k+b+j, k+i) = Z_k,rest(i, j)
      const double* wc = Ws + i * (b + 1);  // column i of W_kk: W_kk(t, i)
      for (int t = 0; t < i; ++t) s -= wc[t] * Xs[t * 65 + tid];
      Xs[i * 65 + tid] = s / wc[i];
    }
  }
  __syncthreads();
  // X(i, j): rows i of W's panel block, coalesced along j
  for (int idx = tid; idx < b * 64; idx += 64) {
    const int i = idx / 64, col = idx % 64;
    const int jj = blockIdx.x * 64 + col;
    if (jj < ncols) X[i + (int64_t)jj * ldx] = Xs[i * 65 + col];
  }
}

void launch_panel_trsm(Ctx& ctx, const DMat& Wkk, const DMat& Zr, const DMat& X) {
  const int b = (int)Wkk.rows, ncols = (int)Zr.rows;
  const size_t smem = ((size_t)b * (b + 1) + (size_t)b * 65) * 8;
  func_attr(panel_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)((128 * 129 + 128 * 65) * 8));
  panel_trsm_kernel<<<(ncols + 63) / 64, 64, smem, ctx.stream>>>(Wkk.ptr(), Wkk.ld, Zr.ptr(), Zr.ld,
                                                                X.ptr(), X.ld, b, ncols);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

// Recursive Cholesky-and-inverse on the diagonal block [r0, r0+n):
//   (W11, W11^-1) = rec(Z11);  W12 = W11^-T Z12;  Z22 -= W12^T W12;
//   (W22, W22^-1) = rec(Z22);  W^-1_12 = -W11^-1 W12 W22^-1.
// The trailing SYRK of the top level has K = n/2 (vs 128 for a right-looking
// sweep), so almost all flops run at full DMMA rate; leaves are the 128-block
// diag kernel.  Only the lower triangle of Z is read/updated.
void chol_inv_rec(Ctx& ctx, const DMat& Z, const DMat& W, const DMat& Winv, int64_t r0, int64_t n,
                  int nb, int leaf_flags) {
  // sub-trees up to QDWHG_CHOL_DAG_TMAX tiles: one tile-DAG kernel (W^{-1} only)
  if (nb == 128 && (leaf_flags & kDiagNoW) && chol_dag_applicable(n)) {
    chol_dag(ctx, Z.sub(r0, r0, n, n), Winv.sub(r0, r0, n, n));
    return;
  }
  if (n <= nb) {
    launch_diag(ctx, Z.sub(r0, r0, n, n), W.sub(r0, r0, n, n), Winv.sub(r0, r0, n, n), leaf_flags);
    return;
  }
  int64_t n1 = ((n / 2 + nb - 1) / nb) * nb;
  if (n1 >= n) n1 = n - nb;
  const int64_t n2 = n - n1;
  chol_inv_rec(ctx, Z, W, Winv, r0, n1, nb, leaf_flags);
  const int64_t r1 = r0 + n1;
  GemmExtra e1;
  e1.krange = KRange::ALower;  // op(A) = W11^-T lower
  gemm(ctx, Op::T, Op::T, 1.0, Winv.sub(r0, r0, n1, n1), Z.sub(r1, r0, n2, n1), 0.0,
       W.sub(r0, r1, n1, n2), e1);
  GemmExtra e2;
  e2.out = OutMode::Lower;
  const DMat W12 = W.sub(r0, r1, n1, n2);
  gemm(ctx, Op::T, Op::N, -1.0, W12, W12, 1.0, Z.sub(r1, r1, n2, n2), e2);
  chol_inv_rec(ctx, Z, W, Winv, r1, n2, nb, leaf_flags);
  const Arena::Mark mark = ctx.arena->mark();
  DMat T = ctx.arena->alloc(n1, n2);
  GemmExtra e3;
  e3.krange = KRange::BUpper;  // W22^-1 upper
  gemm(ctx, Op::N, Op::N, 1.0, W12, Winv.sub(r1, r1, n2, n2), 0.0, T, e3);
  GemmExtra e4;
  e4.krange = KRange::AUpper;  // W11^-1 upper
  gemm(ctx, Op::N, Op::N, -1.0, Winv.sub(r0, r0, n1, n1), T, 0.0, Winv.sub(r0, r1, n1, n2), e4);
  ctx.arena->release_to(mark);
}

}  // namespace

// Top level of the fast recursive Cholesky-and-inverse with hooks so a caller
// can overlap independent work on its side stream (qdwh_chol_step):
//   z22_ready(): enqueued right before Z22 is first read (the caller may have
//                produced Z22 on another stream and waits for it here);
//   left_done(): enqueued once W11 and W11^-1 are final (they are not written
//                again), e.g. to start Y(:, 0:n1) = X(:, 0:n1) W11^-1.
// Z is overwritten (lower triangle workspace), Winv receives W^-1 (upper).
void potrf_fast_split(Ctx& ctx, const DMat& Z, const DMat& Winv, int64_t n1,
                      const std::function<void()>& z22_ready,
                      const std::function<void()>& left_done, bool winv_lower_zeroed) {
  const int64_t n = Z.rows;
  const int nb = 128;
  if (n1 % nb || n1 <= 0 || n1 >= n) throw InvalidArgument("potrf_fast_split: bad split");
  if (!ctx.defer_pivot_check) QDWHG_CUDA(cudaMemsetAsync(ctx.dflag, 0, sizeof(int), ctx.stream));
  const Arena::Mark mark = ctx.arena->mark();
  DMat W = ctx.arena->alloc(n, n);
  // W: only its off-diagonal upper blocks W12 are used, each written before it is
  // read (no fill).  W^-1: the chain writes every upper entry (upper-only leaves,
  // W^-1_12 blocks); the strictly lower part must read as zero — zeroed here, or
  // by the caller (on its side stream, overlapping the SYRK)
  if (!winv_lower_zeroed) zero_strict_lower(ctx, Winv);
  const int64_t n2 = n - n1;
  const int leaf = kDiagUpperOnly | kDiagNoW;
  chol_inv_rec(ctx, Z, W, Winv, 0, n1, nb, leaf);
  left_done();
  GemmExtra e1;
  e1.krange = KRange::ALower;  // op(A) = W11^-T lower
  gemm(ctx, Op::T, Op::T, 1.0, Winv.sub(0, 0, n1, n1), Z.sub(n1, 0, n2, n1), 0.0, W.sub(0, n1, n1, n2), e1);
  z22_ready();
  GemmExtra e2;
  e2.out = OutMode::Lower;
  const DMat W12 = W.sub(0, n1, n1, n2);
  gemm(ctx, Op::T, Op::N, -1.0, W12, W12, 1.0, Z.sub(n1, n1, n2, n2), e2);
  chol_inv_rec(ctx, Z, W, Winv, n1, n2, nb, leaf);
  DMat T = ctx.arena->alloc(n1, n2);
  GemmExtra e3;
  e3.krange = KRange::BUpper;  // W22^-1 upper
  gemm(ctx, Op::N, Op::N, 1.0, W12, Winv.sub(n1, n1, n2, n2), 0.0, T, e3);
  GemmExtra e4;
  e4.krange = KRange::AUpper;  // W11^-1 upper
  gemm(ctx, Op::N, Op::N, -1.0, Winv.sub(0, 0, n1, n1), T, 0.0, Winv.sub(0, n1, n1, n2), e4);
  ctx.arena->release_to(mark);
  if (ctx.defer_pivot_check) return;
  int hflag = 0;
  QDWHG_CUDA(cudaMemcpyAsync(&hflag, ctx.dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  if (hflag) throw NotPositiveDefinite("cholesky: pivot is not positive");
}

bool trtri_upper(Ctx& ctx, const DMat& R, const DMat& Rinv) {
  // R^{-1} of an upper-triangular R: 128-block inverses by the leaf kernel in
  // invert-only mode, then the recursive block assembly used for W^{-1}
  const int64_t n = R.rows;
  if (R.cols != n) throw InvalidArgument("trtri: matrix not square");
  const int nb = 128;
  QDWHG_CUDA(cudaMemsetAsync(ctx.dflag, 0, sizeof(int), ctx.stream));
  fill(ctx, Rinv, 0.0, 0.0);
  for (int64_t k = 0; k < n; k += nb) {
    const int64_t b = std::min<int64_t>(nb, n - k);
    launch_diag(ctx, R.sub(k, k, b, b), Rinv.sub(k, k, b, b), Rinv.sub(k, k, b, b),
                kDiagInvertOnly | kDiagUpperOnly);
  }
  const int64_t nblk = n / nb;
  if (n % nb == 0 && (nblk & (nblk - 1)) == 0)
    trtri_levels(ctx, R, Rinv, n, nb);
  else
    trtri_rec(ctx, R, Rinv, 0, n, nb);
  int hflag = 0;
  QDWHG_CUDA(cudaMemcpyAsync(&hflag, ctx.dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  return hflag == 0;
}

void potrf_upper_and_inverse(Ctx& ctx, const DMat& Z, const DMat& Winv, bool want_w, bool stable) {
  const int64_t n = Z.rows;
  if (Z.cols != n) throw InvalidArgument("cholesky: matrix not square");
  static const int nb_env = getenv("QDWHG_POTRF_NB") ? atoi(getenv("QDWHG_POTRF_NB")) : 0;
  const int nb = (nb_env == 32 || nb_env == 64 || nb_env == 96 || nb_env == 128) ? nb_env : 128;
  const bool defer = ctx.defer_pivot_check && !stable && !want_w;
  if (!defer) QDWHG_CUDA(cudaMemsetAsync(ctx.dflag, 0, sizeof(int), ctx.stream));
  const Arena::Mark mark = ctx.arena->mark();
  DMat W = ctx.arena->alloc(n, n);
  // (the fast path without W output reads only W12 blocks it wrote first)
  if (stable || want_w) fill(ctx, W, 0.0, 0.0);
  if (stable) fill(ctx, Winv, 0.0, 0.0);
  else zero_strict_lower(ctx, Winv);  // upper part fully written by the chain
  if (!stable) {
    chol_inv_rec(ctx, Z, W, Winv, 0, n, nb, kDiagUpperOnly | (want_w ? 0 : kDiagNoW));
  } else {
    // right-looking, panel by forward substitution (no explicit inverse in the
    // factorisation: backward stable like the reference's dot-product Cholesky)
    for (int64_t k = 0; k < n; k += nb) {
      const int64_t b = std::min<int64_t>(nb, n - k);
      const int64_t rest = n - k - b;
      launch_diag(ctx, Z.sub(k, k, b, b), W.sub(k, k, b, b), Winv.sub(k, k, b, b), kDiagUpperOnly);
      if (rest > 0) {
        launch_panel_trsm(ctx, W.sub(k, k, b, b), Z.sub(k + b, k, rest, b), W.sub(k, k + b, b, rest));
        GemmExtra e2;
        e2.out = OutMode::Lower;
        const DMat Wp = W.sub(k, k + b, b, rest);
        gemm(ctx, Op::T, Op::N, -1.0, Wp, Wp, 1.0, Z.sub(k + b, k + b, rest, rest), e2);
      }
    }
    const int64_t nblk = n / nb;
    if (n % nb == 0 && (nblk & (nblk - 1)) == 0)
      trtri_levels(ctx, W, Winv, n, nb);
    else
      trtri_rec(ctx, W, Winv, 0, n, nb);
  }
  // one pivot check for the whole factorisation (a failed pivot poisons what
  // follows with NaN, which is discarded: the call throws)
  if (defer) {
    ctx.arena->release_to(mark);
    return;
  }
  int hflag = 0;
  QDWHG_CUDA(cudaMemcpyAsync(&hflag, ctx.dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  if (hflag) {
    ctx.arena->release_to(mark);
    throw NotPositiveDefinite("cholesky: pivot is not positive");
  }
  if (want_w) copy(ctx, W, Z);  // W (upper, zero strict lower) back in Z for qdwhg_cholesky
  ctx.arena->release_to(mark);
}

}  // namespace qdwhg
