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

#include "common.cuh"
#include "internal.hpp"

namespace qdwhg {

namespace {

constexpr int kDiagThreads = 256;

// 1/sqrt(d) without the libdevice slow-path call (which forces the unrolled
// register row to the stack): float seed + 3 Newton steps, exponent-scaled so
// any positive double works.  Non-positive d returns NaN (the caller flags it).
QDWHG_DEV double rsqrt_newton(double d) {
  if (!(d > 0.0)) return __longlong_as_double(0x7ff8000000000000ll);
  const int e = ((__double2hiint(d) >> 20) & 0x7ff) - 1023;  // d = m * 2^e, m in [1, 2)
  const int h = e >> 1;                                       // floor(e/2)
  const double m = __hiloint2double(__double2hiint(d) - (h << 21), __double2loint(d));  // d / 4^h
  double y = (double)rsqrtf((float)m);
#pragma unroll
  for (int it = 0; it < 3; ++it) y = y * (1.5 - 0.5 * m * y * y);
  return __hiloint2double(__double2hiint(y) - (h << 20), __double2loint(y));  // y / 2^h
}
constexpr int kSB = 32;          // sub-block handled by one warp
constexpr int kLDA = 129;        // padded smem leading dimension (odd -> conflict free)

// One right-looking Cholesky column step of a 32x32 block held as one row per
// lane; template recursion guarantees compile-time register indices.
template <int J>
struct CholStep {
  static QDWHG_DEV void run(double (&row)[kSB], int lane, bool& bad, double& my_inv) {
    const double djj = __shfl_sync(0xffffffffu, row[J], J);
    if (!(djj > 0.0)) bad = true;
    const double inv = rsqrt_newton(djj);
    if (lane > J) row[J] *= inv;
    if (lane == J) {
      row[J] = djj * inv;
      my_inv = inv;
    }
#pragma unroll
    for (int c = J + 1; c < kSB; ++c) {
      const double lcj = __shfl_sync(0xffffffffu, row[J], c);
      if (lane >= c) row[c] -= row[J] * lcj;
    }
    CholStep<J + 1>::run(row, lane, bad, my_inv);
  }
};
template <>
struct CholStep<kSB> {
  static QDWHG_DEV void run(double (&)[kSB], int, bool&, double&) {}
};

// Factor the nb x nb diagonal block (nb <= 128, reads the lower triangle of Z)
// -> W_kk = L^T (upper, to W) and W_kk^{-1} = L^{-T} (upper, to Winv), one CTA,
// all in shared memory, blocked by 32:
//   per 32-column step: warp 0 factors + inverts the 32x32 diagonal block in
//   registers (shuffles, no CTA barrier), the panel below is L_p = Z_p D^{-T},
//   the trailing lower triangle gets a rank-32 update with 4x4 register tiles;
//   then L^{-1} column block by column block: Linv_ij = -D_i^{-1} sum_k L_ik Linv_kj.
// The block is padded to a multiple of 32 with an identity (chol([Z 0;0 I]) = [L 0;0 I]).
__global__ void __launch_bounds__(kDiagThreads, 1)
    potrf_diag_kernel(const double* Z, int64_t ldz, double* W, int64_t ldw, double* Winv,
                      int64_t ldwi, int nb, int* flag) {
  extern __shared__ double sm[];
  double* A = sm;                          // 128 x kLDA, column-major, lower = L
  double* Dinv = A + 128 * kLDA;           // 4 blocks of 32 x 33 (column-major, lower)
  double* T = Dinv + 4 * kSB * 33;         // 32 columns x kLDA: panel temp / Linv column block
  double* S = T + kSB * kLDA;              // 32 x 33 scratch
  __shared__ int bad_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nbp = ((nb + kSB - 1) / kSB) * kSB;
  const int nsb = nbp / kSB;
  if (tid == 0) bad_s = 0;

  for (int idx = tid; idx < nbp * nbp; idx += kDiagThreads) {
    const int r = idx % nbp, c = idx / nbp;
    double v = 0.0;
    if (r >= c) v = (r < nb && c < nb) ? Z[r + (int64_t)c * ldz] : (r == c ? 1.0 : 0.0);
    A[c * kLDA + r] = v;
  }
  __syncthreads();

  for (int kb = 0; kb < nsb; ++kb) {
    const int b0 = kb * kSB;
    double* D = Dinv + kb * kSB * 33;
    if (warp == 0) {
      // ---- factor the 32x32 diagonal block in registers: lane i owns row i.
      // No division/sqrt library calls in here (their slow-path CALL would push
      // the unrolled register rows to the stack): pivots use rsqrt_newton.
      double row[kSB];
#pragma unroll
      for (int c = 0; c < kSB; ++c) row[c] = (c <= lane) ? A[(b0 + c) * kLDA + b0 + lane] : 0.0;
      bool bad = false;
      double my_inv = 0.0;
      CholStep<0>::run(row, lane, bad, my_inv);  // fully unrolled: registers stay registers
#pragma unroll
      for (int c = 0; c < kSB; ++c)
        if (c <= lane) A[(b0 + c) * kLDA + b0 + lane] = row[c];
      if (bad && lane == 0) bad_s = 1;
      S[lane] = my_inv;  // 1 / L_ii
      __syncwarp();
      // ---- D^{-1}: lane j computes column j by forward substitution (registers)
      double x[kSB];
#pragma unroll
      for (int i = 0; i < kSB; ++i) {
        double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < i; ++k)
          if (k >= lane) s -= A[(b0 + k) * kLDA + b0 + i] * x[k];
        x[i] = (i >= lane) ? s * S[i] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < kSB; ++i) D[lane * 33 + i] = x[i];
    }
    __syncthreads();
    const int p0 = b0 + kSB, R = nbp - p0;
    if (R > 0) {
      // ---- panel rows below the block by forward substitution (one thread per
      // row; no multiplication by the explicit inverse, which would cost
      // u*kappa(D)^2 accuracy on ill-conditioned blocks):
      // L(i, b0+c) = (Z(i, b0+c) - sum_{t<c} L(i, b0+t) L(b0+c, b0+t)) / L(b0+c, b0+c)
      for (int i = tid; i < R; i += kDiagThreads) {
        for (int c = 0; c < kSB; ++c) {
          double s = A[(b0 + c) * kLDA + p0 + i];
          for (int t = 0; t < c; ++t) s -= A[(b0 + t) * kLDA + p0 + i] * A[(b0 + t) * kLDA + b0 + c];
          A[(b0 + c) * kLDA + p0 + i] = s * S[c];
        }
      }
      __syncthreads();
      // ---- trailing rank-32 update of the lower triangle, 4x4 register tiles
      const int tr = R / 4;
      const int ntiles = tr * (tr + 1) / 2;
      for (int t = tid; t < ntiles; t += kDiagThreads) {
        int tj = 0, rem = t;
        while (rem >= tr - tj) {
          rem -= tr - tj;
          ++tj;
        }
        const int ti = tj + rem;
        const int i0 = p0 + 4 * ti, j0 = p0 + 4 * tj;
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        for (int c = 0; c < kSB; ++c) {
          const double* col = A + (b0 + c) * kLDA;
          double li[4], lj[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            li[a] = col[i0 + a];
            lj[a] = col[j0 + a];
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] += li[a] * lj[b];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (i0 + a >= j0 + b) A[(j0 + b) * kLDA + i0 + a] -= acc[a][b];
      }
      __syncthreads();
    }
  }
  if (tid == 0 && bad_s) atomicExch(flag, 1);

  // ---- W = L^T (upper) with explicit zeros below
  for (int idx = tid; idx < nb * nb; idx += kDiagThreads) {
    const int r = idx % nb, c = idx / nb;
    W[r + (int64_t)c * ldw] = (r <= c) ? A[r * kLDA + c] : 0.0;
  }

  // ---- L^{-1} by 32-column blocks; Winv = L^{-T}
  for (int jb = 0; jb < nsb; ++jb) {
    const int c0 = jb * kSB;
    for (int idx = tid; idx < kSB * nbp; idx += kDiagThreads) {
      const int r = idx % nbp, c = idx / nbp;
      double v = 0.0;
      if (r >= c0 && r < c0 + kSB) v = Dinv[jb * kSB * 33 + c * 33 + (r - c0)];
      T[c * kLDA + r] = v;
    }
    __syncthreads();
    for (int ib = jb + 1; ib < nsb; ++ib) {
      const int r0 = ib * kSB;
      // S = sum_{k in [c0, r0)} L(r0 + r, k) * Linv(k, c0 + c)
      {
        const int r = tid & 31, cb = tid >> 5;  // columns cb + 8q
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = c0; k < r0; ++k) {
          const double a = A[k * kLDA + r0 + r];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] += a * T[(cb + 8 * q) * kLDA + k];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) S[(cb + 8 * q) * 33 + r] = acc[q];
      }
      __syncthreads();
      const double* Di = Dinv + ib * kSB * 33;
      {
        const int r = tid & 31, cb = tid >> 5;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int t = 0; t <= r; ++t) {
          const double d = Di[t * 33 + r];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] += d * S[(cb + 8 * q) * 33 + t];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) T[(cb + 8 * q) * kLDA + r0 + r] = -acc[q];
      }
      __syncthreads();
    }
    // Winv(c0 + c, row) = Linv(row, c0 + c)
    for (int idx = tid; idx < kSB * nb; idx += kDiagThreads) {
      const int c = idx & 31, row = idx >> 5;
      if (c0 + c < nb) Winv[(c0 + c) + (int64_t)row * ldwi] = (row >= c0 + c) ? T[c * kLDA + row] : 0.0;
    }
    __syncthreads();
  }
}

void launch_diag(Ctx& ctx, const DMat& Zkk, const DMat& Wkk, const DMat& Wikk) {
  const size_t smem = (size_t)(128 * kLDA + 4 * kSB * 33 + kSB * kLDA + kSB * 33) * 8;
  static bool set = false;
  if (!set) {
    QDWHG_CUDA(cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    set = true;
  }
  potrf_diag_kernel<<<1, kDiagThreads, smem, ctx.stream>>>(Zkk.ptr(), Zkk.ld, Wkk.ptr(), Wkk.ld,
                                                           Wikk.ptr(), Wikk.ld, (int)Zkk.rows,
                                                           ctx.dflag);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void trtri_rec(Ctx& ctx, const DMat& W, const DMat& Winv, int64_t r0, int64_t n, int nb) {
  if (n <= nb) return;
  int64_t n1 = ((n / 2 + nb - 1) / nb) * nb;
  if (n1 >= n) n1 = n - nb;
  const int64_t n2 = n - n1;
  trtri_rec(ctx, W, Winv, r0, n1, nb);
  trtri_rec(ctx, W, Winv, r0 + n1, n2, nb);
  const Arena::Mark mark = ctx.arena->mark();
  DMat T = ctx.arena->alloc(n1, n2);
  GemmExtra e1;
  e1.krange = KRange::BUpper;  // B = W22^-1 upper
  gemm(ctx, Op::N, Op::N, 1.0, W.sub(r0, r0 + n1, n1, n2), Winv.sub(r0 + n1, r0 + n1, n2, n2), 0.0,
       T, e1);
  GemmExtra e2;
  e2.krange = KRange::AUpper;  // A = W11^-1 upper
  gemm(ctx, Op::N, Op::N, -1.0, Winv.sub(r0, r0, n1, n1), T, 0.0, Winv.sub(r0, r0 + n1, n1, n2),
       e2);
  ctx.arena->release_to(mark);
}

// Same recursion, level by level for n = nb * 2^L: all merges of one level are
// independent, so each level is two batched GEMM launches instead of 2 * pairs.
void trtri_levels(Ctx& ctx, const DMat& W, const DMat& Winv, int64_t n, int nb) {
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
    gemm(ctx, Op::N, Op::N, 1.0, W.sub(0, h, h, h), Winv.sub(h, h, h, h), 0.0, T.sub(0, 0, h, h), e1);
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
  static bool set = false;
  if (!set) {
    QDWHG_CUDA(cudaFuncSetAttribute(panel_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)((128 * 129 + 128 * 65) * 8)));
    set = true;
  }
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
                  int nb) {
  if (n <= nb) {
    launch_diag(ctx, Z.sub(r0, r0, n, n), W.sub(r0, r0, n, n), Winv.sub(r0, r0, n, n));
    return;
  }
  int64_t n1 = ((n / 2 + nb - 1) / nb) * nb;
  if (n1 >= n) n1 = n - nb;
  const int64_t n2 = n - n1;
  chol_inv_rec(ctx, Z, W, Winv, r0, n1, nb);
  const int64_t r1 = r0 + n1;
  GemmExtra e1;
  e1.krange = KRange::ALower;  // op(A) = W11^-T lower
  gemm(ctx, Op::T, Op::T, 1.0, Winv.sub(r0, r0, n1, n1), Z.sub(r1, r0, n2, n1), 0.0,
       W.sub(r0, r1, n1, n2), e1);
  GemmExtra e2;
  e2.out = OutMode::Lower;
  const DMat W12 = W.sub(r0, r1, n1, n2);
  gemm(ctx, Op::T, Op::N, -1.0, W12, W12, 1.0, Z.sub(r1, r1, n2, n2), e2);
  chol_inv_rec(ctx, Z, W, Winv, r1, n2, nb);
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

void potrf_upper_and_inverse(Ctx& ctx, const DMat& Z, const DMat& Winv, bool want_w, bool stable) {
  const int64_t n = Z.rows;
  if (Z.cols != n) throw InvalidArgument("cholesky: matrix not square");
  static const int nb_env = getenv("QDWHG_POTRF_NB") ? atoi(getenv("QDWHG_POTRF_NB")) : 0;
  const int nb = (nb_env == 32 || nb_env == 64 || nb_env == 96 || nb_env == 128) ? nb_env : 128;
  QDWHG_CUDA(cudaMemsetAsync(ctx.dflag, 0, sizeof(int), ctx.stream));
  const Arena::Mark mark = ctx.arena->mark();
  DMat W = ctx.arena->alloc(n, n);
  fill(ctx, W, 0.0, 0.0);
  fill(ctx, Winv, 0.0, 0.0);
  if (!stable) {
    chol_inv_rec(ctx, Z, W, Winv, 0, n, nb);
  } else {
    // right-looking, panel by forward substitution (no explicit inverse in the
    // factorisation: backward stable like the reference's dot-product Cholesky)
    for (int64_t k = 0; k < n; k += nb) {
      const int64_t b = std::min<int64_t>(nb, n - k);
      const int64_t rest = n - k - b;
      launch_diag(ctx, Z.sub(k, k, b, b), W.sub(k, k, b, b), Winv.sub(k, k, b, b));
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
