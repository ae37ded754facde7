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
#include "common.cuh"
#include "internal.hpp"

namespace qdwhg {

namespace {

constexpr int kDiagThreads = 512;

// Factor the nb x nb block Zkk (symmetric; reads the lower triangle) -> W_kk
// (upper, written to W) and W_kk^{-1} (upper, written to Winv).
template <int NB>
__global__ void __launch_bounds__(kDiagThreads, 1)
    potrf_diag_kernel(const double* Z, int64_t ldz, double* W, int64_t ldw, double* Winv,
                      int64_t ldwi, int nb, int* flag) {
  extern __shared__ double sm[];
  constexpr int LDS = NB + 1;
  double* L = sm;                  // column-major L[c*LDS + r], lower
  double* X = sm + NB * LDS;       // inverse scratch: 64 columns X[g*LDS + r]
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kDiagThreads / 32;

  // load lower triangle (column-major, coalesced down columns)
  for (int c = warp; c < nb; c += NW)
    for (int r = lane; r < nb; r += 32) L[c * LDS + r] = (r >= c) ? Z[r + (int64_t)c * ldz] : 0.0;
  __syncthreads();

  // right-looking, one barrier per column: the trailing update of step j uses
  // the unscaled column j and the pivot d_j; column j-1 is scaled during step j.
  bool bad = false;
  for (int j = 0; j < nb; ++j) {
    const double d = L[j * LDS + j];
    if (!(d > 0.0)) bad = true;
    const double inv_d = 1.0 / d;
    if (j > 0) {
      const double sp = sqrt(L[(j - 1) * LDS + (j - 1)]);
      // scale column j-1 below the diagonal (not read in this step)
      for (int r = j + tid; r < nb; r += kDiagThreads) L[(j - 1) * LDS + r] /= sp;
    }
    for (int c = j + 1 + warp; c < nb; c += NW) {
      const double f = L[j * LDS + c] * inv_d;
      for (int r = c + lane; r < nb; r += 32) L[c * LDS + r] -= L[j * LDS + r] * f;
    }
    __syncthreads();
  }
  // last column has no sub-diagonal; now take sqrt of every pivot
  __syncthreads();
  for (int j = tid; j < nb; j += kDiagThreads) L[j * LDS + j] = sqrt(L[j * LDS + j]);
  __syncthreads();
  if (bad && lane == 0) atomicExch(flag, 1);

  // W_kk = L^T: W(r, c) = L(c, r) for r <= c
  for (int c = warp; c < nb; c += NW)
    for (int r = lane; r < nb; r += 32) W[r + (int64_t)c * ldw] = (r <= c) ? L[r * LDS + c] : 0.0;

  // Linv by forward substitution, 8 lanes per column of Linv (column j solves
  // L x = e_j); X holds the partial results.  Winv_kk = Linv^T.
  constexpr int G = 8;
  const int grp = tid / G, sub = tid % G;
  constexpr int NGRP = kDiagThreads / G;
  for (int j0 = 0; j0 < nb; j0 += NGRP) {
    const int j = j0 + grp;
    const bool live = j < nb;
    double* x = X + grp * LDS;
    // all groups of a warp walk the same i range so the warp stays converged
    for (int i = j0; i < nb; ++i) {
      const bool act = live && i >= j;
      double s = 0.0;
      if (act)
        for (int k = j + sub; k < i; k += G) s += L[k * LDS + i] * x[k];
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, G);
      if (act && sub == 0) x[i] = ((i == j ? 1.0 : 0.0) - s) / L[i * LDS + i];
      __syncwarp();
    }
    // Winv(j, i) = Linv(i, j) for i >= j  -> row j of Winv
    if (live)
      for (int i = sub; i < nb; i += G) Winv[j + (int64_t)i * ldwi] = (i >= j) ? x[i] : 0.0;
    __syncthreads();
  }
}

template <int NB>
void launch_diag(Ctx& ctx, const DMat& Zkk, const DMat& Wkk, const DMat& Wikk) {
  const size_t smem = (size_t)(NB + kDiagThreads / 8) * (NB + 1) * 8;
  static bool set = false;
  if (!set) {
    QDWHG_CUDA(cudaFuncSetAttribute(potrf_diag_kernel<NB>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = true;
  }
  potrf_diag_kernel<NB><<<1, kDiagThreads, smem, ctx.stream>>>(
      Zkk.ptr(), Zkk.ld, Wkk.ptr(), Wkk.ld, Wikk.ptr(), Wikk.ld, (int)Zkk.rows, ctx.dflag);
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

}  // namespace

void potrf_upper_and_inverse(Ctx& ctx, const DMat& Z, const DMat& Winv) {
  const int64_t n = Z.rows;
  if (Z.cols != n) throw InvalidArgument("cholesky: matrix not square");
  const int nb = n >= 1024 ? 128 : 64;
  QDWHG_CUDA(cudaMemsetAsync(ctx.dflag, 0, sizeof(int), ctx.stream));
  const Arena::Mark mark = ctx.arena->mark();
  DMat W = ctx.arena->alloc(n, n);
  fill(ctx, W, 0.0, 0.0);
  fill(ctx, Winv, 0.0, 0.0);
  for (int64_t k = 0; k < n; k += nb) {
    const int64_t b = std::min<int64_t>(nb, n - k);
    const int64_t rest = n - k - b;
    if (nb == 128)
      launch_diag<128>(ctx, Z.sub(k, k, b, b), W.sub(k, k, b, b), Winv.sub(k, k, b, b));
    else
      launch_diag<64>(ctx, Z.sub(k, k, b, b), W.sub(k, k, b, b), Winv.sub(k, k, b, b));
    if (rest > 0) {
      // W_k,rest = W_kk^{-T} Z_k,rest   (op(A) = Winv_kk^T is lower -> ALower)
      GemmExtra e1;
      e1.krange = KRange::ALower;
      gemm(ctx, Op::T, Op::N, 1.0, Winv.sub(k, k, b, b), Z.sub(k, k + b, b, rest), 0.0,
           W.sub(k, k + b, b, rest), e1);
      // Z_rest -= W_k,rest^T W_k,rest   (symmetric, lower tiles mirrored)
      GemmExtra e2;
      e2.out = OutMode::LowerMirror;
      const DMat Wp = W.sub(k, k + b, b, rest);
      gemm(ctx, Op::T, Op::N, -1.0, Wp, Wp, 1.0, Z.sub(k + b, k + b, rest, rest), e2);
    }
  }
  // pivot check before the inverse is trusted
  int hflag = 0;
  QDWHG_CUDA(cudaMemcpyAsync(&hflag, ctx.dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  if (hflag) {
    ctx.arena->release_to(mark);
    throw NotPositiveDefinite("cholesky: pivot is not positive");
  }
  trtri_rec(ctx, W, Winv, 0, n, nb);
  // hand W back in Z's upper triangle (zero strict lower) for callers that want it
  copy(ctx, W, Z);
  ctx.arena->release_to(mark);
}

}  // namespace qdwhg
