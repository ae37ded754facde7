// Device building blocks of the 128 x 128 Cholesky-and-inverse leaf, shared by
// the stand-alone leaf kernel (potrf.cu: potrf_diag_kernel) and the tile-DAG
// Cholesky (chol_dag.cu).  256 threads; the block lives in shared memory,
// column-major with leading dimension kLDA, lower triangle = L (then L^{-1}).
#pragma once
#include "common.cuh"

namespace qdwhg {
#ifndef QDWHG_LEAF_MARK
#define QDWHG_LEAF_MARK(i)
#endif
#ifndef QDWHG_LEAF_MARK_T
#define QDWHG_LEAF_MARK_T(i, t)
#endif
namespace leaf {

constexpr int kThreads = 256;
constexpr int kDiagThreads = kThreads;
// 1/sqrt(d) without the libdevice slow-path call (which forces the unrolled
// register row to the stack): hardware double-precision estimate
// (rsqrt.approx.f64) refined by one third-order step.  Non-positive d returns NaN
// (the caller flags it).
QDWHG_DEV double rsqrt_newton(double d) {
  // branch-free (a branch here splits the unrolled Cholesky step into basic
  // blocks and stops the scheduler from hiding this chain behind the updates)
  // One third-order step from the ~2^-20 hardware estimate: with
  // e = 1 - d y^2, y' = y + y e (1/2 + 3/8 e) (error 5/16 e^3 < 2^-56),
  // dependency depth 4 instead of 6 for two Newton steps.
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;\n" : "=d"(y) : "d"(d));
  const double e = fma(-d * y, y, 1.0);
  const double p = fma(e, 0.375, 0.5);
  y = fma(y * e, p, y);
  return (d > 0.0) ? y : __longlong_as_double(0x7ff8000000000000ll);
}
constexpr int kSB = 32;          // sub-block handled by one warp
// padded smem leading dimension: 132 = 4 (mod 16) makes the DMMA fragment loads
// (8 rows x 4 k, or 4 k x 8 columns, one double per lane) bank-conflict free
constexpr int kLDA = 132;

// One right-looking Cholesky column step of a 32x32 block held as one row per
// lane (template recursion: compile-time register indices).  The pivot comes
// by one shuffle; the scaled column J goes to shared memory (its final place
// in L) and every lane reads the entries it needs as broadcast loads — half
// the instructions of shuffling each double.
template <int J>
struct CholStep {
  // djj: the pivot L_JJ^2, already broadcast by the previous step (look-ahead)
  static QDWHG_DEV void run(double (&row)[kSB], double* L, int lane, bool& bad, double& my_inv,
                            double djj) {
    if (!(djj > 0.0)) bad = true;
    const double inv = rsqrt_newton(djj);
    if (lane > J) row[J] *= inv;
    if (lane == J) {
      row[J] = djj * inv;
      my_inv = inv;
    }
    // look-ahead: lane J+1 updates its own diagonal from its own register
    // (same fma as the loop below) and broadcasts the next pivot right away, so
    // the next step's rsqrt does not wait for the shared-memory round trip
    double dnext = 0.0;
    if (J + 1 < kSB) dnext = __shfl_sync(0xffffffffu, fma(-row[J], row[J], row[(J + 1) % kSB]), (J + 1) % kSB);
    if (lane >= J) L[J * kLDA + lane] = row[J];
    __syncwarp();
    // unpredicated: entries above a lane's diagonal pick up junk that is never
    // read (the pivot and the written column only use entries on/below it)
#pragma unroll
    for (int c = J + 1; c < kSB; ++c) row[c] -= row[J] * L[J * kLDA + c];
    CholStep<J + 1>::run(row, L, lane, bad, my_inv, dnext);
  }
};
template <>
struct CholStep<kSB> {
  static QDWHG_DEV void run(double (&)[kSB], double*, int, bool&, double&, double) {}
};

// D^{-1} of a factored 32x32 lower block by forward substitution, one warp,
// lane j computing column j in registers (x[i] = 0 above the diagonal)
QDWHG_DEV void block_inverse(const double* Lb, const double* sinv, int lane, double (&x)[kSB]) {
#pragma unroll
  for (int i = 0; i < kSB; ++i) {
    double s[4] = {(i == lane) ? 1.0 : 0.0, 0.0, 0.0, 0.0};  // 4 chains
#pragma unroll
    for (int k = 0; k < i; ++k) s[k & 3] -= Lb[k * kLDA + i] * x[k];  // x[k] == 0 for k < lane
    x[i] = (i >= lane) ? ((s[0] + s[1]) + (s[2] + s[3])) * sinv[i] : 0.0;
  }
}

constexpr int kLDT = 68;  // T (<= 64 x 64, the doubling products' scratch) leading dimension
// shared-memory doubles used by factor + invert: A (128 x kLDA), T (64 x kLDT), Sinv (128)
constexpr int kSmemDoubles = 128 * kLDA + 64 * kLDT + 128;

// Right-looking blocked Cholesky of the nbp x nbp lower block in A (strict upper
// zero; nbp a multiple of 32, <= 128): L in place, Sinv[i] = 1 / L_ii.  A
// non-positive pivot sets *bad_s.  Per 32-column step: warp 0 factors the
// diagonal block in registers, the panel rows below by forward substitution (one
// row per thread), the trailing lower triangle by a rank-32 DMMA update.
QDWHG_DEV void factor(double* A, double* Sinv, int nbp, int* bad_s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;  // DMMA fragment coordinates
  const int nsb = nbp / kSB;
  for (int kb = 0; kb < nsb; ++kb) {
    const int b0 = kb * kSB;
    if (warp == 0) {
      // ---- factor the 32x32 diagonal block in registers: lane i owns row i.
      // No division/sqrt library calls in here (their slow-path CALL would push
      // the unrolled register rows to the stack): pivots use rsqrt_newton.
      double row[kSB];
#pragma unroll
      for (int c = 0; c < kSB; ++c) row[c] = A[(b0 + c) * kLDA + b0 + lane];  // strict upper is 0
      bool bad = false;
      double my_inv = 0.0;
      CholStep<0>::run(row, A + b0 * kLDA + b0, lane, bad, my_inv,
                       __shfl_sync(0xffffffffu, row[0], 0));  // writes L in place
      if (bad && lane == 0) *bad_s = 1;
      Sinv[b0 + lane] = my_inv;
    }
    __syncthreads();
    const int p0 = b0 + kSB, R = nbp - p0;
    if (R > 0) {
      // ---- panel rows by forward substitution, one row per thread:
      // L(i, b0+c) = (Z(i, b0+c) - sum_{t<c} L(i, b0+t) L(b0+c, b0+t)) / L(b0+c, b0+c)
      if (tid < R) {
        const int i = p0 + tid;
        double x[kSB];
#pragma unroll
        for (int c = 0; c < kSB; ++c) x[c] = A[(b0 + c) * kLDA + i];
#pragma unroll
        for (int c = 0; c < kSB; ++c) {
          double s0 = x[c], s1 = 0.0;  // two chains: half the FMA latency
#pragma unroll
          for (int t = 0; t < c; ++t) {
            const double l = A[(b0 + t) * kLDA + b0 + c];  // broadcast
            if (t & 1) s1 -= x[t] * l;
            else s0 -= x[t] * l;
          }
          x[c] = (s0 + s1) * Sinv[b0 + c];
        }
#pragma unroll
        for (int c = 0; c < kSB; ++c) A[(b0 + c) * kLDA + i] = x[c];
      }
      __syncthreads();
      // ---- trailing rank-32 update of the lower triangle on 8x8 DMMA tiles:
      // A(i, j) -= sum_t L(i, b0+t) L(j, b0+t),  i >= j >= p0.  A work unit is
      // one row tile x up to 4 column tiles (4 independent accumulator chains).
      const int nt = R / 8;
      int nunits = 0;
      for (int ti = 0; ti < nt; ++ti) nunits += ti / 4 + 1;
      for (int u = warp; u < nunits; u += kDiagThreads / 32) {
        int ti = 0, rem = u;
        while (rem >= ti / 4 + 1) {
          rem -= ti / 4 + 1;
          ++ti;
        }
        const int tj0 = 4 * rem;
        const int i0 = p0 + 8 * ti;
        double c[4][2];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int j0 = p0 + 8 * min(tj0 + v, ti);
          c[v][0] = A[(j0 + 2 * q) * kLDA + i0 + g];
          c[v][1] = A[(j0 + 2 * q + 1) * kLDA + i0 + g];
        }
#pragma unroll
        for (int k4 = 0; k4 < kSB / 4; ++k4) {
          const double* lc = A + (b0 + 4 * k4 + q) * kLDA;
          const double a = -lc[i0 + g];
#pragma unroll
          for (int v = 0; v < 4; ++v)
            dmma_8x8x4(c[v][0], c[v][1], a, lc[p0 + 8 * min(tj0 + v, ti) + g]);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int tj = tj0 + v;
          if (tj > ti) break;
          const int j0 = p0 + 8 * tj;
          if (tj != ti || g >= 2 * q) A[(j0 + 2 * q) * kLDA + i0 + g] = c[v][0];
          if (tj != ti || g >= 2 * q + 1) A[(j0 + 2 * q + 1) * kLDA + i0 + g] = c[v][1];
        }
      }
      __syncthreads();
    }
  }
}

// L^{-1} in place (lower) from the factored block: the 32x32 diagonal-block
// inverses in parallel (one warp each), then recursive doubling over the
// diagonal blocks, L^{-1}_QP = -Q^{-1} (L_QP P^{-1}), on DMMA tiles (T scratch).
QDWHG_DEV void invert(double* A, double* T, const double* Sinv, int nbp) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int nsb = nbp / kSB;
  // ---- D_kb^{-1} (lower 32x32) of every diagonal block, one warp each, in place
  if (warp < nsb) {
    const int b0 = warp * kSB;
    double x[kSB];
    block_inverse(A + b0 * kLDA + b0, Sinv + b0, lane, x);
    __syncwarp();
    double* D = A + (b0 + lane) * kLDA + b0;  // column lane of the block (zeros above)
#pragma unroll
    for (int i = 0; i < kSB; ++i) D[i] = x[i];
  }
  __syncthreads();

  // ---- L^{-1} by recursive doubling over the diagonal blocks: for each pair of
  // adjacent groups (P = [a0, a0+h), Q = [a0+h, a0+2h)) with P^{-1}, Q^{-1} in
  // place:  L^{-1}_QP = -Q^{-1} (L_QP P^{-1}).  Two levels for nb = 128, each
  // two DMMA products over all pairs at once (a unit = one 8-row tile x 32 columns).
  for (int h = kSB; h < nbp; h *= 2) {
    const int npairs = (nbp - h + 2 * h - 1) / (2 * h);  // pairs with a non-empty Q
    const int cgs = h / kSB;                             // 32-column groups per pair
    int units = 0;
    for (int p = 0; p < npairs; ++p) units += min(h, nbp - (2 * p + 1) * h) / 8 * cgs;
    // phase 1: T_p = L_QP * P^{-1}   (P^{-1} lower: k >= column)
    for (int u = warp; u < units; u += kDiagThreads / 32) {
      int p = 0, rem = u;
      while (rem >= min(h, nbp - (2 * p + 1) * h) / 8 * cgs) {
        rem -= min(h, nbp - (2 * p + 1) * h) / 8 * cgs;
        ++p;
      }
      const int ti = rem / cgs, cg = rem % cgs;
      const int a0 = 2 * p * h, q0 = a0 + h;
      double c[4][2] = {};
      for (int k4 = 8 * cg; k4 < h / 4; ++k4) {
        const int k = a0 + 4 * k4 + q;
        const double a = A[k * kLDA + q0 + 8 * ti + g];
#pragma unroll
        for (int tj = 0; tj < 4; ++tj)
          dmma_8x8x4(c[tj][0], c[tj][1], a, A[(a0 + kSB * cg + 8 * tj + g) * kLDA + k]);
      }
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) {
        const int col = p * h + kSB * cg + 8 * tj + 2 * q;
        T[col * kLDT + 8 * ti + g] = c[tj][0];
        T[(col + 1) * kLDT + 8 * ti + g] = c[tj][1];
      }
    }
    __syncthreads();
    // phase 2: L^{-1}_QP = -Q^{-1} T_p   (Q^{-1} lower: k <= row), heaviest rows first
    for (int u = warp; u < units; u += kDiagThreads / 32) {
      int p = 0, rem = u;
      while (rem >= min(h, nbp - (2 * p + 1) * h) / 8 * cgs) {
        rem -= min(h, nbp - (2 * p + 1) * h) / 8 * cgs;
        ++p;
      }
      const int nti = min(h, nbp - (2 * p + 1) * h) / 8;
      const int ti = nti - 1 - rem / cgs, cg = rem % cgs;
      const int a0 = 2 * p * h, q0 = a0 + h;
      double c[4][2] = {};
      for (int k4 = 0; k4 < 2 * (ti + 1); ++k4) {
        const int k = 4 * k4 + q;
        const double a = -A[(q0 + k) * kLDA + q0 + 8 * ti + g];
#pragma unroll
        for (int tj = 0; tj < 4; ++tj)
          dmma_8x8x4(c[tj][0], c[tj][1], a, T[(p * h + kSB * cg + 8 * tj + g) * kLDT + k]);
      }
#pragma unroll
      for (int tj = 0; tj < 4; ++tj) {
        const int col = a0 + kSB * cg + 8 * tj + 2 * q;
        A[col * kLDA + q0 + 8 * ti + g] = c[tj][0];
        A[(col + 1) * kLDA + q0 + 8 * ti + g] = c[tj][1];
      }
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// Fused, software-pipelined factor-and-invert of a 128 x 128 tile for the fast
// path (kappa(Z) small: the QDWH step's Z = I + c X^T X, Gram matrices of
// well-conditioned blocks).  Same result as factor() + invert() up to rounding,
// but the latency-bound chain of the four 32 x 32 diagonal-block factorisations
// is the only thing left on the critical path:
//   * warp 0 factors diagonal block kb in registers (the plain right-looking
//     Cholesky: 6.2K cycles, the pivot chain) and publishes its columns four at a
//     time on mbarriers; the helper warp (warp 1, another SM sub-partition) applies
//     the same column operations to the identity right behind it — lane i holds
//     row i of U = L^{-T} — and writes D_kb^{-1} over the block ~0.7K cycles after
//     warp 0 is done.  (Both in warp 0 — one register array serves the row of L
//     below the diagonal and the row of U from it on, but U's part must be zeroed
//     at every step — measured 8.2K cycles per block.)
//   * the panel below is one DMMA product with D_kb^{-T} (no forward
//     substitution), the next diagonal block's update runs first (all warps,
//     ~2 x 400 cycles), then warp 0 goes on with block kb + 1;
//   * meanwhile warps 2, 3, 5, 6, 7 (warp 4 shares warp 0's sub-partition and FP64
//     pipe: it only joins the all-warp phases) finish the trailing update and
//     build block row kb of L^{-1}:  S_kb,j = sum_m L_kb,m X_m,j (ahead of D_kb),
//     X_kb,j = -D_kb^{-1} S_kb,j, in place over the dead L blocks.  This
//     background (DMMA-issue bound on three sub-partitions, ~8K cycles) is now what
//     a block step waits for, not warp 0.
// A: 128 x kLDA tile (lower triangle = Z, strict upper zero) -> L^{-1} (lower,
// strict upper zero).  S: 192 x kLDS scratch.  256 threads, barriers 1 and 2.
constexpr int kLDS = 36;  // = 4 (mod 16): conflict-free DMMA fragment loads
constexpr int kFusedSmemDoubles = 128 * kLDA + 192 * kLDS;

QDWHG_DEV void bar_all() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }
QDWHG_DEV void bar_workers() { asm volatile("bar.sync 2, 160;\n" ::: "memory"); }  // warps 2, 3, 5, 6, 7

// L(r0 .. r0+8, b0 .. b0+32) = Z(same) * D^{-T}, D^{-1} lower in the diagonal block at b0
QDWHG_DEV void fused_panel_tile(double* A, int b0, int r0, int g, int q) {
  double c[4][2] = {};
#pragma unroll
  for (int k4 = 0; k4 < kSB / 4; ++k4) {
    const double* col = A + (b0 + 4 * k4 + q) * kLDA;
    const double a = col[r0 + g];
#pragma unroll
    for (int tj = 0; tj < 4; ++tj)
      if (k4 <= 2 * tj + 1) dmma_8x8x4(c[tj][0], c[tj][1], a, col[b0 + 8 * tj + g]);
  }
  __syncwarp();
#pragma unroll
  for (int tj = 0; tj < 4; ++tj) {
    A[(b0 + 8 * tj + 2 * q) * kLDA + r0 + g] = c[tj][0];
    A[(b0 + 8 * tj + 2 * q + 1) * kLDA + r0 + g] = c[tj][1];
  }
}

// rank-32 update of one 8 x 8 tile (ti >= tj) of the trailing lower triangle at p0
QDWHG_DEV void fused_update_tile(double* A, int b0, int p0, int ti, int tj, int g, int q) {
  const int i0 = p0 + 8 * ti, j0 = p0 + 8 * tj;
  double c0 = A[(j0 + 2 * q) * kLDA + i0 + g], c1 = A[(j0 + 2 * q + 1) * kLDA + i0 + g];
#pragma unroll
  for (int k4 = 0; k4 < kSB / 4; ++k4) {
    const double* lc = A + (b0 + 4 * k4 + q) * kLDA;
    dmma_8x8x4(c0, c1, -lc[i0 + g], lc[j0 + g]);
  }
  if (ti != tj || g >= 2 * q) A[(j0 + 2 * q) * kLDA + i0 + g] = c0;
  if (ti != tj || g >= 2 * q + 1) A[(j0 + 2 * q + 1) * kLDA + i0 + g] = c1;
}

// trailing update of the rows below the next diagonal block (row tiles >= 4 of
// the trailing matrix at p0), units of one row tile x up to 4 column tiles; a warp
// runs two units at a time (eight accumulator chains: the 8-step DMMA chains are
// latency-bound, ~100 cycles a step)
QDWHG_DEV void fused_rest_update(double* A, int b0, int p0, int nt, int w, int nw, int g, int q) {
  int nunits = 0;
  for (int ti = 4; ti < nt; ++ti) nunits += ti / 4 + 1;
  for (int u0 = w; u0 < nunits; u0 += 2 * nw) {
    int ti[2], tj0[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int rem = min(u0 + h * nw, nunits - 1);  // (a missing second unit repeats the last one: not stored)
      int t = 4;
      while (rem >= t / 4 + 1) {
        rem -= t / 4 + 1;
        ++t;
      }
      ti[h] = t;
      tj0[h] = 4 * rem;
    }
    const bool two = u0 + nw < nunits;
    double c[2][4][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i0 = p0 + 8 * ti[h], j0 = p0 + 8 * min(tj0[h] + v, ti[h]);
        c[h][v][0] = A[(j0 + 2 * q) * kLDA + i0 + g];
        c[h][v][1] = A[(j0 + 2 * q + 1) * kLDA + i0 + g];
      }
#pragma unroll
    for (int k4 = 0; k4 < kSB / 4; ++k4) {
      const double* lc = A + (b0 + 4 * k4 + q) * kLDA;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double a = -lc[p0 + 8 * ti[h] + g];
#pragma unroll
        for (int v = 0; v < 4; ++v)
          dmma_8x8x4(c[h][v][0], c[h][v][1], a, lc[p0 + 8 * min(tj0[h] + v, ti[h]) + g]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && !two) break;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int tj = tj0[h] + v;
        if (tj > ti[h]) break;
        const int i0 = p0 + 8 * ti[h], j0 = p0 + 8 * tj;
        if (tj != ti[h] || g >= 2 * q) A[(j0 + 2 * q) * kLDA + i0 + g] = c[h][v][0];
        if (tj != ti[h] || g >= 2 * q + 1) A[(j0 + 2 * q + 1) * kLDA + i0 + g] = c[h][v][1];
      }
    }
  }
}

// S_kn,j = sum_{m = j}^{kn-1} L_kn,m X_m,j for j < kn (X = L^{-1}: diagonal blocks
// D_m^{-1}, finished rows below), into Sk (32 rows x 32 kn columns).  Units of one
// 8-row tile x 16 columns, heaviest (smallest j) first.
QDWHG_DEV void fused_inv_sums(const double* A, double* Sk, int kn, int w, int nw, int g, int q) {
  const int nunits = kn * 8;
  for (int u = w; u < nunits; u += nw) {
    const int j = u >> 3, ri = (u & 7) >> 1, h = u & 1;
    const int c0 = kSB * j + 16 * h;
    double c[2][2] = {};
    for (int k4 = 8 * j + 4 * h; k4 < 8 * kn; ++k4) {
      const int k = 4 * k4 + q;
      const double a = A[k * kLDA + kSB * kn + 8 * ri + g];
#pragma unroll
      for (int v = 0; v < 2; ++v) dmma_8x8x4(c[v][0], c[v][1], a, A[(c0 + 8 * v + g) * kLDA + k]);
    }
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      Sk[(c0 + 8 * v + 2 * q) * kLDS + 8 * ri + g] = c[v][0];
      Sk[(c0 + 8 * v + 2 * q + 1) * kLDS + 8 * ri + g] = c[v][1];
    }
  }
}

// X_kb,j = -D_kb^{-1} S_kb,j for j < kb, in place over block row kb of A.  Units
// of one 8-row tile x 8 NV columns, heaviest (last row tile) first.
template <int NV>
QDWHG_DEV void fused_inv_rows(double* A, const double* Sk, int kb, int w, int nw, int g, int q) {
  const int b0 = kSB * kb, ncg = 4 * kb / NV;
  for (int u = w; u < 4 * ncg; u += nw) {
    const int ri = 3 - u / ncg, cg = u % ncg;
    double c[NV][2] = {};
#pragma unroll 2
    for (int k4 = 0; k4 <= 2 * ri + 1; ++k4) {
      const int k = 4 * k4 + q;
      const double a = -A[(b0 + k) * kLDA + b0 + 8 * ri + g];
#pragma unroll
      for (int v = 0; v < NV; ++v)
        dmma_8x8x4(c[v][0], c[v][1], a, Sk[(8 * NV * cg + 8 * v + g) * kLDS + k]);
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      A[(8 * NV * cg + 8 * v + 2 * q) * kLDA + b0 + 8 * ri + g] = c[v][0];
      A[(8 * NV * cg + 8 * v + 2 * q + 1) * kLDA + b0 + 8 * ri + g] = c[v][1];
    }
  }
}

QDWHG_DEV double* fused_s_region(double* S, int kb) {  // S_kb: 32 kb columns after S_1 .. S_kb-1
  return S + kLDS * kSB * (kb * (kb - 1) / 2);
}

// Plain right-looking Cholesky step of warp 0 (as CholStep) that also leaves
// 1 / L_JJ in sinv[J] and publishes its progress every four columns (one mbarrier
// per group of four, a phase per block: release / acquire at CTA scope; a
// st.release flag cost 100 cycles per column): the helper warp applies the same column operations to the identity right behind it.
// (sinv / prog as 32-bit shared-window addresses: through generic pointers each
// step's store first converts the address — an S2R the in-order warp waits on —
// and the block took 8.9K cycles instead of 5.7K)
QDWHG_DEV void sts_f64(uint32_t addr, double x) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(addr), "d"(x));
}
QDWHG_DEV void mbar_arrive_s(uint32_t addr) {
  asm volatile("{\n.reg .b64 t;\nmbarrier.arrive.shared::cta.b64 t, [%0];\n}\n" ::"r"(addr) : "memory");
}
template <int J>
struct CholPubStep {
  static QDWHG_DEV void run(double (&row)[kSB], double* L, uint32_t sinv, uint32_t prog, int lane,
                            bool& bad, double djj) {
    if (!(djj > 0.0)) bad = true;
    const double inv = rsqrt_newton(djj);
    if (lane > J) row[J] *= inv;
    if (lane == J) row[J] = djj * inv;
    sts_f64(sinv + 8 * J, inv);  // every lane, same value: no branch in the step
    double dnext = 0.0;
    if (J + 1 < kSB) dnext = __shfl_sync(0xffffffffu, fma(-row[J], row[J], row[(J + 1) % kSB]), (J + 1) % kSB);
    if (lane >= J) L[J * kLDA + lane] = row[J];
    __syncwarp();
    if ((J & 3) == 3) mbar_arrive_s(prog + 8 * (J >> 2));  // columns J-3 .. J are out (32 arrivals)
#pragma unroll
    for (int c = J + 1; c < kSB; ++c) row[c] -= row[J] * L[J * kLDA + c];
    CholPubStep<J + 1>::run(row, L, sinv, prog, lane, bad, dnext);
  }
};
template <>
struct CholPubStep<kSB> {
  static QDWHG_DEV void run(double (&)[kSB], double*, uint32_t, uint32_t, int, bool&, double) {}
};

// Warp 0's part of a block step, as a function of its own: its 32-step unrolled
// chain is sensitive to register allocation, and inlined into the 255-register
// kernels any edit elsewhere reshuffles it (measured 8.2K <-> 10.2K cycles per block).
// It only factors (5.7K cycles: the pivot chain); D^{-1} comes from the helper warp.
// (Both in this warp: one pass, the inverse rows' registers zeroed at each step,
// 8.2K; two passes 9.7K.)
static __device__ __noinline__ void fused_factor_block(double* Ablk, uint32_t sinv, uint32_t prog, int lane,
                                                       int* bad_s) {
  __builtin_assume(__isShared(Ablk));  // not inlined: keep the column broadcasts LDS
  double v[kSB];
#pragma unroll
  for (int c = 0; c < kSB; ++c) v[c] = Ablk[c * kLDA + lane];
  bool bad = false;
  CholPubStep<0>::run(v, Ablk, sinv, prog, lane, bad, __shfl_sync(0xffffffffu, v[0], 0));
  if (bad && lane == 0) *bad_s = 1;
}

// The helper warp (warp 4, warp 0's neighbour on its SM sub-partition): row
// `lane` of U = L^{-T} by the column operations of the factorisation applied to
// the identity, four columns behind warp 0; then D^{-1} over the block (warp 0 is
// done with it: all eight groups are out).
static __device__ __noinline__ void fused_inverse_block(double* Ablk, const double* sinv, uint64_t* prog,
                                                        uint32_t parity, int lane) {
  __builtin_assume(__isShared(Ablk));
  __builtin_assume(__isShared(sinv));
  __builtin_assume(__isShared(prog));
  double u[kSB];
#pragma unroll
  for (int c = 0; c < kSB; ++c) u[c] = (c == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int J = 0; J < kSB; ++J) {
    if ((J & 3) == 0) mbar_wait(&prog[J >> 2], parity);
    u[J] *= sinv[J];
#pragma unroll
    for (int c = J + 1; c < kSB; ++c) u[c] = fma(-u[J], Ablk[J * kLDA + c], u[c]);
  }
  __syncwarp();
  double* D = Ablk + lane * kLDA;  // column `lane` of D^{-1}: U(lane, c) = D^{-1}(c, lane)
#pragma unroll
  for (int c = 0; c < kSB; ++c)
    if (c >= lane) D[c] = u[c];
}

QDWHG_DEV void factor_invert_fused(double* A, double* S, int* bad_s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  // warp 0 factors, warp 1 (another SM sub-partition: on warp 0's own, warp 4, it
  // slowed the pivot chain from 5.7K to 9.4K cycles) inverts behind it, warp 4 only
  // joins the all-warp phases, warps 2, 3, 5, 6, 7 are the background workers
  constexpr int NA = 5;
  const int ai = (warp == 2 || warp == 3) ? warp - 2 : (warp >= 5 ? warp - 3 : -1);
  constexpr int nblk = 128 / kSB;
  __shared__ double s_sinv[kSB];
  __shared__ uint64_t s_prog[kSB / 4];
  if (tid == 0) {
    for (int i = 0; i < kSB / 4; ++i) mbar_init(&s_prog[i], 32);
    fence_barrier_init();
  }
  bar_all();
#pragma unroll 1
  for (int kb = 0; kb < nblk; ++kb) {
    const int b0 = kSB * kb, p0 = b0 + kSB, R = 128 - p0;
    if (warp == 0) {
      fused_factor_block(A + b0 * kLDA + b0, smem_u32(s_sinv), smem_u32(s_prog), lane, bad_s);
      QDWHG_LEAF_MARK(24 + 4 * kb);
    } else if (warp == 1) {
      fused_inverse_block(A + b0 * kLDA + b0, s_sinv, s_prog, (uint32_t)(kb & 1), lane);
      QDWHG_LEAF_MARK_T(40 + kb, 32);
    } else if (kb > 0 && warp != 4) {
      // ---- background of step kp = kb - 1, while warp 0 factors block kb
      const int kp = kb - 1, pb0 = kSB * kp, pp0 = pb0 + kSB, pnt = (128 - pp0) / 8;
      if (ai >= 0) {
        for (int t = 8 + ai; t < pnt; t += NA) fused_panel_tile(A, pb0, pp0 + 8 * t, g, q);
        if (kp > 0) fused_inv_rows<2>(A, fused_s_region(S, kp), kp, ai, NA, g, q);
      }
      if (kb == 1) { QDWHG_LEAF_MARK_T(60, 64); }
      bar_workers();
      if (kb == 1) { QDWHG_LEAF_MARK_T(61, 64); }
      if (ai >= 0) {
        fused_rest_update(A, pb0, pp0, pnt, ai, NA, g, q);
        if (kb == 1) { QDWHG_LEAF_MARK_T(62, 64); }
        fused_inv_sums(A, fused_s_region(S, kb), kb, ai, NA, g, q);
        if (kb == 1) { QDWHG_LEAF_MARK_T(63, 64); }
      }
    }
    bar_all();
    QDWHG_LEAF_MARK(25 + 4 * kb);
    if (R > 0) {
      // ---- panel row tiles 0-7 (0-3 feed the next diagonal block), one per warp
      if (8 * warp < R) fused_panel_tile(A, b0, p0 + 8 * warp, g, q);
      QDWHG_LEAF_MARK_T(44 + kb, 32);
      QDWHG_LEAF_MARK_T(48 + kb, 64);
      QDWHG_LEAF_MARK_T(52 + kb, 128);
      QDWHG_LEAF_MARK_T(56 + kb, 224);
      bar_all();
      QDWHG_LEAF_MARK(26 + 4 * kb);
      // ---- next diagonal block's rank-32 update: 10 tiles over 8 warps
      {
        // tile u -> (ti, tj), row-major over the lower triangle: u = ti (ti + 1) / 2 + tj
        const int ti = (warp >= 6) ? 3 : (warp >= 3) ? 2 : (warp >= 1) ? 1 : 0;
        fused_update_tile(A, b0, p0, ti, warp - ti * (ti + 1) / 2, g, q);
        if (warp == 2 || warp == 3) fused_update_tile(A, b0, p0, 3, warp, g, q);  // u = 8, 9
      }
      bar_all();
      QDWHG_LEAF_MARK(27 + 4 * kb);
    }
  }
  // ---- last block row of L^{-1}: S_3 is ready, D_3^{-1} just arrived
  fused_inv_rows<6>(A, fused_s_region(S, nblk - 1), nblk - 1, warp, 8, g, q);
  bar_all();
}

}  // namespace leaf
}  // namespace qdwhg
