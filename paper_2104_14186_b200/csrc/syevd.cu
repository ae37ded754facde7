// Symmetric eigensolver for the large Rayleigh-Ritz blocks (ell in the
// thousands: partial.cpp:80-81 sym_eig_dense of Q2^T A Q2, and eig(H) of the
// polar-based SVD, fullsolve.cpp:82-103).  The reference uses cyclic Jacobi
// (kernels.cpp:148-215), which is hours at ell ~ 5000; the values/vectors are
// the same mathematical objects, computed here by
//   1. SYTRD  A = Q T Q^T, Householder, blocked (LAPACK dsytrd/dlatrd shape):
//      a cooperative panel kernel does the per-column work (column update with
//      the panel's V/W, reflector, SYMV of the stale trailing matrix + panel
//      corrections, w) with 4 grid barriers per column; the trailing update
//      A -= V W^T + W V^T is two DMMA GEMMs;
//   2. bisection (Sturm counts), one thread per eigenvalue -> ascending values
//      to ~u*||T||;
//   3. inverse iteration with partial pivoting (LAPACK dlagtf/dlagts shape),
//      one thread per eigenvector, vectors stored transposed for coalescing;
//   4. Lowdin orthogonalisation Z <- Z (I - E/2 + 3E^2/8), E = Z^T Z - I, for
//      the O(u*||T||/gap) inner-product defects of inverse iteration
//      (falls back to the QDWH divide-and-conquer if E is not small);
//   5. back-transform Z_A = Q Z with the compact-WY blocks (Gram + larft + GEMMs).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

namespace qdwhg {

void larft_launch(Ctx& ctx, const DMat& G, const double* tau_dev, const DMat& T);  // geqrf.cu

namespace {

#ifdef QDWHG_TRD_TRACE
__device__ long long g_trd_trace[16];
#define TRD_MARK(k, col) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && (col) == 5) g_trd_trace[k] = clock64()
#else
#define TRD_MARK(k, col)
#endif
constexpr int kTrdThreads = 512;
constexpr size_t kTrdDynSmem = (kTrdThreads / 32) * (32 * 33 + 64) * sizeof(double);
constexpr int kTrdNB = 32;


// Block-wide sum into one atomic on `dst` (skip zeros).
QDWHG_DEV void block_atomic_sum(double v, double* dst, double* scratch) {
  v = block_sum(v, scratch);
  if (threadIdx.x == 0 && v != 0.0) atomicAdd(dst, v);
  __syncthreads();
}

struct TrdArgs {
  double* A;  // n x n full symmetric (lower triangle used), ld
  int64_t lda;
  double* V;  // n x nb panel reflectors (unit at row c+1, zeros above)
  double* W;  // n x nb
  int64_t ldp;
  double* d;    // diag (n)
  double* e;    // sub-diagonal (n-1)
  double* tau;  // n
  double* y;    // n scratch (virtual-column dots t1/t2 at [m, m + 2i))
  double* ypart;  // SYMV tile partials: [TI][TI * 32] (TI = ceil(m / 32)), L2-resident
  double* red;  // 4 x 8 rotating reduction slots
  unsigned* bar;
  int n, j0, nb;
};

// One panel of dlatrd (lower).  Columns c = j0 .. j0+nb-1, three grid barriers
// per column:
//   A   a_c(r) -= sum_t V(r,t) W(c,t) + W(r,t) V(c,t)  (r >= c), with W taken as
//       W_raw + a2_t V (the rank-one correction of each W column is applied
//       lazily, see D); partial sums of |a_c(c+2:)|^2 and a_c(c+1)   | barrier
//   BC  reflector scalars (every CTA), V(:, i) = scal x + (1 - scal x0) e_{c+1}
//       written, and the SYMV run on the UNnormalised x = a_c(c+1:): y_raw =
//       A22 x, t1_raw = W_raw^T x, t2_raw = V^T x (linear in x, so the
//       normalisation is folded in afterwards — no barrier between the
//       reflector and the SYMV)                                     | barrier
//   D   y, t1, t2 assembled; w = tau (y - V t1 - W t2); w . v partial sums;
//       W_raw(:, i) = w                                              | barrier
//   a2_i = -tau/2 (w . v) is known to every CTA after the last barrier; at the
//   end of the panel each thread applies W += a2 V to its rows.
__global__ void __launch_bounds__(kTrdThreads, 1) sytrd_panel_kernel(TrdArgs a) {
  __shared__ double scratch[32];
  __shared__ double vw[2 * kTrdNB];   // V(c, 0:i), W_true(c, 0:i)  /  t1, t2
  __shared__ double a2s[kTrdNB];      // lazy W corrections
  const int n = a.n;
  const int tid = threadIdx.x;
  const int gtid = blockIdx.x * kTrdThreads + tid;
  const int gsz = gridDim.x * kTrdThreads;
  const int warps_total = gsz / 32;
  const int gwarp = gtid / 32, lane = tid & 31;
  unsigned epoch = 0;
  for (int i = 0; i < a.nb; ++i) {
    const int c = a.j0 + i;
    double* red = a.red + (i % 4) * 8;
    // zero the slot used two columns ahead (last read before the barrier below)
    if (blockIdx.x == 0 && tid < 8) a.red[((i + 2) % 4) * 8 + tid] = 0.0;
    TRD_MARK(0, i);
    // ---- A: column update with the panel so far (W_true = W_raw + a2 V)
    if (tid < i) {
      const double vct = a.V[c + (int64_t)tid * a.ldp];
      vw[tid] = vct;
      vw[kTrdNB + tid] = a.W[c + (int64_t)tid * a.ldp] + a2s[tid] * vct;
    }
    __syncthreads();
    double xs = 0.0, alpha_part = 0.0;
    for (int r = c + gtid; r < n; r += gsz) {
      double v = a.A[r + (int64_t)c * a.lda];
      for (int t = 0; t < i; ++t) {
        const double vr = a.V[r + (int64_t)t * a.ldp];
        const double wr = a.W[r + (int64_t)t * a.ldp] + a2s[t] * vr;
        v -= vr * vw[kTrdNB + t] + wr * vw[t];
      }
      a.A[r + (int64_t)c * a.lda] = v;
      if (r >= c + 2) xs += v * v;
      if (r == c + 1) alpha_part = v;
      if (r == c) a.d[c] = v;
    }
    TRD_MARK(1, i);
    block_atomic_sum(xs, &red[0], scratch);
    block_atomic_sum(alpha_part, &red[1], scratch);
    TRD_MARK(2, i);
    grid_sync(a.bar, epoch);
    TRD_MARK(3, i);
    // ---- BC: reflector + SYMV on the unnormalised column
    const double alpha = __ldcg(&red[1]);
    const double xnorm = sqrt(__ldcg(&red[0]));
    double beta = alpha, taui = 0.0, scal = 0.0;
    if (c + 1 < n && xnorm > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xnorm * xnorm), alpha);
      taui = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    const double head = 1.0 - scal * alpha;  // v = scal x + head e_{c+1}
    for (int r = gtid; r < n; r += gsz) {
      double v = 0.0;
      if (r == c + 1) v = 1.0;
      else if (r > c + 1) v = __ldcg(&a.A[r + (int64_t)c * a.lda]) * scal;
      a.V[r + (int64_t)i * a.ldp] = v;
    }
    if (gtid == 0) {
      if (c + 1 < n) a.e[c] = beta;
      a.tau[c] = taui;
    }
    TRD_MARK(4, i);
    const int m = n - c - 1;
    const double* xcol = a.A + (int64_t)c * a.lda;  // x(r) = A(r, c), r > c
    // SYMV over the LOWER triangle of A22 only (half the HBM traffic): one warp
    // per 32x32 lower tile (ti >= tj); the tile serves both y_ti += A x_tj
    // and (off the diagonal) y_tj += A^T x_ti, accumulated into y by FP64
    // atomics (y is zeroed row by row in phase D after its use).
    const int TI = (m + 31) / 32, mpad = TI * 32;
    const int ntiles = TI * (TI + 1) / 2;
    {
      // per-warp 32x33 tile + 64 x values in dynamic shared memory
      extern __shared__ double trd_dyn[];
      double(*tl)[33] = reinterpret_cast<double(*)[33]>(trd_dyn + (tid >> 5) * (32 * 33 + 64));
      double* xw = trd_dyn + (tid >> 5) * (32 * 33 + 64) + 32 * 33;
      for (int tt = gwarp; tt < ntiles + 2 * i; tt += warps_total) {
        if (tt >= ntiles) {  // virtual columns: t1_raw = W_raw^T x, t2_raw = V^T x
          const int jv = tt - ntiles;
          const double* col = (jv < i) ? a.W + (int64_t)jv * a.ldp : a.V + (int64_t)(jv - i) * a.ldp;
          double s0 = 0.0, s1 = 0.0;
          int r = c + 1 + lane;
          for (; r + 32 < n; r += 64) {
            s0 = fma(col[r], __ldcg(&xcol[r]), s0);
            s1 = fma(col[r + 32], __ldcg(&xcol[r + 32]), s1);
          }
          if (r < n) s0 = fma(col[r], __ldcg(&xcol[r]), s0);
          const double sm = warp_sum(s0 + s1);
          if (lane == 0) a.y[m + jv] = sm;
          continue;
        }
        int tj = 0, rem = tt;  // column-major enumeration of the lower tiles
        while (rem >= TI - tj) {
          rem -= TI - tj;
          ++tj;
        }
        const int ti = tj + rem;
        const int lr = ti * 32 + lane, lc0 = tj * 32;  // local row / first local column
        const int r = c + 1 + lr;
        const bool diag = (ti == tj);
        {
          // all 32 column loads of the tile in flight at once (8 KB per warp)
          double v[32];
          const double* base = a.A + r + (int64_t)(c + 1 + lc0) * a.lda;
          const int ncol = min(32, m - lc0);
#pragma unroll
          for (int cc = 0; cc < 32; ++cc)
            v[cc] = (lr < m && cc < ncol && (!diag || lane >= cc)) ? base[(int64_t)cc * a.lda] : 0.0;
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) tl[lane][cc] = v[cc];
        }
        xw[lane] = (lc0 + lane < m) ? __ldcg(&xcol[c + 1 + lc0 + lane]) : 0.0;
        xw[32 + lane] = (lr < m) ? __ldcg(&xcol[r]) : 0.0;
        __syncwarp();
        double yr = 0.0, yc = 0.0;
        if (diag) {
#pragma unroll 8
          for (int cc = 0; cc < 32; ++cc) {
            const double v = (cc <= lane) ? tl[lane][cc] : tl[cc][lane];
            yr = fma(v, xw[cc], yr);
          }
        } else {
#pragma unroll 8
          for (int cc = 0; cc < 32; ++cc) {
            yr = fma(tl[lane][cc], xw[cc], yr);        // row part: rows of ti
            yc = fma(tl[cc][lane], xw[32 + cc], yc);   // column part: rows of tj
          }
        }
        // y (zeroed by phase D of the previous column) accumulates by atomics
        if (lr < m) atomicAdd(&a.y[lr], yr);
        if (!diag && lc0 + lane < m) atomicAdd(&a.y[lc0 + lane], yc);
        __syncwarp();
      }
    }
    TRD_MARK(5, i);
    grid_sync(a.bar, epoch);
    TRD_MARK(6, i);
    // ---- D: w = tau (y - V t1 - W_true t2) with y = scal y_raw + head A22(:, 0),
    // t = scal t_raw + head (row c+1);  W_true t2 = W_raw t2 + V (a2 .* t2)
    if (tid < i) {
      const double t2 = scal * __ldcg(&a.y[m + i + tid]) + head * a.V[(c + 1) + (int64_t)tid * a.ldp];
      const double wrow = a.W[(c + 1) + (int64_t)tid * a.ldp];
      const double t1raw = scal * __ldcg(&a.y[m + tid]) + head * wrow;  // W_raw^T v
      // coefficient of V(:, t): t1_true + a2 t2 = t1raw + 2 a2 t2 (t1_true = t1raw + a2 t2)
      vw[tid] = t1raw + 2.0 * a2s[tid] * t2;
      vw[kTrdNB + tid] = t2;
    }
    __syncthreads();
    double dotp = 0.0;
    for (int r = gtid; r < n; r += gsz) {
      double w = 0.0;
      if (r > c) {
        const int lr = r - c - 1;
        const double yraw = __ldcg(&a.y[lr]);
        a.y[lr] = 0.0;  // ready for the next column's atomics
        w = scal * yraw + head * a.A[r + (int64_t)(c + 1) * a.lda];
        for (int t = 0; t < i; ++t)
          w -= a.V[r + (int64_t)t * a.ldp] * vw[t] + a.W[r + (int64_t)t * a.ldp] * vw[kTrdNB + t];
        w *= taui;
        dotp += w * __ldcg(&a.V[r + (int64_t)i * a.ldp]);
      }
      a.W[r + (int64_t)i * a.ldp] = w;
    }
    TRD_MARK(7, i);
    block_atomic_sum(dotp, &red[2], scratch);
    grid_sync(a.bar, epoch);
    TRD_MARK(8, i);
    if (tid == 0) a2s[i] = -0.5 * taui * __ldcg(&red[2]);
    __syncthreads();
  }
  // ---- W += a2 V (the deferred corrections), rows owned by this thread
  for (int r = gtid; r < n; r += gsz)
    for (int t = 0; t < a.nb; ++t)
      a.W[r + (int64_t)t * a.ldp] += a2s[t] * a.V[r + (int64_t)t * a.ldp];
}

// Sturm count: number of eigenvalues of T (d, e) strictly below x.
QDWHG_DEV int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < n; ++i) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = d[i] - x - e2[i - 1] / q;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

// Eigenvalue k (ascending) by multisection on [lo, hi]: one warp per
// eigenvalue, the 32 lanes evaluate 32 Sturm counts at once, so every round
// shrinks the bracket 33x (~11 rounds to full precision instead of ~55).
__global__ void bisect_kernel(const double* d, const double* e2, int n, double lo0, double hi0,
                              double pivmin, double abstol, double* w) {
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= n) return;
  double lo = lo0, hi = hi0;
  for (int it = 0; it < 40; ++it) {
    if (hi - lo <= abstol + 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi))) break;
    const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
    const bool above = sturm_count(d, e2, n, x, pivmin) > k;  // lambda_k < x
    const unsigned m = __ballot_sync(0xffffffffu, above);
    // first lane whose point lies above lambda_k
    const int f = m ? (__ffs(m) - 1) : 32;
    const double nlo = (f == 0) ? lo : lo + (hi - lo) * (double)f / 33.0;
    const double nhi = (f == 32) ? hi : lo + (hi - lo) * (double)(f + 1) / 33.0;
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) w[k] = 0.5 * (lo + hi);
}

// Inverse iteration for eigenvalue lam: (T - lam I) z = b with partial pivoting,
// 3 solves, normalised.  Element i of this thread's vector / factor arrays is at
// [i * zs] (Z) and [i * s] (u1 diag, u2 super, u3 super2, l, piv): strided so
// consecutive threads touch consecutive words (global or shared memory).
QDWHG_DEV void inviter_one(const double* d, const double* e, int n, double lam, double tnorm,
                           double* Z, int zs, double* U1, double* U2, double* U3, double* L,
                           unsigned char* P, int s) {
  const double eps = 2.220446049250313e-16;
  const double tiny = eps * tnorm;
  // ---- LU with partial pivoting of the tridiagonal (dlagtf shape)
  double a = d[0] - lam;                  // current diagonal
  double b = (n > 1) ? e[0] : 0.0;        // current super
  for (int i = 0; i < n - 1; ++i) {
    const double cc = e[i];              // sub-diagonal below row i
    const double dn = d[i + 1] - lam;
    const double bn = (i + 2 < n) ? e[i + 1] : 0.0;
    const size_t o = (size_t)i * s;
    if (fabs(a) >= fabs(cc)) {
      // no swap: row i stays; multiplier l = cc / a
      const double piv = (a == 0.0) ? tiny : a;
      const double l = cc / piv;
      U1[o] = piv;
      U2[o] = b;
      U3[o] = 0.0;
      L[o] = l;
      P[o] = 0;
      a = dn - l * b;
      b = bn;
    } else {
      // swap rows i and i+1
      const double l = a / cc;
      U1[o] = cc;
      U2[o] = dn;
      U3[o] = bn;
      L[o] = l;
      P[o] = 1;
      a = b - l * dn;
      b = -l * bn;
    }
  }
  {
    const size_t o = (size_t)(n - 1) * s;
    U1[o] = (a == 0.0) ? tiny : a;
    U2[o] = 0.0;
    U3[o] = 0.0;
  }
  // ---- iterations: forward apply L (with pivots), back-solve U
  // start vector: ones (dstein uses random; ones is adequate after 3 solves)
  for (int i = 0; i < n; ++i) Z[(size_t)i * zs] = 1.0;
  for (int it = 0; it < 3; ++it) {
    if (it > 0) {
      // forward: apply the row swaps/multipliers to the rhs
      for (int i = 0; i < n - 1; ++i) {
        const size_t o = (size_t)i * s;
        double zi = Z[(size_t)i * zs], zn = Z[(size_t)(i + 1) * zs];
        if (P[o]) {
          const double t = zi;
          zi = zn;
          zn = t;
        }
        zn -= L[o] * zi;
        Z[(size_t)i * zs] = zi;
        Z[(size_t)(i + 1) * zs] = zn;
      }
    }
    // back substitution U z = rhs, with scaling against overflow
    double z2 = 0.0, z1 = 0.0, nrm = 0.0;
    for (int i = n - 1; i >= 0; --i) {
      const size_t o = (size_t)i * s;
      double v = Z[(size_t)i * zs] - U2[o] * z1 - U3[o] * z2;
      v /= U1[o];
      Z[(size_t)i * zs] = v;
      z2 = z1;
      z1 = v;
      nrm = fmax(nrm, fabs(v));
    }
    // normalise (inf-norm first, then 2-norm at the end)
    const double sc = (nrm > 0.0) ? 1.0 / nrm : 1.0;
    for (int i = 0; i < n; ++i) Z[(size_t)i * zs] *= sc;
  }
  double s2 = 0.0;
  for (int i = 0; i < n; ++i) {
    const double v = Z[(size_t)i * zs];
    s2 += v * v;
  }
  const double inv = 1.0 / sqrt(s2);
  for (int i = 0; i < n; ++i) Z[(size_t)i * zs] *= inv;
}

// Eigenvectors k0 .. k0+cnt-1, one thread each, arrays in global memory
// (transposed, stride cnt): Zt[k + i*cnt] = z_k(i).
__global__ void inviter_kernel(const double* d, const double* e, int n, const double* w, int k0,
                               int cnt, double tnorm, double* Zt, double* U1, double* U2,
                               double* U3, double* L, unsigned char* P) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= cnt) return;
  inviter_one(d, e, n, w[k0 + k], tnorm, Zt + k, cnt, U1 + k, U2 + k, U3 + k, L + k, P + k, cnt);
}

// Small tridiagonals (n <= kSmallTrd): 32 eigenvectors per CTA with the factor
// and vector arrays in shared memory (an L1-latency recurrence instead of an
// L2 round trip per step); Z (n x cnt, column-major) written directly.
__global__ void __launch_bounds__(32)
    inviter_small_kernel(const double* d, const double* e, int n, const double* w, int k0, int cnt,
                         double tnorm, double* Z, int64_t ldz) {
  extern __shared__ double ism[];
  const int lane = threadIdx.x;
  double* Zs = ism;                       // [n][33]
  double* U1 = Zs + (size_t)n * 33;       // [n][32] each
  double* U2 = U1 + (size_t)n * 32;
  double* U3 = U2 + (size_t)n * 32;
  double* Lm = U3 + (size_t)n * 32;
  unsigned char* P = reinterpret_cast<unsigned char*>(Lm + (size_t)n * 32);
  const int k = blockIdx.x * 32 + lane;
  if (k < cnt)
    inviter_one(d, e, n, w[k0 + k], tnorm, Zs + lane, 33, U1 + lane, U2 + lane, U3 + lane, Lm + lane,
                P + lane, 32);
  __syncwarp();
  const int nv = min(32, cnt - blockIdx.x * 32);
  for (int v = 0; v < nv; ++v)
    for (int i = lane; i < n; i += 32) Z[i + (int64_t)(blockIdx.x * 32 + v) * ldz] = Zs[i * 33 + v];
}

size_t inviter_small_smem(int n) { return (size_t)n * (33 + 4 * 32) * sizeof(double) + (size_t)n * 32; }

void inviter_small_launch(Ctx& ctx, const double* dd, const double* ee, int n, const double* wv, int k0,
                          int cnt, double tnorm, double* Z, int64_t ldz) {
  func_attr(inviter_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)inviter_small_smem(160));
  inviter_small_kernel<<<(cnt + 31) / 32, 32, inviter_small_smem(n), ctx.stream>>>(dd, ee, n, wv, k0, cnt,
                                                                                  tnorm, Z, ldz);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

// Z(i, k) = Zt[k + i*cnt]   (i < n rows, k < cnt vectors)
__global__ void transpose_kernel(const double* Zt, int n, int cnt, double* Z, int64_t ldz) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = by + r, k = bx + threadIdx.x;
    tile[r][threadIdx.x] = (i < n && k < cnt) ? Zt[(size_t)k + (size_t)i * cnt] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = bx + r, i = by + threadIdx.x;
    if (i < n && k < cnt) Z[i + (int64_t)k * ldz] = tile[threadIdx.x][r];
  }
}

__global__ void square_kernel(const double* e, int n, double* e2) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x)
    e2[i] = e[i] * e[i];
}

// ---------------------------------------------------------------- small blocks
// Rayleigh-Ritz blocks up to kSmallTrd (cfg1/cfg2: ell ~ 50-130) in ONE CTA:
// the whole matrix lives in shared memory, so a column costs three CTA barriers
// instead of the cooperative panel's three grid barriers plus the per-panel
// trailing GEMMs.  Unblocked dsytd2 (lower), same reflector convention as
// sytrd_panel_kernel (beta = -sign(alpha) ||x||, tau = (beta - alpha)/beta,
// v = [1; x(2:)/(alpha - beta)]).
constexpr int kSmallTrd = 160;
constexpr int kSmallThreads = 1024;

__global__ void __launch_bounds__(kSmallThreads, 1)
    sytd2_small_kernel(const double* S, int64_t lds, int n, double* d, double* e, double* tau,
                       double* V, int64_t ldv) {
  extern __shared__ double sm[];
  const int LD = n | 1;              // odd stride: column reads by row groups are conflict-free
  double* A = sm;                    // column-major A[c * LD + r], both triangles kept current
  double* vs = A + (size_t)n * LD;   // reflector (n)
  double* ps = vs + n + 1;           // p = tau A22 v (n)
  double* sc = ps + n + 1;           // [0] tau, [1] p.v accumulator
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = warp; c < n; c += (int)(blockDim.x / 32))
    for (int r = c + lane; r < n; r += 32)  // lower triangle (all the kernel reads)
      A[c * LD + r] = 0.5 * (S[r + (int64_t)c * lds] + S[c + (int64_t)r * lds]);
  // V(:, j): zeros above row j+1 (every column written in full below)
  for (int c = warp; c < n - 1; c += (int)(blockDim.x / 32))
    for (int r = lane; r <= c; r += 32) V[r + (int64_t)c * ldv] = 0.0;
  __syncthreads();
  for (int i = 0; i + 1 < n; ++i) {
    const int m = n - i - 1;  // rows i+1 .. n-1
    const double* x = A + (size_t)i * LD + i + 1;
    // ---- (a) reflector: one warp (m <= 159: <= 5 entries per lane)
    if (warp == 0) {
      double s2 = 0.0;
      for (int r = 1 + lane; r < m; r += 32) s2 = fma(x[r], x[r], s2);
      s2 = warp_sum(s2);
      const double alpha = x[0];
      double beta = alpha, taui = 0.0, scal = 0.0;
      if (s2 > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s2), alpha);
        taui = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int r = lane; r < m; r += 32) {
        const double v = (r == 0) ? 1.0 : (s2 > 0.0 ? x[r] * scal : 0.0);
        vs[r] = v;
        V[(i + 1 + r) + (int64_t)i * ldv] = v;
      }
      if (lane == 0) {
        d[i] = A[(size_t)i * LD + i];
        e[i] = beta;
        tau[i] = taui;
        sc[0] = taui;
      }
    }
    __syncthreads();
    const double taui = sc[0];
    if (taui != 0.0) {
      // ---- (b) p = tau A22 v: 8 threads per row r of A22 read column r (A symmetric)
      // (loop bound uniform per warp: the shuffles need all 32 lanes)
      const int k = tid & 7;
      for (int r0 = warp * 4; r0 < m; r0 += (int)(blockDim.x / 8)) {
        const int r = r0 + ((tid >> 3) & 3);
        // lower triangle only: A22(r, c) = row r left of the diagonal, column r below it
        const double* A22 = A + (size_t)(i + 1) * LD + i + 1;
        double acc = 0.0;
        if (r < m)
          for (int c = k; c < m; c += 8)
            acc = fma(c < r ? A22[(size_t)c * LD + r] : A22[(size_t)r * LD + c], vs[c], acc);
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (k == 0 && r < m) ps[r] = taui * acc;
      }
      __syncthreads();
      // ---- (c) A22 -= v w^T + w v^T,  w = p - (tau/2)(p.v) v; p.v summed by
      // every warp redundantly (same order everywhere, no extra barrier)
      double pv = 0.0;
      for (int r = lane; r < m; r += 32) pv = fma(ps[r], vs[r], pv);
      const double a2 = -0.5 * taui * warp_sum(pv);
      // (lower triangle only; lane = row within a 32-row strip, warp = column)
      for (int c = warp; c < m; c += (int)(blockDim.x / 32)) {
        const double vc = vs[c], wc = ps[c] + a2 * vc;
        double* col = A + (size_t)(i + 1 + c) * LD + i + 1;
        for (int r = c + lane; r < m; r += 32) col[r] -= vs[r] * wc + (ps[r] + a2 * vs[r]) * vc;
      }
    }
    __syncthreads();  // (also orders sc[0] reads before the next column's write)
  }
  if (tid == 0) d[n - 1] = A[(size_t)(n - 1) * LD + n - 1];
}

int small_threads() {
  static const int t = getenv("QDWHG_SMALL_THREADS") ? atoi(getenv("QDWHG_SMALL_THREADS")) : kSmallThreads;
  return (t == 256 || t == 512 || t == 1024) ? t : kSmallThreads;
}

size_t sytd2_small_smem(int n) { return ((size_t)n * (n | 1) + 2 * (n + 1) + 2) * sizeof(double); }

}  // namespace

void syev_dc_fallback(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout);

// Returns false if the eigenvectors could not be orthogonalised cheaply (caller falls back).
bool syev_tridiag(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout, double vlo,
                  double vhi, int64_t* sel0) {
  const int n = (int)S.rows;
  const Arena::Mark mark = ctx.arena->mark();
  const bool small = n <= kSmallTrd;
  DMat A = ctx.arena->alloc(n, n);
  if (!small) copy(ctx, S, A);
  const int nb = kTrdNB;
  const int npan = (n - 1 + nb - 1) / nb;  // columns 0 .. n-2 carry reflectors
  DMat Vfull = ctx.arena->alloc(n, std::max(npan * nb, 1));
  DMat Wp = ctx.arena->alloc(n, nb);
  double* dd = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (n + 8)));
  double* ee = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (n + 8)));
  double* tau = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (npan * nb + 8)));
  double* y = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (n + 2 * nb + 8)));
  const int64_t tin = (n + 31) / 32;
  double* ypart = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * tin * tin * 32 + 64));
  double* red = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * 64));
  unsigned* bar = static_cast<unsigned*>(ctx.arena->alloc_bytes(256));
  QDWHG_CUDA(cudaMemsetAsync(tau, 0, sizeof(double) * (npan * nb + 8), ctx.stream));
  QDWHG_CUDA(cudaMemsetAsync(ee, 0, sizeof(double) * (n + 8), ctx.stream));
  if (!small)  // (Vfull needs no fill: every panel writes its V columns in full)
    QDWHG_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * (n + 2 * nb + 8), ctx.stream));  // SYMV atomics
  if (Wp.ld != Vfull.ld) throw CudaError("syev_tridiag: panel V/W leading dimensions differ");
  func_attr(sytrd_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrdDynSmem);
  if (small) {
    func_attr(sytd2_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sytd2_small_smem(kSmallTrd));
    sytd2_small_kernel<<<1, small_threads(), sytd2_small_smem(n), ctx.stream>>>(S.ptr(), S.ld, n, dd, ee, tau,
                                                                             Vfull.ptr(), Vfull.ld);
    QDWHG_CUDA(cudaGetLastError());
    ctx.count();
  }
  // all SMs: the per-column SYMV streams the trailing matrix (HBM/L2 bound)
  const int grid = std::max(1, std::min(ctx.num_sms, (n + 31) / 32));
  for (int p = 0; p < (small ? 0 : npan); ++p) {
    const int j0 = p * nb;
    const int b = std::min(nb, n - 1 - j0);
    QDWHG_CUDA(cudaMemsetAsync(red, 0, sizeof(double) * 64, ctx.stream));
    QDWHG_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), ctx.stream));
    // the panel's reflectors go straight into their columns of Vfull
    const DMat Vpan = Vfull.sub(0, j0, n, nb);
    TrdArgs args{A.ptr(), A.ld, Vpan.ptr(), Wp.ptr(), Vfull.ld, dd, ee, tau, y, ypart, red, bar, n, j0, b};
    void* kargs[] = {&args};
    QDWHG_CUDA(cudaLaunchCooperativeKernel((void*)sytrd_panel_kernel, dim3(grid), dim3(kTrdThreads),
                                           kargs, kTrdDynSmem, ctx.stream));
    ctx.count();
    const int r0 = j0 + b;
    const int rest = n - r0;
    if (rest > 0) {
      const DMat Vr = Vpan.sub(r0, 0, rest, b), Wr = Wp.sub(r0, 0, rest, b);
      const DMat At = A.sub(r0, r0, rest, rest);
      GemmExtra lo;  // the panel kernel reads only the lower triangle of A
      lo.out = OutMode::Lower;
      gemm(ctx, Op::N, Op::T, -1.0, Vr, Wr, 1.0, At, lo);
      gemm(ctx, Op::N, Op::T, -1.0, Wr, Vr, 1.0, At, lo);
    }
  }
  // last diagonal entry (and the one before if the last panel ended early)
  if (!small) {
    // d[n-1] = A(n-1, n-1) after all updates (no reflector column touches it again)
    QDWHG_CUDA(cudaMemcpyAsync(dd + (n - 1), A.ptr() + (n - 1) + (int64_t)(n - 1) * A.ld,
                               sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
  }
  // ---- tridiagonal eigenvalues (bisection) and vectors (inverse iteration)
  std::vector<double> hd(n), he(n);
  QDWHG_CUDA(cudaMemcpyAsync(hd.data(), dd, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaMemcpyAsync(he.data(), ee, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  double lo = 1e308, hi = -1e308, tnorm = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? std::abs(he[i - 1]) : 0.0) + (i + 1 < n ? std::abs(he[i]) : 0.0);
    lo = std::min(lo, hd[i] - r);
    hi = std::max(hi, hd[i] + r);
    tnorm = std::max(tnorm, std::abs(hd[i]) + r);
  }
  if (!(tnorm > 0.0)) tnorm = 1.0;
  const double eps = 2.220446049250313e-16;
  lo -= 2 * eps * tnorm + 1e-300;
  hi += 2 * eps * tnorm + 1e-300;
  double* e2 = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (n + 8)));
  double* wv = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (n + 8)));
  square_kernel<<<std::max(1, std::min(148, (n + 255) / 256)), 256, 0, ctx.stream>>>(ee, n, e2);
  const double pivmin = std::max(1e-300, eps * eps * tnorm * tnorm * 1e-10);
  bisect_kernel<<<(32 * n + 127) / 128, 128, 0, ctx.stream>>>(dd, e2, n, lo, hi, pivmin, 2 * eps * tnorm * 1e-3,
                                                     wv);
  // eigenvalues to the host now: only the selected eigenvectors are formed
  vals.resize(n);
  QDWHG_CUDA(cudaMemcpyAsync(vals.data(), wv, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  int i0 = 0;
  while (i0 < n && !(vals[i0] > vlo)) ++i0;
  int i1 = i0;
  while (i1 < n && vals[i1] < vhi) ++i1;
  const int cnt = i1 - i0;
  *sel0 = i0;
  if (cnt == 0) {
    ctx.arena->release_to(mark);
    return true;
  }
  const size_t nc = (size_t)n * cnt;
  double* Zt = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * nc));
  double* U1 = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * nc));
  double* U2 = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * nc));
  double* U3 = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * nc));
  double* Lm = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * nc));
  unsigned char* Pv = static_cast<unsigned char*>(ctx.arena->alloc_bytes(nc));
  DMat Z = ctx.arena->alloc(n, cnt);
  if (small) {
    inviter_small_launch(ctx, dd, ee, n, wv, i0, cnt, tnorm, Z.ptr(), Z.ld);
    ctx.count(2);
  } else {
    inviter_kernel<<<(cnt + 63) / 64, 64, 0, ctx.stream>>>(dd, ee, n, wv, i0, cnt, tnorm, Zt, U1, U2,
                                                          U3, Lm, Pv);
    transpose_kernel<<<dim3((cnt + 31) / 32, (n + 31) / 32), dim3(32, 8), 0, ctx.stream>>>(
        Zt, n, cnt, Z.ptr(), Z.ld);
    ctx.count(4);
  }
  QDWHG_CUDA(cudaGetLastError());
  // ---- Lowdin: E = Z^T Z - I;  Z <- Z (I - E/2 + 3/8 E^2)
  DMat E = ctx.arena->alloc(cnt, cnt);
  GemmExtra gr;
  gr.out = OutMode::LowerMirror;
  gr.diag_add = -1.0;
  gemm(ctx, Op::T, Op::N, 1.0, Z, Z, 0.0, E, gr);
  const MatStats es = mat_stats(ctx, E, false);
  if (!(es.maxabs < 1e-4)) {
    ctx.arena->release_to(mark);
    return false;
  }
  DMat F = ctx.arena->alloc(cnt, cnt);
  GemmExtra f2;
  f2.cin = &E;  // F = 3/8 E^2 - 1/2 E + I
  f2.diag_add = 1.0;
  gemm(ctx, Op::N, Op::N, 0.375, E, E, -0.5, F, f2);
  // ---- back-transform: Vout = Q Z F, Q = H_0 ... H_{n-2}, blocks applied last to first
  const DMat Vsel = Vout.sub(0, 0, n, cnt);
  gemm(ctx, Op::N, Op::N, 1.0, Z, F, 0.0, Vsel);
  // (small blocks too: the sytd2_small reflectors use the same unit-lower layout;
  // compact-WY blocks on the GEMM engine instead of the former one-CTA
  // reflector-by-reflector back-transform: 0.30 ms at l = 132)
  // blocks of 64 reflectors (the larft limit; twice the SYTRD panel width: half
  // the launches, K = 64 GEMMs)
  constexpr int bw = 64;
  const int nbt = (n - 1 + bw - 1) / bw;
  DMat G = ctx.arena->alloc(bw, bw), Tb = ctx.arena->alloc(bw, bw);
  for (int p = nbt - 1; p >= 0; --p) {
    const int j0 = p * bw;
    const int b = std::min(bw, n - 1 - j0);
    const int r0 = j0 + 1;  // reflectors of this panel act on rows >= j0+1
    const int mp = n - r0;
    const DMat Vb = Vfull.sub(r0, j0, mp, b);
    gemm(ctx, Op::T, Op::N, 1.0, Vb, Vb, 0.0, G.sub(0, 0, b, b));
    larft_launch(ctx, G.sub(0, 0, b, b), tau + j0, Tb.sub(0, 0, b, b));
    const Arena::Mark m2 = ctx.arena->mark();
    DMat W1 = ctx.arena->alloc(b, cnt), W2 = ctx.arena->alloc(b, cnt);
    const DMat C = Vout.sub(r0, 0, mp, cnt);
    gemm(ctx, Op::T, Op::N, 1.0, Vb, C, 0.0, W1);
    GemmExtra eu;
    eu.krange = KRange::AUpper;
    gemm(ctx, Op::N, Op::N, 1.0, Tb.sub(0, 0, b, b), W1, 0.0, W2, eu);
    gemm(ctx, Op::N, Op::N, -1.0, Vb, W2, 1.0, C);
    ctx.arena->release_to(m2);
  }
  ctx.arena->release_to(mark);
  return true;
}

void tridiag_lowest(Ctx& ctx, const std::vector<double>& d, const std::vector<double>& e,
                    double* theta, double* z_last) {
  const int n = (int)d.size();
  if (n == 0) throw InvalidArgument("tridiag_lowest: empty");
  if (n == 1) {
    *theta = d[0];
    *z_last = 1.0;
    return;
  }
  double lo = 1e308, hi = -1e308, tnorm = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? std::abs(e[i - 1]) : 0.0) + (i + 1 < n ? std::abs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
    tnorm = std::max(tnorm, std::abs(d[i]) + r);
  }
  if (!(tnorm > 0.0)) tnorm = 1.0;
  const double eps = 2.220446049250313e-16;
  lo -= 2 * eps * tnorm + 1e-300;
  hi += 2 * eps * tnorm + 1e-300;
  const double pivmin = std::max(1e-300, eps * eps * tnorm * tnorm * 1e-10);
  // one packed upload: [d | e | e^2], then w (1), z (n) and the LU scratch
  std::vector<double> h((size_t)3 * n, 0.0);
  for (int i = 0; i < n; ++i) h[i] = d[i];
  for (int i = 0; i + 1 < n; ++i) {
    h[n + i] = e[i];
    h[2 * n + i] = e[i] * e[i];
  }
  const Arena::Mark mark = ctx.arena->mark();
  double* dev = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (size_t)(5 * n + 8)));
  double *dd = dev, *ee = dev + n, *e2 = dev + 2 * n, *wv = dev + 3 * n, *Zt = wv + 1;
  QDWHG_CUDA(cudaMemcpyAsync(dev, h.data(), sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx.stream));
  bisect_kernel<<<1, 32, 0, ctx.stream>>>(dd, e2, n, lo, hi, pivmin, 2 * eps * tnorm * 1e-3, wv);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
  inviter_small_launch(ctx, dd, ee, n, wv, 0, 1, tnorm, Zt, n);
  double out[2];
  QDWHG_CUDA(cudaMemcpyAsync(&out[0], wv, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaMemcpyAsync(&out[1], Zt + (n - 1), sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  ctx.arena->release_to(mark);
  *theta = out[0];
  *z_last = out[1];
}

}  // namespace qdwhg
