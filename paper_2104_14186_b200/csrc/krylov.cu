// HBM-bound Krylov scalars of the partial drivers:
//   two_norm_estimate  — power iteration on A^T A (kernels.cpp:332-360), alpha for Alg. 2
//   lanczos_min_bound  — 30-step Lanczos with two-pass full reorthogonalisation
//                        (kernels.cpp:362-439), mu for Alg. 1
// Start vectors are generated on the host with the reference's own counter
// generator (bit-identical, see host_gaussian in qdwhg.cpp), so mu and alpha
// differ from the reference only by summation order.  GEMVs stream A once per
// product at full HBM bandwidth (column-dot form for A^T x, row-split form with
// a deterministic two-stage reduction for A x).
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

namespace qdwhg {

std::vector<double> host_gaussian(int64_t count, uint64_t seed);  // qdwhg.cpp
void syev_jacobi(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout);

namespace {

// Normalised start vector of the reference's counter generator (host glibc
// log/cos: ~0.3 ms at n = 4096), cached per (n, seed) — it is the same vector on
// every call of a given size.
// (returned by value: a copy of n doubles is nothing next to the generation, and
// no caller holds a reference into the cache while another thread evicts it)
std::vector<double> start_vector(int64_t n, uint64_t seed) {
  static std::mutex mu;
  static std::map<std::pair<int64_t, uint64_t>, std::vector<double>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({n, seed});
  if (it != cache.end()) return it->second;
  std::vector<double> v = host_gaussian(n, seed);
  double s = 0.0;
  for (double x : v) s += x * x;
  const double nv = std::sqrt(s);
  for (double& x : v) x /= nv;
  if (cache.size() >= 64) cache.clear();
  cache.emplace(std::make_pair(n, seed), v);
  return v;
}

// z_j = sum_i A(i,j) x_i  (one warp per column; coalesced down the column)
__global__ void gemv_t_kernel(const double* A, int64_t lda, int64_t m, int64_t n, const double* x,
                              double* z) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
    const double* a = A + j * lda;
    double s0 = 0.0, s1 = 0.0;
    int64_t i = lane;
    for (; i + 32 < m; i += 64) {
      s0 += a[i] * x[i];
      s1 += a[i + 32] * x[i + 32];
    }
    if (i < m) s0 += a[i] * x[i];
    const double s = warp_sum(s0 + s1);
    if (lane == 0) z[j] = s;
  }
}

// partial[s][i] = sum_{j in split s} A(i,j) x_j
__global__ void gemv_n_partial_kernel(const double* A, int64_t lda, int64_t m, int64_t n,
                                      const double* x, int64_t cols_per_split, double* partial) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j0 = blockIdx.y * cols_per_split;
  const int64_t j1 = std::min<int64_t>(n, j0 + cols_per_split);
  if (i >= m) return;
  double s0 = 0.0, s1 = 0.0;
  int64_t j = j0;
  for (; j + 1 < j1; j += 2) {
    s0 += A[i + j * lda] * x[j];
    s1 += A[i + (j + 1) * lda] * x[j + 1];
  }
  if (j < j1) s0 += A[i + j * lda] * x[j];
  partial[blockIdx.y * m + i] = s0 + s1;
}

__global__ void reduce_partial_kernel(const double* partial, int splits, int64_t m, double* y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += partial[k * m + i];
    y[i] = s;
  }
}

// out[slot] = x . y  (two-stage: per-block partials, then final by block 0 of a 2nd launch)
__global__ void dot_partial_kernel(const double* x, const double* y, int64_t n, double* partial) {
  __shared__ double scratch[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s += x[i] * y[i];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
__global__ void dot_final_kernel(const double* partial, int nblk, double* out) {
  __shared__ double scratch[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) s += partial[i];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) *out = s;
}

// x = y / sqrt(*nrm2)
__global__ void scale_by_invnorm_kernel(const double* y, const double* nrm2, int64_t n, double* x) {
  const double inv = 1.0 / sqrt(*nrm2);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = y[i] * inv;
}

// w_i -= sum_k Q(i,k) h_k   (k < kcount <= 64)
__global__ void sub_qh_kernel(const double* Q, int64_t ldq, int64_t n, int kcount, const double* h,
                              double* w) {
  __shared__ double hs[64];
  if (threadIdx.x < kcount) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < kcount; ++k) s += Q[i + k * ldq] * hs[k];
    w[i] -= s;
  }
}


// ---------------------------------------------------------------- Lanczos
// The whole m-step Lanczos with two-pass classical Gram-Schmidt
// reorthogonalisation as ONE cooperative kernel (one CTA per SM): CTA g owns
// rows [g*chunk, (g+1)*chunk) of every vector; w = A q_j is formed column by
// column (A symmetric) for the owned indices, so the reorthogonalisation and
// norms only need cross-CTA sums of short vectors: three grid barriers per
// step (two CGS passes, the norm), no host round trips, no kernel launches.
// Partial sums are combined in fixed order (deterministic).
constexpr int kLzThreads = 512;
constexpr int kLzSlotsPerLane = 5;  // 160 >= the grid (<= 148 CTAs)
struct LanczosArgs {
  const double* A;
  int64_t lda;
  int n, m;
  double* Q;  // n x (m+1), column 0 = q_0 (set by the host)
  int64_t ldq;
  double* wbuf;        // [2][n] unnormalised next vector, by step parity
  double* slots;       // [2 passes][G][64] CGS partials
  double* bslots;      // [2 parity][G] norm partials
  double* alpha_part;  // [G][64] alpha partials (summed by the host)
  double* beta2;       // [64]
  unsigned* bar;
};

__global__ void __launch_bounds__(kLzThreads, 1) lanczos_kernel(LanczosArgs a) {
  extern __shared__ double lz_sm[];
  const int G = gridDim.x, g = blockIdx.x;
  const int n = a.n;
  const int chunk = (n + G - 1) / G;
  const int r0 = min(n, g * chunk), nown = max(0, min(n, r0 + chunk) - r0);
  double* w_own = lz_sm;       // [chunk]
  double* hsm = w_own + chunk; // [64]
  double* red = hsm + 64;      // [32]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kLzThreads / 32;
  unsigned epoch = 0;
  double inv_beta = 1.0;
  const bool vec2 = ((a.lda & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.A) & 15) == 0) && ((n & 1) == 0);
  for (int j = 0; j < a.m; ++j) {
    const double* qsrc = (j == 0) ? a.Q : a.wbuf + ((j - 1) & 1) * (int64_t)n;
    const double qs = (j == 0) ? 1.0 : inv_beta;
    double* Qj = a.Q + (int64_t)j * a.ldq;
    if (j > 0)
      for (int i = tid; i < nown; i += kLzThreads) Qj[r0 + i] = qsrc[r0 + i] * qs;
    // ---- w_i = (A q_j)_i for owned i, reading only the LOWER triangle of A (A is
    // symmetric): the n^2/2 footprint stays L2-resident across the steps for
    // n up to ~5000, and every element is read twice (column strip of its
    // column owner, row strip of its row owner) — n * chunk reads per CTA.
    //  (a) column strip: sum_{r >= i} A(r, i) q_r, warp per owned column i
    for (int ii = warp; ii < nown; ii += NW) {
      const int i = r0 + ii;
      const double* col = a.A + (int64_t)i * a.lda;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (vec2) {
        const double2* c2 = reinterpret_cast<const double2*>(col);
        const double2* q2 = reinterpret_cast<const double2*>(qsrc);
        const int n2 = n / 2;
        const int p0 = i >> 1;  // first pair holding row i (row i-1 masked when i is odd)
        int r = p0 + lane;
        for (; r + 32 < n2; r += 64) {
          const double2 x = c2[r], y = c2[r + 32];
          const double2 u = q2[r], v = q2[r + 32];
          s0 = fma((2 * r >= i) ? x.x : 0.0, u.x, s0);
          s1 = fma(x.y, u.y, s1);
          s2 = fma(y.x, v.x, s2);
          s3 = fma(y.y, v.y, s3);
        }
        if (r < n2) {
          const double2 x = c2[r], u = q2[r];
          s0 = fma((2 * r >= i) ? x.x : 0.0, u.x, s0);
          s1 = fma(x.y, u.y, s1);
        }
      } else {
        for (int r = i + lane; r < n; r += 32) s0 = fma(col[r], qsrc[r], s0);
      }
      const double wv = warp_sum((s0 + s1) + (s2 + s3));
      //  (c) the diagonal block left of the diagonal: sum_{r0 <= c < i} A(i, c) q_c
      double dc = 0.0;
      for (int cc = r0 + lane; cc < i; cc += 32) dc = fma(a.A[i + (int64_t)cc * a.lda], qsrc[cc], dc);
      dc = warp_sum(dc);
      if (lane == 0) w_own[ii] = wv + dc;
    }
    //  (b) row strip left of the diagonal block: sum_{c < r0} A(i, c) q_c, lanes
    //      over the owned rows (coalesced column segments), warps over columns
    //      in a fixed interleave, partials summed in warp order
    {
      double* rpart = red + 32;  // [NW][chunk]
      for (int rb = 0; rb < nown; rb += 32) {
        const int ii = rb + lane;
        const bool own = ii < nown;
        const double* rowp = a.A + (r0 + (own ? ii : 0));
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int cc = warp;
        for (; cc + 3 * NW < r0; cc += 4 * NW) {
          const double x0 = rowp[(int64_t)cc * a.lda], x1 = rowp[(int64_t)(cc + NW) * a.lda];
          const double x2 = rowp[(int64_t)(cc + 2 * NW) * a.lda], x3 = rowp[(int64_t)(cc + 3 * NW) * a.lda];
          s0 = fma(x0, qsrc[cc], s0);
          s1 = fma(x1, qsrc[cc + NW], s1);
          s2 = fma(x2, qsrc[cc + 2 * NW], s2);
          s3 = fma(x3, qsrc[cc + 3 * NW], s3);
        }
        for (; cc < r0; cc += NW) s0 = fma(rowp[(int64_t)cc * a.lda], qsrc[cc], s0);
        if (own) rpart[warp * chunk + ii] = (s0 + s1) + (s2 + s3);
      }
      __syncthreads();
      for (int ii = tid; ii < nown; ii += kLzThreads) {
        double sm = 0.0;
        for (int k = 0; k < NW; ++k) sm += rpart[k * chunk + ii];
        w_own[ii] = (w_own[ii] + sm) * qs;
      }
      __syncthreads();
    }
    double alpha_acc = 0.0;
    for (int ii = tid; ii < nown; ii += kLzThreads) alpha_acc = fma(qsrc[r0 + ii] * qs, w_own[ii], alpha_acc);
    alpha_acc = warp_sum(alpha_acc);
    if (lane == 0) red[warp] = alpha_acc;
    __syncthreads();
    if (tid == 0) {
      double sa = 0.0;
      for (int k = 0; k < NW; ++k) sa += red[k];
      a.alpha_part[g * 64 + j] = sa;
    }
    // ---- two CGS passes: h = Q(:, 0:j)^T w, w -= Q(:, 0:j) h
    for (int pass = 0; pass < 2; ++pass) {
      double* sl = a.slots + (int64_t)pass * G * 64;
      for (int t = warp; t <= j; t += NW) {
        const double* qt = a.Q + (int64_t)t * a.ldq + r0;
        double sm = 0.0;
        for (int ii = lane; ii < nown; ii += 32) sm = fma(qt[ii], w_own[ii], sm);
        sm = warp_sum(sm);
        if (lane == 0) sl[g * 64 + t] = sm;
      }
      grid_sync(a.bar, epoch);
      // h_t = sum over the G CTAs' slots: every load of a warp's (up to two) t issued
      // before any add (the reduction is L2-latency bound: one round trip, not five)
      for (int t = warp; t <= j; t += 2 * NW) {
        const int t2 = t + NW;
        double v[2][kLzSlotsPerLane];
#pragma unroll
        for (int u = 0; u < kLzSlotsPerLane; ++u) {
          const int gg = lane + 32 * u;
          v[0][u] = gg < G ? __ldcg(&sl[gg * 64 + t]) : 0.0;
          v[1][u] = (gg < G && t2 <= j) ? __ldcg(&sl[gg * 64 + t2]) : 0.0;
        }
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int u = 0; u < kLzSlotsPerLane; ++u) {
          s0 += v[0][u];
          s1 += v[1][u];
        }
        s0 = warp_sum(s0);
        s1 = warp_sum(s1);
        if (lane == 0) {
          hsm[t] = s0;
          if (t2 <= j) hsm[t2] = s1;
        }
      }
      __syncthreads();
      for (int ii = tid; ii < nown; ii += kLzThreads) {
        double sm = 0.0;
        for (int t = 0; t <= j; ++t) sm = fma(a.Q[(int64_t)t * a.ldq + r0 + ii], hsm[t], sm);
        w_own[ii] -= sm;
      }
      __syncthreads();
    }
    // ---- beta^2 = w^T w; publish the unnormalised w for the next product
    double* wout = a.wbuf + (j & 1) * (int64_t)n;
    double b2 = 0.0;
    for (int ii = tid; ii < nown; ii += kLzThreads) {
      const double x = w_own[ii];
      wout[r0 + ii] = x;
      b2 = fma(x, x, b2);
    }
    b2 = block_sum(b2, red);
    double* bs = a.bslots + (j & 1) * G;
    if (tid == 0) bs[g] = b2;
    grid_sync(a.bar, epoch);
    if (warp == 0) {
      double v[kLzSlotsPerLane];
#pragma unroll
      for (int u = 0; u < kLzSlotsPerLane; ++u) v[u] = (lane + 32 * u < G) ? __ldcg(&bs[lane + 32 * u]) : 0.0;
      double sm = 0.0;
#pragma unroll
      for (int u = 0; u < kLzSlotsPerLane; ++u) sm += v[u];
      sm = warp_sum(sm);
      if (lane == 0) hsm[0] = sm;
    }
    __syncthreads();
    const double beta2 = hsm[0];
    if (g == 0 && tid == 0) a.beta2[j] = beta2;
    inv_beta = 1.0 / sqrt(beta2);
    __syncthreads();
  }
}

struct Vec {
  double* p;
};

class Krylov {
 public:
  explicit Krylov(Ctx& c) : ctx(c) {
    nblk = 2 * ctx.num_sms;
    partial = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * nblk));
  }
  void gemv_t(const DMat& A, const double* x, double* z) {
    const int blocks = (int)std::min<int64_t>((A.cols + 7) / 8, 16LL * ctx.num_sms);
    gemv_t_kernel<<<blocks, 256, 0, ctx.stream>>>(A.ptr(), A.ld, A.rows, A.cols, x, z);
    QDWHG_CUDA(cudaGetLastError());
    ctx.count();
  }
  void gemv_n(const DMat& A, const double* x, double* y, double* part, int splits) {
    const int64_t cps = (A.cols + splits - 1) / splits;
    dim3 grid((unsigned)((A.rows + 255) / 256), (unsigned)splits);
    gemv_n_partial_kernel<<<grid, 256, 0, ctx.stream>>>(A.ptr(), A.ld, A.rows, A.cols, x, cps, part);
    reduce_partial_kernel<<<(int)std::min<int64_t>((A.rows + 255) / 256, 4LL * ctx.num_sms), 256, 0,
                            ctx.stream>>>(part, splits, A.rows, y);
    QDWHG_CUDA(cudaGetLastError());
    ctx.count(2);
  }
  void dot(const double* x, const double* y, int64_t n, double* out) {
    const int b = (int)std::min<int64_t>(nblk, std::max<int64_t>(1, (n + 255) / 256));
    dot_partial_kernel<<<b, 256, 0, ctx.stream>>>(x, y, n, partial);
    dot_final_kernel<<<1, 256, 0, ctx.stream>>>(partial, b, out);
    QDWHG_CUDA(cudaGetLastError());
    ctx.count(2);
  }
  Ctx& ctx;
  int nblk;
  double* partial;
};

}  // namespace

double two_norm_estimate(Ctx& ctx, const DMat& A) {
  const int64_t m = A.rows, n = A.cols;
  const MatStats st = mat_stats(ctx, A, false);
  if (st.fro2 == 0.0) throw InvalidArgument("two_norm_estimate: zero matrix");
  const Arena::Mark mark = ctx.arena->mark();
  Krylov K(ctx);
  const std::vector<double> v0 = start_vector(n, 0x6e6f726d32ull);  // kernels.cpp:336
  double* v = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * n));
  double* y = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * m));
  double* z = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * n));
  const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(64, (2LL * ctx.num_sms * 256) / std::max<int64_t>(m, 1)));
  double* part = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * splits * m));
  double* sc = ctx.dscratch;  // [0] = ||y||^2, [1] = ||z||^2
  QDWHG_CUDA(cudaMemcpyAsync(v, v0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx.stream));
  double est = 0.0;
  for (int it = 0; it < 100; ++it) {
    K.gemv_n(A, v, y, part, splits);
    K.dot(y, y, m, sc + 0);
    K.gemv_t(A, y, z);
    K.dot(z, z, n, sc + 1);
    QDWHG_CUDA(cudaMemcpyAsync(ctx.hscratch, sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
    const double ny = std::sqrt(ctx.hscratch[0]);
    if (ny == 0.0) {
      // start vector in the null space: restart from an axis (kernels.cpp:345-350)
      std::vector<double> e(n, 0.0);
      e[it % n] = 1.0;
      QDWHG_CUDA(cudaMemcpyAsync(v, e.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx.stream));
      QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
      continue;
    }
    const double nz = std::sqrt(ctx.hscratch[1]);
    const double prev = est;
    est = ny;
    if (nz == 0.0) break;
    scale_by_invnorm_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4LL * ctx.num_sms), 256, 0,
                              ctx.stream>>>(z, sc + 1, n, v);
    QDWHG_CUDA(cudaGetLastError());
    ctx.count();
    if (it > 0 && std::abs(est - prev) < 1e-3 * est) break;
  }
  ctx.arena->release_to(mark);
  return 1.05 * est;
}

double lanczos_min_bound(Ctx& ctx, const DMat& A, int steps, const MatStats* pre) {
  const int64_t n = A.rows;
  if (A.cols != n) throw InvalidArgument("lanczos_min_bound: matrix not square");
  if (steps < 1) throw InvalidArgument("lanczos_min_bound: steps must be >= 1");
  const MatStats st = pre ? *pre : mat_stats(ctx, A, true);
  const double fro = std::sqrt(st.fro2);
  const double eps = 2.220446049250313e-16;
  if (st.asym > 1e3 * (double)n * eps * std::max(1.0, fro))
    throw InvalidArgument("lanczos_min_bound: input not symmetric within tolerance");
  const int m = (int)std::min<int64_t>(steps, n);
  if (m > 63) throw InvalidArgument("lanczos_min_bound: at most 63 steps supported");
  const Arena::Mark mark = ctx.arena->mark();
  DMat Q = ctx.arena->alloc(n, m + 1);
  const std::vector<double> q0 = start_vector(n, 0x6c616e637aull);  // kernels.cpp:379
  QDWHG_CUDA(cudaMemcpyAsync(Q.ptr(), q0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx.stream));
  // All steps run in one cooperative kernel without host round trips; a
  // breakdown (beta <= tol) is detected afterwards and the recurrence
  // truncated there, exactly like the reference's early exit (later entries
  // are never read).
  // one CTA per SM (co-resident for the grid barriers), at least 16 rows each
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(ctx.num_sms, 32 * kLzSlotsPerLane), n / 16));
  const int chunk = (int)((n + G - 1) / G);
  const size_t smem = (size_t)(chunk + 96 + (kLzThreads / 32) * chunk) * 8;
  if (smem > 200 * 1024) throw InvalidArgument("lanczos_min_bound: matrix too large");
  func_attr(lanczos_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  double* wbuf = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * 2 * n));
  double* slots = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * 2 * G * 64));
  double* bslots = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * 2 * G));
  double* apart = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * G * 64));
  double* beta2 = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * 64));
  unsigned* bar = static_cast<unsigned*>(ctx.arena->alloc_bytes(256));
  QDWHG_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), ctx.stream));
  LanczosArgs la{A.ptr(), A.ld, (int)n, m, Q.ptr(), Q.ld, wbuf, slots, bslots, apart, beta2, bar};
  void* largs[] = {&la};
  QDWHG_CUDA(cudaLaunchCooperativeKernel((void*)lanczos_kernel, dim3(G), dim3(kLzThreads), largs, smem,
                                         ctx.stream));
  ctx.count();
  std::vector<double> hap((size_t)G * 64), hb2(64);
  QDWHG_CUDA(cudaMemcpyAsync(hap.data(), apart, sizeof(double) * G * 64, cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaMemcpyAsync(hb2.data(), beta2, sizeof(double) * 64, cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  std::vector<double> hab(128, 0.0);
  for (int j = 0; j < m; ++j) {
    double sa = 0.0;
    for (int gg = 0; gg < G; ++gg) sa += hap[(size_t)gg * 64 + j];
    hab[j] = sa;
    hab[64 + j] = hb2[j];
  }
  const double breakdown_tol = (double)n * eps * std::max(1.0, fro);
  std::vector<double> alpha, beta;
  double beta_last = 0.0;
  for (int j = 0; j < m; ++j) {
    alpha.push_back(hab[j]);
    const double bj = std::sqrt(hab[64 + j]);
    beta_last = bj;
    if (j + 1 == m || bj <= breakdown_tol) {
      if (bj <= breakdown_tol) beta_last = 0.0;
      break;
    }
    beta.push_back(bj);
  }
  const int k = (int)alpha.size();
  // smallest eigenpair of the tridiagonal T (kernels.cpp:426-433 uses Jacobi on
  // the dense T; T is tridiagonal, so Sturm multisection + inverse iteration on
  // the device give the same theta_min and |s_last| in microseconds)
  double theta = 0.0, s_last = 0.0;
  tridiag_lowest(ctx, alpha, beta, &theta, &s_last);
  double mu = theta - beta_last * std::abs(s_last);
  if (mu < 0.0) mu *= 1.1;
  ctx.arena->release_to(mark);
  return mu;
}

}  // namespace qdwhg
