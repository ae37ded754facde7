// Dense symmetric eigensolver for the Rayleigh-Ritz block (partial.cpp:80-81),
// the 30x30 Lanczos tridiagonal (kernels.cpp:426-438) and the leaves of the
// spectral divide-and-conquer.  Reference: cyclic Jacobi sym_eig_dense,
// kernels.cpp:148-215 — same rotation formula, same skip threshold
// rotate_tol = 0.5*u*||S||_F/n, same "stop after a sweep without rotations",
// at most 64 sweeps, ascending order.
//
// B200 shape: one CTA, the matrix lives in shared memory (n <= kJacobiMax), the
// n/2 disjoint rotations of a round-robin round are computed and applied in
// parallel (A <- J^T A J, V <- V J) — 3 barriers per round instead of n/2
// sequential rotations.
#include <algorithm>
#include <numeric>

#include "common.cuh"
#include "internal.hpp"

namespace qdwhg {

constexpr int kJacobiMax = 160;
extern const int kJacobiMaxN = kJacobiMax;

namespace {

constexpr int kJThreads = 512;

QDWHG_DEV int rr_index(int pos, int r, int ne) {
  return pos == 0 ? 0 : ((pos - 1 + r) % (ne - 1)) + 1;
}

// A (n x n, lda) -> eigenvalues (unsorted, diag of the converged matrix) in
// evals, eigenvectors V (n x n, ldv).  info[0] = sweeps, info[1] = rotations.
__global__ void __launch_bounds__(kJThreads, 1)
    jacobi_kernel(const double* A, int64_t lda, double* V, int64_t ldv, double* evals, int n,
                  int* info) {
  extern __shared__ double sm[];
  const int LDS = n + 1;
  double* S = sm;                           // column-major S[c*LDS + r]
  double* rc = S + (size_t)n * LDS;         // per pair c
  double* rs = rc + kJacobiMax / 2 + 1;     // per pair s
  int* rp = reinterpret_cast<int*>(rs + kJacobiMax / 2 + 1);
  int* rq = rp + kJacobiMax / 2 + 1;
  __shared__ double scratch[32];
  __shared__ int rot_count;
  const int tid = threadIdx.x;

  double fro2 = 0.0;
  for (int i = tid; i < n * n; i += kJThreads) {
    const int r = i % n, c = i / n;
    const double a = A[r + (int64_t)c * lda];
    const double b = A[c + (int64_t)r * lda];
    const double v = 0.5 * (a + b);  // symmetrize (kernels.cpp:161)
    S[c * LDS + r] = v;
    fro2 += a * a;
    V[r + (int64_t)c * ldv] = (r == c) ? 1.0 : 0.0;
  }
  const double norm = sqrt(block_sum(fro2, scratch));
  __syncthreads();
  const double rotate_tol = 0.5 * 2.220446049250313e-16 * norm / (double)n;
  const int ne = n + (n & 1);  // even count with a dummy index for odd n
  const int npairs = ne / 2;
  int sweeps = 0, total_rot = 0;
  if (norm > 0.0 && n > 1) {
    for (int sweep = 0; sweep < 64; ++sweep) {
      if (tid == 0) rot_count = 0;
      __syncthreads();
      for (int r = 0; r < ne - 1; ++r) {
        // 1. rotation parameters per pair
        if (tid < npairs) {
          int a = rr_index(tid, r, ne), b = rr_index(ne - 1 - tid, r, ne);
          int p = min(a, b), q = max(a, b);
          double c = 1.0, s = 0.0;
          bool act = false;
          if (q < n) {
            const double apq = S[q * LDS + p];
            if (fabs(apq) > rotate_tol) {
              act = true;
              const double app = S[p * LDS + p], aqq = S[q * LDS + q];
              const double theta = (aqq - app) / (2.0 * apq);
              const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
              c = 1.0 / sqrt(1.0 + t * t);
              s = t * c;
            }
          }
          rp[tid] = act ? p : -1;
          rq[tid] = q;
          rc[tid] = c;
          rs[tid] = s;
          if (act) atomicAdd(&rot_count, 1);
        }
        __syncthreads();
        // 2. columns: A <- A J, V <- V J
        for (int i = tid; i < npairs * n; i += kJThreads) {
          const int k = i / n, row = i % n;
          const int p = rp[k];
          if (p < 0) continue;
          const int q = rq[k];
          const double c = rc[k], s = rs[k];
          const double akp = S[p * LDS + row], akq = S[q * LDS + row];
          S[p * LDS + row] = c * akp - s * akq;
          S[q * LDS + row] = s * akp + c * akq;
          const double vkp = V[row + (int64_t)p * ldv], vkq = V[row + (int64_t)q * ldv];
          V[row + (int64_t)p * ldv] = c * vkp - s * vkq;
          V[row + (int64_t)q * ldv] = s * vkp + c * vkq;
        }
        __syncthreads();
        // 3. rows: A <- J^T A
        for (int i = tid; i < npairs * n; i += kJThreads) {
          const int k = i / n, col = i % n;
          const int p = rp[k];
          if (p < 0) continue;
          const int q = rq[k];
          const double c = rc[k], s = rs[k];
          const double apk = S[col * LDS + p], aqk = S[col * LDS + q];
          S[col * LDS + p] = c * apk - s * aqk;
          S[col * LDS + q] = s * apk + c * aqk;
        }
        __syncthreads();
        if (tid < npairs && rp[tid] >= 0) {
          const int p = rp[tid], q = rq[tid];
          S[q * LDS + p] = 0.0;
          S[p * LDS + q] = 0.0;
        }
        __syncthreads();
      }
      ++sweeps;
      total_rot += rot_count;
      const int rc_now = rot_count;
      __syncthreads();
      if (rc_now == 0) break;
    }
  }
  for (int i = tid; i < n; i += kJThreads) evals[i] = S[i * LDS + i];
  if (tid == 0) {
    info[0] = sweeps;
    info[1] = total_rot;
  }
}

// Vout(:, j) = V(:, order[j])
__global__ void permute_cols_kernel(const double* V, int64_t ldv, const int* order, double* Vo,
                                    int64_t ldo, int64_t m, int64_t n) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    Vo[i + j * ldo] = V[i + (int64_t)order[j] * ldv];
  }
}

}  // namespace

// Vout(:, j) = V(:, order[j]) for a host permutation.
void permute_cols(Ctx& ctx, const DMat& V, const std::vector<int>& order, const DMat& Vout) {
  const int64_t n = (int64_t)order.size();
  int* od = static_cast<int*>(ctx.arena->alloc_bytes(sizeof(int) * (n + 1)));
  QDWHG_CUDA(cudaMemcpyAsync(od, order.data(), sizeof(int) * n, cudaMemcpyHostToDevice, ctx.stream));
  const int64_t total = V.rows * n;
  permute_cols_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 8 * 148)), 256, 0,
                        ctx.stream>>>(V.ptr(), V.ld, od, Vout.ptr(), Vout.ld, V.rows, n);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
}

void syev_jacobi(Ctx& ctx, const DMat& S, std::vector<double>& vals, const DMat& Vout) {
  const int n = (int)S.rows;
  if (n > kJacobiMax) throw InvalidArgument("syev_jacobi: n exceeds the single-CTA limit");
  const size_t smem = ((size_t)n * (n + 1) + 2 * (kJacobiMax / 2 + 1)) * 8 + 2 * (kJacobiMax / 2 + 1) * 4;
  func_attr(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
            (int)(((size_t)kJacobiMax * (kJacobiMax + 1) + 2 * (kJacobiMax / 2 + 1)) * 8 +
                  2 * (kJacobiMax / 2 + 1) * 4));
  const Arena::Mark mark = ctx.arena->mark();
  DMat Vt = ctx.arena->alloc(n, n);
  double* ev = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (n + 1)));
  int* info = static_cast<int*>(ctx.arena->alloc_bytes(64));
  int* order_d = static_cast<int*>(ctx.arena->alloc_bytes(sizeof(int) * (n + 1)));
  jacobi_kernel<<<1, kJThreads, smem, ctx.stream>>>(S.ptr(), S.ld, Vt.ptr(), Vt.ld, ev, n, info);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
  std::vector<double> d(n);
  QDWHG_CUDA(cudaMemcpyAsync(d.data(), ev, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  // ascending sort (kernels.cpp:203-214), ties keep std::sort semantics
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int i, int j) { return d[i] < d[j]; });
  vals.resize(n);
  for (int j = 0; j < n; ++j) vals[j] = d[order[j]];
  QDWHG_CUDA(cudaMemcpyAsync(order_d, order.data(), sizeof(int) * n, cudaMemcpyHostToDevice,
                             ctx.stream));
  permute_cols_kernel<<<std::max(1, std::min(148, (n * n + 255) / 256)), 256, 0, ctx.stream>>>(
      Vt.ptr(), Vt.ld, order_d, Vout.ptr(), Vout.ld, n, n);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  ctx.arena->release_to(mark);
}

}  // namespace qdwhg
