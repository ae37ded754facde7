// HBM-bound O(n^2) passes of the QDWHpartial path, each one fused pass:
//   scaled/add/symmetrize/shift   (matrix.cpp:72-105, partial.cpp:55-58, 67-68, 134-135)
//   require_finite / symmetry check / frobenius norm (matrix.cpp:114-145, partial.cpp:15-22)
//   counter-based Gaussian (kernels.cpp:14-32, 441-447; device log/cos, not bit-identical)
// Grids are sized to a multiple of the SM count; columns are walked by warps
// so every access is a coalesced column segment.
#include "common.cuh"
#include "internal.hpp"

namespace qdwhg {

namespace {

inline int grid_for(Ctx& ctx, int64_t elems, int threads) {
  int64_t want = (elems + threads - 1) / threads;
  int64_t cap = 8LL * ctx.num_sms;
  return (int)std::max<int64_t>(1, std::min(want, cap));
}

__global__ void fill_kernel(double* X, int64_t ld, int64_t m, int64_t n, double v, double diag) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    X[i + j * ld] = v + (i == j ? diag : 0.0);
  }
}

__global__ void axpby_identity_kernel(const double* X, int64_t ldx, double* Y, int64_t ldy,
                                      int64_t m, int64_t n, double a, double diag) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    Y[i + j * ldy] = a * X[i + j * ldx] + (i == j ? diag : 0.0);
  }
}

// Y(i,j) = a * 0.5 * (X(i,j) + X(j,i)) + diag*[i==j].  Processes 32x32 tiles
// pairwise through shared memory so both reads are coalesced; in-place safe
// because each (tile, mirror tile) pair is owned by one block.
// Y = a sym(X) + diag I and, when Y2 != nullptr, Y2 = a2 Y + diag2 I from the
// same read (the EIG driver's A/|mu| and (1-s) A/|mu| - s I in one pass)
__global__ void symmetrize_kernel(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t n,
                                  double a, double diag, double* Y2, int64_t ldy2, double a2,
                                  double diag2) {
  __shared__ double t1[32][33], t2[32][33];
  const int64_t nt = (n + 31) / 32;
  const int64_t npairs = nt * (nt + 1) / 2;
  for (int64_t pid = blockIdx.x; pid < npairs; pid += gridDim.x) {
    // pid -> (ti >= tj)
    int64_t tj = 0, rem = pid;
    while (rem >= nt - tj) {
      rem -= nt - tj;
      ++tj;
    }
    const int64_t ti = tj + rem;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
      const int64_t i1 = ti * 32 + tx, j1 = tj * 32 + r;  // tile (ti,tj) element (tx, r)
      t1[r][tx] = (i1 < n && j1 < n) ? X[i1 + j1 * ldx] : 0.0;
      const int64_t i2 = tj * 32 + tx, j2 = ti * 32 + r;  // tile (tj,ti)
      t2[r][tx] = (i2 < n && j2 < n) ? X[i2 + j2 * ldx] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      // element (ti*32+tx, tj*32+r): X(i,j) = t1[r][tx], X(j,i) = t2[tx][r]
      const int64_t i1 = ti * 32 + tx, j1 = tj * 32 + r;
      if (i1 < n && j1 < n) {
        const double v = a * (0.5 * (t1[r][tx] + t2[tx][r])) + (i1 == j1 ? diag : 0.0);
        Y[i1 + j1 * ldy] = v;
        if (Y2) Y2[i1 + j1 * ldy2] = a2 * v + (i1 == j1 ? diag2 : 0.0);
      }
      const int64_t i2 = tj * 32 + tx, j2 = ti * 32 + r;
      if (ti != tj && i2 < n && j2 < n) {
        const double v = a * (0.5 * (t2[r][tx] + t1[tx][r]));
        Y[i2 + j2 * ldy] = v;
        if (Y2) Y2[i2 + j2 * ldy2] = a2 * v;
      }
    }
    __syncthreads();
  }
}

__global__ void copy_kernel(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t m,
                            int64_t n) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    Y[i + j * ldy] = X[i + j * ldx];
  }
}

// Y = X^T through 32x32 shared-memory tiles (both sides coalesced)
__global__ void transpose_kernel(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t m,
                                 int64_t n) {
  __shared__ double t[32][33];
  const int64_t i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;  // tile of X: rows i0.., cols j0..
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 256 threads: 8 rows per pass
  for (int r = ty; r < 32; r += 8)
    if (i0 + tx < m && j0 + r < n) t[r][tx] = X[(i0 + tx) + (j0 + r) * ldx];
  __syncthreads();
  for (int r = ty; r < 32; r += 8)
    if (j0 + tx < n && i0 + r < m) Y[(j0 + tx) + (i0 + r) * ldy] = t[tx][r];
}

// per-block partials: [0] sum x^2, [1] max |x_ij - x_ji|, [2] nonfinite count, [3] max |x|
__global__ void stats_kernel(const double* X, int64_t ld, int64_t m, int64_t n, int want_asym,
                             double* partial) {
  __shared__ double scratch[32];
  double s = 0.0, asym = 0.0, nf = 0.0, mx = 0.0;
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    const double x = X[i + j * ld];
    if (!isfinite(x)) {
      nf += 1.0;
    } else {
      s += x * x;
      mx = fmax(mx, fabs(x));
    }
    if (want_asym && i < j) asym = fmax(asym, fabs(x - X[j + i * ld]));
  }
  s = block_sum(s, scratch);
  __syncthreads();
  asym = block_max(asym, scratch);
  __syncthreads();
  nf = block_sum(nf, scratch);
  __syncthreads();
  mx = block_max(mx, scratch);
  if (threadIdx.x == 0) {
    partial[4 * blockIdx.x + 0] = s;
    partial[4 * blockIdx.x + 1] = asym;
    partial[4 * blockIdx.x + 2] = nf;
    partial[4 * blockIdx.x + 3] = mx;
  }
}

__global__ void stats_final_kernel(const double* partial, int nblk, double* out) {
  __shared__ double scratch[32];
  double s = 0, a = 0, nf = 0, mx = 0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    s += partial[4 * b];
    a = fmax(a, partial[4 * b + 1]);
    nf += partial[4 * b + 2];
    mx = fmax(mx, partial[4 * b + 3]);
  }
  s = block_sum(s, scratch);
  __syncthreads();
  a = block_max(a, scratch);
  __syncthreads();
  nf = block_sum(nf, scratch);
  __syncthreads();
  mx = block_max(mx, scratch);
  if (threadIdx.x == 0) {
    out[0] = s;
    out[1] = a;
    out[2] = nf;
    out[3] = mx;
  }
}

QDWHG_DEV uint64_t hash64(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gaussian_kernel(double* X, int64_t ld, int64_t m, int64_t n, uint64_t seed) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    const double u1 = (double)((hash64(seed, 2ull * idx) >> 11) + 1ull) * 0x1.0p-53;
    const double u2 = (double)((hash64(seed, 2ull * idx + 1ull) >> 11) + 1ull) * 0x1.0p-53;
    X[i + j * ld] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

__global__ void mirror_kernel(double* X, int64_t ld, int64_t n) {
  // upper (i < j) <- lower (j, i)
  const int64_t total = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    if (i < j) X[i + j * ld] = X[j + i * ld];
  }
}

__global__ void zero_strict_lower_kernel(double* X, int64_t ld, int64_t m, int64_t n) {
  // block per column (grid-stride), threads down the rows below the diagonal
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x)
    for (int64_t i = j + 1 + threadIdx.x; i < m; i += blockDim.x) X[i + j * ld] = 0.0;
}

}  // namespace

void fill(Ctx& ctx, const DMat& X, double v, double diag) {
  if (X.rows * X.cols == 0) return;
  fill_kernel<<<grid_for(ctx, X.rows * X.cols, 256), 256, 0, ctx.stream>>>(X.ptr(), X.ld, X.rows,
                                                                           X.cols, v, diag);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void axpby_identity(Ctx& ctx, const DMat& X, double a, double diag, const DMat& Y) {
  if (X.rows * X.cols == 0) return;
  axpby_identity_kernel<<<grid_for(ctx, X.rows * X.cols, 256), 256, 0, ctx.stream>>>(
      X.ptr(), X.ld, Y.ptr(), Y.ld, X.rows, X.cols, a, diag);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void symmetrize_scale(Ctx& ctx, const DMat& X, double a, double diag, const DMat& Y) {
  if (X.rows != X.cols) throw InvalidArgument("symmetrize: matrix not square");
  const int64_t nt = (X.rows + 31) / 32;
  const int64_t npairs = nt * (nt + 1) / 2;
  const int blocks = (int)std::min<int64_t>(npairs, 8LL * ctx.num_sms);
  symmetrize_kernel<<<blocks, 256, 0, ctx.stream>>>(X.ptr(), X.ld, Y.ptr(), Y.ld, X.rows, a, diag,
                                                    nullptr, 0, 0.0, 0.0);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void symmetrize_scale2(Ctx& ctx, const DMat& X, double a, double diag, const DMat& Y, double a2,
                       double diag2, const DMat& Y2) {
  if (X.rows != X.cols) throw InvalidArgument("symmetrize: matrix not square");
  const int64_t nt = (X.rows + 31) / 32;
  const int64_t npairs = nt * (nt + 1) / 2;
  const int blocks = (int)std::min<int64_t>(npairs, 8LL * ctx.num_sms);
  symmetrize_kernel<<<blocks, 256, 0, ctx.stream>>>(X.ptr(), X.ld, Y.ptr(), Y.ld, X.rows, a, diag,
                                                    Y2.ptr(), Y2.ld, a2, diag2);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void copy(Ctx& ctx, const DMat& X, const DMat& Y) {
  if (X.rows * X.cols == 0) return;
  copy_kernel<<<grid_for(ctx, X.rows * X.cols, 256), 256, 0, ctx.stream>>>(X.ptr(), X.ld, Y.ptr(),
                                                                           Y.ld, X.rows, X.cols);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void transpose(Ctx& ctx, const DMat& X, const DMat& Y) {
  if (X.rows * X.cols == 0) return;
  dim3 grid((unsigned)((X.rows + 31) / 32), (unsigned)((X.cols + 31) / 32));
  transpose_kernel<<<grid, 256, 0, ctx.stream>>>(X.ptr(), X.ld, Y.ptr(), Y.ld, X.rows, X.cols);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void copy_from_host(Ctx& ctx, const double* h, int64_t ldh, const DMat& Y) {
  QDWHG_CUDA(cudaMemcpy2DAsync(Y.ptr(), Y.ld * 8, h, ldh * 8, Y.rows * 8, Y.cols,
                               cudaMemcpyHostToDevice, ctx.stream));
}

void copy_to_host(Ctx& ctx, const DMat& X, double* h, int64_t ldh) {
  QDWHG_CUDA(cudaMemcpy2DAsync(h, ldh * 8, X.ptr(), X.ld * 8, X.rows * 8, X.cols,
                               cudaMemcpyDeviceToHost, ctx.stream));
}

// Square matrices with the symmetry check: 32x32 tile pairs (T_ij, T_ji) through
// shared memory, so both the direct and the transposed reads are coalesced.
__global__ void stats_sym_kernel(const double* X, int64_t ld, int64_t n, double* partial) {
  __shared__ double scratch[32];
  __shared__ double t1[32][33], t2[32][33];
  const int64_t nt = (n + 31) / 32;
  const int64_t npairs = nt * (nt + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 rows per pass
  double s = 0.0, asym = 0.0, nf = 0.0, mx = 0.0;
  // contiguous chunk of the column-major lower-tile enumeration per block: the
  // (ti, tj) of the first pair is found once, then stepped
  const int64_t chunk = (npairs + gridDim.x - 1) / gridDim.x;
  const int64_t p0 = blockIdx.x * chunk, p1 = min(npairs, p0 + chunk);
  int64_t tj = 0, ti = 0;
  {
    int64_t rem = p0;
    while (tj < nt && rem >= nt - tj) {
      rem -= nt - tj;
      ++tj;
    }
    ti = tj + rem;
  }
  for (int64_t pidx = p0; pidx < p1; ++pidx, ++ti) {
    if (ti >= nt) {
      ++tj;
      ti = tj;
    }
    const int64_t i0 = ti * 32, j0 = tj * 32;
    for (int r = ty; r < 32; r += 8) {
      // t1(r, tx) = X(i0 + tx, j0 + r) (column j0+r of tile ij), t2 likewise for tile ji
      const int64_t ia = i0 + tx, ja = j0 + r, ib = j0 + tx, jb = i0 + r;
      t1[r][tx] = (ia < n && ja < n) ? X[ia + ja * ld] : 0.0;
      t2[r][tx] = (ib < n && jb < n) ? X[ib + jb * ld] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int64_t ia = i0 + tx, ja = j0 + r;
      if (ia < n && ja < n) {
        const double x = t1[r][tx];  // X(ia, ja), ia >= ja region of the pair
        if (!isfinite(x)) nf += 1.0;
        else {
          s += x * x;
          mx = fmax(mx, fabs(x));
        }
        // X(ja, ia) = t2(tx, r)
        if (ti != tj || tx > r) asym = fmax(asym, fabs(x - t2[tx][r]));
      }
      if (ti != tj) {  // the transposed tile's own entries
        const int64_t ib = j0 + tx, jb = i0 + r;
        if (ib < n && jb < n) {
          const double y = t2[r][tx];
          if (!isfinite(y)) nf += 1.0;
          else {
            s += y * y;
            mx = fmax(mx, fabs(y));
          }
        }
      }
    }
    __syncthreads();
  }
  s = block_sum(s, scratch);
  __syncthreads();
  asym = block_max(asym, scratch);
  __syncthreads();
  nf = block_sum(nf, scratch);
  __syncthreads();
  mx = block_max(mx, scratch);
  if (threadIdx.x == 0) {
    partial[4 * blockIdx.x + 0] = s;
    partial[4 * blockIdx.x + 1] = asym;
    partial[4 * blockIdx.x + 2] = nf;
    partial[4 * blockIdx.x + 3] = mx;
  }
}

MatStats mat_stats(Ctx& ctx, const DMat& X, bool want_asym) {
  MatStats st;
  if (X.rows * X.cols == 0) return st;
  int blocks = std::min(grid_for(ctx, X.rows * X.cols, 256), 2 * ctx.num_sms);
  double* partial = ctx.dscratch + 64;
  if (want_asym && X.rows == X.cols) {
    const int64_t nt = (X.rows + 31) / 32;
    blocks = (int)std::max<int64_t>(1, std::min<int64_t>(nt * (nt + 1) / 2, 4LL * ctx.num_sms));
    stats_sym_kernel<<<blocks, 256, 0, ctx.stream>>>(X.ptr(), X.ld, X.rows, partial);
  } else {
    stats_kernel<<<blocks, 256, 0, ctx.stream>>>(X.ptr(), X.ld, X.rows, X.cols, want_asym ? 1 : 0,
                                                 partial);
  }
  stats_final_kernel<<<1, 256, 0, ctx.stream>>>(partial, blocks, ctx.dscratch);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count(2);
  QDWHG_CUDA(cudaMemcpyAsync(ctx.hscratch, ctx.dscratch, 4 * 8, cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  st.fro2 = ctx.hscratch[0];
  st.asym = ctx.hscratch[1];
  st.nonfinite = ctx.hscratch[2];
  st.maxabs = ctx.hscratch[3];
  return st;
}

void gaussian_fill(Ctx& ctx, const DMat& X, uint64_t seed) {
  if (X.rows * X.cols == 0) return;
  gaussian_kernel<<<grid_for(ctx, X.rows * X.cols, 256), 256, 0, ctx.stream>>>(X.ptr(), X.ld,
                                                                               X.rows, X.cols, seed);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void mirror_lower_to_upper(Ctx& ctx, const DMat& X) {
  mirror_kernel<<<grid_for(ctx, X.rows * X.rows, 256), 256, 0, ctx.stream>>>(X.ptr(), X.ld, X.rows);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void zero_strict_lower(Ctx& ctx, const DMat& X) {
  zero_strict_lower_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(X.cols, 8LL * ctx.num_sms)), 256, 0,
                             ctx.stream>>>(X.ptr(), X.ld, X.rows, X.cols);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

}  // namespace qdwhg
