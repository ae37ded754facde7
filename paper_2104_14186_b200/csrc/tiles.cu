// Local-array kernels of the distributed driver (HBM-bound):
//   * batched tile copies (pack / unpack / place of broadcast panels, optional
//     transpose through 32x32 shared-memory tiles) — one launch per batch of up
//     to kMaxBatch tiles, descriptors passed by value (no upload),
//   * Y = a X + b Y, diagonal adds, strict-triangle zeroing,
//   * the counter-based Gaussian at global coordinates (a tile of the global
//     matrix draws the same entries as the whole-matrix generator).
#include "common.cuh"
#include "internal.hpp"

namespace qdwhg {

namespace {

constexpr int kMaxBatch = 400;
struct TileBatch {
  int count;
  TileDesc d[kMaxBatch];
};

__global__ void __launch_bounds__(256) copy_tiles_kernel(const TileBatch b) {
  const TileDesc t = b.d[blockIdx.y];
  if (!t.trans) {
    // block-strided columns, threads down the rows (coalesced both sides)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c = blockIdx.x * 8 + warp; c < t.cols; c += gridDim.x * 8) {
      const double* s = t.src + (int64_t)c * t.lds;
      double* d = t.dst + (int64_t)c * t.ldd;
      for (int r = lane; r < t.rows; r += 32) d[r] = s[r];
    }
    return;
  }
  // transpose: dst (cols x rows) = src^T, 32 x 32 sub-tiles through shared memory
  __shared__ double sm[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int sr = (t.rows + 31) / 32, sc = (t.cols + 31) / 32;
  for (int st = blockIdx.x; st < sr * sc; st += gridDim.x) {
    const int r0 = (st % sr) * 32, c0 = (st / sr) * 32;
    for (int k = ty; k < 32; k += 8) {
      const int r = r0 + tx, c = c0 + k;
      if (r < t.rows && c < t.cols) sm[k][tx] = t.src[r + (int64_t)c * t.lds];
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
      const int c = c0 + tx, r = r0 + k;  // dst(c, r) = src(r, c)
      if (r < t.rows && c < t.cols) t.dst[c + (int64_t)r * t.ldd] = sm[tx][k];
    }
    __syncthreads();
  }
}

__global__ void axpby_kernel(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t m, int64_t n,
                             double a, double b) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); c < n; c += warps) {
    double* y = Y + c * ldy;
    const double* x = X ? X + c * ldx : nullptr;
    for (int64_t r = lane; r < m; r += 32) {
      const double xv = x ? a * x[r] : 0.0;
      y[r] = b == 0.0 ? xv : fma(b, y[r], xv);
    }
  }
}

__global__ void add_diag_kernel(double* Y, int64_t ld, int64_t len, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
    Y[i + i * ld] += v;
}

__global__ void zero_strict_upper_kernel(double* X, int64_t ld, int64_t m, int64_t n) {
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x)
    for (int64_t i = threadIdx.x; i < j && i < m; i += blockDim.x) X[i + j * ld] = 0.0;
}

QDWHG_DEV uint64_t hash64_g(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gaussian_at_kernel(double* X, int64_t ld, int64_t m, int64_t n, uint64_t seed, int64_t gr0,
                                   int64_t gc0, int64_t gm) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m, j = idx / m;
    const uint64_t g = (uint64_t)((gr0 + i) + (gc0 + j) * gm);  // column-major global index
    const double u1 = (double)((hash64_g(seed, 2ull * g) >> 11) + 1ull) * 0x1.0p-53;
    const double u2 = (double)((hash64_g(seed, 2ull * g + 1ull) >> 11) + 1ull) * 0x1.0p-53;
    X[i + j * ld] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

int grid_cap(Ctx& ctx, int64_t want) { return (int)std::max<int64_t>(1, std::min<int64_t>(want, 8LL * ctx.num_sms)); }

}  // namespace

void copy_tiles(Ctx& ctx, const std::vector<TileDesc>& list) {
  static TileBatch b;  // (host staging for the by-value parameter)
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  for (size_t s = 0; s < list.size(); s += kMaxBatch) {
    const int cnt = (int)std::min<size_t>(kMaxBatch, list.size() - s);
    b.count = cnt;
    int64_t maxel = 0;
    for (int i = 0; i < cnt; ++i) {
      b.d[i] = list[s + i];
      maxel = std::max<int64_t>(maxel, (int64_t)b.d[i].rows * b.d[i].cols);
    }
    if (maxel == 0) continue;
    // ~8K elements per block, at least one wave over the machine per batch
    const int bx = (int)std::max<int64_t>(1, std::min<int64_t>((maxel + 8191) / 8192,
                                                                std::max<int64_t>(1, 2LL * ctx.num_sms / cnt)));
    copy_tiles_kernel<<<dim3(bx, cnt), 256, 0, ctx.stream>>>(b);
    QDWHG_CUDA(cudaGetLastError());
    ctx.count();
  }
}

void axpby(Ctx& ctx, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t m, int64_t n, double a,
           double b) {
  if (m <= 0 || n <= 0) return;
  axpby_kernel<<<grid_cap(ctx, (n + 7) / 8), 256, 0, ctx.stream>>>(X, ldx, Y, ldy, m, n, a, b);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void add_diag(Ctx& ctx, double* Y, int64_t ld, int64_t len, double v) {
  if (len <= 0) return;
  add_diag_kernel<<<grid_cap(ctx, (len + 255) / 256), 256, 0, ctx.stream>>>(Y, ld, len, v);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void zero_strict_upper(Ctx& ctx, const DMat& X) {
  if (X.rows * X.cols == 0) return;
  zero_strict_upper_kernel<<<grid_cap(ctx, X.cols), 256, 0, ctx.stream>>>(X.ptr(), X.ld, X.rows, X.cols);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void gaussian_fill_at(Ctx& ctx, double* X, int64_t ld, int64_t m, int64_t n, uint64_t seed, int64_t gr0,
                      int64_t gc0, int64_t gm) {
  if (m * n == 0) return;
  gaussian_at_kernel<<<grid_cap(ctx, (m * n + 255) / 256), 256, 0, ctx.stream>>>(X, ld, m, n, seed, gr0, gc0, gm);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

}  // namespace qdwhg
