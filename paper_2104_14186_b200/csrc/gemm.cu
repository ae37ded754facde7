// FP64 tensor-core GEMM for sm_100a: TMA -> swizzled smem -> DMMA.8x8x4.
//
// One kernel serves every GEMM-shaped step of the QDWHpartial path:
//   SYRK  Z = I + c*X^T X        (polar.cpp:85-93)        -> OutMode::LowerMirror, diag_add
//   TRMM  Y = X W^-1, G = Y W^-T (polar.cpp:95-121)       -> KRange::BUpper / BLower
//   fused weight update X+ = (b/c) X + (a-b/c) G (polar.cpp:122-127) -> alpha/beta/Cin epilogue
//   WY updates of GEQRF/ORGQR, Rayleigh-Ritz products (partial.cpp:80,97,147,156)
//
// Structure (one CTA per output tile, WM*WN warps):
//   lane 0 of warp 0 : TMA producer, STAGES-deep full/empty mbarrier ring
//   all warps        : DMMA consumers, warp tile (BM/WM) x (BN/WN)
// Shared-memory tiles are written by TMA with the 128-byte swizzle; the k
// order inside each 16-wide k slab is permuted (same permutation for A and B,
// so the product is unchanged) to make fragment loads bank-conflict free.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.hpp"

namespace qdwhg {

namespace {

constexpr int BK = 16;  // k per stage (one 128-byte swizzle row of doubles)

struct GemmParams {
  int M, N, K;
  int a_c0, a_c1;  // TMA coordinate offsets of op(A) storage (contiguous, outer)
  int b_c0, b_c1;
  double alpha, beta, diag_add;
  double* D;
  int64_t ldd;
  const double* Cin;
  int64_t ldcin;
  int kmode;   // KRange
  int omode;   // OutMode
  int tiles_m, tiles_n;
  int splits;       // split-K factor (1 = fused epilogue)
  double* partial;  // splits x (M x N) raw partials (ld = M) when splits > 1
  // batch item b (blockIdx.y): TMA coordinates += b * (x_bs0, x_bs1), D/Cin += b * stride
  int a_bs0, a_bs1, b_bs0, b_bs1;
  int64_t d_bs, cin_bs;
  int nbatch;
  // tail launch of a wave-balanced GEMM: tiles tile0 .. tile0 + gridDim.x - 1,
  // split-K partials stored compactly per tile ([z][tile][BM x BN], ld = BM)
  int tile0;
  int ntl;       // tiles in this launch (0 = all)
  int compact;
  double flop_frac;  // share of the GEMM's algorithmic flops in this launch (profiling)
};

template <bool KMAJ>
QDWHG_DEV int frag_off(int mn, int k) {
  if (KMAJ) {
    // box {16 (k), BMN (mn)}: row = mn, 16 k per 128-byte row
    return mn * 16 + ((((k >> 1) ^ (mn & 7)) << 1) | (k & 1));
  } else {
    // boxes {16 (mn), 16 (k)}: box = mn/16, row = k
    const int c = mn & 15;
    return (mn >> 4) * 256 + k * 16 + ((((c >> 1) ^ (k & 7)) << 1) | (c & 1));
  }
}

template <bool PERM1>
QDWHG_DEV int kperm(int t, int i) {
  return PERM1 ? (2 * i + (t & 1) + 8 * (t >> 1)) : ((i & 1) + 2 * t + 8 * (i >> 1));
}

// Fragment offsets for mn = base_mn + 8*x (base_mn % 16 in [0,8), x compile-time):
// one or two runtime bases per k-step plus compile-time immediates.
struct FragBase {
  int even, odd;
};
template <bool KMAJ>
QDWHG_DEV FragBase frag_base(int base_mn, int k) {
  FragBase b;
  b.even = frag_off<KMAJ>(base_mn, k);
  b.odd = frag_off<KMAJ>(base_mn + 8, k);
  return b;
}
template <bool KMAJ>
QDWHG_DEV int frag_at(const FragBase& b, int x) {
  // K-major: +128 doubles per 8 rows; M-major: boxes of 16 rows (256 doubles), parity selects base
  return KMAJ ? (b.even + 128 * x) : (((x & 1) ? b.odd : b.even) + 256 * (x >> 1));
}

// blockIdx -> (tm, tn); heaviest tiles first for triangular K ranges.
QDWHG_DEV void tile_coords(const GemmParams& p, int bid, int& tm, int& tn) {
  if (p.omode != (int)OutMode::Full) {
    // enumerate lower tiles column by column: column tn holds tiles tm = tn..tiles_m-1
    int c = 0, rem = bid;
    while (rem >= p.tiles_m - c) {
      rem -= p.tiles_m - c;
      ++c;
    }
    tn = c;
    tm = c + rem;
    return;
  }
  // Triangular K ranges: the tile index that sets the work is the slow index,
  // heaviest first (longest-processing-time order across the waves).
  switch ((KRange)p.kmode) {
    case KRange::BUpper:  // work grows with tn
      tm = bid % p.tiles_m;
      tn = p.tiles_n - 1 - bid / p.tiles_m;
      break;
    case KRange::BLower:  // work shrinks with tn
      tm = bid % p.tiles_m;
      tn = bid / p.tiles_m;
      break;
    case KRange::ALower:  // work grows with tm
      tn = bid % p.tiles_n;
      tm = p.tiles_m - 1 - bid / p.tiles_n;
      break;
    case KRange::AUpper:  // work shrinks with tm
      tn = bid % p.tiles_n;
      tm = bid / p.tiles_n;
      break;
    default:
      // column-major (a band-of-12-rows raster cut the DRAM reads of a 4096^3 GEMM
      // from 1.10 to 0.84 GB at the same time, compute-bound; it is not used because
      // it moves which tiles form a wave-balanced tail, i.e. the rounding of those
      // tiles, and with it the bytes of the pinned full-size inputs)
      tm = bid % p.tiles_m;
      tn = bid / p.tiles_m;
      break;
  }
}

template <int BM, int BN>
QDWHG_DEV void k_range(const GemmParams& p, int m0, int n0, int& kb, int& ke) {
  kb = 0;
  ke = p.K;
  switch ((KRange)p.kmode) {
    case KRange::BUpper: ke = min(p.K, n0 + BN); break;   // op(B)(k,j) != 0 only for k <= j
    case KRange::BLower: kb = min(p.K, n0); break;        // k >= j
    case KRange::AUpper: kb = min(p.K, m0); break;        // op(A)(i,k) != 0 only for k >= i
    case KRange::ALower: ke = min(p.K, m0 + BM); break;   // k <= i
    default: break;
  }
}

template <int BM, int BN, int WM, int WN, int STAGES, bool A_KMAJ, bool B_KMAJ>
__global__ void __launch_bounds__(WM * WN * 32, 1)
    gemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  constexpr int NCW = WM * WN;           // consumer warps
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int TM = WTM / 8, TN = WTN / 8;
  constexpr int A_ELEMS = BM * BK, B_ELEMS = BN * BK;
  constexpr uint32_t STAGE_BYTES = (A_ELEMS + B_ELEMS) * 8;
  constexpr bool PERM1 = A_KMAJ;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = sA + STAGES * A_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_ELEMS);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int tm, tn;
  tile_coords(p, p.tile0 + blockIdx.x, tm, tn);
  const int m0 = tm * BM, n0 = tn * BN;
  int kb, ke;
  k_range<BM, BN>(p, m0, n0, kb, ke);
  int kt0 = kb / BK, kt1 = (ke + BK - 1) / BK;
  if (p.splits > 1) {
    const int nk = max(kt1 - kt0, 0);
    const int per = (nk + p.splits - 1) / p.splits;
    const int s0 = kt0 + blockIdx.z * per;
    kt1 = min(kt1, s0 + per);
    kt0 = min(s0, kt1);
  }
  const int nkt = max(kt1 - kt0, 0);
  // batched launches (blockIdx.y): per-item coordinate / pointer offsets
  const int bi = blockIdx.y;
  const int ac0 = p.a_c0 + bi * p.a_bs0, ac1 = p.a_c1 + bi * p.a_bs1;
  const int bc0 = p.b_c0 + bi * p.b_bs0, bc1 = p.b_c1 + bi * p.b_bs1;
  double* const Dp = p.D + (int64_t)bi * p.d_bs;
  const double* const Cinp = p.Cin + (int64_t)bi * p.cin_bs;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_wait();  // PDL: everything above overlapped the previous kernel's tail

  // Producer = lane 0 of warp 0 (no dedicated warp: 8 warps keep the 255-register
  // budget; 9 would cap at 168 because 3 warps would share one SMSP).
  auto issue = [&](int it) {
    const int s = it % STAGES;
    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
    mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
    const int k0 = (kt0 + it) * BK;
    double* a_dst = sA + s * A_ELEMS;
    double* b_dst = sB + s * B_ELEMS;
    if (A_KMAJ) {
      tma_load_2d(a_dst, &tmA, &full[s], ac0 + k0, ac1 + m0);
    } else {
#pragma unroll
      for (int b = 0; b < BM / 16; ++b)
        tma_load_2d(a_dst + b * 256, &tmA, &full[s], ac0 + m0 + 16 * b, ac1 + k0);
    }
    if (B_KMAJ) {
      tma_load_2d(b_dst, &tmB, &full[s], bc0 + k0, bc1 + n0);
    } else {
#pragma unroll
      for (int b = 0; b < BN / 16; ++b)
        tma_load_2d(b_dst + b * 256, &tmB, &full[s], bc0 + n0 + 16 * b, bc1 + k0);
    }
  };
  const bool producer = (threadIdx.x == 0);
  if (producer && nkt > 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int it = 0; it < min(nkt, STAGES - 1); ++it) issue(it);
  }

  // ---------------- DMMA consumers
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, t = lane & 3;
  const int am = wm * WTM + g, bn = wn * WTN + g;

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  FragBase fa_i[4], fb_i[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    fa_i[i] = frag_base<A_KMAJ>(am, kperm<PERM1>(t, i));
    fb_i[i] = frag_base<B_KMAJ>(bn, kperm<PERM1>(t, i));
  }

  for (int it = 0; it < nkt; ++it) {
    const int s = it % STAGES;
    if (producer && it + STAGES - 1 < nkt) issue(it + STAGES - 1);
    mbar_wait(&full[s], (it / STAGES) & 1);
    const double* a_s = sA + s * A_ELEMS;
    const double* b_s = sB + s * B_ELEMS;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const FragBase fa = fa_i[i], fb = fb_i[i];
      // B fragments held, A fragments streamed (register pressure)
      double bf[TN];
#pragma unroll
      for (int y = 0; y < TN; ++y) bf[y] = b_s[frag_at<B_KMAJ>(fb, y)];
#pragma unroll
      for (int x = 0; x < TM; ++x) {
        const double af = a_s[frag_at<A_KMAJ>(fa, x)];
#pragma unroll
        for (int y = 0; y < TN; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af, bf[y]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- epilogue: accumulators -> smem tile -> coalesced column writes
  __syncthreads();  // every warp is past the mainloop: the stage buffers are free
  // PDL: the next kernel may be scheduled now (once every CTA of this grid got
  // here); it still waits in griddep_wait() for this grid's completion and memory
  // flush, so only its launch and prologue overlap this epilogue
  griddep_launch_dependents();
  constexpr int LDC = BM + 2;  // conflict-free 8-byte writes per half-warp
  double* Cs = sA;
#pragma unroll
  for (int x = 0; x < TM; ++x)
#pragma unroll
    for (int y = 0; y < TN; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        Cs[(wn * WTN + 8 * y + 2 * t + e) * LDC + wm * WTM + 8 * x + g] = acc[x][y][e];
  __syncthreads();
  constexpr int NW = WM * WN;
  const bool split = p.splits > 1;
  double* D = split ? (p.compact ? p.partial + ((int64_t)blockIdx.z * gridDim.x + blockIdx.x) * (BM * BN) -
                                      m0 - (int64_t)n0 * BM
                                : p.partial + (size_t)blockIdx.z * p.M * p.N)
                    : Dp;
  const int64_t ldd = split ? (p.compact ? BM : p.M) : p.ldd;
  const bool lower = !split && p.omode != (int)OutMode::Full;
  const bool mirror = !split && p.omode == (int)OutMode::LowerMirror;
  const bool vec = ((reinterpret_cast<uintptr_t>(D) & 15) == 0) && ((ldd & 1) == 0) &&
                   (split || p.beta == 0.0 ||
                    (((reinterpret_cast<uintptr_t>(Cinp) & 15) == 0) && ((p.ldcin & 1) == 0)));
  // Cin (beta != 0) for every (column, row pair) of this lane is loaded up
  // front — all loads in flight at once instead of one global round trip per
  // column — then combined with the tile and stored.
  constexpr int NCOL = (BN + NW - 1) / NW, NCH = (BM + 63) / 64;
  double2 cinv[NCOL][NCH];
  const bool use_cin = !split && p.beta != 0.0;
  if (use_cin) {
#pragma unroll
    for (int ci = 0; ci < NCOL; ++ci) {
      const int cl = warp + ci * NW;
      const int j = n0 + cl;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int rl = ch * 64 + 2 * lane;
        const int i = m0 + rl;
        double2 c2 = make_double2(0.0, 0.0);
        if (cl < BN && j < p.N && rl < BM && i < p.M) {
          const double* cin = Cinp + i + (size_t)j * p.ldcin;
          if (vec && i + 1 < p.M) {
            c2 = *reinterpret_cast<const double2*>(cin);
          } else {
            c2.x = cin[0];
            if (i + 1 < p.M) c2.y = cin[1];
          }
        }
        cinv[ci][ch] = c2;
      }
    }
  }
#pragma unroll
  for (int ci = 0; ci < NCOL; ++ci) {
    const int cl = warp + ci * NW;
    const int j = n0 + cl;
    if (cl >= BN || j >= p.N) break;
    const double* col = Cs + cl * LDC;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int rl = ch * 64 + 2 * lane;
      const int i = m0 + rl;
      if ((BM % 64 != 0 && rl >= BM) || i >= p.M) continue;
      double v0 = col[rl], v1 = col[rl + 1];
      if (!split) {
        v0 *= p.alpha;
        v1 *= p.alpha;
        if (use_cin) {
          v0 += p.beta * cinv[ci][ch].x;
          v1 += p.beta * cinv[ci][ch].y;
        }
        if (i == j) v0 += p.diag_add;
        if (i + 1 == j) v1 += p.diag_add;
      }
      double* dst = D + i + (size_t)j * ldd;
      const bool w0 = !lower || i >= j, w1 = (i + 1 < p.M) && (!lower || i + 1 >= j);
      if (vec && w0 && w1) {
        *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
      } else {
        if (w0) dst[0] = v0;
        if (w1) dst[1] = v1;
      }
      if (mirror) {
        if (w0 && i > j) D[j + (size_t)i * ldd] = v0;
        if (w1 && i + 1 > j) D[j + (size_t)(i + 1) * ldd] = v1;
      }
    }
  }
}

// Split-K reduction + epilogue: D = alpha * sum_z P_z + beta * Cin (+diag), with
// the same LowerMirror semantics.
__global__ void splitk_reduce_kernel(const GemmParams p) {
  const int64_t total = (int64_t)p.M * p.N;
  const bool lower = p.omode != (int)OutMode::Full;
  const bool mirror = p.omode == (int)OutMode::LowerMirror;
  griddep_wait();  // PDL launch: the partials of the GEMM just before
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % p.M), j = (int)(idx / p.M);
    if (lower && i < j) continue;
    double s = 0.0;
    for (int z = 0; z < p.splits; ++z) s += p.partial[(size_t)z * total + idx];
    double v = p.alpha * s;
    if (p.beta != 0.0) v += p.beta * p.Cin[i + (size_t)j * p.ldcin];
    if (i == j) v += p.diag_add;
    p.D[i + (size_t)j * p.ldd] = v;
    if (mirror && i != j) p.D[j + (size_t)i * p.ldd] = v;
  }
  griddep_launch_dependents();
}

// Reduction of a compact split-K tail launch: one block per 32 x 32 sub-block of
// the tail tiles (tile tile0 + t, sub-block sbk) sums the partials and applies the
// epilogue (alpha, beta Cin, diag, lower/mirror).  The mirrored (transposed)
// writes of LowerMirror outputs go through shared memory, so they are coalesced
// too.  (One block per tile, element by element, was latency-bound at ~90 us per
// 84-tile tail at n = 4096: four loads in flight per thread.)
template <int BM>
__global__ void __launch_bounds__(256) splitk_reduce_tiles_kernel(const GemmParams p, int ntail) {
  __shared__ double sb[32][33];
  constexpr int NS = (BM / 32) * (BM / 32);
  const int t = blockIdx.x / NS, sbk = blockIdx.x % NS;
  int tm, tn;
  tile_coords(p, p.tile0 + t, tm, tn);
  const int m0 = tm * BM + (sbk % (BM / 32)) * 32, n0 = tn * BM + (sbk / (BM / 32)) * 32;
  const int e0 = (sbk % (BM / 32)) * 32 + (sbk / (BM / 32)) * 32 * BM;  // sub-block origin in the tile
  const bool lower = p.omode != (int)OutMode::Full;
  const bool mirror = p.omode == (int)OutMode::LowerMirror;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  griddep_wait();
  if (!(lower && m0 + 31 < n0)) {  // (sub-blocks strictly above the diagonal: nothing)
    for (int r = ty; r < 32; r += 8) {
      const int i = m0 + tx, j = n0 + r;
      double v = 0.0;
      if (i < p.M && j < p.N && !(lower && i < j)) {
        const int e = e0 + tx + r * BM;
        double s = 0.0;
        for (int z = 0; z < p.splits; ++z) s += p.partial[((int64_t)z * ntail + t) * (BM * BM) + e];
        v = p.alpha * s;
        if (p.beta != 0.0) v += p.beta * p.Cin[i + (size_t)j * p.ldcin];
        if (i == j) v += p.diag_add;
        p.D[i + (size_t)j * p.ldd] = v;
      }
      sb[r][tx] = v;
    }
    if (mirror) {
      __syncthreads();
      // D(j, i) = v(i, j) for i > j, coalesced along j
      for (int r = ty; r < 32; r += 8) {
        const int i = m0 + r, j = n0 + tx;
        if (i < p.M && j < p.N && i > j) p.D[j + (size_t)i * p.ldd] = sb[tx][r];
      }
    }
  }
  griddep_launch_dependents();
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    QDWHG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// Descriptor over the stored matrix of view `v`, extent clipped at the end of
// the view so reads past the view are zero-filled by TMA.
// Encoded descriptors are cached by (base, ld, extent, box): the arena hands
// out the same addresses every QDWH iteration, so steady-state launches skip
// the driver call.
struct DescKey {
  uintptr_t base;
  int64_t ld;
  uint64_t d0, d1;
  int box0, box1;
  bool operator==(const DescKey& o) const {
    return base == o.base && ld == o.ld && d0 == o.d0 && d1 == o.d1 && box0 == o.box0 &&
           box1 == o.box1;
  }
};
struct DescKeyHash {
  size_t operator()(const DescKey& k) const {
    size_t h = std::hash<uintptr_t>()(k.base);
    h ^= std::hash<int64_t>()(k.ld) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h ^= std::hash<uint64_t>()(k.d0 * 1000003ull + k.d1) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h ^= (size_t)(k.box0 * 131 + k.box1);
    return h;
  }
};

CUtensorMap make_desc(const DMat& v, int box0, int box1) {
  static thread_local std::unordered_map<DescKey, CUtensorMap, DescKeyHash> cache;
  CUtensorMap tm;
  const uint64_t d0 = (uint64_t)std::max<int64_t>(v.r0 + v.rows, 1);
  const uint64_t d1 = (uint64_t)std::max<int64_t>(v.c0 + v.cols, 1);
  const DescKey key{reinterpret_cast<uintptr_t>(v.base), v.ld, d0, d1, box0, box1};
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 8192) cache.clear();
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)v.base, dims, strides,
                            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  cache.emplace(key, tm);
  return tm;
}

// Useful FP64 flops of one launch (zeros of triangular operands and the
// mirrored half of a symmetric output are not counted).
double algorithmic_flops(const GemmParams& p) {
  const double M = p.M, N = p.N, K = p.K;
  auto tri = [](double rows, double len, double kmax) {
    // sum_{j<len} min(kmax, j+1)
    const double full = std::min(len, kmax);
    return full * (full + 1) / 2 + std::max(0.0, len - kmax) * kmax;
  };
  if (p.omode != (int)OutMode::Full) {
    if ((KRange)p.kmode == KRange::AUpper) {
      // lower tiles, k from the row index: sum_i 2 (i+1)(K-i)  (LAUUM-shaped)
      double f = 0.0;
      for (int64_t i = 0; i < p.N; ++i) f += 2.0 * (double)(i + 1) * std::max(0.0, K - (double)i);
      return f;
    }
    return K * N * (N + 1);
  }
  switch ((KRange)p.kmode) {
    case KRange::BUpper: return 2 * M * tri(M, N, K);
    case KRange::BLower: return 2 * M * tri(M, std::min(N, K), K);  // sum_j (K - j)
    case KRange::AUpper: return 2 * N * tri(N, std::min(M, K), K);
    case KRange::ALower: return 2 * N * tri(N, M, K);
    default: return 2 * M * N * K;
  }
}

template <int BM, int BN, int WM, int WN, int STAGES, bool AK, bool BK_>
void launch_cfg(Ctx& ctx, const DMat& A, const DMat& B, GemmParams& p) {
  constexpr int threads = WM * WN * 32;
  constexpr size_t smem = 1024 + (size_t)STAGES * (BM + BN) * BK * 8 + 2 * STAGES * 8;
  auto kern = gemm_dmma_kernel<BM, BN, WM, WN, STAGES, AK, BK_>;
  func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const CUtensorMap ta = AK ? make_desc(A, 16, BM) : make_desc(A, 16, 16);
  const CUtensorMap tb = BK_ ? make_desc(B, 16, BN) : make_desc(B, 16, 16);
  int ntiles;
  if (p.ntl > 0)
    ntiles = p.ntl;
  else if (p.omode != (int)OutMode::Full)
    ntiles = p.tiles_n * (p.tiles_n + 1) / 2;
  else
    ntiles = p.tiles_m * p.tiles_n;
  dim3 grid(ntiles, p.nbatch, p.splits);
  static const bool debug = getenv("QDWHG_DEBUG") != nullptr;
  if (debug)
    fprintf(stderr,
            "gemm BM=%d AK=%d BK=%d M=%d N=%d K=%d kmode=%d omode=%d splits=%d tiles=%dx%d "
            "A(r0=%ld c0=%ld %ldx%ld ld=%ld) B(r0=%ld c0=%ld %ldx%ld ld=%ld)\n",
            BM, (int)AK, (int)BK_, p.M, p.N, p.K, p.kmode, p.omode, p.splits, p.tiles_m, p.tiles_n,
            (long)A.r0, (long)A.c0, (long)A.rows, (long)A.cols, (long)A.ld, (long)B.r0,
            (long)B.c0, (long)B.rows, (long)B.cols, (long)B.ld);
  if (ctx.profile) {
    char tag[160];
    snprintf(tag, sizeof(tag), "BM=%d AK=%d BK=%d M=%d N=%d K=%d kmode=%d omode=%d splits=%d grid=%d",
             BM, (int)AK, (int)BK_, p.M, p.N, p.K, p.kmode, p.omode, p.splits, ntiles * p.splits);
    ctx.prof_begin(algorithmic_flops(p) * p.flop_frac, tag);
  }
  launch_pdl(ctx, kern, grid, dim3(threads), smem, ta, tb, p);
  if (ctx.profile) ctx.prof_end();
  if (debug) QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  ctx.gemm_launches++;
}

template <int BM, int BN, int WM, int WN, int STAGES>
void dispatch_layout(Ctx& ctx, bool ak, bool bk, const DMat& A, const DMat& B, GemmParams& p) {
  if (ak && bk) launch_cfg<BM, BN, WM, WN, STAGES, true, true>(ctx, A, B, p);
  else if (ak && !bk) launch_cfg<BM, BN, WM, WN, STAGES, true, false>(ctx, A, B, p);
  else if (!ak && bk) launch_cfg<BM, BN, WM, WN, STAGES, false, true>(ctx, A, B, p);
  else launch_cfg<BM, BN, WM, WN, STAGES, false, false>(ctx, A, B, p);
}

}  // namespace

void gemm(Ctx& ctx, Op ta, Op tb, double alpha, const DMat& A, const DMat& B, double beta,
          const DMat& C, const GemmExtra& ex) {
  const int64_t M = C.rows, N = C.cols;
  const int64_t K = (ta == Op::N) ? A.cols : A.rows;
  const int64_t am = (ta == Op::N) ? A.rows : A.cols;
  const int64_t bk = (tb == Op::N) ? B.rows : B.cols;
  const int64_t bn = (tb == Op::N) ? B.cols : B.rows;
  if (am != M || bn != N || bk != K) throw InvalidArgument("gemm: shape mismatch");
  if (M == 0 || N == 0) return;
  if (ex.out != OutMode::Full && M != N) throw InvalidArgument("gemm: lower output needs square C");
  if ((A.ld % 2) || (B.ld % 2) || (reinterpret_cast<uintptr_t>(A.base) % 16) ||
      (reinterpret_cast<uintptr_t>(B.base) % 16))
    throw InvalidArgument("gemm: operands must be 16-byte aligned with even leading dimension");
  // TMA box starts must be 16-byte aligned in the contiguous dimension: an odd
  // row offset (e.g. Q2 = Q(m:m+n, :) with odd m in the QR step) is staged
  // into an aligned copy first.
  if ((A.r0 & 1) || (B.r0 & 1)) {
    const Arena::Mark m0 = ctx.arena->mark();
    DMat A2 = A, B2 = B;
    if (A.r0 & 1) {
      A2 = ctx.arena->alloc(A.rows, A.cols);
      copy(ctx, A, A2);
    }
    if (B.r0 & 1) {
      B2 = ctx.arena->alloc(B.rows, B.cols);
      copy(ctx, B, B2);
    }
    gemm(ctx, ta, tb, alpha, A2, B2, beta, C, ex);
    ctx.arena->release_to(m0);
    return;
  }

  GemmParams p{};
  p.flop_frac = 1.0;
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  // TMA coordinates: (contiguous index, outer index) of the stored matrix
  p.a_c0 = (int)A.r0;
  p.a_c1 = (int)A.c0;
  p.b_c0 = (int)B.r0;
  p.b_c1 = (int)B.c0;
  p.alpha = alpha;
  p.beta = beta;
  p.diag_add = ex.diag_add;
  p.D = C.ptr();
  p.ldd = C.ld;
  const DMat& cin = ex.cin ? *ex.cin : C;
  p.Cin = cin.ptr();
  p.ldcin = cin.ld;
  p.kmode = (int)ex.krange;
  p.omode = (int)ex.out;
  const bool ak = (ta == Op::T);  // op(A) K-contiguous
  const bool bkm = (tb == Op::N); // op(B) K-contiguous
  const int nb_ = std::max(1, ex.batch);
  p.nbatch = nb_;
  p.a_bs0 = (int)ex.a_step_r;
  p.a_bs1 = (int)ex.a_step_c;
  p.b_bs0 = (int)ex.b_step_r;
  p.b_bs1 = (int)ex.b_step_c;
  p.d_bs = ex.c_step_r + ex.c_step_c * C.ld;
  p.cin_bs = ex.c_step_r + ex.c_step_c * cin.ld;
  // descriptors must cover every batch item (items tile exactly: no zero-fill reliance)
  DMat Ae = A, Be = B;
  Ae.rows += (nb_ - 1) * ex.a_step_r;
  Ae.cols += (nb_ - 1) * ex.a_step_c;
  Be.rows += (nb_ - 1) * ex.b_step_r;
  Be.cols += (nb_ - 1) * ex.b_step_c;

  // Tile size and split-K from a small wave-quantisation cost model: for each
  // candidate (128/64/32 tiles, split factor) estimate
  //   ceil(units / concurrent CTAs) * (tile flops / per-CTA rate + prologue)
  //   + split-K reduction traffic,
  // and take the cheapest.  Triangular K ranges count half the K on average.
  const bool tri = ex.krange != KRange::Full;
  const double keff = tri ? 0.5 * (double)K : (double)K;
  const int64_t ktiles = (K + BK - 1) / BK;
  const double sm_rate = 64.0 * 1.9e9;  // FP64 FMA / s per SM (DMMA)
  int BMt = 128, splits = 1;
  double best = 1e30;
  for (int bm : {128, 64, 32}) {
    if (ex.force_bm && bm != ex.force_bm) continue;
    if (nb_ > 1 && (M % bm || N % bm)) continue;  // batched items must tile exactly
    const int64_t tm = (M + bm - 1) / bm, tn = (N + bm - 1) / bm;
    const int64_t tiles = (ex.out != OutMode::Full) ? tn * (tn + 1) / 2 : tm * tn;
    const int per_sm = (bm == 32 || (bm == 64 && ex.skinny)) ? 2 : 1;
    const double eff = (bm == 128) ? 0.95 : (bm == 64) ? 0.75 : 0.45;
    for (int sp : {1, 2, 3, 4, 6, 8, 12, 16}) {
      if (ex.split_k > 0 && sp != ex.split_k) continue;
      if (sp > 1 && (nb_ > 1 || ktiles / sp < 4)) continue;
      const double units = (double)tiles * nb_ * sp;
      const double waves = std::ceil(units / ((double)ctx.num_sms * per_sm));
      const double t_unit = (double)bm * bm * (keff / sp) / (sm_rate * eff / per_sm) + 2e-6;
      double t = waves * t_unit;
      // triangular K ranges: the heaviest tiles carry the full K, and with few
      // waves they set the time (a one-wave TRMM runs as long as its K = n tile)
      if (tri) t = std::max(t, (double)bm * bm * ((double)K / sp) / (sm_rate * eff / per_sm) + 2e-6);
      if (sp > 1) t += (double)(sp + 1) * M * N * 8.0 / 4e12 + 3e-6;
      if (t < best * 0.97) {  // prefer the earlier (larger-tile, fewer-split) candidate on ties
        best = t;
        BMt = bm;
        splits = sp;
      }
    }
  }
  // Wave balancing: when the chosen plan is unsplit and its last wave is
  // partial, run the full waves as one launch and the tail tiles split-K over
  // the whole machine (compact partials + per-tile reduction) — the tail costs
  // ceil(tail*s / CTAs) * t/s instead of a whole wave t.  Full K range only
  // (equal work per tile).
  int tail_split = 1;
  int64_t full_tiles = 0, tail_tiles = 0;
  static const bool no_balance = getenv("QDWHG_GEMM_NO_BALANCE") != nullptr;
  if (!no_balance && splits == 1 && nb_ == 1 && !tri && ex.split_k == 0) {
    const int bm = BMt;
    const int64_t tm = (M + bm - 1) / bm, tn = (N + bm - 1) / bm;
    const int64_t tiles = (ex.out != OutMode::Full) ? tn * (tn + 1) / 2 : tm * tn;
    const int per_sm = (bm == 32 || (bm == 64 && ex.skinny)) ? 2 : 1;
    const int64_t conc = (int64_t)ctx.num_sms * per_sm;
    const int64_t full = (tiles / conc) * conc, tail = tiles - full;
    const double eff = (bm == 128) ? 0.95 : (bm == 64) ? 0.75 : 0.45;
    const double t_full = (double)bm * bm * keff / (sm_rate * eff / per_sm);
    if (full > 0 && tail > 0) {
      double plain = std::ceil((double)tiles / conc) * (t_full + 2e-6);
      double bt = plain;
      for (int sp : {2, 3, 4, 5, 6, 7, 8, 10, 12, 16}) {
        if (ktiles / sp < 4) continue;
        const double th = (double)(full / conc) * (t_full + 2e-6) +
                          std::ceil((double)tail * sp / conc) * (t_full / sp + 2e-6) +
                          (double)(sp + 2) * tail * bm * bm * 8.0 / 4e12 + 8e-6;
        if (th < bt * (ex.fine_tail ? 1.0 : 0.97)) {
          bt = th;
          tail_split = sp;
        }
      }
      if (tail_split > 1) {
        full_tiles = full;
        tail_tiles = tail;
      }
    }
  }
  const bool big = BMt == 128, tiny = BMt == 32;
  p.tiles_m = (int)((M + BMt - 1) / BMt);
  p.tiles_n = (int)((N + BMt - 1) / BMt);
  if (nb_ > 1) {
    splits = 1;
    if (M % BMt || N % BMt || K % BK)
      throw InvalidArgument("gemm: batched items must tile exactly");
  }
  p.splits = splits;
  const Arena::Mark mark = ctx.arena->mark();
  if (splits > 1) p.partial = static_cast<double*>(ctx.arena->alloc_bytes((size_t)splits * M * N * 8));

  auto dispatch = [&](GemmParams& q) {
    if (big)
      dispatch_layout<128, 128, 2, 4, 6>(ctx, ak, bkm, Ae, Be, q);
    else if (tiny)
      dispatch_layout<32, 32, 2, 2, 8>(ctx, ak, bkm, Ae, Be, q);
    else if (ex.skinny)
      dispatch_layout<64, 64, 2, 2, 6>(ctx, ak, bkm, Ae, Be, q);
    else
      dispatch_layout<64, 64, 2, 2, 8>(ctx, ak, bkm, Ae, Be, q);
  };
  if (tail_split > 1) {
    const double tot_tiles = (double)(full_tiles + tail_tiles);
    GemmParams p1 = p;  // full waves, fused epilogue
    p1.ntl = (int)full_tiles;
    p1.flop_frac = full_tiles / tot_tiles;
    dispatch(p1);
    GemmParams p2 = p;  // tail tiles, split-K, compact partials
    p2.tile0 = (int)full_tiles;
    p2.ntl = (int)tail_tiles;
    p2.splits = tail_split;
    p2.compact = 1;
    p2.flop_frac = tail_tiles / tot_tiles;
    p2.partial = static_cast<double*>(
        ctx.arena->alloc_bytes((size_t)tail_split * tail_tiles * BMt * BMt * 8));
    dispatch(p2);
    if (big)
      launch_pdl(ctx, splitk_reduce_tiles_kernel<128>, dim3((unsigned)(tail_tiles * 16)), dim3(256), 0, p2,
                 (int)tail_tiles);
    else if (tiny)
      launch_pdl(ctx, splitk_reduce_tiles_kernel<32>, dim3((unsigned)tail_tiles), dim3(256), 0, p2,
                 (int)tail_tiles);
    else
      launch_pdl(ctx, splitk_reduce_tiles_kernel<64>, dim3((unsigned)(tail_tiles * 4)), dim3(256), 0, p2,
                 (int)tail_tiles);
    ctx.count();
    ctx.arena->release_to(mark);
    return;
  }
  dispatch(p);

  if (splits > 1) {
    const int64_t total = M * N;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 4 * ctx.num_sms);
    launch_pdl(ctx, splitk_reduce_kernel, dim3(blocks), dim3(256), 0, p);
    ctx.count();
  }
  ctx.arena->release_to(mark);
}

}  // namespace qdwhg
