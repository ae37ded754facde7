// Blocked Householder QR + trailing-column Q formation for the subspace
// extraction of Alg. 1/2 (partial.cpp:71-79, 138-146) and the stacked QR of
// the QR-based QDWH step (polar.cpp:56-72).  Reference kernels:
// householder_qr kernels.cpp:41-80 and accumulate_q kernels.cpp:84-101.
//
// Same reflector convention as the reference (R_jj = -sign(x0)*||x||,
// p = min(m-1, n) reflectors, tau = 0 for a zero column), stored LAPACK style
// (v_jj = 1, tau' = tau * v0^2) so each nb-column panel becomes a compact-WY
// block (I - V T V^T) and every update is a DMMA GEMM:
//   panel:    geqr2_panel_kernel — cooperative persistent kernel, the panel
//             lives in shared memory across up to 148 CTAs; ONE grid barrier
//             per column (norm, pivot and all v^T a_c dot products reduced
//             together with FP64 atomics);
//   T:        Gram V^T V by GEMM, then larft_kernel (one CTA);
//   trailing: C -= V T^T (V^T C)  — three GEMMs;
//   ORGQR:    only the requested Q columns (Q2 = Q(:, ind-1:n)), reflector
//             blocks applied last to first, skipping columns still equal to e_i.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "internal.hpp"

namespace qdwhg {

namespace {

constexpr int kPanelThreads = 256;
constexpr int kBW = 64;  // max panel width (one thread column per panel column)

QDWHG_DEV unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
QDWHG_DEV void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Monotonic grid barrier (counter zeroed before launch; all CTAs co-resident
// via cooperative launch).
QDWHG_DEV void grid_barrier(unsigned* bar, unsigned nblocks, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) {
    // bar.sync orders the CTA's prior writes/atomics before thread 0's
    // gpu-scope release (cumulativity); acquire on the poll orders what follows.
    red_release_add(bar, 1u);
    const unsigned target = epoch * nblocks;
    while (ld_acquire(bar) < target) {
    }
  }
  __syncthreads();
}

// Partial sums for pivot column `col` over this CTA's rows:
//   top[c]  = A(col, c)                       (row owner only)
//   dbel[c] = sum_{r > col} A(r, col) A(r, c) (dbel[col] = sigma^2 below the pivot)
// for c >= col, written to this CTA's out = [top(BW) | dbel(BW)] (zeros elsewhere).
QDWHG_DEV void panel_partials(const double* S, int RP, int nr, int rbeg, int b, int col, double* red,
                              double* out) {
  const int c = threadIdx.x % kBW, rg = threadIdx.x / kBW;
  double d = 0.0;
  if (c < b && c >= col) {
    const double* sc = S + c * RP;
    const double* sp = S + col * RP;
    int r0 = max(col + 1 - rbeg, 0);
    for (int r = r0 + rg; r < nr; r += kPanelThreads / kBW) d += sp[r] * sc[r];
  }
  red[rg * kBW + c] = d;
  __syncthreads();
  if (rg == 0) {
    double s = 0.0, top = 0.0;
    if (c < b && c >= col) {
#pragma unroll
      for (int q = 0; q < kPanelThreads / kBW; ++q) s += red[q * kBW + c];
      const int rl = col - rbeg;
      if (rl >= 0 && rl < nr) top = S[c * RP + rl];
    }
    out[c] = top;
    out[kBW + c] = s;
  }
  __syncthreads();
}

// Unblocked Householder QR of an mp x b panel (b <= 64) whose rows are spread
// over the CTAs of the launch, each CTA keeping its rows in shared memory.
// Per column ONE cross-CTA reduction of [x0, sigma^2, a_jj,c, x^T a_c] gives the
// pivot, tau and all v^T a_c at once.
//   CLUSTER = true : one thread-block cluster (<= 16 CTAs): partial vectors are
//                    read from the peers' shared memory (DSMEM) in fixed order
//                    (deterministic) behind one hardware cluster barrier;
//   CLUSTER = false: any number of co-resident CTAs (cooperative launch): FP64
//                    atomics into a rotating global buffer + a grid barrier.
template <bool CLUSTER>
__global__ void __launch_bounds__(kPanelThreads, 1)
    geqr2_panel_kernel(double* A, int64_t lda, double* V, int64_t ldv, double* tau_out, int mp,
                       int b, int rpc, double* acc, unsigned* bar) {
  extern __shared__ double smem[];
  const int RP = rpc | 1;
  double* S = smem;                                  // [b][RP] panel rows of this CTA
  double* red = S + kBW * RP;                        // [4][kBW]
  double* coef = red + (kPanelThreads / kBW) * kBW;  // [kBW] w_c
  double* part = coef + kBW;                         // [2][2*kBW] this CTA's partials (by parity)
  double* tot = part + 4 * kBW;                      // [2*kBW] reduced vector
  const int rbeg = blockIdx.x * rpc;
  const int nr = max(0, min(rpc, mp - rbeg));
  const int c = threadIdx.x % kBW, rg = threadIdx.x / kBW;
  constexpr int NRG = kPanelThreads / kBW;
  unsigned epoch = 0;
  namespace cg = cooperative_groups;

  for (int cc = 0; cc < b; ++cc)
    for (int r = threadIdx.x; r < nr; r += kPanelThreads) S[cc * RP + r] = A[(rbeg + r) + cc * lda];
  __syncthreads();

  // publish this CTA's partials for column `col` and make the reduced vector
  // visible in `tot`
  auto reduce = [&](int col) {
    double* mine = part + (col & 1) * (2 * kBW);
    panel_partials(S, RP, nr, rbeg, b, col, red, mine);
    if (CLUSTER) {
      cg::cluster_group cluster = cg::this_cluster();
      cluster.sync();
      if (threadIdx.x < 2 * kBW) {
        const int nb_ = (int)cluster.num_blocks();
        double v[16];
#pragma unroll
        for (int p = 0; p < 16; ++p)  // all remote loads in flight before the sum
          v[p] = (p < nb_) ? cluster.map_shared_rank(mine, p)[threadIdx.x] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < 16; ++p) s += v[p];
        tot[threadIdx.x] = s;
      }
      __syncthreads();
    } else {
      double* buf = acc + (col % 3) * (2 * kBW);
      if (threadIdx.x < 2 * kBW) {
        const int cc = threadIdx.x % kBW;
        if (cc < b && cc >= col && mine[threadIdx.x] != 0.0) atomicAdd(&buf[threadIdx.x], mine[threadIdx.x]);
      }
      grid_barrier(bar, gridDim.x, epoch);
      if (threadIdx.x < 2 * kBW) tot[threadIdx.x] = __ldcg(&buf[threadIdx.x]);
      if (blockIdx.x == 0) {  // buffer col+2 was last read before this barrier
        double* z = acc + ((col + 2) % 3) * (2 * kBW);
        if (threadIdx.x < 2 * kBW) z[threadIdx.x] = 0.0;
      }
      __syncthreads();
    }
  };

  reduce(0);
  for (int jj = 0; jj < b; ++jj) {
    const double x0 = tot[jj];
    const double sig2 = tot[kBW + jj];
    const double normx = sqrt(x0 * x0 + sig2);
    const bool reflect = (jj < mp - 1) && normx > 0.0;
    double beta = x0, v0 = 1.0, taup = 0.0;
    if (reflect) {
      const double sign = x0 >= 0.0 ? 1.0 : -1.0;
      beta = -sign * normx;
      v0 = x0 - beta;
      taup = (beta - x0) / beta;
    }
    if (threadIdx.x < kBW) {
      const int cc = threadIdx.x;
      double w = 0.0;
      if (reflect && cc > jj && cc < b) w = taup * (tot[cc] + tot[kBW + cc] / v0);
      coef[cc] = w;
    }
    __syncthreads();
    // apply H_jj to this CTA's rows; column jj -> v' (to V), R_jj
    if (c < b) {
      const double* sj = S + jj * RP;
      double* sc = S + c * RP;
      const double inv_v0 = 1.0 / v0;
      if (c > jj) {
        const double w = coef[c];
        if (w != 0.0) {
          for (int r = rg; r < nr; r += NRG) {
            const int rgl = rbeg + r;
            if (rgl == jj) sc[r] -= w;
            else if (rgl > jj) sc[r] -= w * (sj[r] * inv_v0);
          }
        }
      } else if (c == jj) {
        for (int r = rg; r < nr; r += NRG) {
          const int rgl = rbeg + r;
          double v;
          if (rgl < jj) v = 0.0;
          else if (rgl == jj) v = 1.0;
          else v = reflect ? sj[r] * inv_v0 : 0.0;
          V[rgl + (int64_t)jj * ldv] = v;
        }
      }
    }
    __syncthreads();
    if (c == jj && rg == 0) {
      const int rl = jj - rbeg;
      if (rl >= 0 && rl < nr) S[jj * RP + rl] = beta;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) tau_out[jj] = taup;
    if (jj + 1 < b) reduce(jj + 1);
  }
  if (CLUSTER) cg::this_cluster().sync();  // peers may still read our partials
  __syncthreads();
  // write back R (upper part) with explicit zeros below the diagonal
  for (int cc = 0; cc < b; ++cc)
    for (int r = threadIdx.x; r < nr; r += kPanelThreads) {
      const int rgl = rbeg + r;
      A[rgl + cc * lda] = (rgl <= cc) ? S[cc * RP + r] : 0.0;
    }
}

// T (b x b upper) from G = V^T V and tau' (LAPACK dlarft, forward/columnwise),
// by recursive doubling instead of the column recurrence:
//   T = [T11, -T11 (V1^T V2) T22; 0, T22],  V1^T V2 = G12,
// block size s = 1, 2, 4, ... — 2 barriers per level, log2(b) levels.
__global__ void larft_kernel(const double* G, int64_t ldg, const double* tau, double* T,
                             int64_t ldt, int b) {
  extern __shared__ double larft_sm[];
  double(*Ts)[kBW + 1] = reinterpret_cast<double(*)[kBW + 1]>(larft_sm);
  double(*M)[kBW + 1] = reinterpret_cast<double(*)[kBW + 1]>(larft_sm + kBW * (kBW + 1));
  const int t = threadIdx.x;
  for (int i = t; i < kBW * kBW; i += blockDim.x) {
    const int r = i % kBW, c = i / kBW;
    Ts[r][c] = (r == c && r < b) ? tau[r] : 0.0;
  }
  __syncthreads();
  for (int s = 1; s < b; s *= 2) {
    // M(a+r, a+s+c) = sum_{k=r}^{s-1} T11(r, k) G(a+k, a+s+c)
    for (int i = t; i < b * s; i += blockDim.x) {
      const int r = i % s, rest = i / s;          // rest = a/(2s) * s + c  over all pairs
      const int pair = rest / s, c = rest % s;
      const int a = pair * 2 * s;
      if (a + s + c >= b) continue;
      double acc = 0.0;
      for (int k = r; k < s; ++k) acc += Ts[a + r][a + k] * G[(a + k) + (int64_t)(a + s + c) * ldg];
      M[a + r][a + s + c] = acc;
    }
    __syncthreads();
    // T12(r, c) = -sum_{k=0}^{c} M(a+r, a+s+k) T22(k, c)
    for (int i = t; i < b * s; i += blockDim.x) {
      const int r = i % s, rest = i / s;
      const int pair = rest / s, c = rest % s;
      const int a = pair * 2 * s;
      if (a + s + c >= b) continue;
      double acc = 0.0;
      for (int k = 0; k <= c; ++k) acc += M[a + r][a + s + k] * Ts[a + s + k][a + s + c];
      Ts[a + r][a + s + c] = -acc;
    }
    __syncthreads();
  }
  for (int i = t; i < b * b; i += blockDim.x) {
    const int r = i % b, cc = i / b;
    T[r + (int64_t)cc * ldt] = Ts[r][cc];
  }
}

__global__ void diag_kernel(const double* R, int64_t ld, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = R[i + i * ld];
}

size_t panel_smem(int rpc) {
  return ((size_t)kBW * (rpc | 1) + (kPanelThreads / kBW) * kBW + kBW + 4 * kBW + 2 * kBW) * 8;
}

constexpr size_t kPanelSmemMax = 220 * 1024;

// Largest cluster the device allows for the panel (16 non-portable, else 8).
int cluster_size_limit() {
  static int cs = -1;
  if (cs < 0) {
    cs = 8;
    if (cudaFuncSetAttribute(geqr2_panel_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(kPanelThreads);
      cfg.dynamicSmemBytes = kPanelSmemMax;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = 16;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, geqr2_panel_kernel<true>, &cfg) == cudaSuccess && n > 0)
        cs = 16;
    }
    cudaGetLastError();
  }
  return cs;
}

void panel_factor(Ctx& ctx, const DMat& P, const DMat& Vp, double* tau_dev, double* acc,
                  unsigned* bar) {
  int mp = (int)P.rows, b = (int)P.cols;
  static bool set = false;
  if (!set) {
    QDWHG_CUDA(cudaFuncSetAttribute(geqr2_panel_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPanelSmemMax));
    QDWHG_CUDA(cudaFuncSetAttribute(geqr2_panel_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPanelSmemMax));
    set = true;
  }
  double* Ap = P.ptr();
  int64_t lda = P.ld;
  double* Vptr = Vp.ptr();
  int64_t ldv = Vp.ld;
  const int csmax = cluster_size_limit();
  // cluster path when <= 64 rows per CTA fit in one cluster (deterministic,
  // cheapest barrier); taller panels spread over more SMs with the grid path,
  // whose per-column work shrinks with the CTA count (measured faster at n=4096).
  int cs = std::max(1, (mp + 63) / 64);
  int rpc = (mp + cs - 1) / cs;
  if (cs <= csmax) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kPanelThreads);
    cfg.dynamicSmemBytes = panel_smem(rpc);
    cfg.stream = ctx.stream;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cs;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    QDWHG_CUDA(cudaLaunchKernelEx(&cfg, geqr2_panel_kernel<true>, Ap, lda, Vptr, ldv, tau_dev, mp, b,
                                  rpc, acc, bar));
    ctx.count();
    return;
  }
  // grid path (tall panels): cooperative launch over up to all SMs
  const int nblk = std::max(1, std::min(ctx.num_sms, (mp + 63) / 64));
  rpc = (mp + nblk - 1) / nblk;
  if (panel_smem(rpc) > kPanelSmemMax) throw InvalidArgument("geqrf: panel too tall for shared memory");
  QDWHG_CUDA(cudaMemsetAsync(acc, 0, 3 * 2 * kBW * sizeof(double), ctx.stream));
  QDWHG_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), ctx.stream));
  void* args[] = {&Ap, &lda, &Vptr, &ldv, &tau_dev, &mp, &b, &rpc, &acc, &bar};
  QDWHG_CUDA(cudaLaunchCooperativeKernel((void*)geqr2_panel_kernel<false>, dim3(nblk),
                                         dim3(kPanelThreads), args, panel_smem(rpc), ctx.stream));
  ctx.count();
}

}  // namespace

// T (b x b, b <= 64) of a compact-WY block from its Gram G = V^T V and taus.
void larft_launch(Ctx& ctx, const DMat& G, const double* tau_dev, const DMat& T) {
  static bool larft_attr = false;
  if (!larft_attr) {
    QDWHG_CUDA(cudaFuncSetAttribute(larft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    2 * kBW * (kBW + 1) * 8));
    larft_attr = true;
  }
  larft_kernel<<<1, 256, 2 * kBW * (kBW + 1) * 8, ctx.stream>>>(G.ptr(), G.ld, tau_dev, T.ptr(),
                                                               T.ld, (int)G.rows);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
}

void geqrf(Ctx& ctx, const DMat& A, QrWork& w) {
  const int64_t m = A.rows, n = A.cols;
  if (m < n) throw InvalidArgument("geqrf: requires rows >= cols");
  // Two-level blocking: 64-column panels (one cooperative/cluster kernel each)
  // inside 256-column outer blocks.  Inner updates touch only the outer block;
  // the outer T (256 x 256) is assembled by merging the panel T's
  // (T = [T1, -T1 (V1^T V2) T2; 0, T2]) so the trailing update of the rest of
  // the matrix — the O(n^3) part — runs as GEMMs with K = 256.
  const int nbi = kBW;
  const int nbo = 4 * kBW;
  w.nb = nbo;
  const int64_t nout = (n + nbo - 1) / nbo;
  w.V = ctx.arena->alloc(m, n);
  w.T = ctx.arena->alloc(nbo, nout * nbo);
  fill(ctx, w.T, 0.0, 0.0);
  double* tau_dev = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (n + 64)));
  double* acc = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * 3 * 2 * kBW));
  unsigned* bar = static_cast<unsigned*>(ctx.arena->alloc_bytes(256));
  DMat G = ctx.arena->alloc(nbo, nbo);
  const Arena::Mark mark = ctx.arena->mark();
  for (int64_t po = 0; po < nout; ++po) {
    const int64_t jo = po * nbo;
    const int64_t bo = std::min<int64_t>(nbo, n - jo);
    const int64_t mo = m - jo;
    const DMat To = w.T.sub(0, po * nbo, bo, bo);
    std::vector<std::pair<int64_t, int64_t>> blocks;  // (offset in outer block, width)
    for (int64_t ji = 0; ji < bo; ji += nbi) {
      const int64_t bi = std::min<int64_t>(nbi, bo - ji);
      const int64_t j0 = jo + ji;
      const int64_t mp = m - j0;
      const DMat Vp = w.V.sub(j0, j0, mp, bi);
      panel_factor(ctx, A.sub(j0, j0, mp, bi), Vp, tau_dev + j0, acc, bar);
      if (j0 > 0) fill(ctx, w.V.sub(0, j0, j0, bi), 0.0, 0.0);  // V above the panel is zero
      const DMat Gp = G.sub(0, 0, bi, bi);
      gemm(ctx, Op::T, Op::N, 1.0, Vp, Vp, 0.0, Gp);
      const DMat Ti = To.sub(ji, ji, bi, bi);
      larft_launch(ctx, Gp, tau_dev + j0, Ti);
      blocks.push_back({ji, bi});
      const int64_t nc = bo - ji - bi;  // rest of the outer block
      if (nc > 0) {
        const DMat C = A.sub(j0, j0 + bi, mp, nc);
        DMat W1 = ctx.arena->alloc(bi, nc), W2 = ctx.arena->alloc(bi, nc);
        gemm(ctx, Op::T, Op::N, 1.0, Vp, C, 0.0, W1);
        GemmExtra e;
        e.krange = KRange::ALower;  // op(A) = T^T lower
        gemm(ctx, Op::T, Op::N, 1.0, Ti, W1, 0.0, W2, e);
        gemm(ctx, Op::N, Op::N, -1.0, Vp, W2, 1.0, C);
        ctx.arena->release_to(mark);
      }
    }
    const int64_t nc = n - jo - bo;
    // ---- outer T (also needed by ORGQR for the last block) by pairwise merges of the panel T's
    if (blocks.size() > 1) {
      const DMat Vo = w.V.sub(jo, jo, mo, bo);
      const DMat Go = G.sub(0, 0, bo, bo);
      gemm(ctx, Op::T, Op::N, 1.0, Vo, Vo, 0.0, Go);
      while (blocks.size() > 1) {
        std::vector<std::pair<int64_t, int64_t>> next;
        for (size_t q = 0; q + 1 < blocks.size(); q += 2) {
          const auto [o1, s1] = blocks[q];
          const auto [o2, s2] = blocks[q + 1];
          DMat M1 = ctx.arena->alloc(s1, s2);
          GemmExtra a1;
          a1.krange = KRange::AUpper;  // T11 upper
          gemm(ctx, Op::N, Op::N, 1.0, To.sub(o1, o1, s1, s1), Go.sub(o1, o2, s1, s2), 0.0, M1, a1);
          GemmExtra a2;
          a2.krange = KRange::BUpper;  // T22 upper
          gemm(ctx, Op::N, Op::N, -1.0, M1, To.sub(o2, o2, s2, s2), 0.0, To.sub(o1, o2, s1, s2), a2);
          ctx.arena->release_to(mark);
          next.push_back({o1, s1 + s2});
        }
        if (blocks.size() % 2) next.push_back(blocks.back());
        blocks.swap(next);
      }
    }
    // ---- trailing update of the rest: C = C - V T^T (V^T C), K = bo
    if (nc > 0) {
      const DMat Vo = w.V.sub(jo, jo, mo, bo);
      const DMat C = A.sub(jo, jo + bo, mo, nc);
      DMat W1 = ctx.arena->alloc(bo, nc), W2 = ctx.arena->alloc(bo, nc);
      gemm(ctx, Op::T, Op::N, 1.0, Vo, C, 0.0, W1);
      GemmExtra e;
      e.krange = KRange::ALower;
      gemm(ctx, Op::T, Op::N, 1.0, To, W1, 0.0, W2, e);
      gemm(ctx, Op::N, Op::N, -1.0, Vo, W2, 1.0, C);
      ctx.arena->release_to(mark);
    }
  }
}

void orgqr_cols(Ctx& ctx, const QrWork& w, int64_t m, int64_t n, int64_t c0, const DMat& Q) {
  const int64_t ncols = Q.cols;
  const int nb = w.nb;
  // Q = E(:, c0 : c0+ncols)
  fill(ctx, Q, 0.0, 0.0);
  {
    // identity entries (c0 + i, i)
    DMat D = Q.sub(c0, 0, std::min<int64_t>(ncols, m - c0), std::min<int64_t>(ncols, m - c0));
    fill(ctx, D, 0.0, 1.0);
  }
  const int64_t npan = (n + nb - 1) / nb;
  const Arena::Mark mark = ctx.arena->mark();
  for (int64_t p = npan - 1; p >= 0; --p) {
    const int64_t j0 = p * nb;
    const int64_t b = std::min<int64_t>(nb, n - j0);
    const int64_t mp = m - j0;
    const int64_t i0 = std::max<int64_t>(0, j0 - c0);  // first affected Q column
    if (i0 >= ncols) continue;
    const int64_t nc = ncols - i0;
    const DMat Vp = w.V.sub(j0, j0, mp, b);
    const DMat Tp = w.T.sub(0, p * nb, b, b);
    const DMat C = Q.sub(j0, i0, mp, nc);
    DMat W1 = ctx.arena->alloc(b, nc);
    DMat W2 = ctx.arena->alloc(b, nc);
    gemm(ctx, Op::T, Op::N, 1.0, Vp, C, 0.0, W1);
    GemmExtra e;
    e.krange = KRange::AUpper;  // T upper
    gemm(ctx, Op::N, Op::N, 1.0, Tp, W1, 0.0, W2, e);
    gemm(ctx, Op::N, Op::N, -1.0, Vp, W2, 1.0, C);
    ctx.arena->release_to(mark);
  }
}

void diag_to_host(Ctx& ctx, const DMat& R, std::vector<double>& d) {
  const int64_t n = std::min(R.rows, R.cols);
  d.resize(n);
  double* tmp = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (n + 1)));
  diag_kernel<<<std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148)), 256, 0, ctx.stream>>>(
      R.ptr(), R.ld, n, tmp);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
  QDWHG_CUDA(cudaMemcpyAsync(d.data(), tmp, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
}

}  // namespace qdwhg
