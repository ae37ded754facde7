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

#ifdef QDWHG_PANEL_TRACE
__device__ long long g_panel_trace[16];
#define PANEL_MARK(i, col) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && (col) == 10) g_panel_trace[i] = clock64()
#else
#define PANEL_MARK(i, col)
#endif

constexpr int kPanelThreads = 256;
constexpr int kBW = 64;  // max panel width (one thread column per panel column)
// Deterministic grid-path reduction (the shared-memory grid panel always, the
// register panel when Ctx::deterministic): per-CTA slots
// [2 parity][kMaxGridCtas][2*kBW] after the atomic accumulators, summed in CTA
// order by every CTA after the grid barrier — bitwise reproducible run to run.
constexpr int kMaxGridCtas = 160;
constexpr size_t kAccDoubles = 3 * 2 * kBW;  // atomic accumulators (zero between launches)
constexpr size_t kSlotDoubles = (size_t)2 * kMaxGridCtas * 2 * kBW;


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

// tot[s] = sum of slots[g][s] over CTAs g = 0..G-1 in a fixed order (strided
// groups of nthreads / (2 kBW) threads, then the groups in order): every CTA
// computes the same bits.  `scratch` holds nthreads doubles of shared memory.
__device__ __forceinline__ void slot_sum(const double* slots, int G, double* scratch, double* tot,
                                         int nthreads) {
  const int tid = threadIdx.x;
  const int np = nthreads / (2 * kBW);
  const int s = tid % (2 * kBW), part = tid / (2 * kBW);
  if (part < np) {
    double acc0 = 0.0;
    const double* p = slots + (size_t)part * 2 * kBW + s;
#pragma unroll 4
    for (int g = part; g < G; g += np, p += (size_t)np * 2 * kBW) acc0 += __ldcg(p);
    scratch[part * 2 * kBW + s] = acc0;
  }
  __syncthreads();
  if (tid < 2 * kBW) {
    double t = 0.0;
    for (int q = 0; q < np; ++q) t += scratch[q * 2 * kBW + tid];
    tot[tid] = t;
  }
}

// Unblocked Householder QR of an mp x b panel (b <= 64) whose rows are spread
// over the CTAs of the launch, each CTA keeping its rows in shared memory.
// Per column ONE cross-CTA reduction of [x0, sigma^2, a_jj,c, x^T a_c] gives the
// pivot, tau and all v^T a_c at once.
//   CLUSTER = true : one thread-block cluster (<= 16 CTAs): partial vectors are
//                    read from the peers' shared memory (DSMEM) in fixed order
//                    (deterministic) behind one hardware cluster barrier;
//   CLUSTER = false: any number of co-resident CTAs (cooperative launch): per-CTA
//                    slots + a grid barrier, summed in CTA order (deterministic).
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
    PANEL_MARK(3, col);
    panel_partials(S, RP, nr, rbeg, b, col, red, mine);
    PANEL_MARK(4, col);
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
      // slot per CTA, double-buffered by parity: a CTA writes column col+2's
      // slot only after the barrier of col+1, which every CTA reaches after
      // reading column col's slots
      double* buf = acc + kAccDoubles + (size_t)(col & 1) * kMaxGridCtas * (2 * kBW);
      if (threadIdx.x < 2 * kBW) {
        const int cc = threadIdx.x % kBW;
        __stcg(&buf[(size_t)blockIdx.x * 2 * kBW + threadIdx.x],
               (cc < b && cc >= col) ? mine[threadIdx.x] : 0.0);
      }
      PANEL_MARK(5, col);
      grid_sync(bar, epoch);
      PANEL_MARK(6, col);
      slot_sum(buf, (int)gridDim.x, red, tot, kPanelThreads);
      __syncthreads();
    }
    PANEL_MARK(7, col);
  };

  reduce(0);
  for (int jj = 0; jj < b; ++jj) {
    PANEL_MARK(0, jj);
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
    PANEL_MARK(1, jj);
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
    PANEL_MARK(2, jj);
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

// Register-resident panel factorization (the default for panels up to
// 148 * 256 rows): thread (c, rg) — c = tid % 64 the panel column, rg = tid / 64
// the row group — keeps column c of rows rg + NRG*t (t < RPT) of its CTA's row
// block in registers for the whole panel.  Per column jj there is ONE pass over
// the registers that applies H_jj to the thread's column AND accumulates the
// partial sums of column jj+1 (x0, sigma^2, v^T a_c) from column jj+1's updated
// values, which every thread recomputes from a shared-memory snapshot
// (bit-identical to the owner's update: same inputs, same fma).  Then one
// in-CTA combine and one cross-CTA reduction (cluster DSMEM or grid atomics),
// i.e. two CTA barriers + one cluster/grid barrier per column.
// T (b x b upper) from G = V^T V and tau' (LAPACK dlarft, forward/columnwise),
// by recursive doubling instead of the column recurrence:
//   T = [T11, -T11 (V1^T V2) T22; 0, T22],  V1^T V2 = G12,
// block size s = 1, 2, 4, ... — 2 barriers per level, log2(b) levels.
// One doubling level of larft with compile-time block size S: the k loops are
// fully unrolled (zero terms by predicate) so every thread's shared loads are
// in flight together instead of one load-FMA round trip per term.
template <int S>
QDWHG_DEV void larft_level(double (*Ts)[kBW + 1], double (*M)[kBW + 1], double (*Gs)[kBW + 1], int b,
                           int t) {
  if (S >= b) return;
  // M(a+r, a+S+c) = sum_{k=r}^{S-1} T11(r, k) G(a+k, a+S+c)
  for (int i = t; i < b * S; i += blockDim.x) {
    const int r = i % S, rest = i / S;
    const int pair = rest / S, c = rest % S;
    const int a = pair * 2 * S;
    if (a + S + c >= b) continue;
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const double v = (k >= r) ? Ts[a + r][a + k] * Gs[a + k][a + S + c] : 0.0;
      if (k & 1) acc1 += v;
      else acc0 += v;
    }
    M[a + r][a + S + c] = acc0 + acc1;
  }
  __syncthreads();
  // T12(r, c) = -sum_{k=0}^{c} M(a+r, a+S+k) T22(k, c)
  for (int i = t; i < b * S; i += blockDim.x) {
    const int r = i % S, rest = i / S;
    const int pair = rest / S, c = rest % S;
    const int a = pair * 2 * S;
    if (a + S + c >= b) continue;
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const double v = (k <= c) ? M[a + r][a + S + k] * Ts[a + S + k][a + S + c] : 0.0;
      if (k & 1) acc1 += v;
      else acc0 += v;
    }
    Ts[a + r][a + S + c] = -(acc0 + acc1);
  }
  __syncthreads();
}

// Fused panel tail (PanelTail): the compact-WY T of the panel is built inside
// the column loop.  G(c, j) = v_c^T v_j for c < j rides in the otherwise unused
// slots c < j of the per-column reduction vector (threads of finished columns
// accumulate a_c . u over their rows during the same register pass), and CTA 0
// extends T by the LAPACK dlarft column recurrence
//   T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j)
// while the next reduction is in flight — no Gram GEMM, no larft launch.  The
// kernel also zeroes V above the panel inside its outer block and (grid path)
// leaves its barrier/accumulator buffers zeroed for the next launch.
struct PanelTail {
  double* T;          // b x b upper T (zeros below) of the panel, ld ldt
  int64_t ldt;
  double* vz;         // V rows above the panel that must be zero: zrows x b, ld ldv
  int zrows;
  unsigned* ticket;   // grid path: last-CTA election for the buffer cleanup
};

template <bool CLUSTER, int NRG, int RPT, bool DET>
__global__ void __launch_bounds__(64 * NRG, 1)
    geqr2_panel_reg_kernel(double* A, int64_t lda, double* V, int64_t ldv, double* tau_out, int mp,
                           int b, int rpc, double* acc, unsigned* bar, PanelTail tl) {
  constexpr int NT = kBW * NRG;
  constexpr int RB = NRG * RPT;  // row capacity per CTA (>= rpc)
  constexpr int RBP = RB + 1;
  extern __shared__ double smem[];
  double* stage = smem;                 // [kBW][RBP]: coalesced load / store staging
  // [2 parity][RB] x (u, p): column jj and column jj+1 interleaved, so each
  // row's pair is ONE broadcast 16-byte shared load in the hot loop
  double* snap = stage + kBW * RBP;
  double* red = snap + 4 * RB;          // [NRG][2*kBW]
  double* part = red + NRG * 2 * kBW;   // [2 parity][2*kBW] this CTA's partials
  double* tot = part + 4 * kBW;         // [2*kBW] reduced (top | below)
  double* gbuf = tot + 2 * kBW;         // CLUSTER: [2 parity][16 ranks][2*kBW] pushed partials
  double* colsc = gbuf + 2 * 16 * 2 * kBW;  // [kBW] 1/v0 (0: no reflector) | [kBW] beta, per column
  uint64_t* mbar = reinterpret_cast<uint64_t*>(colsc + 2 * kBW);  // CLUSTER: [2] gather barriers
  // CTA 0: G = V^T V (strict upper; tau_j kept on the diagonal) for the T of the tail
  double(*Gs)[kBW + 1] = reinterpret_cast<double(*)[kBW + 1]>(mbar + 2);
  // larft work arrays after the panel: the staging area when large enough, else
  // appended after Gs
  double* lwork = (kBW * (RB + 1) >= 2 * kBW * (kBW + 1)) ? stage : &Gs[kBW][0];
  const int tid = threadIdx.x;
  const int c = tid % kBW, rg = tid / kBW;
  const int rbeg = blockIdx.x * rpc;
  const int nr = max(0, min(rpc, mp - rbeg));
  unsigned epoch = 0;
  namespace cg = cooperative_groups;

  // ---- coalesced load through shared memory, then into registers
  for (int cc = 0; cc < b; ++cc)  // cp.async: every element in flight at once
    for (int i = tid; i < nr; i += NT) cp_async8(stage + cc * RBP + i, A + (rbeg + i) + (int64_t)cc * lda);
  cp_async_wait_all();
  __syncthreads();
  double a[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int i = rg + NRG * t;
    a[t] = (c < b && i < nr) ? stage[c * RBP + i] : 0.0;  // rows past nr stay exactly 0
    if (c == 0) snap[2 * i] = a[t];
    if (c == 1) snap[2 * i + 1] = a[t];
  }
  for (int i = tid; i < 2 * RB; i += NT) snap[2 * RB + i] = 0.0;
  if (CLUSTER) {
    // gather barriers: column col's partials from all ranks land in
    // gbuf[col & 1] via st.async, completing tx bytes on mbar[col & 1]
    if (tid == 0) {
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      fence_barrier_init();
    }
    cg::this_cluster().sync();
    if (tid == 0) {
      const uint32_t bytes = (uint32_t)cg::this_cluster().num_blocks() * 2 * kBW * 8;
      mbar_arrive_expect_tx(&mbar[0], bytes);
      mbar_arrive_expect_tx(&mbar[1], bytes);  // reductions run for col = 0 .. b
    }
  }
  __syncthreads();

  // cross-CTA sum of the per-row-group partials in `red` -> tot
  // side(): work for threads that are not on the reduction's critical path
  // (snapshot writes), run while the partials are in flight
  auto reduce = [&](int col, auto&& side) {
    double* mine = part + (col & 1) * (2 * kBW);
    if (tid < 2 * kBW) {
      double s = 0.0;
#pragma unroll
      for (int g = 0; g < NRG; ++g) s += red[g * 2 * kBW + tid];
      mine[tid] = s;
    }
    if (CLUSTER) {
      // all-gather by st.async: this CTA's vector goes into slot [my rank] of
      // every peer, each store completing bytes on the peer's mbar[col & 1];
      // the local wait then sums the slots in fixed rank order (deterministic)
      cg::cluster_group cluster = cg::this_cluster();
      const int nb_ = (int)cluster.num_blocks();
      const int me = (int)cluster.block_rank();
      const int q = col & 1;
      double* g = gbuf + q * (16 * 2 * kBW);
      __syncthreads();  // `mine` complete
      if (tid < kBW) {
        const uint32_t src = smem_u32(g + me * (2 * kBW) + 2 * tid);
        const uint32_t mb = smem_u32(&mbar[q]);
        const double x = mine[2 * tid], y = mine[2 * tid + 1];
        for (int p = 0; p < nb_; ++p) st_async_v2(mapa_u32(src, p), x, y, mapa_u32(mb, p));
      }
      side();
      if (tid < 2 * kBW) {
        mbar_wait_cluster(&mbar[q], (col >> 1) & 1);
        double s = 0.0;
        for (int p = 0; p < nb_; ++p) s += g[p * 2 * kBW + tid];
        tot[tid] = s;
        // re-arm for column col + 2 by a thread that sent nothing (a sender's
        // release-arrive would wait for its own remote stores to land)
        if (tid == kBW && col + 2 <= b) mbar_arrive_expect_tx(&mbar[q], (uint32_t)nb_ * 2 * kBW * 8);
      }
      __syncthreads();
    } else {
      if constexpr (DET) {
        // per-CTA slots, parity double-buffered (see geqr2_panel_kernel)
        double* buf = acc + kAccDoubles + (size_t)(col & 1) * kMaxGridCtas * (2 * kBW);
        if (tid < 2 * kBW) __stcg(&buf[(size_t)blockIdx.x * 2 * kBW + tid], mine[tid]);
        side();
        grid_sync(bar, epoch);
        slot_sum(buf, (int)gridDim.x, red, tot, NT);
        __syncthreads();
        return;
      }
      double* buf = acc + (col % 3) * (2 * kBW);
      if (tid < 2 * kBW) {
        const int cc = tid % kBW;
        if (cc < b && mine[tid] != 0.0) atomicAdd(&buf[tid], mine[tid]);  // (cc < col: Gram slots)
      }
      side();
      grid_sync(bar, epoch);
      if (tid < 2 * kBW) tot[tid] = __ldcg(&buf[tid]);
      if (blockIdx.x == 0) {  // buffer col+2 was last read before this barrier
        double* z = acc + ((col + 2) % 3) * (2 * kBW);
        if (tid < 2 * kBW) z[tid] = 0.0;
      }
      __syncthreads();
    }
  };

  // partials of column 0
  {
    double top = 0.0, below = 0.0;
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int i = rg + NRG * t, gr = rbeg + i;
      if (i < nr && c < b) {
        if (gr == 0) top = a[t];
        else below = fma(snap[2 * i], a[t], below);
      }
    }
    red[rg * 2 * kBW + c] = top;
    red[rg * 2 * kBW + kBW + c] = below;
    __syncthreads();
    reduce(0, [] {});
  }

  // Snapshot conventions (shared memory, per parity):
  //   U = column jj with 0 above row jj (its row-jj entry becomes v0 at step jj),
  //       so u = v0 * v and a_c -= s_c u is the complete H_jj update of any row;
  //   P = column jj+1 (raw); its updated value pv is recomputed by every thread
  //       (same fma as its owner's) for the partial sums of column jj+1.
  // The pivot column itself is left raw (s_jj = 0) and normalised at the end
  // (v = a / v0 below the diagonal, beta on it), from per-column scalars.
  for (int jj = 0; jj < b; ++jj) {
    PANEL_MARK(8, jj);
    const int par = jj & 1;
    const double2* UP = reinterpret_cast<const double2*>(snap) + par * RB;  // (u, p) per row
    double* UPn = snap + (par ^ 1) * 2 * RB;                               // next step's pairs
    const double x0 = tot[jj];
    const double sig2 = tot[kBW + jj];
    const double nx2 = fma(x0, x0, sig2);
    const bool reflect = (jj < mp - 1) && nx2 > 0.0;
    // short dependent chain (FP64 latency is the column's critical path):
    //   rn = 1/||x||, v0 = x0 - beta = x0 + sign(x0) ||x||, tau' = 1 + |x0| rn,
    //   s_c = tau' (v^T a_c) / v0 = sign(x0) rn (a_c(j) + x_b^T a_c / v0)
    double beta = x0, v0 = 1.0, taup = 0.0, inv_v0 = 1.0, srn = 0.0;
    if (reflect) {
      const double rn = fast_rsqrt(nx2);
      const double normx = nx2 * rn;
      v0 = x0 + copysign(normx, x0);
      inv_v0 = fast_rcp(v0);
      beta = -copysign(normx, x0);
      taup = fma(fabs(x0), rn, 1.0);
      srn = copysign(rn, x0);
    }
    // w_c = tau' v^T a_c  (v = [1; x_below / v0]);  s_c = w_c / v0 scales u = v0 v
    double sc = 0.0, s1 = 0.0;
    if (reflect && c > jj && c < b) sc = srn * fma(tot[kBW + c], inv_v0, tot[c]);
    if (reflect && jj + 1 < b) s1 = srn * fma(tot[kBW + jj + 1], inv_v0, tot[jj + 1]);
    if (tid == 0) {  // read after the last step's barriers
      colsc[jj] = reflect ? inv_v0 : 0.0;
      colsc[kBW + jj] = beta;
    }
    if (blockIdx.x == 0) {
      if (tid == 0) {
        tau_out[jj] = taup;
        Gs[jj][jj] = taup;
      }
      // G(c, jj-1), c < jj-1, from the Gram slots of the reduction just completed
      // (v_c = a_c / v0_c below its diagonal, a_c(jj-1) on row jj-1)
      if (jj >= 2 && tid < jj - 1)
        Gs[tid][jj - 1] = colsc[tid] * (tot[tid] + tot[kBW + tid] * colsc[jj - 1]);
    }
    PANEL_MARK(9, jj);
    double top = 0.0, below = 0.0;
    const int kmask = jj + 1 - rbeg - rg;  // element t has row <= jj+1 iff NRG*t <= kmask
    // columns right of the pivot: H_jj update + partials of column jj+1 (rows > jj+1,
    // top = row jj+1); finished columns c < jj (sc = 0, unchanged): Gram partials
    // a_c . u over rows > jj, top = row jj
    const bool gram = c < jj;
    if ((tid % kBW) / 32 * 32 + 31 < jj) {
      // warp of finished columns only: Gram partials, nothing to update
      const double* U = reinterpret_cast<const double*>(UP);
      double bl[4] = {0.0, 0.0, 0.0, 0.0};
      const int lo = kmask - 1;
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const int i = rg + NRG * t;
        bl[t & 3] = (NRG * t > lo) ? fma(U[2 * i], a[t], bl[t & 3]) : bl[t & 3];
      }
      below = (bl[0] + bl[1]) + (bl[2] + bl[3]);
      if (lo >= 0 && lo % NRG == 0) {
#pragma unroll
        for (int t = 0; t < RPT; ++t)
          if (NRG * t == lo) top = a[t];  // row jj
      }
    } else if (kmask < 0) {
      double bl[4] = {0.0, 0.0, 0.0, 0.0};  // 4 chains: FP64 latency, not throughput
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const int i = rg + NRG * t;
        const double2 up = UP[i];
        const double u = up.x;
        const double pv = fma(-s1, u, up.y);
        const double an = fma(-sc, u, a[t]);
        a[t] = an;
        bl[t & 3] = fma(gram ? u : pv, an, bl[t & 3]);
      }
      below = (bl[0] + bl[1]) + (bl[2] + bl[3]);
    } else {
      double bl[4] = {0.0, 0.0, 0.0, 0.0};
      const int lo = gram ? kmask - 1 : kmask;  // rows counted: NRG*t > lo
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const int i = rg + NRG * t;
        const double2 up = UP[i];
        const double u = (NRG * t == kmask - 1) ? v0 : up.x;  // row jj: u = v0 (v = 1)
        const double pv = fma(-s1, u, up.y);
        const double an = fma(-sc, u, a[t]);
        a[t] = an;
        bl[t & 3] = (NRG * t > lo) ? fma(gram ? up.x : pv, an, bl[t & 3]) : bl[t & 3];
      }
      below = (bl[0] + bl[1]) + (bl[2] + bl[3]);
      if (lo >= 0 && lo % NRG == 0) {
#pragma unroll
        for (int t = 0; t < RPT; ++t)
          if (NRG * t == lo) top = a[t];  // row jj+1 (gram: row jj)
      }
    }
    PANEL_MARK(10, jj);
    if (!(c < b && (c > jj ? jj + 1 < b : gram))) top = below = 0.0;
    // snapshots of columns jj+1 (zero above its diagonal) and jj+2 (owners
    // only), written while the partial sums are in flight
    auto snapshots = [&] {
      if (c == jj + 1) {
#pragma unroll
        for (int t = 0; t < RPT; ++t) UPn[2 * (rg + NRG * t)] = (NRG * t < kmask) ? 0.0 : a[t];
      } else if (c == jj + 2) {
#pragma unroll
        for (int t = 0; t < RPT; ++t) UPn[2 * (rg + NRG * t) + 1] = a[t];
      }
    };
    red[rg * 2 * kBW + c] = top;
    red[rg * 2 * kBW + kBW + c] = below;
    PANEL_MARK(11, jj);
    __syncthreads();
    PANEL_MARK(12, jj);
    // (jj + 1 == b: the last reduction carries only the Gram slots of column b-1)
    reduce(jj + 1, snapshots);
    PANEL_MARK(13, jj);
  }
  // last G column (j = b-1) from the final reduction
  if (blockIdx.x == 0 && tid < b - 1)
    Gs[tid][b - 1] = colsc[tid] * (tot[tid] + tot[kBW + tid] * colsc[b - 1]);
  if (CLUSTER) cg::this_cluster().sync();  // peers may still write into our buffers
  __syncthreads();
  // ---- pivot columns: v = a / v0 below the diagonal, beta on it; then R (upper,
  // zeros below) and V (zeros above, unit diagonal) through staging
  if (c < b) {
    const double iv = colsc[c], bt = colsc[kBW + c];
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int i = rg + NRG * t, gr = rbeg + i;
      double x = a[t];
      if (gr == c) x = bt;
      else if (gr > c) x *= iv;
      if (i < nr) stage[c * RBP + i] = x;
    }
  }
  __syncthreads();
  for (int cc = 0; cc < b; ++cc)
    for (int i = tid; i < nr; i += NT) {
      const int gr = rbeg + i;
      const double x = stage[cc * RBP + i];
      A[gr + (int64_t)cc * lda] = (gr <= cc) ? x : 0.0;
      V[gr + (int64_t)cc * ldv] = (gr < cc) ? 0.0 : (gr == cc ? 1.0 : x);
    }
  // ---- T (LAPACK dlarft) of the panel by CTA 0: recursive doubling on G
  if (blockIdx.x == 0) {
    __syncthreads();  // staging reads of the write-out done (lwork may alias it)
    double(*Ts)[kBW + 1] = reinterpret_cast<double(*)[kBW + 1]>(lwork);
    double(*M)[kBW + 1] = reinterpret_cast<double(*)[kBW + 1]>(lwork + kBW * (kBW + 1));
    for (int q = tid; q < kBW * kBW; q += NT) {
      const int r = q % kBW, cc = q / kBW;
      Ts[r][cc] = (r == cc && r < b) ? Gs[r][r] : 0.0;
    }
    __syncthreads();
    larft_level<1>(Ts, M, Gs, b, tid);
    larft_level<2>(Ts, M, Gs, b, tid);
    larft_level<4>(Ts, M, Gs, b, tid);
    larft_level<8>(Ts, M, Gs, b, tid);
    larft_level<16>(Ts, M, Gs, b, tid);
    larft_level<32>(Ts, M, Gs, b, tid);
    for (int q = tid; q < b * b; q += NT) {
      const int r = q % b, cc = q / b;
      tl.T[r + (int64_t)cc * tl.ldt] = Ts[r][cc];
    }
  }
  // V rows above the panel inside its outer block are zero (GEMMs read them)
  for (int q = blockIdx.x * NT + tid; q < tl.zrows * b; q += gridDim.x * NT) {
    const int r = q % tl.zrows, cc = q / tl.zrows;
    tl.vz[r + (int64_t)cc * ldv] = 0.0;
  }
  if (!CLUSTER) {
    // leave the barrier counter and accumulators zeroed for the next launch: the
    // last CTA to get here knows every CTA has passed its final grid barrier
    __shared__ bool last;
    __syncthreads();
    if (tid == 0) last = atomicAdd(tl.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
      for (int q = tid; q < 3 * 2 * kBW; q += NT) acc[q] = 0.0;
      if (tid == 0) {
        *bar = 0u;
        *tl.ticket = 0u;
      }
    }
  }
}

template <int NRG, int RPT>
size_t panel_reg_smem() {
  constexpr int RB = NRG * RPT;
  return ((size_t)kBW * (RB + 1) + 4 * RB + NRG * 2 * kBW + 4 * kBW + 2 * kBW + 2 * 16 * 2 * kBW +
          2 * kBW + 2 + kBW * (kBW + 1) +
          ((kBW * (RB + 1) >= 2 * kBW * (kBW + 1)) ? 0 : 2 * kBW * (kBW + 1))) *
         8;  // (+ G and, unless the staging area holds them, the larft work arrays)
}

__global__ void larft_kernel(const double* G, int64_t ldg, const double* tau, double* T,
                             int64_t ldt, int b) {
  extern __shared__ double larft_sm[];
  double(*Ts)[kBW + 1] = reinterpret_cast<double(*)[kBW + 1]>(larft_sm);
  double(*M)[kBW + 1] = reinterpret_cast<double(*)[kBW + 1]>(larft_sm + kBW * (kBW + 1));
  double(*Gs)[kBW + 1] = reinterpret_cast<double(*)[kBW + 1]>(larft_sm + 2 * kBW * (kBW + 1));
  const int t = threadIdx.x;
  griddep_wait();
  // G (upper part used) and tau staged in shared memory once: the doubling
  // loops below only touch shared memory
  for (int i = t; i < b * b; i += blockDim.x) {
    const int r = i % b, c = i / b;
    Gs[r][c] = G[r + (int64_t)c * ldg];
  }
  for (int i = t; i < kBW * kBW; i += blockDim.x) {
    const int r = i % kBW, c = i / kBW;
    Ts[r][c] = (r == c && r < b) ? tau[r] : 0.0;
  }
  __syncthreads();
  larft_level<1>(Ts, M, Gs, b, t);
  larft_level<2>(Ts, M, Gs, b, t);
  larft_level<4>(Ts, M, Gs, b, t);
  larft_level<8>(Ts, M, Gs, b, t);
  larft_level<16>(Ts, M, Gs, b, t);
  larft_level<32>(Ts, M, Gs, b, t);
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
  return per_device_cached(0, [] {
    int cs = 8;
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
    return cs;
  });
}

// Largest cluster the register-resident panel kernel can use (16 non-portable, else 8).
int reg_cluster_limit() {
  return per_device_cached(1, [] {
    int cs = 8;
    auto kern = geqr2_panel_reg_kernel<true, 8, 32, false>;
    const size_t smem = panel_reg_smem<8, 32>();
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
            cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = 16;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) cs = 16;
    }
    cudaGetLastError();
    return cs;
  });
}

template <bool CL, int RPT, bool DET = false, int NRG = 8>
void launch_panel_reg_t(Ctx& ctx, int nblk, double* Ap, int64_t lda, double* Vptr, int64_t ldv,
                      double* tau_dev, int mp, int b, int rpc, double* acc, unsigned* bar,
                      PanelTail tl) {
  auto kern = geqr2_panel_reg_kernel<CL, NRG, RPT, DET>;
  const size_t smem = panel_reg_smem<NRG, RPT>();
  func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CL) func_attr(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (CL) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblk);
    cfg.blockDim = dim3(64 * NRG);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx.stream;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = nblk;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    QDWHG_CUDA(cudaLaunchKernelEx(&cfg, kern, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl));
  } else {
    // acc / bar / ticket are zero on entry (geqrf zeroes them once; every grid
    // launch leaves them zeroed)
    void* args[] = {&Ap, &lda, &Vptr, &ldv, &tau_dev, &mp, &b, &rpc, &acc, &bar, &tl};
    QDWHG_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(nblk), dim3(64 * NRG), args, smem,
                                           ctx.stream));
  }
  ctx.count();
}

template <bool CL, int RPT>
void launch_panel_reg(Ctx& ctx, int nblk, double* Ap, int64_t lda, double* Vptr, int64_t ldv,
                      double* tau_dev, int mp, int b, int rpc, double* acc, unsigned* bar,
                      PanelTail tl) {
  if (!CL && ctx.deterministic)
    launch_panel_reg_t<CL, RPT, true>(ctx, nblk, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
  else
    launch_panel_reg_t<CL, RPT, false>(ctx, nblk, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
}

// Register-resident panel when the panel fits (cluster of <= 16 CTAs x 256
// rows, or a cooperative grid of <= #SMs CTAs x 256 rows); false otherwise.
bool panel_factor_reg(Ctx& ctx, const DMat& P, const DMat& Vp, double* tau_dev, double* acc,
                      unsigned* bar, const PanelTail& tl) {
  static const bool disabled = getenv("QDWHG_PANEL_SMEM") != nullptr;
  if (disabled) return false;
  const int mp = (int)P.rows, b = (int)P.cols;
  double* Ap = P.ptr();
  const int64_t lda = P.ld;
  double* Vptr = Vp.ptr();
  const int64_t ldv = Vp.ld;
  const int csmax = reg_cluster_limit();
  auto ceil_div = [](int x, int y) { return (x + y - 1) / y; };
  // cluster (deterministic DSMEM reduction, hardware barrier)
  if (ceil_div(mp, 8 * 4) <= csmax) {
    const int cs = ceil_div(mp, 8 * 4), rpc = ceil_div(mp, cs);
    launch_panel_reg<true, 4>(ctx, cs, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
    return true;
  }
  if (ceil_div(mp, 8 * 8) <= csmax) {
    const int cs = ceil_div(mp, 8 * 8), rpc = ceil_div(mp, cs);
    launch_panel_reg<true, 8>(ctx, cs, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
    return true;
  }
  if (ceil_div(mp, 8 * 16) <= csmax) {
    const int cs = ceil_div(mp, 8 * 16), rpc = ceil_div(mp, cs);
    launch_panel_reg<true, 16>(ctx, cs, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
    return true;
  }
  // (a 16-CTA cluster of 256-row CTAs was slower than the grid path at 4096
  // rows: 3.13 vs 2.60 us/column — the per-column register pass dominates)

  // cooperative grid (FP64 atomics + grid barrier); while a look-ahead side
  // stream runs, the grid is capped (ctx.panel_max_ctas) so the panel does not
  // need the whole machine at once
  const int sms = std::min(ctx.num_sms, kMaxGridCtas);  // slot capacity of the grid reduction
  const int max_ctas = ctx.panel_max_ctas > 0 ? std::min(ctx.panel_max_ctas, sms) : sms;
  if (ceil_div(mp, 8 * 8) <= max_ctas) {
    const int nb = ceil_div(mp, 8 * 8), rpc = ceil_div(mp, nb);
    launch_panel_reg<false, 8>(ctx, nb, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
    return true;
  }
  if (ceil_div(mp, 8 * 16) <= max_ctas) {
    const int nb = ceil_div(mp, 8 * 16), rpc = ceil_div(mp, nb);
    launch_panel_reg<false, 16>(ctx, nb, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
    return true;
  }
  if (ceil_div(mp, 8 * 32) <= max_ctas) {
    const int nb = ceil_div(mp, 8 * 32), rpc = ceil_div(mp, nb);
    launch_panel_reg<false, 32>(ctx, nb, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
    return true;
  }
  if (max_ctas < sms) {  // taller than the cap allows: uncapped
    if (ceil_div(mp, 8 * 16) <= sms) {
      const int nb = ceil_div(mp, 8 * 16), rpc = ceil_div(mp, nb);
      launch_panel_reg<false, 16>(ctx, nb, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
      return true;
    }
    if (ceil_div(mp, 8 * 32) <= sms) {
      const int nb = ceil_div(mp, 8 * 32), rpc = ceil_div(mp, nb);
      launch_panel_reg<false, 32>(ctx, nb, Ap, lda, Vptr, ldv, tau_dev, mp, b, rpc, acc, bar, tl);
      return true;
    }
  }
  return false;
}

// Returns true when the panel's T (and the zeroed V rows above it) came out of
// the fused register-panel kernel; false: the caller forms T (Gram + larft).
bool panel_factor(Ctx& ctx, const DMat& P, const DMat& Vp, double* tau_dev, double* acc,
                  unsigned* bar, const PanelTail& tl) {
  if (panel_factor_reg(ctx, P, Vp, tau_dev, acc, bar, tl)) return true;
  // shared-memory panel kernel: panels taller than the register path covers
  int mp = (int)P.rows, b = (int)P.cols;
  func_attr(geqr2_panel_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPanelSmemMax);
  func_attr(geqr2_panel_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPanelSmemMax);
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
    return false;
  }
  // grid path (tall panels): cooperative launch over up to all SMs
  const int nblk = std::max(1, std::min(std::min(ctx.num_sms, kMaxGridCtas), (mp + 63) / 64));
  rpc = (mp + nblk - 1) / nblk;
  if (panel_smem(rpc) > kPanelSmemMax) throw InvalidArgument("geqrf: panel too tall for shared memory");
  QDWHG_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), ctx.stream));
  void* args[] = {&Ap, &lda, &Vptr, &ldv, &tau_dev, &mp, &b, &rpc, &acc, &bar};
  QDWHG_CUDA(cudaLaunchCooperativeKernel((void*)geqr2_panel_kernel<false>, dim3(nblk),
                                         dim3(kPanelThreads), args, panel_smem(rpc), ctx.stream));
  ctx.count();
  // the register kernels expect a zeroed barrier counter on entry (the atomic
  // accumulators were not touched: this kernel reduces through the slots)
  QDWHG_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), ctx.stream));
  return false;
}

}  // namespace

// T (b x b, b <= 64) of a compact-WY block from its Gram G = V^T V and taus.
void larft_launch(Ctx& ctx, const DMat& G, const double* tau_dev, const DMat& T) {
  func_attr(larft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * kBW * (kBW + 1) * 8);
  launch_pdl(ctx, larft_kernel, dim3(1), dim3(512), (size_t)(3 * kBW * (kBW + 1) * 8), G.ptr(), G.ld,
             tau_dev, T.ptr(), T.ld, (int)G.rows);
  ctx.count();
}

void geqrf(Ctx& ctx, const DMat& A, QrWork& w, int64_t top_rows) {
  const int64_t m = A.rows, n = A.cols;
  if (m < n) throw InvalidArgument("geqrf: requires rows >= cols");
  if (top_rows < 0 || top_rows > m) throw InvalidArgument("geqrf: bad structure");
  // Structured stack [T; U] (top_rows > 0: rows [top_rows, m) upper triangular,
  // e.g. the QDWH QR step's [sqrt(c) X; I], polar.cpp:56-72): a reflector of
  // column c touches rows < top_rows + c + 1 only, and the rows below stay zero
  // in every column to its right, so every panel and update of columns
  // [j0, j0 + b) runs on rows [j0, top_rows + j0 + b) — for m = 2n, (n + b) rows
  // instead of (2n - j0): ~40 % fewer flops, shorter panels.  Same reflectors.
  w.top_rows = top_rows;
  auto rend = [&](int64_t c) { return top_rows > 0 ? std::min<int64_t>(m, top_rows + c) : m; };
  // Two-level blocking: 64-column panels (one cooperative/cluster kernel each)
  // inside 256-column outer blocks.  Inner updates touch only the outer block;
  // the outer T (256 x 256) is assembled by merging the panel T's
  // (T = [T1, -T1 (V1^T V2) T2; 0, T2]) so the trailing update of the rest of
  // the matrix — the O(n^3) part — runs as GEMMs with K = 256.
  const int nbi = kBW;
  static const int nbo_env = getenv("QDWHG_QR_NBO") ? atoi(getenv("QDWHG_QR_NBO")) : 0;
  // outer block: 256 columns; 512 for very wide matrices, where the K = 512
  // trailing GEMMs' efficiency gain outweighs the longer inner chain (cfg4:
  // QR 286 -> 265 ms; at n <= 8192 256 is faster)
  const int nbo = (nbo_env == 128 || nbo_env == 256 || nbo_env == 512) ? nbo_env
                  : (n >= 12288) ? 8 * kBW : 4 * kBW;
  w.nb = nbo;
  const int64_t nout = (n + nbo - 1) / nbo;
  w.V = ctx.arena->alloc(m, n);
  if (top_rows > 0) fill(ctx, w.V, 0.0, 0.0);  // V below each panel's row range stays zero
  w.T = ctx.arena->alloc(nbo, nout * nbo);
  fill(ctx, w.T, 0.0, 0.0);
  double* tau_dev = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (n + 64)));
  // [atomic accumulators | deterministic slots | barrier, ticket]
  double* acc = static_cast<double*>(ctx.arena->alloc_bytes(sizeof(double) * (kAccDoubles + kSlotDoubles) + 256));
  unsigned* bar = reinterpret_cast<unsigned*>(acc + kAccDoubles + kSlotDoubles);  // [0] barrier, [32] ticket
  QDWHG_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * kAccDoubles, ctx.stream));
  QDWHG_CUDA(cudaMemsetAsync(bar, 0, 256, ctx.stream));
  DMat G = ctx.arena->alloc(nbo, nbo);
  static const bool no_la = getenv("QDWHG_QR_NO_LOOKAHEAD") != nullptr;
  const bool lookahead = !no_la && ctx.side != nullptr && n > 2 * nbo;
  // side-stream scratch lives for the whole factorisation (never rewound
  // while side-stream kernels may still read it)
  DMat SW1, SW2;
  if (lookahead) {
    SW1 = ctx.arena->alloc(nbo, n);
    SW2 = ctx.arena->alloc(nbo, n);
  }
  bool side_pending = false;
  // with look-ahead the latency-bound chain (panels, inner updates, next-block
  // update) runs on the high-priority stream so the side stream's big GEMM
  // tiles yield SMs to it as they retire
  cudaStream_t caller = ctx.stream;
  static const bool no_prio = getenv("QDWHG_NO_PRIORITY") != nullptr;
  const bool use_hi = lookahead && !no_prio && ctx.hi != nullptr;
  if (use_hi) {
    QDWHG_CUDA(cudaEventRecord(ctx.ev_main, caller));
    QDWHG_CUDA(cudaStreamWaitEvent(ctx.hi, ctx.ev_main, 0));
    ctx.stream = ctx.hi;
  }
  // measured: cap 64 -> cfg4 QR 247 -> 239 ms, cfg3 66.8 -> 63.2 ms
  static const int pcap_env = getenv("QDWHG_PANEL_CAP") ? atoi(getenv("QDWHG_PANEL_CAP")) : 64;
  const int saved_cap = ctx.panel_max_ctas;
  ctx.panel_max_ctas = lookahead ? pcap_env : 0;
  const Arena::Mark mark = ctx.arena->mark();
  for (int64_t po = 0; po < nout; ++po) {
    const int64_t jo = po * nbo;
    const int64_t bo = std::min<int64_t>(nbo, n - jo);
    const int64_t mo = rend(jo + bo) - jo;
    const DMat To = w.T.sub(0, po * nbo, bo, bo);
    std::vector<std::pair<int64_t, int64_t>> blocks;  // (offset in outer block, width)
    for (int64_t ji = 0; ji < bo; ji += nbi) {
      const int64_t bi = std::min<int64_t>(nbi, bo - ji);
      const int64_t j0 = jo + ji;
      const int64_t mp = rend(j0 + bi) - j0;
      const DMat Vp = w.V.sub(j0, j0, mp, bi);
      const DMat Ti = To.sub(ji, ji, bi, bi);
      PanelTail tl;
      tl.T = Ti.ptr();
      tl.ldt = Ti.ld;
      tl.zrows = (int)ji;  // V rows jo .. j0-1 of the panel columns (read by the outer-block GEMMs)
      tl.vz = w.V.sub(jo, j0, std::max<int64_t>(ji, 1), bi).ptr();
      tl.ticket = bar + 32;
      if (!panel_factor(ctx, A.sub(j0, j0, mp, bi), Vp, tau_dev + j0, acc, bar, tl)) {
        if (j0 > 0) fill(ctx, w.V.sub(0, j0, j0, bi), 0.0, 0.0);  // V above the panel is zero
        const DMat Gp = G.sub(0, 0, bi, bi);
        gemm(ctx, Op::T, Op::N, 1.0, Vp, Vp, 0.0, Gp);
        larft_launch(ctx, Gp, tau_dev + j0, Ti);
      }
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
    // ---- trailing update of the rest: C = C - V T^T (V^T C), K = bo.
    // Look-ahead: the next outer block's columns are updated first on the main
    // stream (its panels can start right away); the remaining columns are
    // updated on the side stream, overlapping the next block's latency-bound
    // panel chain.  Column ranges are disjoint; events order the hand-offs.
    if (nc > 0) {
      const DMat Vo = w.V.sub(jo, jo, mo, bo);
      const int64_t bn = lookahead ? std::min<int64_t>(nbo, nc) : nc;
      if (side_pending) QDWHG_CUDA(cudaStreamWaitEvent(ctx.stream, ctx.ev_side, 0));
      {
        const DMat C = A.sub(jo, jo + bo, mo, bn);
        DMat W1 = ctx.arena->alloc(bo, bn), W2 = ctx.arena->alloc(bo, bn);
        gemm(ctx, Op::T, Op::N, 1.0, Vo, C, 0.0, W1);
        GemmExtra e;
        e.krange = KRange::ALower;
        gemm(ctx, Op::T, Op::N, 1.0, To, W1, 0.0, W2, e);
        gemm(ctx, Op::N, Op::N, -1.0, Vo, W2, 1.0, C);
        ctx.arena->release_to(mark);
      }
      if (nc > bn) {
        QDWHG_CUDA(cudaEventRecord(ctx.ev_main, ctx.stream));
        cudaStream_t main_stream = ctx.stream;
        ctx.stream = ctx.side;
        QDWHG_CUDA(cudaStreamWaitEvent(ctx.stream, ctx.ev_main, 0));
        const int64_t nr = nc - bn;
        // The side GEMMs run in column chunks of at most ~64 128x128 tiles:
        // the next panel is a cooperative launch that needs its SMs free at
        // once, so the side stream must never occupy the whole machine.
        GemmExtra e0;
        e0.split_k = 1;  // no arena scratch on the side stream
        e0.force_bm = 128;
        GemmExtra e;
        e.krange = KRange::ALower;
        e.split_k = 1;
        e.force_bm = 128;
        // cap only for mid-size matrices (measured: helps at 4096^2, hurts at
        // 8192^2, 16384^2 and 32768 x 4546, where the side work dominates and
        // the grid panels need most SMs anyway)
        static const int64_t cap_env = getenv("QDWHG_QR_SIDE_CAP") ? atoll(getenv("QDWHG_QR_SIDE_CAP")) : 0;
        const int64_t cap_tiles =
            cap_env > 0 ? cap_env : ((m <= 6144 && n <= 6144) ? 64 : (int64_t)1 << 40);
        const int64_t cw1 = std::max<int64_t>(128, (cap_tiles / ((bo + 127) / 128)) * 128);
        const int64_t cw2 = std::max<int64_t>(128, (cap_tiles / ((mo + 127) / 128)) * 128);
        const DMat C = A.sub(jo, jo + bo + bn, mo, nr);
        const DMat W1 = SW1.sub(0, 0, bo, nr), W2 = SW2.sub(0, 0, bo, nr);
        for (int64_t c0 = 0; c0 < nr; c0 += cw1) {
          const int64_t w = std::min(cw1, nr - c0);
          gemm(ctx, Op::T, Op::N, 1.0, Vo, C.col_block(c0, w), 0.0, W1.col_block(c0, w), e0);
          gemm(ctx, Op::T, Op::N, 1.0, To, W1.col_block(c0, w), 0.0, W2.col_block(c0, w), e);
        }
        for (int64_t c0 = 0; c0 < nr; c0 += cw2) {
          const int64_t w = std::min(cw2, nr - c0);
          gemm(ctx, Op::N, Op::N, -1.0, Vo, W2.col_block(c0, w), 1.0, C.col_block(c0, w), e0);
        }
        QDWHG_CUDA(cudaEventRecord(ctx.ev_side, ctx.stream));
        ctx.stream = main_stream;
        side_pending = true;
      } else {
        side_pending = false;
      }
    }
  }
  if (side_pending) QDWHG_CUDA(cudaStreamWaitEvent(ctx.stream, ctx.ev_side, 0));
  if (use_hi) {
    QDWHG_CUDA(cudaEventRecord(ctx.ev_main, ctx.hi));
    QDWHG_CUDA(cudaStreamWaitEvent(caller, ctx.ev_main, 0));
    ctx.stream = caller;
  }
  ctx.panel_max_ctas = saved_cap;
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
    // (structured stacks: the block's reflectors act on rows < top_rows + j0 + b)
    const int64_t mp = (w.top_rows > 0 ? std::min<int64_t>(m, w.top_rows + j0 + b) : m) - j0;
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

void ormqr_left(Ctx& ctx, const QrWork& w, int64_t m, int64_t n, const DMat& C) {
  // C <- Q C with Q = H_0 ... H_{p-1} of geqrf (p = min(m-1, n)): blocks applied
  // last to first, C(j0:, :) -= V T (V^T C(j0:, :)) — ORGQR without the
  // identity start, so Q (m x n) never has to be formed when only Q M is needed
  const int64_t nc = C.cols;
  const int nb = w.nb;
  const int64_t npan = (n + nb - 1) / nb;
  const Arena::Mark mark = ctx.arena->mark();
  for (int64_t p = npan - 1; p >= 0; --p) {
    const int64_t j0 = p * nb;
    const int64_t b = std::min<int64_t>(nb, n - j0);
    const int64_t mp = (w.top_rows > 0 ? std::min<int64_t>(m, w.top_rows + j0 + b) : m) - j0;
    const DMat Vp = w.V.sub(j0, j0, mp, b);
    const DMat Tp = w.T.sub(0, p * nb, b, b);
    const DMat Cp = C.sub(j0, 0, mp, nc);
    DMat W1 = ctx.arena->alloc(b, nc);
    DMat W2 = ctx.arena->alloc(b, nc);
    gemm(ctx, Op::T, Op::N, 1.0, Vp, Cp, 0.0, W1);
    GemmExtra e;
    e.krange = KRange::AUpper;  // T upper
    gemm(ctx, Op::N, Op::N, 1.0, Tp, W1, 0.0, W2, e);
    gemm(ctx, Op::N, Op::N, -1.0, Vp, W2, 1.0, Cp);
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


// detect_deficiency_index (partial.cpp:32-38) on the device: the 1-based index of
// the first diagonal entry of R with |R_ii| < tol (reciprocal: R_ii = 1 / X_ii of
// the given X, e.g. X = W^{-1}), 0 when none.  One int comes back to the host
// instead of the whole diagonal.
__global__ void first_deficient_kernel(const double* R, int64_t ld, int64_t n, double tol, int reciprocal,
                                       unsigned long long* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = R[i + i * ld];
    const bool hit = reciprocal ? !(1.0 / fabs(d) >= tol) : (fabs(d) < tol);
    if (hit) atomicMin(out, (unsigned long long)(i + 1));
  }
}

int64_t first_deficient(Ctx& ctx, const DMat& R, double tol, bool reciprocal) {
  const int64_t n = std::min(R.rows, R.cols);
  auto* dv = static_cast<unsigned long long*>(ctx.arena->alloc_bytes(sizeof(unsigned long long)));
  auto* hv = reinterpret_cast<unsigned long long*>(ctx.hscratch);
  QDWHG_CUDA(cudaMemsetAsync(dv, 0xff, sizeof(unsigned long long), ctx.stream));
  first_deficient_kernel<<<std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148)), 256, 0, ctx.stream>>>(
      R.ptr(), R.ld, n, tol, reciprocal ? 1 : 0, dv);
  QDWHG_CUDA(cudaGetLastError());
  ctx.count();
  QDWHG_CUDA(cudaMemcpyAsync(hv, dv, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx.stream));
  QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
  return *hv == ~0ull ? 0 : (int64_t)*hv;
}

}  // namespace qdwhg
