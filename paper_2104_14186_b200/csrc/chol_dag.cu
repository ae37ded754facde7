// Tile-DAG Cholesky for the QDWH Cholesky step (polar.cpp:82-128; reference
// kernel kernels.cpp:124-146): one persistent kernel instead of the recursive
// chain of ~190 launches per factorisation.
//
// Z (n x n, lower triangle read, n = 128 T) is factored Z = L L^T by the
// right-looking tile algorithm on 128 x 128 tiles:
//   LEAF(k)       L_kk = chol(Z_kk) and L_kk^{-1} (one CTA, shared memory:
//                 potrf_leaf.cuh), W^{-1}_kk = L_kk^{-T} -> Winv, L_kk^{-1} -> Z_kk
//   PANEL(i, k)   L_ik = Z_ik L_kk^{-T}                      (i > k, in place)
//   UPDATE(i,j,k) Z_ij -= L_ik L_jk^T                         (k < j <= i)
// Tasks run from a queue in a topological order (sorted by their earliest
// start in the infinite-machine schedule), each CTA of a persistent grid taking
// the next index with one atomic, waiting on per-tile completion counters
// (acquire / release at gpu scope), and running the task.  Because every task
// only waits on tasks taken earlier, no co-residency is needed and there is no
// deadlock; the queue order gives the look-ahead: while one CTA factors the
// latency-bound diagonal tile, the others run the trailing updates of earlier
// steps.  The critical tasks (all PANELs and the updates of the next tile
// column) are split into 32-row strips so the chain between two leaves crosses
// the machine in a few microseconds.
//
// Afterwards W^{-1} is assembled from the diagonal-tile inverses and the
// off-diagonal L blocks by the level-batched TRTRI (potrf.cu: two GEMM launches
// per level, log2(T) levels).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <queue>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "potrf_leaf.cuh"

namespace qdwhg {

namespace {

constexpr int kTile = 128;
constexpr int kKC = 32;              // K chunk of the tile GEMM pipeline
constexpr int kLDB = kTile + 4;      // smem ld of the B chunk (132 = 4 mod 16: conflict-free fragments)
enum : int { kLeafTask = 0, kPanelTask = 1, kUpdateTask = 2, kAccTask = 3, kFinTask = 4 };

struct DagTask {
  int type, i, j, k;
  int r0, nr;         // row strip of the output tile
  int nk;             // 128-column K steps (1, or 2: steps k and k + 1 in one task)
  int slot;           // completion counter this task increments
  int dep[3];         // tile indices (i * T + j) this task waits on, -1 = none
  unsigned cnt[3];    // ... until their completion counters reach these values
};

struct DagParams {
  double* Z;
  int64_t ldz;
  double* Winv;
  int64_t ldw;
  int T;
  const DagTask* tasks;
  int ntasks;      // queue length (tasks[ntasks + k] = LEAF(k), run by CTA 0)
  unsigned* done;  // T*T completion counters (zero on entry, reset on exit)
  unsigned* ctrl;  // [0] queue head, [1] CTAs exited
  int* flag;       // set on a non-positive pivot
  int fused_leaf;  // pipelined factor-and-invert leaf (QDWHG_LEAF_NO_FUSED unset)
  unsigned long long* trace;  // QDWHG_DAG_TRACE: per task {grab, ready, end, smid} (ns), clocks at ready/end
  unsigned long long* ltrace; // ... and per leaf {loaded, factored, inverted, written}
};

QDWHG_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
QDWHG_DEV unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

QDWHG_DEV void cp_async16_cg(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
QDWHG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
QDWHG_DEV void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// C(R x 128) = C0 -/+ A(R x 128) * Bt(128 x 128)^T with C0 = C (kSub, kAdd) or
// 0 (kSet, kNeg), all column-major with leading dimension ld in global memory (L2:
// the tiles were written by other SMs, so every read bypasses L1).  K streams in
// 32-column chunks through a STAGES-deep cp.async ring (the 32-row strips load
// all four chunks at once: their time is latency); C is read into the
// accumulators while the first chunks are in flight; DMMA m8n8k4 on
// shared-memory fragments (the subtraction is the DMMA's negated A operand).
enum : int { kSet = 0, kSub = 1, kAdd = 2, kNeg = 3 };  // C = [C0] +/- A Bt^T
// (mode is a runtime argument: one instance per strip height keeps the kernel's
// code small — the leaf runs from a warm instruction cache)
template <int R>
QDWHG_DEV void tile_gemm(double* sm, int mode, double* C, int64_t ldc, const double* A, int64_t lda,
                         const double* Bt, int64_t ldb, int nk = 1) {
  // K = 128 nk: step s reads the 128 columns of A and Bt that follow step s - 1
  // C0 - A Bt^T = -(-C0 + A Bt^T): the sign goes on the accumulators' first load
  // and last store, none in the DMMA loop
  const bool loadc = mode == kSub || mode == kAdd;
  const double sgn = (mode == kSub || mode == kNeg) ? -1.0 : 1.0;
  constexpr int LDA = R + 4;
  constexpr int STAGES = (R == 128) ? 3 : 4;
  constexpr int WR = (R == 128) ? 2 : 1;  // warps along the rows
  constexpr int WC = 8 / WR;
  constexpr int MR = R / WR / 8;          // 8-row fragments per warp
  constexpr int NC = kTile / WC / 8;      // 8-column fragments per warp
  constexpr int STAGE = kKC * (LDA + kLDB);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int row0 = (warp % WR) * (R / WR), col0 = (warp / WR) * (kTile / WC);

  auto load_chunk = [&](int ch) {
    // A: 32 columns x R rows (R/2 16-byte pieces per column); Bt: 32 columns x 128 rows
    double* as = sm + (ch % STAGES) * STAGE;
    double* bs = as + kKC * LDA;
    constexpr int AP = kKC * (R / 2), BP = kKC * (kTile / 2);
    const int cs = ch & 3;  // chunk within its 128-column step
    const double* Ap = A + (int64_t)(ch >> 2) * kTile * lda;
    const double* Bp = Bt + (int64_t)(ch >> 2) * kTile * ldb;
#pragma unroll 4
    for (int idx = tid; idx < AP + BP; idx += leaf::kThreads) {
      if (idx < AP) {
        const int c = idx / (R / 2), r2 = idx % (R / 2);
        cp_async16_cg(as + c * LDA + 2 * r2, Ap + 2 * r2 + (int64_t)(cs * kKC + c) * lda);
      } else {
        const int b = idx - AP;
        const int c = b / (kTile / 2), r2 = b % (kTile / 2);
        cp_async16_cg(bs + c * kLDB + 2 * r2, Bp + 2 * r2 + (int64_t)(cs * kKC + c) * ldb);
      }
    }
  };

  const int NCH = 4 * nk;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < NCH) load_chunk(s);
    cp_async_commit();
  }
  double acc[MR][NC][2];
#pragma unroll
  for (int m = 0; m < MR; ++m)
#pragma unroll
    for (int n = 0; n < NC; ++n) {
      if (loadc) {
        const double* p0 = C + row0 + 8 * m + g + (int64_t)(col0 + 8 * n + 2 * q) * ldc;
        acc[m][n][0] = sgn * __ldcg(p0);
        acc[m][n][1] = sgn * __ldcg(p0 + ldc);
      } else {
        acc[m][n][0] = acc[m][n][1] = 0.0;
      }
    }
#pragma unroll 1
  for (int ch = 0; ch < NCH; ++ch) {
    if (ch + STAGES - 1 < NCH) load_chunk(ch + STAGES - 1);
    cp_async_commit();
    cp_async_wait_group<STAGES - 1>();
    __syncthreads();
    const double* as = sm + (ch % STAGES) * STAGE;
    const double* bs = as + kKC * LDA;
#pragma unroll
    for (int k4 = 0; k4 < kKC / 4; ++k4) {
      double a[MR], b[NC];
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        a[m] = as[(4 * k4 + q) * LDA + row0 + 8 * m + g];
      }
#pragma unroll
      for (int n = 0; n < NC; ++n) b[n] = bs[(4 * k4 + q) * kLDB + col0 + 8 * n + g];
#pragma unroll
      for (int m = 0; m < MR; ++m)
#pragma unroll
        for (int n = 0; n < NC; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], a[m], b[n]);
    }
    if (ch + STAGES < NCH) __syncthreads();  // this stage is refilled by the next iteration
  }
#pragma unroll
  for (int m = 0; m < MR; ++m)
#pragma unroll
    for (int n = 0; n < NC; ++n) {
      double* p0 = C + row0 + 8 * m + g + (int64_t)(col0 + 8 * n + 2 * q) * ldc;
      p0[0] = sgn * acc[m][n][0];
      p0[ldc] = sgn * acc[m][n][1];
    }
}
constexpr int kGemmSmemDoubles = 3 * kKC * (2 * kTile + 8);  // the 128-row ring (> the strips' 4 stages)
constexpr int kDagSmemDoubles =
    (kGemmSmemDoubles > leaf::kSmemDoubles) ? kGemmSmemDoubles : leaf::kSmemDoubles;
static_assert(kDagSmemDoubles >= leaf::kFusedSmemDoubles, "fused leaf scratch");

// LEAF(k): factor and invert the (fully updated) diagonal tile.
QDWHG_DEV void leaf_task(double* sm, const DagParams& p, int k, int* bad_s) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* A = sm;
  double* Tm = A + 128 * leaf::kLDA;
  double* Sinv = Tm + 64 * leaf::kLDT;
  double* Zkk = p.Z + (int64_t)k * kTile * (p.ldz + 1);
  for (int idx = tid; idx < kTile * (kTile / 2); idx += leaf::kThreads) {
    const int c = idx / (kTile / 2), r2 = idx % (kTile / 2);
    cp_async16_cg(A + c * leaf::kLDA + 2 * r2, Zkk + 2 * r2 + (int64_t)c * p.ldz);
  }
  cp_async_commit();
  cp_async_wait_group<0>();
  __syncthreads();
  // the strict upper of a diagonal tile is workspace garbage: zero it
  for (int idx = tid; idx < kTile * kTile; idx += leaf::kThreads) {
    const int c = idx / kTile, r = idx % kTile;
    if (r < c) A[c * leaf::kLDA + r] = 0.0;
  }
  __syncthreads();
  if (p.ltrace && tid == 0) p.ltrace[4 * k] = globaltimer();
  if (p.fused_leaf) {
    leaf::factor_invert_fused(A, Tm, bad_s);  // Tm: the 192 x kLDS scratch
    if (p.ltrace && tid == 0) p.ltrace[4 * k + 1] = globaltimer();
  } else {
    leaf::factor(A, Sinv, kTile, bad_s);
    if (p.ltrace && tid == 0) p.ltrace[4 * k + 1] = globaltimer();
    leaf::invert(A, Tm, Sinv, kTile);
  }
  if (p.ltrace && tid == 0) p.ltrace[4 * k + 2] = globaltimer();
  // L_kk^{-1} (lower, zeros above) over Z_kk: the PANEL / FIN tasks' B operand.
  // Released first (the leaf chain continues through PANEL(k+1, k)); the tile's
  // counter is released a second time by the caller once Winv_kk is out (ACC tasks)
  for (int idx = tid; idx < kTile * kTile; idx += leaf::kThreads) {
    const int c = idx / kTile, r = idx % kTile;
    Zkk[r + (int64_t)c * p.ldz] = (r >= c) ? A[c * leaf::kLDA + r] : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    red_release_add_gpu(&p.done[k * p.T + k], 1u);
  }
  // Winv_kk = L^{-T} (upper; the strict lower of Winv is pre-zeroed), transposed
  // shared reads with 8 lanes per column (conflict-free for kLDA = 132)
  {
    double* Wkk = p.Winv + (int64_t)k * kTile * (p.ldw + 1);
    const int j = lane >> 3, rr = lane & 7;
    for (int c0 = 4 * warp; c0 < kTile; c0 += 4 * (leaf::kThreads / 32)) {
      const int c = c0 + j;
      double* wc = Wkk + (int64_t)c * p.ldw;
      for (int r = rr; r < c0 + 4; r += 8)
        if (r <= c) wc[r] = A[r * leaf::kLDA + c];
    }
  }
  if (p.ltrace) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      p.ltrace[4 * k + 3] = globaltimer();
    }
  }
}

__global__ void __launch_bounds__(leaf::kThreads, 1) chol_dag_kernel(const DagParams p) {
  extern __shared__ double sm[];
  __shared__ int s_task, s_last, bad_s;
  const int tid = threadIdx.x;
  if (tid == 0) bad_s = 0;
  griddep_wait();
  if (blockIdx.x == 0) {
    // CTA 0 factors the diagonal tiles, in order (its instruction cache stays
    // warm with the leaf code; the queue CTAs never wait for a free SM to run one)
    for (int k = 0; k < p.T; ++k) {
      const int t = p.ntasks + k;
      const DagTask tk = p.tasks[t];
      if (tid == 0) {
        const unsigned long long tg = p.trace ? globaltimer() : 0ull;
        if (tk.dep[0] >= 0)
          while (ld_acquire_gpu(&p.done[tk.dep[0]]) < tk.cnt[0]) __nanosleep(20);
        __threadfence();
        if (p.trace) {
          p.trace[6 * t] = tg;
          p.trace[6 * t + 1] = globaltimer();
          p.trace[6 * t + 4] = clock64();
        }
      }
      __syncthreads();
      leaf_task(sm, p, k, &bad_s);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        red_release_add_gpu(&p.done[tk.slot], 1u);
        if (p.trace) {
          p.trace[6 * t + 2] = globaltimer();
          p.trace[6 * t + 5] = clock64();
          p.trace[6 * t + 3] = smid();
        }
      }
    }
  } else {
    for (;;) {
      if (tid == 0) s_task = (int)atomicAdd(&p.ctrl[0], 1u);
      __syncthreads();
      const int t = s_task < p.ntasks ? s_task : -1;
      if (t < 0) break;
      const DagTask tk = p.tasks[t];
      if (tid == 0) {
        const unsigned long long tg = p.trace ? globaltimer() : 0ull;
#pragma unroll
        for (int d = 0; d < 3; ++d)
          if (tk.dep[d] >= 0)
            while (ld_acquire_gpu(&p.done[tk.dep[d]]) < tk.cnt[d]) __nanosleep(32);
        __threadfence();
        if (p.trace) {
          p.trace[6 * t] = tg;
          p.trace[6 * t + 1] = globaltimer();
          p.trace[6 * t + 4] = clock64();
        }
      }
      __syncthreads();
      const int64_t ld = p.ldz;
      {
        // one call site per strip height (the kernel's code stays small: the leaf
        // CTA keeps its instructions cached); tiles (a, b) of Z / Winv, row strip r0
        auto zt = [&](int a, int b, int r0) { return p.Z + (int64_t)a * kTile + r0 + (int64_t)b * kTile * ld; };
        auto wt = [&](int a, int b, int r0) {
          return p.Winv + (int64_t)a * kTile + r0 + (int64_t)b * kTile * p.ldw;
        };
        int mode;
        double* C;
        const double *A, *Bt;
        int64_t ldc = ld, lda = ld;
        switch (tk.type) {
          case kPanelTask:  // L_ik = Z_ik L_kk^{-T}  (A aliases C row by row: read before written)
            mode = kSet;
            C = zt(tk.i, tk.k, tk.r0);
            A = C;
            Bt = zt(tk.k, tk.k, 0);
            break;
          case kUpdateTask:  // Z_ij -= sum_{s < nk} L_i,k+s L_j,k+s^T
            mode = kSub;
            C = zt(tk.i, tk.j, tk.r0);
            A = zt(tk.i, tk.k, tk.r0);
            Bt = zt(tk.j, tk.k, 0);
            break;
          case kAccTask:  // S_ij^T (+)= sum_{s < nk} X_k+s,j^T L_i,k+s^T  (X = L^{-1}, X_kj^T = Winv tile (j, k)), S^T in Z tile (j, i)
            mode = tk.k == tk.j ? kSet : kAdd;
            C = zt(tk.j, tk.i, tk.r0);
            A = wt(tk.j, tk.k, tk.r0);
            lda = p.ldw;
            Bt = zt(tk.i, tk.k, 0);
            break;
          default:  // kFinTask: Winv_ji = X_ij^T = -S_ij^T L_ii^{-T}
            mode = kNeg;
            C = wt(tk.j, tk.i, tk.r0);
            ldc = p.ldw;
            A = zt(tk.j, tk.i, tk.r0);
            Bt = zt(tk.i, tk.i, 0);
            break;
        }
        if (tk.nr == 16)
          tile_gemm<16>(sm, mode, C, ldc, A, lda, Bt, ld);
        else if (tk.nr == 32)
          tile_gemm<32>(sm, mode, C, ldc, A, lda, Bt, ld);
        else
          tile_gemm<128>(sm, mode, C, ldc, A, lda, Bt, ld, tk.nk);
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        red_release_add_gpu(&p.done[tk.slot], 1u);
        if (p.trace) {
          p.trace[6 * t + 2] = globaltimer();
          p.trace[6 * t + 5] = clock64();
          p.trace[6 * t + 3] = smid();
        }
      }
    }
  }
  if (tid == 0 && bad_s) atomicExch(p.flag, 1);
  // the last CTA out resets the counters for the next launch (every task is
  // complete: a CTA leaves only after its last task and an empty queue)
  if (tid == 0) {
    __threadfence();
    s_last = (atomicAdd(&p.ctrl[1], 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    for (int idx = tid; idx < p.T * p.T; idx += leaf::kThreads) p.done[idx] = 0u;
    if (tid == 0) p.ctrl[0] = p.ctrl[1] = 0u;
  }
}

// Task list of a T x T tile grid in queue order.  The order is the start order
// of a list schedule of the DAG on P processors (the CTAs) with measured task
// durations, highest bottom level (longest path to the end) first among the
// ready tasks — so a leaf enters the queue as soon as it can run, ahead of the
// trailing updates that only fill the machine.  Start times respect every
// dependency, so the order is topological (required: a CTA blocks on the tasks
// taken before its own).
std::vector<DagTask> build_tasks(int T, int P, int* nqueue) {
  const double kLeafUs = 34.0, kChainUs = 6.0, kStripUs = 8.6, kTileUs = 24.0;
  std::vector<DagTask> tasks;
  std::vector<double> dur;
  std::vector<std::vector<int>> succ;
  std::vector<int> indeg;
  std::vector<unsigned> cnt((size_t)T * T, 0u);
  std::vector<std::vector<int>> last((size_t)T * T);  // task ids of the tile's latest step
  auto tile = [T](int i, int j) { return i * T + j; };
  int nk = 1;  // K steps of the next task added (bulk groups: steps k .. k + nk - 1)
  // measured with the fused leaf (n = 4096 / 2048 / 1024 DAG, us): 1 step 2640 / 754 /
  // 361, 2: 2406 / 800 / 384, 3: 2340 / 881 / 416, 4: 2333 / 955 / 455, 6: 2412 /
  // 1123 / 510 — longer tasks pay where the trailing work is large, short ones
  // where the leaf chain dominates
  static const int group_env = getenv("QDWHG_DAG_GROUP") ? atoi(getenv("QDWHG_DAG_GROUP")) : 0;
  const int kGroup = group_env > 0 ? group_env : (T >= 24) ? 3 : (T >= 20) ? 2 : 1;
  auto addx = [&](int type, int i, int j, int k, int nstrips, const int (&dt)[3], double d, int slot) {
    DagTask base{};
    base.type = type;
    base.i = i;
    base.j = j;
    base.k = k;
    std::vector<int> preds;
    for (int x = 0; x < 3; ++x) {
      base.dep[x] = -1;
      base.cnt[x] = 0;
      if (dt[x] >= 0 && cnt[dt[x]] > 0) {
        base.dep[x] = dt[x];
        base.cnt[x] = cnt[dt[x]];
        preds.insert(preds.end(), last[dt[x]].begin(), last[dt[x]].end());
      }
    }
    const int t = slot;
    std::vector<int> ids;
    for (int s = 0; s < nstrips; ++s) {
      DagTask x = base;
      x.slot = slot;
      x.nk = nk;
      x.nr = kTile / nstrips;
      x.r0 = s * x.nr;
      const int id = (int)tasks.size();
      tasks.push_back(x);
      dur.push_back(d);
      succ.emplace_back();
      indeg.push_back((int)preds.size());
      for (int pr : preds) succ[pr].push_back(id);
      ids.push_back(id);
    }
    cnt[t] += nstrips;
    last[t] = ids;
  };
  auto add = [&](int type, int i, int j, int k, int nstrips, const int (&dt)[3], double d) {
    addx(type, i, j, k, nstrips, dt, d, tile(i, j));
  };
  for (int k = 0; k < T; ++k) {
    {
      const int dt[3] = {tile(k, k), -1, -1};
      add(kLeafTask, k, k, k, 1, dt, kLeafUs);
      // the leaf releases its tile twice: L_kk^{-1} (in Z_kk) first, Winv_kk second
      cnt[tile(k, k)] += 1;
    }
    // tasks that read only L_kk^{-1} (dependency 1 = tile (k, k)) wait for the first release
    auto first_release_only = [&](int nstrips) {
      for (int s = 1; s <= nstrips; ++s) tasks[tasks.size() - s].cnt[1] -= 1;
    };
    for (int i = k + 1; i < T; ++i) {
      const int dt[3] = {tile(i, k), tile(k, k), -1};
      // the leaf chain LEAF(k) -> PANEL(k+1, k) -> UPDATE(k+1, k+1, k) -> LEAF(k+1)
      // crosses the machine in 16-row strips, the rest of the next column in 32
      add(kPanelTask, i, k, k, i == k + 1 ? 8 : 4, dt, i == k + 1 ? kChainUs : kStripUs);
      first_release_only(i == k + 1 ? 8 : 4);
    }
    for (int j = k + 1; j < T; ++j)
      for (int i = j; i < T; ++i) {
        const bool c = (j == k + 1);  // the next tile column: on the leaf chain
        const bool chain = c && i == j;
        if (!c) {
          // bulk updates of a tile in groups of kGroup steps (K = 128 kGroup: fewer
          // tasks, less C traffic), aligned at multiples of kGroup and cut at the
          // tile's last bulk step j - 2; emitted at the group's last step
          const int gs = (k / kGroup) * kGroup, ge = std::min(gs + kGroup - 1, j - 2);
          if (k != ge) continue;
          if (ge > gs) {
            // tile (i, j) through gs - 1, panels (i, ge), (j, ge) (which imply the earlier ones)
            const int dt[3] = {tile(i, j), tile(i, ge), i == j ? -1 : tile(j, ge)};
            nk = ge - gs + 1;
            add(kUpdateTask, i, j, gs, 1, dt, nk * (kTileUs - 4.0) + 4.0);
            nk = 1;
            continue;
          }
        }
        const int dt[3] = {tile(i, j), tile(i, k), i == j ? -1 : tile(j, k)};
        add(kUpdateTask, i, j, k, chain ? 8 : c ? 4 : 1, dt, chain ? kChainUs : c ? kStripUs : kTileUs);
      }
    // row k of X = L^{-1} (W^{-1} = X^T): X_kj = -L_kk^{-1} sum_{m=j}^{k-1} L_km X_mj,
    // accumulated (S_kj^T in Z's unused upper tile (j, k)) as soon as X_mj and
    // L_km exist; slot counters use the upper index (j, k)
    for (int j = 0; j < k; ++j) {
      // accumulations in groups of kGroup m (K = 128 kGroup), the last one
      // (m = k - 1, the one FIN(k, j) waits for) alone
      for (int m = j; m < k;) {
        const int m2 = (m == k - 1) ? m : std::min(m + kGroup - 1, k - 2);  // last step of this task
        const int dt[3] = {tile(j, k), tile(j, m2), tile(k, m2)};  // S, X_m2,j (leaf / FIN), L_k,m2
        nk = m2 - m + 1;
        addx(kAccTask, k, j, m, 1, dt, nk * (kTileUs - 4.0) + 4.0, tile(j, k));
        nk = 1;
        m = m2 + 1;
      }
      const int dt[3] = {tile(j, k), tile(k, k), -1};  // all of S, L_kk^{-1}
      addx(kFinTask, k, j, k, 4, dt, kStripUs, tile(j, k));
      first_release_only(4);
    }
  }
  const int N = (int)tasks.size();
  // bottom levels (generation order is topological: successors have larger ids)
  std::vector<double> bl(N, 0.0);
  for (int t = N - 1; t >= 0; --t) {
    double m = 0.0;
    for (int s : succ[t]) m = std::max(m, bl[s]);
    bl[t] = dur[t] + m;
  }
  // list schedule: leaves on their own processor (CTA 0) as soon as ready, the
  // rest on P - 1
  using RItem = std::pair<double, int>;  // (-bottom level, id)
  std::priority_queue<RItem, std::vector<RItem>, std::greater<RItem>> ready;
  using EItem = std::pair<double, int>;  // (finish time, id)
  std::priority_queue<EItem, std::vector<EItem>, std::greater<EItem>> running;
  std::vector<double> start(N, 0.0);
  double now = 0.0;
  int free_p = P - 1, scheduled = 0;
  auto release = [&](int t) {
    if (tasks[t].type == kLeafTask) {  // the leaf processor is idle whenever a leaf is ready
      start[t] = now;
      running.push({now + dur[t], t});
      ++scheduled;
    } else {
      ready.push({-bl[t], t});
    }
  };
  for (int t = 0; t < N; ++t)
    if (indeg[t] == 0) release(t);
  while (scheduled < N) {
    while (free_p > 0 && !ready.empty()) {
      const int t = ready.top().second;
      ready.pop();
      start[t] = now;
      running.push({now + dur[t], t});
      --free_p;
      ++scheduled;
    }
    // advance to the next completion (and everything finishing at that time)
    const double tn = running.top().first;
    now = tn;
    while (!running.empty() && running.top().first <= tn) {
      const int t = running.top().second;
      running.pop();
      if (tasks[t].type != kLeafTask) ++free_p;
      for (int s : succ[t])
        if (--indeg[s] == 0) release(s);
    }
  }
  // queue = non-leaf tasks by start time (topological: a start follows every
  // dependency's finish); the leaves follow, in order
  std::vector<int> ord;
  for (int x = 0; x < N; ++x)
    if (tasks[x].type != kLeafTask) ord.push_back(x);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return start[a] < start[b]; });
  *nqueue = (int)ord.size();
  for (int x = 0; x < N; ++x)
    if (tasks[x].type == kLeafTask) ord.push_back(x);
  std::vector<DagTask> out(N);
  for (int x = 0; x < N; ++x) out[x] = tasks[ord[x]];
  return out;
}

}  // namespace

// Per-handle DAG state: one task list per tile count (built and uploaded once),
// one set of completion counters sized for the largest grid seen.
struct DagCache {
  struct Entry {
    DagTask* d_tasks = nullptr;
    int ntasks = 0, nqueue = 0;  // tasks[0, nqueue): queue; then the T leaves
    std::vector<DagTask> h_tasks;
    unsigned long long* d_trace = nullptr;   // QDWHG_DAG_TRACE only
    unsigned long long* d_ltrace = nullptr;
  };
  std::map<int, Entry> entries;
  unsigned* d_done = nullptr;  // tmax^2 counters + 2 control words
  int tmax = 0;
  ~DagCache() {
    for (auto& kv : entries) {
      cudaFree(kv.second.d_tasks);
      cudaFree(kv.second.d_trace);
      cudaFree(kv.second.d_ltrace);
    }
    cudaFree(d_done);
  }
};

bool chol_dag_applicable(int64_t n) {
  static const bool off = getenv("QDWHG_CHOL_NO_DAG") != nullptr;
  static const int tmax_env = getenv("QDWHG_CHOL_DAG_TMAX") ? atoi(getenv("QDWHG_CHOL_DAG_TMAX")) : 32;
  return !off && n % kTile == 0 && n / kTile >= 2 && n / kTile <= tmax_env;
}

void chol_dag(Ctx& ctx, const DMat& Z, const DMat& Winv) {
  const int64_t n = Z.rows;
  const int T = (int)(n / kTile);
  if (!ctx.dag) ctx.dag = std::make_shared<DagCache>();
  DagCache& dc = *ctx.dag;
  auto it = dc.entries.find(T);
  if (it == dc.entries.end()) {
    // task list per tile count (a synchronous upload, once per size per handle)
    DagCache::Entry e;
    e.h_tasks = build_tasks(T, ctx.num_sms, &e.nqueue);
    e.ntasks = (int)e.h_tasks.size();
    QDWHG_CUDA(cudaMalloc(&e.d_tasks, e.h_tasks.size() * sizeof(DagTask)));
    QDWHG_CUDA(cudaMemcpy(e.d_tasks, e.h_tasks.data(), e.h_tasks.size() * sizeof(DagTask),
                          cudaMemcpyHostToDevice));
    it = dc.entries.emplace(T, std::move(e)).first;
  }
  DagCache::Entry& c = it->second;
  if (dc.tmax < T) {
    if (dc.d_done) {
      QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
      QDWHG_CUDA(cudaFree(dc.d_done));
    }
    dc.d_done = nullptr;
    QDWHG_CUDA(cudaMalloc(&dc.d_done, ((size_t)T * T + 2) * sizeof(unsigned)));
    QDWHG_CUDA(cudaMemset(dc.d_done, 0, ((size_t)T * T + 2) * sizeof(unsigned)));
    dc.tmax = T;
  }
  DagParams p;
  p.Z = Z.ptr();
  p.ldz = Z.ld;
  p.Winv = Winv.ptr();
  p.ldw = Winv.ld;
  p.T = T;
  p.tasks = c.d_tasks;
  p.ntasks = c.nqueue;
  p.done = dc.d_done;
  p.ctrl = dc.d_done + (size_t)dc.tmax * dc.tmax;
  p.flag = ctx.dflag;
  static const bool no_fused = getenv("QDWHG_LEAF_NO_FUSED") != nullptr;
  p.fused_leaf = no_fused ? 0 : 1;
  static const char* trace_path = getenv("QDWHG_DAG_TRACE");
  p.trace = p.ltrace = nullptr;
  if (trace_path) {
    if (!c.d_trace) QDWHG_CUDA(cudaMalloc(&c.d_trace, (size_t)c.ntasks * 6 * sizeof(unsigned long long)));
    if (!c.d_ltrace) QDWHG_CUDA(cudaMalloc(&c.d_ltrace, (size_t)T * 4 * sizeof(unsigned long long)));
    p.trace = c.d_trace;
    p.ltrace = c.d_ltrace;
  }
  const size_t smem = (size_t)kDagSmemDoubles * 8;
  func_attr(chol_dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = std::min(ctx.num_sms, c.nqueue + 1);
  // (profiling: events around the launch break its PDL overlap, as for the GEMMs)
  if (ctx.profile) ctx.prof_begin(2.0 / 3.0 * (double)n * n * n, "chol_dag n=" + std::to_string(n), 1);
  launch_pdl(ctx, chol_dag_kernel, dim3(grid), dim3(leaf::kThreads), smem, p);
  if (ctx.profile) ctx.prof_end();
  ctx.count();
  if (trace_path) {
    // debug: append {type,i,j,k,r0,nr, grab,ready,end,smid} rows of this launch
    std::vector<unsigned long long> tr((size_t)c.ntasks * 6), lt((size_t)T * 4);
    QDWHG_CUDA(cudaStreamSynchronize(ctx.stream));
    QDWHG_CUDA(cudaMemcpy(tr.data(), c.d_trace, tr.size() * 8, cudaMemcpyDeviceToHost));
    QDWHG_CUDA(cudaMemcpy(lt.data(), c.d_ltrace, lt.size() * 8, cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(trace_path, "a")) {
      fprintf(f, "# launch T=%d ntasks=%d grid=%d\n", T, c.ntasks, grid);
      for (int t = 0; t < c.ntasks; ++t) {
        const DagTask& x = c.h_tasks[t];
        fprintf(f, "%d %d %d %d %d %d %llu %llu %llu %llu %llu\n", x.type, x.i, x.j, x.k, x.r0, x.nr, tr[6 * t],
                tr[6 * t + 1], tr[6 * t + 2], tr[6 * t + 3], tr[6 * t + 5] - tr[6 * t + 4]);
      }
      for (int k = 0; k < T; ++k)
        fprintf(f, "L %d %llu %llu %llu %llu\n", k, lt[4 * k], lt[4 * k + 1], lt[4 * k + 2], lt[4 * k + 3]);
      fclose(f);
    }
  }
}

}  // namespace qdwhg
