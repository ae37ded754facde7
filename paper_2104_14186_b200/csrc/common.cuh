// Shared device primitives for the sm_100a FP64 kernels of libqdwhg.
//  - DMMA: mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4).  tcgen05 has
//    no kind::f64 (ptxas rejects it), so FP64 tensor work on B200 is DMMA fed
//    from shared memory; measured 37.1 TFLOP/s issue-bound (profiles/r01_fp64_peak_probe.txt).
//  - TMA (cp.async.bulk.tensor.2d) + mbarrier transaction pipelines.
//  - warp / block reductions in FP64.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define QDWHG_DEV __device__ __forceinline__

namespace qdwhg {

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------- DMMA
// D(8x8) += A(8x4, row) * B(4x8, col).  Lane l holds A[l>>2][l&3], B[l&3][l>>2],
// C[l>>2][2(l&3)+{0,1}].
QDWHG_DEV void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- smem addressing
QDWHG_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- cp.async
QDWHG_DEV void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
QDWHG_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---------------------------------------------------------------- mbarrier
QDWHG_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
QDWHG_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
QDWHG_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

QDWHG_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
QDWHG_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
QDWHG_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Cluster-scope acquire wait (data delivered by peers' st.async).
QDWHG_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- DSMEM
// Address of the same shared-memory location in CTA `rank` of the cluster.
QDWHG_DEV uint32_t mapa_u32(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
// 16-byte asynchronous store into a peer CTA's shared memory that completes
// 16 transaction bytes on the peer's mbarrier (no cluster barrier needed).
QDWHG_DEV void st_async_v2(uint32_t remote_addr, double x, double y, uint32_t remote_mbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
          remote_addr),
      "d"(x), "d"(y), "r"(remote_mbar)
      : "memory");
}

// ---------------------------------------------------------------- TMA
QDWHG_DEV void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}
// 2D tiled load: box at element coordinates (c0 = contiguous dim, c1 = outer dim).
QDWHG_DEV void tma_load_2d(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// ---------------------------------------------------------------- programmatic dependent launch
// A kernel launched with cudaLaunchAttributeProgrammaticStreamSerialization may
// start while its predecessor finishes; it must call griddep_wait() before its
// first global-memory access.  griddep_launch_dependents() lets the next such
// kernel start its prologue.
QDWHG_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
QDWHG_DEV void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// ---------------------------------------------------------------- grid barrier
QDWHG_DEV unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
QDWHG_DEV void red_release_add_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Monotonic grid barrier for cooperative launches (counter zeroed before the
// launch, all CTAs co-resident).  bar.sync orders the CTA's prior writes before
// thread 0's gpu-scope release (cumulativity); the acquire poll orders what follows.
QDWHG_DEV void grid_sync(unsigned* bar, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) {
    red_release_add_gpu(bar, 1u);
    const unsigned target = epoch * gridDim.x;
    while (ld_acquire_gpu(bar) < target) {
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- reductions
// Latency-lean reciprocal / square root for scalar critical paths (panel
// pivots): hardware f64 estimates + Newton steps, ~1 ulp (not correctly rounded,
// no library slow path).  x must be finite and nonzero (sqrt: positive).
QDWHG_DEV double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;\n" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
// 1/sqrt(x) to ~1 ulp: hardware estimate + two Newton steps (x > 0, finite)
QDWHG_DEV double fast_rsqrt(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(x));
  const double h = 0.5 * x;
  r = r * fma(-h * r, r, 1.5);
  return r * fma(-h * r, r, 1.5);
}
QDWHG_DEV double fast_sqrt(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(x));
  const double h = 0.5 * x;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  const double s = x * r;
  return fma(0.5 * r, fma(-s, s, x), s);  // one residual correction
}

QDWHG_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
QDWHG_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// Block-wide sum; every thread gets the result.  scratch >= 32 doubles.
QDWHG_DEV double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = (lane < nw) ? scratch[lane] : 0.0;
  t = warp_sum(t);
  return t;
}
QDWHG_DEV double block_max(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = (lane < nw) ? scratch[lane] : 0.0;
  t = warp_max(t);
  return t;
}

}  // namespace qdwhg
