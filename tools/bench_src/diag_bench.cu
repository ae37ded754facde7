// Microbenchmark of the POTRF leaf kernel (potrf_diag_kernel) with per-phase
// clock64 marks.  Build: make -C tools/bench_src diag_bench
#define QDWHG_DIAG_TRACE 1
// kernels compiled into this binary are registered with ITS runtime: their
// attributes must be set here, not through libqdwhg's (statically linked) one
#define func_attr bench_func_attr
#include "../../paper_2104_14186_b200/csrc/potrf.cu"
namespace qdwhg {
void bench_func_attr(const void* kern, cudaFuncAttribute attr, int value) {
  cudaFuncSetAttribute(kern, attr, value);
}
}  // namespace qdwhg

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

using namespace qdwhg;

__global__ void rsqrt_probe(const double* d, double* y, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = leaf::rsqrt_newton(d[i]);
}

static void check_rsqrt() {
  const int n = 1 << 20;
  std::vector<double> d(n), y(n);
  uint64_t st = 12345;
  for (int i = 0; i < n; ++i) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    const double u = (double)(st >> 11) / 9007199254740992.0;
    d[i] = std::ldexp(1.0 + u, (int)(st % 200) - 100);
  }
  double *dd, *dy;
  cudaMalloc(&dd, 8 * n);
  cudaMalloc(&dy, 8 * n);
  cudaMemcpy(dd, d.data(), 8 * n, cudaMemcpyHostToDevice);
  rsqrt_probe<<<n / 256, 256>>>(dd, dy, n);
  cudaMemcpy(y.data(), dy, 8 * n, cudaMemcpyDeviceToHost);
  double worst = 0;
  for (int i = 0; i < n; ++i) {
    const long double ref = 1.0L / sqrtl((long double)d[i]);
    worst = std::max(worst, (double)(fabsl((long double)y[i] - ref) / ref));
  }
  printf("rsqrt_newton max rel err %.3e (%.2f ulp)\n", worst, worst / 1.1102230246251565e-16);
  cudaFree(dd);
  cudaFree(dy);
}

int main() {
  check_rsqrt();
  const int nb = 128;
  const int64_t ld = 128;
  std::vector<double> h(ld * nb);
  // SPD: Z = I*nb + small symmetric
  // SPD like the QDWH step's Z = I + c X^T X (c = 17: kappa up to ~18 .. 100)
  {
    std::vector<double> x(ld * nb);
    uint64_t st = 777;
    for (auto& v : x) {
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      v = ((double)(st >> 11) / 9007199254740992.0 - 0.5) * 0.35;
    }
    for (int j = 0; j < nb; ++j)
      for (int i = 0; i < nb; ++i) {
        double s = 0;
        for (int k = 0; k < nb; ++k) s += x[k + i * ld] * x[k + j * ld];
        h[i + j * ld] = (i == j ? 1.0 : 0.0) + 17.0 * s;
      }
  }
  double *Z, *W, *Wi;
  int* flag;
  cudaMalloc(&Z, 8 * ld * nb);
  cudaMalloc(&W, 8 * ld * nb);
  cudaMalloc(&Wi, 8 * ld * nb);
  cudaMalloc(&flag, 4);
  cudaMemset(flag, 0, 4);
  cudaMemcpy(Z, h.data(), 8 * ld * nb, cudaMemcpyHostToDevice);
  Ctx ctx;
  ctx.dflag = flag;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 5; ++it) launch_diag(ctx, DMat{Z, ld, 0, 0, nb, nb}, DMat{W, ld, 0, 0, nb, nb}, DMat{Wi, ld, 0, 0, nb, nb});
  cudaEventRecord(e0);
  const int reps = 50;
  for (int it = 0; it < reps; ++it) launch_diag(ctx, DMat{Z, ld, 0, 0, nb, nb}, DMat{W, ld, 0, 0, nb, nb}, DMat{Wi, ld, 0, 0, nb, nb});
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("potrf_diag nb=%d: %.2f us/launch (%s)\n", nb, 1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  cudaEventRecord(e0);
  for (int it = 0; it < reps; ++it)
    launch_diag(ctx, DMat{Z, ld, 0, 0, nb, nb}, DMat{W, ld, 0, 0, nb, nb}, DMat{Wi, ld, 0, 0, nb, nb},
                kDiagNoW | kDiagUpperOnly);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("potrf_diag nb=%d (no W, upper only): %.2f us/launch\n", nb, 1e3 * ms / reps);
  // the fused, pipelined leaf (kDiagNoW path) against the classic one's W^{-1}
  {
    std::vector<double> wi0(ld * nb), wi1(ld * nb);
    cudaMemset(Wi, 0, 8 * ld * nb);
    launch_diag(ctx, DMat{Z, ld, 0, 0, nb, nb}, DMat{W, ld, 0, 0, nb, nb}, DMat{Wi, ld, 0, 0, nb, nb});
    cudaMemcpy(wi0.data(), Wi, 8 * ld * nb, cudaMemcpyDeviceToHost);
    cudaMemset(Wi, 0xff, 8 * ld * nb);
    launch_diag_fused(ctx, DMat{Z, ld, 0, 0, nb, nb}, DMat{Wi, ld, 0, 0, nb, nb}, 0);
    cudaMemcpy(wi1.data(), Wi, 8 * ld * nb, cudaMemcpyDeviceToHost);
    printf("fused launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    double d = 0, mx = 0;
    for (size_t i = 0; i < wi0.size(); ++i) {
      d = std::max(d, std::abs(wi0[i] - wi1[i]));
      mx = std::max(mx, std::abs(wi0[i]));
    }
    printf("fused vs classic W^-1: max abs diff %.3e (max |W^-1| %.3e)\n", d, mx);
    for (int it = 0; it < 5; ++it) launch_diag_fused(ctx, DMat{Z, ld, 0, 0, nb, nb}, DMat{Wi, ld, 0, 0, nb, nb}, kDiagUpperOnly);
    cudaEventRecord(e0);
    for (int it = 0; it < reps; ++it) launch_diag_fused(ctx, DMat{Z, ld, 0, 0, nb, nb}, DMat{Wi, ld, 0, 0, nb, nb}, kDiagUpperOnly);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("potrf_diag_fused nb=%d (upper only): %.2f us/launch (%s)\n", nb, 1e3 * ms / reps,
           cudaGetErrorString(cudaGetLastError()));
    cudaDeviceSynchronize();
    long long tf[64];
    cudaMemcpyFromSymbol(tf, g_diag_trace, sizeof(tf));
    printf("  fused: load %lld  factor+invert %lld  write %lld  total %lld cycles\n", tf[0] - tf[20],
           tf[15] - tf[0], tf[16] - tf[15], tf[16] - tf[20]);
    printf("  fused steps:");
    for (int i = 24; i < 40; ++i) printf(" %lld", tf[i] - tf[0]);
    printf("\n  helper end / panel end (warps 1, 2, 4, 7):");
    for (int i = 40; i < 64; ++i) printf(" %lld", tf[i] - tf[0]);
    printf("\n");
  }
  for (int it = 0; it < 2; ++it) launch_diag(ctx, DMat{Z, ld, 0, 0, nb, nb}, DMat{W, ld, 0, 0, nb, nb}, DMat{Wi, ld, 0, 0, nb, nb});
  cudaDeviceSynchronize();
  long long t[64];
  cudaMemcpyFromSymbol(t, g_diag_trace, sizeof(t));
  const char* names[21] = {"load", "kb0 chol+Dinv", "kb0 panel", "kb0 trail", "kb1 chol+Dinv", "kb1 panel",
                           "kb1 trail", "kb2 chol+Dinv", "kb2 panel", "kb2 trail", "kb3 chol+Dinv",
                           "kb3 panel", "kb3 trail", "W write", "D^-1 blocks", "L^-1 doubling", "Winv write",
                           "", "", "", "start"};
  long long prev = t[20];
  for (int i = 0; i <= 16; ++i) {
    if (i == 11 || i == 12) continue;  // no panel / trailing update in the last block
    printf("  %-16s %8lld cycles\n", names[i], t[i] - prev);
    prev = t[i];
  }
  printf("  total %lld cycles\n", t[16] - t[20]);
  printf("  inverse: level32 %lld level64 %lld\n", t[22] - t[14], t[23] - t[22]);
  // check: W^T W == Z
  std::vector<double> w(ld * nb), wi(ld * nb);
  cudaMemcpy(w.data(), W, 8 * ld * nb, cudaMemcpyDeviceToHost);
  cudaMemcpy(wi.data(), Wi, 8 * ld * nb, cudaMemcpyDeviceToHost);
  double e = 0, ei = 0;
  for (int j = 0; j < nb; ++j)
    for (int i = 0; i < nb; ++i) {
      double s = 0, si = 0;
      for (int k = 0; k < nb; ++k) {
        s += w[k + i * ld] * w[k + j * ld];
        si += w[i + k * ld] * wi[k + j * ld];
      }
      e = std::max(e, std::abs(s - h[i + j * ld]));
      ei = std::max(ei, std::abs(si - (i == j)));
    }
  printf("  max|W^T W - Z| %.3e  max|W Winv - I| %.3e\n", e, ei);
  return 0;
}
