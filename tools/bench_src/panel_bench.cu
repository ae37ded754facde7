// Microbenchmark of the GEQRF panel kernel (geqr2_panel_kernel, cluster and
// grid variants) with per-phase clock marks for column 10 of CTA 0.
// Build: make -C tools/bench_src panel_bench
#ifndef NO_TRACE
#define QDWHG_PANEL_TRACE 1
#endif
#include "../../paper_2104_14186_b200/csrc/geqrf.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace qdwhg;

int main() {
  for (int mp : {1024, 2048, 4096, 8192, 16384}) {
    const int b = 64;
    const int64_t ld = mp;
    std::vector<double> h((size_t)ld * b);
    uint64_t st = 12345;
    for (auto& x : h) {
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      x = (double)(st >> 11) / 9007199254740992.0 - 0.5;
    }
    double *A, *A0, *V, *tau, *acc;
    unsigned* bar;
    int* flag;
    cudaMalloc(&A, 8 * ld * b);
    cudaMalloc(&A0, 8 * ld * b);
    cudaMalloc(&V, 8 * ld * b);
    cudaMalloc(&tau, 8 * 64);
    cudaMalloc(&acc, 8 * 3 * 128 + 256);
    cudaMemset(acc, 0, 8 * 3 * 128 + 256);
    bar = reinterpret_cast<unsigned*>(acc + 3 * 128);
    double* T;
    cudaMalloc(&T, 8 * 64 * 64);
    cudaMalloc(&flag, 4);
    cudaMemcpy(A0, h.data(), 8 * ld * b, cudaMemcpyHostToDevice);
    Ctx ctx;
    if (getenv("CAP")) ctx.panel_max_ctas = atoi(getenv("CAP"));
    ctx.dflag = flag;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 20;
    float total = 0;
    for (int it = 0; it < reps + 3; ++it) {
      cudaMemcpy(A, A0, 8 * ld * b, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      PanelTail tl;
      tl.T = T;
      tl.ldt = 64;
      tl.vz = V;
      tl.zrows = 0;
      tl.ticket = bar + 32;
      panel_factor(ctx, DMat{A, ld, 0, 0, mp, b}, DMat{V, ld, 0, 0, mp, b}, tau, acc, bar, tl);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 3) total += ms;
    }
    long long t[16] = {};
#ifndef NO_TRACE
    cudaMemcpyFromSymbol(t, g_panel_trace, sizeof(t));
#endif
    printf("panel %5d x %d: %7.1f us  (%.2f us/column) %s\n", mp, b, 1e3 * total / reps,
           1e3 * total / reps / b, cudaGetErrorString(cudaGetLastError()));
    printf("  col10: scalars %lld loop %lld snap %lld sync %lld reduce %lld\n", t[9]-t[8], t[10]-t[9], t[11]-t[10], t[12]-t[11], t[13]-t[12]);
    // host Householder QR (same convention) for R, V, tau
    std::vector<double> hr(h), hv((size_t)ld * b, 0.0), htau(b, 0.0);
    for (int j = 0; j < b; ++j) {
      double sig2 = 0;
      for (int i = j + 1; i < mp; ++i) sig2 += hr[i + j * ld] * hr[i + j * ld];
      const double x0 = hr[j + j * ld], normx = std::sqrt(x0 * x0 + sig2);
      const bool reflect = (j < mp - 1) && normx > 0;
      double beta = x0, v0 = 1, taup = 0;
      if (reflect) {
        beta = -(x0 >= 0 ? 1.0 : -1.0) * normx;
        v0 = x0 - beta;
        taup = (beta - x0) / beta;
      }
      hv[j + j * ld] = 1.0;
      for (int i = j + 1; i < mp; ++i) hv[i + j * ld] = reflect ? hr[i + j * ld] / v0 : 0.0;
      htau[j] = taup;
      for (int cc = j + 1; cc < b; ++cc) {
        double d = hr[j + cc * ld];
        for (int i = j + 1; i < mp; ++i) d += hv[i + j * ld] * hr[i + cc * ld];
        const double w = taup * d;
        hr[j + cc * ld] -= w;
        for (int i = j + 1; i < mp; ++i) hr[i + cc * ld] -= w * hv[i + j * ld];
      }
      hr[j + j * ld] = beta;
      for (int i = j + 1; i < mp; ++i) hr[i + j * ld] = 0.0;
    }
    std::vector<double> gr((size_t)ld * b), gv((size_t)ld * b), gt(b);
    cudaMemcpy(gr.data(), A, 8 * ld * b, cudaMemcpyDeviceToHost);
    cudaMemcpy(gv.data(), V, 8 * ld * b, cudaMemcpyDeviceToHost);
    cudaMemcpy(gt.data(), tau, 8 * b, cudaMemcpyDeviceToHost);
    double er = 0, ev = 0, et = 0, rmax = 0;
    for (size_t k = 0; k < (size_t)ld * b; ++k) {
      er = std::max(er, std::abs(gr[k] - hr[k]));
      ev = std::max(ev, std::abs(gv[k] - hv[k]));
      rmax = std::max(rmax, std::abs(hr[k]));
    }
    for (int j = 0; j < b; ++j) et = std::max(et, std::abs(gt[j] - htau[j]));
    printf("  max|dR| %.2e (|R| %.1f)  max|dV| %.2e  max|dtau| %.2e\n", er, rmax, ev, et);
    cudaFree(A); cudaFree(A0); cudaFree(V); cudaFree(tau); cudaFree(acc); cudaFree(T); cudaFree(flag);
  }
  return 0;
}
