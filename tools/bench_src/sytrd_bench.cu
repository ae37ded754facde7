// Per-phase clock marks of the SYTRD panel kernel (column 5 of the first panel).
// Build: make -C tools/bench_src sytrd_bench
#define QDWHG_TRD_TRACE 1
#include "../../paper_2104_14186_b200/csrc/syevd.cu"

#include <cstdio>
#include <vector>

using namespace qdwhg;

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 5016;
  const int nb = kTrdNB;
  std::vector<double> h((size_t)n * n);
  uint64_t st = 7;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j; ++i) {
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      const double v = (double)(st >> 11) / 9007199254740992.0 - 0.5;
      h[i + (size_t)j * n] = h[j + (size_t)i * n] = v;
    }
  double *A, *V, *W, *d, *e, *tau, *y, *red, *ypart;
  unsigned* bar;
  cudaMalloc(&A, 8ull * n * n);
  cudaMalloc(&V, 8ull * n * nb);
  cudaMalloc(&W, 8ull * n * nb);
  cudaMalloc(&d, 8ull * (n + 8));
  cudaMalloc(&e, 8ull * (n + 8));
  cudaMalloc(&tau, 8ull * (n + 64));
  cudaMalloc(&y, 8ull * (n + 2 * nb + 8));
  cudaMalloc(&red, 8 * 64);
  cudaMalloc(&ypart, 8ull * ((n + 31) / 32) * ((n + 31) / 32) * 32 + 64);
  cudaMalloc(&bar, 256);
  cudaMemcpy(A, h.data(), 8ull * n * n, cudaMemcpyHostToDevice);
  cudaMemset(y, 0, 8ull * (n + 2 * nb + 8));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = std::max(1, std::min(sms, (n + 31) / 32));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaMemset(red, 0, 8 * 64);
  cudaMemset(bar, 0, 4);
  cudaFuncSetAttribute(sytrd_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrdDynSmem);
  TrdArgs args{A, n, V, W, n, d, e, tau, y, ypart, red, bar, n, 0, nb};
  for (int warm = 0; warm < 2; ++warm) {
    cudaMemset(y, 0, 8ull * (n + 2 * nb + 8));
    cudaMemset(red, 0, 8 * 64);
    cudaMemset(bar, 0, 4);
    void* ka[] = {&args};
    cudaLaunchCooperativeKernel((void*)sytrd_panel_kernel, dim3(grid), dim3(kTrdThreads), ka, kTrdDynSmem, 0);
  }
  cudaMemcpy(A, h.data(), 8ull * n * n, cudaMemcpyHostToDevice);
  void* kargs[] = {&args};
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((void*)sytrd_panel_kernel, dim3(grid), dim3(kTrdThreads), kargs, kTrdDynSmem, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long t[16];
  cudaMemcpyFromSymbol(t, g_trd_trace, sizeof(t));
  printf("n=%d panel of %d columns: %.1f us (%.2f us/column) %s\n", n, nb, 1e3 * ms, 1e3 * ms / nb,
         cudaGetErrorString(cudaGetLastError()));
  printf("col5 cycles: A %lld | A-reduce %lld | bar1 %lld | refl+V %lld | SYMV %lld | bar3 %lld | D %lld | bar4 %lld\n",
         t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[5] - t[4], t[6] - t[5], t[7] - t[6], t[8] - t[7]);
  return 0;
}
