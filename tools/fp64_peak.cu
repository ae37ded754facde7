// FP64 peak probe for the roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
// Measures: (1) DMMA m8n8k4 issue-bound throughput, (2) DFMA throughput,
// both register-resident (no memory traffic), with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
  double* d; cudaMalloc(&d, 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16}) {
    int iters = 20000;
    dmma_loop<<<sms * 2, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms * 2, warps * 32>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 16 * (double)iters * warps * sms * 2;
    printf("DMMA m8n8k4 warps/CTA=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int warps : {8, 16, 32}) {
    int iters = 20000;
    dfma_loop<<<sms * 2, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms * 2, warps * 32>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * (double)iters * warps * 32 * sms * 2;
    printf("DFMA warps/CTA=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
