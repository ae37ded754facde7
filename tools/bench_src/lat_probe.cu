// Dependent-chain latency of FP64 ops on this GPU (clock64 around 256 chained
// ops in one thread): DFMA, DMUL, DADD, MUFU.RCP64H/RSQ64H, FFMA for reference,
// and shared-memory load-to-use.  Build: nvcc -arch=sm_100a -O3 lat_probe.cu
#include <cstdio>

__global__ void probe(double* out, long long* cyc, double x0, float f0) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x * 1e-3;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double x = x0, y = 1.0000001;
  float f = f0;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 256; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 256; ++i) x = x + 1e-9;
  t1 = clock64();
  cyc[1] = t1 - t0;
  // FFMA chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 256; ++i) f = fmaf(f, 1.0000001f, 1e-9f);
  t1 = clock64();
  cyc[2] = t1 - t0;
  // rcp.approx.f64 chain
  double r = x;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(r));
  t1 = clock64();
  cyc[3] = t1 - t0;
  // rsqrt.approx.f64 chain
  double q = x;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(q));
  t1 = clock64();
  cyc[4] = t1 - t0;
  // shared load-to-use (pointer chase through indices)
  int idx = 1;
  int* smi = reinterpret_cast<int*>(sm);
  for (int i = 0; i < 64; ++i) smi[i] = (i * 7 + 1) & 63;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) idx = smi[idx];
  t1 = clock64();
  cyc[5] = t1 - t0;
  // double-precision divide (IEEE, library sequence)
  double d = x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) d = 1.0000001 / d;
  t1 = clock64();
  cyc[6] = t1 - t0;
  out[0] = x + f + r + q + idx + d;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8 * 8);
  for (int rep = 0; rep < 3; ++rep) probe<<<1, 64>>>(out, cyc, 1.0, 1.0f);
  long long h[8];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("DFMA %.1f  DADD %.1f  FFMA %.1f  RCP64 %.1f  RSQ64 %.1f  LDS %.1f  DDIV %.1f cycles/op\n",
         h[0] / 256.0, h[1] / 256.0, h[2] / 256.0, h[3] / 64.0, h[4] / 64.0, h[5] / 64.0, h[6] / 64.0);
  return 0;
}
