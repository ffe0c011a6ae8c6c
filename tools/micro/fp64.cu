// microbenchmark: dependent-chain latency of FP64 ops on one warp (clock64)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed, int n) {
  double x = seed + threadIdx.x * 1e-3, y = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = exp(x * 1e-3 - 0.5);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.5);
  long long t3 = clock64();
  float f = (float)x;
  for (int i = 0; i < n; ++i) f = __expf(f * 1e-3f - 0.5f);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) f = fmaf(f, 1.0000001f, 1e-9f);
  long long t5 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x + f;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 64);
  int n = 1000;
  for (int blocks : {1, 148, 148 * 8}) {
    k<<<blocks, 32>>>(out, cyc, 0.3, n); cudaDeviceSynchronize();
    printf("blocks=%d per-op cycles: dfma %.1f  exp(f64) %.1f  ddiv %.1f  __expf %.1f  ffma %.1f\n", blocks,
           cyc[0] / (double)n, cyc[1] / (double)n, cyc[2] / (double)n, cyc[3] / (double)n, cyc[4] / (double)n);
  }
  k<<<1, 256>>>(out, cyc, 0.3, n); cudaDeviceSynchronize();
  printf("1 block x 8 warps: dfma %.1f  exp(f64) %.1f  ddiv %.1f\n", cyc[0] / (double)n, cyc[1] / (double)n, cyc[2] / (double)n);
  return 0;
}
