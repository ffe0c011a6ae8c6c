// correctness + latency of the warp sorting networks in wsort.cuh
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/micro/wsort.cu -o tools/micro/wsort
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include "../../paper_2512_00719_b200/csrc/wsort.cuh"
using namespace dp;

__global__ void kern(const uint64_t* in, int n, uint64_t* out, long long* cyc) {
  const uint32_t lane = threadIdx.x;
  Item a = lane < (uint32_t)n ? Item{in[lane], lane} : item_worst();
  Item b = 32 + lane < (uint32_t)n ? Item{in[32 + lane], 32 + lane} : item_worst();
  long long t0 = clock64();
  warp_sort64_desc(a, b);
  long long t1 = clock64();
  // fold the remaining chunks of 64 in with merges
  long long tm = 0;
  for (int base = 64; base < n; base += 64) {
    Item c = base + lane < (uint32_t)n ? Item{in[base + lane], base + lane} : item_worst();
    Item d = base + 32 + lane < (uint32_t)n ? Item{in[base + 32 + lane], base + 32 + lane} : item_worst();
    long long m0 = clock64();
    warp_sort64_desc(c, d);
    warp_merge64_desc(a, b, c, d);
    tm += clock64() - m0;
  }
  out[lane] = a.k;
  out[32 + lane] = b.k;
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = tm; }
}

int main() {
  const int n = 300;
  std::vector<uint64_t> h(n);
  srand(1);
  for (int i = 0; i < n; ++i) h[i] = ((uint64_t)rand() << 32) | (uint64_t)rand();
  uint64_t *din, *dout; long long* cyc;
  cudaMalloc(&din, n * 8); cudaMalloc(&dout, 64 * 8); cudaMallocManaged(&cyc, 16);
  cudaMemcpy(din, h.data(), n * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) { kern<<<1, 32>>>(din, n, dout, cyc); cudaDeviceSynchronize(); }
  std::vector<uint64_t> g(64);
  cudaMemcpy(g.data(), dout, 64 * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end(), [](uint64_t x, uint64_t y) { return x > y; });
  bool ok = true;
  for (int i = 0; i < 64; ++i) ok &= g[i] == h[i];
  printf("top-64 of %d: %s; sort64 %lld cycles, %d x (sort64+merge) %lld cycles\n", n, ok ? "OK" : "WRONG", cyc[0],
         (n - 1) / 64, cyc[1]);
  return ok ? 0 : 1;
}
