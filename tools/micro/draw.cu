// microbenchmark: cycles of warp_filter_draw on one warp, k = 50, sorted input
#include <cstdio>
#include "../../paper_2512_00719_b200/csrc/sampler.cuh"
using namespace dp;
__global__ void kern(double* out, long long* cyc, int k, int iters) {
  __shared__ double r[1024], w[1024], cum[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) r[i] = -0.01 * i;
  __syncwarp();
  dp_params_t p;
  p.temperature = 0.8; p.top_k = k; p.top_p = 0.9; p.min_p = 0.05;
  p.rep_penalty = 1.1; p.presence_penalty = 0.5; p.frequency_penalty = 0.1; p.seed = 0;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    DrawResult d = warp_filter_draw(r, k, knobs_of(p), 0.3 + 1e-4 * it, w, cum);
    acc += d.logprob + d.index;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / iters; out[0] = acc; }
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 64); cudaMallocManaged(&cyc, 64);
  for (int k : {50, 200}) {
    kern<<<1, 32>>>(out, cyc, k, 100); cudaDeviceSynchronize();
    printf("k=%d: %lld cycles per warp_filter_draw\n", k, cyc[0]);
  }
  return 0;
}
