// microbenchmark: latency (cycles) of the per-row final-stage primitives on
// one warp / one 128-thread CTA of an idle GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/micro/prims.cu -o tools/micro/prims
#include <cstdio>
#include "../../paper_2512_00719_b200/csrc/finish.cuh"
using namespace dp;

__global__ void kern(long long* cyc, double* sink) {
  __shared__ uint64_t key[1024];
  __shared__ uint32_t pos[1024];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t bcast[4];
  __shared__ double fr[1024], w[1024], cum[1024];
  const uint32_t t = threadIdx.x, lane = t & 31u;
  dp_params_t p;
  p.temperature = 0.8; p.top_k = 50; p.top_p = 0.9; p.min_p = 0.05;
  p.rep_penalty = 1.1; p.presence_penalty = 0.5; p.frequency_penalty = 0.1; p.seed = 0;
  double acc = 0;
  auto fill = [&](int n) {
    for (int i = t; i < 1024; i += blockDim.x) {
      uint32_t h = (uint32_t)i * 2654435761u;
      key[i] = i < n ? (((uint64_t)(h >> 4) << 32) | (0xFFFFFFFFu - i)) : 0ull;
      pos[i] = i;
      fr[i] = -0.01 * i;
    }
    __syncthreads();
  };
  long long t0, t1;
  // 1. warp_filter_draw_reg, k=50
  fill(0);
  if (t < 32) {
    t0 = clock64();
    for (int it = 0; it < 20; ++it) {
      DrawResult d = warp_filter_draw_reg(fr, 50, p, 0.3 + 1e-4 * it);
      acc += d.logprob + d.index;
    }
    t1 = clock64();
    if (t == 0) cyc[0] = (t1 - t0) / 20;
  }
  __syncthreads();
  // 2. warp_select_threshold over 350 keys, need 150
  fill(350);
  if (t < 32) {
    t0 = clock64();
    uint64_t th = 0;
    for (int it = 0; it < 20; ++it) th += warp_select_threshold(key, 350, 150 + (it & 1), hist);
    t1 = clock64();
    if (t == 0) cyc[1] = (t1 - t0) / 20;
    acc += (double)(th & 0xFF);
  }
  __syncthreads();
  // 3. warp_topk_sort 150 keys -> k=50 (destructive: refill each time)
  long long s3 = 0;
  for (int it = 0; it < 10; ++it) {
    fill(150);
    if (t < 32) {
      t0 = clock64();
      warp_topk_sort(key, pos, 150, 50, hist);
      t1 = clock64();
      s3 += t1 - t0;
    }
    __syncthreads();
  }
  if (t == 0) cyc[2] = s3 / 10;
  // 4. get_uniforms
  if (t < 32) {
    double u[3];
    t0 = clock64();
    for (int it = 0; it < 20; ++it) {
      row_uniforms(p.seed + it, 7, 9, u);
      acc += u[0] + u[1];
    }
    t1 = clock64();
    if (t == 0) cyc[3] = (t1 - t0) / 20;
  }
  // 5. f64 exp chain (dependent)
  if (t < 32) {
    double x = -0.5 + 1e-3 * lane;
    t0 = clock64();
    for (int it = 0; it < 20; ++it) x = exp(x - 1.0) - 0.5;
    t1 = clock64();
    if (t == 0) cyc[4] = (t1 - t0) / 20;
    acc += x;
  }
  // 6. ready_penalized dependent chain (ddiv x3)
  if (t < 32) {
    float xf = 1.0f + lane;
    double z = 0;
    t0 = clock64();
    for (int it = 0; it < 20; ++it) { z += ready_penalized(xf, it & 3, p); xf = (float)(z * 1e-9) + 1.0f; }
    t1 = clock64();
    if (t == 0) cyc[5] = (t1 - t0) / 20;
    acc += z;
  }
  __syncthreads();
  // 7. block (128) group_select_threshold over 350 keys, need 50
  fill(350);
  t0 = clock64();
  uint64_t th2 = 0;
  for (int it = 0; it < 10; ++it) {
    auto get = [&](uint32_t i, uint64_t& k) -> bool { k = key[i]; return true; };
    th2 += group_select_threshold<128>(get, 350, 350, 50 + (it & 1), hist, bcast, t, [] { __syncthreads(); });
  }
  t1 = clock64();
  if (t == 0) cyc[6] = (t1 - t0) / 10;
  acc += (double)(th2 & 0xFF);
  // 8. __syncthreads cost (128 threads)
  t0 = clock64();
  for (int it = 0; it < 100; ++it) __syncthreads();
  t1 = clock64();
  if (t == 0) cyc[7] = (t1 - t0) / 100;
  // 9. smem atomicAdd same-address from 32 lanes
  t0 = clock64();
  for (int it = 0; it < 20; ++it) atomicAdd(&hist[it & 3], 1u);
  __syncwarp();
  t1 = clock64();
  if (t == 0) cyc[8] = (t1 - t0) / 20;
  sink[t] = acc;
}

int main() {
  long long* cyc;
  double* sink;
  cudaMallocManaged(&cyc, 64 * sizeof(long long));
  cudaMalloc(&sink, 1024 * sizeof(double));
  for (int rep = 0; rep < 2; ++rep) {
    kern<<<1, 128>>>(cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  }
  const char* names[] = {"warp_filter_draw_reg k=50", "warp_select_threshold 350->150", "warp_topk_sort 150->50",
                         "row_uniforms", "f64 exp (dependent)", "ready_penalized (dependent)",
                         "group_select_threshold<128> 350->50", "__syncthreads (128)", "smem atomicAdd (32 lanes)"};
  for (int i = 0; i < 9; ++i) printf("%-40s %8lld cycles\n", names[i], cyc[i]);
  return 0;
}
