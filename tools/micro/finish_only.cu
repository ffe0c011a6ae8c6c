// microbenchmark: latency of finish_row (the per-row final stage of the top-k
// kernel) in a 256-thread CTA, with the top-k kernel's launch bounds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/micro/finish.cu -o tools/micro/finish
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2512_00719_b200/csrc/finish.cuh"
#ifndef FNT
#define FNT 256
#endif
using namespace dp;

template <int MB>
__global__ void __launch_bounds__(FNT, MB) kern(SampleArgs a, const float* row, int n, int plen, int nsel_in,
                                                long long* cyc) {
  extern __shared__ __align__(16) uint8_t smem[];
  const FinLayout F = fin_layout(a.lcap);
  __shared__ uint64_t sel[1024];
  __shared__ FinishScratch fs;
  const uint32_t t = threadIdx.x;
  for (int i = t; i < nsel_in; i += FNT) sel[i] = comp_key(row[i], (uint32_t)i);
  const dp_params_t p = a.params[0];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < 16; ++it) {
    finish_row<float, kFull, FNT, false, false>(a, 0, p, plen, row, 0, n, sel, nsel_in, 0.0, 0.0, smem, F, fs, t,
                                  [] { __syncthreads(); });
    __syncthreads();
  }
  long long t1 = clock64();
  if (t == 0) { cyc[0] = (t1 - t0) / 16; cyc[1] = cyc[2] = cyc[5] = cyc[6] = 0; }
}

int main(int argc, char** argv) {
  const int nblk = argc > 1 ? atoi(argv[1]) : 1;
  const int n = 8192, cap = 256;
  const int nsel = argc > 2 ? atoi(argv[2]) : 150, plen = argc > 3 ? atoi(argv[3]) : 100;
  std::vector<float> h(n);
  for (int i = 0; i < n; ++i) h[i] = (i < 1000) ? 5.0f - 0.004f * i : -3.0f - 1e-4f * i;
  float* row; cudaMalloc(&row, n * 4); cudaMemcpy(row, h.data(), n * 4, cudaMemcpyHostToDevice);
  std::vector<int> ids(cap), cnt(cap, 1);
  for (int j = 0; j < plen; ++j) ids[j] = (j * 37) % n;
  int *d_ids, *d_cnt, *d_len, *d_plen; cudaMalloc(&d_ids, cap * 4); cudaMalloc(&d_cnt, cap * 4);
  cudaMalloc(&d_len, 4); cudaMalloc(&d_plen, 4);
  cudaMemcpy(d_ids, ids.data(), cap * 4, cudaMemcpyHostToDevice); cudaMemcpy(d_cnt, cnt.data(), cap * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_len, &plen, 4, cudaMemcpyHostToDevice); cudaMemcpy(d_plen, &plen, 4, cudaMemcpyHostToDevice);
  dp_params_t hp{}; hp.temperature = 0.8; hp.top_k = 50; hp.top_p = 0.9; hp.min_p = 0.05; hp.rep_penalty = 1.1;
  hp.presence_penalty = 0.5; hp.frequency_penalty = 0.1; hp.seed = 0;
  dp_params_t* d_p; cudaMalloc(&d_p, sizeof(hp)); cudaMemcpy(d_p, &hp, sizeof(hp), cudaMemcpyHostToDevice);
  double hu[3] = {0.3, 0.5, 0.7}; double* d_u; cudaMalloc(&d_u, 24); cudaMemcpy(d_u, hu, 24, cudaMemcpyHostToDevice);
  int32_t* tok; double* lp; uint8_t* fl; cudaMalloc(&tok, 4); cudaMalloc(&lp, 8); cudaMalloc(&fl, 1);
  cudaMemset(fl, 0, 1);
  long long* cyc; cudaMallocManaged(&cyc, 64);
  long long* st; cudaMallocManaged(&st, 24 * 8);
  SampleArgs a; memset(&a, 0, sizeof(a));
  a.logits = row; a.ld = n; a.V = n; a.H = 0; a.params = d_p;
  a.pen.ids = d_ids; a.pen.out_count = d_cnt; a.pen.len = d_len; a.pen.prompt_len = d_plen; a.pen.cap = cap;
  a.pen.vocab_size = n; a.uniforms = d_u; a.n_rows = 1; a.token = tok; a.logprob = lp; a.flags = fl;
  a.dbg.stats = getenv("LAPS") ? (int64_t*)st : nullptr;
  a.kcap = 256; a.lcap = 512; a.wcap = 1024; a.split = 1; a.nt = 256;
  const FinLayout F = fin_layout(a.lcap);
  for (int mb : {1, 2, 4}) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mb == 1) { cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, F.bytes); kern<1><<<nblk, FNT, F.bytes>>>(a, row, n, plen, nsel, cyc); }
      if (mb == 2) { cudaFuncSetAttribute(kern<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, F.bytes); kern<2><<<nblk, FNT, F.bytes>>>(a, row, n, plen, nsel, cyc); }
      if (mb == 4) { cudaFuncSetAttribute(kern<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, F.bytes); kern<4><<<nblk, FNT, F.bytes>>>(a, row, n, plen, nsel, cyc); }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    int tk; cudaMemcpy(&tk, tok, 4, cudaMemcpyDeviceToHost);
    printf("  laps/row:");
    for (int sl : {8, 12, 9, 10, 11, 13, 14, 16, 15}) printf(" %d:%lld", sl, st[sl] / (32 * nblk));
    printf("\n");
    for (int i = 0; i < 24; ++i) st[i] = 0;
    printf("[%d CTAs] finish_row minBlocks=%d: %lld cycles (token %d); draw in loop %lld, draw once %lld, draw interleaved with finish_row %lld, draw COLD %lld\n", nblk, mb, cyc[0], tk, cyc[1], cyc[2], cyc[5], cyc[6]);
  }
#ifdef DP_DRAW_PROBE
  long long hprobe[32];
  cudaMemcpyFromSymbol(hprobe, g_probe, sizeof(hprobe));
  printf("probe (finish_row ctx, cumulative): %lld %lld %lld %lld %lld\n", hprobe[0], hprobe[1], hprobe[2], hprobe[3], hprobe[4]);
  printf("probe (standalone ctx, cumulative): %lld %lld %lld %lld %lld\n", hprobe[8], hprobe[9], hprobe[10], hprobe[11], hprobe[12]);
  printf("probe (finish_row ctx, 2nd run):    %lld %lld %lld %lld %lld\n", hprobe[16], hprobe[17], hprobe[18], hprobe[19], hprobe[20]);
#endif
  return 0;
}
