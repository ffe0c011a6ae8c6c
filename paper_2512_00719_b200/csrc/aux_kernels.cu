// aux_kernels.cu — per-row uniforms, penalty-state maintenance, debug ready
// rows and the synthetic logits producer.
#include "common.cuh"

namespace dp {

// rng.pregenerate_slice per row (rng.py:94-113; seed per row: service.py:761)
__global__ void uniforms_kernel(const dp_params_t* params, const uint64_t* seq_ids, int64_t B,
                                uint64_t iteration, double* out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double u[3];
  row_uniforms(params[b].seed, iteration, seq_ids[b], u);
  out[3 * b] = u[0];
  out[3 * b + 1] = u[1];
  out[3 * b + 2] = u[2];
}

// update_output_histogram (penalty.py:18-32): one warp per row scans the
// row's sparse list; hit -> count+1, miss -> append (id, 1).
__global__ void penalty_update_kernel(dp_penalty_t pen, const int32_t* token, int64_t B,
                                      uint8_t* flags) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= B) return;
  const uint32_t lane = threadIdx.x & 31u;
  if (flags && (flags[row] & DP_FLAG_DEGENERATE)) return;
  const int32_t tok = token[row];
  if (tok < 0 || tok >= pen.vocab_size) {
    if (lane == 0 && flags) flags[row] |= DP_FLAG_DEGENERATE;
    return;
  }
  int32_t* ids = pen.ids + row * pen.cap;
  int32_t* cnt = pen.out_count + row * pen.cap;
  const int32_t len = pen.len[row];
  // all loads of a 256-entry window in flight at once (one memory round trip
  // for the usual list sizes), then the first match
  int32_t hit = -1;
  for (int32_t base = 0; base < len && hit < 0; base += 256) {
    int32_t v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int32_t j = base + r * 32 + (int32_t)lane;
      v[r] = j < len ? ids[j] : -1;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const uint32_t m = __ballot_sync(0xffffffffu, v[r] == tok);
      if (m && hit < 0) hit = base + r * 32 + __ffs(m) - 1;
    }
  }
  if (lane == 0) {
    if (hit >= 0) {
      cnt[hit] += 1;
    } else if (len < pen.cap) {
      ids[len] = tok;
      cnt[len] = 1;
      pen.len[row] = len + 1;
    } else if (flags) {
      flags[row] |= DP_FLAG_PEN_OVERFLOW;
    }
  }
}

// new_sequence_state (core.py:144-169): keep the prompt prefix, zero counts
__global__ void penalty_reset_kernel(dp_penalty_t pen, int64_t B) {
  const int64_t row = blockIdx.x;
  if (row >= B) return;
  const int32_t pl = pen.prompt_len[row];
  for (int32_t j = threadIdx.x; j < pl; j += blockDim.x) pen.out_count[row * pen.cap + j] = 0;
  if (threadIdx.x == 0) pen.len[row] = pl;
}

// ReadyColumn.full (service.py:236-241) materialised in f64
template <typename T>
__global__ void ready_rows_kernel(const T* logits, int64_t V, int64_t ld, const dp_params_t* params,
                                  dp_penalty_t pen, double* out) {
  const int64_t row = blockIdx.y;
  const dp_params_t p = params[row];
  const T* x = logits + row * ld;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    out[row * V + v] = ready_plain(Elem<T>::get(x, v), p);
}
template <typename T>
__global__ void ready_rows_pen_kernel(const T* logits, int64_t V, int64_t ld, const dp_params_t* params,
                                      dp_penalty_t pen, double* out) {
  const int64_t row = blockIdx.x;
  const dp_params_t p = params[row];
  if (penalties_neutral(p)) return;
  const int32_t len = pen.len[row];
  for (int32_t j = threadIdx.x; j < len; j += blockDim.x) {
    const int32_t id = pen.ids[row * pen.cap + j];
    out[row * V + id] = ready_penalized(Elem<T>::get(logits + row * ld, id), pen.out_count[row * pen.cap + j], p);
  }
}

// SyntheticSource.column (service.py:459-463): base + noise * Gumbel(u),
// u keyed by (seed, DOMAIN_LOGITS, iteration, seq, v), clamped at 2^-60.
template <typename T>
DP_DEV float synth_value(const double* base, double noise, uint64_t h0, int64_t id, T* dst) {
  double u = unit53(mix64(h0 ^ (uint64_t)id));
  u = fmax(u, 8.673617379884035e-19);   // 2^-60
  const double g = -log(-log(u));
  const double z = base[id] + noise * g;
  if constexpr (sizeof(T) == 4) {
    *dst = (float)z;
    return (float)z;
  } else {
    *dst = __float2bfloat16_rn((float)z);
    return __bfloat162float(*dst);
  }
}

template <typename T>
__global__ void synth_kernel(const double* base, double noise, uint64_t seed, uint64_t iteration,
                             const uint64_t* seq_ids, int64_t V, int64_t ld, const int32_t* perm, T* out) {
  const int64_t row = blockIdx.y;
  const uint64_t h0 = mix64(hash_prefix(seed, kDomainLogits, iteration) ^ seq_ids[row]);
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < V; pos += (int64_t)gridDim.x * blockDim.x)
    synth_value<T>(base, noise, h0, perm ? (int64_t)perm[pos] : pos, out + row * ld + pos);
}

// The producer-fused summary (make_shard_blocks, service.py:470-504; paper:
// "w can be pre-computed on GPUs when writing logits"): the same generator,
// one 8-CTA cluster per row (rank r writes positions r*NT + tid + k*8*NT, so
// the grid is as fine-grained as the plain generator's), every CTA folding
// the values it writes (as rounded to T) into an online ExpSum; rank 0
// combines the ranks' (max, sum) over DSMEM and emits the penalty-free
// (row_max, total_expsum) of the row / tau — dp_row_summary_raw's output —
// without re-reading the row.
constexpr int kSynthCluster = 8;

template <typename T, int NT>
__global__ void __launch_bounds__(NT) synth_summary_kernel(const double* base, double noise, uint64_t seed,
                                                           uint64_t iteration, const uint64_t* seq_ids, int64_t B,
                                                           int64_t V, int64_t ld, const int32_t* perm, T* out,
                                                           const dp_params_t* params, double* row_max,
                                                           double* total) {
  __shared__ float redf[NT / 32];
  __shared__ double redd[NT / 32];
  __shared__ float cta_m;
  __shared__ double cta_s;
  constexpr int C = kSynthCluster;
  const uint32_t rank = cluster_ctarank();
  const int64_t row = blockIdx.x / C;
  const uint64_t h0 = mix64(hash_prefix(seed, kDomainLogits, iteration) ^ seq_ids[row]);
  const double tau = params[row].temperature;
  const float s2 = (float)(1.4426950408889634 / tau);
  T* o = out + row * ld;
  ExpSum acc;
  for (int64_t p0 = (int64_t)rank * NT + threadIdx.x; p0 < V; p0 += 4 * C * NT) {
    float x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t pos = p0 + (int64_t)j * C * NT;
      x[j] = pos < V ? synth_value<T>(base, noise, h0, perm ? (int64_t)perm[pos] : pos, o + pos) : -INFINITY;
    }
#ifdef DP_SYNTH_NOSUM   // A-B build: the fused kernel's structure without the summary arithmetic
    acc.m = fmaxf(acc.m, fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3])));
#else
    acc.add(x, s2);
#endif
  }
  float m = warp_max(acc.m);
  if ((threadIdx.x & 31u) == 0) redf[threadIdx.x >> 5] = m;
  __syncthreads();
  m = redf[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) m = fmaxf(m, redf[w]);
  const double sr = warp_sum(acc.rel(m, s2));
  if ((threadIdx.x & 31u) == 0) redd[threadIdx.x >> 5] = sr;
  __syncthreads();
  if (threadIdx.x == 0) {
    double S = 0.0;
    for (int w = 0; w < NT / 32; ++w) S += redd[w];   // fixed order: deterministic
    cta_m = m;
    cta_s = S;
  }
  cluster_sync();   // every rank's (cta_m, cta_s) is visible cluster-wide
  if (rank == 0 && threadIdx.x == 0) {
    float rm[C];
    double rs[C];
    float M = -INFINITY;
    for (int r = 0; r < C; ++r) {
      rm[r] = __uint_as_float(ld_dsmem_u32(dsmem_addr(&cta_m, r)));
      rs[r] = __longlong_as_double((long long)ld_dsmem_u64(dsmem_addr(&cta_s, r)));
      M = fmaxf(M, rm[r]);
    }
    double S = 0.0;
    for (int r = 0; r < C; ++r)
      if (rm[r] != -INFINITY) S += rs[r] * exp2((double)(rm[r] - M) * (double)s2);
    row_max[row] = M == -INFINITY ? -INFINITY : (tau != 1.0 ? __ddiv_rn((double)M, tau) : (double)M);
    total[row] = S;
  }
  cluster_sync();   // rank 0 has read every peer's shared memory before anyone exits
}

// DecisionBatch wire payload (transport.py:173-184): u32 count, then per row
// u64 seq_id, u32 token_id, u8 flags (bit0 eos, bit1 accepted_hot,
// bit2 has_logprob), f32 logprob — 17 unaligned little-endian bytes per row.
__global__ void encode_decisions_kernel(const int32_t* token, const double* logprob, const uint8_t* flags,
                                        const uint64_t* seq_ids, int64_t B, uint8_t* out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) {
    const uint32_t n = (uint32_t)B;
    for (int i = 0; i < 4; ++i) out[i] = (uint8_t)(n >> (8 * i));
  }
  if (b >= B) return;
  uint8_t* r = out + 4 + 17 * b;
  const uint64_t s = seq_ids[b];
  const uint32_t t = (uint32_t)token[b];
  const uint8_t f = flags[b];
  const uint8_t wf = (uint8_t)((f & DP_FLAG_EOS) | (f & DP_FLAG_ACCEPTED_HOT) | 0x04u);
  const uint32_t lp = __float_as_uint((float)logprob[b]);
  for (int i = 0; i < 8; ++i) r[i] = (uint8_t)(s >> (8 * i));
  for (int i = 0; i < 4; ++i) r[8 + i] = (uint8_t)(t >> (8 * i));
  r[12] = wf;
  for (int i = 0; i < 4; ++i) r[13 + i] = (uint8_t)(lp >> (8 * i));
}

}  // namespace dp

using namespace dp;

cudaError_t dp_launch_encode(const int32_t* token, const double* logprob, const uint8_t* flags,
                             const uint64_t* seq_ids, int64_t B, uint8_t* out, cudaStream_t st) {
  encode_decisions_kernel<<<(unsigned)((B + 255) / 256 > 0 ? (B + 255) / 256 : 1), 256, 0, st>>>(token, logprob, flags,
                                                                                               seq_ids, B, out);
  return cudaGetLastError();
}

cudaError_t dp_launch_uniforms(const dp_params_t* params, const uint64_t* seq_ids, int64_t B,
                               uint64_t iteration, double* out, cudaStream_t st) {
  uniforms_kernel<<<(unsigned)((B + 127) / 128), 128, 0, st>>>(params, seq_ids, B, iteration, out);
  return cudaGetLastError();
}
cudaError_t dp_launch_penalty_update(const dp_penalty_t& pen, const int32_t* token, int64_t B,
                                     uint8_t* flags, cudaStream_t st) {
  penalty_update_kernel<<<(unsigned)((B + 7) / 8), 256, 0, st>>>(pen, token, B, flags);
  return cudaGetLastError();
}
cudaError_t dp_launch_penalty_reset(const dp_penalty_t& pen, int64_t B, cudaStream_t st) {
  penalty_reset_kernel<<<(unsigned)B, 128, 0, st>>>(pen, B);
  return cudaGetLastError();
}
cudaError_t dp_launch_ready_rows(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                                 const dp_params_t* params, const dp_penalty_t& pen, double* out,
                                 cudaStream_t st) {
  dim3 g((unsigned)((V + 255) / 256 < 64 ? (V + 255) / 256 : 64), (unsigned)B);
  if (dtype == DP_F32) {
    ready_rows_kernel<float><<<g, 256, 0, st>>>((const float*)logits, V, ld, params, pen, out);
    ready_rows_pen_kernel<float><<<(unsigned)B, 128, 0, st>>>((const float*)logits, V, ld, params, pen, out);
  } else {
    ready_rows_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16*)logits, V, ld, params, pen, out);
    ready_rows_pen_kernel<__nv_bfloat16><<<(unsigned)B, 128, 0, st>>>((const __nv_bfloat16*)logits, V, ld, params,
                                                                        pen, out);
  }
  return cudaGetLastError();
}
cudaError_t dp_launch_synth(const double* base, double noise, uint64_t seed, uint64_t iteration,
                            const uint64_t* seq_ids, int64_t B, int64_t V, int64_t ld, const int32_t* perm,
                            int dtype, void* out, const dp_params_t* params, double* row_max, double* total,
                            cudaStream_t st) {
  if (row_max) {
    constexpr int NT = 256;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * kSynthCluster));
    cfg.blockDim = dim3(NT);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kSynthCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (dtype == DP_F32)
      return cudaLaunchKernelEx(&cfg, synth_summary_kernel<float, NT>, base, noise, seed, iteration, seq_ids, B, V,
                                ld, perm, (float*)out, params, row_max, total);
    return cudaLaunchKernelEx(&cfg, synth_summary_kernel<__nv_bfloat16, NT>, base, noise, seed, iteration, seq_ids,
                              B, V, ld, perm, (__nv_bfloat16*)out, params, row_max, total);
  }
  dim3 g((unsigned)((V + 255) / 256 < 148 ? (V + 255) / 256 : 148), (unsigned)B);
  if (dtype == DP_F32)
    synth_kernel<float><<<g, 256, 0, st>>>(base, noise, seed, iteration, seq_ids, V, ld, perm, (float*)out);
  else
    synth_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(base, noise, seed, iteration, seq_ids, V, ld, perm,
                                                   (__nv_bfloat16*)out);
  return cudaGetLastError();
}
