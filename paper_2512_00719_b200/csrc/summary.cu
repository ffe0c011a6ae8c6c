// summary.cu — producer row summary (K2) and the hot-mass curve (K6).
//
// K2 is make_shard_blocks' per-row (row_max, total_expsum) over the penalized,
// temperature-scaled row (service.py:470-504, shvs.row_summary shvs.py:157-168):
// one streaming pass with a per-thread online (max, sum) pair (ExpSum,
// common.cuh); penalized ids are excluded from the stream through a
// shared-memory bitmap and added back exactly in f64, so heavy penalties
// cannot cancel catastrophically.
#include "sampler.cuh"

namespace dp {

template <int NT>
DP_DEV double block_sum_f64(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < NT / 32; ++w) s += red[w];   // fixed order: deterministic
    red[32] = s;
  }
  __syncthreads();
  s = red[32];
  __syncthreads();
  return s;
}
template <int NT>
DP_DEV float block_max_f32(float v, float* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = red[0];
    for (int w = 1; w < NT / 32; ++w) m = fmaxf(m, red[w]);
    red[32] = m;
  }
  __syncthreads();
  v = red[32];
  __syncthreads();
  return v;
}

// One CTA per row, 16-byte streaming loads (U per thread in flight), the
// online ExpSum per vector (one max + compare, SFU exp2 terms centred on the
// running maximum, one f64 add per vector).  PEN: penalized positions are
// masked to -inf through the shared bitmap (one funnel shift per vector) and
// added back exactly in f64 after the stream.
template <typename T, int NT, int U, bool PEN>
__global__ void __launch_bounds__(NT, 2048 / NT / 2) row_summary_kernel(const T* logits, int64_t V, int64_t ld,
                                                                      const dp_params_t* params, dp_penalty_t pen,
                                                                      const int32_t* inv_perm, double* row_max,
                                                                      double* total) {
  constexpr int EPV = Elem<T>::kPerVec;
  extern __shared__ __align__(16) uint8_t smem[];
  double* redd = reinterpret_cast<double*>(smem);
  float* redf = reinterpret_cast<float*>(smem + 40 * 8);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem + 40 * 8 + 40 * 4);
  const int64_t row = blockIdx.x;
  const dp_params_t p = params[row];
  const T* x = logits + row * ld;
  const int32_t plen = (!PEN || penalties_neutral(p) || pen.len == nullptr) ? 0 : pen.len[row];
  const int32_t* pids = pen.ids + row * pen.cap;
  const int32_t* pcnt = pen.out_count + row * pen.cap;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(x);
  const int32_t a0 = (int32_t)min64(V, (int64_t)(((16u - (addr & 15u)) & 15u) / sizeof(T)));
  const int32_t nvec = (int32_t)((V - a0) / EPV);
  const int32_t tail0 = a0 + nvec * EPV;
  if (PEN) {
    const uint32_t words = (uint32_t)((V + 31) / 32) + 1u;   // +1: funnel-shift window
    for (uint32_t i = threadIdx.x; i < words; i += NT) bitmap[i] = 0u;
    __syncthreads();
    for (int32_t j = threadIdx.x; j < plen; j += NT) {
      const int64_t pos = inv_perm ? inv_perm[pids[j]] : pids[j];
      atomicOr(&bitmap[pos >> 5], 1u << (pos & 31));
    }
    __syncthreads();
  }
  const float s2 = (float)(1.4426950408889634 / p.temperature);
  auto masked = [&](float v, int64_t pos) -> float {
    return (PEN && plen > 0 && ((bitmap[pos >> 5] >> (pos & 31)) & 1u)) ? -INFINITY : v;
  };
  ExpSum acc;
  if (threadIdx.x < 32) {   // scalar head / tail elements
    const int32_t i = threadIdx.x, ti = tail0 + threadIdx.x;
    float h[2] = {i < a0 ? masked(Elem<T>::get(x, i), i) : -INFINITY,
                  ti < V ? masked(Elem<T>::get(x, ti), ti) : -INFINITY};
    acc.add(h, s2);
  }
  const uint4* vp = reinterpret_cast<const uint4*>(x + a0);
  auto fold = [&](const uint4& vv, int32_t idx) {
    float e[EPV];
#pragma unroll
    for (int i = 0; i < EPV; ++i) e[i] = vec_elem<T>(vv, i);
    if (PEN && plen > 0) {
      const uint32_t p0 = (uint32_t)(a0 + idx * EPV);
      const uint32_t pm = __funnelshift_r(bitmap[p0 >> 5], bitmap[(p0 >> 5) + 1], p0 & 31u);
#pragma unroll
      for (int i = 0; i < EPV; ++i) if ((pm >> i) & 1u) e[i] = -INFINITY;
    }
    acc.add(e, s2);
  };
  int32_t base = threadIdx.x;
  for (; base + (U - 1) * NT < nvec; base += NT * U) {   // full batches: unpredicated loads
    uint4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) v[j] = ld_stream16(vp + base + j * NT);
#pragma unroll
    for (int j = 0; j < U; ++j) fold(v[j], base + j * NT);
  }
  for (int32_t idx = base; idx < nvec; idx += NT) fold(ld_stream16(vp + idx), idx);
  // combine thread states: raw maximum, then every partial sum rescaled to it
  const float mnp = block_max_f32<NT>(acc.m, redf);
  const double snp = block_sum_f64<NT>(acc.rel(mnp, s2), redd);
  // penalized ids, exact f64 (penalty.py:66-78)
  double rpen = -INFINITY, sp = 0.0;
  if (PEN) {
    double rmax_pen = -INFINITY;
    for (int32_t j = threadIdx.x; j < plen; j += NT) {
      const int64_t pos = inv_perm ? inv_perm[pids[j]] : pids[j];
      rmax_pen = fmax(rmax_pen, ready_penalized(Elem<T>::get(x, pos), pcnt[j], p));
    }
    rmax_pen = warp_max(rmax_pen);
    if ((threadIdx.x & 31u) == 0) redd[threadIdx.x >> 5] = rmax_pen;
    __syncthreads();
    if (threadIdx.x == 0) {
      double mm = redd[0];
      for (int w = 1; w < NT / 32; ++w) mm = fmax(mm, redd[w]);
      redd[33] = mm;
    }
    __syncthreads();
    rpen = redd[33];
    __syncthreads();
  }
  const double rnp = mnp == -INFINITY ? -INFINITY : ready_plain(mnp, p);
  const double M = fmax(rnp, rpen);
  if (PEN) {
    double spen = 0.0;
    for (int32_t j = threadIdx.x; j < plen; j += NT) {
      const int64_t pos = inv_perm ? inv_perm[pids[j]] : pids[j];
      spen += exp(ready_penalized(Elem<T>::get(x, pos), pcnt[j], p) - M);
    }
    sp = block_sum_f64<NT>(spen, redd);
  }
  if (threadIdx.x == 0) {
    row_max[row] = M;
    total[row] = (rnp == -INFINITY ? 0.0 : snp * exp(rnp - M)) + sp;
  }
}

// K6: out[row, g] = ready mass of hot positions [0, grid[g]) / total_expsum
template <typename T, int NT>
__global__ void __launch_bounds__(NT) hot_mass_curve_kernel(const T* logits, int64_t V, int64_t ld,
                                                            const double* row_max, const double* total,
                                                            const dp_params_t* params, dp_penalty_t pen,
                                                            const int32_t* inv_perm, const int32_t* col_of_pos,
                                                            const int32_t* grid, int32_t n_grid, double* out) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* redd = reinterpret_cast<double*>(smem);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem + 40 * 8);
  const int64_t row = blockIdx.x;
  const dp_params_t p = params[row];
  const T* x = logits + row * ld;
  const int32_t plen = penalties_neutral(p) ? 0 : pen.len[row];
  const int32_t* pids = pen.ids + row * pen.cap;
  const int32_t* pcnt = pen.out_count + row * pen.cap;
  const int64_t hmax = grid[n_grid - 1];
  const uint32_t words = plen > 0 ? (uint32_t)((hmax + 31) / 32) : 0u;
  for (uint32_t i = threadIdx.x; i < words; i += NT) bitmap[i] = 0u;
  __syncthreads();
  for (int32_t j = threadIdx.x; j < plen; j += NT) {
    const int64_t pos = inv_perm ? inv_perm[pids[j]] : pids[j];
    if (pos < hmax) atomicOr(&bitmap[pos >> 5], 1u << (pos & 31));
  }
  __syncthreads();
  const double M = row_max[row], S = total[row];
  const double c = M * p.temperature;
  const float c_hi = (float)c, c_lo = (float)(c - (double)(float)c);
  const float inv_tau = (float)(1.0 / p.temperature);
  double acc = 0.0;
  int64_t lo = 0;
  for (int32_t g = 0; g < n_grid; ++g) {
    const int64_t hi = grid[g];
    double s = 0.0;
    // 4 independent loads in flight per thread (one at a time was L2/HBM
    // latency-bound)
    int64_t pos = lo + threadIdx.x;
    for (; pos + 3 * NT < hi; pos += 4 * NT) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t q = pos + u * NT;
        v[u] = Elem<T>::get(x, col_of_pos ? (int64_t)col_of_pos[q] : q);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t q = pos + u * NT;
        if (plen > 0 && ((bitmap[q >> 5] >> (q & 31)) & 1u)) continue;
        s += (double)expf(((v[u] - c_hi) - c_lo) * inv_tau);
      }
    }
    for (; pos < hi; pos += NT) {
      if (plen > 0 && ((bitmap[pos >> 5] >> (pos & 31)) & 1u)) continue;
      const float v = Elem<T>::get(x, col_of_pos ? (int64_t)col_of_pos[pos] : pos);
      s += (double)expf(((v - c_hi) - c_lo) * inv_tau);
    }
    for (int32_t j = threadIdx.x; j < plen; j += NT) {
      const int64_t pos = inv_perm ? inv_perm[pids[j]] : pids[j];
      if (pos >= lo && pos < hi)
        s += exp(ready_penalized(Elem<T>::get(x, col_of_pos ? (int64_t)col_of_pos[pos] : pos), pcnt[j], p) - M);
    }
    acc += block_sum_f64<NT>(s, redd);
    if (threadIdx.x == 0) out[row * n_grid + g] = S > 0.0 ? fmin(acc / S, 1.0) : 0.0;
    lo = hi;
  }
}

// Exact re-decision of the SHVS accept tests that defer_accept (sampler.cuh)
// left open: the row's ready total S relative to the producer's row max,
// summed exactly (f64 exp of every ready value; penalized positions excluded
// from the stream by a bitmap and added with their penalized values), then
// alpha = S_H / S and the accept test of shvs.py:223-236.  An accepted row
// keeps the hot decision the hot pass wrote and records its token (fused
// update); a rejected one joins the reject list for the tail pass, which runs
// after this kernel.
template <typename T, int NT>
__global__ void __launch_bounds__(NT) resum_kernel(SampleArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* redd = reinterpret_cast<double*>(smem);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem + 40 * 8);
  const int nrows = *a.resum_count;
  const uint32_t words = (uint32_t)((a.V + 31) / 32);
  for (int ridx = blockIdx.x; ridx < nrows; ridx += gridDim.x) {
    const int row = a.resum_rows[ridx];
    const dp_params_t p = a.params[row];
    const int32_t plen = pen_len(a, row, p);
    const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
    const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;
    const double mrow = a.row_max[row];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < words; i += NT) bitmap[i] = 0u;
    __syncthreads();
    double s = 0.0;
    for (int32_t j = threadIdx.x; j < plen; j += NT) {
      const int64_t pos = id_to_pos(a, pids[j]);
      atomicOr(&bitmap[pos >> 5], 1u << (pos & 31));
      s += exp(ready_penalized(row_value<T>(a, row, pos), pcnt[j], p) - mrow);
    }
    __syncthreads();
    for (int64_t pos = threadIdx.x; pos < a.V; pos += NT) {
      if ((bitmap[pos >> 5] >> (pos & 31)) & 1u) continue;
      s += exp(ready_plain(row_value<T>(a, row, pos), p) - mrow);
    }
    const double S = block_sum_f64<NT>(s, redd);
    if (threadIdx.x == 0) {
      double u[3];
      get_uniforms(a, row, p, u);
      const double sH = a.resum_sh[row];
      const bool ok = S > 0.0 && isfinite(S);
      const double alpha = ok ? fmin(sH / S, 1.0) : 1.0;
      const bool near = fabs(u[1] - alpha) < kBoundaryEps;
      if (a.dbg.alpha) a.dbg.alpha[row] = alpha;
      touch_bytes(a, row, (uint64_t)(a.V + plen) * sizeof(T));   // the whole row + the penalty values
      if (a.dbg.stats) atomicAdd((unsigned long long*)&a.dbg.stats[2], 1ull);
      if (!ok) {
        a.token[row] = -1;
        a.logprob[row] = 0.0;
        a.flags[row] = DP_FLAG_REJECTED | DP_FLAG_DEGENERATE;
      } else if (u[1] <= alpha) {
        a.flags[row] |= near ? DP_FLAG_NEAR_BOUNDARY : 0;
        if (a.dbg.margin) a.dbg.margin[row] = fmin(a.dbg.margin[row], fabs(u[1] - alpha));
        thread_record_token(a, row, a.token[row]);   // fused K5
      } else {
        a.flags[row] = DP_FLAG_REJECTED | (near ? DP_FLAG_NEAR_BOUNDARY : 0);
        if (a.dbg.margin) a.dbg.margin[row] = fabs(u[1] - alpha);
        a.reject_rows[atomicAdd(a.reject_count, 1)] = row;
      }
    }
  }
}

cudaError_t launch_resum(const SampleArgs& a, int dtype, cudaStream_t st) {
  constexpr int NT = 256;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // deferred accept tests are rare (usually none): a small grid keeps the
  // empty launch cheap; CTAs loop over the list when there are more
#ifndef DP_RESUM_GRID
#define DP_RESUM_GRID 16
#endif
  const int cap_grid = DP_RESUM_GRID < sms ? DP_RESUM_GRID : sms;
  const int grid = a.n_rows < cap_grid ? (a.n_rows > 0 ? a.n_rows : 1) : cap_grid;
  const size_t smem = 40 * 8 + (size_t)((a.V + 31) / 32) * 4;
  if (dtype == DP_F32) {
    auto k = resum_kernel<float, NT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, NT, smem, st>>>(a);
  } else {
    auto k = resum_kernel<__nv_bfloat16, NT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, NT, smem, st>>>(a);
  }
  return cudaGetLastError();
}

template <typename T, bool PEN>
static void row_summary_t(const void* logits, int64_t B, int64_t V, int64_t ld, const dp_params_t* params,
                          const dp_penalty_t& pen, const int32_t* inv_perm, double* row_max, double* total,
                          cudaStream_t st) {
  constexpr int NT = 256, U = 4;
  const size_t smem = 40 * 8 + 40 * 4 + (PEN ? (size_t)((V + 31) / 32 + 1) * 4 : 0);
  auto k = row_summary_kernel<T, NT, U, PEN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<(unsigned)B, NT, smem, st>>>((const T*)logits, V, ld, params, pen, inv_perm, row_max, total);
}

cudaError_t launch_row_summary(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                               const dp_params_t* params, const dp_penalty_t& pen, const int32_t* inv_perm,
                               double* row_max, double* total, cudaStream_t st) {
  const bool pen_on = pen.len != nullptr;   // dp_row_summary_raw passes no penalty state
  if (dtype == DP_F32) {
    if (pen_on) row_summary_t<float, true>(logits, B, V, ld, params, pen, inv_perm, row_max, total, st);
    else row_summary_t<float, false>(logits, B, V, ld, params, pen, inv_perm, row_max, total, st);
  } else {
    if (pen_on) row_summary_t<__nv_bfloat16, true>(logits, B, V, ld, params, pen, inv_perm, row_max, total, st);
    else row_summary_t<__nv_bfloat16, false>(logits, B, V, ld, params, pen, inv_perm, row_max, total, st);
  }
  return cudaGetLastError();
}

cudaError_t launch_hot_mass_curve(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                                  const double* row_max, const double* total, const dp_params_t* params,
                                  const dp_penalty_t& pen, const int32_t* inv_perm, const int32_t* col_of_pos,
                                  const int32_t* grid, int32_t n_grid, double* out, cudaStream_t st) {
  constexpr int NT = 256;
  const size_t smem = 40 * 8 + (size_t)((V + 31) / 32) * 4;
  if (dtype == DP_F32) {
    auto k = hot_mass_curve_kernel<float, NT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)B, NT, smem, st>>>((const float*)logits, V, ld, row_max, total, params, pen, inv_perm,
                                     col_of_pos, grid, n_grid, out);
  } else {
    auto k = hot_mass_curve_kernel<__nv_bfloat16, NT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)B, NT, smem, st>>>((const __nv_bfloat16*)logits, V, ld, row_max, total, params, pen, inv_perm,
                                     col_of_pos, grid, n_grid, out);
  }
  return cudaGetLastError();
}

}  // namespace dp
