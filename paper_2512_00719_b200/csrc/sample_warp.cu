// sample_warp.cu — warp-per-row sampler (K1w) for short top-k, sm_100a.
//
// One warp decides one row with no block-level barrier anywhere: for the
// SHVS hot pass (rows of H <= 64K logits) and other short rows at large batch
// the per-row CTA kernel spends most of its time in __syncthreads while one
// warp sorts / draws; here every warp streams, selects and draws its own row
// and the SM overlaps the phases of ~8 independent rows.
//
// Same decision law as sample_topk.cu (filtering.py:38-162, penalty.py:66-78,
// shvs.py:223-236):
//  1. threshold: the first batch of every lane is a strided sample of the row
//     (batch b, slot j reads vectors (j*nb + b)*32 + lane); each lane keeps
//     its top-4 sample values and a bitwise search over the warp's 128 values
//     gives t_lb (the kp-th: a proven lower bound of the row's kp-th largest)
//     and t_est (an estimate admitting ~2 kp elements);
//  2. stream: elements >= threshold are appended as unique (value desc,
//     position asc) keys to a 512-entry warp buffer; a full buffer is cut to
//     its kp largest, which also raises the threshold (exact: nothing below the
//     kp-th largest of a subset can reach the top-kp);  fewer than kp
//     survivors re-stream with t_lb;
//  3. exact top-kp (raw top-(k + |penalty list|), the superset argument of
//     _tail_preselect, service.py:309-336), sparse penalties in IEEE f64,
//     radix cut to the top-k, register sort, exact top-p / min-p / draw.
// kHot accumulates the raw hot mass of every element (f32 exp2 of the
// max-centred argument, f64 sum) and replaces the penalized ids' raw terms by
// their exact penalized mass: the subtracted terms are the bit-identical f32
// values that were added, so no per-element penalty test is needed.

#include "sampler.cuh"
#include "select.cuh"
#include "finish.cuh"

namespace dp {

constexpr int kWXcap = 512;   // candidate keys per warp (>= kWarpKpMax + one vector slot of the warp)
constexpr int kWHcap = 512;   // penalty hash slots (>= 2 * kWarpPenCap)
constexpr int kWPC = 2;       // warps per CTA
constexpr int kWU = 16;       // 16-byte vectors in flight per lane

struct WarpSmem {
  uint64_t key[kWXcap];   // stream candidates, then the final list keys
  uint32_t pos[kWXcap];   // final list positions
  uint32_t hist[256];
  uint32_t hash[kWHcap];
  double fr[kWarpKMax];
};

template <typename T, int MODE>
__global__ void __launch_bounds__(kWPC * 32) warp_sample_kernel(SampleArgs a) {
  constexpr int EPV = Elem<T>::kPerVec;
  constexpr int U = kWU;
  __shared__ WarpSmem sm_all[kWPC];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  WarpSmem& S = sm_all[warp];
  const int ridx = blockIdx.x * kWPC + (int)warp;
  const int nrows = a.row_count ? *a.row_count : a.n_rows;
  if (ridx >= nrows) return;
  const int row = a.rows ? a.rows[ridx] : ridx;
  const dp_params_t p = a.params[row];
  const int32_t plen = pen_len(a, row, p);
  const int64_t n = dom_n(a, MODE), lo = dom_lo(a, MODE);
  const int32_t k = p.top_k;
  if (route_row(a, MODE, k, plen, n) != kRouteWarp) return;
  const uint32_t kp = (uint32_t)min64(n, (int64_t)k + plen);
  const T* rowp = reinterpret_cast<const T*>(a.logits) + (int64_t)row * a.ld + lo;
  const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
  const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;

  // hot mass: exp((x - m tau)/tau) = 2^(((x - hi) - lo) * log2e/tau), with
  // m tau = hi + lo split so that x - m tau is exact near the row maximum
  double mrow = 0.0;
  float m_hi = 0.f, m_lo = 0.f, s2 = 0.f;
  if (MODE == kHot) {
    mrow = a.row_max[row];
    const double c = mrow * p.temperature;
    m_hi = (float)c;
    m_lo = (float)(c - (double)m_hi);
    s2 = (float)(1.4426950408889634 / p.temperature);
  }
  auto hot_exp = [&](float x) -> float { return ex2_fast(__fmul_rn(__fsub_rn(__fsub_rn(x, m_hi), m_lo), s2)); };

  // ---- geometry: 16-byte vectors (32-bit indices, V < 2^31)
  const uintptr_t addr = reinterpret_cast<uintptr_t>(rowp);
  const int32_t a0 = (int32_t)min64(n, (int64_t)(((16u - (addr & 15u)) & 15u) / sizeof(T)));
  const int32_t nvec = (int32_t)((n - a0) / EPV);
  const int32_t tail0 = a0 + nvec * EPV;
  const int32_t nb = max(1, (nvec + 32 * U - 1) / (32 * U));
  const uint4* vp = reinterpret_cast<const uint4*>(rowp + a0);
  auto vidx = [&](int32_t b, int j) -> int32_t { return (j * nb + b) * 32 + (int32_t)lane; };

  uint4 v[U];
#pragma unroll
  for (int j = 0; j < U; ++j) {
    const int32_t idx = vidx(0, j);
    v[j] = idx < nvec ? ld_stream16(vp + idx) : neg_inf_vec<T>();
  }

  // ---- thresholds from the strided first batch (per-lane top-4)
  float t4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int j = 0; j < U; ++j) {
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      float x = vec_elem<T>(v[j], e);
      if (x > t4[3]) {
        t4[3] = x;
        if (t4[3] > t4[2]) { const float q = t4[2]; t4[2] = t4[3]; t4[3] = q; }
        if (t4[2] > t4[1]) { const float q = t4[1]; t4[1] = t4[2]; t4[2] = q; }
        if (t4[1] > t4[0]) { const float q = t4[0]; t4[0] = t4[1]; t4[1] = q; }
      }
    }
  }
  // padding lanes hold -inf, which only lowers the thresholds (safe)
  uint32_t kk4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) kk4[i] = f32_key(t4[i]);
  // r-th largest of the warp's 128 kept sample values (bitwise search)
  auto kth = [&](uint32_t r) -> float {
    uint32_t t = 0u;
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t c = t | (1u << bit);
      uint32_t cnt = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) cnt += __popc(__ballot_sync(0xffffffffu, kk4[i] >= c));
      if (cnt >= r) t = c;
    }
    return key_f32(t);
  };
  const int64_t sampled = min64(n, (int64_t)32 * U * EPV);
  const float t_lb = kp <= 128u ? kth(kp) : -INFINITY;
  uint32_t r_est = (uint32_t)ceil(2.0 * (double)kp * (double)sampled / (double)n);
  r_est = max(1u, r_est);
  const float t_est = r_est <= 128u ? fmaxf(kth(r_est), t_lb) : t_lb;

  // ---- stream
  float thr_f = t_est;
  uint64_t thr_k = thr_f == -INFINITY ? 0ull : ((uint64_t)f32_key(thr_f) << 32);
  uint32_t cnt = 0;     // warp-uniform buffer fill
  double sh = 0.0;      // kHot: raw hot mass of this lane's elements
  // cut the buffer to its kp largest keys; raises the admission threshold
  auto cut = [&]() {
    __syncwarp();
    const uint64_t t = warp_select_threshold(S.key, cnt, kp, S.hist);
    cnt = warp_compact(S.key, cnt, t);
    if (t > thr_k) {
      thr_k = t;
      thr_f = comp_val(t);
    }
  };
  // append this lane's elements (mask m of admitted candidates, keys ks[])
  auto append = [&](uint32_t m, const uint64_t* ks, int nk) {
    const uint32_t c = __popc(m);
    const uint32_t incl = warp_incl_scan(c);
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t o = cnt + incl - c;
    for (int e = 0; e < nk; ++e)
      if ((m >> e) & 1u) S.key[o++] = ks[e];
    cnt += tot;
  };
  // vector j of the register batch: hot mass + admission
  auto consume = [&](const uint4& vv, int32_t idx, bool first_pass) {
    const bool valid = idx < nvec;
    if (MODE == kHot && first_pass && valid) {
#pragma unroll
      for (int e = 0; e < EPV; ++e) sh += (double)hot_exp(vec_elem<T>(vv, e));
    }
    bool any = false;
#pragma unroll
    for (int e = 0; e < EPV; ++e) any |= vec_elem<T>(vv, e) >= thr_f;
    any = any && valid;
    if (__any_sync(0xffffffffu, any)) {
      uint64_t ks[EPV];
      uint32_t m = 0;
#pragma unroll
      for (int e = 0; e < EPV; ++e) {
        ks[e] = comp_key(vec_elem<T>(vv, e), (uint32_t)(a0 + idx * EPV + e));
        if (valid && ks[e] >= thr_k) m |= 1u << e;
      }
      const uint32_t tot = __reduce_add_sync(0xffffffffu, __popc(m));
      if (cnt + tot > (uint32_t)kWXcap) {
        cut();
#pragma unroll
        for (int e = 0; e < EPV; ++e)
          if (ks[e] < thr_k) m &= ~(1u << e);
      }
      append(m, ks, EPV);
    }
  };

  for (int pass_no = 0;; ++pass_no) {
    const bool first = pass_no == 0;
    // scalar head / tail elements (at most 2*EPV-2)
    {
      const int32_t hi_i = (int32_t)lane, ti = tail0 + (int32_t)lane;
      const bool hv = hi_i < a0, tv = ti < n;
      const float hx = hv ? Elem<T>::get(rowp, hi_i) : -INFINITY;
      const float tx = tv ? Elem<T>::get(rowp, ti) : -INFINITY;
      if (MODE == kHot && first) {
        if (hv) sh += (double)hot_exp(hx);
        if (tv) sh += (double)hot_exp(tx);
      }
      uint64_t ks[2] = {comp_key(hx, (uint32_t)hi_i), comp_key(tx, (uint32_t)ti)};
      uint32_t m = (hv && ks[0] >= thr_k ? 1u : 0u) | (tv && ks[1] >= thr_k ? 2u : 0u);
      append(m, ks, 2);   // <= 14 keys: always fits
    }
    for (int32_t b = 0; b < nb; ++b) {
      if (b > 0 || !first) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int32_t idx = vidx(b, j);
          v[j] = idx < nvec ? ld_stream16(vp + idx) : neg_inf_vec<T>();
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j) consume(v[j], vidx(b, j), first);
    }
    if (cnt >= kp || thr_f <= t_lb) break;
    // the estimate was too high: re-stream with the proven bound
    thr_f = t_lb;
    thr_k = t_lb == -INFINITY ? 0ull : ((uint64_t)f32_key(t_lb) << 32);
    cnt = 0;
    if (a.dbg.stats && lane == 0) atomicAdd((unsigned long long*)&a.dbg.stats[1], 1ull);
  }
  __syncwarp();
  if (a.dbg.stats && lane == 0) {
    atomicAdd((unsigned long long*)&a.dbg.stats[0], 1ull);
    atomicAdd((unsigned long long*)&a.dbg.stats[3], (unsigned long long)cnt);
  }
  // exact raw top-kp
  if (cnt > kp) cut();
  __syncwarp();

  // ---- penalized ids of the domain -> hash set; kHot mass correction
  uint32_t hcap = 32;
  while (hcap < 2u * (uint32_t)plen) hcap <<= 1;
  const uint32_t hmask = hcap - 1u;
  for (uint32_t i = lane; i < hcap; i += 32) S.hash[i] = 0xFFFFFFFFu;
  __syncwarp();
  double spen = 0.0, sraw = 0.0;
  for (int32_t j = lane; j < plen; j += 32) {
    const int64_t q = id_to_pos(a, pids[j]) - lo;
    if (q >= 0 && q < n) {
      uint32_t h = ((uint32_t)q * 2654435761u) & hmask;
      while (atomicCAS(&S.hash[h], 0xFFFFFFFFu, (uint32_t)q) != 0xFFFFFFFFu) h = (h + 1u) & hmask;
      if (MODE == kHot) {
        const float x = Elem<T>::get(rowp, q);
        spen += exp(ready_penalized(x, pcnt[j], p) - mrow);
        sraw += (double)hot_exp(x);
      }
    }
  }
  __syncwarp();
  double u[3];
  get_uniforms(a, row, p, u);

  // ---- kHot: alpha and the accept test (shvs.py:223-236)
  double alpha = 1.0;
  bool imprecise = false;
  if (MODE == kHot) {
    const double sH = fmax(0.0, warp_sum(sh) - warp_sum(sraw) + warp_sum(spen));
    double corr = 0.0;
    if (a.summary_raw)
      corr = warp_sum(raw_summary_correction(a, row, p, plen, mrow, lane, 32u,
                                             [&](int64_t pos) { return Elem<T>::get(rowp - lo, pos); }));
    const double S_prod = a.total_expsum[row];
    const double Stot = S_prod + corr;
    imprecise = a.summary_raw && S_prod > 16.0 * Stot;
    const bool tail_empty = a.V == a.H;
    bool degenerate = false;
    if (!tail_empty) {
      if (!(Stot > 0.0) || !isfinite(Stot)) degenerate = true;
      else alpha = fmin(sH / Stot, 1.0);
    }
    const bool accept = !degenerate && sH > 0.0 && (tail_empty || u[1] <= alpha);
    if (!accept) {
      if (lane == 0) {
        uint8_t fl = DP_FLAG_REJECTED;
        if (degenerate || (tail_empty && !(sH > 0.0))) fl |= DP_FLAG_DEGENERATE;
        else if (fabs(u[1] - alpha) < kBoundaryEps || imprecise) fl |= DP_FLAG_NEAR_BOUNDARY;
        a.flags[row] = fl;
        if (a.dbg.alpha) a.dbg.alpha[row] = alpha;
        if (a.dbg.margin) a.dbg.margin[row] = fabs(u[1] - alpha);
        if (a.dbg.bytes_touched) a.dbg.bytes_touched[row] = (uint64_t)n * sizeof(T);
        if (!(fl & DP_FLAG_DEGENERATE)) {
          a.reject_rows[atomicAdd(a.reject_count, 1)] = row;
        } else {
          a.token[row] = -1;
          a.logprob[row] = 0.0;
        }
      }
      return;
    }
  }

  // ---- final list: raw candidates that are not penalized (ready = x/tau),
  // then the penalized ids of the domain (exact f64 penalties)
  uint32_t nl = 0;
  for (uint32_t base = 0; base < cnt; base += 32) {
    const uint32_t i = base + lane;
    const uint64_t key = i < cnt ? S.key[i] : 0ull;
    const uint32_t pos = comp_pos(key);
    bool keep = i < cnt;
    if (keep && plen > 0) {
      uint32_t h = (pos * 2654435761u) & hmask;
      while (true) {
        const uint32_t hv = S.hash[h];
        if (hv == pos) { keep = false; break; }
        if (hv == 0xFFFFFFFFu) break;
        h = (h + 1u) & hmask;
      }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) {
      const uint32_t o = nl + __popc(m & lanemask_lt());
      S.key[o] = f64_key(ready_plain(comp_val(key), p));
      S.pos[o] = pos;
    }
    nl += __popc(m);
    __syncwarp();
  }
  for (int32_t base = 0; base < plen; base += 32) {
    const int32_t j = base + (int32_t)lane;
    int64_t q = -1;
    if (j < plen) q = id_to_pos(a, pids[j]) - lo;
    const bool in = j < plen && q >= 0 && q < n;
    const uint32_t m = __ballot_sync(0xffffffffu, in);
    if (in) {
      const uint32_t o = nl + __popc(m & lanemask_lt());
      S.key[o] = f64_key(ready_penalized(Elem<T>::get(rowp, q), pcnt[j], p));
      S.pos[o] = (uint32_t)q;
    }
    nl += __popc(m);
  }
  __syncwarp();

  // ---- top-k in canonical order, exact filter + draw
  warp_topk_sort(S.key, S.pos, nl, (uint32_t)k, S.hist);
  const uint32_t kk = min((uint32_t)k, nl);
  for (uint32_t i = lane; i < kk; i += 32) {
    const uint64_t key = S.key[i];
    const uint64_t bb = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
    S.fr[i] = __longlong_as_double((long long)bb);
  }
  __syncwarp();
  const DrawResult d = warp_filter_draw_reg(S.fr, (int32_t)kk, p, u[0]);
  if (lane == 0) {
    a.token[row] = pos_to_id(a, (int64_t)S.pos[d.index] + lo);
    a.logprob[row] = d.logprob;
    uint8_t fl = MODE == kHot ? DP_FLAG_ACCEPTED_HOT : 0;
    double margin = d.margin;
    if (MODE == kHot && a.V != a.H) margin = fmin(margin, fabs(u[1] - alpha));
    if (margin < kBoundaryEps || imprecise) fl |= DP_FLAG_NEAR_BOUNDARY;
    a.flags[row] = fl;
    if (a.dbg.margin) a.dbg.margin[row] = margin;
    if (a.dbg.kept) a.dbg.kept[row] = d.kept;
    if (MODE == kHot && a.dbg.alpha) a.dbg.alpha[row] = alpha;
    if (a.dbg.bytes_touched) a.dbg.bytes_touched[row] = (uint64_t)n * sizeof(T);
  }
  if (a.dbg.topk_ids) {
    const int32_t m = min((int32_t)kk, a.dbg.topk_stride);
    for (int32_t j = lane; j < m; j += 32) {
      a.dbg.topk_ids[(int64_t)row * a.dbg.topk_stride + j] = pos_to_id(a, (int64_t)S.pos[j] + lo);
      if (a.dbg.topk_ready) a.dbg.topk_ready[(int64_t)row * a.dbg.topk_stride + j] = S.fr[j];
    }
  }
}

// ---------------------------------------------------------------------------
// host launcher (kFull / kHot; grid covers the call's rows)

template <typename T, int MODE>
static cudaError_t launch_warp_t(const SampleArgs& a, int grid_rows, cudaStream_t st) {
  const int grid = (grid_rows + kWPC - 1) / kWPC;
  warp_sample_kernel<T, MODE><<<grid, kWPC * 32, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_warp(const SampleArgs& a, int dtype, int mode, int grid_rows, cudaStream_t st) {
  if (dtype == DP_F32) {
    return mode == kHot ? launch_warp_t<float, kHot>(a, grid_rows, st) : launch_warp_t<float, kFull>(a, grid_rows, st);
  }
  return mode == kHot ? launch_warp_t<__nv_bfloat16, kHot>(a, grid_rows, st)
                      : launch_warp_t<__nv_bfloat16, kFull>(a, grid_rows, st);
}

}  // namespace dp
