// sample_warp.cu — short-row sampler (K1w): one 4-warp CTA per row with no
// block barrier inside the stream, sm_100a.
//
// For the SHVS hot pass (rows of H <= 64K logits) and other short rows at
// large batch the per-row CTA kernel spends most of its time in
// __syncthreads while one warp sorts / draws.  Here the four warps stream
// disjoint, interleaved quarters of the row into private candidate buffers
// (two CTA barriers per row: thresholds, end of stream), then warp 0 merges
// and decides while the SM's other CTAs keep streaming.  CTAs loop over rows
// when the batch exceeds one wave.
//
// Same decision law as sample_topk.cu (filtering.py:38-162, penalty.py:66-78,
// shvs.py:223-236):
//  1. threshold: the first batch is a strided sample of the row (batch b,
//     slot j of warp w reads vectors ((j*nb + b)*4 + w)*32 + lane); each lane
//     keeps its top-4 sample values and a bitwise search over the CTA's 512
//     values gives t_lb (the kp-th: a proven lower bound of the row's kp-th
//     largest) and t_est (an estimate admitting ~2 kp elements);
//  2. stream: elements >= threshold are appended as unique (value desc,
//     position asc) keys to the warp's 512-entry buffer; a full buffer is cut
//     to its kp largest, which also raises that warp's threshold (exact:
//     nothing below the kp-th largest of a subset can reach the top-kp); fewer
//     than kp survivors over the CTA re-stream with t_lb;
//  3. warp 0: merge, exact top-kp (raw top-(k + |penalty list|), the superset
//     argument of _tail_preselect, service.py:309-336), sparse penalties in
//     IEEE f64, radix cut to the top-k, register sort, exact top-p / min-p /
//     draw.
// kHot accumulates the raw hot mass of every element (f32 exp2 of the
// max-centred argument, pairwise f32 per vector, f64 across vectors) and
// replaces the penalized ids' raw terms by their exact penalized mass: the
// subtracted terms are the bit-identical f32 values that were added, so no
// per-element penalty test is needed.

#include <type_traits>

#include "sampler.cuh"
#include "select.cuh"
#include "finish.cuh"

namespace dp {

constexpr int kWXcap = 512;   // candidate keys per warp buffer (>= kWarpKpMax + one batch of admissions)
constexpr int kWHcap = 512;   // penalty hash slots (>= 2 * kWarpPenCap)
constexpr int kMW = 4;        // warps per row (one CTA per row)
constexpr int kWU = 4;        // 16-byte vectors in flight per lane
constexpr int kMWBlocks = 7;
constexpr int kWQcap = 256;   // admitted-vector queue per warp (>= 32 lanes * kWU)
constexpr int kFLcap = 320;   // final list (k <= 64 cut keys + <= 256 penalized), in the queue area  // resident CTAs per SM the register budget targets (1,024 rows in one wave)

struct MWSmem {
  uint64_t key[kMW * kWXcap];   // warp w streams into key[w*kWXcap ...]; warp 0 merges into key[0 ...]
  uint32_t hist[kMW][256];
  uint32_t q[kMW][kWQcap];      // per-warp queue of admitted vector indices
  uint64_t pkey[kWarpPenCap];   // penalty list: f64 key of the penalized ready value
  int32_t pq[kWarpPenCap];      //   and its domain position (-1: outside the domain)
  uint32_t phash[kWHcap];       // penalized domain positions (open addressing; empty at row start)
  double pm[kMW][3];            // per-warp partials: penalized hot mass, raw hot mass, summary correction
  uint32_t cnt[kMW];
  double sh[kMW];
  float thr[kMW];               // per-warp lower bounds (CTA t_lb = their minimum)
  uint32_t bcast[4];
  uint32_t nl;                  // final list fill
};
// warp 0's final-stage scratch aliases the stream buffers of warps 1..3, which
// are free once the merged list is cut to kp <= kWXcap keys
struct MWFinish {
  double fr[kWarpKMax];
};
static_assert(kWarpPenCap <= 2 * kMW * 32, "two penalty entries per thread");
static_assert(kFLcap * 12 <= kMW * kWQcap * 4, "final list must fit the queue area");
static_assert(sizeof(MWFinish) <= (kMW - 1) * kWXcap * sizeof(uint64_t), "finish scratch must fit");

template <typename T, int MODE>
__global__ void __launch_bounds__(kMW * 32, kMWBlocks) warp_sample_kernel(SampleArgs a) {
  constexpr int EPV = Elem<T>::kPerVec;
  constexpr int U = kWU;
  __shared__ MWSmem S;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const int nrows = a.row_count ? *a.row_count : a.n_rows;
  uint64_t* wkey = S.key + warp * kWXcap;
  MWFinish& F = *reinterpret_cast<MWFinish*>(S.key + kWXcap);
  uint32_t* whist = S.hist[warp];
  // phase profile (debug only): warp 0 lane 0 accumulates clock64 laps into
  // stats[4..7]; stats[21]/[22] = min start / max end globaltimer (ns)
#ifdef DP_PHASE_PROF
  const bool prof = a.dbg.stats != nullptr && threadIdx.x == 0;
#else
  constexpr bool prof = false;   // build with -DDP_PHASE_PROF for the phase profile
#endif
  long long pc = 0;
  auto lap = [&](int slot) {
    if (prof) {
      const long long now = clock64();
      atomicAdd((unsigned long long*)&a.dbg.stats[slot], (unsigned long long)(now - pc));
      pc = now;
    }
  };
  auto gtime = []() -> unsigned long long {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  };
  if (prof) atomicMin((unsigned long long*)&a.dbg.stats[21], gtime());
  for (uint32_t i = threadIdx.x; i < (uint32_t)kWHcap; i += kMW * 32) S.phash[i] = 0xFFFFFFFFu;

  for (int ridx = blockIdx.x; ridx < nrows; ridx += gridDim.x) {
    const int row = a.rows ? a.rows[ridx] : ridx;
    // params are read from global / L1 where used, not held in registers
    // across the stream (register pressure: the stream loop must not spill)
    const dp_params_t& p = a.params[row];
    const int32_t plen = pen_len(a, row, p);
    const int64_t n = dom_n(a, MODE), lo = dom_lo(a, MODE);
    const int32_t k = p.top_k;
    if (route_row(a, MODE, k, plen, n) != kRouteWarp) continue;   // CTA-uniform
    const uint32_t kp = (uint32_t)min64(n, (int64_t)k + plen);
    const T* rowp = domain_row<T>(a, row, MODE);
    const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
    const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;

    // hot mass: exp((x - m tau)/tau) = 2^((x - hi) * log2e/tau - lo * log2e/tau),
    // m tau = hi + lo split so that x - hi is exact near the row maximum
    double mrow = 0.0;
    float m_hi = 0.f, nlo_s2 = 0.f, s2 = 0.f;
    if (MODE == kHot) {
      mrow = a.row_max[row];
      const double c = mrow * p.temperature;
      m_hi = (float)c;
      s2 = (float)(1.4426950408889634 / p.temperature);
      nlo_s2 = -(float)((c - (double)m_hi) * (double)s2);
    }
    auto hot_exp = [&](float x) -> float { return ex2_fast(__fmaf_rn(__fsub_rn(x, m_hi), s2, nlo_s2)); };

    // ---- geometry: 16-byte vectors (32-bit indices, V < 2^31).  Batch b,
    // slot j of warp w reads vectors ((j*nb + b)*kMW + w)*32 + lane, so the
    // first batch is a strided sample of the whole row.
    const uintptr_t addr = reinterpret_cast<uintptr_t>(rowp);
    const int32_t a0 = (int32_t)min64(n, (int64_t)(((16u - (addr & 15u)) & 15u) / sizeof(T)));
    const int32_t nvec = (int32_t)((n - a0) / EPV);
    const int32_t tail0 = a0 + nvec * EPV;
    const int32_t nb = max(1, (nvec + kMW * 32 * U - 1) / (kMW * 32 * U));
    const uint4* vp = reinterpret_cast<const uint4*>(rowp + a0);
    const int32_t wl = (int32_t)(warp * 32u + lane);
    auto vidx = [&](int32_t b, int j) -> int32_t { return (j * nb + b) * (kMW * 32) + wl; };

    __syncthreads();   // the previous row's finish (warp 0) is done with the shared buffers
    if (prof) pc = clock64();
    uint4 v[U];
    const int32_t stride = nb * (kMW * 32);
    // load vectors [J0, J0 + UH) of batch b (the register file holds one batch;
    // the halves are refilled in turn so a half is always in flight while the
    // other is consumed)
    constexpr int UH = U / 2;
    auto load_half = [&](int32_t b, auto j0c) {
      constexpr int J0 = decltype(j0c)::value;
      const int32_t base = b * (kMW * 32) + wl;
      if (b * (kMW * 32) + (kMW * 32 - 1) + (J0 + UH - 1) * stride < nvec) {   // CTA-uniform: all valid
#pragma unroll
        for (int j = J0; j < J0 + UH; ++j) v[j] = ld_stream16(vp + base + j * stride);
      } else {
#pragma unroll
        for (int j = J0; j < J0 + UH; ++j) {
          const int32_t idx = base + j * stride;
          v[j] = idx < nvec ? ld_stream16(vp + idx) : neg_inf_vec<T>();
        }
      }
    };
    using H0 = std::integral_constant<int, 0>;
    using H1 = std::integral_constant<int, UH>;
    load_half(0, H0{});
    load_half(0, H1{});
    // penalty list ids -> absolute row positions, fetched while the first
    // batch is in flight (consumed after the stream; kWarpPenCap = 2 * 128)
    int32_t pa_r[2] = {-1, -1}, pc_r[2] = {0, 0};
    float px_r[2] = {0.f, 0.f};   // their raw logits, gathered during the stream too
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int32_t j = (int32_t)threadIdx.x + i * kMW * 32;
      if (j < plen) {
        pa_r[i] = (int32_t)id_to_pos(a, pids[j]);
        pc_r[i] = pcnt[j];
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
      if (pa_r[i] >= 0) px_r[i] = row_value<T>(a, row, pa_r[i]);

    // ---- threshold from the strided first batch: each lane keeps its top-2
    // sample values; warp w takes the ceil(kp/4)-th largest of its 64 kept
    // values, so >= ceil(kp/4) row elements reach it; the minimum over the 4
    // warps is reached by >= kp elements: a proven lower bound t_lb of the
    // row's kp-th largest, used directly for admission (no re-stream)
    {
      float t1 = -INFINITY, t2 = -INFINITY;
#pragma unroll
      for (int j = 0; j < U; ++j) {
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          const float x = vec_elem<T>(v[j], e);
          t2 = fmaxf(t2, fminf(t1, x));
          t1 = fmaxf(t1, x);
        }
      }
      // padding lanes hold -inf, which only lowers the bound (safe)
      const uint32_t r = (kp + kMW - 1) / kMW;
      const uint32_t k1 = f32_key(t1), k2 = f32_key(t2);
      uint32_t tk = 0u;
      if (r <= 64u) {
        for (int bit = 31; bit >= 0; --bit) {
          const uint32_t c = tk | (1u << bit);
          const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, k1 >= c)) + __popc(__ballot_sync(0xffffffffu, k2 >= c));
          if (cnt >= r) tk = c;
        }
      }
      if (lane == 0) S.thr[warp] = tk > f32_key(-INFINITY) ? key_f32(tk) : -INFINITY;
    }
    __syncthreads();
    lap(4);
    float t_lb = S.thr[0];
#pragma unroll
    for (int w = 1; w < kMW; ++w) t_lb = fminf(t_lb, S.thr[w]);
    const float t_est = t_lb;

    // ---- stream
    float thr_f = t_est;
    uint64_t thr_k = thr_f == -INFINITY ? 0ull : ((uint64_t)f32_key(thr_f) << 32);
    uint32_t cnt = 0;     // warp-uniform buffer fill
    double sh = 0.0;      // kHot: raw hot mass of this lane's elements
    // cut the warp buffer to its kp largest keys; raises the admission threshold
    // (exact: nothing below the kp-th largest of a subset can reach the top-kp)
    auto cut = [&]() {
      __syncwarp();
      const uint64_t t = warp_select_threshold(wkey, cnt, kp, whist);
      cnt = warp_compact(wkey, cnt, t);
      if (t > thr_k) {
        thr_k = t;
        thr_f = comp_val(t);
      }
    };
    // append this lane's admitted keys (mask m over ks[0..nk))
    auto append = [&](uint32_t m, const uint64_t* ks, int nk) {
      const uint32_t c = __popc(m);
      const uint32_t incl = warp_incl_scan(c);
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      uint32_t o = cnt + incl - c;
      for (int e = 0; e < nk; ++e)
        if ((m >> e) & 1u) wkey[o++] = ks[e];
      cnt += tot;
    };
    // queued vectors -> exact keys: one queued vector per lane per round
    // (re-read from L2), unique (value, position) keys >= thr_k appended
    uint32_t* wq = S.q[warp];
    uint32_t qn = 0;   // warp-uniform queue fill
    // R rounds of 32 queued vectors are loaded together (R > 1 only where the
    // stream registers are free, i.e. after the last batch)
    auto flush_r = [&](auto rc) {
      constexpr int R = decltype(rc)::value;
      __syncwarp();
      for (uint32_t base = 0; base < qn; base += 32 * R) {
        uint4 vv[R];
        int32_t idx[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t i = base + 32u * r + lane;
          idx[r] = i < qn ? (int32_t)wq[i] : -1;
          vv[r] = idx[r] >= 0 ? __ldg(vp + idx[r]) : neg_inf_vec<T>();
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (base + 32u * r >= qn) break;   // warp-uniform
          const bool has = idx[r] >= 0;
          uint64_t ks[EPV];
          uint32_t m = 0;
#pragma unroll
          for (int e = 0; e < EPV; ++e) {
            ks[e] = comp_key(vec_elem<T>(vv[r], e), (uint32_t)(a0 + idx[r] * EPV + e));
            if (has && ks[e] >= thr_k) m |= 1u << e;
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
      }
      qn = 0;
      __syncwarp();
    };
    auto flush = [&]() { flush_r(std::integral_constant<int, 1>{}); };
    // vectors [J0, J0 + UH) of batch b: hot mass (first pass) + per-vector
    // admission test (vector max >= threshold) -> queue of vector indices
    auto consume_half = [&](int32_t b, bool first_pass, auto j0c) {
      constexpr int J0 = decltype(j0c)::value;
      const int32_t base = b * (kMW * 32) + wl;
      uint32_t vm = 0;
      float bs[UH];
#pragma unroll
      for (int jj = 0; jj < UH; ++jj) {
        const int j = J0 + jj;
        float mx = vec_elem<T>(v[j], 0);
#pragma unroll
        for (int e = 1; e < EPV; ++e) mx = fmaxf(mx, vec_elem<T>(v[j], e));
        vm |= (mx >= thr_f ? 1u : 0u) << jj;
        if (MODE == kHot && first_pass) {   // padding vectors are -inf: exp = 0
          float e4[EPV];
#pragma unroll
          for (int e = 0; e < EPV; ++e) e4[e] = hot_exp(vec_elem<T>(v[j], e));
#pragma unroll
          for (int st = 1; st < EPV; st <<= 1)
#pragma unroll
            for (int e = 0; e < EPV; e += 2 * st) e4[e] += e4[e + st];
          bs[jj] = e4[0];
        }
      }
      if (MODE == kHot && first_pass) {
#pragma unroll
        for (int st = 1; st < UH; st <<= 1)
#pragma unroll
          for (int jj = 0; jj < UH; jj += 2 * st) bs[jj] += bs[jj + st];
        sh += (double)bs[0];
      }
      if (thr_f == -INFINITY) {   // padding would pass: keep valid vectors only
#pragma unroll
        for (int jj = 0; jj < UH; ++jj)
          if (base + (J0 + jj) * stride >= nvec) vm &= ~(1u << jj);
      }
      if (!__any_sync(0xffffffffu, vm != 0u)) return;
      const uint32_t c = __popc(vm);
      const uint32_t incl = warp_incl_scan(c);
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      if (qn + tot > (uint32_t)kWQcap) flush();
      uint32_t o = qn + incl - c;
      for (uint32_t mm = vm; mm; mm &= mm - 1u) wq[o++] = (uint32_t)(base + (J0 + __ffs(mm) - 1) * stride);
      qn += tot;
    };
    int npass = 0;
    for (int pass_no = 0;; ++pass_no) {
      const bool first = pass_no == 0;
      npass = pass_no + 1;
      if (warp == 0) {   // scalar head / tail elements (at most 2*EPV-2)
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
      if (!first) {   // re-stream: reload the first batch
        load_half(0, H0{});
        load_half(0, H1{});
      }
      for (int32_t b = 0; b < nb; ++b) {
        consume_half(b, first, H0{});
        if (b + 1 < nb) load_half(b + 1, H0{});
        consume_half(b, first, H1{});
        if (b + 1 < nb) load_half(b + 1, H1{});
      }
      lap(8);
      flush_r(std::integral_constant<int, 4>{});
      lap(9);
      if (lane == 0) S.cnt[warp] = cnt;
      __syncthreads();
      uint32_t total = 0;
#pragma unroll
      for (int w = 0; w < kMW; ++w) total += S.cnt[w];
      // a cut leaves kp keys in its warp, so total < kp means no warp cut and
      // every warp still admits with t_est (the decision is CTA-uniform)
      if (total >= kp || thr_f <= t_lb) break;
      // the estimate was too high: re-stream with the proven bound
      thr_f = t_lb;
      thr_k = t_lb == -INFINITY ? 0ull : ((uint64_t)f32_key(t_lb) << 32);
      cnt = 0;
      if (a.dbg.stats && threadIdx.x == 0) atomicAdd((unsigned long long*)&a.dbg.stats[1], 1ull);
      __syncthreads();   // everyone has read S.cnt before it is rewritten
    }
    if (MODE == kHot) {
      const double s = warp_sum(sh);
      if (lane == 0) S.sh[warp] = s;
    }
    // every pass loads the row's vectors once plus its scalar head / tail;
    // the penalty values are gathered once below
    if (threadIdx.x == 0)
      touch_bytes(a, row, (uint64_t)npass * ((uint64_t)nvec * 16u + (uint64_t)(a0 + (n - tail0)) * sizeof(T)) +
                              (uint64_t)plen * sizeof(T));
    __syncthreads();
    lap(5);
    // ---- penalty list (after the stream: the row and the id maps are L2-hot;
    // keeping it out of the stream loop keeps that loop free of spills):
    // domain positions into a shared hash set, exact f64 ready values as keys,
    // and the kHot mass terms
    uint32_t hcap = 32;
    while (hcap < 2u * (uint32_t)plen) hcap <<= 1;
    const uint32_t hmask = hcap - 1u;
    {
      double spen = 0.0, sraw = 0.0, corr = 0.0;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int32_t j = (int32_t)threadIdx.x + i * kMW * 32;
        if (j >= plen) continue;
        const int64_t pa = pa_r[i];   // absolute row position
        const int64_t q = pa - lo;
        const bool in = q >= 0 && q < n;
        const float x = px_r[i];
        const double r = ready_penalized(x, pc_r[i], p);
        S.pq[j] = in ? (int32_t)q : -1;
        S.pkey[j] = f64_key(r);
        if (in) {
          uint32_t h = ((uint32_t)q * 2654435761u) & hmask;
          while (atomicCAS(&S.phash[h], 0xFFFFFFFFu, (uint32_t)q) != 0xFFFFFFFFu) h = (h + 1u) & hmask;
        }
        if (MODE == kHot) {
          const double ep = exp(r - mrow);
          if (in) {
            spen += ep;
            sraw += (double)hot_exp(x);   // bit-identical to the streamed term
          }
          // raw producer summary: S = S_raw + sum_j [exp(r_j - m) - exp(x_j/tau - m)]
          if (a.summary_raw) corr += ep - exp(ready_plain(x, p) - mrow);
        }
      }
      if (MODE == kHot) {
        spen = warp_sum(spen);
        sraw = warp_sum(sraw);
        corr = warp_sum(corr);
        if (lane == 0) {
          S.pm[warp][0] = spen;
          S.pm[warp][1] = sraw;
          S.pm[warp][2] = corr;
        }
      }
    }

    __syncthreads();
    lap(10);
    // ---- decision inputs, evaluated by every thread (CTA-uniform)
    double u[3];
    get_uniforms(a, row, p, u);
    double alpha = 1.0, sH = 0.0;
    bool deferred = false;   // accept test left to the exact re-sum (defer_accept)
    if (MODE == kHot) {   // alpha and the accept test (shvs.py:223-236)
      double sh_row = 0.0, spen = 0.0, sraw = 0.0, corr = 0.0;
#pragma unroll
      for (int w = 0; w < kMW; ++w) {   // fixed order: deterministic
        sh_row += S.sh[w];
        spen += S.pm[w][0];
        sraw += S.pm[w][1];
        corr += S.pm[w][2];
      }
      sH = fmax(0.0, sh_row - sraw + spen);
      const double S_prod = a.total_expsum[row];
      const double Stot = S_prod + corr;
      const bool tail_empty = a.V == a.H;
      bool degenerate = false;
      if (!tail_empty) {
        if (!(Stot > 0.0) || !isfinite(Stot)) degenerate = true;
        else alpha = fmin(sH / Stot, 1.0);
      }
      deferred = sH > 0.0 && defer_accept(a, S_prod, Stot, alpha, u[1]);
      const bool accept = deferred || (!degenerate && sH > 0.0 && (tail_empty || u[1] <= alpha));
      if (!accept) {
        if (threadIdx.x == 0) {
          uint8_t fl = DP_FLAG_REJECTED;
          if (degenerate || (tail_empty && !(sH > 0.0))) fl |= DP_FLAG_DEGENERATE;
          else if (fabs(u[1] - alpha) < kBoundaryEps) fl |= DP_FLAG_NEAR_BOUNDARY;
          a.flags[row] = fl;
          if (a.dbg.alpha) a.dbg.alpha[row] = alpha;
          if (a.dbg.margin) a.dbg.margin[row] = fabs(u[1] - alpha);
          if (!(fl & DP_FLAG_DEGENERATE)) {
            a.reject_rows[atomicAdd(a.reject_count, 1)] = row;
          } else {
            a.token[row] = -1;
            a.logprob[row] = 0.0;
          }
        }
        for (uint32_t i = threadIdx.x; i < hcap; i += kMW * 32) S.phash[i] = 0xFFFFFFFFu;   // empty for the next row
        continue;
      }
    }

    // ---- 1. every warp drops the penalized ids from its buffer (in place)
    if (a.dbg.stats && lane == 0) atomicAdd((unsigned long long*)&a.dbg.stats[3], (unsigned long long)cnt);
    if (plen > 0) {
      uint32_t out = 0;
      for (uint32_t base = 0; base < cnt; base += 32) {
        const uint32_t i = base + lane;
        const uint64_t key = i < cnt ? wkey[i] : 0ull;
        const uint32_t pos = comp_pos(key);
        bool keep = i < cnt;
        if (keep) {
          uint32_t h = (pos * 2654435761u) & hmask;
          while (true) {
            const uint32_t hv = S.phash[h];
            if (hv == pos) { keep = false; break; }
            if (hv == 0xFFFFFFFFu) break;
            h = (h + 1u) & hmask;
          }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) wkey[out + __popc(m & lanemask_lt())] = key;
        out += __popc(m);
        __syncwarp();
      }
      cnt = out;
    }
    if (lane == 0) S.cnt[warp] = cnt;
    if (threadIdx.x == 0) S.nl = 0u;
    __syncthreads();
    lap(11);

    // ---- 2. CTA-level exact cut: the k largest unpenalized raw keys.  Their
    // ready values keep the raw order, so together with the penalized ids they
    // contain the ready top-k (superset argument of _tail_preselect,
    // service.py:309-336; every raw top-(k + |list|) element was admitted)
    const uint32_t c0 = S.cnt[0], c1 = c0 + S.cnt[1], c2 = c1 + S.cnt[2], ctot = c2 + S.cnt[3];
    auto get_u = [&](uint32_t i, uint64_t& key) -> bool {
      const uint32_t w = i < c0 ? 0u : (i < c1 ? 1u : (i < c2 ? 2u : 3u));
      const uint32_t b0 = w == 0u ? 0u : (w == 1u ? c0 : (w == 2u ? c1 : c2));
      key = S.key[w * kWXcap + (i - b0)];
      return true;
    };
    const uint64_t tk = group_select_threshold<kMW * 32>(get_u, ctot, ctot, (uint32_t)k, S.hist[0], S.bcast,
                                                          threadIdx.x, [] { __syncthreads(); });
    lap(23);

    // ---- 3. final list (in the now free queue area): those keys as exact f64
    // ready keys, plus the penalized ids of the domain with their exact keys
    uint64_t* fkey = reinterpret_cast<uint64_t*>(&S.q[0][0]);
    uint32_t* fpos = reinterpret_cast<uint32_t*>(fkey + kFLcap);
    for (uint32_t i = lane; i < cnt; i += 32) {
      const uint64_t key = wkey[i];
      if (key >= tk) {
        const uint32_t o = atomicAdd(&S.nl, 1u);
        fkey[o] = f64_key(ready_plain(comp_val(key), p));
        fpos[o] = comp_pos(key);
      }
    }
    // a penalized id can enter the ready top-k only if it reaches the k-th
    // unpenalized candidate's ready value (ties kept: the sort breaks them)
    const uint64_t pk_thr = (tk == 0ull || ctot < (uint32_t)k) ? 0ull : f64_key(ready_plain(comp_val(tk), p));
    for (int32_t j = (int32_t)threadIdx.x; j < plen; j += kMW * 32) {
      const int32_t q = S.pq[j];
      if (q >= 0 && S.pkey[j] >= pk_thr) {
        const uint32_t o = atomicAdd(&S.nl, 1u);
        fkey[o] = S.pkey[j];
        fpos[o] = (uint32_t)q;
      }
    }
    __syncthreads();
    lap(6);
    if (warp != 0) {
      for (uint32_t i = threadIdx.x - 32u; i < hcap; i += (kMW - 1) * 32) S.phash[i] = 0xFFFFFFFFu;   // next row
      continue;
    }

    // ---- 4. warp 0: top-k in canonical order, exact filter + draw
    const uint32_t nl = S.nl;
    warp_topk_sort(fkey, fpos, nl, (uint32_t)k, S.hist[0]);
    const uint32_t kk = min((uint32_t)k, nl);
    for (uint32_t i = lane; i < kk; i += 32) {
      const uint64_t key = fkey[i];
      const uint64_t bb = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
      F.fr[i] = __longlong_as_double((long long)bb);
    }
    __syncwarp();
    if (!(kk > 0 && F.fr[0] > -INFINITY)) {   // no usable mass (DegenerateRowError, core.py:19-20)
      if (lane == 0) {
        a.token[row] = -1;
        a.logprob[row] = 0.0;
        a.flags[row] = DP_FLAG_DEGENERATE;
      }
      continue;
    }
    const DrawResult d = warp_filter_draw_reg(F.fr, (int32_t)kk, knobs_of(p), u[0]);
    lap(7);
    if (prof) atomicMax((unsigned long long*)&a.dbg.stats[22], gtime());
    if (lane == 0) {
      a.token[row] = pos_to_id(a, (int64_t)fpos[d.index] + lo);
      a.logprob[row] = d.logprob;
      uint8_t fl = MODE == kHot ? DP_FLAG_ACCEPTED_HOT : 0;
      double margin = d.margin;
      if (MODE == kHot && a.V != a.H && !deferred) margin = fmin(margin, fabs(u[1] - alpha));
      if (margin < kBoundaryEps) fl |= DP_FLAG_NEAR_BOUNDARY;
      a.flags[row] = fl;
      if (a.dbg.margin) a.dbg.margin[row] = margin;
      if (a.dbg.kept) a.dbg.kept[row] = d.kept;
      if (MODE == kHot && a.dbg.alpha) a.dbg.alpha[row] = alpha;
      if (a.dbg.stats) atomicAdd((unsigned long long*)&a.dbg.stats[0], 1ull);
    }
    if (deferred) {
      if (lane == 0) push_resum(a, row, sH);   // the exact re-sum decides, then records
    } else {
      warp_record_token(a, row, pos_to_id(a, (int64_t)fpos[d.index] + lo));   // fused K5
    }
    if (a.dbg.topk_ids) {
      const int32_t m = min((int32_t)kk, a.dbg.topk_stride);
      for (int32_t j = lane; j < m; j += 32) {
        a.dbg.topk_ids[(int64_t)row * a.dbg.topk_stride + j] = pos_to_id(a, (int64_t)fpos[j] + lo);
        if (a.dbg.topk_ready) a.dbg.topk_ready[(int64_t)row * a.dbg.topk_stride + j] = F.fr[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host launcher (kFull / kHot; grid covers the call's rows)

template <typename T, int MODE>
static cudaError_t launch_warp_t(const SampleArgs& a, int grid_rows, cudaStream_t st) {
  // one CTA per row while they fit in one wave; beyond that CTAs loop over rows
  static int max_grid = 0;
  if (max_grid == 0) {
    int dev = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, warp_sample_kernel<T, MODE>, kMW * 32, 0) !=
            cudaSuccess || per_sm < 1)
      per_sm = 1;
    max_grid = sms * per_sm;
  }
  const int grid = grid_rows < max_grid ? grid_rows : max_grid;
  if (grid < 1) return cudaSuccess;
  warp_sample_kernel<T, MODE><<<grid, kMW * 32, 0, st>>>(a);
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
