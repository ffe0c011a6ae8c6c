// sampler.cuh — shared per-row decision logic: domain description, penalty
// entries, and the exact filter/draw over a sorted candidate list
// (filtering.py:61-162 at tau_eff = 1).
#pragma once

#include "common.cuh"

namespace dp {

enum Mode : int { kFull = 0, kHot = 1, kTail = 2 };
// Admission threshold estimate of the streaming top-k kernels: the first
// batch's sample estimates the (est * kp)-th largest of the segment.  A
// too-high estimate (fewer than kp admitted) costs a whole re-stream of the
// row, which the C2 distribution hits at est = 2 (1,000 steps: 150 vs 131 us
// at est = 4); every extra admission costs select work, which nucleus rows
// (kp >= 256) pay for at est = 4 (C5 full path 2.42 vs 2.75 ms;
// profiles/r2/est_over_ab.txt).
DP_DEV float est_over(uint32_t kp, bool nucleus) {
  (void)kp;
  return nucleus ? 2.0f : 4.0f;
}
constexpr int kHotSortMax = 4096;   // SHVS hot prefixes up to this size take K1h (sample_hot.cu)
constexpr int kMaxShards = 8;

struct SampleArgs {
  const void* logits;
  int64_t ld, V, H;             // H = hot size (kHot/kTail), V for kFull
  const int32_t* perm;          // position -> token id (NULL = identity)
  const int32_t* inv_perm;      // token id -> position (NULL = identity)
  const dp_params_t* params;
  dp_penalty_t pen;
  const double* uniforms;       // [B,3] or NULL (derive from seeds)
  const uint64_t* seq_ids;
  uint64_t iteration;
  const double* row_max;        // producer summary (kHot)
  const double* total_expsum;
  int32_t* rows;                // row list (kTail: reject list) or NULL
  int32_t* row_count;           // device count for `rows` (kTail) or NULL
  int32_t n_rows;               // host row count when row_count == NULL
  int32_t* token;
  double* logprob;
  uint8_t* flags;
  dp_debug_t dbg;
  int32_t* reject_rows;         // kHot: rows appended on rejection
  int32_t* reject_count;
  int32_t wcap, kcap, lcap, split;
  int32_t nt;                   // threads per CTA of the top-k kernel (128 / 256)
  int32_t summary_raw;          // kHot: row_max/total_expsum are the producer's raw summary
  int32_t use_warp;             // this call runs the warp-per-row kernel (sample_warp.cu)
  const void* tail_logits;      // split SHVS storage: positions [H, V) of row b at
  int64_t tail_ld;              //   tail_logits + b * tail_ld (device or mapped host memory)
  int32_t* fb_rows;             // nucleus rows whose kept set left the candidate list:
  int32_t* fb_count;            //   appended here for the general kernel (NULL: none routed)
  int32_t force_general;        // the general kernel decides every listed row
  int32_t update_pen;           // record each decided token in the penalty state (fused K5)
  // TP-sharded kFull rows (nshard > 0): vocab shard s = positions
  // [s * shard_n, (s + 1) * shard_n) of row b at shard[s] + b * ld, read in
  // place by cluster rank s of the top-k kernel (split == nshard)
  const void* shard[kMaxShards];
  int64_t shard_n;
  int32_t nshard;
  int32_t shard_per_cta;        // shards one CTA streams (nshard = split * shard_per_cta)
  // kHot with a raw producer summary: rows whose accept test the cancelling
  // correction cannot decide are listed here (hot decision written, penalty
  // update withheld) and re-decided by the exact re-sum (resum_kernel)
  int32_t* resum_rows;
  int32_t* resum_count;
  double* resum_sh;             // [B] the row's hot mass S_H (relative to row_max)
  int32_t force_resum;          // DP_PLAN_FORCE_RESUM (test hook)
  int32_t use_hot_sort;         // kHot: 1 = nucleus rows go to K1h (sample_hot.cu), 2 = every row
  int32_t pen_excl;             // kFull / kTail: penalized ids leave the streaming selection
                                //   (shared bitmap, kp = k) — long penalty lists (finish.cuh)
};
// penalty lists longer than this stream with the penalized ids excluded
// (pen_excl) instead of widening the selection to k + |list|
constexpr int kPenExclMin = 256;
// the streaming kernel keeps at most this many penalized candidates per row
// for its final merge (the best ones by ready value; finish.cuh)
constexpr int kPenSelCap = 256;

// upper bound of the penalty-list length over the call's rows (sizes lists)
__host__ __device__ inline int32_t pen_bound(const dp_penalty_t& pen) {
  return (pen.max_len > 0 && pen.max_len < pen.cap) ? pen.max_len : pen.cap;
}

DP_DEV int64_t dom_lo(const SampleArgs& a, int mode) { return mode == kTail ? a.H : 0; }
DP_DEV int64_t dom_n(const SampleArgs& a, int mode) {
  return mode == kFull ? a.V : (mode == kHot ? a.H : a.V - a.H);
}
// the row's domain [dom_lo, dom_lo + dom_n) as a pointer to its first element
template <typename T>
DP_DEV const T* domain_row(const SampleArgs& a, int row, int mode) {
  if (mode == kTail && a.tail_logits) return reinterpret_cast<const T*>(a.tail_logits) + (int64_t)row * a.tail_ld;
  return reinterpret_cast<const T*>(a.logits) + (int64_t)row * a.ld + dom_lo(a, mode);
}
// VisitCounter (instrument.py:6-33) on the device: bytes this launch loaded
// for `row` — every streaming pass (re-streams included), scalar head / tail
// elements and gathered penalty values — accumulated per row across the
// kernels of one call (the host zeroes the counters before a debug call).
DP_DEV void touch_bytes(const SampleArgs& a, int row, uint64_t bytes) {
  if (a.dbg.bytes_touched && bytes)
    atomicAdd(reinterpret_cast<unsigned long long*>(a.dbg.bytes_touched + row), (unsigned long long)bytes);
}

// raw logit at an absolute row position (either storage)
template <typename T>
DP_DEV float row_value(const SampleArgs& a, int row, int64_t pos) {
  if (a.tail_logits && pos >= a.H)
    return Elem<T>::get(reinterpret_cast<const T*>(a.tail_logits) + (int64_t)row * a.tail_ld, pos - a.H);
  return Elem<T>::get(reinterpret_cast<const T*>(a.logits) + (int64_t)row * a.ld, pos);
}
// raw logit at domain position q of a row whose domain starts at rowp
// (TP-sharded kFull rows: the owning shard's element)
template <typename T>
DP_DEV float dom_value(const SampleArgs& a, int row, const T* rowp, int64_t q) {
  if (a.nshard > 0) {
    const int64_t s = q / a.shard_n;
    return Elem<T>::get(reinterpret_cast<const T*>(a.shard[s]) + (int64_t)row * a.ld, q - s * a.shard_n);
  }
  return Elem<T>::get(rowp, q);
}
DP_DEV int32_t pos_to_id(const SampleArgs& a, int64_t pos) {
  return a.perm ? __ldg(a.perm + pos) : (int32_t)pos;
}
DP_DEV int64_t id_to_pos(const SampleArgs& a, int32_t id) {
  return a.inv_perm ? (int64_t)__ldg(a.inv_perm + id) : (int64_t)id;
}
DP_DEV void get_uniforms(const SampleArgs& a, int row, const dp_params_t& p, double u[3]) {
  if (a.uniforms) {
    u[0] = a.uniforms[3 * (int64_t)row];
    u[1] = a.uniforms[3 * (int64_t)row + 1];
    u[2] = a.uniforms[3 * (int64_t)row + 2];
  } else {
    row_uniforms(p.seed, a.iteration, a.seq_ids[row], u);
  }
}
// number of penalty entries that can change values for this row
DP_DEV int32_t pen_len(const SampleArgs& a, int row, const dp_params_t& p) {
  return penalties_neutral(p) ? 0 : a.pen.len[row];
}

// ---------------------------------------------------------------------------
// update_output_histogram (penalty.py:18-32) fused into the kernel that
// decides the row: C_o[tok] += 1, a first-seen id is appended.  The row's list
// is read by no other kernel of the call after its decision (SHVS tail and
// fallback passes only see rows the first pass left undecided).
DP_DEV void record_token_hit(const SampleArgs& a, int row, int32_t tok, int32_t hit, int32_t len) {
  int32_t* ids = a.pen.ids + (int64_t)row * a.pen.cap;
  int32_t* cnt = a.pen.out_count + (int64_t)row * a.pen.cap;
  if (hit >= 0) {
    cnt[hit] += 1;
  } else if (len < a.pen.cap) {
    ids[len] = tok;
    cnt[len] = 1;
    a.pen.len[row] = len + 1;
  } else {
    a.flags[row] |= DP_FLAG_PEN_OVERFLOW;
  }
}
// one warp (all lanes, tok uniform)
DP_DEV void warp_record_token(const SampleArgs& a, int row, int32_t tok) {
  if (!a.update_pen || tok < 0) return;
  const uint32_t lane = lane_id();
  const int32_t* ids = a.pen.ids + (int64_t)row * a.pen.cap;
  const int32_t len = a.pen.len[row];
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
  if (lane == 0) record_token_hit(a, row, tok, hit, len);
  __syncwarp();
}
// one thread
DP_DEV void thread_record_token(const SampleArgs& a, int row, int32_t tok) {
  if (!a.update_pen || tok < 0) return;
  const int32_t* ids = a.pen.ids + (int64_t)row * a.pen.cap;
  const int32_t len = a.pen.len[row];
  int32_t hit = -1;
  for (int32_t j = 0; j < len; ++j)
    if (ids[j] == tok) { hit = j; break; }
  record_token_hit(a, row, tok, hit, len);
}

// ---------------------------------------------------------------------------
// Row routing: every row of a call is decided by exactly one kernel.
//  * warp-per-row kernel (short top-k, sample_warp.cu) when the call uses it;
//  * per-row CTA / cluster streaming top-k kernel (sample_topk.cu);
//  * general radix kernel (no top-k / oversized lists, sample_general.cu).
enum Route : int { kRouteGeneral = 0, kRouteTopk = 1, kRouteWarp = 2, kRouteHotSort = 3 };
// Rows with top-k off (top-p only, min-p only, neutral) take the top-k kernel
// as "nucleus" rows: it keeps the exact kNucK largest ready values plus the
// mass of the whole domain, and decides the row when the kept set (and the
// draw) lies inside that list — the usual case for LLM distributions.
// Otherwise the row goes to the general kernel (fb_rows).
constexpr int kNucK = 256;
DP_DEV bool nucleus_row(int32_t k, int64_t n) { return k <= 0 || (int64_t)k >= n; }
DP_DEV int32_t effective_k(int32_t k, int64_t n) {
  return nucleus_row(k, n) ? (int32_t)min64(n, (int64_t)kNucK) : k;
}
constexpr int kWarpKMax = 64;     // top_k limit of the warp kernel
constexpr int kWarpKpMax = 256;   // raw candidates kept (k + penalty list)
constexpr int kWarpPenCap = 256;  // penalty-list capacity it can hash

DP_DEV bool warp_row_ok(const SampleArgs& a, int32_t k, int32_t plen, int64_t n) {
  return k > 0 && (int64_t)k < n && k <= kWarpKMax && min64(n, (int64_t)k + plen) <= kWarpKpMax &&
         plen <= kWarpPenCap;
}
DP_DEV int route_row(const SampleArgs& a, int mode, int32_t k, int32_t plen, int64_t n) {
  if (mode == kHot && (a.use_hot_sort == 2 || (a.use_hot_sort == 1 && nucleus_row(k, n)))) return kRouteHotSort;
  if (a.force_general) return kRouteGeneral;
  if (a.use_warp && warp_row_ok(a, k, plen, n)) return kRouteWarp;
  if (nucleus_row(k, n)) {
    if (!a.fb_rows || (int64_t)kNucK * 2 > n) return kRouteGeneral;   // no fallback list / short domain
    k = kNucK;
  }
  const bool excl = mode == kHot || a.pen_excl;
  const uint32_t kp = (uint32_t)min64(n, (int64_t)k + (excl ? 0 : plen));
  // the final stage holds k + 2 |list| entries, or (penalized ids excluded
  // from the stream) at most the k + kPenSelCap best ones
  const int32_t pl = (excl && plen > kPenSelCap) ? kPenSelCap : plen;
  if (k > 0 && (int64_t)k < n && kp <= (uint32_t)a.kcap && (uint32_t)(k + 2 * pl) <= (uint32_t)a.lcap)
    return kRouteTopk;
  return kRouteGeneral;
}

// Total mass S of the ready row relative to `mrow` when the producer summary is
// raw (no penalties): S = S_raw + sum over the penalty list of
// [exp(r_j - m) - exp(x_j/tau - m)], exact f64 per entry.  Runs on NT threads
// (index t), returns the per-thread partial of the correction; `x_at` reads a
// raw logit at an absolute row position.  The caller reduces the partials.
template <typename XAt>
DP_DEV double raw_summary_correction(const SampleArgs& a, int row, const dp_params_t& p, int32_t plen, double mrow,
                                     uint32_t t, uint32_t nt, XAt x_at) {
  const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
  const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;
  double c = 0.0;
  for (int32_t j = t; j < plen; j += nt) {
    const float x = x_at(id_to_pos(a, pids[j]));
    c += exp(ready_penalized(x, pcnt[j], p) - mrow) - exp(ready_plain(x, p) - mrow);
  }
  return c;
}

// ---------------------------------------------------------------------------
// SHVS accept test against a RAW producer summary (plan->summary_raw): the
// ready total is S = S_prod + corr, where S_prod (the producer's sum of f32
// exp terms, relative error <= kRawSumRelErr) may hold mostly mass that the
// penalties have since removed.  The computed alpha = S_H / S then carries an
// absolute error up to kRawSumRelErr * alpha * S_prod / S.  Whenever that
// exceeds the 1e-6 decision band and the draw u_accept lies inside it — or S
// came out non-positive — the accept test is deferred to an exact re-sum of
// the penalized row (resum_kernel, summary.cu); every other row is decided
// here (a decision inside the band is flagged NEAR_BOUNDARY as usual).
constexpr double kRawSumRelErr = 1e-6;
DP_DEV bool defer_accept(const SampleArgs& a, double S_prod, double S, double alpha, double u_accept) {
  if (!a.summary_raw || a.resum_rows == nullptr || a.V == a.H) return false;
  if (!(S > 0.0) || !isfinite(S) || a.force_resum) return true;
  const double err = kRawSumRelErr * fmax(alpha, 1e-300) * (fabs(S_prod) / S);
  return err > kBoundaryEps && fabs(u_accept - alpha) <= err;
}
DP_DEV void push_resum(const SampleArgs& a, int row, double sH) {
  a.resum_sh[row] = sH;
  a.resum_rows[atomicAdd(a.resum_count, 1)] = row;
}

// ---------------------------------------------------------------------------
// Exact filter + inverse-CDF draw over candidates already sorted by
// (ready desc, pos asc): _filter_core / filtered_draw / categorical_draw.
// Executed by ONE warp.  r[0..n) ready values (f64, sorted), n >= 1;
// `k` = number of candidates entering the top-p / min-p stages (the top-k
// set, or the whole domain when top-k is off).  w / cum are scratch [n].
// the filter knobs a draw needs, passed by value: a `const dp_params_t&`
// argument of a non-inlined draw would force the caller's params into local
// memory
struct DrawKnobs {
  double top_p, min_p;
};
DP_DEV DrawKnobs knobs_of(const dp_params_t& p) { return DrawKnobs{p.top_p, p.min_p}; }

struct DrawResult {
  int32_t index;     // position in the sorted list
  int32_t kept;
  double logprob;
  double margin;
};

DP_DEV DrawResult warp_filter_draw_smem(const double* r, int32_t k, const DrawKnobs p, double u, double* w,
                                        double* cum) {
  const uint32_t lane = lane_id();
  const double r0 = r[0];
  // w_j = exp(r_j - r_0) (filtering.py:90), inclusive cumsum in f64
  double carry = 0.0;
  for (int32_t base = 0; base < k; base += 32) {
    const int32_t j = base + lane;
    const double wj = j < k ? exp(r[j] - r0) : 0.0;
    const double c = warp_incl_scan(wj) + carry;
    if (j < k) {
      w[j] = wj;
      cum[j] = c;
    }
    carry = __shfl_sync(0xffffffffu, c, 31);
  }
  __syncwarp();
  int32_t kept = k;
  double margin = 1e30;
  const double total = cum[k - 1];
  if (p.top_p < 1.0) {                               // filtering.py:91-95
    const double thr = p.top_p * total;
    int32_t below = 0;
    for (int32_t base = 0; base < k; base += 32) {
      const int32_t j = base + lane;
      below += __popc(__ballot_sync(0xffffffffu, j < k && cum[j] < thr));
    }
    const int32_t kp = below + 1;
    kept = min(kept, kp);
    for (int32_t j = max(0, kp - 2); j < min(k, kp + 1); ++j) margin = fmin(margin, fabs(cum[j] - thr));
    margin = (double)__fdividef((float)margin, (float)total);   // flag only: f32 ratio
  }
  if (p.min_p > 0.0) {                               // filtering.py:96-98
    const double floor_ = p.min_p * w[0];
    int32_t ge = 0;
    for (int32_t base = 0; base < k; base += 32) {
      const int32_t j = base + lane;
      ge += __popc(__ballot_sync(0xffffffffu, j < k && w[j] >= floor_));
    }
    kept = min(kept, ge);
    for (int32_t j = max(0, ge - 1); j < min(k, ge + 1); ++j) margin = fmin(margin, fabs(w[j] - floor_));
  }
  kept = max(1, kept);                               // filtering.py:99
  const double S = cum[kept - 1];
  const double us = u * S;
  // j* = #(cdf_j <= u), clamped (filtering.py:158-162)
  int32_t le = 0;
  for (int32_t base = 0; base < kept; base += 32) {
    const int32_t j = base + lane;
    le += __popc(__ballot_sync(0xffffffffu, j < kept && cum[j] <= us));
  }
  const int32_t js = min(le, kept - 1);
  double dm = fabs(cum[js] - us);
  if (js > 0) dm = fmin(dm, fabs(cum[js - 1] - us));
  DrawResult res;
  res.index = js;
  res.kept = kept;
  res.logprob = (r[js] - r0) - log(S);   // ln(w_j / S), w_j = exp(r_j - r_0)
  res.margin = fmin(margin, (double)__fdividef((float)dm, (float)S));
  return res;
}

// k <= 64: everything in registers (two candidates per lane)
DP_DEV DrawResult warp_filter_draw_reg(const double* r, int32_t k, const DrawKnobs p, double u) {
  // compact on purpose: this runs once per row with a cold instruction cache,
  // so every instruction it does not have is ~20 cycles saved
  const uint32_t lane = lane_id();
  const int32_t j0 = lane, j1 = lane + 32;
  const double r0 = __shfl_sync(0xffffffffu, r[0], 0);
  // both candidates of a lane through ONE exp call on a lane-local pair: a
  // loop over an array (rr[h]) would put the pair in local memory, whose
  // store -> load round trip costs more than the whole draw
  const double ra = j0 < k ? r[j0] : 0.0;
  const double rb = j1 < k ? r[j1] : 0.0;
  double wa = 0.0, wb = 0.0;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {   // one copy of the f64 exp
    const bool in = (h == 0 ? j0 : j1) < k;
    const double e = in ? exp((h == 0 ? ra : rb) - r0) : 0.0;
    if (h == 0) wa = e;
    else wb = e;
  }
  const double ca = warp_incl_scan(wa);
  const double tot_a = __shfl_sync(0xffffffffu, ca, 31);
  const double cb = warp_incl_scan(wb) + tot_a;
  const double total = __shfl_sync(0xffffffffu, cb, 31);
  // value at global index j (any lane): cum / w / r via shuffles
  auto cum_at = [&](int32_t j) -> double { return __shfl_sync(0xffffffffu, j < 32 ? ca : cb, j & 31); };
  auto w_at = [&](int32_t j) -> double { return __shfl_sync(0xffffffffu, j < 32 ? wa : wb, j & 31); };
  auto r_at = [&](int32_t j) -> double { return __shfl_sync(0xffffffffu, j < 32 ? ra : rb, j & 31); };
  // margins only feed the 1e-6 boundary flag: f32 ratios are plenty
  auto ratio = [](double a, double b) -> double { return (double)__fdividef((float)a, (float)b); };
  int32_t kept = k;
  double margin = 1e30;
  if (p.top_p < 1.0) {
    const double thr = p.top_p * total;
    const int32_t below = __popc(__ballot_sync(0xffffffffu, j0 < k && ca < thr)) +
                          __popc(__ballot_sync(0xffffffffu, j1 < k && cb < thr));
    const int32_t kp = below + 1;
    kept = min(kept, kp);
#pragma unroll 1
    for (int32_t j = max(0, kp - 2); j < min(k, kp + 1); ++j) margin = fmin(margin, fabs(cum_at(j) - thr));
    margin = ratio(margin, total);
  }
  if (p.min_p > 0.0) {
    const double floor_ = p.min_p * 1.0;   // w_0 = exp(0) = 1
    const int32_t ge = __popc(__ballot_sync(0xffffffffu, j0 < k && wa >= floor_)) +
                       __popc(__ballot_sync(0xffffffffu, j1 < k && wb >= floor_));
    kept = min(kept, ge);
#pragma unroll 1
    for (int32_t j = max(0, ge - 1); j < min(k, ge + 1); ++j) margin = fmin(margin, fabs(w_at(j) - floor_));
  }
  kept = max(1, kept);
  const double S = cum_at(kept - 1);
  const double us = u * S;
  const int32_t le = __popc(__ballot_sync(0xffffffffu, j0 < kept && ca <= us)) +
                     __popc(__ballot_sync(0xffffffffu, j1 < kept && cb <= us));
  const int32_t js = min(le, kept - 1);
  double dm = fabs(cum_at(js) - us);
  if (js > 0) dm = fmin(dm, fabs(cum_at(js - 1) - us));
  DrawResult res;
  res.index = js;
  res.kept = kept;
  // ln p_j = ln(w_j / S) = (r_j - r_0) - ln S (w_j = exp(r_j - r_0))
  res.logprob = (r_at(js) - r0) - log(S);
  res.margin = fmin(margin, ratio(dm, S));
  return res;
}

// Nucleus rows (top-k off): r[0..K) are the K largest ready values of the
// domain (sorted), `total` the mass of the WHOLE domain relative to r[0].
// Same law as warp_filter_draw over the full domain (filtering.py:61-162);
// exact whenever the kept set — and for neutral rows the draw — lies inside
// the list.  `fallback` is set otherwise (the general kernel decides).
DP_DEV DrawResult warp_filter_draw_nuc(const double* r, int32_t K, const DrawKnobs p, double u, double total,
                                       double* w, double* cum, bool& fallback) {
  const uint32_t lane = lane_id();
  const double r0 = r[0];
  double carry = 0.0;
  for (int32_t base = 0; base < K; base += 32) {
    const int32_t j = base + lane;
    const double wj = j < K ? exp(r[j] - r0) : 0.0;
    const double c = warp_incl_scan(wj) + carry;
    if (j < K) {
      w[j] = wj;
      cum[j] = c;
    }
    carry = __shfl_sync(0xffffffffu, c, 31);
  }
  __syncwarp();
  fallback = false;
  int32_t kept = K;
  double margin = 1e30;
  const bool neutral = !(p.top_p < 1.0) && !(p.min_p > 0.0);
  bool p_open = false, m_open = false;
  if (p.top_p < 1.0) {                               // filtering.py:91-95 over the whole domain
    const double thr = p.top_p * total;
    int32_t below = 0;
    for (int32_t base = 0; base < K; base += 32) {
      const int32_t j = base + lane;
      below += __popc(__ballot_sync(0xffffffffu, j < K && cum[j] < thr));
    }
    p_open = below >= K;                             // the nucleus may extend past the list
    const int32_t kp = below + 1;
    kept = min(kept, kp);
    for (int32_t j = max(0, kp - 2); j < min(K, kp + 1); ++j) margin = fmin(margin, fabs(cum[j] - thr));
    margin = (double)__fdividef((float)margin, (float)total);   // flag only: f32 ratio
  }
  if (p.min_p > 0.0) {                               // filtering.py:96-98
    const double floor_ = p.min_p;                   // w_0 = 1
    int32_t ge = 0;
    for (int32_t base = 0; base < K; base += 32) {
      const int32_t j = base + lane;
      ge += __popc(__ballot_sync(0xffffffffu, j < K && w[j] >= floor_));
    }
    m_open = ge >= K;                                // more kept ids may follow the list
    kept = min(kept, ge);
    for (int32_t j = max(0, ge - 1); j < min(K, ge + 1); ++j) margin = fmin(margin, fabs(w[j] - floor_));
  }
  // the kept count is known once either active filter closes inside the list
  // (kept = min of the two); both open -> the general kernel decides
  if (!neutral && (p.top_p < 1.0 ? p_open : true) && (p.min_p > 0.0 ? m_open : true)) fallback = true;
  kept = max(1, kept);
  const double S = neutral ? total : cum[kept - 1];
  const double us = u * S;
  int32_t le = 0;
  for (int32_t base = 0; base < kept; base += 32) {
    const int32_t j = base + lane;
    le += __popc(__ballot_sync(0xffffffffu, j < kept && cum[j] <= us));
  }
  if (neutral && le >= kept) fallback = true;        // the draw lands past the list
  const int32_t js = min(le, kept - 1);
  double dm = fabs(cum[js] - us);
  if (js > 0) dm = fmin(dm, fabs(cum[js - 1] - us));
  DrawResult res;
  res.index = js;
  res.kept = kept;
  res.logprob = (r[js] - r0) - log(S);   // ln(w_j / S), w_j = exp(r_j - r_0)
  res.margin = fmin(margin, (double)__fdividef((float)dm, (float)S));
  return res;
}

// A real call, not inlined: one compiled copy shared by every final stage
// (smaller code), ~2.4k cycles on an idle SM (tools/micro/finish.cu)
#ifndef DP_DRAW_INLINE
static __device__ __noinline__
#else
DP_DEV
#endif
DrawResult warp_filter_draw(const double* r, int32_t k, const DrawKnobs p, double u, double* w,
                                   double* cum, int64_t* prof = nullptr) {
  (void)prof;
  return k <= 64 ? warp_filter_draw_reg(r, k, p, u) : warp_filter_draw_smem(r, k, p, u, w, cum);
}

}  // namespace dp
