// sample_general.cu — general filter/draw path: rows whose top-k stage is off
// (top_k == 0 or >= n: top-p only, min-p only, neutral) or too wide for the
// streaming top-k kernel.  Exact law of _filter_core / filtered_draw /
// categorical_draw (filtering.py:61-162) over the whole domain.
//
// One CTA per row.  Elements are ordered by a unique 64-bit composite key
// (f32 value key << 32 | ~position), i.e. (value desc, position asc) — the
// reference's lexsort order (filtering.py:83).  Penalised ids get an exact
// *virtual* composite key: the smallest f32 value whose f64(x)/tau reaches
// their f64 ready value (binary search), so they sort among the unpenalised
// elements exactly as the f64 oracle orders them.
//
// Weights w = exp(r - r_max) are accumulated in u64 fixed point (2^40 per
// unit): integer sums are exact and associative, so every bucket / prefix
// mass is deterministic.  Per-element relative error ~2e-7 comes from the
// f32 exp of unpenalised elements (penalised ones are f64); decisions within
// 1e-6 of a flip point are flagged DP_FLAG_NEAR_BOUNDARY.
//
// Passes over the domain (from L2 / shared memory when it fits):
//   A  max of unpenalised values -> r_max;
//   B  2048-bucket histogram of (count, mass) by relative log-weight
//      (bucket width tau/16 in raw units, monotone in the key order), totals,
//      min-p count/mass;
//   then each cut (top-k count, top-p mass, draw mass) finds its crossing
//   bucket, refines it by composite-key digits while it holds more than
//   kCollect elements, collects it, sorts it and scans it exactly.

#include "finish.cuh"
#include "sampler.cuh"
#include "select.cuh"

namespace dp {

constexpr int kGenNT = 512;
constexpr int kGenNB = 2048;          // level-1 buckets
constexpr int kCollect = 2048;        // max elements sorted in shared memory
constexpr double kFix = 1099511627776.0;   // 2^40 fixed-point unit of weight
constexpr float kBucketsPerNat = 16.f;

struct GenSmem {
  uint32_t cnt[kGenNB];
  unsigned long long mass[kGenNB];
  unsigned long long ckey[kCollect];
  unsigned long long cw[kCollect];
  double red_d[32];
  unsigned long long red_u[32];
  float red_f[32];
  uint32_t red_c[32];
  uint32_t ncol;
  int32_t bsel;
  uint32_t rbits;
  unsigned long long rlo, rhi;   // refine range of composite keys (inclusive)
  unsigned long long above_m;    // mass strictly above the range
  uint32_t above_c;              // count strictly above the range
  uint32_t digit_cnt[2048];
  unsigned long long digit_mass[2048];
};

struct PenEntry {
  double r;                      // exact ready value
  unsigned long long vkey;       // virtual composite key
  unsigned long long wfp;        // fixed-point weight
  uint32_t pos;                  // domain position
  uint32_t bucket;
};

// 64-bit shared-memory add as two native 32-bit atomics (sm_100 has no
// native 64-bit shared atomic add: the compiler emits a CAS loop, which
// serialises hard on the popular buckets).  The low word's carry-out of THIS
// addition goes to the high word, so the 64-bit total is exact.
DP_DEV void smem_add_u64(unsigned long long* addr, unsigned long long w) {
  uint32_t* p = reinterpret_cast<uint32_t*>(addr);
  const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
  const uint32_t old = atomicAdd(p, lo);
  const uint32_t up = hi + ((uint32_t)(old + lo) < old ? 1u : 0u);
  if (up) atomicAdd(p + 1, up);
}

// Every element of a row domain, 16-byte vector loads (8 bf16 / 4 f32 per
// load; the passes re-read the row from L2): fn(position, value).
template <typename T, typename F>
DP_DEV void for_each_elem(const T* rowp, int64_t n, uint32_t tid, F fn) {
  constexpr int EPV = Elem<T>::kPerVec;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(rowp);
  const int64_t a0 = min64(n, (int64_t)(((16u - (addr & 15u)) & 15u) / sizeof(T)));
  for (int64_t i = tid; i < a0; i += kGenNT) fn(i, Elem<T>::get(rowp, i));
  const int64_t nvec = (n - a0) / EPV;
  const uint4* vp = reinterpret_cast<const uint4*>(rowp + a0);
  // kGenU independent 16-byte loads in flight per thread: one CTA walks a
  // whole row per pass, so a single outstanding load per thread made every
  // pass L2-latency-bound
  constexpr int kGenU = 4;
  int64_t v = tid;
  for (; v + (kGenU - 1) * kGenNT < nvec; v += kGenU * kGenNT) {
    uint4 q[kGenU];
#pragma unroll
    for (int u = 0; u < kGenU; ++u) q[u] = __ldg(vp + v + u * kGenNT);
#pragma unroll
    for (int u = 0; u < kGenU; ++u)
#pragma unroll
      for (int e = 0; e < EPV; ++e) fn(a0 + (v + u * kGenNT) * EPV + e, vec_elem<T>(q[u], e));
  }
  for (; v < nvec; v += kGenNT) {
    const uint4 q = __ldg(vp + v);
#pragma unroll
    for (int e = 0; e < EPV; ++e) fn(a0 + v * EPV + e, vec_elem<T>(q, e));
  }
  for (int64_t i = a0 + nvec * EPV + tid; i < n; i += kGenNT) fn(i, Elem<T>::get(rowp, i));
}

// block reductions over kGenNT threads
template <typename F>
DP_DEV double blk_sum_d(double v, GenSmem& g, F sync) {
  v = warp_sum(v);
  if ((threadIdx.x & 31u) == 0) g.red_d[threadIdx.x >> 5] = v;
  sync();
  double s = 0.0;
  for (int w = 0; w < kGenNT / 32; ++w) s += g.red_d[w];
  sync();
  return s;
}
template <typename F>
DP_DEV unsigned long long blk_sum_u(unsigned long long v, GenSmem& g, F sync) {
  v = warp_sum(v);
  if ((threadIdx.x & 31u) == 0) g.red_u[threadIdx.x >> 5] = v;
  sync();
  unsigned long long s = 0;
  for (int w = 0; w < kGenNT / 32; ++w) s += g.red_u[w];
  sync();
  return s;
}
template <typename F>
DP_DEV uint32_t blk_sum_c(uint32_t v, GenSmem& g, F sync) {
  v = warp_sum(v);
  if ((threadIdx.x & 31u) == 0) g.red_c[threadIdx.x >> 5] = v;
  sync();
  uint32_t s = 0;
  for (int w = 0; w < kGenNT / 32; ++w) s += g.red_c[w];
  sync();
  return s;
}
template <typename F>
DP_DEV float blk_max_f(float v, GenSmem& g, F sync) {
  v = warp_max(v);
  if ((threadIdx.x & 31u) == 0) g.red_f[threadIdx.x >> 5] = v;
  sync();
  float m = g.red_f[0];
  for (int w = 1; w < kGenNT / 32; ++w) m = fmaxf(m, g.red_f[w]);
  sync();
  return m;
}

// Crossing search over n bins in descending-key order (bin 0 = highest keys).
// kind 0: first bin where cumulative count >= target_c
// kind 1: first bin where cumulative mass >= target_m   (top-p, inclusive)
// kind 2: first bin where cumulative mass >  target_m   (draw, strict)
// Executed by warp 0; returns bin, count and mass strictly above it.
struct Cross {
  int32_t bin;
  uint32_t above_c;
  unsigned long long above_m;
};
DP_DEV Cross warp_cross(const uint32_t* cnt, const unsigned long long* mass, int nbins, int kind, uint32_t target_c,
                        double target_m) {
  const uint32_t lane = lane_id();
  const int per = (nbins + 31) / 32;
  const int lo = lane * per, hi = min(nbins, lo + per);
  uint32_t sc = 0;
  unsigned long long sm = 0;
  for (int i = lo; i < hi; ++i) {
    sc += cnt[i];
    sm += mass[i];
  }
  const uint32_t ic = warp_incl_scan(sc);
  const unsigned long long im = warp_incl_scan(sm);
  const uint32_t ec = ic - sc;
  const unsigned long long em = im - sm;
  bool hit;
  if (kind == 0) hit = ec < target_c && target_c <= ic;
  else if (kind == 1) hit = (double)em < target_m && (double)im >= target_m;
  else hit = (double)em <= target_m && (double)im > target_m;
  const uint32_t b = __ballot_sync(0xffffffffu, hit);
  Cross r;
  r.bin = -1;
  r.above_c = 0;
  r.above_m = 0;
  int L = b ? __ffs(b) - 1 : -1;
  int bin = -1;
  uint32_t ac = 0;
  unsigned long long am = 0;
  if ((int)lane == L) {
    uint32_t c = ec;
    unsigned long long m = em;
    for (int i = lo; i < hi; ++i) {
      bool h;
      if (kind == 0) h = c + cnt[i] >= target_c;
      else if (kind == 1) h = (double)(m + mass[i]) >= target_m;
      else h = (double)(m + mass[i]) > target_m;
      if (h) {
        bin = i;
        ac = c;
        am = m;
        break;
      }
      c += cnt[i];
      m += mass[i];
    }
  }
  if (L >= 0) {
    r.bin = __shfl_sync(0xffffffffu, bin, L);
    r.above_c = __shfl_sync(0xffffffffu, ac, L);
    r.above_m = __shfl_sync(0xffffffffu, am, L);
  }
  return r;
}

template <typename T, int MODE>
__global__ void __launch_bounds__(kGenNT, 1) general_sample_kernel(SampleArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  GenSmem& g = *reinterpret_cast<GenSmem*>(smem);
  PenEntry* pen = reinterpret_cast<PenEntry*>(smem + ((sizeof(GenSmem) + 15) & ~15));
  const int64_t n = dom_n(a, MODE);
  const int64_t lo = dom_lo(a, MODE);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(pen) + (size_t)pen_bound(a.pen) * sizeof(PenEntry));
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  auto sync = [] { __syncthreads(); };

  const int nrows = a.row_count ? *a.row_count : a.n_rows;
  // CTAs loop over the rows (grid sized to the resident CTAs): rows routed to
  // the streaming kernels cost one parameter read here
  for (int ridx = blockIdx.x; ridx < nrows; ridx += gridDim.x) {
  const int row = a.rows ? a.rows[ridx] : ridx;
  const dp_params_t p = a.params[row];
  const int32_t plen_all = pen_len(a, row, p);
  if (route_row(a, MODE, p.top_k, plen_all, n) != kRouteGeneral) continue;   // a streaming kernel's row
  sync();   // the previous row is done with the shared buffers
  const T* rowp = domain_row<T>(a, row, MODE);
  const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
  const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;
  const double tau = p.temperature;

  // ---- penalty entries inside the domain -> pen[], bitmap
  const uint32_t words = (uint32_t)((n + 31) / 32);
  for (uint32_t i = tid; i < words; i += kGenNT) bitmap[i] = 0u;
  if (tid == 0) g.ncol = 0u;
  sync();
  for (int32_t j = tid; j < plen_all; j += kGenNT) {
    const int64_t pos = id_to_pos(a, pids[j]) - lo;
    if (pos >= 0 && pos < n) {
      const uint32_t s = atomicAdd(&g.ncol, 1u);
      pen[s].pos = (uint32_t)pos;
      pen[s].r = ready_penalized(Elem<T>::get(rowp, pos), pcnt[j], p);
      atomicOr(&bitmap[pos >> 5], 1u << (pos & 31));
    }
  }
  sync();
  const uint32_t np = g.ncol;
  if (tid == 0) touch_bytes(a, row, (uint64_t)np * sizeof(T));   // gathered penalty values
  auto is_pen = [&](int64_t pos) -> bool { return np > 0 && ((bitmap[pos >> 5] >> (pos & 31)) & 1u); };
  auto val = [&](int64_t i) -> float { return Elem<T>::get(rowp, i); };

  // ---- pass A: max of unpenalised values
  float mx = -INFINITY;
  if (tid == 0) touch_bytes(a, row, (uint64_t)n * sizeof(T));   // one more pass over the domain
  for_each_elem(rowp, n, tid, [&](int64_t i, float x) {
    if (!is_pen(i)) mx = fmaxf(mx, x);
  });
  mx = blk_max_f(mx, g, sync);
  double rmax = mx == -INFINITY ? -INFINITY : ready_plain(mx, p);
  {
    double pm = -INFINITY;
    for (uint32_t j = tid; j < np; j += kGenNT) pm = fmax(pm, pen[j].r);
    pm = warp_max(pm);
    if (lane == 0) g.red_d[warp] = pm;
    sync();
    for (int w = 0; w < kGenNT / 32; ++w) rmax = fmax(rmax, g.red_d[w]);
    sync();
  }
  double u[3];
  get_uniforms(a, row, p, u);
  if (!isfinite(rmax)) {                                    // no usable mass
    if (tid == 0) {
      a.token[row] = -1;
      a.logprob[row] = 0.0;
      a.flags[row] = DP_FLAG_DEGENERATE;
    }
    continue;
  }
  // raw-unit anchor of the weights: w = exp((x - c)/tau), c = rmax*tau (hi/lo)
  const double cd = rmax * tau;
  const float c_hi = (float)cd, c_lo = (float)(cd - (double)(float)cd);
  const float inv_tau = (float)(1.0 / tau);
  const float bscale = kBucketsPerNat * inv_tau;
  auto bucket_of = [&](float x) -> uint32_t {
    float d = ((c_hi - x) + c_lo) * bscale;
    d = fmaxf(d, 0.f);
    return d >= (float)(kGenNB - 1) ? (uint32_t)(kGenNB - 1) : (uint32_t)d;
  };
  auto wfix = [&](float x) -> unsigned long long {
    const float w = expf(((x - c_hi) - c_lo) * inv_tau);
    return (unsigned long long)fminf(w * (float)kFix + 0.5f, 1.8e19f);
  };
  auto ready_of_key = [&](uint32_t k32) -> double { return ready_plain(key_f32(k32), p); };

  // ---- penalised entries: virtual keys (exact order), weights, buckets.
  // K = smallest f32 key with f64(x_K)/tau >= r (binary search over
  // [key(-inf), key(+inf)]); equal -> tie with real elements of value x_K,
  // ordered by position; otherwise strictly between K-1 and K, below every
  // real key K, and penalised entries sharing the gap ordered (r desc, pos asc)
  for (uint32_t j = tid; j < np; j += kGenNT) {
    const double r = pen[j].r;
    uint32_t lo_k = 0x007FFFFFu, hi_k = 0xFF800000u;
    if (!(ready_of_key(hi_k) >= r)) lo_k = hi_k;
    while (lo_k < hi_k) {
      const uint32_t mid = lo_k + ((hi_k - lo_k) >> 1);
      if (ready_of_key(mid) >= r) hi_k = mid;
      else lo_k = mid + 1;
    }
    const bool eq = ready_of_key(lo_k) == r;
    pen[j].vkey = ((unsigned long long)lo_k << 32) | (eq ? 1ull : 0ull);   // low bit: eq flag (temporary)
    const double w = exp(r - rmax);
    pen[j].wfp = (unsigned long long)(w * kFix + 0.5);
    pen[j].bucket = bucket_of(key_f32(lo_k));
  }
  sync();
  for (uint32_t j = tid; j < np; j += kGenNT) {
    const uint32_t kj = (uint32_t)(pen[j].vkey >> 32);
    const bool eqj = (pen[j].vkey & 1ull) != 0ull;
    uint32_t low = 0xFFFFFFFFu - pen[j].pos;
    if (!eqj) {
      uint32_t before = 0;
      for (uint32_t q = 0; q < np; ++q) {
        if (q == j || (uint32_t)(pen[q].vkey >> 32) != kj || (pen[q].vkey & 1ull)) continue;
        if (pen[q].r > pen[j].r || (pen[q].r == pen[j].r && pen[q].pos < pen[j].pos)) ++before;
      }
      low = 0x7FFFFFFFu - before;
    }
    g.ckey[j] = ((unsigned long long)kj << 32) | low;   // staged: vkey still read by others
  }
  sync();
  for (uint32_t j = tid; j < np; j += kGenNT) pen[j].vkey = g.ckey[j];
  sync();
  // min-p floor: keep w >= min_p (w_0 = 1 is the max): smallest f32 key with
  // exp(ready - rmax) >= min_p (f64, the reference's test, filtering.py:96-98)
  uint32_t minp_key = 0u;
  if (p.min_p > 0.0) {
    uint32_t lo_k = 0x007FFFFFu, hi_k = 0xFF800000u;
    while (lo_k < hi_k) {
      const uint32_t mid = lo_k + ((hi_k - lo_k) >> 1);
      if (exp(ready_of_key(mid) - rmax) >= p.min_p * 1.0) hi_k = mid;
      else lo_k = mid + 1;
    }
    minp_key = lo_k;
  }

  // ---- pass B: level-1 histogram + totals
  for (uint32_t i = tid; i < kGenNB; i += kGenNT) {
    g.cnt[i] = 0u;
    g.mass[i] = 0ull;
  }
  sync();
  unsigned long long wsum = 0, wminp = 0;
  uint32_t cminp = 0, cnp = 0;
  if (tid == 0) touch_bytes(a, row, (uint64_t)n * sizeof(T));   // one more pass over the domain
  for_each_elem(rowp, n, tid, [&](int64_t i, float x) {
    if (is_pen(i)) return;
    const uint32_t b = bucket_of(x);
    const unsigned long long w = wfix(x);
    atomicAdd(&g.cnt[b], 1u);
    if (w) smem_add_u64(&g.mass[b], w);
    wsum += w;
    ++cnp;
    if (p.min_p > 0.0 && f32_key(x) >= minp_key) {
      wminp += w;
      ++cminp;
    }
  });
  for (uint32_t j = tid; j < np; j += kGenNT) {
    atomicAdd(&g.cnt[pen[j].bucket], 1u);
    smem_add_u64(&g.mass[pen[j].bucket], pen[j].wfp);
    wsum += pen[j].wfp;
    if (p.min_p > 0.0 && exp(pen[j].r - rmax) >= p.min_p) {
      wminp += pen[j].wfp;
      ++cminp;
    }
  }
  sync();
  const unsigned long long W = blk_sum_u(wsum, g, sync);
  const uint32_t n_np = blk_sum_c(cnp, g, sync);
  const uint32_t kept_m_cnt = p.min_p > 0.0 ? blk_sum_c(cminp, g, sync) : 0u;
  const unsigned long long W_m = p.min_p > 0.0 ? blk_sum_u(wminp, g, sync) : 0ull;

  // kHot: alpha and the accept test (shvs.py:223-236); S_H relative to the
  // producer's row max m: S_H = W * exp(rmax - m)
  double alpha = 1.0, sH = 0.0;
  bool deferred = false;   // accept test left to the exact re-sum (defer_accept)
  if (MODE == kHot) {
    const double mrow = a.row_max[row];
    sH = ((double)W / kFix) * exp(rmax - mrow);
    double corr = 0.0;
    if (a.summary_raw) {
      corr = raw_summary_correction(a, row, p, plen_all, mrow, tid, kGenNT,
                                    [&](int64_t pos) { return row_value<T>(a, row, pos); });
      corr = blk_sum_d(corr, g, sync);
    }
    const double S_prod = a.total_expsum[row];
    const double S = S_prod + corr;
    const bool tail_empty = a.V == a.H;
    bool degenerate = false;
    if (!tail_empty) {
      if (!(S > 0.0) || !isfinite(S)) degenerate = true;
      else alpha = fmin(sH / S, 1.0);
    }
    deferred = sH > 0.0 && defer_accept(a, S_prod, S, alpha, u[1]);
    const bool accept = deferred || (!degenerate && sH > 0.0 && (tail_empty || u[1] <= alpha));
    if (!accept) {
      if (tid == 0) {
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
      continue;
    }
  }

  // ---- exact crossing search: returns the element (key, weight), its rank
  // and the mass strictly above it, for a count or mass target
  struct Hit {
    unsigned long long key, w, above_m;
    uint32_t above_c;
    bool ok;
  };
  auto in_range = [&](unsigned long long k) -> bool { return k >= g.rlo && k <= g.rhi; };
  // key of element i (unpenalised) and its bucket
  auto ekey = [&](int64_t i, float x) -> unsigned long long { return comp_key(x, (uint32_t)i); };
  auto find = [&](int kind, uint32_t target_c, double target_m) -> Hit {
    Hit h;
    h.ok = false;
    h.key = h.w = h.above_m = 0;
    h.above_c = 0;
    // level 1: buckets
    if (warp == 0) {
      const Cross c = warp_cross(g.cnt, g.mass, kGenNB, kind, target_c, target_m);
      if (lane == 0) {
        g.bsel = c.bin;
        g.above_c = c.above_c;
        g.above_m = c.above_m;
      }
    }
    sync();
    const int32_t bsel = g.bsel;
    if (bsel < 0) return h;
    // key range of the bucket: all keys whose bucket is bsel
    if (tid == 0) {
      g.rlo = 0ull;
      g.rhi = ~0ull;
      g.rbits = 64u;
    }
    sync();
    uint32_t in_cnt = g.cnt[bsel];
    // refine by composite-key digits (11 bits) while the range is too large
    uint32_t shift = 53;
    bool use_bucket = true;   // level-1 membership is by bucket, deeper by key prefix
    while (in_cnt > (uint32_t)kCollect) {
      for (uint32_t i = tid; i < 2048; i += kGenNT) {
        g.digit_cnt[i] = 0u;
        g.digit_mass[i] = 0ull;
      }
      sync();
      const unsigned long long pmask = shift >= 53 ? 0ull : (~0ull << (shift + 11));
      const unsigned long long pref = g.rlo & pmask;
      auto member = [&](unsigned long long k, uint32_t b) -> bool {
        return (use_bucket ? b == (uint32_t)bsel : true) && (k & pmask) == pref && in_range(k);
      };
      if (tid == 0) touch_bytes(a, row, (uint64_t)n * sizeof(T));   // one more pass over the domain
  for_each_elem(rowp, n, tid, [&](int64_t i, float x) {
        if (is_pen(i)) return;
        const uint32_t b = bucket_of(x);
        if (b != (uint32_t)bsel) return;
        const unsigned long long k = ekey(i, x);
        if (!member(k, b)) return;
        const uint32_t d = (uint32_t)(k >> shift) & 2047u;
        // descending key order: digit 2047 first
        atomicAdd(&g.digit_cnt[2047u - d], 1u);
        const unsigned long long w = wfix(x);
        if (w) smem_add_u64(&g.digit_mass[2047u - d], w);
      });
      for (uint32_t j = tid; j < np; j += kGenNT) {
        const unsigned long long k = pen[j].vkey;
        if (pen[j].bucket == (uint32_t)bsel && member(k, pen[j].bucket)) {
          const uint32_t d = (uint32_t)(k >> shift) & 2047u;
          atomicAdd(&g.digit_cnt[2047u - d], 1u);
          smem_add_u64(&g.digit_mass[2047u - d], pen[j].wfp);
        }
      }
      sync();
      if (warp == 0) {
        const uint32_t tc = target_c > g.above_c ? target_c - g.above_c : 0u;
        const double tm = target_m - (double)g.above_m;
        const Cross c = warp_cross(g.digit_cnt, g.digit_mass, 2048, kind, tc, tm);
        if (lane == 0) {
          const uint32_t d = 2047u - (uint32_t)max(c.bin, 0);
          const unsigned long long pref2 = pref | ((unsigned long long)d << shift);
          const unsigned long long m2 = shift >= 53 ? (~0ull << shift) : (pmask | (2047ull << shift));
          g.rlo = pref2 & m2;
          g.rhi = (pref2 & m2) | ~m2;
          g.above_c += c.above_c;
          g.above_m += c.above_m;
          g.bsel = c.bin < 0 ? -1 : bsel;
          g.rbits = g.digit_cnt[max(c.bin, 0)];
        }
      }
      sync();
      if (g.bsel < 0) return h;
      in_cnt = g.rbits;
      if (shift < 11) break;   // fully resolved key (unique)
      shift -= 11;
    }
    // collect the range: unpenalised + penalised members
    if (tid == 0) g.ncol = 0u;
    sync();
    if (tid == 0) touch_bytes(a, row, (uint64_t)n * sizeof(T));   // one more pass over the domain
  for_each_elem(rowp, n, tid, [&](int64_t i, float x) {
      if (is_pen(i)) return;
      if (bucket_of(x) != (uint32_t)bsel) return;
      const unsigned long long k = ekey(i, x);
      if (!in_range(k)) return;
      const uint32_t s = atomicAdd(&g.ncol, 1u);
      if (s < (uint32_t)kCollect) {
        g.ckey[s] = k;
        g.cw[s] = wfix(x);
      }
    });
    for (uint32_t j = tid; j < np; j += kGenNT) {
      if (pen[j].bucket == (uint32_t)bsel && in_range(pen[j].vkey)) {
        const uint32_t s = atomicAdd(&g.ncol, 1u);
        if (s < (uint32_t)kCollect) {
          g.ckey[s] = pen[j].vkey;
          g.cw[s] = pen[j].wfp;
        }
      }
    }
    sync();
    const uint32_t nc = min(g.ncol, (uint32_t)kCollect);
    uint32_t p2 = 1;
    while (p2 < nc) p2 <<= 1;
    for (uint32_t i = nc + tid; i < p2; i += kGenNT) {
      g.ckey[i] = 0ull;
      g.cw[i] = 0ull;
    }
    sync();
    // bitonic sort, descending by key (keys unique), weights ride along
    for (uint32_t size = 2; size <= p2; size <<= 1)
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t i = tid; i < p2 / 2; i += kGenNT) {
          const uint32_t lo_i = 2 * stride * (i / stride) + (i % stride);
          const uint32_t hi_i = lo_i + stride;
          const bool desc = ((lo_i & size) == 0);
          const unsigned long long ka = g.ckey[lo_i], kb = g.ckey[hi_i];
          if ((ka > kb) != desc) {
            g.ckey[lo_i] = kb;
            g.ckey[hi_i] = ka;
            const unsigned long long t0 = g.cw[lo_i];
            g.cw[lo_i] = g.cw[hi_i];
            g.cw[hi_i] = t0;
          }
        }
        sync();
      }
    // sequential exact scan by one thread (nc is small)
    if (tid == 0) {
      uint32_t c = g.above_c;
      unsigned long long m = g.above_m;
      int32_t found = -1;
      for (uint32_t i = 0; i < nc; ++i) {
        bool hit;
        if (kind == 0) hit = c + 1 >= target_c;
        else if (kind == 1) hit = (double)(m + g.cw[i]) >= target_m;
        else hit = (double)(m + g.cw[i]) > target_m;
        if (hit) {
          found = (int32_t)i;
          break;
        }
        ++c;
        m += g.cw[i];
      }
      g.bsel = found;
      g.above_c = c;
      g.above_m = m;
      if (found >= 0) {
        g.rlo = g.ckey[found];
        g.rhi = g.cw[found];
      }
    }
    sync();
    if (g.bsel >= 0) {
      h.ok = true;
      h.key = g.rlo;
      h.w = g.rhi;
      h.above_c = g.above_c;
      h.above_m = g.above_m;
    }
    sync();
    return h;
  };

  // ---- the cuts (filtering.py:77-99)
  const int64_t ndom = (int64_t)n_np + np;
  const int32_t k = p.top_k;
  uint32_t kept = (uint32_t)ndom;
  unsigned long long S_kept = W;   // mass of the kept prefix
  double margin = 1e300;
  unsigned long long W_K = W;
  if (k > 0 && (int64_t)k < ndom) {                           // wide top-k (count cut)
    const Hit hk = find(0, (uint32_t)k, 0.0);
    W_K = hk.above_m + hk.w;
    kept = (uint32_t)k;
    S_kept = W_K;
  }
  if (p.top_p < 1.0) {
    const double thr = p.top_p * (double)W_K;
    const Hit hp = find(1, 0u, thr);
    if (hp.ok) {
      const uint32_t kp = hp.above_c + 1;
      margin = fmin(margin, fabs((double)(hp.above_m + hp.w) - thr) / (double)W_K);
      margin = fmin(margin, fabs((double)hp.above_m - thr) / (double)W_K);
      if (kp < kept) {
        kept = kp;
        S_kept = hp.above_m + hp.w;
      }
    }
  }
  if (p.min_p > 0.0) {
    const uint32_t km = max(kept_m_cnt, 1u);
    if (km < kept) {
      kept = km;
      S_kept = W_m;
    }
  }
  if (kept < 1) kept = 1;
  // ---- inverse-CDF draw over the kept prefix (filtering.py:158-162)
  const double target = u[MODE == kTail ? 2 : 0] * (double)S_kept;
  Hit hd = find(2, 0u, target);
  if (!hd.ok || hd.above_c >= kept) hd = find(0, kept, 0.0);   // clamp to the last kept element
  if (tid == 0) {
    const unsigned long long key = hd.key;
    // position: real keys carry ~pos, virtual (penalised) keys need a lookup
    uint32_t pos;
    double r;
    if ((uint32_t)(key & 0xFFFFFFFFull) >= 0x80000000u) {
      pos = comp_pos(key);
      r = ready_plain(comp_val(key), p);
      for (uint32_t j = 0; j < np; ++j)
        if (pen[j].vkey == key) r = pen[j].r;
    } else {
      pos = 0;
      r = rmax;
      for (uint32_t j = 0; j < np; ++j)
        if (pen[j].vkey == key) {
          pos = pen[j].pos;
          r = pen[j].r;
        }
    }
    const double dm = fmin(fabs((double)(hd.above_m + hd.w) - target), fabs((double)hd.above_m - target)) /
                      (double)S_kept;
    margin = fmin(margin, dm);
    const int64_t gpos = (int64_t)pos + lo;
    a.token[row] = pos_to_id(a, gpos);
    a.logprob[row] = (r - rmax) - log((double)S_kept / kFix);
    uint8_t fl = MODE == kHot ? DP_FLAG_ACCEPTED_HOT : (MODE == kTail ? DP_FLAG_REJECTED : 0);
    if (MODE == kHot && a.V != a.H && !deferred) margin = fmin(margin, fabs(u[1] - alpha));
    if (margin < kBoundaryEps) fl |= DP_FLAG_NEAR_BOUNDARY;
    if (MODE == kTail) fl |= a.flags[row] & DP_FLAG_NEAR_BOUNDARY;
    a.flags[row] = fl;
    if (a.dbg.margin) a.dbg.margin[row] = MODE == kTail ? fmin(margin, a.dbg.margin[row]) : margin;
    if (a.dbg.kept) a.dbg.kept[row] = (int32_t)kept;
    if (MODE == kHot && a.dbg.alpha) a.dbg.alpha[row] = alpha;
    if (deferred) push_resum(a, row, sH);   // the exact re-sum decides, then records
    else thread_record_token(a, row, pos_to_id(a, gpos));   // fused K5
  }
  }
}

template <typename T, int MODE>
static cudaError_t launch_general_t(const SampleArgs& a, int grid_rows, cudaStream_t st) {
  const int64_t n = MODE == kFull ? a.V : (MODE == kHot ? a.H : a.V - a.H);
  const size_t smem = ((sizeof(GenSmem) + 15) & ~15) + (size_t)pen_bound(a.pen) * sizeof(PenEntry) +
                      (size_t)((n + 31) / 32) * 4;
  auto kern = general_sample_kernel<T, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGenNT, smem) != cudaSuccess || per_sm < 1) per_sm = 1;
  const int grid = grid_rows < sms * per_sm ? grid_rows : sms * per_sm;
  if (grid < 1) return cudaSuccess;
  kern<<<grid, kGenNT, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_general(const SampleArgs& a, int dtype, int mode, int grid_rows, cudaStream_t st) {
  if (dtype == DP_F32) {
    if (mode == kFull) return launch_general_t<float, kFull>(a, grid_rows, st);
    if (mode == kHot) return launch_general_t<float, kHot>(a, grid_rows, st);
    return launch_general_t<float, kTail>(a, grid_rows, st);
  }
  if (mode == kFull) return launch_general_t<__nv_bfloat16, kFull>(a, grid_rows, st);
  if (mode == kHot) return launch_general_t<__nv_bfloat16, kHot>(a, grid_rows, st);
  return launch_general_t<__nv_bfloat16, kTail>(a, grid_rows, st);
}

}  // namespace dp
