// sample_hot.cu — K1h: SHVS hot pass for short hot sets (H <= 4096) by an
// exact sort, sm_100a.
//
// A hot prefix of H <= 4096 logits fits one CTA's shared memory, so instead
// of threshold estimation, admission and a candidate select (K1 / K1w) the
// CTA materialises every hot position's ready value exactly (IEEE f64:
// x / tau, penalized ids by penalty.py:66-78), sums the hot mass S_H in f64,
// runs the accept test (shvs.py:223-236) and, for accepted rows, sorts the
// hot prefix by (ready desc, position asc) — the canonical order of
// _top_k_ids / _filter_core (filtering.py:38-105) — and decides with the
// exact top-k / top-p / min-p / inverse-CDF law (filtering.py:124-162) over
// the first min(k, H) entries (all H with top-k off).  No estimate, no
// re-stream, no fallback: nucleus rows (top-p / min-p without top-k), which
// K1 decides through a 256-entry list plus a general-kernel fallback, are
// exact here too.  Nucleus rows skip the full sort in the common case: the
// top-224 by a block radix select (digits from the keys' highest differing
// bit), one warp sorts them, and warp_filter_draw_nuc decides against the
// exact f64 mass of the whole hot set; the full sort runs only when the kept
// set (or a neutral row's draw) leaves that list.  Opt-in (DP_PLAN_HOT_SORT:
// nucleus rows, route_row use_hot_sort 1; DP_PLAN_HOT_SORT_ALL: every row,
// 2): the streaming kernels stay faster at the bench shapes — C2 top-k rows
// 36 vs ~70 us, C5 nucleus rows 1,045 vs 1,306 us per step at H = 2,048
// (per row, two f64 exps and an f64 divide per hot value dominate;
// profiles/r2/k1h).  One CTA per row (grid-stride over rows).
#include "sampler.cuh"
#include "select.cuh"
#include "finish.cuh"

namespace dp {

constexpr int kHSNT = 256;          // threads per CTA
constexpr int kHSW = kHSNT / 32;
constexpr int kHSCumMin = 1152;     // doubles: the nucleus path's scratch (2 KB keys + 1 KB pos + 3 x 256 doubles)
constexpr int kHSNucM = 224;        // nucleus rows: the M largest are selected first (ties may add up to 256)

DP_DEV double key_f64(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

struct HotSortShared {
  double red[kHSW];
  double red2[kHSW];
  uint32_t cnt[kHSW];
  uint32_t cnt2[kHSW];
  double bc[4];
  uint32_t bcu[4];
};

// fixed-order block sums / counts (deterministic)
DP_DEV double hs_sum(double v, double* red, double* bc) {
  v = warp_sum(v);
  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kHSW; ++w) s += red[w];
    bc[0] = s;
  }
  __syncthreads();
  const double s = bc[0];
  __syncthreads();
  return s;
}
DP_DEV uint32_t hs_count(bool pred, uint32_t* cnt, uint32_t* bcu) {
  const uint32_t c = __popc(__ballot_sync(0xffffffffu, pred));
  if ((threadIdx.x & 31u) == 0) cnt[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kHSW; ++w) s += cnt[w];
    bcu[0] = s;
  }
  __syncthreads();
  const uint32_t s = bcu[0];
  __syncthreads();
  return s;
}

template <typename T>
__global__ void __launch_bounds__(kHSNT) hot_sort_kernel(SampleArgs a, int hp) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int ccap_d = hp > kHSCumMin ? hp : kHSCumMin;   // prefix masses / nucleus scratch (doubles)
  uint64_t* key = reinterpret_cast<uint64_t*>(smem);   // [hp] ready keys
  double* cum = reinterpret_cast<double*>(key + hp);    // [ccap_d] prefix masses
  uint32_t* pos = reinterpret_cast<uint32_t*>(cum + ccap_d);   // [hp] hot positions
  __shared__ HotSortShared S;
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  const int64_t H = a.H;
  const int nrows = a.row_count ? *a.row_count : a.n_rows;
  for (int ridx = blockIdx.x; ridx < nrows; ridx += gridDim.x) {
    const int row = a.rows ? a.rows[ridx] : ridx;
    const dp_params_t p = a.params[row];
    const int32_t plen = pen_len(a, row, p);
    const int32_t k = p.top_k;
    if (route_row(a, kHot, k, plen, a.H) != kRouteHotSort) continue;   // a streaming kernel's row
    const T* rowp = domain_row<T>(a, row, kHot);
    const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
    const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;
    const double mrow = a.row_max[row];
    __syncthreads();   // the previous row is done with the shared arrays
    // ---- 1. ready keys of the hot prefix (unpenalized form: x / tau)
    for (int i = (int)tid; i < hp; i += kHSNT) {
      key[i] = i < H ? f64_key(ready_plain(Elem<T>::get(rowp, i), p)) : 0ull;
      pos[i] = (uint32_t)i;
    }
    __syncthreads();
    // ---- 2. penalized ids: exact ready values inside the hot prefix; the raw
    // producer summary's correction over the whole list (sampler.cuh)
    double corr = 0.0;
    for (int32_t j = (int32_t)tid; j < plen; j += kHSNT) {
      const int64_t q = id_to_pos(a, pids[j]);
      const float x = row_value<T>(a, row, q);
      const double r = ready_penalized(x, pcnt[j], p);
      if (q < H) key[q] = f64_key(r);
      if (a.summary_raw) corr += exp(r - mrow) - exp(ready_plain(x, p) - mrow);
    }
    __syncthreads();
    // ---- 3. hot mass S_H (f64) and the accept test (shvs.py:223-236)
    double sh = 0.0;
    for (int i = (int)tid; i < H; i += kHSNT) sh += exp(key_f64(key[i]) - mrow);
    const double sH = hs_sum(sh, S.red, S.bc);
    corr = hs_sum(corr, S.red2, S.bc);
    if (tid == 0) touch_bytes(a, row, (uint64_t)(H + plen) * sizeof(T));
    double u[3];
    get_uniforms(a, row, p, u);
    const double S_prod = a.total_expsum[row];
    const double Stot = S_prod + corr;
    const bool tail_empty = a.V == a.H;
    bool degenerate = false;
    double alpha = 1.0;
    if (!tail_empty) {
      if (!(Stot > 0.0) || !isfinite(Stot)) degenerate = true;
      else alpha = fmin(sH / Stot, 1.0);
    }
    const bool deferred = sH > 0.0 && defer_accept(a, S_prod, Stot, alpha, u[1]);
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
    // ---- 4. canonical order (ready desc, position asc) of the first n entries
    const int n = (k > 0 && (int64_t)k < H) ? k : (int)H;
    bool sorted = false;
    if (n < (int)H && n <= 256) {
      // top-k rows: radix threshold of the k-th largest key (ties at it
      // included), the >= k survivors compacted and ordered by one warp
      auto get_k = [&](uint32_t i, uint64_t& kk) -> bool { kk = key[i]; return true; };
      uint32_t* hist = reinterpret_cast<uint32_t*>(pos + hp);   // 256 u32 past the arrays (smem sized for it)
      const uint64_t t = group_select_threshold<kHSNT>(get_k, (uint32_t)H, (uint32_t)H, (uint32_t)n, hist, S.bcu,
                                                       tid, [] { __syncthreads(); });
      uint64_t* ck = reinterpret_cast<uint64_t*>(cum);          // survivors (scratch in the prefix array)
      uint32_t* cp = reinterpret_cast<uint32_t*>(ck + 256);
      if (tid == 0) S.bcu[3] = 0u;
      __syncthreads();
      for (int i = (int)tid; i < (int)H; i += kHSNT) {
        const uint64_t kk = key[i];
        if (kk >= t) {
          const uint32_t o = atomicAdd(&S.bcu[3], 1u);
          if (o < 256u) {
            ck[o] = kk;
            cp[o] = pos[i];
          }
        }
      }
      __syncthreads();
      const uint32_t c = S.bcu[3];
      if (c <= 256u) {   // else (massive ties) the full sort below
        if (tid < 32) {
          warp_topk_sort(ck, cp, c, (uint32_t)n, hist);
          for (int j = (int)lane; j < n; j += 32) {
            key[j] = ck[j];
            pos[j] = cp[j];
          }
        }
        __syncthreads();
        sorted = true;
      }
    }
    if (!sorted && n == (int)H && H > 256) {
      // nucleus rows (top-k off): the top-M by a block radix select (digits
      // start at the keys' highest differing bit, so the histogram spreads),
      // one warp sorts them, and warp_filter_draw_nuc decides against the
      // exact mass of the whole hot set — the full sort only when the kept
      // set (or, for neutral rows, the draw) leaves the M (fallback)
      uint32_t* hist = reinterpret_cast<uint32_t*>(pos + hp);
      uint64_t* ck = reinterpret_cast<uint64_t*>(cum);      // [256] survivors
      uint32_t* cpos = reinterpret_cast<uint32_t*>(ck + 256);   // [256]
      double* fr = reinterpret_cast<double*>(cpos + 256);    // [256] sorted ready values
      double* fw = fr + 256;
      double* fc = fw + 256;
      // kmax / kmin of the keys of the hot set, and r0 / the mass relative to it
      uint64_t kmx = 0ull, kmn = ~0ull;
      for (int i = (int)tid; i < (int)H; i += kHSNT) {
        kmx = key[i] > kmx ? key[i] : kmx;
        kmn = key[i] < kmn ? key[i] : kmn;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t a1 = __shfl_xor_sync(0xffffffffu, kmx, o), b1 = __shfl_xor_sync(0xffffffffu, kmn, o);
        kmx = a1 > kmx ? a1 : kmx;
        kmn = b1 < kmn ? b1 : kmn;
      }
      __shared__ uint64_t s_mx[kHSW], s_mn[kHSW];
      if (lane == 0) {
        s_mx[tid >> 5] = kmx;
        s_mn[tid >> 5] = kmn;
      }
      __syncthreads();
      kmx = s_mx[0];
      kmn = s_mn[0];
      for (int w = 1; w < kHSW; ++w) {
        kmx = s_mx[w] > kmx ? s_mx[w] : kmx;
        kmn = s_mn[w] < kmn ? s_mn[w] : kmn;
      }
      const double rtop = key_f64(kmx);
      double tw = 0.0;
      for (int i = (int)tid; i < (int)H; i += kHSNT) tw += exp(key_f64(key[i]) - rtop);
      const double total_w = hs_sum(tw, S.red, S.bc);   // hot-set mass relative to the top value
      // threshold t: >= M keys are >= t (ties at it included)
      uint64_t t = kmn;
      if (kmx != kmn) {
        const int hb = 63 - __clzll((long long)(kmx ^ kmn));
        uint64_t prefix = kmx & ~((hb == 63) ? 0ull : ((2ull << hb) - 1ull));
        uint32_t need = (uint32_t)kHSNucM;
        for (int hi = hb;; hi -= 8) {
          const int lo = hi >= 7 ? hi - 7 : 0;
          const uint64_t hmask = (hi == 63) ? ~0ull : ((2ull << hi) - 1ull);   // bits <= hi
          for (int i = (int)tid; i < 256; i += kHSNT) hist[i] = 0u;
          __syncthreads();
          for (int i = (int)tid; i < (int)H; i += kHSNT) {
            const uint64_t kk = key[i];
            if ((kk & ~hmask) == prefix) atomicAdd(&hist[(uint32_t)((kk & hmask) >> lo)], 1u);
          }
          __syncthreads();
          if (tid < 32) {
            const DigitHit h = warp_find_digit(hist, need);
            if (tid == 0) {
              S.bcu[0] = h.digit;
              S.bcu[1] = h.above;
              S.bcu[2] = h.inbin;
            }
          }
          __syncthreads();
          prefix |= (uint64_t)S.bcu[0] << lo;
          need -= S.bcu[1];
          const bool done = S.bcu[2] == need || lo == 0;
          __syncthreads();
          if (done) break;
        }
        t = prefix;
      }
      if (tid == 0) S.bcu[3] = 0u;
      __syncthreads();
      for (int i = (int)tid; i < (int)H; i += kHSNT) {
        const uint64_t kk = key[i];
        if (kk >= t) {
          const uint32_t o = atomicAdd(&S.bcu[3], 1u);
          if (o < 256u) {
            ck[o] = kk;
            cpos[o] = pos[i];
          }
        }
      }
      __syncthreads();
      const uint32_t c = S.bcu[3];
      if (c <= 256u) {
        if (tid < 32) {
          warp_topk_sort(ck, cpos, c, c, hist);   // c > 64: sort only (no cut)
          for (uint32_t j = lane; j < c; j += 32) fr[j] = key_f64(ck[j]);
          __syncwarp();
          bool fb = false;
          const DrawResult d = warp_filter_draw_nuc(fr, (int32_t)c, knobs_of(p), u[0], total_w, fw, fc, fb);
          if (lane == 0) S.bcu[2] = fb ? 1u : 0u;
          if (!fb) {
            double margin = d.margin;
            if (!tail_empty && !deferred) margin = fmin(margin, fabs(u[1] - alpha));
            const int32_t tok = pos_to_id(a, (int64_t)cpos[d.index]);
            if (lane == 0) {
              a.token[row] = tok;
              a.logprob[row] = d.logprob;
              uint8_t fl = DP_FLAG_ACCEPTED_HOT;
              if (margin < kBoundaryEps) fl |= DP_FLAG_NEAR_BOUNDARY;
              a.flags[row] = fl;
              if (a.dbg.margin) a.dbg.margin[row] = margin;
              if (a.dbg.kept) a.dbg.kept[row] = d.kept;
              if (a.dbg.alpha) a.dbg.alpha[row] = alpha;
              if (deferred) push_resum(a, row, sH);   // the exact re-sum decides, then records
            }
            if (!deferred) warp_record_token(a, row, tok);   // fused K5
            if (a.dbg.topk_ids) {
              const int m = min((int)c, a.dbg.topk_stride);
              for (int j = (int)lane; j < m; j += 32) {
                a.dbg.topk_ids[(int64_t)row * a.dbg.topk_stride + j] = pos_to_id(a, (int64_t)cpos[j]);
                if (a.dbg.topk_ready) a.dbg.topk_ready[(int64_t)row * a.dbg.topk_stride + j] = fr[j];
              }
            }
          }
        }
        __syncthreads();
        const bool fb_all = S.bcu[2] != 0u;
        __syncthreads();
        if (!fb_all) continue;   // decided
      }
    }
    if (!sorted) {
      // bitonic over hp in shared memory; pairs of a warp stay inside its own
      // 64-entry segment while stride <= 32, so a stage needs only a warp sync
      // when it and the stage before it both have stride <= 32
      int prev = hp;
      for (int size = 2; size <= hp; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          if (stride > 32 || prev > 32) __syncthreads();
          else __syncwarp();
          prev = stride;
          const int sh_ = __ffs(stride) - 1;
          for (int i = (int)tid; i < hp / 2; i += kHSNT) {
            const int lo = ((i >> sh_) << (sh_ + 1)) + (i & (stride - 1));
            const int hi = lo + stride;
            const bool desc = (lo & size) == 0;
            const uint64_t ka = key[lo], kb = key[hi];
            const uint32_t pa = pos[lo], pb = pos[hi];
            const bool a_first = ka > kb || (ka == kb && pa < pb);
            if (a_first != desc) {
              key[lo] = kb; key[hi] = ka;
              pos[lo] = pb; pos[hi] = pa;
            }
          }
        }
      }
      __syncthreads();
    }
    // ---- 5. filter + draw over the first n entries (filtering.py:61-162)
    const double r0 = key_f64(key[0]);
    if (!(r0 > -INFINITY)) {   // no usable mass (DegenerateRowError, core.py:19-20)
      if (tid == 0) {
        a.token[row] = -1;
        a.logprob[row] = 0.0;
        a.flags[row] = DP_FLAG_DEGENERATE;
      }
      continue;
    }
    // contiguous chunk per thread: local f64 prefix, then the chunk offsets
    const int chunk = (n + kHSNT - 1) / kHSNT;
    const int j0 = min(n, (int)tid * chunk), j1 = min(n, j0 + chunk);
    double run = 0.0;
    for (int j = j0; j < j1; ++j) {
      run += exp(key_f64(key[j]) - r0);
      cum[j] = run;
    }
    // exclusive scan of the chunk totals (warp scan + warp offsets)
    double incl = warp_incl_scan(run);
    if (lane == 31) S.red[tid >> 5] = incl;
    __syncthreads();
    double woff = 0.0;
    for (uint32_t w = 0; w < (tid >> 5); ++w) woff += S.red[w];
    const double off = woff + incl - run;
    for (int j = j0; j < j1; ++j) cum[j] += off;
    __syncthreads();
    const double total = cum[n - 1];
    int kept = n;
    double margin = 1e30;
    if (p.top_p < 1.0) {   // filtering.py:91-95: 1 + first j with c_j >= top_p * c_{n-1}
      const double thr = p.top_p * total;
      uint32_t below = 0;
      for (int j = (int)tid; j < n; j += kHSNT) below += cum[j] < thr ? 1u : 0u;
      below = warp_sum(below);
      if (lane == 0) S.cnt[tid >> 5] = below;
      __syncthreads();
      uint32_t b2 = 0;
      for (int w = 0; w < kHSW; ++w) b2 += S.cnt[w];
      __syncthreads();
      const int kpp = (int)b2 + 1;
      kept = min(kept, kpp);
      for (int j = max(0, kpp - 2); j < min(n, kpp + 1); ++j) margin = fmin(margin, fabs(cum[j] - thr));
      margin = (double)__fdividef((float)margin, (float)total);
    }
    if (p.min_p > 0.0) {   // filtering.py:96-98 (w_0 = 1)
      uint32_t ge = 0;
      for (int j = (int)tid; j < n; j += kHSNT) ge += exp(key_f64(key[j]) - r0) >= p.min_p ? 1u : 0u;
      ge = warp_sum(ge);
      if (lane == 0) S.cnt2[tid >> 5] = ge;
      __syncthreads();
      uint32_t g2 = 0;
      for (int w = 0; w < kHSW; ++w) g2 += S.cnt2[w];
      __syncthreads();
      kept = min(kept, (int)g2);
      for (int j = max(0, (int)g2 - 1); j < min(n, (int)g2 + 1); ++j)
        margin = fmin(margin, fabs(exp(key_f64(key[j]) - r0) - p.min_p));
    }
    kept = max(1, kept);   // filtering.py:99
    const double Sk = cum[kept - 1];
    const double us = u[0] * Sk;
    uint32_t le = 0;   // j* = #(cdf_j <= u), clamped (filtering.py:158-162)
    for (int j = (int)tid; j < kept; j += kHSNT) le += cum[j] <= us ? 1u : 0u;
    le = warp_sum(le);
    if (lane == 0) S.cnt[tid >> 5] = le;
    __syncthreads();
    uint32_t le2 = 0;
    for (int w = 0; w < kHSW; ++w) le2 += S.cnt[w];
    const int js = min((int)le2, kept - 1);
    const int64_t hp_pos = (int64_t)pos[js];
    const int32_t tok = pos_to_id(a, hp_pos);
    if (tid == 0) {
      double dm = fabs(cum[js] - us);
      if (js > 0) dm = fmin(dm, fabs(cum[js - 1] - us));
      margin = fmin(margin, (double)__fdividef((float)dm, (float)Sk));
      if (!tail_empty && !deferred) margin = fmin(margin, fabs(u[1] - alpha));
      a.token[row] = tok;
      a.logprob[row] = (key_f64(key[js]) - r0) - log(Sk);   // ln(w_j / S), w_j = exp(r_j - r_0)
      uint8_t fl = DP_FLAG_ACCEPTED_HOT;
      if (margin < kBoundaryEps) fl |= DP_FLAG_NEAR_BOUNDARY;
      a.flags[row] = fl;
      if (a.dbg.margin) a.dbg.margin[row] = margin;
      if (a.dbg.kept) a.dbg.kept[row] = kept;
      if (a.dbg.alpha) a.dbg.alpha[row] = alpha;
      if (deferred) push_resum(a, row, sH);   // the exact re-sum decides, then records
    }
    if (!deferred && tid < 32) warp_record_token(a, row, tok);   // fused K5
    if (a.dbg.topk_ids) {
      const int m = min(n, a.dbg.topk_stride);
      for (int j = (int)tid; j < m; j += kHSNT) {
        a.dbg.topk_ids[(int64_t)row * a.dbg.topk_stride + j] = pos_to_id(a, (int64_t)pos[j]);
        if (a.dbg.topk_ready) a.dbg.topk_ready[(int64_t)row * a.dbg.topk_stride + j] = key_f64(key[j]);
      }
    }
  }
}

size_t hot_sort_smem(int64_t H) {
  int hp = 512;   // the top-k scratch (256 keys + positions) lives in the prefix array
  while (hp < H) hp <<= 1;
  const int cd = hp > kHSCumMin ? hp : kHSCumMin;
  return (size_t)hp * 12u + (size_t)cd * 8u + 1024u;   // keys + positions, prefix masses, radix histogram
}

cudaError_t launch_hot_sort(const SampleArgs& a, int dtype, cudaStream_t st) {
  int hp = 512;   // as hot_sort_smem
  while (hp < a.H) hp <<= 1;
  const size_t smem = hot_sort_smem(a.H);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e;
  if (dtype == DP_F32) {
    auto k = hot_sort_kernel<float>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kHSNT, smem);
  } else {
    auto k = hot_sort_kernel<__nv_bfloat16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kHSNT, smem);
  }
  if (e != cudaSuccess) return e;
  const int64_t slots = (int64_t)(per_sm > 0 ? per_sm : 1) * sms;
  const unsigned grid = (unsigned)(a.n_rows < slots ? (a.n_rows > 0 ? a.n_rows : 1) : slots);
  if (dtype == DP_F32) hot_sort_kernel<float><<<grid, kHSNT, smem, st>>>(a, hp);
  else hot_sort_kernel<__nv_bfloat16><<<grid, kHSNT, smem, st>>>(a, hp);
  return cudaGetLastError();
}

}  // namespace dp
