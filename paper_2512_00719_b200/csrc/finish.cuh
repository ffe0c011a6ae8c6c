// finish.cuh — per-row final stage shared by the streaming samplers: exact
// penalties on the sparse list (penalty.py:66-78), /tau (service.py:236-241),
// canonical ordering (filtering.py:83), top-p / min-p / inverse-CDF draw
// (filtering.py:61-162), and for SHVS the accept test (shvs.py:223-236).
#pragma once

#include "sampler.cuh"
#include "select.cuh"

namespace dp {

// shared-memory carve-up of the final stage
struct FinLayout {
  uint32_t key, r, w, cum, pos, hash, hash_cap, bytes, cap;   // cap: entries of each list array
};
__host__ __device__ inline FinLayout fin_layout(int lcap) {
  FinLayout f;
  f.hash_cap = 256;   // also the radix histogram of the top-k cut
  while (f.hash_cap < 2u * (uint32_t)lcap) f.hash_cap <<= 1;
  if (lcap < 256) lcap = 256;   // the sorts pad the list to a power of two >= 128
  f.cap = (uint32_t)lcap;
  uint32_t o = 0;
  f.key = o; o += lcap * 8u;
  f.r = o; o += lcap * 8u;
  f.w = o; o += lcap * 8u;
  f.cum = o; o += lcap * 8u;
  f.pos = o; o += lcap * 4u;
  f.hash = o; o += f.hash_cap * 4u;
  f.bytes = o;
  return f;
}

struct FinishScratch {
  uint32_t nl;
  uint32_t np;       // penalized entries of the domain (rank-merge path)
  uint32_t nq;       // ... that can enter the top-k
  uint32_t wc[32];   // per-warp counts of a block scan
  double sh_pen[32];
  double corr[32];
};

// Penalty entries of a row whose loads are issued early (before the
// selection) so their latency overlaps it: entries j = t + i*NT, i < 2.
struct PenPrefetch {
  float x[2];
  int32_t cnt[2];
  int32_t pos[2];   // domain position, -1 if absent / outside the domain
};

template <typename T, int NT>
DP_DEV PenPrefetch pen_prefetch(const SampleArgs& a, int row, int32_t plen, const T* rowp, int64_t lo, int64_t n,
                                uint32_t t) {
  PenPrefetch pp;
  const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
  const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int32_t j = (int32_t)t + i * NT;
    pp.pos[i] = -1;
    pp.x[i] = 0.f;
    pp.cnt[i] = 0;
    if (j < plen) {
      const int64_t pos = id_to_pos(a, pids[j]) - lo;
      if (pos >= 0 && pos < n) {
        pp.pos[i] = (int32_t)pos;
        pp.x[i] = dom_value<T>(a, row, rowp, pos);
        pp.cnt[i] = pcnt[j];
      }
    }
  }
  return pp;
}

// Descending bitonic sort of 32*E (u64 key, u32 pos) pairs held in registers
// by one warp; element i = j*32 + lane lives in slot j of lane `lane`.
// Order: key desc, pos asc (the canonical (value desc, id asc) rule).
// The (size, stride) stages are a rolled loop: the sort runs once per row with
// a cold instruction cache, and the fully unrolled network (thousands of
// instructions for E = 8) was fetched from L2 line by line every row
// (no_instructions stalls, profiles/r2); only the slot loop is unrolled so the
// register arrays stay in registers.
template <int E, int JS>
DP_DEV void warp_reg_sort_cross(uint64_t (&key)[E], uint32_t (&pos)[E], uint32_t lane, int size) {
#pragma unroll
  for (int j = 0; j < E; ++j) {
    if ((j & JS) == 0) {
      const int jp = j | JS;
      const uint32_t i = (uint32_t)j * 32u + lane;
      const bool desc = (i & (uint32_t)size) == 0u;
      const bool a_first = key[j] > key[jp] || (key[j] == key[jp] && pos[j] < pos[jp]);
      if (a_first != desc) {
        const uint64_t tk = key[j]; key[j] = key[jp]; key[jp] = tk;
        const uint32_t tp = pos[j]; pos[j] = pos[jp]; pos[jp] = tp;
      }
    }
  }
}
template <int E>
DP_DEV void warp_reg_sort(uint64_t (&key)[E], uint32_t (&pos)[E]) {
  const uint32_t lane = lane_id();
  constexpr int N = 32 * E;
#pragma unroll 1
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll 1
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int js = stride / 32;
        if constexpr (E >= 2) { if (js == 1) warp_reg_sort_cross<E, 1>(key, pos, lane, size); }
        if constexpr (E >= 4) { if (js == 2) warp_reg_sort_cross<E, 2>(key, pos, lane, size); }
        if constexpr (E >= 8) { if (js == 4) warp_reg_sort_cross<E, 4>(key, pos, lane, size); }
      } else {
        const bool lower = (lane & (uint32_t)stride) == 0u;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const uint64_t ok = __shfl_xor_sync(0xffffffffu, key[j], stride);
          const uint32_t op = __shfl_xor_sync(0xffffffffu, pos[j], stride);
          const uint32_t i = (uint32_t)j * 32u + lane;
          const bool desc = (i & (uint32_t)size) == 0u;
          const bool mine_first = key[j] > ok || (key[j] == ok && pos[j] < op);
          const bool keep_mine = (lower == desc) ? mine_first : !mine_first;
          if (!keep_mine) {
            key[j] = ok;
            pos[j] = op;
          }
        }
      }
    }
  }
}

// The k largest of fkey[0,nl) (duplicates allowed) by (key desc, pos asc),
// sorted into fkey/fpos[0, min(k,nl)).  One warp; arrays hold >= 256 entries
// (>= nl).  For k <= 64 a radix cut first keeps every key >= the k-th largest
// (ties at the cut included), so usually only 64 entries are sorted; nl <= 256
// otherwise.  hist: 256 u32 scratch.
template <int E>
DP_DEV void warp_sort_regs(uint64_t* fkey, uint32_t* fpos);

// k rounds of warp arg-max: only for lists of > 256 tied survivors
DP_DEV void warp_select_sort_slow(uint64_t* fkey, uint32_t* fpos, uint32_t c, uint32_t k) {
  const uint32_t lane = lane_id();
  for (uint32_t i = 0; i < k && i < c; ++i) {
    uint64_t bk = 0ull;
    uint32_t bp = 0xFFFFFFFFu, bi = 0xFFFFFFFFu;
    for (uint32_t j = i + lane; j < c; j += 32) {
      const uint64_t kk = fkey[j];
      const uint32_t pp = fpos[j];
      if (bi == 0xFFFFFFFFu || kk > bk || (kk == bk && pp < bp)) { bk = kk; bp = pp; bi = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const uint32_t op = __shfl_xor_sync(0xffffffffu, bp, o);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oi != 0xFFFFFFFFu && (bi == 0xFFFFFFFFu || ok > bk || (ok == bk && op < bp))) { bk = ok; bp = op; bi = oi; }
    }
    __syncwarp();
    if (lane == 0) {
      fkey[bi] = fkey[i];
      fpos[bi] = fpos[i];
      fkey[i] = bk;
      fpos[i] = bp;
    }
    __syncwarp();
  }
}

DP_DEV void warp_topk_sort(uint64_t* fkey, uint32_t* fpos, uint32_t nl, uint32_t k, uint32_t* hist) {
  const uint32_t lane = lane_id();
  uint32_t c = nl;
  if (k <= 64 && nl > 64) {
    uint64_t prefix = 0, mask = 0;
    uint32_t need = k;
    for (int shift = 56; shift >= 0; shift -= 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) hist[lane + 32 * i] = 0u;
      __syncwarp();
      for (uint32_t i = lane; i < nl; i += 32) {
        const uint64_t kk = fkey[i];
        if ((kk & mask) == prefix) atomicAdd(&hist[(uint32_t)(kk >> shift) & 255u], 1u);
      }
      __syncwarp();
      const DigitHit h = warp_find_digit(hist, need);
      prefix |= (uint64_t)h.digit << shift;
      mask |= 255ull << shift;
      need -= h.above;
      __syncwarp();
      if (h.inbin == need) break;
    }
    // keys >= prefix: the whole cut bucket, or (walk ran to the last digit)
    // everything above plus all ties at the k-th value
    uint32_t out = 0;
    for (uint32_t base = 0; base < nl; base += 32) {
      const uint32_t i = base + lane;
      const uint64_t kk = i < nl ? fkey[i] : 0ull;
      const uint32_t pp = i < nl ? fpos[i] : 0u;
      const bool keep = i < nl && kk >= prefix;
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) {
        const uint32_t o = out + __popc(m & lanemask_lt());
        fkey[o] = kk;
        fpos[o] = pp;
      }
      out += __popc(m);
      __syncwarp();
    }
    c = out;
  }
  if (c > 256) {
    warp_select_sort_slow(fkey, fpos, c, k);
    return;
  }
  const uint32_t cp = c <= 64 ? 64u : (c <= 128 ? 128u : 256u);
  for (uint32_t i = c + lane; i < cp; i += 32) {
    fkey[i] = 0ull;
    fpos[i] = 0xFFFFFFFFu;
  }
  __syncwarp();
  if (c <= 64) warp_sort_regs<2>(fkey, fpos);
  else if (c <= 128) warp_sort_regs<4>(fkey, fpos);
  else warp_sort_regs<8>(fkey, fpos);
}

template <int E>
DP_DEV void warp_sort_regs(uint64_t* fkey, uint32_t* fpos) {
  const uint32_t lane = lane_id();
  uint64_t k[E];
  uint32_t p[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    k[j] = fkey[j * 32 + lane];
    p[j] = fpos[j * 32 + lane];
  }
  warp_reg_sort<E>(k, p);
#pragma unroll
  for (int j = 0; j < E; ++j) {
    fkey[j * 32 + lane] = k[j];
    fpos[j * 32 + lane] = p[j];
  }
  __syncwarp();
}

// Runs on NT cooperating threads (thread index `t`); `sync` is their barrier.
// sel[0..nsel): unique (value desc, position asc) keys of the raw candidates.
// `pp` holds the prefetched first 2*NT penalty entries.
// Returns false when a kHot row was rejected (token left to the tail pass).
template <typename T, int MODE, int NT, bool NUC, bool PX, typename Sync>
DP_DEV bool finish_row(const SampleArgs& a, int row, const dp_params_t& p, int32_t plen, const T* rowp,
                       int64_t lo, int64_t n, const uint64_t* sel, uint32_t nsel, double sh_unpen, double mrow,
                       uint8_t* fin, const FinLayout& F, FinishScratch& fs, uint32_t t, Sync sync,
                       const PenPrefetch* pp = nullptr, float cref = 0.f) {
  const uint32_t warp = t >> 5, lane = t & 31u;
  // nucleus rows (top-k off): the list holds the kNucK largest; sh_unpen is
  // the domain mass (kHot: hot mass relative to mrow; kFull / kTail: every
  // element's f32 term relative to cref, penalized ones swapped below)
  const bool nuc = NUC && nucleus_row(p.top_k, n);
  const int32_t k = nuc ? effective_k(p.top_k, n) : p.top_k;
  const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
  const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;
  uint64_t* fkey = reinterpret_cast<uint64_t*>(fin + F.key);
  double* fr = reinterpret_cast<double*>(fin + F.r);
  double* fw = reinterpret_cast<double*>(fin + F.w);
  double* fcum = reinterpret_cast<double*>(fin + F.cum);
  uint32_t* fpos = reinterpret_cast<uint32_t*>(fin + F.pos);
  uint32_t* hash = reinterpret_cast<uint32_t*>(fin + F.hash);
  uint32_t hcap = 64;
  while (hcap < 2u * (uint32_t)plen) hcap <<= 1;
  if (hcap > F.hash_cap) hcap = F.hash_cap;
  const uint32_t hmask = hcap - 1u;
  double u[3];
  get_uniforms(a, row, p, u);
#ifdef DP_TIMELINE   // A-B build: globaltimer marks of the final stage's phases -> dbg.topk_ready[row * stride + 5..7]
  uint64_t tm[4] = {0, 0, 0, 0};
  auto tmark = [&](int i) {
    if (t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm[i]));
  };
#else
  auto tmark = [](int) {};
#endif
  tmark(0);
  const bool prof = a.dbg.stats != nullptr && t == 0;
  long long pc = prof ? clock64() : 0;
  auto lap = [&](int slot) {
    if (prof) {
      const long long now = clock64();
      atomicAdd((unsigned long long*)&a.dbg.stats[slot], (unsigned long long)(now - pc));
      pc = now;
    }
  };

  if (t == 0) touch_bytes(a, row, (uint64_t)plen * sizeof(T));   // gathered penalty values
  // penalty entry e: (domain position, x, count), from the prefetch or memory
  auto pen_entry = [&](int32_t j, int32_t& pos, float& x, int32_t& c) {
    const int i = (j - (int32_t)t) / NT;
    if (pp != nullptr && i < 2) {
      pos = pp->pos[i];
      x = pp->x[i];
      c = pp->cnt[i];
      return;
    }
    const int64_t q = id_to_pos(a, pids[j]) - lo;
    pos = (q >= 0 && q < n) ? (int32_t)q : -1;
    x = pos >= 0 ? dom_value<T>(a, row, rowp, q) : 0.f;
    c = pcnt[j];
  };

  // kHot: alpha and the accept test first (shvs.py:223-236)
  double alpha = 1.0;
  bool deferred = false;     // kHot: accept test left to the exact re-sum
  double s_dom = sh_unpen;   // nucleus: mass of the whole domain (see above)
  if (MODE == kHot) {
    double spen = 0.0;   // exact mass of penalized hot ids (f64)
    for (int32_t j = t; j < plen; j += NT) {
      int32_t pos, c;
      float x;
      pen_entry(j, pos, x, c);
      if (pos >= 0) spen += exp(ready_penalized(x, c, p) - mrow);
    }
    double scorr = 0.0;   // raw producer summary -> penalized total (shvs.py:148-154 needs the ready row)
    if (a.summary_raw)
      scorr = raw_summary_correction(a, row, p, plen, mrow, t, NT,
                                     [&](int64_t pos) { return row_value<T>(a, row, pos); });
    spen = warp_sum(spen);
    scorr = warp_sum(scorr);
    if (lane == 0) {
      fs.sh_pen[warp] = spen;
      fs.corr[warp] = scorr;
    }
    sync();
    double sH = sh_unpen, corr = 0.0;
    for (int w = 0; w < NT / 32; ++w) {   // fixed order: deterministic
      sH += fs.sh_pen[w];
      corr += fs.corr[w];
    }
    s_dom = sH;
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
      if (t == 0) {
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
      sync();
      return false;
    }
  }

  // penalized positions of this domain -> hash set (raw candidates defer to
  // them).  kHot, and long lists (a.pen_excl), streamed around the penalized
  // ids already: no hash set needed
  constexpr bool excl = MODE == kHot || PX;   // PX: penalized ids outside the stream (a.pen_excl)
  if (t == 0) {
    fs.nl = 0u;
    fs.np = 0u;
    fs.nq = 0u;
  }
  if (!excl)
    for (uint32_t i = t; i < hcap; i += NT) hash[i] = 0xFFFFFFFFu;
  sync();
  lap(8);
  const bool nuc_mass = nuc && MODE != kHot;
  const float s2 = (float)(1.4426950408889634 / p.temperature);
  const double cref_r = (double)cref / p.temperature;   // cref in ready units
  // Long lists with the penalized ids outside the stream: only the k best
  // penalized entries (ties at the k-th value included) can enter the ready
  // top-k, so only those are kept — a radix threshold over their exact f64
  // keys, computed on the fly from the (L2-hot) list and logits.
  // rank merge (O(nsel^2 / NT) compares per thread) for short candidate lists;
  // longer ones (long penalty lists: kp = k + |list|) take the radix cut +
  // register sort of one warp
// Rank sort when nsel^2 / NT compares per thread stay small.  On an idle SM
// (latency: the SHVS hot / tail passes) it beats the one-warp radix cut +
// register sort up to ~240 compares per thread (tools/micro/finish_only.cu:
// NT 96, nsel 80: 20.9k -> 9.8k cycles; NT 256, nsel 150: 20.9k -> 13.6k;
// SHVS C2 71.3 -> 70.0 us).  With full rows streaming beside it (throughput:
// K1 / K1p) its extra issue slots cost more than they save (C4 unchanged,
// C2 +0.4 us at 240), so the full path keeps the tighter bound.
#ifndef DP_RANK_MAX_ITERS
#define DP_RANK_MAX_ITERS 48
#endif
#ifndef DP_RANK_MAX_ITERS_SHVS
#define DP_RANK_MAX_ITERS_SHVS 240
#endif
  const bool fast = nsel * nsel <= (uint32_t)(MODE == kFull ? DP_RANK_MAX_ITERS : DP_RANK_MAX_ITERS_SHVS) * NT;
  // with the penalized ids outside the stream the fast path keeps them only
  // once the k-th unpenalized ready value rk is known: one pass, entries
  // >= rk (late_pen); the other paths pick the k best by a radix threshold
  const bool late_pen = PX && fast && plen > 0;
  auto get_p = [&](uint32_t j, uint64_t& key) -> bool {
    int32_t pos, c;
    float x;
    pen_entry((int32_t)j, pos, x, c);
    if (pos < 0) return false;
    key = f64_key(ready_penalized(x, c, p));
    return true;
  };
  // the k best penalized entries' threshold key (ties at the k-th included)
  auto pen_threshold = [&]() -> uint64_t {
    uint32_t cv = 0;
    for (int32_t j = t; j < plen; j += NT) {
      uint64_t kk;
      cv += get_p((uint32_t)j, kk) ? 1u : 0u;
    }
    cv = warp_sum(cv);
    if (lane == 0) fs.wc[warp] = cv;
    sync();
    uint32_t cnt_p = 0;
    for (int w = 0; w < NT / 32; ++w) cnt_p += fs.wc[w];
    sync();
    return group_select_threshold<NT>(get_p, (uint32_t)plen, cnt_p, (uint32_t)k, hash, fs.wc, t, sync);
  };
  uint64_t p_thr = 0ull;
  const bool psel = excl && !late_pen && plen > kPenSelCap;
  if (psel) p_thr = pen_threshold();
  const uint32_t pcap = F.cap - (uint32_t)k - 1u;   // penalized slots next to the k unpenalized ones
  // the rank-merge path keeps the penalized entries apart: ready values in
  // fcum, positions at the top of fpos (k + 2 |kept list| < lcap: no overlap)
  double m_sub = 0.0, m_add = 0.0;
  for (int32_t j = t; j < plen && (!late_pen || nuc_mass); j += NT) {
    int32_t pos, c;
    float x;
    pen_entry(j, pos, x, c);
    if (pos >= 0) {
      if (!excl) {
        uint32_t h = ((uint32_t)pos * 2654435761u) & hmask;
        while (atomicCAS(&hash[h], 0xFFFFFFFFu, (uint32_t)pos) != 0xFFFFFFFFu) h = (h + 1u) & hmask;
      }
      const double r = ready_penalized(x, c, p);
      if (!late_pen && (!psel || f64_key(r) >= p_thr)) {
        if (fast) {
          const uint32_t s = atomicAdd(&fs.np, 1u);
          if (s < pcap) {   // (ties at the k-th penalized value beyond kPenSelCap - k: not kept)
            fcum[s] = r;
            fpos[F.cap - 1u - s] = (uint32_t)pos;
          }
        } else {
          const uint32_t s = atomicAdd(&fs.nl, 1u);
          if (s < F.cap) {
            fkey[s] = f64_key(r);
            fpos[s] = (uint32_t)pos;
          }
        }
      }
      if (nuc_mass) {   // swap the streamed f32 term (bit-identical) for the exact one
        m_sub += (double)ex2_fast(((x - cref) - 0.f) * s2);
        m_add += exp(r - cref_r);
      }
    }
  }
  if (nuc_mass) {
    m_sub = warp_sum(m_sub);
    m_add = warp_sum(m_add);
    if (lane == 0) {
      fs.sh_pen[warp] = m_sub;
      fs.corr[warp] = m_add;
    }
  }
  sync();
  if (t == 0) {
    if (fs.np > pcap) fs.np = pcap;
    if (fs.nl > F.cap) fs.nl = F.cap;
  }
  sync();
  if (nuc_mass) {
    for (int w = 0; w < NT / 32; ++w) s_dom += fs.corr[w] - fs.sh_pen[w];   // fixed order
  }
  lap(12);
  tmark(1);
  auto penalized = [&](uint32_t pos) -> bool {
    if (excl || plen == 0) return false;
    uint32_t h = (pos * 2654435761u) & hmask;
    while (true) {
      const uint32_t hv = hash[h];
      if (hv == pos) return true;
      if (hv == 0xFFFFFFFFu) return false;
      h = (h + 1u) & hmask;
    }
  };
  uint32_t nl;
  if (fast) {
    // (1) rank sort of the raw candidates (unique composite keys): O(nsel^2 / NT)
    for (uint32_t i = t; i < nsel; i += NT) {
      const uint64_t key = sel[i];
      uint32_t rank = 0;
      for (uint32_t j = 0; j < nsel; ++j) rank += sel[j] > key ? 1u : 0u;
      fkey[rank] = key;
    }
    sync();
    lap(9);
    // (2) the k largest unpenalized, in order: their ready values keep the raw
    // order (x / tau is monotone), so a prefix count over the sorted keys ranks
    // them; list U -> (fw, fpos)[0 .. nu)
    uint32_t base_u = 0;
    for (uint32_t c0 = 0; c0 < nsel; c0 += NT) {
      const uint32_t i = c0 + t;
      const uint64_t key = i < nsel ? fkey[i] : 0ull;
      const uint32_t pos = comp_pos(key);
      const bool unpen = i < nsel && !penalized(pos);
      const uint32_t bal = __ballot_sync(0xffffffffu, unpen);
      if (lane == 0) fs.wc[warp] = __popc(bal);
      sync();
      uint32_t before = base_u, total = 0;
      for (int w = 0; w < NT / 32; ++w) {
        if (w < (int)warp) before += fs.wc[w];
        total += fs.wc[w];
      }
      before += __popc(bal & lanemask_lt());
      if (unpen && before < (uint32_t)k) {
        fw[before] = ready_plain(comp_val(key), p);
        fpos[before] = pos;
      }
      base_u += total;
      sync();
    }
    const uint32_t nu = min(base_u, (uint32_t)k);
    lap(10);
    // (3) a penalized id can enter the ready top-k only if it reaches the k-th
    // unpenalized (ties kept: the merge orders them)
    const bool full_k = base_u >= (uint32_t)k;
    const double rk = full_k ? fw[k - 1] : -INFINITY;
    if (late_pen) {
      // keep the penalized entries >= rk; if more than fit, only the k best
      // of them can matter (radix threshold), so keep those >= both
      // batched: each thread issues the list loads of 4 entries, then their
      // 4 logit gathers, so 4 entries cost two memory round trips, not 8
      auto keep_pen = [&](uint64_t floor_key) {
        constexpr int UB = 4;
        for (int32_t base = (int32_t)t; base < plen; base += NT * UB) {
          int32_t q[UB], c[UB];
          float x[UB];
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int32_t j = base + u * NT;
            q[u] = -1;
            c[u] = 0;
            if (j < plen) {
              const int64_t qq = id_to_pos(a, pids[j]) - lo;
              q[u] = (qq >= 0 && qq < n) ? (int32_t)qq : -1;
              c[u] = pcnt[j];
            }
          }
#pragma unroll
          for (int u = 0; u < UB; ++u) x[u] = q[u] >= 0 ? dom_value<T>(a, row, rowp, q[u]) : 0.f;
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            if (q[u] < 0) continue;
            const double r = ready_penalized(x[u], c[u], p);
            if (r >= rk && f64_key(r) >= floor_key) {
              const uint32_t s2i = atomicAdd(&fs.np, 1u);
              if (s2i < pcap) {
                fcum[s2i] = r;
                fpos[F.cap - 1u - s2i] = (uint32_t)q[u];
              }
            }
          }
        }
        sync();
      };
      keep_pen(0ull);
      if (fs.np > pcap) {
        const uint64_t thr_k = pen_threshold();
        if (t == 0) fs.np = 0u;
        sync();
        keep_pen(thr_k);
      }
      if (t == 0 && fs.np > pcap) fs.np = pcap;
      sync();
    }
    const uint32_t np = fs.np;
    lap(11);
    // (4) rank merge of U and the qualifying penalized entries P into
    // (fr, hash)[0 .. m), m = min(k, nu + |P|); order (ready desc, pos asc)
    auto before_ = [](double ra, uint32_t pa, double rb, uint32_t pb) -> bool {
      return ra > rb || (ra == rb && pa < pb);
    };
    for (uint32_t i = t; i < nu; i += NT) {
      const double r = fw[i];
      const uint32_t pos = fpos[i];
      uint32_t f = i;
      for (uint32_t j = 0; j < np; ++j)
        if (fcum[j] >= rk && before_(fcum[j], fpos[F.cap - 1u - j], r, pos)) ++f;
      if (f < (uint32_t)k) {
        fr[f] = r;
        hash[f] = pos;
      }
    }
    for (uint32_t j = t; j < np; j += NT) {
      const double r = fcum[j];
      if (!(r >= rk)) continue;
      atomicAdd(&fs.nq, 1u);
      const uint32_t pos = fpos[F.cap - 1u - j];
      uint32_t f = 0;
      for (uint32_t q = 0; q < np; ++q)
        if (fcum[q] >= rk && before_(fcum[q], fpos[F.cap - 1u - q], r, pos)) ++f;
      for (uint32_t q = 0; q < nu; ++q)
        if (before_(fw[q], fpos[q], r, pos)) ++f;
      if (f < (uint32_t)k) {
        fr[f] = r;
        hash[f] = pos;
      }
    }
    sync();
    nl = min((uint32_t)k, nu + fs.nq);
    for (uint32_t i = t; i < nl; i += NT) fpos[i] = hash[i];
    sync();
  } else {
    for (uint32_t i = t; i < nsel; i += NT) {
      const uint64_t key = sel[i];
      const uint32_t pos = comp_pos(key);
      if (!penalized(pos)) {
        const uint32_t s = atomicAdd(&fs.nl, 1u);
        fkey[s] = f64_key(ready_plain(comp_val(key), p));
        fpos[s] = pos;
      }
    }
    sync();
    nl = fs.nl;
    uint32_t p2 = 128;
    while (p2 < nl) p2 <<= 1;
    for (uint32_t i = nl + t; i < p2; i += NT) {
      fkey[i] = 0ull;
      fpos[i] = 0xFFFFFFFFu;
    }
    sync();
    lap(13);
    // canonical order (ready desc, position asc): one warp through registers
    // for short lists, all NT threads in shared memory otherwise
    if (p2 <= 256 || k <= 64) {   // warp_topk_sort cuts any list to the top k <= 64 first
      if (warp == 0) {
        warp_topk_sort(fkey, fpos, nl, (uint32_t)k, hash);
        const uint32_t m = min((uint32_t)k, nl);
        for (uint32_t i = lane; i < m; i += 32) {
          const uint64_t kk = fkey[i];
          const uint64_t bb = (kk >> 63) ? (kk & 0x7FFFFFFFFFFFFFFFull) : ~kk;
          fr[i] = __longlong_as_double((long long)bb);
        }
        __syncwarp();
      }
    } else {
      for (uint32_t size = 2; size <= p2; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
          for (uint32_t i = t; i < p2 / 2; i += NT) {
            const uint32_t lo_i = 2 * stride * (i / stride) + (i % stride);
            const uint32_t hi_i = lo_i + stride;
            const bool desc = ((lo_i & size) == 0);
            const uint64_t ka = fkey[lo_i], kb = fkey[hi_i];
            const uint32_t pa = fpos[lo_i], pb = fpos[hi_i];
            const bool a_first = ka > kb || (ka == kb && pa < pb);
            if (a_first != desc) {
              fkey[lo_i] = kb; fkey[hi_i] = ka;
              fpos[lo_i] = pb; fpos[hi_i] = pa;
            }
          }
          sync();
        }
      for (uint32_t i = t; i < nl; i += NT) {
        const uint64_t kk = fkey[i];
        const uint64_t bb = (kk >> 63) ? (kk & 0x7FFFFFFFFFFFFFFFull) : ~kk;
        fr[i] = __longlong_as_double((long long)bb);
      }
      sync();
    }
  }

  lap(14);
  tmark(2);
  if (warp == 0) {
    const double ud = u[MODE == kTail ? 2 : 0];
    // no usable mass: every candidate is -inf (DegenerateRowError, core.py:19-20)
    const bool degen = !(nl > 0 && fr[0] > -INFINITY);
    bool fb = false;
    DrawResult d;
    if (degen) {
    } else if (nuc) {
      // domain mass relative to the top ready value r[0]
      const double ref = MODE == kHot ? mrow : cref_r;
      const double total = s_dom * exp(ref - fr[0]);
      if (!(total > 0.0) || !isfinite(total)) fb = true;   // e.g. the first batch missed the row's scale
      else d = warp_filter_draw_nuc(fr, (int32_t)min((uint32_t)k, nl), knobs_of(p), ud, total, fw, fcum, fb);
    } else {
      d = warp_filter_draw(fr, (int32_t)min((uint32_t)k, nl), knobs_of(p), ud, fw, fcum, a.dbg.stats);
    }
    lap(16);
    tmark(3);

    if (degen) {
      if (lane == 0) {
        a.token[row] = -1;
        a.logprob[row] = 0.0;
        a.flags[row] = DP_FLAG_DEGENERATE | (MODE == kTail ? DP_FLAG_REJECTED : 0);
      }
    } else if (fb) {
      if (lane == 0) a.fb_rows[atomicAdd(a.fb_count, 1)] = row;   // the general kernel decides it
    } else if (lane == 0) {
      const int64_t pos = (int64_t)fpos[d.index] + lo;
      a.token[row] = pos_to_id(a, pos);
      a.logprob[row] = d.logprob;
      uint8_t fl = MODE == kHot ? DP_FLAG_ACCEPTED_HOT : (MODE == kTail ? DP_FLAG_REJECTED : 0);
      double margin = d.margin;
      if (MODE == kHot && a.V != a.H && !deferred) margin = fmin(margin, fabs(u[1] - alpha));
      if (margin < kBoundaryEps) fl |= DP_FLAG_NEAR_BOUNDARY;
      if (MODE == kTail) fl |= a.flags[row] & DP_FLAG_NEAR_BOUNDARY;
      a.flags[row] = fl;
      if (a.dbg.margin) a.dbg.margin[row] = MODE == kTail ? fmin(margin, a.dbg.margin[row]) : margin;
      if (a.dbg.kept) a.dbg.kept[row] = d.kept;
      if (MODE == kHot && a.dbg.alpha) a.dbg.alpha[row] = alpha;
    }
    if (deferred && !fb && !degen && lane == 0) push_resum(a, row, s_dom);   // re-sum decides, then records
    if (!fb && !degen && !deferred) warp_record_token(a, row, pos_to_id(a, (int64_t)fpos[d.index] + lo));   // fused K5
    if (a.dbg.topk_ids && !fb && !degen) {
      const int32_t m = min(k, a.dbg.topk_stride);
      for (int32_t j = lane; j < m; j += 32) {
        a.dbg.topk_ids[(int64_t)row * a.dbg.topk_stride + j] = pos_to_id(a, (int64_t)fpos[j] + lo);
        if (a.dbg.topk_ready) a.dbg.topk_ready[(int64_t)row * a.dbg.topk_stride + j] = fr[j];
      }
    }
  }
  sync();
  lap(15);
#ifdef DP_TIMELINE   // (after the top-k debug values, which share the row's slots)
  if (t == 0 && a.dbg.topk_ready && a.dbg.topk_stride >= 8) {
    double* tl = a.dbg.topk_ready + (int64_t)row * a.dbg.topk_stride;
    tl[5] = (double)(tm[1] - tm[0]);
    tl[6] = (double)(tm[2] - tm[1]);
    tl[7] = (double)(tm[3] - tm[2]);
  }
#endif
  return true;
}

}  // namespace dp
