// sample_stream.cu — persistent, warp-specialised, TMA-fed top-k sampler
// (K1 for batches that fill the GPU).
//
// One CTA per SM, three warp roles:
//   * producer (1 warp): pulls rows from a device work counter and streams
//     each row through a ring of S shared-memory stages with 1-D TMA bulk
//     copies (cp.async.bulk ... mbarrier::complete_tx, L2 evict_first),
//     running ahead into the next row;
//   * streamers (8 warps): per stage, compare every element with the row's
//     admission threshold and append whole 16-byte vectors holding a survivor
//     to one of two candidate buffers;
//   * finishers (4 warps): while the streamers already consume row r+1, take
//     row r's candidate buffer, verify it, run the exact radix selection of the
//     raw top-(k + |penalty list|) (the _tail_preselect superset,
//     service.py:309-336) and the exact final stage (finish.cuh).
// In-flight bytes live in shared memory (128 KB ring), so the SM's share of
// HBM stays busy through every per-row step, and the grid has no
// wave-quantisation tail.
//
// Threshold: from the first stage of a row, t_est = the r-th largest of the
// streamers' lane maxima, r sized to admit ~3 kp elements; t_lb = a proven
// lower bound of the kp-th largest.  The finishers verify that >= kp
// survivors passed; otherwise (or on buffer overflow) they re-stream the row
// from global memory with t_lb (or the buffer's kp-th key), so the result
// never depends on the estimate.

#include "finish.cuh"
#include "sampler.cuh"
#include "select.cuh"

namespace dp {

constexpr int kStreamChunk = 16384;   // bytes per ring stage
constexpr int kStreamStages = 8;
constexpr int kNS = 256;              // streamer threads (8 warps)
constexpr int kNF = 128;              // finisher threads per group (4 warps)
constexpr int kNG = 2;                // finisher groups (rows alternate)
constexpr int kNB = 3;                // candidate buffers (streamers + 2 groups)
constexpr int kStreamThreads = kNS + 32 + kNG * kNF;
constexpr int kProducerWarp = kNS / 32;
constexpr int kFirstFinisherWarp = kProducerWarp + 1;

struct StageMeta {
  int32_t row;      // -1: no more work
  int32_t chunk;
  int32_t nchunks;
  int32_t nvec;     // 16-byte vectors in this stage
};

// hand-off record of one candidate buffer (streamers -> finishers)
struct RowRec {
  int32_t row;      // -1: no more rows
  uint32_t kp;
  uint64_t thr;
  float t_lb;
  int32_t a0, nvec, plen;
  uint32_t cnt, overflow;
  double sh;        // kHot: unpenalized hot mass of the streamed elements
};

struct StreamSmem {
  uint64_t full[kStreamStages];
  uint64_t empty[kStreamStages];
  uint64_t cfull[kNB];
  uint64_t cempty[kNB];
  StageMeta meta[kStreamStages];
  RowRec rec[kNB];
  float thr_warp[8];
  uint32_t top4[32];
  double sh_warp[8];
  uint32_t tmp[kNG];
  uint32_t bcast[kNG][4];
  FinishScratch fin[kNG];
};

struct StreamLayout {
  uint32_t ring, cand, cand_bytes, fin, fin_bytes, sel, sel_bytes, hist_s, hist_f, bitmap, bitmap_bytes, misc, total;
};
__host__ __device__ inline StreamLayout stream_layout(int ccap, int kcap, int lcap, int bitmap_words) {
  StreamLayout L;
  uint32_t o = 0;
  L.ring = o; o += kStreamStages * kStreamChunk;
  L.cand_bytes = ((uint32_t)ccap * 8u + 127u) & ~127u;   // composite keys
  L.cand = o; o += kNB * L.cand_bytes;
  L.fin_bytes = (fin_layout(lcap).bytes + 127u) & ~127u;  // per finisher group
  L.fin = o; o += kNG * L.fin_bytes;
  L.sel_bytes = ((uint32_t)kcap * 8u + 15u) & ~15u;
  L.sel = o; o += kNG * L.sel_bytes;
  L.hist_s = o; o += 256u * 4u;
  L.hist_f = o; o += kNG * 256u * 4u;
  L.bitmap_bytes = ((uint32_t)bitmap_words * 4u + 15u) & ~15u;
  L.bitmap = o; o += kNB * L.bitmap_bytes;
  L.misc = o; o += (sizeof(StreamSmem) + 15u) & ~15u;
  L.total = o;
  return L;
}

// same routing rule as topk_sample_kernel / the general path
template <int MODE>
DP_DEV bool topk_route(const SampleArgs& a, const dp_params_t& p, int32_t plen, int64_t n) {
  return route_row(a, MODE, p.top_k, plen, n) == kRouteTopk;
}

template <typename T, int MODE>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_sample_kernel(SampleArgs a, int32_t* work) {
  constexpr int NWS = kNS / 32;
  constexpr int EPV = Elem<T>::kPerVec;
  constexpr int VPS = kStreamChunk / 16;   // vectors per stage
  extern __shared__ __align__(128) uint8_t smem[];
  const int64_t n = dom_n(a, MODE);
  const int64_t lo = dom_lo(a, MODE);
  const uint32_t bm_words = MODE == kHot ? (uint32_t)((n + 31) / 32) : 0u;
  const StreamLayout L = stream_layout(a.wcap, a.kcap, a.lcap, (int)bm_words);
  const uint8_t* ring = smem + L.ring;
  const uint32_t ccap = (uint32_t)a.wcap;   // candidate keys per buffer
  StreamSmem& ms = *reinterpret_cast<StreamSmem*>(smem + L.misc);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;

  auto cbuf = [&](int b) { return reinterpret_cast<uint64_t*>(smem + L.cand + b * L.cand_bytes); };
  auto bmap = [&](int b) { return reinterpret_cast<uint32_t*>(smem + L.bitmap + b * L.bitmap_bytes); };

  if (tid == 0) {
    for (int s = 0; s < kStreamStages; ++s) {
      mbar_init(&ms.full[s], 1);
      mbar_init(&ms.empty[s], NWS);
    }
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&ms.cfull[b], 1);
      mbar_init(&ms.cempty[b], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int nrows = a.row_count ? *a.row_count : a.n_rows;

  // ================================================================ producer
  if (warp == kProducerWarp) {
    if (lane != 0) return;
    const uint64_t pol = l2_evict_first_policy();
    int stage = 0;
    uint32_t phase = 0;
    while (true) {
      const int ridx = atomicAdd(work, 1);
      if (ridx >= nrows) break;
      const int row = a.rows ? a.rows[ridx] : ridx;
      const dp_params_t p = a.params[row];
      const int32_t plen = pen_len(a, row, p);
      if (!topk_route<MODE>(a, p, plen, n)) continue;          // general-path row
      const T* rowp = domain_row<T>(a, row, MODE);
      const uintptr_t addr = reinterpret_cast<uintptr_t>(rowp);
      const int64_t a0 = min64(n, (int64_t)(((16u - (addr & 15u)) & 15u) / sizeof(T)));
      const int32_t nvec = (int32_t)((n - a0) / EPV);
      const int32_t nchunks = nvec > 0 ? (nvec + VPS - 1) / VPS : 1;
      const uint4* vp = reinterpret_cast<const uint4*>(rowp + a0);
      for (int32_t c = 0; c < nchunks; ++c) {
        {
          const long long w0 = clock64();
          mbar_wait(&ms.empty[stage], phase ^ 1u);
          if (a.dbg.stats) atomicAdd((unsigned long long*)&a.dbg.stats[8], (unsigned long long)(clock64() - w0));
        }
        const int32_t nv = nvec > 0 ? min(VPS, nvec - c * VPS) : 0;
        ms.meta[stage] = StageMeta{row, c, nchunks, nv};
        if (nv > 0) {
          mbar_arrive_expect_tx(&ms.full[stage], (uint32_t)nv * 16u);
          tma_load_1d((void*)(ring + stage * kStreamChunk), vp + (int64_t)c * VPS, (uint32_t)nv * 16u,
                      &ms.full[stage], pol);
        } else {
          mbar_arrive(&ms.full[stage]);
        }
        if (++stage == kStreamStages) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    mbar_wait(&ms.empty[stage], phase ^ 1u);
    ms.meta[stage].row = -1;
    mbar_arrive(&ms.full[stage]);
    return;
  }

  // ================================================================ finishers
  if (warp >= kFirstFinisherWarp) {
    const uint32_t g = (warp - kFirstFinisherWarp) / (kNF / 32);     // finisher group
    const uint32_t t = tid - kFirstFinisherWarp * 32 - g * kNF;
    const uint32_t bar_id = 2 + g;
    auto fsync = [bar_id] { named_bar_sync(bar_id, kNF); };
    uint64_t* sel = reinterpret_cast<uint64_t*>(smem + L.sel + g * L.sel_bytes);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L.hist_f + g * 1024u);
    uint8_t* fin = smem + L.fin + g * L.fin_bytes;
    uint32_t& tmp = ms.tmp[g];
    uint32_t* bcast = ms.bcast[g];
    for (uint32_t seq = g;; seq += kNG) {
      const int b = seq % kNB;
      mbar_wait(&ms.cfull[b], (seq / kNB) & 1u);
      RowRec& R = ms.rec[b];
      const int row = R.row;
      if (row < 0) return;
      const dp_params_t p = a.params[row];
      const T* rowp = domain_row<T>(a, row, MODE);
      uint64_t* ckey = cbuf(b);
      const uint32_t* bitmap = bmap(b);
      const int32_t a0 = R.a0;
      const uint32_t kp = R.kp;
      uint64_t thr = R.thr;
      auto pen_bit = [&](int64_t pos) -> bool {
        return MODE == kHot && ((bitmap[pos >> 5] >> (pos & 31)) & 1u);
      };
      auto get_k = [&](uint32_t i, uint64_t& key) -> bool {
        key = ckey[i];
        return key >= thr;
      };
      // issue the penalty-entry loads now; they are consumed after selection
      const PenPrefetch pp = pen_prefetch<T, kNF>(a, row, R.plen, rowp, lo, n, t);
      long long c0 = clock64();
      uint32_t n_valid = min(R.cnt, ccap);
      if (a.dbg.stats && t == 0) {
        atomicAdd((unsigned long long*)&a.dbg.stats[0], 1ull);
        atomicAdd((unsigned long long*)&a.dbg.stats[3], (unsigned long long)n_valid);
      }
      // verification: fewer than kp survivors (estimate too high) or overflow
      // -> re-stream the row from global memory with a proven threshold
      while (R.overflow != 0u ||
             (n_valid < kp && thr != 0ull && key_f32((uint32_t)(thr >> 32)) > R.t_lb)) {
        if (a.dbg.stats && t == 0) atomicAdd((unsigned long long*)&a.dbg.stats[R.overflow ? 2 : 1], 1ull);
        if (R.overflow != 0u) {
          // the buffer holds a subset of the survivors: its kp-th key is a
          // valid, strictly higher threshold
          const uint64_t t1 = group_select_threshold<kNF>(get_k, ccap, ccap, kp, hist, bcast, t, fsync);
          thr = t1 > thr ? t1 : thr;
        } else {
          thr = R.t_lb == -INFINITY ? 0ull : ((uint64_t)f32_key(R.t_lb) << 32);
        }
        float thr_f = thr == 0ull ? -INFINITY : key_f32((uint32_t)(thr >> 32));
        if (thr_f != thr_f) thr_f = -INFINITY;
        fsync();
        if (t == 0) {
          R.cnt = 0u;
          R.overflow = 0u;
        }
        fsync();
        const uint4* vp = reinterpret_cast<const uint4*>(rowp + a0);
        auto take = [&](float x, int64_t pos) {
          if (x >= thr_f && !pen_bit(pos)) {
            const uint64_t key = comp_key(x, (uint32_t)pos);
            if (key >= thr) {
              const uint32_t slot = atomicAdd(&R.cnt, 1u);
              if (slot < ccap) ckey[slot] = key;
              else R.overflow = 1u;
            }
          }
        };
        for (int32_t i = t; i < R.nvec; i += kNF) {
          const uint4 v = ld_stream16(vp + i);
#pragma unroll
          for (int e = 0; e < EPV; ++e) take(vec_elem<T>(v, e), (int64_t)a0 + (int64_t)i * EPV + e);
        }
        if (t < 32) {   // scalar head / tail
          const int64_t hi_i = t, ti = (int64_t)a0 + (int64_t)R.nvec * EPV + t;
          if (hi_i < a0) take(Elem<T>::get(rowp, hi_i), hi_i);
          if (ti < n) take(Elem<T>::get(rowp, ti), ti);
        }
        fsync();
        n_valid = min(R.cnt, ccap);
      }
      long long c1 = clock64();
      // exact top-kp of the survivors (unique value-desc / position-asc keys)
      {
        const uint64_t tt = group_select_threshold<kNF>(get_k, n_valid, n_valid, kp, hist, bcast, t, fsync);
        if (t == 0) tmp = 0u;
        fsync();
        for (uint32_t i = t; i < n_valid; i += kNF) {
          const uint64_t kk = ckey[i];
          if (kk >= thr && kk >= tt) sel[atomicAdd(&tmp, 1u)] = kk;
        }
        fsync();
      }
      const uint32_t nsel = tmp;
      long long c2 = clock64();
      const FinLayout F = fin_layout(a.lcap);
      finish_row<T, MODE, kNF, false>(a, row, p, R.plen, rowp, lo, n, sel, nsel, R.sh,
                               MODE == kHot ? a.row_max[row] : 0.0, fin, F, ms.fin[g], t, fsync, &pp);
      if (a.dbg.stats && t == 0) {
        long long c3 = clock64();
        atomicAdd((unsigned long long*)&a.dbg.stats[4], (unsigned long long)(c1 - c0));
        atomicAdd((unsigned long long*)&a.dbg.stats[5], (unsigned long long)(c2 - c1));
        atomicAdd((unsigned long long*)&a.dbg.stats[6], (unsigned long long)(c3 - c2));
      }
      if (t == 0) mbar_arrive(&ms.cempty[b]);
    }
  }

  // ================================================================ streamers
  auto ssync = [] { named_bar_sync(1, kNS); };
  const uint32_t t = tid;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L.hist_s);
  int stage = 0;
  uint32_t phase = 0;
  uint32_t seq = 0;       // rows handed to the finishers
  // per-row state (uniform across streamers)
  int b = 0;
  uint64_t* ckey = cbuf(0);
  uint32_t* bitmap = bmap(0);
  const T* rowp = nullptr;
  int32_t a0 = 0, nvec = 0, tail0 = 0;
  float thr_f = -INFINITY;
  double sh = 0.0;
  float mtau_hi = 0.f, mtau_lo = 0.f, inv_tau = 1.f;

  auto pen_bit = [&](int64_t pos) -> bool {
    return MODE == kHot && ((bitmap[pos >> 5] >> (pos & 31)) & 1u);
  };
  auto accum = [&](float x, int64_t pos) {
    if (MODE == kHot && !pen_bit(pos)) sh += (double)expf(((x - mtau_hi) - mtau_lo) * inv_tau);
  };

  while (true) {
    {
      const long long w0 = clock64();
      mbar_wait(&ms.full[stage], phase);
      if (a.dbg.stats && t == 0) atomicAdd((unsigned long long*)&a.dbg.stats[9], (unsigned long long)(clock64() - w0));
    }
    const StageMeta m = ms.meta[stage];
    const uint4* sv = reinterpret_cast<const uint4*>(ring + stage * kStreamChunk);
    if (m.row < 0) {
      // hand every finisher group a terminating record
      if (t == 0) {
        for (int q = 0; q < kNG; ++q, ++seq) {
          b = seq % kNB;
          mbar_wait(&ms.cempty[b], ((seq / kNB) & 1u) ^ 1u);
          ms.rec[b].row = -1;
          mbar_arrive(&ms.cfull[b]);
        }
      }
      break;
    }

    const long long rb0 = clock64();
    if (m.chunk == 0) {
      // ---- row begin: claim a candidate buffer, threshold from this stage
      b = seq % kNB;
      RowRec& R = ms.rec[b];
      if (t == 0) {
        const long long w0 = clock64();
        mbar_wait(&ms.cempty[b], ((seq / kNB) & 1u) ^ 1u);   // finishers released it
        if (a.dbg.stats) atomicAdd((unsigned long long*)&a.dbg.stats[7], (unsigned long long)(clock64() - w0));
      }
      ckey = cbuf(b);
      bitmap = bmap(b);
      const int row = m.row;
      const dp_params_t p = a.params[row];
      const int32_t plen = pen_len(a, row, p);
      const uint32_t kp = (uint32_t)min64(n, (int64_t)p.top_k + (MODE == kHot ? 0 : plen));
      rowp = domain_row<T>(a, row, MODE);
      const uintptr_t addr = reinterpret_cast<uintptr_t>(rowp);
      a0 = (int32_t)min64(n, (int64_t)(((16u - (addr & 15u)) & 15u) / sizeof(T)));
      nvec = (int32_t)((n - a0) / EPV);
      tail0 = a0 + nvec * EPV;
      sh = 0.0;
      ssync();   // buffer b is free (thread 0 waited) before anyone writes it
      if (MODE == kHot) {
        inv_tau = (float)(1.0 / p.temperature);
        for (uint32_t i = t; i < bm_words; i += kNS) bitmap[i] = 0u;
        ssync();
        const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
        for (int32_t j = t; j < plen; j += kNS) {
          const int64_t pos = id_to_pos(a, pids[j]) - lo;
          if (pos >= 0 && pos < n) atomicOr(&bitmap[pos >> 5], 1u << (pos & 31));
        }
        const double c = a.row_max[row] * p.temperature;
        mtau_hi = (float)c;
        mtau_lo = (float)(c - (double)(float)c);
        ssync();
      }
      // each streamer's maximum over its vectors of this stage
      float mx = -INFINITY;
      for (int32_t i = t; i < m.nvec; i += kNS) {
        const uint4 v = lds128(sv + i);
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          const float x = vec_elem<T>(v, e);
          if (MODE != kHot || !pen_bit((int64_t)a0 + (int64_t)i * EPV + e)) mx = fmaxf(mx, x);
        }
      }
      // t_lb: min over warps of the ceil(kp/NW)-th largest lane maximum (each
      // lane maximum is a distinct element, so >= kp elements reach it).
      // t_est: the r-th largest of the union of every warp's top-4 lane
      // maxima (a subset of all lane maxima, so never above their r-th
      // largest), r sized so that ~3 kp row elements are expected to pass.
      const uint32_t kw = (kp + NWS - 1) / NWS;
      const uint32_t sorted = warp_sort_desc(f32_key(mx));
      const uint32_t t_lbk = __shfl_sync(0xffffffffu, sorted, kw <= 32 ? kw - 1 : 31);
      if (lane == 0) ms.thr_warp[warp] = kw <= 32 ? key_f32(t_lbk) : -INFINITY;
      if (lane < 4) ms.top4[warp * 4 + lane] = sorted;
      ssync();
      float tl = ms.thr_warp[0];
#pragma unroll
      for (int w = 1; w < NWS; ++w) tl = fminf(tl, ms.thr_warp[w]);
      float te;
      {
        const uint32_t u = warp_sort_desc(ms.top4[lane]);   // every streamer warp, redundantly
        const float sample = (float)max(1, m.nvec * EPV);
        int r = (int)ceilf(3.0f * (float)kp * sample / (float)max(1, nvec * EPV));
        r = max(1, min(32, r));
        te = key_f32(__shfl_sync(0xffffffffu, u, r - 1));
      }
      if (te != te) te = -INFINITY;
      te = fmaxf(te, tl);
      thr_f = te;
      const uint64_t thr = te == -INFINITY ? 0ull : ((uint64_t)f32_key(te) << 32);
      if (t == 0) {
        R.row = row;
        R.kp = kp;
        R.thr = thr;
        R.t_lb = tl;
        R.a0 = a0;
        R.nvec = nvec;
        R.plen = plen;
        R.cnt = 0u;
        R.overflow = 0u;
      }
      ssync();
      if (warp == 0 && (a0 > 0 || tail0 < n)) {   // scalar head / tail elements
        const int32_t hi_i = lane, ti = tail0 + lane;
        const bool hv = hi_i < a0, tv = ti < n;
        const float hx = hv ? Elem<T>::get(rowp, hi_i) : -INFINITY;
        const float tx = tv ? Elem<T>::get(rowp, ti) : -INFINITY;
        if (hv) accum(hx, hi_i);
        if (tv) accum(tx, ti);
        __syncwarp();
        if (hv && !pen_bit(hi_i) && hx >= thr_f) {
          const uint32_t slot = atomicAdd(&R.cnt, 1u);
          if (slot < ccap) ckey[slot] = comp_key(hx, (uint32_t)hi_i);
        }
        if (tv && !pen_bit(ti) && tx >= thr_f) {
          const uint32_t slot = atomicAdd(&R.cnt, 1u);
          if (slot < ccap) ckey[slot] = comp_key(tx, (uint32_t)ti);
        }
      }
      ssync();
    }

    if (a.dbg.stats && t == 0 && m.chunk == 0)
      atomicAdd((unsigned long long*)&a.dbg.stats[10], (unsigned long long)(clock64() - rb0));
    const long long cs0 = clock64();
    // ---- consume this stage (all loads of a thread first, then the tests)
    {
      RowRec& R = ms.rec[b];
      const int32_t vbase = m.chunk * VPS;
      constexpr int PER = VPS / kNS;
      uint4 v[PER];
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int32_t i = (int32_t)t + j * kNS;
        v[j] = i < m.nvec ? lds128(sv + i) : neg_inf_vec<T>();
      }
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int32_t i = (int32_t)t + j * kNS;
        if (MODE == kHot && i < m.nvec) {
#pragma unroll
          for (int e = 0; e < EPV; ++e) accum(vec_elem<T>(v[j], e), (int64_t)a0 + (int64_t)(vbase + i) * EPV + e);
        }
        bool any = false;
#pragma unroll
        for (int e = 0; e < EPV; ++e) any |= vec_elem<T>(v[j], e) >= thr_f;
        if (any && i < m.nvec) {   // rare (~0.1% of vectors): append survivors' keys
#pragma unroll
          for (int e = 0; e < EPV; ++e) {
            const float x = vec_elem<T>(v[j], e);
            const int64_t pos = (int64_t)a0 + (int64_t)(vbase + i) * EPV + e;
            if (x >= thr_f && !pen_bit(pos)) {
              const uint32_t slot = atomicAdd(&R.cnt, 1u);
              if (slot < ccap) ckey[slot] = comp_key(x, (uint32_t)pos);
              else R.overflow = 1u;
            }
          }
        }
      }
    }
    __syncwarp();
    if (a.dbg.stats && t == 0) atomicAdd((unsigned long long*)&a.dbg.stats[11], (unsigned long long)(clock64() - cs0));
    if (lane == 0) mbar_arrive(&ms.empty[stage]);
    if (++stage == kStreamStages) {
      stage = 0;
      phase ^= 1u;
    }
    if (m.chunk != m.nchunks - 1) continue;

    // ---- row end: hand the buffer to the finishers
    if (MODE == kHot) {
      const double s = warp_sum(sh);
      if (lane == 0) ms.sh_warp[warp] = s;
    }
    ssync();
    if (t == 0) {
      double s = 0.0;
      if (MODE == kHot)
        for (int w = 0; w < NWS; ++w) s += ms.sh_warp[w];   // fixed order: deterministic
      ms.rec[b].sh = s;
      mbar_arrive(&ms.cfull[b]);
    }
    ++seq;
  }
}

// ---------------------------------------------------------------------------

template <typename T, int MODE>
static cudaError_t launch_stream_t(const SampleArgs& a, int grid, int32_t* work, cudaStream_t st) {
  const int64_t n = MODE == kFull ? a.V : (MODE == kHot ? a.H : a.V - a.H);
  const int bm_words = MODE == kHot ? (int)((n + 31) / 32) : 0;
  const StreamLayout L = stream_layout(a.wcap, a.kcap, a.lcap, bm_words);
  auto kern = stream_sample_kernel<T, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(work, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  kern<<<grid, kStreamThreads, L.total, st>>>(a, work);
  return cudaGetLastError();
}

cudaError_t launch_stream(const SampleArgs& a, int dtype, int mode, int grid, int32_t* work, cudaStream_t st) {
  if (dtype == DP_F32) {
    if (mode == kFull) return launch_stream_t<float, kFull>(a, grid, work, st);
    if (mode == kHot) return launch_stream_t<float, kHot>(a, grid, work, st);
    return launch_stream_t<float, kTail>(a, grid, work, st);
  }
  if (mode == kFull) return launch_stream_t<__nv_bfloat16, kFull>(a, grid, work, st);
  if (mode == kHot) return launch_stream_t<__nv_bfloat16, kHot>(a, grid, work, st);
  return launch_stream_t<__nv_bfloat16, kTail>(a, grid, work, st);
}

size_t stream_smem_bytes(const SampleArgs& a, int mode) {
  const int64_t n = mode == kFull ? a.V : (mode == kHot ? a.H : a.V - a.H);
  return stream_layout(a.wcap, a.kcap, a.lcap, mode == kHot ? (int)((n + 31) / 32) : 0).total;
}

}  // namespace dp
