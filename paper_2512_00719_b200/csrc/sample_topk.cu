// sample_topk.cu — fused single-pass top-k sampler (K1), sm_100a.
//
// One thread-block CLUSTER per row; the row's domain is split across the
// cluster's CTAs, each streaming its segment exactly once from HBM with
// 16-byte non-allocating loads (U vectors in flight per lane).
//
// Selection is exact and keeps the raw top-(k + |penalty list|): an
// unpenalized element below the raw (k + |touched|)-th largest is dominated by
// k unpenalized elements whose ready value keeps its raw order, so it cannot
// reach the top-k — the superset argument of _Sampler._tail_preselect
// (service.py:309-336).  Per CTA:
//   1. threshold: from the first register batch, each warp sorts its lanes'
//      maxima and takes the ceil(kp/NW)-th; the CTA minimum is a proven lower
//      bound of the segment's kp-th largest (>= kp distinct elements reach it);
//   2. stream: elements >= threshold are appended (warp-aggregated) to one
//      shared candidate buffer — ~1-2% of the row, no in-loop compaction;
//      overflow (adversarial order) re-streams with the buffer's kp-th key;
//   3. exact radix select on unique (value desc, position asc) keys — the
//      canonical boundary-tie rule of _top_k_ids (filtering.py:38-58).
// Non-leader CTAs push their survivors into CTA 0's shared memory over DSMEM
// and arrive on its mbarrier, then exit; CTA 0 merges, applies the sparse
// penalties in IEEE f64 (penalty.py:66-78), divides by tau
// (service.py:236-241), sorts, and runs the exact top-p / min-p /
// inverse-CDF draw (filtering.py:61-162).
//
// kHot excludes penalized ids from the stream (shared bitmap), accumulates the
// hot mass S_H (shvs.py:223-230) and decides acceptance; kTail serves the rows
// the hot pass rejected.

#include "sampler.cuh"
#include "select.cuh"
#include "finish.cuh"

#include <type_traits>

namespace dp {

template <int NT>
struct TopkSmem {
  static constexpr int NW = NT / 32;
  uint64_t mbar;              // CTA 0: arrivals of the other cluster CTAs
  double sh_warp[NW];
  double sh_recv[8];          // CTA 0: per-rank hot mass (kHot) / nucleus mass
  float c_recv[8];            // CTA 0: per-rank nucleus mass reference
  float max_warp[NW];
  double sh_pen[NW];
  float thr_warp[NW];
  float est_warp[NW];
  uint32_t cnt;               // candidate buffer fill
  uint32_t overflow;
  uint32_t nsel;
  uint32_t bcast[4];
  uint32_t recv_n[8];         // CTA 0: per-rank survivor counts
  uint32_t nl;
  uint32_t nscal;
  uint32_t tmp;
  unsigned long long kor, kand;   // OR / AND of the valid candidate keys (group_compact_valid)
  uint64_t scal[64];          // scalar head/tail candidates (CTA 0; every rank of a sharded row: <= 8 fp32 / 4 bf16 shards)
  FinishScratch fin;
};

// shared-memory carve-up, shared by host sizing and device code
struct TopkLayout {
  uint32_t cand, recv, sel, bhist, bitmap, misc, total, ccap;
};
template <int NT>
__host__ __device__ inline TopkLayout topk_layout(int ccap, int kcap, int lcap, int bitmap_words, int split) {
  TopkLayout L;
  L.ccap = (uint32_t)ccap;
  const uint32_t fin = fin_layout(lcap).bytes;
  uint32_t region = (uint32_t)ccap * 20u;
  const uint32_t merge = (uint32_t)split * kcap * 8u;   // CTA 0 merge scratch
  region = region > merge ? region : merge;
  region = region > fin ? region : fin;
  uint32_t o = 0;
  L.cand = o; o += (region + 15u) & ~15u;
  L.recv = o; o += (split > 1 ? (uint32_t)(split - 1) * kcap * 8u : 0u);
  L.sel = o; o += kcap * 8u;
  L.bhist = o; o += 256u * 4u;
  L.bitmap = o; o += ((uint32_t)bitmap_words * 4u + 15u) & ~15u;
  L.misc = o; o += (sizeof(TopkSmem<NT>) + 15u) & ~15u;
  L.total = o;
  return L;
}


// NUC: the call may hold nucleus rows (top-k off); the plain top-k
// instantiation carries none of that code
#ifndef DP_PREFETCH
#define DP_PREFETCH 1
#endif
constexpr int kPrefetch = DP_PREFETCH;   // L2 prefetch distance, in batches

// SH: TP-sharded kFull rows (a.nshard > 0), a separate instantiation so the
// contiguous-row code keeps its single-segment stream
template <typename T, int MODE, int NT, int U, bool NUC, bool SH, bool PX = false>
__global__ void __launch_bounds__(NT, MODE == kTail ? 2 : 1024 / NT) topk_sample_kernel(SampleArgs a) {
  constexpr int NW = NT / 32;
  constexpr int EPV = Elem<T>::kPerVec;
  extern __shared__ __align__(16) uint8_t smem[];
  const int64_t n = dom_n(a, MODE);
  const int64_t lo = dom_lo(a, MODE);
  // kHot, and long penalty lists (pen_excl), stream around the penalized ids
  // PX: a separate instantiation, so the plain path carries no bitmap code
  constexpr bool excl = MODE == kHot || PX;
  const uint32_t bm_words = excl ? (uint32_t)((n + 31) / 32) + 1u : 0u;   // +1: vector window
  const TopkLayout L = topk_layout<NT>(a.wcap, a.kcap, a.lcap, (int)bm_words, a.split);
  uint64_t* cand = reinterpret_cast<uint64_t*>(smem + L.cand);
  uint64_t* recv = reinterpret_cast<uint64_t*>(smem + L.recv);
  uint64_t* sel = reinterpret_cast<uint64_t*>(smem + L.sel);
  uint32_t* bhist = reinterpret_cast<uint32_t*>(smem + L.bhist);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem + L.bitmap);
  TopkSmem<NT>& ms = *reinterpret_cast<TopkSmem<NT>*>(smem + L.misc);

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  const uint32_t split = (uint32_t)a.split;
#ifdef DP_TIMELINE   // A-B build: per-row globaltimer marks into dbg.topk_ready[row * stride + 0..4]
  auto gt = [] { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
  uint64_t tl0 = 0, tl1 = 0, tl2 = 0;
#endif
  const uint32_t rank = split > 1 ? cluster_ctarank() : 0u;
  const int nrows = a.row_count ? *a.row_count : a.n_rows;
  // clusters loop over rows (the tail pass launches fewer clusters than rows);
  // CTA 0's mbarrier completes one phase per row
  if (split > 1 && rank == 0 && tid == 0) {
    mbar_init(&ms.mbar, split - 1);
    fence_mbar_init();
  }
  uint32_t phase = 0;
  for (int ridx = blockIdx.x / (int)split; ridx < nrows; ridx += gridDim.x / split) {
  const int row = a.rows ? a.rows[ridx] : ridx;
  const dp_params_t p = a.params[row];
  const int32_t plen = pen_len(a, row, p);
  const int32_t k = p.top_k;
  // nucleus rows (top-k off) keep the kNucK largest plus the domain mass;
  // kHot's mass is the hot mass it accumulates anyway, kFull / kTail
  // accumulate it relative to the first batch's maximum (nuc_mass)
  const bool nuc = NUC && nucleus_row(k, n);
  const int32_t ke = nuc ? effective_k(k, n) : k;
  const bool nuc_mass = nuc && MODE != kHot;
  // kHot excludes penalized ids from the stream (bitmap) so it needs no widening
  const uint32_t kp = (uint32_t)min64(n, (int64_t)ke + (excl ? 0 : plen));
  if (route_row(a, MODE, k, plen, n) != kRouteTopk) continue;   // another kernel's row (cluster-uniform)

#ifdef DP_TIMELINE
  tl0 = gt();
#endif
  const T* rowp = domain_row<T>(a, row, MODE);
  const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
  const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;
  const uint32_t ccap = L.ccap;

  // ---- setup
  const bool prof = a.dbg.stats != nullptr && threadIdx.x == 0;
  long long pc0 = prof ? clock64() : 0;
  auto lapk = [&](int slot) {
    if (prof) {
      const long long now = clock64();
      atomicAdd((unsigned long long*)&a.dbg.stats[slot], (unsigned long long)(now - pc0));
      pc0 = now;
    }
  };
  if (tid == 0) {
    ms.cnt = 0u;
    ms.overflow = 0u;
    ms.nsel = 0u;
    ms.nl = 0u;
    ms.nscal = 0u;
  }
  double mrow = 0.0;
  float mtau_hi = 0.f, mtau_lo = 0.f;
  const float s2 = (float)(1.4426950408889634 / p.temperature);
  if (excl) {
    for (uint32_t i = tid; i < bm_words; i += NT) bitmap[i] = 0u;
    __syncthreads();
    // 4 list entries per thread in flight (long lists: fewer round trips)
    for (int32_t base = tid; base < plen; base += NT * 4) {
      int32_t pos[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t j = base + u * NT;
        pos[u] = j < plen ? (int32_t)(id_to_pos(a, pids[j]) - lo) : -1;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (pos[u] >= 0 && pos[u] < n) atomicOr(&bitmap[pos[u] >> 5], 1u << (pos[u] & 31));
    }
  }
  if (MODE == kHot) {
    mrow = a.row_max[row];
    const double c = mrow * p.temperature;
    mtau_hi = (float)c;
    mtau_lo = (float)(c - (double)(float)c);
  }
  if (split > 1) cluster_sync();   // CTA 0's mbarrier is initialised before anyone arrives
  else __syncthreads();

  lapk(17);
  // ---- segment geometry (32-bit vector indices: V < 2^31)
  // TP-sharded rows: this CTA's segment is its own vocab shard, read in place
  // (positions offset by pos0); otherwise a vector-aligned chunk of the row
  constexpr bool sharded = SH && MODE == kFull;
  // a sharded row's CTA streams shards [rank * spc, (rank + 1) * spc), one
  // segment after another (set_segment)
  const int spc = sharded ? a.shard_per_cta : 1;   // 1 at compile time unless SH
  const bool own_scal = rank == 0 || sharded;   // this CTA holds scalar head / tail elements
  const T* segp = rowp;
  int64_t n_seg = n;
  uint32_t pos0 = 0u;
  int32_t a0 = 0, nvec = 0, tail0 = 0, v_lo = 0, v_hi = 0;
  const uint4* vp = nullptr;
  auto set_segment = [&](int g) {
    if (sharded) {
      const int s = (int)rank * spc + g;
      segp = reinterpret_cast<const T*>(a.shard[s]) + (int64_t)row * a.ld;
      n_seg = a.shard_n;
      pos0 = (uint32_t)s * (uint32_t)a.shard_n;
    }
    const uintptr_t addr = reinterpret_cast<uintptr_t>(segp);
    a0 = (int32_t)min64(n_seg, (int64_t)(((16u - (addr & 15u)) & 15u) / sizeof(T)));
    nvec = (int32_t)((n_seg - a0) / EPV);
    tail0 = a0 + nvec * EPV;
    const int32_t chunk = sharded ? nvec : ((nvec + (int32_t)split - 1) / (int32_t)split + 31) & ~31;
    v_lo = sharded ? 0 : min(nvec, (int32_t)rank * chunk);
    v_hi = min(nvec, v_lo + chunk);
    vp = reinterpret_cast<const uint4*>(segp + a0);
  };
  set_segment(0);
  const int64_t seg_elems = sharded ? (int64_t)spc * a.shard_n : (int64_t)(v_hi - v_lo) * EPV;
  uint4* cvec = reinterpret_cast<uint4*>(cand);                 // admitted vectors
  int32_t* cidx = reinterpret_cast<int32_t*>(cvec + ccap);      // their first element's row position
  const T* celem = reinterpret_cast<const T*>(cvec);
  auto pen_bit = [&](int64_t pos) -> bool {
    return excl && ((bitmap[pos >> 5] >> (pos & 31)) & 1u);
  };

  uint64_t thr = 0ull;     // admit keys >= thr
  float thr_f = -INFINITY;
  double sh = 0.0;         // kHot: unpenalized hot mass of this thread's elements
  // hot mass: exp((x - m tau) / tau) = 2^(((x - hi) - lo) * log2e / tau); the
  // argument is centred on the row maximum (hi/lo split keeps x - m tau
  // exact near the top), pairwise f32 sums per vector, one f64 add per vector
  auto hot_exp = [&](float x) -> float { return ex2_fast(((x - mtau_hi) - mtau_lo) * s2); };
  auto accum = [&](float x, int64_t pos) {
    if ((MODE == kHot && !pen_bit(pos)) || nuc_mass) sh += (double)hot_exp(x);
  };
  // nucleus mass of kFull / kTail: every element (penalized ones are swapped
  // for their exact terms in the final stage)
  auto accum_vec_all = [&](const uint4& vv) {
    float e[EPV];
#pragma unroll
    for (int i = 0; i < EPV; ++i) e[i] = hot_exp(vec_elem<T>(vv, i));
#pragma unroll
    for (int st = 1; st < EPV; st <<= 1)
#pragma unroll
      for (int i = 0; i < EPV; i += 2 * st) e[i] += e[i + st];
    sh += (double)e[0];
  };
  auto accum_vec = [&](const uint4& vv, int32_t idx) {
    const uint32_t p0 = (uint32_t)(a0 + idx * EPV);
    const uint32_t w = p0 >> 5;
    const uint32_t pm = __funnelshift_r(bitmap[w], bitmap[w + 1], p0 & 31u);
    float e[EPV];
#pragma unroll
    for (int i = 0; i < EPV; ++i) e[i] = ((pm >> i) & 1u) ? 0.f : hot_exp(vec_elem<T>(vv, i));
#pragma unroll
    for (int st = 1; st < EPV; st <<= 1)
#pragma unroll
      for (int i = 0; i < EPV; i += 2 * st) e[i] += e[i + st];
    sh += (double)e[0];
  };
  // scalar head / tail elements (at most 2*EPV-2) belong to CTA 0 (warp 0)
  uint32_t nscal_acc = 0u;   // warp 0: scalar keys appended so far this pass
  auto head_tail = [&](bool first) {
    const int32_t hi_i = lane, ti = tail0 + lane;
    const bool hv = hi_i < a0, tv = ti < n_seg;
    const float hx = hv ? Elem<T>::get(segp, hi_i) : -INFINITY;
    const float tx = tv ? Elem<T>::get(segp, ti) : -INFINITY;
    if (first && hv) accum(hx, hi_i);
    if (first && tv) accum(tx, ti);
    const bool hp = hv && !pen_bit(hi_i) && comp_key(hx, pos0 + (uint32_t)hi_i) >= thr;
    const bool tp = tv && !pen_bit(ti) && comp_key(tx, pos0 + (uint32_t)ti) >= thr;
    const uint32_t mh = __ballot_sync(0xffffffffu, hp), mt = __ballot_sync(0xffffffffu, tp);
    if (hp) ms.scal[nscal_acc + __popc(mh & lanemask_lt())] = comp_key(hx, pos0 + (uint32_t)hi_i);
    if (tp) ms.scal[nscal_acc + __popc(mh) + __popc(mt & lanemask_lt())] = comp_key(tx, pos0 + (uint32_t)ti);
    nscal_acc += (uint32_t)(__popc(mh) + __popc(mt));
    if (lane == 0) ms.nscal = nscal_acc;
  };

  // candidate source for the exact selection: elements of admitted vectors
  // (>= thr, not penalized in kHot) plus CTA 0's scalar head/tail keys
  auto get_c = [&](uint32_t i, uint64_t& key) -> bool {
    const uint32_t ne = min(ms.cnt, ccap) * EPV;
    if (i >= ne) {
      key = ms.scal[i - ne];
      return true;
    }
    const float x = to_f32(celem[i]);
    const uint32_t pos = (uint32_t)cidx[i / EPV] + i % EPV;
    key = comp_key(x, pos);
    return key >= thr && !pen_bit(pos);
  };

  // ---- threshold -> stream the segment.  The first register batch gives
  //  * t_lb: min over warps of the ceil(kp/NW)-th largest lane maximum — a
  //    proven lower bound of the segment's kp-th largest;
  //  * t_est: an estimate of the segment's (2 kp)-th largest from the same
  //    sample (median over warps), ~5-10x fewer admissions.
  // Admission uses t_est; if the CTA then holds fewer than kp survivors the
  // segment is re-streamed with t_lb, so results never depend on the estimate.
  // Admission is per 16-byte vector: a lane appends every vector holding an
  // element >= threshold (one aggregated atomic per lane per batch).
  float t_lb = -INFINITY;
  uint32_t n_valid = 0;
  // the valid keys, compacted into the candidate region's unused slots
  // (select rounds then read n_valid keys, not every element slot)
  uint64_t* dense = nullptr;
  uint32_t dcap = 0u;
  DenseStats ds{};
  uint64_t loaded = 0;   // tid 0: bytes this CTA streamed for the row (every pass)
  for (int pass_no = 0;; ++pass_no) {
  nscal_acc = 0u;
  for (int g = 0; g < spc; ++g) {
    if (g > 0 || (sharded && pass_no > 0)) set_segment(g);
    if (tid == 0)
      loaded += (uint64_t)(v_hi - v_lo) * 16u + (own_scal ? (uint64_t)(a0 + (n_seg - tail0)) * sizeof(T) : 0u);
    int32_t base = v_lo + (int32_t)warp * 32 * U;
    if (lane == 0) {   // the first kPrefetch chunks after the first batch -> L2
#pragma unroll
      for (int d = 1; d <= kPrefetch; ++d)
        if (base + d * NT * U + 32 * U <= v_hi) prefetch_l2(vp + base + d * NT * U, 32u * U * 16u);
    }
    uint4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int32_t idx = base + j * 32 + (int32_t)lane;
      v[j] = idx < v_hi ? ld_stream16(vp + idx) : neg_inf_vec<T>();
    }
    if (pass_no == 0 && g == 0) {
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int32_t idx = base + j * 32 + (int32_t)lane;
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          const float x = vec_elem<T>(v[j], e);
          if (!excl || (idx < v_hi && !pen_bit((int64_t)a0 + (int64_t)idx * EPV + e))) mx = fmaxf(mx, x);
        }
      }
      const uint32_t kw = (kp + NW - 1) / NW;
      const float seg = (float)max((int64_t)1, seg_elems);
      int rw = (int)ceilf(est_over(kp, nuc) * (float)kp * (float)(32 * U * EPV) / seg);
      rw = max(1, min(32, rw));
      const uint32_t sorted = warp_sort_desc(f32_key(mx));
      const uint32_t t_lbk = __shfl_sync(0xffffffffu, sorted, kw <= 32 ? kw - 1 : 31);
      const uint32_t t_ek = __shfl_sync(0xffffffffu, sorted, rw - 1);
      const float mx_w = warp_max(mx);
      if (lane == 0) {
        ms.thr_warp[warp] = kw <= 32 ? key_f32(t_lbk) : -INFINITY;
        ms.est_warp[warp] = key_f32(t_ek);
        ms.max_warp[warp] = mx_w;
      }
      __syncthreads();
      if (nuc_mass) {   // mass reference: the maximum of this CTA's first batch
        float c = ms.max_warp[0];
#pragma unroll
        for (int w = 1; w < NW; ++w) c = fmaxf(c, ms.max_warp[w]);
        mtau_hi = c;
        mtau_lo = 0.f;
      }
      float tl = ms.thr_warp[0];
      float ev[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        tl = fminf(tl, ms.thr_warp[w]);
        ev[w] = ms.est_warp[w];
      }
      // upper median of the warp estimates (NW small: insertion sort, desc)
#pragma unroll
      for (int i = 1; i < NW; ++i)
#pragma unroll
        for (int j2 = i; j2 > 0; --j2)
          if (ev[j2] > ev[j2 - 1]) { const float tmp = ev[j2]; ev[j2] = ev[j2 - 1]; ev[j2 - 1] = tmp; }
      t_lb = tl;
      const float te = fmaxf(ev[(NW - 1) / 2], t_lb);
      thr_f = te;
      thr = te == -INFINITY ? 0ull : ((uint64_t)f32_key(te) << 32);
    }
    if (own_scal && warp == 0) head_tail(pass_no == 0);
    // consume batches.  While the threshold is a plain value (low key bits
    // zero) "x >= thr_f" IS the exact admission test: one max + compare per
    // vector.  After an overflow cut it is a full composite key and the exact
    // (value, position) test runs (ties at its value must not re-admit, so
    // every re-stream admits strictly fewer elements).
    const bool exact_mode = (uint32_t)thr != 0u;
    while (true) {
      uint32_t vm = 0;
      const bool full = base + 32 * U <= v_hi;   // warp-uniform: every vector of the batch is valid
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int32_t idx = base + j * 32 + (int32_t)lane;
        if (MODE == kHot && pass_no == 0 && (full || idx < v_hi)) accum_vec(v[j], idx);
        else if (nuc_mass && pass_no == 0 && (full || idx < v_hi)) accum_vec_all(v[j]);
        float mx = vec_elem<T>(v[j], 0);
#pragma unroll
        for (int e = 1; e < EPV; ++e) mx = fmaxf(mx, vec_elem<T>(v[j], e));
        vm |= (mx >= thr_f ? 1u : 0u) << j;
      }
      if (!full) {
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (base + j * 32 + (int32_t)lane >= v_hi) vm &= ~(1u << j);
      }
      if (exact_mode && vm) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          if ((vm >> j) & 1u) {
            const int32_t idx = base + j * 32 + (int32_t)lane;
            bool ex = false;
#pragma unroll
            for (int e = 0; e < EPV; ++e)
              ex |= comp_key(vec_elem<T>(v[j], e), pos0 + (uint32_t)(a0 + idx * EPV + e)) >= thr;
            if (!ex) vm &= ~(1u << j);
          }
        }
      }
      if (vm) {
        uint32_t slot = atomicAdd(&ms.cnt, (uint32_t)__popc(vm));
#pragma unroll
        for (int j = 0; j < U; ++j) {
          if ((vm >> j) & 1u) {
            if (slot < ccap) {
              cvec[slot] = v[j];
              cidx[slot] = (int32_t)(pos0 + (uint32_t)(a0 + (base + j * 32 + (int32_t)lane) * EPV));
            } else {
              ms.overflow = 1u;
            }
            ++slot;
          }
        }
      }
      base += NT * U;
      if (base >= v_hi) break;
      // this warp's chunk kPrefetch iterations ahead -> L2 (one lane, 4 KB)
      if (lane == 0 && base + kPrefetch * NT * U + 32 * U <= v_hi)
        prefetch_l2(vp + base + kPrefetch * NT * U, 32u * U * 16u);
      if (base + 32 * U <= v_hi) {   // full batch: unpredicated loads at immediate offsets
        const uint4* q = vp + base + (int32_t)lane;
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = ld_stream16(q + j * 32);
      } else {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int32_t idx = base + j * 32 + (int32_t)lane;
          v[j] = idx < v_hi ? ld_stream16(vp + idx) : neg_inf_vec<T>();
        }
      }
    }
  }   // shards of this CTA
    __syncthreads();
    const bool overflow = ms.overflow != 0u;
    {
      const uint32_t nc = min(ms.cnt, ccap);
      dense = reinterpret_cast<uint64_t*>(cvec + nc);
      dcap = overflow ? 0u : (ccap - nc) * 2u;
      ds = group_compact_valid<NT>(get_c, nc * EPV + (own_scal ? ms.nscal : 0u), dense, dcap, &ms.tmp, &ms.kor,
                                   &ms.kand, tid, [] { __syncthreads(); });
      n_valid = ds.n;
    }
    bool again = false;
    if (overflow) {
      // the buffer holds a subset of the admitted elements: its kp-th largest
      // key is a valid, strictly higher threshold
      const uint64_t t1 = block_select_threshold<NT>(get_c, ccap * EPV + (own_scal ? ms.nscal : 0u), n_valid,
                                                     kp, bhist, ms.bcast, ds.kor ^ ds.kand, ds.kand);
      if (t1 > thr) thr = t1;
      again = true;
    } else if (n_valid < kp && thr_f > t_lb) {
      thr = t_lb == -INFINITY ? 0ull : ((uint64_t)f32_key(t_lb) << 32);   // estimate too aggressive
      again = true;
    }
    if (!again) break;
    if (a.dbg.stats && tid == 0) atomicAdd((unsigned long long*)&a.dbg.stats[1], 1ull);
    thr_f = key_f32((uint32_t)(thr >> 32));
    if (thr_f != thr_f || thr == 0ull) thr_f = -INFINITY;
    __syncthreads();
    if (tid == 0) {
      ms.cnt = 0u;
      ms.overflow = 0u;
    }
    __syncthreads();
  }

  lapk(18);
#ifdef DP_TIMELINE
  tl1 = gt();
#endif
  if (tid == 0) touch_bytes(a, row, loaded);
  // ---- CTA-level exact top-kp
  if (n_valid <= dcap) {
    auto get_d = [&](uint32_t i, uint64_t& key) -> bool { key = dense[i]; return true; };
    const uint64_t t = block_select_threshold<NT>(get_d, n_valid, n_valid, kp, bhist, ms.bcast, ds.kor ^ ds.kand,
                                                  ds.kand);
    for (uint32_t i = tid; i < n_valid; i += NT) {
      const uint64_t kk = dense[i];
      if (kk >= t) sel[atomicAdd(&ms.nsel, 1u)] = kk;
    }
  } else {
    const uint32_t ns = min(ms.cnt, ccap) * EPV + (own_scal ? ms.nscal : 0u);
    const uint64_t t = block_select_threshold<NT>(get_c, ns, n_valid, kp, bhist, ms.bcast, ds.kor ^ ds.kand, ds.kand);
    for (uint32_t i = tid; i < ns; i += NT) {
      uint64_t kk;
      if (get_c(i, kk) && kk >= t) sel[atomicAdd(&ms.nsel, 1u)] = kk;
    }
  }
  if (MODE == kHot || nuc_mass) {
    const double s = warp_sum(sh);
    if (lane == 0) ms.sh_warp[warp] = s;
  }
  __syncthreads();
  double sh_cta = 0.0;
  if (MODE == kHot || nuc_mass) {
    for (int w = 0; w < NW; ++w) sh_cta += ms.sh_warp[w];   // fixed order: deterministic
  }
  const uint32_t nsel_own = ms.nsel;

  lapk(19);
  // ---- push-model cluster merge into CTA 0 (DSMEM + mbarrier)
  if (split > 1) {
    if (rank != 0) {
      const uint32_t dst = dsmem_addr(recv + (size_t)(rank - 1) * a.kcap, 0);
      for (uint32_t i = tid; i < nsel_own; i += NT) st_dsmem_u64(dst + 8u * i, sel[i]);
      if (tid == 0) {
        st_dsmem_u32(dsmem_addr(&ms.recv_n[rank], 0), nsel_own);
        if (MODE == kHot || nuc_mass) st_dsmem_f64(dsmem_addr(&ms.sh_recv[rank], 0), sh_cta);
        if (nuc_mass) st_dsmem_f32(dsmem_addr(&ms.c_recv[rank], 0), mtau_hi);
      }
      __syncthreads();
      if (tid == 0) mbar_remote_arrive(dsmem_addr(&ms.mbar, 0));
      // without a next row: leave (after the cluster's final barrier)
      if (ridx + (int)(gridDim.x / split) >= nrows) {
#ifndef DP_CLUSTER_EARLY_RETIRE
        // every rank leaves together: no rank exits while a peer may still
        // address the cluster's shared memory (compute-sanitizer racecheck
        // clean; retiring right after the push is the opt-in
        // DP_CLUSTER_EARLY_RETIRE build, ~1% faster SHVS tail)
        cluster_sync();
#endif
        return;
      }
      cluster_sync();   // end of row: CTA 0 is done with the receive buffers
      phase ^= 1u;
      continue;
    }
    if (warp == 0) mbar_wait_parity(&ms.mbar, phase);   // one warp polls; the rest park on the barrier
    __syncthreads();
    // gather own + received survivors into the merge scratch, exact select
    uint64_t* mrg = cand;
    uint32_t off = nsel_own;
    for (uint32_t i = tid; i < nsel_own; i += NT) mrg[i] = sel[i];
    for (uint32_t r = 1; r < split; ++r) {
      const uint32_t nr = ms.recv_n[r];
      const uint64_t* src = recv + (size_t)(r - 1) * a.kcap;
      for (uint32_t i = tid; i < nr; i += NT) mrg[off + i] = src[i];
      off += nr;
      if (MODE == kHot) sh_cta += ms.sh_recv[r];
      // nucleus mass of rank r is relative to its own reference: rescale
      if (nuc_mass) sh_cta += ms.sh_recv[r] * exp(((double)ms.c_recv[r] - (double)mtau_hi) / p.temperature);
    }
    __syncthreads();
    if (tid == 0) ms.nsel = 0u;
    __syncthreads();
    auto get_m = [&](uint32_t i, uint64_t& key) -> bool { key = mrg[i]; return true; };
    const uint64_t t = block_select_threshold<NT>(get_m, off, off, kp, bhist, ms.bcast);
    for (uint32_t i = tid; i < off; i += NT)
      if (mrg[i] >= t) sel[atomicAdd(&ms.nsel, 1u)] = mrg[i];
    __syncthreads();
  }

  lapk(20);
#ifdef DP_TIMELINE
  tl2 = gt();
#endif
  // ---- final stage (CTA 0): penalties, exact sort, filter, draw
  {
    const FinLayout F = fin_layout(a.lcap);
    finish_row<T, MODE, NT, NUC, PX>(a, row, p, plen, rowp, lo, n, sel, ms.nsel, sh_cta, mrow, smem + L.cand, F,
                                     ms.fin, tid, [] { __syncthreads(); }, nullptr, mtau_hi);
  }
#ifdef DP_TIMELINE
  __syncthreads();
  if (tid == 0 && a.dbg.topk_ready) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    double* tl = a.dbg.topk_ready + (int64_t)row * a.dbg.topk_stride;
    tl[0] = (double)tl0; tl[1] = (double)tl1; tl[2] = (double)tl2; tl[3] = (double)gt(); tl[4] = (double)smid;
  }
#endif
  if (split > 1) {
    if (ridx + (int)(gridDim.x / split) >= nrows) {   // last row: the cluster's final barrier, then exit
#ifndef DP_CLUSTER_EARLY_RETIRE
      cluster_sync();
#endif
      return;
    }
    cluster_sync();   // end of row: the receive buffers may be rewritten
    phase ^= 1u;
  } else {
    __syncthreads();
  }
  }
}

// ---------------------------------------------------------------------------
// host launcher

template <typename T, int MODE, bool NUC, bool SH = false, bool PX = false>
static cudaError_t launch_topk_t(const SampleArgs& a, int grid_rows, cudaStream_t st) {
#ifndef DP_TOPK_NT
#define DP_TOPK_NT 256
#define DP_TOPK_U 8
#endif
  constexpr int U = DP_TOPK_U, NT = DP_TOPK_NT;
  const int64_t n = MODE == kFull ? a.V : (MODE == kHot ? a.H : a.V - a.H);
  const int bm_words = (MODE == kHot || PX) ? (int)((n + 31) / 32) + 1 : 0;
  const TopkLayout L = topk_layout<NT>(a.wcap, a.kcap, a.lcap, bm_words, a.split);
  auto kern = topk_sample_kernel<T, MODE, NT, U, NUC, SH, PX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(grid_rows * a.split));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.split;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename T, bool NUC>
static cudaError_t launch_topk_m(const SampleArgs& a, int mode, int grid_rows, cudaStream_t st) {
  if (mode == kFull && a.nshard > 0) return launch_topk_t<T, kFull, false, true>(a, grid_rows, st);
  // long penalty lists (a.pen_excl): the instantiation that streams around
  // the penalized ids
  if (mode == kFull)
    return a.pen_excl ? launch_topk_t<T, kFull, NUC, false, true>(a, grid_rows, st)
                      : launch_topk_t<T, kFull, NUC>(a, grid_rows, st);
  if (mode == kHot) return launch_topk_t<T, kHot, NUC>(a, grid_rows, st);
  return a.pen_excl ? launch_topk_t<T, kTail, NUC, false, true>(a, grid_rows, st)
                    : launch_topk_t<T, kTail, NUC>(a, grid_rows, st);
}

// dynamic shared memory of a top-k launch with the call's capacities
size_t topk_smem_bytes(const SampleArgs& a, int mode) {
  const int64_t n = mode == kFull ? a.V : (mode == kHot ? a.H : a.V - a.H);
  const int bm_words = (mode == kHot || a.pen_excl) ? (int)((n + 31) / 32) + 1 : 0;
  return topk_layout<DP_TOPK_NT>(a.wcap, a.kcap, a.lcap, bm_words, a.split).total;
}

// 256 threads per CTA (the 128-thread variant measured slower at every
// shape); the nucleus instantiation only when the call may hold such rows
cudaError_t launch_topk(const SampleArgs& a, int dtype, int mode, int grid_rows, cudaStream_t st) {
  const bool nuc = a.fb_rows != nullptr;
  if (dtype == DP_F32)
    return nuc ? launch_topk_m<float, true>(a, mode, grid_rows, st) : launch_topk_m<float, false>(a, mode, grid_rows, st);
  return nuc ? launch_topk_m<__nv_bfloat16, true>(a, mode, grid_rows, st)
             : launch_topk_m<__nv_bfloat16, false>(a, mode, grid_rows, st);
}

}  // namespace dp
