// sample_persist.cu — K1p: persistent, warp-specialised full-vocabulary
// top-k sampler (same decision law as K1, sample_topk.cu), sm_100a.
//
// Why: with one CTA per row, every CTA of a wave streams its row, then spends
// ~20 us in the exact select and the final stage (penalties, ordering, draw;
// finish.cuh) — latency chains during which its HBM share idles, and the next
// wave cannot start before the CTA exits.  At B = 1,024 rows on 592 resident
// CTAs that is two such gaps per call (profiles/r2/k1_timeline).
//
// K1p keeps one CTA per resident slot and loops over rows
// (row = blockIdx.x + i * gridDim.x).  Its warps split into two roles joined
// by two double-buffered candidate buffers in shared memory and four
// mbarriers (full[2] / empty[2]):
//   * 5 streaming warps: threshold from the first register batch, 16-byte
//     streaming loads, vector admission into candidate buffer i & 1, the
//     overflow / re-stream rule — exactly K1's stream stage — then hand the
//     buffer over and start the next row at once;
//   * 3 finishing warps: exact radix select of the raw top-(k + |list|)
//     (select.cuh), release the buffer, then finish_row (finish.cuh) on 96
//     threads — penalties in IEEE f64, /tau, canonical order, top-p / min-p,
//     inverse-CDF draw, fused penalty-state update — while the streaming
//     warps already stream the next row.
// Rows with top-k only (no nucleus rows, no TP shards, no clusters): the host
// routes everything else to K1.
#include "sampler.cuh"
#include "select.cuh"
#include "finish.cuh"

namespace dp {

#ifndef DP_PERSIST_NT
#define DP_PERSIST_NT 256
#define DP_PERSIST_MINB 4
#endif
constexpr int kPNT = DP_PERSIST_NT;  // threads per CTA
#ifndef DP_PERSIST_SW
#define DP_PERSIST_SW 5
#endif
// 5 streaming + 3 finishing warps: C2 122 us vs 129 (6 + 2), 145 (7 + 1),
// 132 (3 + 5); 4 + 4 is faster on fresh lists (120) but 140 us once the
// penalty lists grow (profiles/r2/k1p/warp_split_ab.txt)
constexpr int kPSW = DP_PERSIST_SW;  // streaming warps
constexpr int kPSNT = kPSW * 32;     // 192
constexpr int kPFNT = kPNT - kPSNT;  // finishing threads
constexpr uint32_t kBarStream = 1, kBarFin = 2;   // named barriers (0 = __syncthreads)
#ifndef DP_PERSIST_U_BF16
#define DP_PERSIST_U_BF16 4
#endif
constexpr int kPUBf16 = DP_PERSIST_U_BF16;   // bf16 vectors in flight per lane (8 elements each: fewer registers)

struct PBuf {            // one candidate buffer's row description (streamers -> finishers)
  uint32_t cnt;          // admitted vectors (slots used: min(cnt, ccap))
  uint32_t overflow;
  uint32_t nscal;        // scalar head / tail keys in scal[]
  uint32_t n_valid;      // keys >= thr among the buffer's elements + scal
  uint32_t dense;        // n_valid keys compacted at the buffer's unused slots (dense_of)
  uint64_t thr;          // admission threshold (composite key)
  uint64_t kor, kand;    // OR / AND of the valid keys (constant-digit skipping)
  uint64_t scal[16];     // <= 2 * EPV - 2 = 14 keys (bf16)
  uint64_t tl0, tl1;     // DP_TIMELINE: row start / hand-over (globaltimer)
};
DP_DEV uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct PersistSmem {
  uint64_t full[2], empty[2];
  PBuf buf[2];
  float thr_warp[kPSW], est_warp[kPSW];
  uint32_t tmp;                 // streamers' count scratch
  unsigned long long kor_s, kand_s;
  uint32_t bcast_s[4];          // streamers' select broadcast (overflow path)
  uint32_t bcast_f[4];          // finishers' select broadcast
  uint32_t nsel;
  FinishScratch fin;
};

struct PersistLayout {
  uint32_t cand0, cand1, sel, hist_s, hist_f, misc, total;
};
// Each candidate buffer also holds its row's final-stage scratch (fin_layout)
// once the select has copied the survivors out: the finishers release the
// buffer only after finish_row, so 2 x max(candidates, final stage) + small
// keeps 4 CTAs per SM at the bench's penalty-list lengths.
__host__ __device__ inline PersistLayout persist_layout(int ccap, int kcap, int lcap) {
  PersistLayout L;
  uint32_t cb = (uint32_t)ccap * 20u;   // 16-byte vectors + their positions
  const uint32_t fb = fin_layout(lcap).bytes;
  cb = ((cb > fb ? cb : fb) + 15u) & ~15u;
  uint32_t o = 0;
  L.cand0 = o; o += cb;
  L.cand1 = o; o += cb;
  L.sel = o; o += (uint32_t)kcap * 8u;
  L.hist_s = o; o += 1024u;
  L.hist_f = o; o += 1024u;
  L.misc = o; o += (sizeof(PersistSmem) + 15u) & ~15u;
  L.total = o;
  return L;
}

// does a later row of this CTA's sequence go to the top-k kernel?
DP_DEV bool more_topk_rows(const SampleArgs& a, int ridx) {
  for (int r = ridx + (int)gridDim.x; r < a.n_rows; r += (int)gridDim.x) {
    const dp_params_t p = a.params[r];
    if (route_row(a, kFull, p.top_k, pen_len(a, r, p), a.V) == kRouteTopk) return true;
  }
  return false;
}

// The CTA's last row: nothing left to stream, so all 8 warps run its select
// and final stage (the K1 schedule) — the kernel's tail is K1's, not the
// two-warp one.  Entered by every thread once the streamers have described
// buffer b and the finishers are done with the earlier rows.
template <typename T>
DP_DEV void all_hands(const SampleArgs& a, uint8_t* smem, const PersistLayout& L, PersistSmem& ms, int b, int row,
                      const dp_params_t& p, int32_t plen, uint32_t kp) {
  constexpr int EPV = Elem<T>::kPerVec;
  __syncthreads();
  const uint32_t tid = threadIdx.x;
  const uint32_t ccap = (uint32_t)a.wcap;
  const PBuf& pb = ms.buf[b];
  const uint4* cvec = reinterpret_cast<const uint4*>(smem + (b ? L.cand1 : L.cand0));
  const int32_t* cidx = reinterpret_cast<const int32_t*>(cvec + ccap);
  const T* celem = reinterpret_cast<const T*>(cvec);
  const uint64_t thr = pb.thr;
  const uint32_t ne = min(pb.cnt, ccap) * EPV;
  const uint32_t ns = ne + pb.nscal;
  auto get_c = [&](uint32_t i, uint64_t& key) -> bool {
    if (i >= ne) {
      key = pb.scal[i - ne];
      return true;
    }
    key = comp_key(to_f32(celem[i]), (uint32_t)cidx[i / EPV] + i % EPV);
    return key >= thr;
  };
  auto sync = [] { __syncthreads(); };
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L.hist_f);
  uint64_t* sel = reinterpret_cast<uint64_t*>(smem + L.sel);
  const uint64_t* dense = reinterpret_cast<const uint64_t*>(cvec + min(pb.cnt, ccap));
  auto get_d = [&](uint32_t i, uint64_t& key) -> bool { key = dense[i]; return true; };
  const uint64_t kvar = pb.kor ^ pb.kand;
  const uint64_t t = pb.dense
                         ? group_select_threshold<kPNT>(get_d, pb.n_valid, pb.n_valid, kp, hist, ms.bcast_f, tid,
                                                        sync, kvar, pb.kand)
                         : group_select_threshold<kPNT>(get_c, ns, pb.n_valid, kp, hist, ms.bcast_f, tid, sync, kvar,
                                                        pb.kand);
  if (tid == 0) ms.nsel = 0u;
  __syncthreads();
  if (pb.dense) {
    for (uint32_t i = tid; i < pb.n_valid; i += kPNT)
      if (dense[i] >= t) sel[atomicAdd(&ms.nsel, 1u)] = dense[i];
  } else {
    for (uint32_t i = tid; i < ns; i += kPNT) {
      uint64_t kk;
      if (get_c(i, kk) && kk >= t) sel[atomicAdd(&ms.nsel, 1u)] = kk;
    }
  }
  __syncthreads();
#ifdef DP_TIMELINE
  const uint64_t tl0 = pb.tl0, tl1 = pb.tl1, tl2 = gtimer();
#endif
  const T* rowp = reinterpret_cast<const T*>(a.logits) + (int64_t)row * a.ld;
  finish_row<T, kFull, kPNT, false, false>(a, row, p, plen, rowp, 0, a.V, sel, ms.nsel, 0.0, 0.0,
                                    smem + (b ? L.cand1 : L.cand0), fin_layout(a.lcap), ms.fin, tid, sync, nullptr,
                                    0.f);
#ifdef DP_TIMELINE
  __syncthreads();
  if (tid == 0 && a.dbg.topk_ready) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    double* tl = a.dbg.topk_ready + (int64_t)row * a.dbg.topk_stride;
    tl[0] = (double)tl0; tl[1] = (double)tl1; tl[2] = (double)tl2; tl[3] = (double)gtimer(); tl[4] = (double)smid;
  }
#endif
}

template <typename T, int U>
__global__ void __launch_bounds__(kPNT, DP_PERSIST_MINB) topk_persist_kernel(SampleArgs a) {
  constexpr int EPV = Elem<T>::kPerVec;
  extern __shared__ __align__(16) uint8_t smem[];
  const PersistLayout L = persist_layout(a.wcap, a.kcap, a.lcap);
  PersistSmem& ms = *reinterpret_cast<PersistSmem*>(smem + L.misc);
  const uint32_t ccap = (uint32_t)a.wcap;
  const int64_t n = a.V;
  const int nrows = a.n_rows;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&ms.full[0], 1);
    mbar_init(&ms.full[1], 1);
    mbar_init(&ms.empty[0], 1);
    mbar_init(&ms.empty[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // candidate source of buffer b: elements of admitted vectors >= thr, then
  // the scalar head / tail keys
  auto cvec_of = [&](int b) { return reinterpret_cast<uint4*>(smem + (b ? L.cand1 : L.cand0)); };
  auto cidx_of = [&](int b) { return reinterpret_cast<int32_t*>(cvec_of(b) + ccap); };

  // the CTA's last top-k row, finished by all 8 warps at ONE call site after
  // both role loops (every warp then executes the same barrier instructions)
  int ah_row = -1, ah_b = 0;
  if (tid < (uint32_t)kPSNT) {
    // ======================= streaming warps =======================
    const uint32_t warp = tid >> 5, lane = tid & 31u;
    auto sync_s = [] { named_bar_sync(kBarStream, kPSNT); };
    uint32_t* hist_s = reinterpret_cast<uint32_t*>(smem + L.hist_s);
    uint32_t j = 0;   // rows handed over so far
    for (int ridx = blockIdx.x; ridx < nrows; ridx += gridDim.x) {
      const int row = ridx;
      const dp_params_t p = a.params[row];
      const int32_t plen = pen_len(a, row, p);
      const int32_t k = p.top_k;
      if (route_row(a, kFull, k, plen, n) != kRouteTopk) continue;   // another kernel's row
      const uint32_t kp = (uint32_t)min64(n, (int64_t)k + plen);
      const int b = (int)(j & 1u);
      if (j >= 2) mbar_wait(&ms.empty[b], ((j >> 1) - 1u) & 1u);   // the finishers released buffer b
      PBuf& pb = ms.buf[b];
      uint4* cvec = cvec_of(b);
      int32_t* cidx = cidx_of(b);
      const T* celem = reinterpret_cast<const T*>(cvec);
      const T* rowp = reinterpret_cast<const T*>(a.logits) + (int64_t)row * a.ld;
      const uintptr_t addr = reinterpret_cast<uintptr_t>(rowp);
      const int32_t a0 = (int32_t)min64(n, (int64_t)(((16u - (addr & 15u)) & 15u) / sizeof(T)));
      const int32_t nvec = (int32_t)((n - a0) / EPV);
      const int32_t tail0 = a0 + nvec * EPV;
      const uint4* vp = reinterpret_cast<const uint4*>(rowp + a0);
      if (tid == 0) {
        pb.cnt = 0u;
        pb.overflow = 0u;
        pb.nscal = 0u;
#ifdef DP_TIMELINE
        pb.tl0 = gtimer();
#endif
      }
      sync_s();
      uint64_t thr = 0ull;
      float thr_f = -INFINITY, t_lb = -INFINITY;
      uint64_t loaded = 0;
      auto get_c = [&](uint32_t i, uint64_t& key) -> bool {
        const uint32_t ne = min(pb.cnt, ccap) * EPV;
        if (i >= ne) {
          key = pb.scal[i - ne];
          return true;
        }
        const float x = to_f32(celem[i]);
        key = comp_key(x, (uint32_t)cidx[i / EPV] + i % EPV);
        return key >= thr;
      };
      uint32_t n_valid = 0;
      uint64_t kor = 0ull, kand = 0ull;
      bool dense_ok = false;
      for (int pass_no = 0;; ++pass_no) {
        if (tid == 0) loaded += (uint64_t)nvec * 16u + (uint64_t)(a0 + (n - tail0)) * sizeof(T);
        int32_t base = (int32_t)warp * 32 * U;
        uint4 v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int32_t idx = base + q * 32 + (int32_t)lane;
          v[q] = idx < nvec ? ld_stream16(vp + idx) : neg_inf_vec<T>();
        }
        // this warp's next chunk -> L2 (one lane, distance 1 as K1)
        if (lane == 0 && base + kPSNT * U + 32 * U <= nvec) prefetch_l2(vp + base + kPSNT * U, 32u * U * 16u);
        if (pass_no == 0) {
          // t_lb: min over warps of the ceil(kp/NW)-th largest lane maximum of the
          // first batch (a proven lower bound of the row's kp-th largest);
          // t_est: median of the warps' estimates of the (2 kp)-th largest
          float mx = -INFINITY;
#pragma unroll
          for (int q = 0; q < U; ++q)
#pragma unroll
            for (int e = 0; e < EPV; ++e) mx = fmaxf(mx, vec_elem<T>(v[q], e));
          const uint32_t kw = (kp + kPSW - 1) / kPSW;
          int rw = (int)ceilf(est_over(kp, false) * (float)kp * (float)(32 * U * EPV) / (float)max((int64_t)1, n));
          rw = max(1, min(32, rw));
          const uint32_t sorted = warp_sort_desc(f32_key(mx));
          const uint32_t t_lbk = __shfl_sync(0xffffffffu, sorted, kw <= 32 ? kw - 1 : 31);
          const uint32_t t_ek = __shfl_sync(0xffffffffu, sorted, rw - 1);
          if (lane == 0) {
            ms.thr_warp[warp] = kw <= 32 ? key_f32(t_lbk) : -INFINITY;
            ms.est_warp[warp] = key_f32(t_ek);
          }
          sync_s();
          float tl = ms.thr_warp[0];
          float ev[kPSW];
#pragma unroll
          for (int w = 0; w < kPSW; ++w) {
            tl = fminf(tl, ms.thr_warp[w]);
            ev[w] = ms.est_warp[w];
          }
#pragma unroll
          for (int i = 1; i < kPSW; ++i)
#pragma unroll
            for (int j2 = i; j2 > 0; --j2)
              if (ev[j2] > ev[j2 - 1]) { const float t2 = ev[j2]; ev[j2] = ev[j2 - 1]; ev[j2 - 1] = t2; }
          t_lb = tl;
          const float te = fmaxf(ev[(kPSW - 1) / 2], t_lb);
          thr_f = te;
          thr = te == -INFINITY ? 0ull : ((uint64_t)f32_key(te) << 32);
        }
        if (warp == 0) {   // scalar head / tail elements
          const int32_t hi_i = (int32_t)lane, ti = tail0 + (int32_t)lane;
          const bool hv = hi_i < a0, tv = ti < n;
          const float hx = hv ? Elem<T>::get(rowp, hi_i) : -INFINITY;
          const float tx = tv ? Elem<T>::get(rowp, ti) : -INFINITY;
          const bool hp = hv && comp_key(hx, (uint32_t)hi_i) >= thr;
          const bool tp = tv && comp_key(tx, (uint32_t)ti) >= thr;
          const uint32_t mh = __ballot_sync(0xffffffffu, hp), mt = __ballot_sync(0xffffffffu, tp);
          if (hp) pb.scal[__popc(mh & lanemask_lt())] = comp_key(hx, (uint32_t)hi_i);
          if (tp) pb.scal[__popc(mh) + __popc(mt & lanemask_lt())] = comp_key(tx, (uint32_t)ti);
          if (lane == 0) pb.nscal = (uint32_t)(__popc(mh) + __popc(mt));
        }
        const bool exact_mode = (uint32_t)thr != 0u;
        while (true) {
          uint32_t vm = 0;
          const bool full = base + 32 * U <= nvec;
#pragma unroll
          for (int q = 0; q < U; ++q) {
            float mx = vec_elem<T>(v[q], 0);
#pragma unroll
            for (int e = 1; e < EPV; ++e) mx = fmaxf(mx, vec_elem<T>(v[q], e));
            vm |= (mx >= thr_f ? 1u : 0u) << q;
          }
          if (!full) {
#pragma unroll
            for (int q = 0; q < U; ++q)
              if (base + q * 32 + (int32_t)lane >= nvec) vm &= ~(1u << q);
          }
          if (exact_mode && vm) {
#pragma unroll
            for (int q = 0; q < U; ++q) {
              if ((vm >> q) & 1u) {
                const int32_t idx = base + q * 32 + (int32_t)lane;
                bool ex = false;
#pragma unroll
                for (int e = 0; e < EPV; ++e) ex |= comp_key(vec_elem<T>(v[q], e), (uint32_t)(a0 + idx * EPV + e)) >= thr;
                if (!ex) vm &= ~(1u << q);
              }
            }
          }
          if (vm) {
            uint32_t slot = atomicAdd(&pb.cnt, (uint32_t)__popc(vm));
#pragma unroll
            for (int q = 0; q < U; ++q) {
              if ((vm >> q) & 1u) {
                if (slot < ccap) {
                  cvec[slot] = v[q];
                  cidx[slot] = a0 + (base + q * 32 + (int32_t)lane) * EPV;
                } else {
                  pb.overflow = 1u;
                }
                ++slot;
              }
            }
          }
          base += kPSNT * U;
          if (base >= nvec) break;
          if (lane == 0 && base + kPSNT * U + 32 * U <= nvec) prefetch_l2(vp + base + kPSNT * U, 32u * U * 16u);
          if (base + 32 * U <= nvec) {
            const uint4* q0 = vp + base + (int32_t)lane;
#pragma unroll
            for (int q = 0; q < U; ++q) v[q] = ld_stream16(q0 + q * 32);
          } else {
#pragma unroll
            for (int q = 0; q < U; ++q) {
              const int32_t idx = base + q * 32 + (int32_t)lane;
              v[q] = idx < nvec ? ld_stream16(vp + idx) : neg_inf_vec<T>();
            }
          }
        }
        sync_s();
        // keys >= thr in the buffer (+ scalars)
        const bool overflow = pb.overflow != 0u;
        const uint32_t nc = min(pb.cnt, ccap);
        const uint32_t dcap = overflow ? 0u : (ccap - nc) * 2u;
        const DenseStats ds = group_compact_valid<kPSNT>(get_c, nc * EPV + pb.nscal,
                                                         reinterpret_cast<uint64_t*>(cvec + nc), dcap, &ms.tmp,
                                                         &ms.kor_s, &ms.kand_s, tid, sync_s);
        n_valid = ds.n;
        kor = ds.kor;
        kand = ds.kand;
        dense_ok = n_valid <= dcap;
        bool again = false;
        if (overflow) {
          // the buffer holds a subset of the admitted elements: its kp-th largest
          // key is a valid, strictly higher threshold
          const uint64_t t1 = group_select_threshold<kPSNT>(get_c, ccap * EPV + pb.nscal, n_valid, kp, hist_s,
                                                            ms.bcast_s, tid, sync_s, kor ^ kand, kand);
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
        sync_s();
        if (tid == 0) {
          pb.cnt = 0u;
          pb.overflow = 0u;
        }
        sync_s();
      }
      if (tid == 0) {
        pb.thr = thr;
        pb.n_valid = n_valid;
        pb.dense = dense_ok ? 1u : 0u;
        pb.kor = kor;
        pb.kand = kand;
        touch_bytes(a, row, loaded);
#ifdef DP_TIMELINE
        pb.tl1 = gtimer();
#endif
      }
      sync_s();
      if (!more_topk_rows(a, ridx)) {   // the CTA's last row: every warp finishes it (below)
        ah_row = row;
        ah_b = b;
        break;
      }
      if (tid == 0) mbar_arrive(&ms.full[b]);   // release: the buffer and its description
      ++j;
    }
  } else {
    // ======================= finishing warps =======================
    const uint32_t ft = tid - (uint32_t)kPSNT;
    auto sync_f = [] { named_bar_sync(kBarFin, kPFNT); };
    uint32_t* hist_f = reinterpret_cast<uint32_t*>(smem + L.hist_f);
    uint64_t* sel = reinterpret_cast<uint64_t*>(smem + L.sel);
    const FinLayout F = fin_layout(a.lcap);
    uint32_t j = 0;
    for (int ridx = blockIdx.x; ridx < nrows; ridx += gridDim.x) {
      const int row = ridx;
      const dp_params_t p = a.params[row];
      const int32_t plen = pen_len(a, row, p);
      const int32_t k = p.top_k;
      if (route_row(a, kFull, k, plen, n) != kRouteTopk) continue;
      const uint32_t kp = (uint32_t)min64(n, (int64_t)k + plen);
      const int b = (int)(j & 1u);
      if (!more_topk_rows(a, ridx)) {   // the last row: joined by the streaming warps (below)
        ah_row = row;
        ah_b = b;
        break;
      }
      mbar_wait(&ms.full[b], (j >> 1) & 1u);
      PBuf& pb = ms.buf[b];
      const uint4* cvec = cvec_of(b);
      const int32_t* cidx = cidx_of(b);
      const T* celem = reinterpret_cast<const T*>(cvec);
      const uint64_t thr = pb.thr;
#ifdef DP_TIMELINE
      const uint64_t tl0 = pb.tl0, tl1 = pb.tl1;
#endif
      const uint32_t ne = min(pb.cnt, ccap) * EPV;
      const uint32_t ns = ne + pb.nscal;
      auto get_c = [&](uint32_t i, uint64_t& key) -> bool {
        if (i >= ne) {
          key = pb.scal[i - ne];
          return true;
        }
        const float x = to_f32(celem[i]);
        key = comp_key(x, (uint32_t)cidx[i / EPV] + i % EPV);
        return key >= thr;
      };
      // exact top-kp of the row's candidates (unique composite keys): from the
      // streamers' dense copy of the valid keys when it fit
      const uint64_t* dense = reinterpret_cast<const uint64_t*>(cvec + min(pb.cnt, ccap));
      auto get_d = [&](uint32_t i, uint64_t& key) -> bool { key = dense[i]; return true; };
      const uint64_t kvar = pb.kor ^ pb.kand;
      const uint64_t t = pb.dense ? group_select_threshold<kPFNT>(get_d, pb.n_valid, pb.n_valid, kp, hist_f,
                                                                  ms.bcast_f, ft, sync_f, kvar, pb.kand)
                                  : group_select_threshold<kPFNT>(get_c, ns, pb.n_valid, kp, hist_f, ms.bcast_f, ft,
                                                                  sync_f, kvar, pb.kand);
      if (ft == 0) ms.nsel = 0u;
      sync_f();
      if (pb.dense) {
        for (uint32_t i = ft; i < pb.n_valid; i += kPFNT)
          if (dense[i] >= t) sel[atomicAdd(&ms.nsel, 1u)] = dense[i];
      } else {
        for (uint32_t i = ft; i < ns; i += kPFNT) {
          uint64_t kk;
          if (get_c(i, kk) && kk >= t) sel[atomicAdd(&ms.nsel, 1u)] = kk;
        }
      }
      sync_f();
      const uint32_t nsel = ms.nsel;
#ifdef DP_TIMELINE
      const uint64_t tl2 = gtimer();
#endif
      const T* rowp = reinterpret_cast<const T*>(a.logits) + (int64_t)row * a.ld;
      // the final stage's scratch lives in buffer b (its candidates are in sel now)
      finish_row<T, kFull, kPFNT, false, false>(a, row, p, plen, rowp, 0, n, sel, nsel, 0.0, 0.0,
                                         reinterpret_cast<uint8_t*>(const_cast<uint4*>(cvec)), F, ms.fin, ft, sync_f,
                                         nullptr, 0.f);
      sync_f();
      if (ft == 0) mbar_arrive(&ms.empty[b]);   // buffer b may be refilled
#ifdef DP_TIMELINE
      sync_f();
      if (ft == 0 && a.dbg.topk_ready) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        double* tl = a.dbg.topk_ready + (int64_t)row * a.dbg.topk_stride;
        tl[0] = (double)tl0; tl[1] = (double)tl1; tl[2] = (double)tl2; tl[3] = (double)gtimer(); tl[4] = (double)smid;
      }
#endif
      ++j;
    }
  }
  if (ah_row >= 0) {
    const dp_params_t p = a.params[ah_row];
    const int32_t plen = pen_len(a, ah_row, p);
    const uint32_t kp = (uint32_t)min64(n, (int64_t)p.top_k + plen);
    all_hands<T>(a, smem, L, ms, ah_b, ah_row, p, plen, kp);
  }
}

size_t persist_smem_bytes(const SampleArgs& a) { return persist_layout(a.wcap, a.kcap, a.lcap).total; }

// grid = resident CTAs (the kernel loops over rows); 0 when it cannot run
int persist_grid(const SampleArgs& a, int dtype) {
  const size_t smem = persist_smem_bytes(a);
  int per_sm = 0, dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e;
  if (dtype == DP_F32) {
    auto k = topk_persist_kernel<float, 8>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kPNT, smem);
  } else {
    auto k = topk_persist_kernel<__nv_bfloat16, kPUBf16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kPNT, smem);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return per_sm * sms;
}

cudaError_t launch_persist(const SampleArgs& a, int dtype, int grid, cudaStream_t st) {
  const size_t smem = persist_smem_bytes(a);
  if (dtype == DP_F32) {
    auto k = topk_persist_kernel<float, 8>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, kPNT, smem, st>>>(a);
  } else {
    auto k = topk_persist_kernel<__nv_bfloat16, kPUBf16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, kPNT, smem, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace dp
