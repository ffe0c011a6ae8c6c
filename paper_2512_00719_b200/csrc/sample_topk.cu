// sample_topk.cu — fused single-pass top-k sampler (K1), sm_100a.
//
// One thread-block CLUSTER per row; the row's domain is split across the
// cluster's CTAs, each streaming its segment exactly once from HBM with
// 16-byte non-allocating loads (8 in flight per lane).  Selection keeps the
// candidates of the raw top-(k + |penalty list|) — the exact superset argument
// of _Sampler._tail_preselect (service.py:309-336): an unpenalized element
// below the raw (k + |touched|)-th largest is dominated by k unpenalized
// elements whose ready value keeps its raw order, so it cannot reach the top-k.
// Per-warp candidate buffers with a shared running threshold; exact radix
// selection on unique (value desc, position asc) keys gives the canonical
// boundary-tie rule of _top_k_ids (filtering.py:38-58).  The cluster's CTA 0
// pulls the other CTAs' survivors over DSMEM, applies the sparse penalties in
// IEEE f64 (penalty.py:66-78), divides by tau (service.py:236-241), sorts, and
// runs the exact top-p / min-p / inverse-CDF draw (filtering.py:61-162).
//
// kHot additionally accumulates the hot mass S_H (shvs.py:223-230) and decides
// acceptance; kTail serves the rows the hot pass rejected.

#include "sampler.cuh"
#include "select.cuh"

namespace dp {

template <int NT>
struct TopkSmem {
  static constexpr int NW = NT / 32;
  uint64_t cta_thr;
  double sh_part[NW];
  double sh_pen[NW];
  uint32_t wcnt[NW];
  uint32_t nsel;
  uint32_t bcast[4];
  uint32_t offs[16];
  uint32_t nl;
  int32_t decision;     // kHot: 1 accept, 0 reject
  double alpha;
};

// smem carve-up, shared by host sizing and device code
struct TopkLayout {
  uint32_t wbuf, sel, whist, bhist, bitmap, misc, total;
  uint32_t fin_key, fin_pos, fin_r, fin_w, fin_cum, fin_hash, hash_cap;
};
template <int NT>
__host__ __device__ inline TopkLayout topk_layout(int wcap, int kcap, int lcap, int bitmap_words,
                                                 int split) {
  constexpr int NW = NT / 32;
  TopkLayout L;
  uint32_t o = 0;
  L.wbuf = o;
  uint32_t region = (uint32_t)NW * wcap * 8u;
  // the rank-0 merge buffer and the final-stage arrays alias the warp buffers
  uint32_t merge = (uint32_t)split * kcap * 8u;
  L.hash_cap = 1;
  while (L.hash_cap < 2u * (uint32_t)lcap) L.hash_cap <<= 1;
  uint32_t fin = 0;
  L.fin_key = fin; fin += lcap * 8u;
  L.fin_r = fin; fin += lcap * 8u;
  L.fin_w = fin; fin += lcap * 8u;
  L.fin_cum = fin; fin += lcap * 8u;
  L.fin_pos = fin; fin += lcap * 4u;
  L.fin_hash = fin; fin += L.hash_cap * 4u;
  region = region > merge ? region : merge;
  region = region > fin ? region : fin;
  o += (region + 15u) & ~15u;
  L.sel = o; o += kcap * 8u;
  L.whist = o; o += NW * 256u * 4u;
  L.bhist = o; o += 256u * 4u;
  L.bitmap = o; o += ((uint32_t)bitmap_words * 4u + 15u) & ~15u;
  L.misc = o; o += (sizeof(TopkSmem<NT>) + 15u) & ~15u;
  L.total = o;
  return L;
}

template <typename T, int MODE, int NT, int U>
__global__ void __launch_bounds__(NT) topk_sample_kernel(SampleArgs a) {
  constexpr int NW = NT / 32;
  constexpr int EPV = Elem<T>::kPerVec;
  extern __shared__ __align__(16) uint8_t smem[];
  const int64_t n = dom_n(a, MODE);
  const int64_t lo = dom_lo(a, MODE);
  const uint32_t bm_words = MODE == kHot ? (uint32_t)((n + 31) / 32) : 0u;
  const TopkLayout L = topk_layout<NT>(a.wcap, a.kcap, a.lcap, (int)bm_words, a.split);
  uint64_t* wbuf = reinterpret_cast<uint64_t*>(smem + L.wbuf);
  uint64_t* sel = reinterpret_cast<uint64_t*>(smem + L.sel);
  uint32_t* whist = reinterpret_cast<uint32_t*>(smem + L.whist);
  uint32_t* bhist = reinterpret_cast<uint32_t*>(smem + L.bhist);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem + L.bitmap);
  TopkSmem<NT>& ms = *reinterpret_cast<TopkSmem<NT>*>(smem + L.misc);

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  const uint32_t split = (uint32_t)a.split;
  const uint32_t rank = split > 1 ? cluster_ctarank() : 0u;
  const int ridx = blockIdx.x / split;
  const int nrows = a.row_count ? *a.row_count : a.n_rows;
  if (ridx >= nrows) return;                                    // uniform per cluster
  const int row = a.rows ? a.rows[ridx] : ridx;
  const dp_params_t p = a.params[row];
  const int32_t plen = pen_len(a, row, p);
  const int32_t k = p.top_k;
  // kHot excludes penalized ids from the stream (bitmap) so no widening
  const uint32_t kp = (uint32_t)min64(n, (int64_t)k + (MODE == kHot ? 0 : plen));
  if (!(k > 0 && (int64_t)k < n && kp <= (uint32_t)a.kcap && (uint32_t)(k + 2 * plen) <= (uint32_t)a.lcap))
    return;                                                     // general-path row

  const T* rowp = reinterpret_cast<const T*>(a.logits) + (int64_t)row * a.ld + lo;
  const int32_t* pids = a.pen.ids + (int64_t)row * a.pen.cap;
  const int32_t* pcnt = a.pen.out_count + (int64_t)row * a.pen.cap;

  // ---- setup
  if (tid == 0) {
    ms.cta_thr = 0ull;
    ms.nsel = 0u;
    ms.nl = 0u;
  }
  double mrow = 0.0;
  float mtau_hi = 0.f, mtau_lo = 0.f;
  float inv_tau = (float)(1.0 / p.temperature);
  if (MODE == kHot) {
    for (uint32_t i = tid; i < bm_words; i += NT) bitmap[i] = 0u;
    __syncthreads();
    for (int32_t j = tid; j < plen; j += NT) {
      const int64_t pos = id_to_pos(a, pids[j]) - lo;
      if (pos >= 0 && pos < n) atomicOr(&bitmap[pos >> 5], 1u << (pos & 31));
    }
    mrow = a.row_max[row];
    const double c = mrow * p.temperature;
    mtau_hi = (float)c;
    mtau_lo = (float)(c - (double)(float)c);
  }
  __syncthreads();

  // ---- stream this CTA's segment once
  const uintptr_t addr = reinterpret_cast<uintptr_t>(rowp);
  const int64_t a0 = min64(n, (int64_t)(((16u - (addr & 15u)) & 15u) / sizeof(T)));
  const int64_t nvec = (n - a0) / EPV;
  const int64_t tail0 = a0 + nvec * EPV;
  const int64_t chunk = ((nvec + split - 1) / split + 31) & ~31ll;
  const int64_t v_lo = min64(nvec, (int64_t)rank * chunk);
  const int64_t v_hi = min64(nvec, v_lo + chunk);
  const uint4* vp = reinterpret_cast<const uint4*>(rowp + a0);

  uint64_t* mybuf = wbuf + (size_t)warp * a.wcap;
  uint32_t* myhist = whist + warp * 256u;
  uint32_t cnt = 0;
  uint64_t thr = 0ull;
  float thr_f = -INFINITY;
  double sh = 0.0;  // kHot partial hot mass (unpenalized ids)

  auto admit = [&](float x, int64_t pos, bool valid) {
    bool pass = valid && x >= thr_f;
    if (MODE == kHot && pass) pass = !((bitmap[pos >> 5] >> (pos & 31)) & 1u);
    uint64_t key = 0ull;
    if (pass) {
      key = comp_key(x, (uint32_t)pos);
      pass = key >= thr;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, pass);
    if (m) {
      if (pass) mybuf[cnt + __popc(m & lanemask_lt())] = key;
      cnt += __popc(m);
    }
  };
  auto accum = [&](float x, int64_t pos, bool valid) {
    if (MODE == kHot && valid && !((bitmap[pos >> 5] >> (pos & 31)) & 1u)) {
      const float d = (x - mtau_hi) - mtau_lo;
      sh += (double)__expf(d * inv_tau);
    }
  };
  auto compact = [&]() {
    __syncwarp();
    uint64_t t = warp_select_threshold(mybuf, cnt, kp, myhist);
    const uint64_t ct = *reinterpret_cast<volatile uint64_t*>(&ms.cta_thr);
    if (ct > t) t = ct;
    if (t > thr) {
      thr = t;
      const uint32_t hk = (uint32_t)(thr >> 32);
      const float f = key_f32(hk);
      thr_f = (hk < 0x00800000u || f != f) ? -INFINITY : f;   // below -inf key: admit all
    }
    cnt = warp_compact(mybuf, cnt, thr);
    if (lane == 0 && cnt >= kp) atomicMax(reinterpret_cast<unsigned long long*>(&ms.cta_thr),
                                          (unsigned long long)thr);
  };

  // scalar head / tail elements (at most 2*EPV-2) go to CTA 0, warp 0
  if (rank == 0 && warp == 0) {
    const int64_t i = lane;
    const bool hv = i < a0;
    const int64_t ti = tail0 + lane;
    const bool tv = ti < n;
    const float hx = hv ? Elem<T>::get(rowp, i) : -INFINITY;
    const float tx = tv ? Elem<T>::get(rowp, ti) : -INFINITY;
    accum(hx, i, hv);
    accum(tx, ti, tv);
    admit(hx, i, hv);
    admit(tx, ti, tv);
  }

  for (int64_t base = v_lo + (int64_t)warp * 32 * U; base < v_hi; base += (int64_t)NT * U) {
    uint4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t idx = base + j * 32 + lane;
      v[j] = idx < v_hi ? ld_stream16(vp + idx) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t idx = base + j * 32 + lane;
      const bool valid = idx < v_hi;
      const int64_t pos0 = a0 + idx * EPV;
#pragma unroll
      for (int h = 0; h < EPV; h += 4) {
        if (cnt + 128 > (uint32_t)a.wcap) compact();
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = vec_elem<T>(v[j], h + e);
          accum(x, pos0 + h + e, valid);
          admit(x, pos0 + h + e, valid);
        }
      }
    }
  }

  // ---- CTA-level exact top-kp over the warp buffers
  if (lane == 0) ms.wcnt[warp] = cnt;
  if (MODE == kHot) {
    const double s = warp_sum(sh);
    if (lane == 0) ms.sh_part[warp] = s;
  }
  __syncthreads();
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) total += ms.wcnt[w];
  const int wcap = a.wcap;
  auto get_w = [&](uint32_t i, uint64_t& key) -> bool {
    const uint32_t w = i / wcap, j = i - w * wcap;
    if (j >= ms.wcnt[w]) return false;
    key = wbuf[i];
    return true;
  };
  uint64_t t = block_select_threshold<NT>(get_w, (uint32_t)(NW * wcap), total, kp, bhist, ms.bcast);
  for (uint32_t i = tid; i < (uint32_t)(NW * wcap); i += NT) {
    uint64_t key;
    if (get_w(i, key) && key >= t) sel[atomicAdd(&ms.nsel, 1u)] = key;
  }
  if (MODE == kHot && tid == 0) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += ms.sh_part[w];
    ms.sh_part[0] = s;
  }
  __syncthreads();

  // ---- cluster merge into CTA 0 over DSMEM
  if (split > 1) {
    cluster_sync();
    if (rank != 0) {
      cluster_arrive();
      cluster_wait();
      return;
    }
    if (tid == 0) {
      uint32_t off = 0;
      double s = 0.0;
      for (uint32_t r = 0; r < split; ++r) {
        ms.offs[r] = off;
        off += ld_dsmem_u32(dsmem_addr(&ms.nsel, r));
        if (MODE == kHot) s += __longlong_as_double((long long)ld_dsmem_u64(dsmem_addr(&ms.sh_part[0], r)));
      }
      ms.offs[split] = off;
      if (MODE == kHot) ms.sh_part[0] = s;
    }
    __syncthreads();
    const uint32_t ntot = ms.offs[split];
    for (uint32_t r = 0; r < split; ++r) {
      const uint32_t nr = ms.offs[r + 1] - ms.offs[r];
      const uint32_t src = dsmem_addr(sel, r);
      for (uint32_t i = tid; i < nr; i += NT) wbuf[ms.offs[r] + i] = ld_dsmem_u64(src + 8u * i);
    }
    __syncthreads();
    cluster_arrive();   // remote CTAs may exit once everyone has copied
    auto get_m = [&](uint32_t i, uint64_t& key) -> bool {
      key = wbuf[i];
      return true;
    };
    if (tid == 0) ms.nsel = 0u;
    __syncthreads();
    t = block_select_threshold<NT>(get_m, ntot, ntot, kp, bhist, ms.bcast);
    for (uint32_t i = tid; i < ntot; i += NT)
      if (wbuf[i] >= t) sel[atomicAdd(&ms.nsel, 1u)] = wbuf[i];
    __syncthreads();
  }

  // ---- final stage (CTA 0): penalties, exact sort, filter, draw
  uint64_t* fkey = reinterpret_cast<uint64_t*>(smem + L.wbuf + L.fin_key);
  double* fr = reinterpret_cast<double*>(smem + L.wbuf + L.fin_r);
  double* fw = reinterpret_cast<double*>(smem + L.wbuf + L.fin_w);
  double* fcum = reinterpret_cast<double*>(smem + L.wbuf + L.fin_cum);
  uint32_t* fpos = reinterpret_cast<uint32_t*>(smem + L.wbuf + L.fin_pos);
  uint32_t* hash = reinterpret_cast<uint32_t*>(smem + L.wbuf + L.fin_hash);
  const uint32_t hmask = L.hash_cap - 1u;
  const uint32_t nsel = ms.nsel;
  double u[3];
  get_uniforms(a, row, p, u);

  // kHot: alpha and the accept test first (shvs.py:223-236)
  double alpha = 1.0;
  bool degenerate = false;
  if (MODE == kHot) {
    // exact hot mass of penalized hot ids (f64) + unpenalized stream partial
    double spen = 0.0;
    for (int32_t j = tid; j < plen; j += NT) {
      const int64_t pos = id_to_pos(a, pids[j]) - lo;
      if (pos >= 0 && pos < n) spen += exp(ready_penalized(Elem<T>::get(rowp, pos), pcnt[j], p) - mrow);
    }
    spen = warp_sum(spen);
    __syncthreads();
    if (lane == 0) ms.sh_pen[warp] = spen;
    __syncthreads();
    double sH = ms.sh_part[0];
    for (int w = 0; w < NW; ++w) sH += ms.sh_pen[w];     // fixed order: deterministic
    const double S = a.total_expsum[row];
    const bool tail_empty = a.V == a.H;
    if (!tail_empty) {
      if (!(S > 0.0) || !isfinite(S)) degenerate = true;
      else alpha = fmin(sH / S, 1.0);
    }
    const bool accept = !degenerate && sH > 0.0 && (tail_empty || u[1] <= alpha);
    if (!accept) {
      if (tid == 0) {
        uint8_t fl = DP_FLAG_REJECTED;
        if (degenerate || (tail_empty && !(sH > 0.0))) fl |= DP_FLAG_DEGENERATE;
        else if (fabs(u[1] - alpha) < kBoundaryEps) fl |= DP_FLAG_NEAR_BOUNDARY;
        a.flags[row] = fl;
        if (a.dbg.alpha) a.dbg.alpha[row] = alpha;
        if (a.dbg.margin) a.dbg.margin[row] = fabs(u[1] - alpha);
        if (a.dbg.bytes_touched) a.dbg.bytes_touched[row] = (uint64_t)n * sizeof(T);
        if (!(fl & DP_FLAG_DEGENERATE)) a.reject_rows[atomicAdd(a.reject_count, 1)] = row;
        else { a.token[row] = -1; a.logprob[row] = 0.0; }
      }
      if (split > 1) cluster_wait();
      return;
    }
  }

  // penalized positions of this domain -> hash set (raw candidates defer to them)
  for (uint32_t i = tid; i < L.hash_cap; i += NT) hash[i] = 0xFFFFFFFFu;
  __syncthreads();
  for (int32_t j = tid; j < plen; j += NT) {
    const int64_t pos = id_to_pos(a, pids[j]) - lo;
    if (pos >= 0 && pos < n) {
      uint32_t h = ((uint32_t)pos * 2654435761u) & hmask;
      while (atomicCAS(&hash[h], 0xFFFFFFFFu, (uint32_t)pos) != 0xFFFFFFFFu) h = (h + 1u) & hmask;
      const uint32_t s = atomicAdd(&ms.nl, 1u);
      const double r = ready_penalized(Elem<T>::get(rowp, pos), pcnt[j], p);
      fr[s] = r;
      fpos[s] = (uint32_t)pos;
    }
  }
  __syncthreads();
  for (uint32_t i = tid; i < nsel; i += NT) {
    const uint64_t key = sel[i];
    const uint32_t pos = comp_pos(key);
    bool is_pen = false;
    if (plen > 0) {
      uint32_t h = (pos * 2654435761u) & hmask;
      while (true) {
        const uint32_t v = hash[h];
        if (v == pos) { is_pen = true; break; }
        if (v == 0xFFFFFFFFu) break;
        h = (h + 1u) & hmask;
      }
    }
    if (!is_pen) {
      const uint32_t s = atomicAdd(&ms.nl, 1u);
      fr[s] = ready_plain(comp_val(key), p);
      fpos[s] = pos;
    }
  }
  __syncthreads();
  const uint32_t nl = ms.nl;
  uint32_t p2 = 1;
  while (p2 < nl) p2 <<= 1;
  for (uint32_t i = tid; i < p2; i += NT) {
    if (i < nl) {
      fkey[i] = f64_key(fr[i]);
    } else {
      fkey[i] = 0ull;
      fpos[i] = 0xFFFFFFFFu;
    }
  }
  __syncthreads();
  // bitonic sort, descending by (key, -pos)
  for (uint32_t size = 2; size <= p2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = tid; i < p2 / 2; i += NT) {
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
      __syncthreads();
    }
  }
  for (uint32_t i = tid; i < nl; i += NT) {
    const uint64_t kk = fkey[i];
    const uint64_t b = (kk >> 63) ? (kk & 0x7FFFFFFFFFFFFFFFull) : ~kk;
    fr[i] = __longlong_as_double((long long)b);
  }
  __syncthreads();

  if (warp == 0) {
    const DrawResult d = warp_filter_draw(fr, k, p, u[MODE == kTail ? 2 : 0], fw, fcum);
    if (lane == 0) {
      const int64_t pos = (int64_t)fpos[d.index] + lo;
      a.token[row] = pos_to_id(a, pos);
      a.logprob[row] = d.logprob;
      uint8_t fl = MODE == kHot ? DP_FLAG_ACCEPTED_HOT : (MODE == kTail ? DP_FLAG_REJECTED : 0);
      double margin = d.margin;
      if (MODE == kHot && a.V != a.H) margin = fmin(margin, fabs(u[1] - alpha));
      if (margin < kBoundaryEps) fl |= DP_FLAG_NEAR_BOUNDARY;
      if (MODE == kTail) fl |= a.flags[row] & DP_FLAG_NEAR_BOUNDARY;
      a.flags[row] = fl;
      if (a.dbg.margin) a.dbg.margin[row] = MODE == kTail ? fmin(margin, a.dbg.margin[row]) : margin;
      if (a.dbg.kept) a.dbg.kept[row] = d.kept;
      if (MODE == kHot && a.dbg.alpha) a.dbg.alpha[row] = alpha;
      if (a.dbg.bytes_touched)
        a.dbg.bytes_touched[row] = (MODE == kTail ? a.dbg.bytes_touched[row] : 0ull) + (uint64_t)n * sizeof(T);
    }
    if (a.dbg.topk_ids) {
      const int32_t m = min(k, a.dbg.topk_stride);
      for (int32_t j = lane; j < m; j += 32) {
        a.dbg.topk_ids[(int64_t)row * a.dbg.topk_stride + j] = pos_to_id(a, (int64_t)fpos[j] + lo);
        if (a.dbg.topk_ready) a.dbg.topk_ready[(int64_t)row * a.dbg.topk_stride + j] = fr[j];
      }
    }
  }
  if (split > 1) cluster_wait();
}

// ---------------------------------------------------------------------------
// host launcher

template <typename T, int MODE>
static cudaError_t launch_topk_t(const SampleArgs& a0, int grid_rows, cudaStream_t st) {
  constexpr int NT = 256, U = 8;
  SampleArgs a = a0;
  const int64_t n = MODE == kFull ? a.V : (MODE == kHot ? a.H : a.V - a.H);
  const int bm_words = MODE == kHot ? (int)((n + 31) / 32) : 0;
  const TopkLayout L = topk_layout<NT>(a.wcap, a.kcap, a.lcap, bm_words, a.split);
  auto kern = topk_sample_kernel<T, MODE, NT, U>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  if (a.split > 1) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
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

cudaError_t launch_topk(const SampleArgs& a, int dtype, int mode, int grid_rows, cudaStream_t st) {
  if (dtype == DP_F32) {
    if (mode == kFull) return launch_topk_t<float, kFull>(a, grid_rows, st);
    if (mode == kHot) return launch_topk_t<float, kHot>(a, grid_rows, st);
    return launch_topk_t<float, kTail>(a, grid_rows, st);
  }
  if (mode == kFull) return launch_topk_t<__nv_bfloat16, kFull>(a, grid_rows, st);
  if (mode == kHot) return launch_topk_t<__nv_bfloat16, kHot>(a, grid_rows, st);
  return launch_topk_t<__nv_bfloat16, kTail>(a, grid_rows, st);
}

size_t topk_smem_bytes(const SampleArgs& a, int mode) {
  const int64_t n = mode == kFull ? a.V : (mode == kHot ? a.H : a.V - a.H);
  const int bm_words = mode == kHot ? (int)((n + 31) / 32) : 0;
  return topk_layout<256>(a.wcap, a.kcap, a.lcap, bm_words, a.split).total;
}

}  // namespace dp
