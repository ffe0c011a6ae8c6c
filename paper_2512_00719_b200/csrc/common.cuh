// common.cuh — shared device helpers for the sm_100a decision-plane kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "decplane_b200.h"

#define DP_DEV __device__ __forceinline__

namespace dp {

constexpr int kWarp = 32;

DP_DEV int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
DP_DEV int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
constexpr double kBoundaryEps = 1e-6;   // north-star tolerance on CDF / accept boundaries

// ---------------------------------------------------------------------------
// counter RNG — SplitMix64 chain of rng.py:39-57 (bit-exact: u64 integer ops)
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMultA = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMultB = 0x94D049BB133111EBull;
constexpr uint64_t kDomainSampler = 0;
constexpr uint64_t kDomainLogits = 1;

DP_DEV uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * kMultA;
  z = (z ^ (z >> 27)) * kMultB;
  return z ^ (z >> 31);
}
// absorption up to the iteration field (rng.py:80-83)
DP_DEV uint64_t hash_prefix(uint64_t seed, uint64_t domain, uint64_t iteration) {
  uint64_t h = mix64(seed ^ kGolden);
  h = mix64(h ^ domain);
  return mix64(h ^ iteration);
}
DP_DEV double unit53(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }
DP_DEV void row_uniforms(uint64_t seed, uint64_t iteration, uint64_t seq, double u[3]) {
  uint64_t h = mix64(hash_prefix(seed, kDomainSampler, iteration) ^ seq);
#pragma unroll
  for (int i = 0; i < 3; ++i) u[i] = unit53(mix64(h ^ (uint64_t)i));
}

// ---------------------------------------------------------------------------
// order-preserving keys.  -0.0 and +0.0 compare equal in the f64 oracle, so
// both map to the +0 key; NaN is not a supported logit value.
DP_DEV uint32_t f32_key(float x) {
  uint32_t b = __float_as_uint(x);
  if ((b << 1) == 0u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
DP_DEV float key_f32(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(b);
}
DP_DEV uint64_t f64_key(double x) {
  uint64_t b = (uint64_t)__double_as_longlong(x);
  if ((b << 1) == 0ull) b = 0ull;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
// composite selection key: value desc, position asc, unique per element
DP_DEV uint64_t comp_key(float x, uint32_t pos) {
  return ((uint64_t)f32_key(x) << 32) | (uint64_t)(0xFFFFFFFFu - pos);
}
DP_DEV uint32_t comp_pos(uint64_t k) { return 0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull); }
DP_DEV float comp_val(uint64_t k) { return key_f32((uint32_t)(k >> 32)); }

// ---------------------------------------------------------------------------
// element access
template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int kPerVec = 4;   // 16-byte vector
  DP_DEV static float get(const float* p, int64_t i) { return __ldg(p + i); }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kPerVec = 8;
  DP_DEV static float get(const __nv_bfloat16* p, int64_t i) {
    unsigned short s = __ldg(reinterpret_cast<const unsigned short*>(p) + i);
    return __uint_as_float(((uint32_t)s) << 16);
  }
};

DP_DEV float to_f32(float x) { return x; }
DP_DEV float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
DP_DEV uint4 neg_inf_vec() {
  return sizeof(T) == 4 ? make_uint4(0xFF800000u, 0xFF800000u, 0xFF800000u, 0xFF800000u)
                        : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
}

// 16-byte streaming load (read-once data: no L1 allocation)
DP_DEV uint4 ld_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// L2 bulk prefetch (TMA engine, no registers, no completion to wait for):
// pulls a future chunk of the row into L2 so its loads hit there
DP_DEV void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
template <typename T> DP_DEV float vec_elem(const uint4& v, int e);
template <> DP_DEV float vec_elem<float>(const uint4& v, int e) {
  uint32_t w = e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
  return __uint_as_float(w);
}
template <> DP_DEV float vec_elem<__nv_bfloat16>(const uint4& v, int e) {
  uint32_t w = (e >> 1) == 0 ? v.x : (e >> 1) == 1 ? v.y : (e >> 1) == 2 ? v.z : v.w;
  return __uint_as_float((e & 1) ? (w & 0xFFFF0000u) : (w << 16));
}

// ---------------------------------------------------------------------------
// penalties — penalty.py:35-78 + service.py:236-241, IEEE f64 op by op with
// no FMA contraction so penalized values are bit-identical to numpy.
DP_DEV bool penalties_neutral(const dp_params_t& p) {
  return p.rep_penalty == 1.0 && p.presence_penalty == 0.0 && p.frequency_penalty == 0.0;
}
DP_DEV double ready_penalized(float x, int32_t out_count, const dp_params_t& p) {
  double z = (double)x;
  if (p.rep_penalty != 1.0) z = __ddiv_rn(z, p.rep_penalty);
  if ((p.presence_penalty != 0.0 || p.frequency_penalty != 0.0) && out_count > 0) {
    z = __dsub_rn(z, p.presence_penalty);
    z = __dsub_rn(z, __dmul_rn(p.frequency_penalty, (double)out_count));
  }
  if (p.temperature != 1.0) z = __ddiv_rn(z, p.temperature);
  return z;
}
DP_DEV double ready_plain(float x, const dp_params_t& p) {
  double z = (double)x;
  if (p.temperature != 1.0) z = __ddiv_rn(z, p.temperature);
  return z;
}

// 2^x on the SFU (ex2.approx.ftz: relative error ~2^-22).  Used only for the
// hot-mass accumulation, whose arguments are pre-centred on the row maximum.
DP_DEV float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Online (max, Σ exp) of raw values scaled by 1/tau, folded one small group
// of elements at a time (a 16-byte vector or a few strided elements): one max
// per group, the running sum rescaled (f64 exp2) only when the group raises
// the maximum — rare after the first groups — and the group's terms
// 2^((x - m) * log2e / tau) on the SFU, summed pairwise in f32 and added to
// the f64 total once per group.  -inf entries (excluded / empty) contribute 0.
struct ExpSum {
  float m = -INFINITY;   // raw maximum seen so far
  double s = 0.0;        // Σ 2^((x - m) s2)
  template <int N>
  DP_DEV void add(const float (&x)[N], float s2) {
    float vm = x[0];
#pragma unroll
    for (int i = 1; i < N; ++i) vm = fmaxf(vm, x[i]);
    if (vm > m) {
      s = m == -INFINITY ? 0.0 : s * exp2((double)(m - vm) * (double)s2);
      m = vm;
    }
    if (m == -INFINITY) return;
    float e[N];
#pragma unroll
    for (int i = 0; i < N; ++i) e[i] = ex2_fast((x[i] - m) * s2);
#pragma unroll
    for (int st = 1; st < N; st <<= 1)
#pragma unroll
      for (int i = 0; i + st < N; i += 2 * st) e[i] += e[i + st];
    s += (double)e[0];
  }
  // this state's sum relative to another maximum M >= m (f64)
  DP_DEV double rel(float M, float s2) const {
    return m == -INFINITY ? 0.0 : s * exp2((double)(m - M) * (double)s2);
  }
};

// ---------------------------------------------------------------------------
// warp helpers
DP_DEV uint32_t lane_id() { return threadIdx.x & 31u; }
DP_DEV uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
template <typename T> DP_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T> DP_DEV T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { T w = __shfl_xor_sync(0xffffffffu, v, o); v = w > v ? w : v; }
  return v;
}
// inclusive prefix sum across the warp
template <typename T> DP_DEV T warp_incl_scan(T v) {
  const int l = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T w = __shfl_up_sync(0xffffffffu, v, o);
    if (l >= o) v += w;
  }
  return v;
}

// cluster helpers (sm_90+ ISA, used on sm_100a)
DP_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
DP_DEV void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
DP_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
DP_DEV void cluster_sync() { cluster_arrive(); cluster_wait(); }
// map a local shared address to the same offset in CTA `rank` of the cluster
DP_DEV uint32_t dsmem_addr(const void* local, uint32_t rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(local), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
DP_DEV uint64_t ld_dsmem_u64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
DP_DEV uint32_t ld_dsmem_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
DP_DEV void st_dsmem_u64(uint32_t addr, uint64_t v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
DP_DEV void st_dsmem_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
DP_DEV void st_dsmem_f32(uint32_t addr, float v) { st_dsmem_u32(addr, __float_as_uint(v)); }
DP_DEV void st_dsmem_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

// mbarrier helpers (local CTA barrier, remote arrive from cluster peers)
DP_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(count) : "memory");
}
DP_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// arrive on the barrier at a shared::cluster address (release at cluster scope)
DP_DEV void mbar_remote_arrive(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
DP_DEV void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done) : "r"(a), "r"(parity), "r"(1000000u) : "memory");
  }
}

DP_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
DP_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
DP_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  // suspend in hardware until the phase completes (or the hint expires)
  // instead of re-polling: spinning warps would steal issue slots from the
  // warps doing real work on the same SM sub-partition
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done) : "r"(a), "r"(parity), "r"(1000000u) : "memory");
  }
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0)
DP_DEV void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)), "l"(policy)
      : "memory");
}
DP_DEV uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
DP_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
DP_DEV uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}

// descending bitonic sort of one u32 key per lane across a warp
DP_DEV uint32_t warp_sort_desc(uint32_t k) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, k, stride);
      const bool lower = (lane & stride) == 0;
      const bool desc = (lane & size) == 0 || size == 32;
      const uint32_t hi = k > o ? k : o, lo = k > o ? o : k;
      k = (lower == desc) ? hi : lo;
    }
  }
  return k;
}

}  // namespace dp
