// capi.cu — the extern "C" boundary (include/decplane_b200.h).  Argument
// validation, launch planning and error mapping live here; kernels live in
// sample_topk.cu / sample_general.cu / aux_kernels.cu.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sampler.cuh"

namespace dp {
cudaError_t launch_topk(const SampleArgs& a, int dtype, int mode, int grid_rows, cudaStream_t st);
cudaError_t launch_general(const SampleArgs& a, int dtype, int mode, int grid_rows, cudaStream_t st);
size_t topk_smem_bytes(const SampleArgs& a, int mode);
cudaError_t launch_resum(const SampleArgs& a, int dtype, cudaStream_t st);
cudaError_t launch_warp(const SampleArgs& a, int dtype, int mode, int grid_rows, cudaStream_t st);
int persist_grid(const SampleArgs& a, int dtype);
size_t persist_smem_bytes(const SampleArgs& a);
cudaError_t launch_persist(const SampleArgs& a, int dtype, int grid, cudaStream_t st);
cudaError_t launch_hot_sort(const SampleArgs& a, int dtype, cudaStream_t st);
cudaError_t launch_row_summary(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                               const dp_params_t* params, const dp_penalty_t& pen, const int32_t* inv_perm,
                               double* row_max, double* total, cudaStream_t st);
cudaError_t launch_hot_mass_curve(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                                  const double* row_max, const double* total, const dp_params_t* params,
                                  const dp_penalty_t& pen, const int32_t* inv_perm, const int32_t* col_of_pos,
                                  const int32_t* grid, int32_t n_grid, double* out, cudaStream_t st);
}  // namespace dp

cudaError_t dp_launch_uniforms(const dp_params_t*, const uint64_t*, int64_t, uint64_t, double*, cudaStream_t);
cudaError_t dp_launch_penalty_update(const dp_penalty_t&, const int32_t*, int64_t, uint8_t*, cudaStream_t);
cudaError_t dp_launch_penalty_reset(const dp_penalty_t&, int64_t, cudaStream_t);
cudaError_t dp_launch_ready_rows(const void*, int, int64_t, int64_t, int64_t, const dp_params_t*,
                                 const dp_penalty_t&, double*, cudaStream_t);
cudaError_t dp_launch_encode(const int32_t*, const double*, const uint8_t*, const uint64_t*, int64_t, uint8_t*,
                             cudaStream_t);
cudaError_t dp_launch_synth(const double*, double, uint64_t, uint64_t, const uint64_t*, int64_t, int64_t,
                            int64_t, const int32_t*, int, void*, const dp_params_t*, double*, double*,
                            cudaStream_t);

// the ctypes mirrors (_native.py) and every caller rely on these layouts
static_assert(sizeof(dp_params_t) == 64, "dp_params_t layout");
static_assert(sizeof(dp_penalty_t) == 48, "dp_penalty_t layout");
static_assert(sizeof(dp_plan_t) == 48, "dp_plan_t layout");

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, const char* detail = nullptr) {
  std::snprintf(g_err, sizeof(g_err), fmt, detail ? detail : "");
  return code;
}
int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return DP_OK;
  std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return DP_ERR_CUDA;
}
int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}
uint32_t pow2_at_least(uint32_t v) {
  uint32_t p = 1;
  while (p < v) p <<= 1;
  return p;
}
// some row may have top-k off (the plan's lower bound does not exclude it)
bool nucleus_possible(const dp_plan_t* plan) { return !(plan && plan->min_top_k > 0); }
// Caller-owned workspace (dp_plan_t.workspace, dp_workspace_len(B) int32
// elements): three fallback row lists [count, rows...] of B + 1 entries
// (slot 0: full path, 1: SHVS hot pass, 2: SHVS tail pass), the re-sum list
// (slot 3) and B f64 hot masses (8-byte aligned).  Without a workspace
// nucleus rows go straight to the general kernel (route_row).
int64_t workspace_len(int64_t B) { return 4 * (B + 1) + 2 * B + 2; }
int32_t* fallback_list(const dp_plan_t* plan, int slot, int64_t B) {
  if (!plan || !plan->workspace || plan->workspace_len < workspace_len(B)) return nullptr;
  return plan->workspace + slot * (B + 1);
}
double* resum_mass(const dp_plan_t* plan, int64_t B) {
  int32_t* p = plan->workspace + 4 * (B + 1);
  if ((reinterpret_cast<uintptr_t>(p) & 7u) != 0) ++p;
  return reinterpret_cast<double*>(p);
}
// arm the fallback list of a call (nucleus rows routed to the top-k kernel);
// false: no workspace, nucleus rows take the general kernel directly
bool arm_fallback(dp::SampleArgs& a, const dp_plan_t* plan, int slot, int64_t B, cudaStream_t st, cudaError_t& e) {
  int32_t* fb = fallback_list(plan, slot, B);
  e = cudaSuccess;
  if (!fb) return false;
  a.fb_count = fb;
  a.fb_rows = fb + 1;
  e = cudaMemsetAsync(fb, 0, sizeof(int32_t), st);
  return true;
}
// the general kernel over the fallback list (after the top-k kernel)
cudaError_t launch_fallback(const dp::SampleArgs& a, int dtype, int mode, int64_t B, cudaStream_t st) {
  dp::SampleArgs g = a;
  g.rows = a.fb_rows;
  g.row_count = a.fb_count;
  g.fb_rows = nullptr;
  g.fb_count = nullptr;
  g.force_general = 1;
  return dp::launch_general(g, dtype, mode, (int)B, st);
}

// Which kernels a call launches.  Every row is routed to exactly one kernel by
// route_row (sampler.cuh); a kernel is skipped only when the plan's top-k
// bounds (promises, see dp_plan_t) prove no row routes to it.
struct Launches {
  bool warp, topk, general;
};
Launches plan_launches(dp::SampleArgs& a, const dp_plan_t* plan, int mode, int64_t B, int64_t n) {
  Launches L;
  const int kernel = plan ? plan->kernel : 0;
  const int64_t kmax = plan ? plan->max_top_k : 0, kmin = plan ? plan->min_top_k : 0;
  // kHot with K1h taking the nucleus rows: the top-k rows are bounded by kmax alone
  const bool nuc_elsewhere = a.use_hot_sort == 1 && mode == dp::kHot;
  const bool bounded = kmax > 0 && (kmin > 0 || nuc_elsewhere) && kmax < n;
  const int64_t cap = dp::pen_bound(a.pen);
  a.use_warp = 0;
  if (mode != dp::kTail && kernel != 1) {
    const bool auto_warp = mode == dp::kHot && B >= sm_count() && n <= 65536;
    a.use_warp = (kernel == 2 || auto_warp) ? 1 : 0;
  }
  // every row with top-k on fits the warp kernel / the top-k kernel
  const bool all_warp = a.use_warp && bounded && kmax <= dp::kWarpKMax && cap <= dp::kWarpPenCap &&
                        (kmax + cap <= dp::kWarpKpMax || n <= dp::kWarpKpMax);
  // penalized ids outside the stream (kHot, long lists): kp = k, and the
  // final stage keeps at most kPenSelCap penalized entries
  const bool excl = mode == dp::kHot || a.pen_excl;
  const int64_t pl = (excl && cap > dp::kPenSelCap) ? dp::kPenSelCap : cap;
  const int64_t kp_topk = kmax + (excl ? 0 : cap);
  const bool k_rows_fit = kmax > 0 && kmax < n && (kp_topk < n ? kp_topk : n) <= a.kcap && kmax + 2 * pl <= a.lcap;
  const bool all_topk = bounded && k_rows_fit;
  // top-k-off rows present (kmin == 0): they are nucleus rows of the top-k
  // kernel (the general kernel then only sees the fallback list) when the
  // nucleus list fits; rows with top-k on fit by k_rows_fit
  const int64_t kp_nuc = dp::kNucK + (excl ? 0 : cap);
  const bool nuc_all = a.fb_rows != nullptr && n >= 2 * (int64_t)dp::kNucK && kp_nuc <= a.kcap &&
                       dp::kNucK + 2 * pl <= a.lcap;
  const bool mixed_topk = kmin == 0 && k_rows_fit && nuc_all;
  L.warp = a.use_warp != 0;
  L.topk = !all_warp;
  L.general = !(all_warp || all_topk || mixed_topk);
  return L;
}

// Shrink the top-k kernel's capacities until its shared memory fits one CTA
// (final-list capacity first, then the admission buffer, then the selection).
// Rows whose k + |list| no longer fit route to the general kernel (route_row).
void fit_topk(dp::SampleArgs& a, int mode) {
  int dev = 0, optin = 232448;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  while (dp::topk_smem_bytes(a, mode) > (size_t)optin) {
    if (a.lcap > 256) a.lcap >>= 1;
    else if (a.wcap > 1024) a.wcap >>= 1;
    else if (a.kcap > 256) a.kcap >>= 1;
    else break;
  }
}

bool valid_pen(const dp_penalty_t* pen, int64_t V) {
  return pen && pen->ids && pen->out_count && pen->len && pen->cap >= 0 && pen->vocab_size == V;
}

// resident CTAs of K1p for the call's shared-memory footprint (occupancy query
// cached per (device, dtype, bytes): it runs once per shape, not per call)
int persist_grid_cached(const dp::SampleArgs& a, int dtype) {
  static thread_local int c_dev = -1, c_dtype = -1, c_grid = 0;
  static thread_local size_t c_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t smem = dp::persist_smem_bytes(a);
  if (dev != c_dev || dtype != c_dtype || smem != c_smem) {
    c_grid = dp::persist_grid(a, dtype);
    c_dev = dev;
    c_dtype = dtype;
    c_smem = smem;
  }
  return c_grid;
}

// capacities for the streaming top-k kernel (see sample_topk.cu)
void plan_topk(dp::SampleArgs& a, const dp_plan_t* plan, int64_t B, int64_t n, int elem_bytes, int mode) {
  int32_t kmax = (plan && plan->max_top_k > 0) ? plan->max_top_k : 256;
  if (nucleus_possible(plan) && kmax < dp::kNucK) kmax = dp::kNucK;   // nucleus rows keep kNucK
  // long penalty lists: the streaming selection excludes the penalized ids
  // (shared bitmap) instead of widening to k + |list|, and the final stage
  // keeps only the best kPenSelCap penalized entries (finish.cuh)
  const int32_t pb = dp::pen_bound(a.pen);
  a.pen_excl = (mode != dp::kHot && a.nshard == 0 && pb > dp::kPenExclMin) ? 1 : 0;
  const bool excl = mode == dp::kHot || a.pen_excl;
  const int32_t pl = (excl && pb > dp::kPenSelCap) ? dp::kPenSelCap : pb;
  const uint32_t kcap = pow2_at_least((uint32_t)kmax + (uint32_t)(a.pen_excl ? 0 : pb));
  a.kcap = (int32_t)(kcap < 32u ? 32u : kcap);
  if (a.kcap > 2048) a.kcap = 2048;
  // vector slots of the streaming stage's candidate buffer (wcap field): the
  // estimated threshold admits ~2-3 kp elements per segment; overflow is
  // handled exactly (re-stream), so this only sizes the common case
  a.wcap = (int32_t)(4u * (uint32_t)a.kcap > 1024u ? 4u * (uint32_t)a.kcap : 1024u);
  if (a.wcap > 4096) a.wcap = 4096;
  a.lcap = (int32_t)pow2_at_least((uint32_t)kmax + 2u * (uint32_t)pl + 1u);
  if (a.lcap > 4096) a.lcap = 4096;
  int split = plan && plan->split > 0 ? plan->split : 0;
  if (split == 0) {
    // one CTA per row once the batch fills the GPU (measured fastest at
    // V=152k, B=1024); small batches split rows over a cluster so every SM
    // streams, keeping >= 16K elements per CTA
    const int64_t sms = sm_count();
    split = B >= sms ? 1 : (int)((2 * sms + B - 1) / B);
    const int64_t by_len = n / 16384;
    if (split > by_len) split = (int)by_len;
    if (split < 1) split = 1;
  }
  if (split > 8) split = 8;
  a.split = split;
  // threads per CTA: 256 by default; plan->reserved[0] may request 128
  a.nt = (plan && plan->threads == 128) ? 128 : 256;
  a.summary_raw = (plan && plan->summary_raw) ? 1 : 0;
  a.update_pen = (plan && plan->fuse_update) ? 1 : 0;
  (void)elem_bytes;
}

}  // namespace

namespace dp {
// other translation units (collective.cu) report through dp_last_error
int set_last_error(int code, const char* msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}
}  // namespace dp

extern "C" {

int dp_version(void) { return 100; }

const char* dp_last_error(void) { return g_err; }

int64_t dp_workspace_len(int64_t B) { return B < 0 ? 0 : workspace_len(B); }

int dp_device_check(int device) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDeviceProperties");
  if (prop.major != 10) {
    std::snprintf(g_err, sizeof(g_err), "device %d is sm_%d%d; this build targets sm_100a", device, prop.major,
                  prop.minor);
    return DP_ERR_UNSUPPORTED;
  }
  return DP_OK;
}

int dp_uniforms(const dp_params_t* params, const uint64_t* seq_ids, int64_t B, uint64_t iteration, double* out,
                void* stream) {
  if (!params || !seq_ids || !out || B < 0) return fail(DP_ERR_ARG, "dp_uniforms: null argument%s");
  if (B == 0) return DP_OK;
  return cuda_status(dp_launch_uniforms(params, seq_ids, B, iteration, out, (cudaStream_t)stream), "dp_uniforms");
}

int dp_sample_full(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld, const dp_params_t* params,
                   const dp_penalty_t* pen_host, const double* uniforms, const uint64_t* seq_ids,
                   uint64_t iteration, int32_t* token, double* logprob, uint8_t* flags,
                   const dp_debug_t* debug_host, const dp_plan_t* plan_host, void* stream) {
  if (!logits || !params || !token || !logprob || !flags) return fail(DP_ERR_ARG, "dp_sample_full: null argument%s");
  if (!uniforms && !seq_ids) return fail(DP_ERR_ARG, "dp_sample_full: need uniforms or seq_ids%s");
  if (dtype != DP_F32 && dtype != DP_BF16) return fail(DP_ERR_UNSUPPORTED, "dp_sample_full: dtype%s");
  if (B < 0 || V < 1 || ld < V || V >= (1ll << 31)) return fail(DP_ERR_ARG, "dp_sample_full: bad shape%s");
  if (!valid_pen(pen_host, V)) return fail(DP_ERR_ARG, "dp_sample_full: penalty state does not match V%s");
  if (B == 0) return DP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dp::SampleArgs a;
  std::memset(&a, 0, sizeof(a));
  a.logits = logits;
  a.ld = ld;
  a.V = V;
  a.H = V;
  a.params = params;
  a.pen = *pen_host;
  a.uniforms = uniforms;
  a.seq_ids = seq_ids;
  a.iteration = iteration;
  a.n_rows = (int32_t)B;
  a.token = token;
  a.logprob = logprob;
  a.flags = flags;
  if (debug_host) a.dbg = *debug_host;
  plan_topk(a, plan_host, B, V, dtype == DP_F32 ? 4 : 2, dp::kFull);
  fit_topk(a, dp::kFull);
  cudaError_t e = cudaSuccess;
  const bool nuc = nucleus_possible(plan_host) && arm_fallback(a, plan_host, 0, B, st, e);
  if (e != cudaSuccess) return cuda_status(e, "dp_sample_full/fallback");
  const Launches L = plan_launches(a, plan_host, dp::kFull, B, V);
  if (L.warp && (e = dp::launch_warp(a, dtype, dp::kFull, (int)B, st)) != cudaSuccess)
    return cuda_status(e, "dp_sample_full/warp");
  if (L.topk) {
    // several waves of rows with top-k only: the persistent warp-specialised
    // K1p overlaps each row's final stage with the next row's stream
    const bool no_persist = plan_host && (plan_host->flags & DP_PLAN_NO_PERSIST);
    const int pg = (!no_persist && a.split == 1 && a.fb_rows == nullptr && !a.use_warp && !a.pen_excl)
                       ? persist_grid_cached(a, dtype)
                                                                                         : 0;
    if (std::getenv("DP_VERBOSE"))
      std::fprintf(stderr, "[dp] full: B=%lld persist_grid=%d smem=%zu topk_smem=%zu kcap=%d wcap=%d lcap=%d\n",
                   (long long)B, pg, dp::persist_smem_bytes(a), dp::topk_smem_bytes(a, dp::kFull), a.kcap, a.wcap,
                   a.lcap);
    // K1p pays off when the batch is one to two waves (C2: 1,024 rows on 592
    // CTAs: the second wave's stream hides the first wave's final stages);
    // with many waves (C4) K1's rows already interleave and its 8 streaming
    // warps win (profiles/r2/k1p_ab.txt)
    const bool force = plan_host && (plan_host->flags & DP_PLAN_FORCE_PERSIST);
#ifdef DP_PERSIST_BALANCE   // A-B: every CTA takes the same number of rows (ceil(B / waves))
    int pgrid = pg;
    if (pg > 0) {
      const int64_t waves = (B + pg - 1) / pg;
      pgrid = (int)((B + waves - 1) / waves);
    }
#else
    const int pgrid = pg;
#endif
    if (pg > 0 && ((B > pg && B <= 2 * (int64_t)pg) || force)) e = dp::launch_persist(a, dtype, pgrid, st);
    else e = dp::launch_topk(a, dtype, dp::kFull, (int)B, st);
    if (e != cudaSuccess) return cuda_status(e, "dp_sample_full/topk");
  }
  if (L.general && (e = dp::launch_general(a, dtype, dp::kFull, (int)B, st)) != cudaSuccess)
    return cuda_status(e, "dp_sample_full/general");
  if (nuc && (e = launch_fallback(a, dtype, dp::kFull, B, st)) != cudaSuccess)
    return cuda_status(e, "dp_sample_full/fallback");
  return DP_OK;
}

int dp_sample_full_sharded(const void* const* shards, int32_t t, int dtype, int64_t B, int64_t V, int64_t ld,
                           const dp_params_t* params, const dp_penalty_t* pen_host, const double* uniforms,
                           const uint64_t* seq_ids, uint64_t iteration, int32_t* token, double* logprob,
                           uint8_t* flags, const dp_debug_t* debug_host, const dp_plan_t* plan_host, void* stream) {
  if (!shards || !params || !token || !logprob || !flags)
    return fail(DP_ERR_ARG, "dp_sample_full_sharded: null argument%s");
  if (!uniforms && !seq_ids) return fail(DP_ERR_ARG, "dp_sample_full_sharded: need uniforms or seq_ids%s");
  if (dtype != DP_F32 && dtype != DP_BF16) return fail(DP_ERR_UNSUPPORTED, "dp_sample_full_sharded: dtype%s");
  if (t < 1 || t > dp::kMaxShards) return fail(DP_ERR_ARG, "dp_sample_full_sharded: shard count outside [1, 8]%s");
  // equal-width tiling from 0 (AssembledLogitsView.__post_init__, transport.py:474-489)
  if (B < 0 || V < 1 || V % t != 0 || ld < V / t || V >= (1ll << 31))
    return fail(DP_ERR_ARG, "dp_sample_full_sharded: shards do not tile [0, V) with equal widths%s");
  for (int32_t s = 0; s < t; ++s)
    if (!shards[s]) return fail(DP_ERR_ARG, "dp_sample_full_sharded: null shard%s");
  if (!valid_pen(pen_host, V)) return fail(DP_ERR_ARG, "dp_sample_full_sharded: penalty state does not match V%s");
  if (B == 0) return DP_OK;
  dp::SampleArgs a;
  std::memset(&a, 0, sizeof(a));
  a.logits = shards[0];
  a.ld = ld;
  a.V = V;
  a.H = V;
  a.params = params;
  a.pen = *pen_host;
  a.uniforms = uniforms;
  a.seq_ids = seq_ids;
  a.iteration = iteration;
  a.n_rows = (int32_t)B;
  a.token = token;
  a.logprob = logprob;
  a.flags = flags;
  if (debug_host) a.dbg = *debug_host;
  a.nshard = t;   // (plan_topk: sharded rows keep the k + |list| selection)
  plan_topk(a, plan_host, B, V, dtype == DP_F32 ? 4 : 2, dp::kFull);
  // one t-CTA cluster per row while the batch leaves SMs idle; otherwise the
  // fewest CTAs per row (a cluster rank's select + push is the per-CTA
  // overhead).  A CTA keeps <= 2 (EPV - 1) scalar head / tail keys per shard
  // in 64 slots: <= 8 fp32 shards, <= 4 bf16 shards
  const int32_t max_spc = dtype == DP_F32 ? 8 : 4;
  int32_t c = t;
  if (B >= (int64_t)sm_count()) {
    c = 1;
    while (t / c > max_spc || t % c != 0) ++c;
  }
  a.split = c;   // cluster rank r streams shards [r t/c, (r+1) t/c) in place
  fit_topk(a, dp::kFull);
  a.shard_per_cta = t / c;
  a.nshard = t;
  a.shard_n = V / t;
  for (int32_t s = 0; s < t; ++s) a.shard[s] = shards[s];
  // zero-copy only through the top-k kernel: every row must carry top-k
  // within the plan's bounds (the other kernels read contiguous rows)
  const Launches L = plan_launches(a, plan_host, dp::kFull, B, V);
  if (L.warp || L.general || !L.topk)
    return fail(DP_ERR_UNSUPPORTED,
                "dp_sample_full_sharded: needs plan min_top_k > 0 and max_top_k within the top-k kernel's "
                "capacity (stitch the shards and call dp_sample_full otherwise)%s");
  return cuda_status(dp::launch_topk(a, dtype, dp::kFull, (int)B, (cudaStream_t)stream), "dp_sample_full_sharded");
}

int dp_row_summary(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld, const dp_params_t* params,
                   const dp_penalty_t* pen_host, const int32_t* inv_perm, double* row_max, double* total_expsum,
                   void* stream) {
  if (!logits || !params || !row_max || !total_expsum) return fail(DP_ERR_ARG, "dp_row_summary: null argument%s");
  if (dtype != DP_F32 && dtype != DP_BF16) return fail(DP_ERR_UNSUPPORTED, "dp_row_summary: dtype%s");
  if (B < 0 || V < 1 || ld < V) return fail(DP_ERR_ARG, "dp_row_summary: bad shape%s");
  if (!valid_pen(pen_host, V)) return fail(DP_ERR_ARG, "dp_row_summary: penalty state does not match V%s");
  if (B == 0) return DP_OK;
  return cuda_status(dp::launch_row_summary(logits, dtype, B, V, ld, params, *pen_host, inv_perm, row_max,
                                            total_expsum, (cudaStream_t)stream),
                     "dp_row_summary");
}

int dp_row_summary_raw(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld, const dp_params_t* params,
                       double* row_max, double* total_expsum, void* stream) {
  if (!logits || !params || !row_max || !total_expsum) return fail(DP_ERR_ARG, "dp_row_summary_raw: null argument%s");
  if (dtype != DP_F32 && dtype != DP_BF16) return fail(DP_ERR_UNSUPPORTED, "dp_row_summary_raw: dtype%s");
  if (B < 0 || V < 1 || ld < V) return fail(DP_ERR_ARG, "dp_row_summary_raw: bad shape%s");
  if (B == 0) return DP_OK;
  dp_penalty_t none;
  std::memset(&none, 0, sizeof(none));
  none.vocab_size = (int32_t)V;
  return cuda_status(dp::launch_row_summary(logits, dtype, B, V, ld, params, none, nullptr, row_max, total_expsum,
                                            (cudaStream_t)stream),
                     "dp_row_summary_raw");
}

}  // extern "C"

namespace {
// device-accessible address of a buffer that may be (mapped) pinned host memory
const void* device_view(const void* p) {
  cudaPointerAttributes at;
  if (p && cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost) {
    void* d = nullptr;
    if (cudaHostGetDevicePointer(&d, const_cast<void*>(p), 0) == cudaSuccess) return d;
    return at.devicePointer ? at.devicePointer : p;
  }
  cudaGetLastError();   // unregistered pageable pointers report an error: clear it
  return p;
}

int sample_shvs_impl(const void* logits, int dtype, int64_t B, int64_t V, int64_t H, int64_t ld,
                     const void* tail_logits, int64_t tail_ld, const int32_t* perm, const int32_t* inv_perm,
                     const double* row_max, const double* total_expsum, const dp_params_t* params,
                     const dp_penalty_t* pen_host, const double* uniforms, const uint64_t* seq_ids,
                     uint64_t iteration, int32_t* token, double* logprob, uint8_t* flags,
                     const dp_debug_t* debug_host, const dp_plan_t* plan_host, int32_t* scratch_rows, void* stream) {
  if (!logits || !params || !token || !logprob || !flags || !row_max || !total_expsum || !scratch_rows)
    return fail(DP_ERR_ARG, "dp_sample_shvs: null argument%s");
  if (!uniforms && !seq_ids) return fail(DP_ERR_ARG, "dp_sample_shvs: need uniforms or seq_ids%s");
  if (dtype != DP_F32 && dtype != DP_BF16) return fail(DP_ERR_UNSUPPORTED, "dp_sample_shvs: dtype%s");
  if (B < 0 || V < 1 || H < 1 || H > V || V >= (1ll << 31) || (tail_logits ? (ld < H || tail_ld < V - H) : ld < V))
    return fail(DP_ERR_ARG, "dp_sample_shvs: bad shape (need 1 <= H <= V <= ld, or ld >= H and ld_tail >= V - H)%s");
  if ((perm == nullptr) != (inv_perm == nullptr)) return fail(DP_ERR_ARG, "dp_sample_shvs: perm/inv_perm%s");
  if (!valid_pen(pen_host, V)) return fail(DP_ERR_ARG, "dp_sample_shvs: penalty state does not match V%s");
  if (B == 0) return DP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dp::SampleArgs a;
  std::memset(&a, 0, sizeof(a));
  a.logits = logits;
  a.ld = ld;
  a.V = V;
  a.H = H;
  a.tail_logits = tail_logits ? device_view(tail_logits) : nullptr;
  a.tail_ld = tail_ld;
  a.perm = perm;
  a.inv_perm = inv_perm;
  a.params = params;
  a.pen = *pen_host;
  a.uniforms = uniforms;
  a.seq_ids = seq_ids;
  a.iteration = iteration;
  a.row_max = row_max;
  a.total_expsum = total_expsum;
  a.n_rows = (int32_t)B;
  a.token = token;
  a.logprob = logprob;
  a.flags = flags;
  if (debug_host) a.dbg = *debug_host;
  int32_t* rej_count = scratch_rows;
  int32_t* rej_rows = scratch_rows + 1;
  cudaError_t e = cudaMemsetAsync(rej_count, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return cuda_status(e, "dp_sample_shvs/memset");
  a.reject_rows = rej_rows;
  a.reject_count = rej_count;
  // raw producer summary: undecidable accept tests are re-summed exactly
  const bool resum = plan_host && plan_host->summary_raw && H < V;
  if (resum) {
    int32_t* rl = fallback_list(plan_host, 3, B);
    if (!rl) return fail(DP_ERR_ARG, "dp_sample_shvs: summary_raw needs the plan workspace (dp_workspace_len)%s");
    a.resum_count = rl;
    a.resum_rows = rl + 1;
    a.resum_sh = resum_mass(plan_host, B);
    a.force_resum = (plan_host->flags & DP_PLAN_FORCE_RESUM) ? 1 : 0;
    if ((e = cudaMemsetAsync(rl, 0, sizeof(int32_t), st)) != cudaSuccess) return cuda_status(e, "dp_sample_shvs/memset");
  }
  // hot pass over [0, H): short hot sets by the exact sort (K1h), longer ones
  // by the streaming kernels
  plan_topk(a, plan_host, B, H, dtype == DP_F32 ? 4 : 2, dp::kHot);
  fit_topk(a, dp::kHot);
  const int kern = plan_host ? plan_host->kernel : 0;
  const int pf = plan_host ? plan_host->flags : 0;
  const bool hot_sort = H <= dp::kHotSortMax && kern != 1 && kern != 2 &&
                        (pf & (DP_PLAN_HOT_SORT | DP_PLAN_HOT_SORT_ALL));
  const bool sort_all = hot_sort && (pf & DP_PLAN_HOT_SORT_ALL);
  a.use_hot_sort = sort_all ? 2 : (hot_sort ? 1 : 0);
  // nucleus rows (top-k off) go to K1h when it is on: the streaming kernels
  // then only see top-k rows and need no nucleus list / fallback
  const bool nuc_rows = nucleus_possible(plan_host);
  if (a.use_hot_sort && (nuc_rows || sort_all)) {
    if ((e = dp::launch_hot_sort(a, dtype, st)) != cudaSuccess) return cuda_status(e, "dp_sample_shvs/hot-sort");
  }
  bool nuc = false;
  const bool any_stream_rows = !sort_all && !(a.use_hot_sort && plan_host && plan_host->max_top_k <= 0);
  if (any_stream_rows) {
    if (!a.use_hot_sort) nuc = nuc_rows && arm_fallback(a, plan_host, 1, B, st, e);
    if (e != cudaSuccess) return cuda_status(e, "dp_sample_shvs/fallback");
    const Launches L = plan_launches(a, plan_host, dp::kHot, B, H);
    if (L.warp && (e = dp::launch_warp(a, dtype, dp::kHot, (int)B, st)) != cudaSuccess)
      return cuda_status(e, "dp_sample_shvs/hot-warp");
    if (L.topk && (e = dp::launch_topk(a, dtype, dp::kHot, (int)B, st)) != cudaSuccess)
      return cuda_status(e, "dp_sample_shvs/hot-topk");
    if (L.general && (e = dp::launch_general(a, dtype, dp::kHot, (int)B, st)) != cudaSuccess)
      return cuda_status(e, "dp_sample_shvs/hot-general");
    if (nuc && (e = launch_fallback(a, dtype, dp::kHot, B, st)) != cudaSuccess)
      return cuda_status(e, "dp_sample_shvs/hot-fallback");
  }
  nuc = nucleus_possible(plan_host);   // the tail pass may hold nucleus rows either way
  if (H == V) return DP_OK;
  if (resum && (e = dp::launch_resum(a, dtype, st)) != cudaSuccess) return cuda_status(e, "dp_sample_shvs/resum");
  // tail pass over [H, V) for the rows the hot pass rejected
  dp::SampleArgs t = a;
  t.resum_rows = nullptr;
  t.resum_count = nullptr;
  t.rows = rej_rows;
  t.row_count = rej_count;
  t.reject_rows = nullptr;
  t.reject_count = nullptr;
  if (nuc) {
    arm_fallback(t, plan_host, 2, B, st, e);
    if (e != cudaSuccess) return cuda_status(e, "dp_sample_shvs/fallback");
  }
  plan_topk(t, plan_host, B, V - H, dtype == DP_F32 ? 4 : 2, dp::kTail);
  // The tail pass serves only the rejected rows (typically a few percent of
  // B, count known on the device only): 4-CTA clusters split each row over 4
  // SMs, and the clusters loop over the reject list, so a handful of
  // rejections costs one short row time rather than one long one.
  int64_t tail_clusters = B;
  if (!(plan_host && plan_host->split > 0)) {
    t.split = (V - H) >= 4 * 4096 ? 4 : 1;   // 4 measured best at C2 (2: 71, 4: 63, 8: 65 us per SHVS step)
    const int64_t slots = (int64_t)sm_count() * 2 / t.split;   // resident clusters (2 tail CTAs per SM)
    tail_clusters = B < slots ? B : slots;
  }
  fit_topk(t, dp::kTail);
  const Launches LT = plan_launches(t, plan_host, dp::kTail, B, V - H);
  if (LT.topk && (e = dp::launch_topk(t, dtype, dp::kTail, (int)tail_clusters, st)) != cudaSuccess)
    return cuda_status(e, "dp_sample_shvs/tail-topk");
  if (LT.general && (e = dp::launch_general(t, dtype, dp::kTail, (int)B, st)) != cudaSuccess)
    return cuda_status(e, "dp_sample_shvs/tail-general");
  if (nuc && (e = launch_fallback(t, dtype, dp::kTail, B, st)) != cudaSuccess)
    return cuda_status(e, "dp_sample_shvs/tail-fallback");
  return DP_OK;
}

}  // namespace

extern "C" {

int dp_sample_shvs(const void* logits, int dtype, int64_t B, int64_t V, int64_t H, int64_t ld, const int32_t* perm,
                   const int32_t* inv_perm, const double* row_max, const double* total_expsum,
                   const dp_params_t* params, const dp_penalty_t* pen_host, const double* uniforms,
                   const uint64_t* seq_ids, uint64_t iteration, int32_t* token, double* logprob, uint8_t* flags,
                   const dp_debug_t* debug_host, const dp_plan_t* plan_host, int32_t* scratch_rows,
                   void* stream) {
  return sample_shvs_impl(logits, dtype, B, V, H, ld, nullptr, 0, perm, inv_perm, row_max, total_expsum, params,
                          pen_host, uniforms, seq_ids, iteration, token, logprob, flags, debug_host, plan_host,
                          scratch_rows, stream);
}

int dp_sample_shvs_split(const void* logits_hot, int64_t ld_hot, const void* logits_tail, int64_t ld_tail, int dtype,
                         int64_t B, int64_t V, int64_t H, const int32_t* perm, const int32_t* inv_perm,
                         const double* row_max, const double* total_expsum, const dp_params_t* params,
                         const dp_penalty_t* pen_host, const double* uniforms, const uint64_t* seq_ids,
                         uint64_t iteration, int32_t* token, double* logprob, uint8_t* flags,
                         const dp_debug_t* debug_host, const dp_plan_t* plan_host, int32_t* scratch_rows,
                         void* stream) {
  if (!logits_tail && H < V) return fail(DP_ERR_ARG, "dp_sample_shvs_split: null tail%s");
  return sample_shvs_impl(logits_hot, dtype, B, V, H, ld_hot, logits_tail ? logits_tail : logits_hot,
                          logits_tail ? ld_tail : ld_hot, perm, inv_perm, row_max, total_expsum, params, pen_host,
                          uniforms, seq_ids, iteration, token, logprob, flags, debug_host, plan_host, scratch_rows,
                          stream);
}

int dp_stage_hot(const void* logits_host, int64_t ld_host, int dtype, int64_t B, int64_t H, void* hot_dev,
                 int64_t ld_dev, void* stream) {
  if (!logits_host || !hot_dev) return fail(DP_ERR_ARG, "dp_stage_hot: null argument%s");
  if (dtype != DP_F32 && dtype != DP_BF16) return fail(DP_ERR_UNSUPPORTED, "dp_stage_hot: dtype%s");
  if (B < 0 || H < 1 || ld_host < H || ld_dev < H) return fail(DP_ERR_ARG, "dp_stage_hot: bad shape%s");
  if (B == 0) return DP_OK;
  const size_t esz = dtype == DP_F32 ? 4 : 2;
  return cuda_status(cudaMemcpy2DAsync(hot_dev, (size_t)ld_dev * esz, logits_host, (size_t)ld_host * esz,
                                       (size_t)H * esz, (size_t)B, cudaMemcpyHostToDevice, (cudaStream_t)stream),
                     "dp_stage_hot");
}

int dp_penalty_update(const dp_penalty_t* pen_host, const int32_t* token, int64_t B, uint8_t* flags, void* stream) {
  if (!pen_host || !token || !pen_host->ids || !pen_host->out_count || !pen_host->len)
    return fail(DP_ERR_ARG, "dp_penalty_update: null argument%s");
  if (B == 0) return DP_OK;
  return cuda_status(dp_launch_penalty_update(*pen_host, token, B, flags, (cudaStream_t)stream), "dp_penalty_update");
}

int dp_penalty_reset(const dp_penalty_t* pen_host, int64_t B, void* stream) {
  if (!pen_host || !pen_host->prompt_len || !pen_host->len) return fail(DP_ERR_ARG, "dp_penalty_reset: null%s");
  if (B == 0) return DP_OK;
  return cuda_status(dp_launch_penalty_reset(*pen_host, B, (cudaStream_t)stream), "dp_penalty_reset");
}

int dp_ready_rows(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld, const dp_params_t* params,
                  const dp_penalty_t* pen_host, double* out, void* stream) {
  if (!logits || !params || !out) return fail(DP_ERR_ARG, "dp_ready_rows: null argument%s");
  if (!valid_pen(pen_host, V)) return fail(DP_ERR_ARG, "dp_ready_rows: penalty state does not match V%s");
  if (B == 0) return DP_OK;
  return cuda_status(dp_launch_ready_rows(logits, dtype, B, V, ld, params, *pen_host, out, (cudaStream_t)stream),
                     "dp_ready_rows");
}

int dp_synth_logits(const double* base_by_id, double noise, uint64_t seed, uint64_t iteration,
                    const uint64_t* seq_ids, int64_t B, int64_t V, int64_t ld, const int32_t* perm, int dtype,
                    void* out, const dp_params_t* params, double* row_max, double* total_expsum, void* stream) {
  if (!base_by_id || !seq_ids || !out) return fail(DP_ERR_ARG, "dp_synth_logits: null argument%s");
  if (dtype != DP_F32 && dtype != DP_BF16) return fail(DP_ERR_UNSUPPORTED, "dp_synth_logits: dtype%s");
  if (B < 0 || V < 1 || ld < V) return fail(DP_ERR_ARG, "dp_synth_logits: bad shape%s");
  const bool summ = row_max || total_expsum;
  if (summ && (!row_max || !total_expsum || !params))
    return fail(DP_ERR_ARG, "dp_synth_logits: the summary needs params, row_max and total_expsum%s");
  if (B == 0) return DP_OK;
  return cuda_status(dp_launch_synth(base_by_id, noise, seed, iteration, seq_ids, B, V, ld, perm, dtype, out,
                                     summ ? params : nullptr, summ ? row_max : nullptr,
                                     summ ? total_expsum : nullptr, (cudaStream_t)stream),
                     "dp_synth_logits");
}

int dp_encode_decisions(const int32_t* token, const double* logprob, const uint8_t* flags, const uint64_t* seq_ids,
                        int64_t B, uint8_t* out, void* stream) {
  if (!token || !logprob || !flags || !seq_ids || !out || B < 0)
    return fail(DP_ERR_ARG, "dp_encode_decisions: null argument%s");
  return cuda_status(dp_launch_encode(token, logprob, flags, seq_ids, B, out, (cudaStream_t)stream),
                     "dp_encode_decisions");
}

int dp_hot_mass_curve(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld, const double* row_max,
                      const double* total_expsum, const dp_params_t* params, const dp_penalty_t* pen_host,
                      const int32_t* inv_perm, const int32_t* col_of_pos, const int32_t* grid, int32_t n_grid,
                      double* out, void* stream) {
  if (!logits || !row_max || !total_expsum || !params || !grid || !out || n_grid < 1)
    return fail(DP_ERR_ARG, "dp_hot_mass_curve: null argument%s");
  if (!valid_pen(pen_host, V)) return fail(DP_ERR_ARG, "dp_hot_mass_curve: penalty state does not match V%s");
  if (B == 0) return DP_OK;
  return cuda_status(dp::launch_hot_mass_curve(logits, dtype, B, V, ld, row_max, total_expsum, params, *pen_host,
                                               inv_perm, col_of_pos, grid, n_grid, out, (cudaStream_t)stream),
                     "dp_hot_mass_curve");
}

}  // extern "C"
