/*
 * decplane_b200.h — C ABI of the B200-native decision plane (sampling epilogue).
 *
 * Drop-in boundary for the reference's sampler surface (arXiv 2512.00719,
 * reference package `decplane`, /root/reference/pkg/src/decplane).  The
 * reference exposes this path only as Python calls; each entry point below
 * names the reference interface it replaces.  All pointers are DEVICE pointers
 * unless the parameter name ends in `_host`; every call is stream-ordered on
 * `stream` (a cudaStream_t passed as void*), never synchronises, and returns
 * DP_OK (0) or a negative dp_status_t.  Per-row problems are reported in the
 * per-row `flags` byte instead of exceptions (the Python host layer turns
 * them into DegenerateRowError / RangeError like core.py:15-20).
 *
 * Layout conventions
 *   logits   row-major [B, ld] (ld >= V), fp32 or bf16.  This is byte-identical
 *            to the reference's "vocabulary-major" shard of one TP rank
 *            (core.py:184-199: (V, B) in Fortran order).
 *   hot-first rows (SHVS): position p < H holds hot id perm[p] in hot order,
 *            positions H..V-1 hold the tail ids in ascending order
 *            (shvs.py:37-92).  perm maps position -> token id, inv_perm the
 *            inverse.  Identity layout = perm NULL.
 */
#ifndef DECPLANE_B200_H
#define DECPLANE_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define DP_API __attribute__((visibility("default")))
#else
#define DP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DP_OK = 0,
  DP_ERR_ARG = -1,          /* invalid argument (ValueError in the reference)   */
  DP_ERR_CUDA = -2,         /* CUDA launch / runtime failure                    */
  DP_ERR_UNSUPPORTED = -3,  /* shape or dtype outside what this build supports  */
  DP_ERR_CAPACITY = -4      /* a fixed-capacity buffer would overflow           */
} dp_status_t;

typedef enum { DP_F32 = 0, DP_BF16 = 1 } dp_dtype_t;

/* per-row flag bits */
#define DP_FLAG_EOS            0x01u  /* the token is an end-of-sequence id (TokenDecision.is_eos) */
#define DP_FLAG_ACCEPTED_HOT   0x02u  /* SHVS took the hot path (TokenDecision.accepted_hot) */
#define DP_FLAG_NEAR_BOUNDARY  0x04u  /* a draw / accept / top-p / min-p decision was within
                                         1e-6 of its flip point (logged by the host)          */
#define DP_FLAG_REJECTED       0x08u  /* SHVS rejected the hot proposal -> tail pass           */
#define DP_FLAG_PEN_OVERFLOW   0x40u  /* penalty list full; token not recorded                */
#define DP_FLAG_DEGENERATE     0x80u  /* no usable probability mass (DegenerateRowError)      */

/* SamplingParams (core.py:23-34), one per row. top_k 0 = disabled. 64 bytes. */
typedef struct {
  double   temperature;
  int32_t  top_k;
  int32_t  reserved;
  double   top_p;
  double   min_p;
  double   rep_penalty;
  double   presence_penalty;
  double   frequency_penalty;
  uint64_t seed;
} dp_params_t;

/* Sparse, device-resident SequenceState (core.py:100-169).  Row b owns
 * entries [b*cap, b*cap+len[b]) of ids/out_count: every token in prompt ∪
 * output (the reference's touched_ids) with its output count (0 = prompt
 * only).  prompt_len[b] entries form the prompt prefix (for reset). */
typedef struct {
  int32_t* ids;
  int32_t* out_count;
  int32_t* len;
  int32_t* prompt_len;
  int32_t  cap;
  int32_t  vocab_size;
  int32_t  max_len;     /* host-known upper bound of len[b] over the call's rows
                           (prompt uniques + tokens recorded since the last reset);
                           0 = unknown (cap).  Sizes the kernels' candidate lists. */
  int32_t  reserved;
} dp_penalty_t;

/* Optional per-row diagnostics (any field may be NULL). */
typedef struct {
  int32_t* topk_ids;     /* [B, topk_stride] top-k stage ids, sorted (value desc, id asc) */
  double*  topk_ready;   /* [B, topk_stride] their sampling-ready values (penalized / tau) */
  int32_t  topk_stride;
  int32_t  reserved;
  double*  margin;       /* [B] distance of the closest decision to its flip point        */
  int32_t* kept;         /* [B] candidates surviving top-k/top-p/min-p                     */
  double*  alpha;        /* [B] SHVS hot mass alpha (shvs.py:148-154)                      */
  uint64_t* bytes_touched; /* [B] logits bytes streamed for the row (VisitCounter analogue) */
  int64_t* stats;          /* [24] launch counters: 0 rows, 1 re-streams (estimate too high),
                              2 SHVS accept tests re-summed exactly (summary_raw),
                              3 candidates admitted                                        */
} dp_debug_t;

/* Launch plan supplied by the host (nullable -> conservative defaults).
 * max_top_k: upper bound of top_k over the rows of the call (0 = unknown);
 *   it sizes the top-k capacities.  Rows that do not fit take the general
 *   (radix) path unless the bounds below promise there are none.
 * min_top_k: lower bound of top_k over the rows (0 = some row may have top-k
 *   off).  When BOTH bounds are nonzero they are promises about every row of
 *   the call and kernels that no row can need are not launched; a row that
 *   breaks the promise is left undecided.  0 / 0 is always safe.
 * split: CTAs per row cluster for the streaming kernels (0 = auto, <= 8).
 * kernel: 0 = auto, 1 = per-row CTA / cluster kernel, 2 = warp-per-row kernel
 *   for rows with top_k <= 64 (auto picks it for the SHVS hot pass at B >= SMs).
 * Rows with top-k off (top-p only, min-p only, neutral) are decided by the top-k
 *   kernel from their 256 largest values plus the domain mass when min_top_k == 0,
 *   with the general kernel as the exact fallback.  That needs the workspace.
 * workspace: CALLER-OWNED device scratch of workspace_len int32 elements
 *   (>= dp_workspace_len(B)), used stream-ordered by the call only: the
 *   library keeps no global buffers, so calls on different streams with
 *   different workspaces never share state and CUDA-graph capture is safe.
 *   NULL: nucleus rows take the (slower, exact) general kernel directly. */
/* dp_plan_t.flags: test hook — every accept test of a raw-summary SHVS call
 * goes through the exact re-sum (normally only the ones the cancelling
 * correction cannot decide) */
#define DP_PLAN_FORCE_RESUM 0x1
/* dp_sample_full: keep the one-CTA-per-row top-k kernel even when the batch
 * spans several waves (A-B tests of the persistent warp-specialised K1p) */
#define DP_PLAN_NO_PERSIST 0x2
/* dp_sample_full: use K1p whenever its rows allow (tests) */
#define DP_PLAN_FORCE_PERSIST 0x4
/* dp_sample_shvs with H <= 4096: the exact-sort hot pass K1h decides the
 * nucleus rows (top-k off) instead of the streaming kernels' 256-entry list +
 * general-kernel fallback (measured slower at H = 2,048: opt-in) */
#define DP_PLAN_HOT_SORT 0x8
/* ... and every hot row (tests) */
#define DP_PLAN_HOT_SORT_ALL 0x10

typedef struct {
  int32_t max_top_k;
  int32_t split;
  int32_t threads;      /* ignored (kept for ABI stability): the top-k kernel runs 256 threads */
  int32_t summary_raw;  /* dp_sample_shvs: row_max/total_expsum are the producer's raw
                           summary (dp_row_summary_raw); correct it for penalties */
  int32_t min_top_k;
  int32_t kernel;
  int32_t fuse_update;  /* record every decided token in the penalty state inside the
                           deciding kernel (update_output_histogram, penalty.py:18-32),
                           replacing a separate dp_penalty_update launch */
  int32_t flags;        /* DP_PLAN_* bits */
  int32_t* workspace;   /* caller-owned scratch, see above (nullable) */
  int64_t  workspace_len;
} dp_plan_t;

/* Library / device info. dp_device_check returns DP_OK when `device` is sm_100. */
DP_API int dp_version(void);
DP_API int dp_device_check(int device);
/* Human-readable reason of the last failing call on this thread. */
DP_API const char* dp_last_error(void);
/* int32 elements of dp_plan_t.workspace needed by a call over B rows. */
DP_API int64_t dp_workspace_len(int64_t B);

/* rng.pregenerate_slice (rng.py:94-113), keyed per row by params[b].seed:
 * out[b,0..2] = (u_hot, u_accept, u_tail) for (seed_b, iteration, seq_ids[b]). */
DP_API int dp_uniforms(const dp_params_t* params, const uint64_t* seq_ids, int64_t B,
                uint64_t iteration, double* out, void* stream);

/* Full-vocabulary decision: _Sampler("offload-truncate").sample for every row
 * (service.py:381-409) == sample_full (filtering.py:172-201) token law:
 * penalties (penalty.py:66-78) -> /tau (service.py:236-241) -> top-k -> top-p
 * -> min-p (filtering.py:61-105) -> inverse-CDF draw with u_hot
 * (filtering.py:158-162).  uniforms may be NULL: then they are derived on
 * device from (params[b].seed, iteration, seq_ids[b]) exactly as dp_uniforms. */
DP_API int dp_sample_full(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                   const dp_params_t* params, const dp_penalty_t* pen_host,
                   const double* uniforms, const uint64_t* seq_ids, uint64_t iteration,
                   int32_t* token, double* logprob, uint8_t* flags,
                   const dp_debug_t* debug_host, const dp_plan_t* plan_host, void* stream);

/* TP-sharded logits, read in place (replaces AssembledLogitsView +
 * assemble_view, transport.py:460-557): the t vocab shards of equal width
 * W = V / t tile [0, V); row b of shard s (vocab [s*W, (s+1)*W)) is at
 * shards[s] + b * ld elements (ld >= W; the reference's (W, B) Fortran-order
 * LogitsShardBlock.values, core.py:185-201, is exactly this layout).
 * shards is a HOST array of t <= 8 device pointers (peer memory of other TP
 * ranks is addressable once peer access is enabled; untested on >1 GPU).  One cluster of t CTAs decides a
 * row, CTA s streaming shard s; results equal dp_sample_full on the stitched
 * rows.  Rows must all carry top-k: plan->min_top_k > 0 and plan->max_top_k
 * within the top-k kernel's capacity, else DP_ERR_UNSUPPORTED (stitch and
 * call dp_sample_full).  Bad tiling -> DP_ERR_ARG (IncompleteIterationError). */
DP_API int dp_sample_full_sharded(const void* const* shards, int32_t t, int dtype, int64_t B, int64_t V,
                   int64_t ld, const dp_params_t* params, const dp_penalty_t* pen_host,
                   const double* uniforms, const uint64_t* seq_ids, uint64_t iteration,
                   int32_t* token, double* logprob, uint8_t* flags,
                   const dp_debug_t* debug_host, const dp_plan_t* plan_host, void* stream);

/* Producer summary: make_shard_blocks' per-row (row_max, total_expsum) over the
 * penalized, temperature-scaled row (service.py:470-504, shvs.py:157-168).
 * Layout-agnostic (a permutation does not change max or sum). */
DP_API int dp_row_summary(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                   const dp_params_t* params, const dp_penalty_t* pen_host,
                   const int32_t* inv_perm, double* row_max, double* total_expsum,
                   void* stream);

/* Producer-side raw summary: (max, sum exp) of x/tau per row WITHOUT
 * penalties — what a logits producer (LM-head epilogue) can emit while writing
 * the row.  dp_sample_shvs with plan->summary_raw = 1 corrects it exactly for
 * the sparse penalty list (O(|list|) per row), so an SHVS step never streams
 * the full row (the make_shard_blocks contract, service.py:470-504, paper
 * section 5.3 "w can be pre-computed on GPUs when writing logits"). */
DP_API int dp_row_summary_raw(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                              const dp_params_t* params, double* row_max, double* total_expsum,
                              void* stream);

/* Speculative hot-vocab sampling on hot-first rows: split_decision
 * (shvs.py:198-255) as driven by _Sampler SHVS (service.py:354-380).  Touches
 * H positions per row, plus V-H on rejection.  scratch_rows: device int32
 * [B + 1] workspace for the on-device reject list. */
DP_API int dp_sample_shvs(const void* logits_hotfirst, int dtype, int64_t B, int64_t V, int64_t H,
                   int64_t ld, const int32_t* perm, const int32_t* inv_perm,
                   const double* row_max, const double* total_expsum,
                   const dp_params_t* params, const dp_penalty_t* pen_host,
                   const double* uniforms, const uint64_t* seq_ids, uint64_t iteration,
                   int32_t* token, double* logprob, uint8_t* flags,
                   const dp_debug_t* debug_host, const dp_plan_t* plan_host,
                   int32_t* scratch_rows, void* stream);

/* dp_sample_shvs over split storage: hot positions [0, H) of row b at
 * logits_hot + b*ld_hot (device memory), tail positions [H, V) at
 * logits_tail + b*ld_tail — device memory, or pinned (mapped) HOST memory that
 * the tail pass reads zero-copy.  With host-resident logits a caller copies
 * only the hot prefix to the GPU (the paper's hot/tail split, section 4.2):
 * the tail crosses PCIe only for the rows the hot pass rejects.  Same
 * decision law and outputs as dp_sample_shvs (shvs.py:198-255). */
DP_API int dp_sample_shvs_split(const void* logits_hot, int64_t ld_hot, const void* logits_tail, int64_t ld_tail,
                   int dtype, int64_t B, int64_t V, int64_t H, const int32_t* perm, const int32_t* inv_perm,
                   const double* row_max, const double* total_expsum,
                   const dp_params_t* params, const dp_penalty_t* pen_host,
                   const double* uniforms, const uint64_t* seq_ids, uint64_t iteration,
                   int32_t* token, double* logprob, uint8_t* flags,
                   const dp_debug_t* debug_host, const dp_plan_t* plan_host,
                   int32_t* scratch_rows, void* stream);

/* Host-resident logits (the decision plane's CPU-side ring, transport.py:326-386):
 * copy the hot prefix [0, H) of each hot-first host row (pinned, row stride
 * ld_host elements) into a device staging buffer [B, ld_dev] — one strided
 * DMA.  Pair with dp_sample_shvs_split(hot_dev, ld_dev, host_row + H, ld_host,
 * ...) so only the hot prefix crosses PCIe up front. */
DP_API int dp_stage_hot(const void* logits_host, int64_t ld_host, int dtype, int64_t B, int64_t H, void* hot_dev,
                 int64_t ld_dev, void* stream);

/* update_output_histogram (penalty.py:18-32) for every row: C_o[tok] += 1,
 * first-seen ids appended.  Rows whose flags[b] has DP_FLAG_DEGENERATE are
 * skipped; a full list sets DP_FLAG_PEN_OVERFLOW. flags may be NULL. */
DP_API int dp_penalty_update(const dp_penalty_t* pen_host, const int32_t* token, int64_t B,
                      uint8_t* flags, void* stream);

/* Reset rows to their prompt-only state (new_sequence_state, core.py:144-169). */
DP_API int dp_penalty_reset(const dp_penalty_t* pen_host, int64_t B, void* stream);

/* apply_penalties(...)/tau materialised as f64 rows (ReadyColumn.full,
 * service.py:236-241).  Debug / parity use. */
DP_API int dp_ready_rows(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                  const dp_params_t* params, const dp_penalty_t* pen_host,
                  double* out, void* stream);

/* SyntheticSource (service.py:429-467): base_by_id[V] (f64) + noise * Gumbel
 * keyed by (seed, DOMAIN_LOGITS, iteration, seq_ids[b], v), written as
 * fp32 or bf16 rows; perm (position -> id, may be NULL) writes hot-first rows.
 * The producer-fused summary (make_shard_blocks, service.py:470-504): with
 * row_max / total_expsum (and params, for tau) non-NULL the same pass also
 * emits each row's penalty-free (max, Σ exp(x/tau - max)) of the values as
 * written — dp_row_summary_raw's output, without re-reading the rows. */
DP_API int dp_synth_logits(const double* base_by_id, double noise, uint64_t seed, uint64_t iteration,
                    const uint64_t* seq_ids, int64_t B, int64_t V, int64_t ld, const int32_t* perm,
                    int dtype, void* out, const dp_params_t* params, double* row_max,
                    double* total_expsum, void* stream);

/* Batch hit-ratio curve (sizing.estimate_hit_ratio_curve, sizing.py:78-100):
 * out[b, g] = ready mass of the first grid[g] positions of the curve's hot
 * ordering / total_expsum.  inv_perm: token id -> curve position (penalty
 * lookups).  col_of_pos (nullable): curve position -> column of `logits` when
 * the rows are laid out in another order (the online sizing loop measures the
 * master ordering on rows written for the current hot size); NULL: the rows
 * are in curve order. */
DP_API int dp_hot_mass_curve(const void* logits, int dtype, int64_t B, int64_t V, int64_t ld,
                      const double* row_max, const double* total_expsum,
                      const dp_params_t* params, const dp_penalty_t* pen_host,
                      const int32_t* inv_perm, const int32_t* col_of_pos, const int32_t* grid, int32_t n_grid,
                      double* out, void* stream);

/* DecisionBatch wire payload (transport.py:173-184) for B decisions: out =
 * u32 B, then per row u64 seq_id, u32 token, u8 flags (bit0 eos = DP_FLAG_EOS,
 * bit1 accepted_hot, bit2 has_logprob = 1), f32 logprob; 4 + 17 B bytes,
 * little-endian.  The host adds the 20-byte frame header and the CRC32. */
DP_API int dp_encode_decisions(const int32_t* token, const double* logprob, const uint8_t* flags,
                               const uint64_t* seq_ids, int64_t B, uint8_t* out, void* stream);

/* Token-id all-gather across batch shards (partition_batch + DecisionLedger,
 * transport.py:133-144, :400-433; service.py:743-748): one ncclAllGather of
 * rows_per_rank int32 tokens per rank into global[world * rows_per_rank], in
 * rank order, on `stream`.  `comm` is an ncclComm_t (dp_nccl_comm_init, or the
 * caller's own).  NCCL is resolved at run time (dlopen libnccl.so.2, reusing a
 * copy already loaded in the process); without it these return
 * DP_ERR_UNSUPPORTED.  dp_nccl_unique_id writes the 128-byte ncclUniqueId that
 * rank 0 hands to every rank out of band; dp_nccl_comm_init runs on the
 * caller's current device. */
DP_API int dp_nccl_available(void);
DP_API int dp_nccl_unique_id(uint8_t* id128);
DP_API int dp_nccl_comm_init(void** comm, int32_t nranks, const uint8_t* id128, int32_t rank);
DP_API int dp_nccl_comm_destroy(void* comm);
DP_API int dp_allgather_tokens(const int32_t* local, int32_t* global, int64_t rows_per_rank, void* comm,
                               void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DECPLANE_B200_H */
