"""Batched decision plane: logits [B, V] on the GPU -> next-token ids.

`DecisionPlane.sample` is the B200 replacement for the reference's per-row
worker loop (service.py:752-766: uniforms -> _Sampler.sample ->
update_output_histogram) over a whole batch, in two or three kernel launches
and no host synchronisation:

* variant "full"  (service.py:381-409, _Sampler("offload-truncate")): fused
  penalties -> /tau -> top-k -> top-p -> min-p -> inverse-CDF draw;
* variant "shvs"  (service.py:354-380): hot prefix pass with the rejection
  test against the producer summary (row_max, total_expsum), tail pass only
  for rejected rows (on-device reject list).

Per-row uniforms are keyed by (params.seed, iteration, seq_id) exactly as
rng.pregenerate_slice (rng.py:94-113), so tokens are invariant to batching and
to the GPU count.  The functional helpers `sample_full` / `shvs_sample` keep
the reference signatures (filtering.py:172, shvs.py:258) for single rows.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import DegenerateRowError, SamplingParams, TokenDecision, params_bytes, validate_params
from .penalty import PenaltyState
from .shvs import HotVocab

VARIANT_FULL = "full"
VARIANT_SHVS = "shvs"


def _dtype_code(t) -> int:
    import torch

    if t.dtype == torch.float32:
        return N.DP_F32
    if t.dtype == torch.bfloat16:
        return N.DP_BF16
    raise ValueError(f"logits dtype {t.dtype} unsupported (float32 or bfloat16)")


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream() -> C.c_void_p:
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class Decisions:
    """Device-side results of one batched call (all tensors length B)."""

    token: "object"          # int32
    logprob: "object"        # float64
    flags: "object"          # uint8
    alpha: "object" = None   # float64 (SHVS hot mass)
    margin: "object" = None  # float64 (closest decision-boundary distance)
    kept: "object" = None
    bytes_touched: "object" = None
    topk_ids: "object" = None
    topk_ready: "object" = None
    stats: "object" = None   # int64[8] launch counters (see dp_debug_t.stats)


class DecisionPlane:
    """A batch of B sequences with per-row params and GPU penalty state."""

    def __init__(self, vocab_size: int, params, prompts=None, seq_ids=None, hot: HotVocab | None = None,
                 device="cuda", max_generated: int = 256, pen_cap: int | None = None, split: int = 0,
                 kernel: int = 0):
        import torch

        self.device = torch.device(device)
        N.require_device(self.device)
        self.vocab_size = int(vocab_size)
        params = list(params) if isinstance(params, (list, tuple)) else None if params is None else [params]
        if prompts is None:
            prompts = [[] for _ in range(len(params))]
        self.batch = len(prompts)
        if len(params) == 1 and self.batch > 1:
            params = params * self.batch
        self.seq_ids = np.arange(self.batch, dtype=np.uint64) if seq_ids is None else np.asarray(seq_ids, np.uint64)
        if self.seq_ids.shape[0] != self.batch:
            raise ValueError("seq_ids must have one entry per row")
        self._seq_dev = torch.from_numpy(self.seq_ids.view(np.int64)).to(self.device)
        self.state = PenaltyState(prompts, vocab_size, cap=pen_cap, device=self.device, max_generated=max_generated)
        self.hot = hot
        self.split = int(split)
        self.kernel = int(kernel)   # dp_plan_t.kernel: 0 auto, 1 CTA/cluster, 2 warp-per-row
        self.set_params(params)
        self._out = None
        self._scratch = torch.empty(self.batch + 1, dtype=torch.int32, device=self.device)

    # -- configuration -----------------------------------------------------
    def set_params(self, params) -> None:
        import torch

        if len(params) != self.batch:
            raise ValueError("need one SamplingParams per row")
        for p in params:
            errs = validate_params(p, self.vocab_size)
            if errs:
                raise ValueError("; ".join(errs))
        self.params = list(params)
        raw = np.frombuffer(params_bytes(self.params), dtype=np.uint8).copy()
        self._params_dev = torch.from_numpy(raw).to(self.device)
        ks = [p.top_k for p in self.params if p.top_k > 0]
        # exact bounds over the rows: they let the library skip kernels no row needs
        min_k = min(p.top_k for p in self.params) if self.params else 0
        self._plan = N.Plan(max(ks) if ks else 0, self.split)
        self._plan.min_top_k = max(0, min_k) if ks else 0
        self._plan.kernel = self.kernel

    def set_hot(self, hot: HotVocab | None) -> None:
        """Hot-set changes land between iterations (service.py:602-610, :646-648)."""
        self.hot = hot

    @property
    def params_dev(self):
        return self._params_dev

    def _outputs(self, debug: bool, topk_stride: int):
        import torch

        dev, b = self.device, self.batch
        key = (debug, topk_stride)
        if self._out is None or self._out[0] != key:
            d = Decisions(torch.empty(b, dtype=torch.int32, device=dev), torch.empty(b, dtype=torch.float64, device=dev),
                          torch.zeros(b, dtype=torch.uint8, device=dev))
            d.alpha = torch.ones(b, dtype=torch.float64, device=dev)
            if debug:
                d.margin = torch.empty(b, dtype=torch.float64, device=dev)
                d.kept = torch.empty(b, dtype=torch.int32, device=dev)
                d.bytes_touched = torch.zeros(b, dtype=torch.int64, device=dev)
                d.stats = torch.zeros(24, dtype=torch.int64, device=dev)
                if topk_stride:
                    d.topk_ids = torch.full((b, topk_stride), -1, dtype=torch.int32, device=dev)
                    d.topk_ready = torch.full((b, topk_stride), float("nan"), dtype=torch.float64, device=dev)
            self._out = (key, d)
        return self._out[1]

    def _debug_struct(self, d: Decisions, topk_stride: int, debug: bool) -> N.Debug:
        if not debug:
            return N.Debug(None, None, 0, 0, None, None, d.alpha.data_ptr(), None, None)
        return N.Debug(_ptr(d.topk_ids).value, _ptr(d.topk_ready).value, topk_stride, 0, d.margin.data_ptr(),
                       d.kept.data_ptr(), d.alpha.data_ptr(), d.bytes_touched.data_ptr(), d.stats.data_ptr())

    # -- the hot path ----------------------------------------------------------
    def sample(self, logits, iteration: int, variant: str = VARIANT_FULL, uniforms=None, summary=None,
               update: bool = True, debug: bool = False, topk_stride: int = 0,
               summary_raw: bool = False) -> Decisions:
        """One decision per row.  `logits` is a [B, V] CUDA tensor (fp32/bf16,
        unit stride along V) in vocab order for "full" and hot-first order for
        "shvs".  `summary` = (row_max, total_expsum) f64 tensors from the
        producer (make_shard_blocks contract, service.py:470-504); computed here
        with one extra pass when omitted.  With `summary_raw=True` the summary
        is the producer's penalty-free one (`producer_summary`), corrected on
        device for the sparse penalty list, so a step never re-reads the row."""
        if logits.dim() != 2 or logits.shape[0] != self.batch or logits.shape[1] != self.vocab_size:
            raise ValueError(f"logits must be [{self.batch}, {self.vocab_size}]")
        if not logits.is_cuda or logits.stride(1) != 1:
            raise ValueError("logits must be a CUDA tensor with unit stride along the vocabulary")
        dt = _dtype_code(logits)
        d = self._outputs(debug, topk_stride)
        dbg = self._debug_struct(d, topk_stride, debug)
        st = _stream()
        uni = _ptr(uniforms)
        # the penalty update runs inside the deciding kernels (no extra launch)
        self._plan.fuse_update = 1 if update else 0
        if variant == VARIANT_FULL:
            N.call("dp_sample_full", _ptr(logits), dt, self.batch, self.vocab_size, logits.stride(0),
                   _ptr(self._params_dev), C.byref(self.state.native), uni, _ptr(self._seq_dev), int(iteration),
                   _ptr(d.token), _ptr(d.logprob), _ptr(d.flags), C.byref(dbg), C.byref(self._plan), st)
        elif variant == VARIANT_SHVS:
            if self.hot is None:
                raise ValueError("SHVS needs a HotVocab")
            perm, inv = self.hot.device_maps(self.device)
            if summary is None:
                summary = self.row_summary(logits, inv_perm=inv)
            rmax, tot = summary
            self._plan.summary_raw = 1 if summary_raw else 0
            N.call("dp_sample_shvs", _ptr(logits), dt, self.batch, self.vocab_size, self.hot.size,
                   logits.stride(0), _ptr(perm), _ptr(inv), _ptr(rmax), _ptr(tot), _ptr(self._params_dev),
                   C.byref(self.state.native), uni, _ptr(self._seq_dev), int(iteration), _ptr(d.token),
                   _ptr(d.logprob), _ptr(d.flags), C.byref(dbg), C.byref(self._plan), _ptr(self._scratch), st)
        else:
            raise ValueError(f"unknown variant {variant!r}")
        return d

    def sample_sharded(self, shards, iteration: int, uniforms=None, update: bool = True, debug: bool = False,
                       topk_stride: int = 0) -> Decisions:
        """Full-vocabulary decisions over TP-sharded logits, read in place:
        `shards` = t <= 8 CUDA tensors [B, V/t] (vocab [s V/t, (s+1) V/t) in
        shard s), one row stride, unit stride along the vocabulary — the
        AssembledLogitsView / assemble_view contract (transport.py:460-557) on
        the device.  Same decisions as `sample` on the stitched rows.  The
        shards are stitched (one device copy) only when some row has top-k off
        or wider than the top-k kernel takes (dp_sample_full_sharded's
        DP_ERR_UNSUPPORTED) or the shards do not share a row stride."""
        import torch

        t = len(shards)
        if t < 1 or t > 8:
            raise ValueError("need 1..8 vocab shards")
        w = shards[0].shape[1] if shards[0].dim() == 2 else -1
        for x in shards:
            if x.dim() != 2 or x.shape[0] != self.batch or x.shape[1] != w:
                raise ValueError(f"shard tiling broken: every shard must be [{self.batch}, V/t]")
            if not x.is_cuda or x.stride(1) != 1 or x.dtype != shards[0].dtype:
                raise ValueError("shards must be CUDA tensors of one dtype with unit stride along the vocabulary")
        if w * t != self.vocab_size:
            raise ValueError(f"shards cover {w * t} ids, vocabulary has {self.vocab_size}")
        self.last_stitched = True   # read by the tests: which path decided the call
        if any(x.stride(0) != shards[0].stride(0) for x in shards):
            return self.sample(torch.cat(list(shards), dim=1), iteration, uniforms=uniforms, update=update,
                               debug=debug, topk_stride=topk_stride)
        dt = _dtype_code(shards[0])
        d = self._outputs(debug, topk_stride)
        dbg = self._debug_struct(d, topk_stride, debug)
        self._plan.fuse_update = 1 if update else 0
        ptrs = (C.c_void_p * t)(*[x.data_ptr() for x in shards])
        st = N.load().dp_sample_full_sharded(
            ptrs, t, dt, self.batch, self.vocab_size, shards[0].stride(0), _ptr(self._params_dev),
            C.byref(self.state.native), _ptr(uniforms), _ptr(self._seq_dev), int(iteration), _ptr(d.token),
            _ptr(d.logprob), _ptr(d.flags), C.byref(dbg), C.byref(self._plan), _stream())
        if st == N.DP_ERR_UNSUPPORTED:
            return self.sample(torch.cat(list(shards), dim=1), iteration, uniforms=uniforms, update=update,
                               debug=debug, topk_stride=topk_stride)
        N.check(st, "dp_sample_full_sharded")
        self.last_stitched = False
        return d

    def sample_split(self, hot, tail, iteration: int, summary, uniforms=None, update: bool = True,
                     debug: bool = False, topk_stride: int = 0, summary_raw: bool = False) -> Decisions:
        """SHVS over split storage: `hot` = [B, >=H] CUDA tensor with the hot
        prefix of each hot-first row, `tail` = [B, >=V-H] tensor with the rest
        — a CUDA tensor or a PINNED HOST tensor, read zero-copy by the tail pass
        for rejected rows only.  `summary` = the producer's (row_max,
        total_expsum) (required: the full row is not re-read here)."""
        import torch

        if self.hot is None:
            raise ValueError("SHVS needs a HotVocab")
        h = self.hot.size
        if hot.dim() != 2 or hot.shape[0] != self.batch or hot.shape[1] < h or not hot.is_cuda or hot.stride(1) != 1:
            raise ValueError(f"hot must be a CUDA tensor [{self.batch}, >= {h}] with unit stride")
        if tail.dim() != 2 or tail.shape[0] != self.batch or tail.shape[1] < self.vocab_size - h or tail.stride(1) != 1:
            raise ValueError(f"tail must be [{self.batch}, >= {self.vocab_size - h}] with unit stride")
        if not tail.is_cuda and not tail.is_pinned():
            raise ValueError("a host tail must be pinned memory (read zero-copy by the tail pass)")
        if tail.dtype != hot.dtype:
            raise ValueError("hot and tail must share a dtype")
        dt = _dtype_code(hot)
        d = self._outputs(debug, topk_stride)
        dbg = self._debug_struct(d, topk_stride, debug)
        perm, inv = self.hot.device_maps(self.device)
        rmax, tot = summary
        self._plan.summary_raw = 1 if summary_raw else 0
        self._plan.fuse_update = 1 if update else 0
        N.call("dp_sample_shvs_split", _ptr(hot), hot.stride(0), _ptr(tail), tail.stride(0), dt, self.batch,
               self.vocab_size, h, _ptr(perm), _ptr(inv), _ptr(rmax), _ptr(tot), _ptr(self._params_dev),
               C.byref(self.state.native), _ptr(uniforms), _ptr(self._seq_dev), int(iteration), _ptr(d.token),
               _ptr(d.logprob), _ptr(d.flags), C.byref(dbg), C.byref(self._plan), _ptr(self._scratch), _stream())
        return d

    def sample_host(self, logits_host, iteration: int, summary_host, staging=None, update: bool = True,
                    summary_raw: bool = False) -> Decisions:
        """SHVS on HOST-resident hot-first logits (pinned [B, V] tensor): the hot
        prefix is staged to the GPU with one strided DMA (dp_stage_hot), the
        tail is read zero-copy by the tail pass for rejected rows only
        (dp_sample_shvs_split).  `summary_host` = the producer's (row_max,
        total_expsum), host f64 [B] tensors (copied with the logits)."""
        import torch

        if self.hot is None:
            raise ValueError("SHVS needs a HotVocab")
        if logits_host.is_cuda or not logits_host.is_pinned() or logits_host.stride(1) != 1:
            raise ValueError("logits_host must be a pinned host tensor with unit stride along V")
        h = self.hot.size
        if staging is None or staging.shape != (self.batch, h) or staging.dtype != logits_host.dtype:
            staging = torch.empty((self.batch, h), dtype=logits_host.dtype, device=self.device)
        N.call("dp_stage_hot", _ptr(logits_host), logits_host.stride(0), _dtype_code(logits_host), self.batch, h,
               _ptr(staging), staging.stride(0), _stream())
        rmax = summary_host[0].to(self.device, non_blocking=True)
        tot = summary_host[1].to(self.device, non_blocking=True)
        tail = logits_host[:, h:]
        return self.sample_split(staging, tail, iteration, (rmax, tot), update=update, summary_raw=summary_raw)

    def hot_mass_curve(self, logits_hotfirst, grid, summary=None):
        """Per-row hot mass alpha(H) at every grid size H (ready mass of the
        first H hot positions / total), [B, G] f64 on device — the batched
        GPU form of sizing.estimate_hit_ratio_curve (sizing.py:78-100)."""
        import torch

        if self.hot is None:
            raise ValueError("the hit-ratio curve needs a HotVocab")
        g = sorted(int(h) for h in grid)
        if not g or g[0] < 1 or g[-1] > self.vocab_size:
            raise ValueError(f"grid sizes must lie in [1, {self.vocab_size}]")
        perm, inv = self.hot.device_maps(self.device)
        if summary is None:
            summary = self.row_summary(logits_hotfirst, inv_perm=inv)
        rmax, tot = summary
        gd = torch.tensor(g, dtype=torch.int32, device=self.device)
        out = torch.empty((self.batch, len(g)), dtype=torch.float64, device=self.device)
        N.call("dp_hot_mass_curve", _ptr(logits_hotfirst), _dtype_code(logits_hotfirst), self.batch,
               self.vocab_size, logits_hotfirst.stride(0), _ptr(rmax), _ptr(tot), _ptr(self._params_dev),
               C.byref(self.state.native), _ptr(inv), _ptr(gd), len(g), _ptr(out), _stream())
        return out

    def row_summary(self, logits, inv_perm=None):
        """(row_max, total_expsum) of the ready rows (service.py:484-489)."""
        import torch

        rmax = torch.empty(self.batch, dtype=torch.float64, device=self.device)
        tot = torch.empty(self.batch, dtype=torch.float64, device=self.device)
        N.call("dp_row_summary", _ptr(logits), _dtype_code(logits), self.batch, self.vocab_size, logits.stride(0),
               _ptr(self._params_dev), C.byref(self.state.native), _ptr(inv_perm), _ptr(rmax), _ptr(tot), _stream())
        return rmax, tot

    def producer_summary(self, logits):
        """Penalty-free (row_max, total_expsum) of logits/tau: what a logits
        producer emits while writing the rows (dp_row_summary_raw)."""
        import torch

        rmax = torch.empty(self.batch, dtype=torch.float64, device=self.device)
        tot = torch.empty(self.batch, dtype=torch.float64, device=self.device)
        N.call("dp_row_summary_raw", _ptr(logits), _dtype_code(logits), self.batch, self.vocab_size,
               logits.stride(0), _ptr(self._params_dev), _ptr(rmax), _ptr(tot), _stream())
        return rmax, tot

    def uniforms(self, iteration: int):
        """rng.pregenerate_slice for every row, [B,3] f64 on device (rng.py:94-113)."""
        import torch

        out = torch.empty((self.batch, 3), dtype=torch.float64, device=self.device)
        N.call("dp_uniforms", _ptr(self._params_dev), _ptr(self._seq_dev), self.batch, int(iteration),
               _ptr(out), _stream())
        return out

    def to_decisions(self, d: Decisions, iteration: int, eos_ids=frozenset(), raise_degenerate: bool = True):
        """Host TokenDecision list (core.py:172-181); synchronises."""
        tok = d.token.cpu().numpy()
        lp = d.logprob.cpu().numpy()
        fl = d.flags.cpu().numpy()
        out = []
        for b in range(self.batch):
            if fl[b] & N.FLAG_DEGENERATE:
                if raise_degenerate:
                    raise DegenerateRowError(f"row {b} (seq {int(self.seq_ids[b])}) has no usable probability mass")
                out.append(None)
                continue
            t = int(tok[b])
            out.append(TokenDecision(int(iteration), int(self.seq_ids[b]), t, t in eos_ids,
                                     bool(fl[b] & N.FLAG_ACCEPTED_HOT), float(lp[b])))
        return out


# ---------------------------------------------------------------------------
# reference-shaped single-row helpers


def _one_row(logits_row, prompt, generated, params: SamplingParams, draws, vocab_size=None):
    import torch

    row = torch.as_tensor(logits_row)
    if row.dim() != 1:
        raise ValueError("logits_row must be 1-D")
    v = row.shape[0] if vocab_size is None else vocab_size
    if row.dtype not in (torch.float32, torch.bfloat16):
        row = row.to(torch.float32)
    plane = DecisionPlane(v, [params], prompts=[prompt], max_generated=max(len(generated), 1) + 1)
    for t in generated:
        plane.state.update(torch.tensor([t], dtype=torch.int32, device=plane.device))
    u = torch.as_tensor(np.asarray(draws, dtype=np.float64).reshape(1, -1)[:, :3], device=plane.device)
    if u.shape[1] < 3:
        u = torch.nn.functional.pad(u, (0, 3 - u.shape[1]))
    return plane, row.to(plane.device).reshape(1, -1).contiguous(), u


def sample_full(logits_row, state, params: SamplingParams, draws, iteration_id: int = 0,
                eos_ids=frozenset()) -> TokenDecision:
    """filtering.sample_full (filtering.py:172-201) on the GPU for one row.
    `state` is a core.SequenceState (prompt + generated tokens)."""
    plane, row, u = _one_row(logits_row, state.prompt_tokens, state.tokens, params, draws)
    d = plane.sample(row, iteration_id, VARIANT_FULL, uniforms=u, update=False)
    dec = plane.to_decisions(d, iteration_id, eos_ids)[0]
    dec.seq_id = state.seq_id
    return dec


def shvs_sample(logits_row, hot: HotVocab, state, params: SamplingParams, draws, iteration_id: int = 0,
                eos_ids=frozenset()) -> TokenDecision:
    """shvs.shvs_sample (shvs.py:258-289) on the GPU for one vocab-order row."""
    plane, row, u = _one_row(logits_row, state.prompt_tokens, state.tokens, params, draws)
    plane.set_hot(hot)
    hot_row = hot.to_hot_first(row).contiguous()
    d = plane.sample(hot_row, iteration_id, VARIANT_SHVS, uniforms=u, update=False)
    dec = plane.to_decisions(d, iteration_id, eos_ids)[0]
    dec.seq_id = state.seq_id
    return dec
