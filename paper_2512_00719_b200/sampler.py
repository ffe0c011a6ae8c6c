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
import logging
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import (DEFAULT_MAX_GENERATED, DegenerateRowError, SamplingParams, TokenDecision, params_bytes,
                   validate_params)
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


def _stream(device=None) -> C.c_void_p:
    import torch

    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


log = logging.getLogger("paper_2512_00719_b200")


@dataclass
class Decisions:
    """Device-side results of one batched call (all tensors length B).

    The plane reuses two sets of these buffers in turn: a `Decisions` stays
    valid until two further calls of the same kind (so a side stream may
    gather `token` while the next step samples)."""

    token: "object"          # int32
    logprob: "object"        # float64
    flags: "object"          # uint8
    alpha: "object" = None   # float64 (SHVS hot mass)
    margin: "object" = None  # float64 (closest decision-boundary distance)
    kept: "object" = None
    bytes_touched: "object" = None   # int64: bytes the call's kernels loaded per row (debug)
    topk_ids: "object" = None
    topk_ready: "object" = None
    stats: "object" = None   # int64[24] launch counters (see dp_debug_t.stats)


class DecisionPlane:
    """A batch of B sequences with per-row params and GPU penalty state.

    Every native call runs on `device` (its current stream), whatever device
    is current in the caller."""

    def __init__(self, vocab_size: int, params, prompts=None, seq_ids=None, hot: HotVocab | None = None,
                 device="cuda", max_generated: int = DEFAULT_MAX_GENERATED, pen_cap: int | None = None,
                 split: int = 0, kernel: int = 0):
        import torch

        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
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
        with torch.cuda.device(self.device):
            self._seq_dev = torch.from_numpy(self.seq_ids.view(np.int64)).to(self.device)
            self.state = PenaltyState(prompts, vocab_size, cap=pen_cap, device=self.device,
                                      max_generated=max_generated)
            self.hot = hot
            self.split = int(split)
            self.kernel = int(kernel)   # dp_plan_t.kernel: 0 auto, 1 CTA/cluster, 2 warp-per-row
            self.plan_flags = 0         # extra DP_PLAN_* bits (A-B / test hooks)
            # caller-owned library scratch (fallback row lists): one per plane
            wl = int(N.load().dp_workspace_len(self.batch))
            self._workspace = torch.zeros(wl, dtype=torch.int32, device=self.device)
            self.set_params(params)
            self._out = {}
            self._scratch = torch.empty(self.batch + 1, dtype=torch.int32, device=self.device)
        self.boundary_log = []        # (iteration, seq_id) of every decision within 1e-6 of a flip point

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
        self._plan.workspace = self._workspace.data_ptr()
        self._plan.workspace_len = self._workspace.numel()

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
        ring = self._out.setdefault(key, [None, None, 0])
        i = ring[2]
        ring[2] ^= 1
        if ring[i] is None:
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
            ring[i] = d
        return ring[i]

    def _debug_struct(self, d: Decisions, topk_stride: int, debug: bool) -> N.Debug:
        if not debug:
            return N.Debug(None, None, 0, 0, None, None, d.alpha.data_ptr(), None, None)
        d.bytes_touched.zero_()   # the kernels of one call accumulate into it (VisitCounter)
        return N.Debug(_ptr(d.topk_ids).value, _ptr(d.topk_ready).value, topk_stride, 0, d.margin.data_ptr(),
                       d.kept.data_ptr(), d.alpha.data_ptr(), d.bytes_touched.data_ptr(), d.stats.data_ptr())

    def _check_logits(self, x, name="logits"):
        if x.dim() != 2 or x.shape[0] != self.batch or x.shape[1] != self.vocab_size:
            raise ValueError(f"{name} must be [{self.batch}, {self.vocab_size}]")
        if not x.is_cuda or x.stride(1) != 1:
            raise ValueError(f"{name} must be a CUDA tensor with unit stride along the vocabulary")
        if x.device != self.device:
            raise ValueError(f"{name} is on {x.device}, the plane on {self.device}")

    # -- the hot path ----------------------------------------------------------
    def sample(self, logits, iteration: int, variant: str = VARIANT_FULL, uniforms=None, summary=None,
               update: bool = True, debug: bool = False, topk_stride: int = 0,
               summary_raw: bool = False, force_resum: bool = False) -> Decisions:
        """One decision per row.  `logits` is a [B, V] CUDA tensor (fp32/bf16,
        unit stride along V) in vocab order for "full" and hot-first order for
        "shvs".  `summary` = (row_max, total_expsum) f64 tensors from the
        producer (make_shard_blocks contract, service.py:470-504); computed here
        exactly (one extra pass) when omitted.  With `summary_raw=True` the
        given summary is the producer's penalty-free one (`producer_summary`,
        or `synthesize(..., summary=True)`), corrected on device for the sparse
        penalty list, so a step never re-reads the row."""
        import torch

        self._check_logits(logits)
        dt = _dtype_code(logits)
        if summary_raw and summary is None:
            raise ValueError("summary_raw=True needs the producer's raw summary")
        with torch.cuda.device(self.device):
            d = self._outputs(debug, topk_stride)
            dbg = self._debug_struct(d, topk_stride, debug)
            st = _stream(self.device)
            uni = _ptr(uniforms)
            # the penalty update runs inside the deciding kernels (no extra launch)
            self._plan.fuse_update = 1 if update else 0
            if variant == VARIANT_FULL:
                pen = self.state.prepare(update)
                N.call("dp_sample_full", _ptr(logits), dt, self.batch, self.vocab_size, logits.stride(0),
                       _ptr(self._params_dev), C.byref(pen), uni, _ptr(self._seq_dev), int(iteration),
                       _ptr(d.token), _ptr(d.logprob), _ptr(d.flags), C.byref(dbg), C.byref(self._plan), st)
            elif variant == VARIANT_SHVS:
                if self.hot is None:
                    raise ValueError("SHVS needs a HotVocab")
                perm, inv = self.hot.device_maps(self.device)
                if summary is None:
                    summary = self.row_summary(logits, inv_perm=inv)   # exact, penalized
                rmax, tot = summary
                self._plan.summary_raw = 1 if summary_raw else 0
                self._plan.flags = self.plan_flags | (N.PLAN_FORCE_RESUM if force_resum else 0)   # test hooks
                pen = self.state.prepare(update)
                N.call("dp_sample_shvs", _ptr(logits), dt, self.batch, self.vocab_size, self.hot.size,
                       logits.stride(0), _ptr(perm), _ptr(inv), _ptr(rmax), _ptr(tot), _ptr(self._params_dev),
                       C.byref(pen), uni, _ptr(self._seq_dev), int(iteration), _ptr(d.token),
                       _ptr(d.logprob), _ptr(d.flags), C.byref(dbg), C.byref(self._plan), _ptr(self._scratch), st)
            else:
                raise ValueError(f"unknown variant {variant!r}")
            self.state.committed(update)
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
        DP_ERR_UNSUPPORTED) or the shards do not share a row stride.  Shards
        must live on the plane's device (peer-GPU shards are not accepted)."""
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
            if x.device != self.device:
                raise ValueError(f"shard on {x.device}, the plane on {self.device}")
        if w * t != self.vocab_size:
            raise ValueError(f"shards cover {w * t} ids, vocabulary has {self.vocab_size}")
        self.last_stitched = True   # read by the tests: which path decided the call
        if any(x.stride(0) != shards[0].stride(0) for x in shards):
            return self.sample(torch.cat(list(shards), dim=1), iteration, uniforms=uniforms, update=update,
                               debug=debug, topk_stride=topk_stride)
        dt = _dtype_code(shards[0])
        with torch.cuda.device(self.device):
            d = self._outputs(debug, topk_stride)
            dbg = self._debug_struct(d, topk_stride, debug)
            self._plan.fuse_update = 1 if update else 0
            ptrs = (C.c_void_p * t)(*[x.data_ptr() for x in shards])
            pen = self.state.prepare(update)
            st = N.load().dp_sample_full_sharded(
                ptrs, t, dt, self.batch, self.vocab_size, shards[0].stride(0), _ptr(self._params_dev),
                C.byref(pen), _ptr(uniforms), _ptr(self._seq_dev), int(iteration), _ptr(d.token),
                _ptr(d.logprob), _ptr(d.flags), C.byref(dbg), C.byref(self._plan), _stream(self.device))
            if st == N.DP_ERR_UNSUPPORTED:
                return self.sample(torch.cat(list(shards), dim=1), iteration, uniforms=uniforms, update=update,
                                   debug=debug, topk_stride=topk_stride)
            N.check(st, "dp_sample_full_sharded")
            self.state.committed(update)
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
        if hot.device != self.device:
            raise ValueError(f"hot prefix on {hot.device}, the plane on {self.device}")
        if tail.dim() != 2 or tail.shape[0] != self.batch or tail.shape[1] < self.vocab_size - h or tail.stride(1) != 1:
            raise ValueError(f"tail must be [{self.batch}, >= {self.vocab_size - h}] with unit stride")
        if not tail.is_cuda and not tail.is_pinned():
            raise ValueError("a host tail must be pinned memory (read zero-copy by the tail pass)")
        if tail.dtype != hot.dtype:
            raise ValueError("hot and tail must share a dtype")
        dt = _dtype_code(hot)
        with torch.cuda.device(self.device):
            d = self._outputs(debug, topk_stride)
            dbg = self._debug_struct(d, topk_stride, debug)
            perm, inv = self.hot.device_maps(self.device)
            rmax, tot = summary
            self._plan.summary_raw = 1 if summary_raw else 0
            self._plan.fuse_update = 1 if update else 0
            self._plan.flags = self.plan_flags
            pen = self.state.prepare(update)
            N.call("dp_sample_shvs_split", _ptr(hot), hot.stride(0), _ptr(tail), tail.stride(0), dt, self.batch,
                   self.vocab_size, h, _ptr(perm), _ptr(inv), _ptr(rmax), _ptr(tot), _ptr(self._params_dev),
                   C.byref(pen), _ptr(uniforms), _ptr(self._seq_dev), int(iteration), _ptr(d.token),
                   _ptr(d.logprob), _ptr(d.flags), C.byref(dbg), C.byref(self._plan), _ptr(self._scratch),
                   _stream(self.device))
            self.state.committed(update)
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
        with torch.cuda.device(self.device):
            if staging is None or staging.shape != (self.batch, h) or staging.dtype != logits_host.dtype:
                staging = torch.empty((self.batch, h), dtype=logits_host.dtype, device=self.device)
            N.call("dp_stage_hot", _ptr(logits_host), logits_host.stride(0), _dtype_code(logits_host), self.batch, h,
                   _ptr(staging), staging.stride(0), _stream(self.device))
            rmax = summary_host[0].to(self.device, non_blocking=True)
            tot = summary_host[1].to(self.device, non_blocking=True)
        tail = logits_host[:, h:]
        return self.sample_split(staging, tail, iteration, (rmax, tot), update=update, summary_raw=summary_raw)

    def hot_mass_curve(self, logits_hotfirst, grid, summary=None, order: HotVocab | None = None):
        """Per-row hot mass alpha(H) at every grid size H (ready mass of the
        first H hot positions / total), [B, G] f64 on device — the batched
        GPU form of sizing.estimate_hit_ratio_curve (sizing.py:78-100).

        The curve follows the plane's hot ordering, or `order` (e.g. the
        master ordering of the online sizing loop, a longer ordering than the
        current hot set): the rows stay in the plane's current hot-first
        layout and are read through the position map."""
        import torch

        if self.hot is None:
            raise ValueError("the hit-ratio curve needs a HotVocab")
        self._check_logits(logits_hotfirst)
        g = sorted(int(h) for h in grid)
        if not g or g[0] < 1 or g[-1] > self.vocab_size:
            raise ValueError(f"grid sizes must lie in [1, {self.vocab_size}]")
        with torch.cuda.device(self.device):
            perm, inv = self.hot.device_maps(self.device)
            col = None
            if order is not None and not np.array_equal(order.perm, self.hot.perm):
                _, oinv = order.device_maps(self.device)
                col = inv.index_select(0, order.device_maps(self.device)[0].long())   # curve pos -> column
                inv = oinv
            if summary is None:
                summary = self.row_summary(logits_hotfirst, inv_perm=self.hot.device_maps(self.device)[1])
            rmax, tot = summary
            gd = torch.tensor(g, dtype=torch.int32, device=self.device)
            out = torch.empty((self.batch, len(g)), dtype=torch.float64, device=self.device)
            N.call("dp_hot_mass_curve", _ptr(logits_hotfirst), _dtype_code(logits_hotfirst), self.batch,
                   self.vocab_size, logits_hotfirst.stride(0), _ptr(rmax), _ptr(tot), _ptr(self._params_dev),
                   C.byref(self.state.native), _ptr(inv), _ptr(col), _ptr(gd), len(g), _ptr(out),
                   _stream(self.device))
        return out

    def row_summary(self, logits, inv_perm=None):
        """(row_max, total_expsum) of the ready rows (service.py:484-489)."""
        import torch

        self._check_logits(logits)
        with torch.cuda.device(self.device):
            rmax = torch.empty(self.batch, dtype=torch.float64, device=self.device)
            tot = torch.empty(self.batch, dtype=torch.float64, device=self.device)
            N.call("dp_row_summary", _ptr(logits), _dtype_code(logits), self.batch, self.vocab_size,
                   logits.stride(0), _ptr(self._params_dev), C.byref(self.state.native), _ptr(inv_perm), _ptr(rmax),
                   _ptr(tot), _stream(self.device))
        return rmax, tot

    def producer_summary(self, logits):
        """Penalty-free (row_max, total_expsum) of logits/tau: what a logits
        producer emits while writing the rows (dp_row_summary_raw)."""
        import torch

        self._check_logits(logits)
        with torch.cuda.device(self.device):
            rmax = torch.empty(self.batch, dtype=torch.float64, device=self.device)
            tot = torch.empty(self.batch, dtype=torch.float64, device=self.device)
            N.call("dp_row_summary_raw", _ptr(logits), _dtype_code(logits), self.batch, self.vocab_size,
                   logits.stride(0), _ptr(self._params_dev), _ptr(rmax), _ptr(tot), _stream(self.device))
        return rmax, tot

    def uniforms(self, iteration: int):
        """rng.pregenerate_slice for every row, [B,3] f64 on device (rng.py:94-113)."""
        import torch

        with torch.cuda.device(self.device):
            out = torch.empty((self.batch, 3), dtype=torch.float64, device=self.device)
            N.call("dp_uniforms", _ptr(self._params_dev), _ptr(self._seq_dev), self.batch, int(iteration),
                   _ptr(out), _stream(self.device))
        return out

    # -- sequence lifecycle (service.py:709-714) --------------------------------
    def mark_eos(self, d: Decisions, eos_ids) -> None:
        """Set DP_FLAG_EOS on every row whose token is an end-of-sequence id
        (TokenDecision.is_eos; carried by dp_encode_decisions), on device."""
        import torch

        if not eos_ids:
            return
        with torch.cuda.device(self.device):
            key = tuple(sorted(int(e) for e in eos_ids))
            if getattr(self, "_eos_key", None) != key:
                self._eos_key, self._eos_dev = key, torch.tensor(key, dtype=torch.int32, device=self.device)
            hit = torch.isin(d.token, self._eos_dev)
            d.flags.bitwise_or_(hit.to(torch.uint8) * N.FLAG_EOS)

    def select_rows(self, rows) -> None:
        """Keep only `rows` of the batch (in order): params, seq ids, penalty
        table and scratch follow; the hot set is shared.  Lands between
        iterations, like the reference's active-list update."""
        import torch

        rows = np.asarray(rows, dtype=np.int64)
        if rows.ndim != 1 or (rows.size and (rows.min() < 0 or rows.max() >= self.batch)):
            raise ValueError("rows must index the current batch")
        with torch.cuda.device(self.device):
            self.seq_ids = self.seq_ids[rows]
            self._seq_dev = torch.from_numpy(self.seq_ids.view(np.int64).copy()).to(self.device)
            self.state.select(torch.from_numpy(rows).to(self.device))
            self.batch = int(rows.size)
            wl = int(N.load().dp_workspace_len(self.batch))
            self._workspace = torch.zeros(wl, dtype=torch.int32, device=self.device)
            self.set_params([self.params[i] for i in rows.tolist()])
            self._out = {}
            self._scratch = torch.empty(self.batch + 1, dtype=torch.int32, device=self.device)

    def retire_finished(self, d: Decisions, eos_ids=frozenset(), max_tokens: int | None = None) -> np.ndarray:
        """The reference's retirement rule (service.py:709-714): drop every
        row whose token is an EOS id or whose sequence reached `max_tokens`
        generated tokens; returns the kept row indices (of the batch before
        the call).  Synchronises once (the new batch size is a host value)."""
        import torch

        with torch.cuda.device(self.device):
            keep = torch.ones(self.batch, dtype=torch.bool, device=self.device)
            if eos_ids:
                self.mark_eos(d, eos_ids)
                keep &= (d.flags & N.FLAG_EOS) == 0
            rows = torch.nonzero(keep).flatten().cpu().numpy()
        if max_tokens is not None and self.state.recorded >= int(max_tokens):
            rows = rows[:0]
        if rows.size != self.batch:
            self.select_rows(rows)
        return rows

    def to_decisions(self, d: Decisions, iteration: int, eos_ids=frozenset(), raise_degenerate: bool = True):
        """Host TokenDecision list (core.py:172-181); synchronises.

        Raises DegenerateRowError for a row without usable mass (core.py:19-20)
        and OverflowError when a row's penalty list could not record its token
        (the reference's append buffer, core.py:90-92).  Every decision whose
        draw / accept / top-p / min-p test came within 1e-6 of its flip point
        (DP_FLAG_NEAR_BOUNDARY) is logged and appended to `boundary_log`."""
        tok = d.token.cpu().numpy()
        lp = d.logprob.cpu().numpy()
        fl = d.flags.cpu().numpy()
        if (fl & N.FLAG_PEN_OVERFLOW).any():
            rows = np.flatnonzero(fl & N.FLAG_PEN_OVERFLOW)
            raise OverflowError(f"append buffer full: penalty list of rows {rows[:8].tolist()} cannot record "
                                f"their token")
        near = np.flatnonzero(fl & N.FLAG_NEAR_BOUNDARY)
        for b in near:
            self.boundary_log.append((int(iteration), int(self.seq_ids[b])))
            log.info("iteration %d seq %d: decision within 1e-6 of a boundary", iteration, int(self.seq_ids[b]))
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
