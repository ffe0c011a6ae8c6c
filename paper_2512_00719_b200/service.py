"""Drop-in replacements for the reference's per-row sampler surface.

A caller of the reference (`decplane`) swaps these in without edits:

* `Sampler` (alias `_Sampler`) == service._Sampler (service.py:282-420):
  `Sampler(variant, hot, counter).sample(view, col, seq_id, state, params,
  draws, iteration_id, eos_ids) -> TokenDecision`, where `view` is an
  AssembledLogitsView (the reference's or `transport.assemble_view`),
  `state` a SequenceState (the reference's or `core.new_sequence_state`) and
  `params` a SamplingParams (either).  The caller keeps ownership of the
  state and records the token itself with `update_output_histogram(state,
  token)` exactly as the reference worker loop does (service.py:752-766).
  `sample_batch` decides a whole column range in one GPU call.
* `sample_full` == filtering.sample_full (filtering.py:172-201).
* `shvs_sample` == shvs.shvs_sample (shvs.py:258-289) with a ShvsRowContext.
* `make_shard_blocks` == service.make_shard_blocks (service.py:470-504): the
  producer contract — wire logits plus the per-row (row_max, total_expsum)
  of the sampling-ready rows, computed on the GPU.

Every decision runs in the sm_100a kernels (dp_sample_full[_sharded] /
dp_sample_shvs) on identical logits and draws; the per-call penalty table is
built from the caller's host state (touched ids + output counts).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .core import (DegenerateRowError, LogitsShardBlock, SamplingParams, TokenDecision, new_sequence_state,
                   sparse_entries)
from .penalty import update_output_histogram
from .sampler import DecisionPlane, VARIANT_FULL, VARIANT_SHVS
from .shvs import HotVocab
from .transport import AssembledLogitsView, assemble_view, shard_ranges

VARIANT_BASELINE_FULL = "baseline-full"           # service.py:64-68
VARIANT_PARALLEL_FULL = "parallel-full"
VARIANT_OFFLOAD_TRUNCATE = "offload-truncate"
VARIANTS = (VARIANT_BASELINE_FULL, VARIANT_PARALLEL_FULL, VARIANT_OFFLOAD_TRUNCATE, VARIANT_SHVS)


def _params(p) -> SamplingParams:
    """Reference or local SamplingParams -> local (field-identical, core.py:23-34)."""
    if isinstance(p, SamplingParams):
        return p
    return SamplingParams(p.temperature, p.top_k, p.top_p, p.min_p, p.rep_penalty, p.presence_penalty,
                          p.frequency_penalty, p.seed)


def _hot(h, vocab_size: int) -> HotVocab:
    if h is None:
        return HotVocab(vocab_size, np.arange(vocab_size))
    if isinstance(h, HotVocab):
        return h
    return HotVocab(h.vocab_size, np.asarray(h.hot_ids))


class _RowBatch:
    """A reusable device batch for n rows: params, penalty table and uniforms
    reloaded from the caller's host objects on every call."""

    def __init__(self, vocab_size: int, n: int, device):
        self.plane = DecisionPlane(vocab_size, [SamplingParams()] * n, prompts=[[]] * n, device=device,
                                   max_generated=1)
        self.n = n

    def load(self, states, params, draws, seq_ids):
        import torch

        plane = self.plane
        plane.set_params([_params(p) for p in params])
        ent = [sparse_entries(s) for s in states]
        cap = max([len(e[0]) for e in ent] + [1])
        ids = np.zeros((self.n, cap), np.int32)
        cnt = np.zeros((self.n, cap), np.int32)
        ln = np.zeros(self.n, np.int32)
        pl = np.zeros(self.n, np.int32)
        for b, (i, c, np_) in enumerate(ent):
            ids[b, : i.size] = i
            cnt[b, : c.size] = c
            ln[b] = i.size
            pl[b] = np_
        st = plane.state
        dev = plane.device
        st.ids = torch.from_numpy(ids).to(dev)
        st.out_count = torch.from_numpy(cnt).to(dev)
        st.len = torch.from_numpy(ln).to(dev)
        st.prompt_len = torch.from_numpy(pl).to(dev)
        st.cap = st.limit = cap
        st.prompt_max, st.recorded = int(ln.max(initial=0)), 0
        st._native = N.Penalty(st.ids.data_ptr(), st.out_count.data_ptr(), st.len.data_ptr(),
                               st.prompt_len.data_ptr(), cap, plane.vocab_size, 0, 0)
        plane.seq_ids = np.asarray(seq_ids, dtype=np.uint64)
        plane._seq_dev = torch.from_numpy(plane.seq_ids.view(np.int64)).to(dev)
        u = np.asarray(draws, dtype=np.float64).reshape(self.n, -1)
        if u.shape[1] < 3:
            u = np.pad(u, ((0, 0), (0, 3 - u.shape[1])))
        return torch.from_numpy(np.ascontiguousarray(u[:, :3])).to(dev)


class Sampler:
    """service._Sampler on the GPU (service.py:282-420).

    Full variants: truncating rows run the full-vocabulary law
    (_global_filter_draw, token-id ties); rows with neutral filters take the
    hot/tail decomposition with this sampler's hot set (split_decision with
    the producer summary, service.py:392-403), `accepted_hot` cleared.  SHVS:
    split_decision over the hot set with the producer summary of the view."""

    def __init__(self, variant: str, hot, counter=None, device="cuda"):
        if variant not in VARIANTS:
            raise ValueError(f"unknown variant {variant!r}")
        self.variant = variant
        self.hot = hot
        self.counter = counter
        self.device = device
        self._batches = {}
        self._hot_cache = {}

    def _batch(self, vocab_size: int, n: int) -> _RowBatch:
        key = (vocab_size, n)
        if key not in self._batches:
            self._batches[key] = _RowBatch(vocab_size, n, self.device)
        return self._batches[key]

    def sample(self, view, col: int, seq_id: int, state, params, draws, iteration_id: int,
               eos_ids=frozenset()) -> TokenDecision:
        return self.sample_batch(view, [col], [seq_id], [state], [params], [draws], iteration_id, eos_ids)[0]

    def sample_batch(self, view, cols, seq_ids, states, params, draws, iteration_id: int,
                     eos_ids=frozenset()) -> list[TokenDecision]:
        """Decide the view columns `cols` (one GPU call per variant path)."""
        import torch

        v = int(view.vocab_size) if hasattr(view, "vocab_size") else int(states[0].vocab_size)
        n = len(cols)
        rb = self._batch(v, n)
        plane = rb.plane
        u = rb.load(states, params, draws, seq_ids)
        if v not in self._hot_cache:
            self._hot_cache[v] = _hot(self.hot, v)
        hot = self._hot_cache[v]
        plist = [_params(p) for p in params]
        neutral = [p.filters_neutral(v) for p in plist]
        summary = (torch.tensor([view.row_max(c) for c in cols], dtype=torch.float64, device=plane.device),
                   torch.tensor([view.total_expsum(c) for c in cols], dtype=torch.float64, device=plane.device))
        dev = plane.device
        views = view.shard_rows(cols, dev) if hasattr(view, "shard_rows") else \
            AssembledLogitsView(list(view.blocks), view.col_lo, view.col_hi).shard_rows(cols, dev)
        use_split = self.variant == VARIANT_SHVS or (any(neutral) and hot.size < v)
        out = [None] * n
        if self.variant != VARIANT_SHVS and not all(neutral) or not use_split:
            d = plane.sample_sharded(views, iteration_id, uniforms=u, update=False) if len(views) > 1 else \
                plane.sample(views[0].contiguous(), iteration_id, uniforms=u, update=False)
            out = plane.to_decisions(d, iteration_id, eos_ids)
        if use_split:
            plane.set_hot(hot)
            rows = torch.cat(views, dim=1) if len(views) > 1 else views[0]
            perm = hot.device_maps(dev)[0]
            d = plane.sample(rows.index_select(1, perm.long()).contiguous(), iteration_id, variant=VARIANT_SHVS,
                             uniforms=u, summary=summary, update=False)
            dec = plane.to_decisions(d, iteration_id, eos_ids)
            for b in range(n):
                if self.variant == VARIANT_SHVS or neutral[b]:
                    out[b] = dec[b]
                    if self.variant != VARIANT_SHVS:
                        out[b].accepted_hot = False   # flag reserved for the speculative variant
        if self.counter is not None:
            for d in out:
                self.counter.add(hot.size if (self.variant == VARIANT_SHVS and d.accepted_hot) else v)
                self.counter.count_token()
        return out


_Sampler = Sampler


def sample_full(logits_row, state, params, draws, iteration_id: int = 0, eos_ids=frozenset(),
                counter=None) -> TokenDecision:
    """filtering.sample_full (filtering.py:172-201) on the GPU: penalties from
    `state`, full-vocabulary top-k / top-p / min-p, inverse-CDF draw with
    draws[0].  `logits_row` is the [V] wire row (numpy or torch, f32 or bf16;
    f64 values must be f32-representable: the kernels stream f32/bf16)."""
    import torch

    row = _wire_row(logits_row)
    v = row.shape[0]
    blk = LogitsShardBlock(iteration_id, 0, 0, v, row.reshape(v, 1), np.zeros(1), np.ones(1), 1)
    s = Sampler(VARIANT_OFFLOAD_TRUNCATE, None, device=row.device if torch.is_tensor(row) and row.is_cuda else "cuda")
    u = np.atleast_1d(np.asarray(draws, dtype=np.float64))
    d = s.sample(assemble_view([blk], (0, 1)), 0, state.seq_id, state, params, u, iteration_id, eos_ids)
    if counter is not None:
        counter.add(v)
        counter.count_token()
    return d


def _wire_row(x):
    import torch

    if torch.is_tensor(x):
        if x.dtype in (torch.float32, torch.bfloat16):
            return (x if x.is_cuda else x.to("cuda")).reshape(-1)
        x = x.detach().cpu().numpy()
    a = np.asarray(x)
    if a.dtype == np.float32:
        return a.reshape(-1)
    f = a.astype(np.float32)
    if not np.array_equal(f.astype(a.dtype), a, equal_nan=True):
        raise TypeError("logits must be f32 / bf16 wire values (an f64 row must be exactly representable in f32)")
    return f.reshape(-1)


class ShvsRowContext:
    """shvs.ShvsRowContext (shvs.py:171-190): `logits` is a sampling-ready row
    or a penalize-on-gather accessor; row_max / total_expsum cover the full
    vocabulary."""

    def __init__(self, logits, row_max: float, total_expsum: float):
        self.logits, self.row_max, self.total_expsum = logits, float(row_max), float(total_expsum)


def shvs_sample(ctx, hot, params, draws, iteration_id: int = 0, seq_id: int = 0, eos_ids=frozenset(),
                counter=None) -> TokenDecision:
    """shvs.shvs_sample (shvs.py:258-289) on the GPU.

    `ctx.logits` may be (a) a ReadyColumn-style accessor over a view
    (the reference's `service.ReadyColumn`, i.e. penalize-on-gather: its
    view / column / state / params are used directly, penalties applied in
    the kernel), or (b) a sampling-ready row (numpy / torch) whose values are
    f32- or bf16-representable, decided with temperature folded (tau = 1)
    and no penalties — the reference's semantics for a ready row."""
    import torch

    hv = _hot(hot, getattr(hot, "vocab_size", None))
    lg = ctx.logits
    acc = getattr(lg, "_view", None) or getattr(lg, "view", None)
    if acc is not None and not isinstance(lg, np.ndarray) and not torch.is_tensor(lg):
        view, col = acc, getattr(lg, "_col", getattr(lg, "col", 0))
        state, p = getattr(lg, "_state", getattr(lg, "state", None)), getattr(lg, "_params", getattr(lg, "params", None))
        # the context's summary wins over the view's (they agree for engine views)
        blks = [LogitsShardBlock(b.iteration_id, b.rank, b.v_lo, b.v_hi, b.values,
                                 _patched(b.row_max, view.col_lo + col, ctx.row_max),
                                 _patched(b.total_expsum, view.col_lo + col, ctx.total_expsum), b.tp_degree)
                for b in view.blocks]
        v2 = assemble_view(blks, (view.col_lo, view.col_hi))
        d = Sampler(VARIANT_SHVS, hv).sample(v2, col, seq_id, state, p, draws, iteration_id, eos_ids)
    else:
        row = _wire_row(lg)
        v = row.shape[0]
        st = new_sequence_state(seq_id, [], v, max_generated=1)
        p = _params(params)
        p_ready = SamplingParams(1.0, p.top_k, p.top_p, p.min_p, 1.0, 0.0, 0.0, p.seed)
        blk = LogitsShardBlock(iteration_id, 0, 0, v, row.reshape(v, 1), np.array([ctx.row_max]),
                               np.array([ctx.total_expsum]), 1)
        d = Sampler(VARIANT_SHVS, hv).sample(assemble_view([blk], (0, 1)), 0, seq_id, st, p_ready, draws,
                                             iteration_id, eos_ids)
    if counter is not None:
        counter.add(hv.size if d.accepted_hot else hv.vocab_size)
        counter.count_token()
    return d


def _patched(vec, i, val):
    a = np.array(vec.cpu().numpy() if hasattr(vec, "cpu") else vec, dtype=np.float64, copy=True)
    a[i] = val
    return a


def make_shard_blocks(cfg, iteration_id: int, logits, states, params_for, device="cuda") -> list[LogitsShardBlock]:
    """service.make_shard_blocks (service.py:470-504) as a GPU producer.

    `logits`: a CUDA tensor [B, V] (f32 / bf16 wire rows) or the reference's
    (V, B) host matrix (cast to f32 wire values).  The per-row (row_max,
    total_expsum) of the penalized, temperature-scaled rows is computed on
    the device (dp_row_summary); the t = cfg.tp_degree blocks are zero-copy
    vocab slices of the device rows (values = (W, B) Fortran-order views)."""
    import torch

    t = int(getattr(cfg, "tp_degree", cfg) or 1)
    if torch.is_tensor(logits):
        x = logits
    else:
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(logits, dtype=np.float64).astype(np.float32).T))
        x = x.to(device)
    bsz, v = x.shape
    plane = DecisionPlane(v, [_params(params_for(b)) for b in range(bsz)], prompts=[[]] * bsz, device=x.device,
                          max_generated=1)
    rb = _RowBatch.__new__(_RowBatch)
    rb.plane, rb.n = plane, bsz
    rb.load(states, [params_for(b) for b in range(bsz)], np.zeros((bsz, 3)), [s.seq_id for s in states])
    rmax, tot = plane.row_summary(x)
    return [LogitsShardBlock(iteration_id, r, lo, hi, x[:, lo:hi].T, rmax, tot, t)
            for r, (lo, hi) in enumerate(shard_ranges(v, t))]


__all__ = ["Sampler", "_Sampler", "VARIANTS", "VARIANT_BASELINE_FULL", "VARIANT_PARALLEL_FULL",
           "VARIANT_OFFLOAD_TRUNCATE", "VARIANT_SHVS", "sample_full", "shvs_sample", "ShvsRowContext",
           "make_shard_blocks", "update_output_histogram", "DegenerateRowError"]
