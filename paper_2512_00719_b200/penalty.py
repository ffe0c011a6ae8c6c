"""GPU-resident penalty state (sparse SequenceState) and its update.

The reference keeps a dense V-length histogram + masks per sequence
(core.py:100-141) and updates one slot per token (penalty.py:18-32).  Here a
batch of B sequences owns an ELL table on the device: row b has `len[b]`
entries (token id, output count); the first `prompt_len[b]` entries are the
prompt's unique ids (count 0 until generated).  That is exactly the
reference's `touched_ids` list with `output_hist` restricted to it, so the
penalty arithmetic (penalty.py:66-78) reads only these entries.

Capacity follows the reference's append buffers (core.py:80-97, :144-169):
a row may record up to `max_generated` tokens (default 65,536 =
DEFAULT_MAX_GENERATED, core.py:12) and one more raises OverflowError.  The
device table starts small and grows on demand: the host knows an exact upper
bound of every row's list length without synchronising (prompt uniques +
tokens recorded since the last reset — each decision appends at most one
entry per row), so it doubles the table (one device copy, stream-ordered)
before a call could overflow it, and passes the bound to the kernels
(`dp_penalty_t.max_len`) to size their candidate lists.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .core import DEFAULT_MAX_GENERATED, RangeError, SamplingParams

_INITIAL_SLACK = 256   # device slots beyond the prompt before the first growth


def _stream(device=None):
    import torch

    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _capturing() -> bool:
    import torch

    return torch.cuda.is_available() and torch.cuda.is_current_stream_capturing()


class PenaltyState:
    """Per-row sparse (id, out_count) lists for a batch, on one device."""

    def __init__(self, prompts, vocab_size: int, cap: int | None = None, device="cuda",
                 max_generated: int = DEFAULT_MAX_GENERATED):
        import torch

        self.vocab_size = int(vocab_size)
        self.device = torch.device(device)
        self.max_generated = int(max_generated)
        if self.max_generated < 1:
            raise ValueError("max_generated must be >= 1")
        uniq = []
        for pr in prompts:
            a = np.asarray(list(pr), dtype=np.int64)
            if a.size and (a.min() < 0 or a.max() >= vocab_size):
                raise RangeError(f"prompt token outside [0, {vocab_size})")
            uniq.append(np.unique(a).astype(np.int32))          # ascending: core.py:166-168
        self.batch = len(uniq)
        self.prompt_max = max([u.size for u in uniq], default=0)
        # logical per-row limit (touched_ids capacity, core.py:166): prompt uniques + max_generated, <= V
        self.limit = min(self.prompt_max + self.max_generated, self.vocab_size)
        want = cap if cap is not None else self.prompt_max + min(self.max_generated, _INITIAL_SLACK)
        self.cap = int(max(1, min(int(want), self.limit)))
        ids = np.zeros((self.batch, self.cap), np.int32)
        for b, u in enumerate(uniq):
            ids[b, : u.size] = u
        plen = np.array([u.size for u in uniq], np.int32)
        self.ids = torch.from_numpy(ids).to(self.device)
        self.out_count = torch.zeros((self.batch, self.cap), dtype=torch.int32, device=self.device)
        self.prompt_len = torch.from_numpy(plen).to(self.device)
        self.len = self.prompt_len.clone()
        self.recorded = 0            # tokens recorded per row since the last reset (host-side bound)
        self._replayed = False       # captured graphs may have advanced the device state: bound unknown
        self._native = N.Penalty(self.ids.data_ptr(), self.out_count.data_ptr(), self.len.data_ptr(),
                                 self.prompt_len.data_ptr(), self.cap, self.vocab_size, 0, 0)

    # -- capacity ----------------------------------------------------------
    @property
    def bound(self) -> int:
        """Upper bound of len[b] over the rows (exact worst case, no sync)."""
        return min(self.prompt_max + self.recorded, self.limit)

    def _grow(self, need: int) -> None:
        import torch

        if _capturing():
            raise RuntimeError(f"penalty table must grow to {need} slots during CUDA-graph capture; "
                               f"construct the plane with a larger pen_cap")
        new_cap = min(max(2 * self.cap, need), self.limit)
        ids = torch.zeros((self.batch, new_cap), dtype=torch.int32, device=self.device)
        cnt = torch.zeros((self.batch, new_cap), dtype=torch.int32, device=self.device)
        ids[:, : self.cap] = self.ids
        cnt[:, : self.cap] = self.out_count
        self.ids, self.out_count, self.cap = ids, cnt, new_cap
        self._native.ids = self.ids.data_ptr()
        self._native.out_count = self.out_count.data_ptr()
        self._native.cap = self.cap

    def prepare(self, appending: bool):
        """Native descriptor for the next call.  `appending`: the call records
        one token per row (fused update) — raises OverflowError past
        max_generated like the reference's append buffer (core.py:90-92) and
        grows the table first when the bound could exceed it."""
        if appending:
            if self.recorded >= self.max_generated:
                raise OverflowError("append buffer full")
            need = min(self.prompt_max + self.recorded + 1, self.limit)
            if need > self.cap:
                self._grow(need)
        # graph capture: the captured kernels replay from whatever state the
        # device holds, so they get the table capacity, not the host bound;
        # after a capture the host bound is unknown until the next eager reset
        if _capturing():
            self._replayed = True
        self._native.max_len = 0 if self._replayed else self.bound + (1 if appending else 0)
        return self._native

    def committed(self, appending: bool) -> None:
        if appending:
            self.recorded += 1

    @property
    def native(self) -> N.Penalty:
        return self.prepare(False)

    # -- operations ----------------------------------------------------------
    def update(self, tokens, flags=None) -> None:
        """update_output_histogram for every row (penalty.py:18-32), on device."""
        nat = self.prepare(True)
        N.call("dp_penalty_update", C.byref(nat), C.c_void_p(tokens.data_ptr()), self.batch,
               C.c_void_p(flags.data_ptr() if flags is not None else 0), _stream(self.device))
        self.committed(True)

    def reset(self) -> None:
        """Back to prompt-only state (new_sequence_state, core.py:144-169)."""
        N.call("dp_penalty_reset", C.byref(self.prepare(False)), self.batch, _stream(self.device))
        self.recorded = 0
        if not _capturing():
            self._replayed = False

    def select(self, rows) -> None:
        """Keep only `rows` (int64 device/host index, batch order kept): the
        table side of retiring finished sequences at an iteration boundary
        (service.py:709-714).  Device gathers, no host copy of the table."""
        import torch

        idx = torch.as_tensor(rows, dtype=torch.int64, device=self.device)
        self.ids = self.ids.index_select(0, idx).contiguous()
        self.out_count = self.out_count.index_select(0, idx).contiguous()
        self.len = self.len.index_select(0, idx).contiguous()
        self.prompt_len = self.prompt_len.index_select(0, idx).contiguous()
        self.batch = int(idx.numel())
        self._native.ids = self.ids.data_ptr()
        self._native.out_count = self.out_count.data_ptr()
        self._native.len = self.len.data_ptr()
        self._native.prompt_len = self.prompt_len.data_ptr()

    def rows(self):
        """Host copy: list of (ids, out_counts) per row (debug / parity tests)."""
        n = self.len.cpu().numpy()
        ids, cnt = self.ids.cpu().numpy(), self.out_count.cpu().numpy()
        return [(ids[b, : n[b]].copy(), cnt[b, : n[b]].copy()) for b in range(self.batch)]


def update_output_histogram(state, new_token, flags=None):
    """penalty.update_output_histogram (penalty.py:18-32).

    Two forms: `update_output_histogram(state: SequenceState, new_token: int)`
    records one token in a host `core.SequenceState` exactly as the reference
    (RangeError outside [0, V), OverflowError when an append buffer is full);
    `update_output_histogram(state: PenaltyState, tokens)` records a [B]
    device tensor of tokens, one per row, in the batch's GPU table."""
    if isinstance(state, PenaltyState):
        state.update(new_token, flags)
        return state
    from .core import record_token

    return record_token(state, new_token)


def apply_penalties(logits, state: PenaltyState, params_dev, dtype_code: int):
    """ReadyColumn.full (service.py:236-241) for a [B,V] device batch -> f64 [B,V].

    Materialises the sampling-ready rows; the fused samplers never do this.
    `params_dev` is the device dp_params_t table."""
    import torch

    bsz, v = logits.shape
    out = torch.empty((bsz, v), dtype=torch.float64, device=logits.device)
    N.call("dp_ready_rows", C.c_void_p(logits.data_ptr()), dtype_code, bsz, v, logits.stride(0),
           C.c_void_p(params_dev.data_ptr()), C.byref(state.native), C.c_void_p(out.data_ptr()),
           _stream(logits.device))
    return out


__all__ = ["PenaltyState", "update_output_histogram", "apply_penalties", "SamplingParams"]
