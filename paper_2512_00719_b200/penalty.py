"""GPU-resident penalty state (sparse SequenceState) and its update.

The reference keeps a dense V-length histogram + masks per sequence
(core.py:100-141) and updates one slot per token (penalty.py:18-32).  Here a
batch of B sequences owns a fixed-capacity ELL table on the device: row b has
`len[b]` entries (token id, output count); the first `prompt_len[b]` entries are
the prompt's unique ids (count 0 until generated).  That is exactly the
reference's `touched_ids` list with `output_hist` restricted to it, so the
penalty arithmetic (penalty.py:66-78) reads only these entries.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .core import RangeError, SamplingParams


def _stream():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class PenaltyState:
    """Per-row sparse (id, out_count) lists for a batch, on one device."""

    def __init__(self, prompts, vocab_size: int, cap: int | None = None, device="cuda",
                 max_generated: int = 256):
        import torch

        self.vocab_size = int(vocab_size)
        self.device = torch.device(device)
        uniq = []
        for pr in prompts:
            a = np.asarray(list(pr), dtype=np.int64)
            if a.size and (a.min() < 0 or a.max() >= vocab_size):
                raise RangeError(f"prompt token outside [0, {vocab_size})")
            uniq.append(np.unique(a).astype(np.int32))          # ascending: core.py:166-168
        self.batch = len(uniq)
        need = max([u.size for u in uniq], default=0) + int(max_generated)
        self.cap = int(max(cap or 0, need, 1))
        ids = np.zeros((self.batch, self.cap), np.int32)
        for b, u in enumerate(uniq):
            ids[b, : u.size] = u
        plen = np.array([u.size for u in uniq], np.int32)
        self.ids = torch.from_numpy(ids).to(self.device)
        self.out_count = torch.zeros((self.batch, self.cap), dtype=torch.int32, device=self.device)
        self.prompt_len = torch.from_numpy(plen).to(self.device)
        self.len = self.prompt_len.clone()
        self._native = N.Penalty(self.ids.data_ptr(), self.out_count.data_ptr(), self.len.data_ptr(),
                                 self.prompt_len.data_ptr(), self.cap, self.vocab_size)

    @property
    def native(self) -> N.Penalty:
        return self._native

    def update(self, tokens, flags=None) -> None:
        """update_output_histogram for every row (penalty.py:18-32), on device."""
        N.call("dp_penalty_update", C.byref(self._native), C.c_void_p(tokens.data_ptr()), self.batch,
               C.c_void_p(flags.data_ptr() if flags is not None else 0), _stream())

    def reset(self) -> None:
        """Back to prompt-only state (new_sequence_state, core.py:144-169)."""
        N.call("dp_penalty_reset", C.byref(self._native), self.batch, _stream())

    def rows(self):
        """Host copy: list of (ids, out_counts) per row (debug / parity tests)."""
        n = self.len.cpu().numpy()
        ids, cnt = self.ids.cpu().numpy(), self.out_count.cpu().numpy()
        return [(ids[b, : n[b]].copy(), cnt[b, : n[b]].copy()) for b in range(self.batch)]


def update_output_histogram(state: PenaltyState, new_tokens, flags=None) -> PenaltyState:
    """Batched mirror of penalty.update_output_histogram (penalty.py:18-32)."""
    state.update(new_tokens, flags)
    return state


def apply_penalties(logits, state: PenaltyState, params_dev, dtype_code: int):
    """ReadyColumn.full (service.py:236-241) for a [B,V] device batch -> f64 [B,V].

    Materialises the sampling-ready rows; the fused samplers never do this.
    `params_dev` is the device dp_params_t table."""
    import torch

    bsz, v = logits.shape
    out = torch.empty((bsz, v), dtype=torch.float64, device=logits.device)
    N.call("dp_ready_rows", C.c_void_p(logits.data_ptr()), dtype_code, bsz, v, logits.stride(0),
           C.c_void_p(params_dev.data_ptr()), C.byref(state.native), C.c_void_p(out.data_ptr()), _stream())
    return out


__all__ = ["PenaltyState", "update_output_histogram", "apply_penalties", "SamplingParams"]
