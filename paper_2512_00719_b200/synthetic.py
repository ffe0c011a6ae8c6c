"""Synthetic logits producer on the GPU (SyntheticSource, service.py:429-467).

logits[b, v] = -s * ln(rank(v) + 1) + noise * Gumbel(u), u keyed by
(seed, DOMAIN_LOGITS, iteration, seq_id, v) through the counter RNG
(rng.py:116-120) and clamped at 2^-60; rank order = stable argsort of keyed
uniforms on domain 7 (synthetic_hot_ordering).  The f64 base table is built
once on the host (setup, V entries); every element is generated on device and
written as fp32 or bf16, optionally directly in hot-first position order.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

_MASK64 = (1 << 64) - 1
_DOMAIN_PERMUTE = 7


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _mix_int(z: int) -> int:
    z &= _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def hot_ordering(seed: int, vocab_size: int) -> np.ndarray:
    """synthetic_hot_ordering (service.py:429-436): token ids, hottest first."""
    h = _mix_int((seed & _MASK64) ^ 0x9E3779B97F4A7C15)
    h = _mix_int(h ^ _DOMAIN_PERMUTE)
    h = _mix_int(h ^ 0)
    hv = _mix(np.full(vocab_size, h, dtype=np.uint64) ^ np.uint64(0))
    hv = _mix(hv ^ np.arange(vocab_size, dtype=np.uint64))
    u = (hv >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
    return np.argsort(u, kind="stable").astype(np.int64)


class SyntheticSource:
    """Zipf-ranked logits with keyed Gumbel noise, generated on device."""

    def __init__(self, vocab_size: int, seed: int = 0, zipf_exponent: float = 1.2, noise_scale: float = 0.3,
                 device="cuda"):
        import torch

        self.vocab_size, self.seed, self.noise = int(vocab_size), int(seed), float(noise_scale)
        self.device = torch.device(device)
        self.rank_to_token = hot_ordering(seed, vocab_size)
        base = np.empty(vocab_size, dtype=np.float64)
        base[self.rank_to_token] = -zipf_exponent * np.log(np.arange(1, vocab_size + 1, dtype=np.float64))
        self._base = torch.from_numpy(base).to(self.device)

    def hot_ordering(self) -> np.ndarray:
        return self.rank_to_token

    def generate(self, iteration: int, seq_ids, dtype=None, perm=None, out=None, summary_params=None,
                 summary_out=None):
        """[B, V] logits for (iteration, seq_ids); perm (int32 device tensor,
        position -> id) writes hot-first rows.  With `summary_params` (the
        plane's device dp_params_t array, for tau) the same pass also emits
        the producer's penalty-free row summary and the call returns
        (logits, (row_max, total_expsum)) — make_shard_blocks' contract
        (service.py:470-504) with the summary computed while the logits are
        written (into `summary_out` = (row_max, total_expsum) f64 [B] when
        given)."""
        import torch

        dtype = torch.float32 if dtype is None else dtype
        if isinstance(seq_ids, torch.Tensor) and seq_ids.is_cuda:   # device ids: capturable in a CUDA graph
            seq = seq_ids
        else:
            seq = torch.as_tensor(np.asarray(seq_ids, dtype=np.uint64).view(np.int64), device=self.device)
        bsz = seq.shape[0]
        if out is None:
            out = torch.empty((bsz, self.vocab_size), dtype=dtype, device=self.device)
        code = N.DP_F32 if out.dtype == torch.float32 else N.DP_BF16
        rmax = tot = None
        if summary_params is not None and summary_out is not None:
            rmax, tot = summary_out
        elif summary_params is not None:
            rmax = torch.empty(bsz, dtype=torch.float64, device=self.device)
            tot = torch.empty(bsz, dtype=torch.float64, device=self.device)
        ptr = lambda t: C.c_void_p(0 if t is None else t.data_ptr())   # noqa: E731
        N.call("dp_synth_logits", C.c_void_p(self._base.data_ptr()), self.noise, self.seed, int(iteration),
               C.c_void_p(seq.data_ptr()), bsz, self.vocab_size, out.stride(0), ptr(perm), code,
               C.c_void_p(out.data_ptr()), ptr(summary_params), ptr(rmax), ptr(tot),
               C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        return out if summary_params is None else (out, (rmax, tot))
