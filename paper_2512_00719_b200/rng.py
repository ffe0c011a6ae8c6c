"""Counter-based uniforms on the device (mirror of decplane/rng.py).

Every uniform is a pure function of (seed, iteration, seq_id, draw index)
through the SplitMix64 chain of rng.py:39-57, evaluated bit-exactly with u64
integer ops in the kernels; the samplers derive their three draws per row
(u_hot, u_accept, u_tail; rng.py:25-26) inline, so this module is only needed
when callers want the uniforms themselves.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import SamplingParams, params_bytes

DOMAIN_SAMPLER = 0
DOMAIN_LOGITS = 1
DRAWS_PER_SEQUENCE = 3


@dataclass(frozen=True)
class DrawKey:
    seed: int
    iteration_id: int
    seq_id: int
    draw_index: int


def pregenerate_slice(seed: int, iteration_id: int, seq_range, device="cuda"):
    """[n, 3] f64 device tensor, bit-identical to rng.pregenerate_slice (rng.py:94-113)."""
    import torch

    seqs = np.asarray(list(seq_range), dtype=np.uint64)
    n = seqs.shape[0]
    out = torch.empty((n, 3), dtype=torch.float64, device=device)
    if n == 0:
        return out
    raw = np.frombuffer(params_bytes([SamplingParams(seed=seed)] * n), dtype=np.uint8).copy()
    params = torch.from_numpy(raw).to(device)
    seq = torch.from_numpy(seqs.view(np.int64)).to(device)
    N.call("dp_uniforms", C.c_void_p(params.data_ptr()), C.c_void_p(seq.data_ptr()), n, int(iteration_id),
           C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    return out


def draw(key: DrawKey, device="cuda") -> float:
    """Single uniform for a draw key (rng.py:60-63), evaluated on device."""
    return float(pregenerate_slice(key.seed, key.iteration_id, [key.seq_id], device)[0, key.draw_index])
