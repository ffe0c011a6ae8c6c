"""Hot vocabulary for speculative hot-vocab sampling (mirror of decplane/shvs.py).

`HotVocab` keeps the reference's contract (hot ids hottest first, inverse map,
ascending tail, prefix `resize`; shvs.py:37-92) and adds the B200 layout: a
*hot-first* position order `perm = [hot ids in hot order | tail ids ascending]`.
A serving stack that permutes its LM-head rows once by `perm` emits logits in
this order for free, so the hot set is one contiguous H-element prefix of every
row and the tail a contiguous suffix — no gathers on the hot path.  With this
layout "lower position" is exactly the reference tie order (hot position on
the hot side, token id on the tail side; shvs.py:71-77, filtering.py:83).
"""

from __future__ import annotations

import numpy as np


class HotVocab:
    """Ordered hot token-id set with forward/inverse maps (shvs.py:37-92)."""

    def __init__(self, vocab_size: int, hot_ids):
        self.vocab_size = int(vocab_size)
        self.hot_ids = np.asarray(hot_ids, dtype=np.int64)
        if self.hot_ids.size < 1:
            raise ValueError("hot set must contain at least one token")
        if self.hot_ids.size > self.vocab_size:
            raise ValueError("hot set larger than vocabulary")
        if self.hot_ids.min() < 0 or self.hot_ids.max() >= self.vocab_size:
            raise ValueError("hot id outside vocabulary")
        if np.unique(self.hot_ids).size != self.hot_ids.size:
            raise ValueError("hot ids must be distinct")
        self.inverse = np.full(self.vocab_size, -1, dtype=np.int64)
        self.inverse[self.hot_ids] = np.arange(self.hot_ids.size)
        self._dev = {}

    @property
    def size(self) -> int:
        return int(self.hot_ids.shape[0])

    @property
    def tail_size(self) -> int:
        return self.vocab_size - self.size

    @property
    def tail_ids(self) -> np.ndarray:
        return np.flatnonzero(self.inverse < 0).astype(np.int64)

    @property
    def perm(self) -> np.ndarray:
        """position -> token id of the hot-first row layout."""
        return np.concatenate([self.hot_ids, self.tail_ids]).astype(np.int32)

    @property
    def inv_perm(self) -> np.ndarray:
        inv = np.empty(self.vocab_size, dtype=np.int32)
        inv[self.perm] = np.arange(self.vocab_size, dtype=np.int32)
        return inv

    def resize(self, hot_size: int) -> "HotVocab":
        """Prefix of the same ordering (shvs.py:89-92)."""
        if hot_size < 1 or hot_size > self.size:
            raise ValueError(f"hot size {hot_size} outside [1, {self.size}]")
        return HotVocab(self.vocab_size, self.hot_ids[:hot_size].copy())

    def device_maps(self, device):
        """(perm, inv_perm) as int32 device tensors, cached per device."""
        import torch

        key = str(device)
        if key not in self._dev:
            self._dev[key] = (torch.from_numpy(self.perm).to(device), torch.from_numpy(self.inv_perm).to(device))
        return self._dev[key]

    def to_hot_first(self, logits):
        """Reorder vocab-order rows [B, V] into hot-first rows (one gather).

        Production stacks avoid this by permuting the LM head once; it is
        provided for callers whose producer emits vocab order."""
        perm, _ = self.device_maps(logits.device)
        return logits.index_select(1, perm.long())


def build_hot_vocab(freq_trace, hot_size: int, vocab_size: int) -> HotVocab:
    """Top `hot_size` ids by trace count, ties toward smaller id (shvs.py:95-112)."""
    if hot_size < 1 or hot_size > vocab_size:
        raise ValueError(f"hot size {hot_size} outside [1, {vocab_size}]")
    counts = np.zeros(vocab_size, dtype=np.int64)
    seen = set()
    for token_id, count in freq_trace:
        t = int(token_id)
        if t < 0 or t >= vocab_size:
            raise ValueError(f"trace token {t} outside [0, {vocab_size})")
        if count < 0:
            raise ValueError("trace counts must be nonnegative")
        if t in seen:
            raise ValueError(f"duplicate trace token {t}")
        seen.add(t)
        counts[t] = int(count)
    # stable sort on -count keeps ascending id among equal counts
    order = np.argsort(-counts, kind="stable")
    return HotVocab(vocab_size, order[:hot_size])


def load_hot_vocab_trace(path) -> list[tuple[int, int]]:
    """`token_id<TAB>count` lines, descending counts, `#` comments (shvs.py:115-132)."""
    trace, prev = [], None
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, 1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split("\t")
            if len(parts) != 2:
                raise ValueError(f"{path}:{lineno}: expected token_id<TAB>count")
            tok, cnt = int(parts[0]), int(parts[1])
            if prev is not None and cnt > prev:
                raise ValueError(f"{path}:{lineno}: counts must be descending")
            prev = cnt
            trace.append((tok, cnt))
    return trace


def save_hot_vocab_trace(path, trace) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("# token_id\tcount\n")
        for tok, cnt in sorted(trace, key=lambda tc: (-tc[1], tc[0])):
            fh.write(f"{tok}\t{cnt}\n")


def acceptance_rate(decisions) -> float:
    """Fraction of decisions that took the hot path (shvs.py:364-369)."""
    decisions = list(decisions)
    if not decisions:
        raise ValueError("empty decision window")
    return sum(1 for d in decisions if d.accepted_hot) / len(decisions)
