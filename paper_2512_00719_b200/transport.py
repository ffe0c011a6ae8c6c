"""Batch-axis partitioning (transport.partition_batch, transport.py:133-144)."""

from __future__ import annotations


def partition_batch(batch_size: int, workers: int) -> list[tuple[int, int]]:
    """Contiguous row ranges whose sizes differ by at most one, larger first."""
    if batch_size < 1 or workers < 1:
        raise ValueError("batch size and worker count must be >= 1")
    base, rem = divmod(batch_size, workers)
    bounds, lo = [], 0
    for j in range(workers):
        hi = lo + base + (j < rem)
        bounds.append((lo, hi))
        lo = hi
    return bounds
