"""World-size-2 tests of the batch-sharded path on CPU (gloo): row ownership
follows partition_batch (transport.py:133-144), the token all-gather
reassembles batch order, and tokens are invariant to the rank count because
the uniforms are keyed by seq_id (rng.py:94-113; test_rng.py:58-64)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import decplane_oracle as O
from paper_2512_00719_b200.sharded import BatchShard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, batch, vocab, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = BatchShard(batch, world, rank)
        # each rank decides only its rows (oracle stands in for the kernel on CPU)
        src = O.Synthetic(vocab)
        params = O.Params(temperature=0.8, top_k=20, top_p=0.9, rep_penalty=1.1)
        toks = []
        for s in sh.seq_ids.tolist():
            x = src.wire(3, [s])[0]
            st = O.State.new(np.random.default_rng(s).integers(0, vocab, 8), vocab)
            u = O.pregenerate_slice(params.seed, 3, [s])[0]
            toks.append(O.sample_full_row(x, st, params, u).token)
        local = torch.tensor(toks, dtype=torch.int32)
        full = sh.gather(local)
        flags = sh.gather(torch.full((sh.rows,), rank + 1, dtype=torch.uint8))
        q.put((rank, full.numpy().tolist(), flags.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def _run(world, batch, vocab=512):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, vocab, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def _single(batch, vocab=512):
    src = O.Synthetic(vocab)
    params = O.Params(temperature=0.8, top_k=20, top_p=0.9, rep_penalty=1.1)
    toks = []
    for s in range(batch):
        st = O.State.new(np.random.default_rng(s).integers(0, vocab, 8), vocab)
        toks.append(O.sample_full_row(src.wire(3, [s])[0], st, params, O.pregenerate_slice(0, 3, [s])[0]).token)
    return toks


@pytest.mark.parametrize("batch", [8, 7])
def test_gloo_world2_gather_matches_single_process(batch):
    want = _single(batch)
    out = _run(2, batch)
    bounds = BatchShard(batch, 2, 0).bounds
    for rank, full, flags in out:
        assert full == want, f"rank {rank}"
        # flags tell which rank decided each row: contiguous blocks, larger first
        expect = [j + 1 for j, (lo, hi) in enumerate(bounds) for _ in range(lo, hi)]
        assert flags == expect


def test_shard_bounds_follow_partition_batch():
    for b, w in [(8192, 8), (1024, 3), (5, 4), (1, 1)]:
        shards = [BatchShard(b, w, r) for r in range(w)]
        assert shards[0].lo == 0 and shards[-1].hi == b
        for a, c in zip(shards, shards[1:]):
            assert a.hi == c.lo and 0 <= a.rows - c.rows <= 1
        assert np.array_equal(np.concatenate([s.seq_ids for s in shards]), np.arange(b, dtype=np.uint64))


def test_single_rank_gather_is_identity():
    sh = BatchShard(6, 1, 0)
    t = torch.arange(6, dtype=torch.int32)
    assert torch.equal(sh.gather(t), t)
