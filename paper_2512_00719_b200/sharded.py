"""Batch-sharded ("sequence-parallel") decisions across GPUs.

The reference splits a batch's rows over m sampler workers with
`partition_batch` (transport.py:133-144, service.py:743-748) and collects the
decisions per row (DecisionLedger / commit_decisions, transport.py:400-433).
Here each rank is one GPU process: it owns the contiguous row block
`partition_batch(B, world)[rank]` with its penalty state, runs the fused
kernels on it, and the only exchange is an all-gather of the int32 token ids
(plus the flag byte) over NCCL / NVLink.  No vocab-axis collective exists:
every row is decided entirely on the rank that owns it, and the uniforms are
keyed by (seed, iteration, seq_id) (rng.py:94-113), so tokens do not depend on
the GPU count.

The gather runs on a side stream so it overlaps the next step's sampling
kernel (the penalty update only needs the local tokens).
"""

from __future__ import annotations

import numpy as np

from .transport import partition_batch


class BatchShard:
    """Row block owned by one rank and the gather of the decided tokens."""

    def __init__(self, batch_size: int, world: int, rank: int):
        if not 0 <= rank < world:
            raise ValueError("rank outside [0, world)")
        self.batch_size, self.world, self.rank = int(batch_size), int(world), int(rank)
        self.bounds = partition_batch(self.batch_size, self.world)
        self.lo, self.hi = self.bounds[rank]
        # partition sizes differ by at most one (larger first): gather padded
        # blocks of the largest size, then drop the pads
        self.block = self.bounds[0][1] - self.bounds[0][0]
        self._keep = np.concatenate([np.arange(j * self.block, j * self.block + (hi - lo))
                                     for j, (lo, hi) in enumerate(self.bounds)]).astype(np.int64)
        self._keep_dev = {}

    @property
    def rows(self) -> int:
        return self.hi - self.lo

    @property
    def seq_ids(self) -> np.ndarray:
        return np.arange(self.lo, self.hi, dtype=np.uint64)

    @property
    def uniform(self) -> bool:
        return self.block * self.world == self.batch_size

    def _keep_index(self, device):
        import torch

        key = str(device)
        if key not in self._keep_dev:
            self._keep_dev[key] = torch.from_numpy(self._keep).to(device)
        return self._keep_dev[key]

    def gather(self, local, group=None, out=None):
        """All-gather the rank's [rows] tensor into the batch-ordered [B] tensor
        on every rank (ncclAllGather over NVLink for CUDA tensors)."""
        import torch
        import torch.distributed as dist

        if local.shape[0] != self.rows:
            raise ValueError(f"rank {self.rank} owns {self.rows} rows, got {local.shape[0]}")
        if self.world == 1:
            if out is not None:
                out.copy_(local)
                return out
            return local
        if self.rows < self.block:
            pad = torch.zeros(self.block, dtype=local.dtype, device=local.device)
            pad[: self.rows] = local
            local = pad
        full = torch.empty(self.block * self.world, dtype=local.dtype, device=local.device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(full, local.contiguous(), group=group)
        else:   # gloo (CPU tests): list form
            parts = list(full.chunk(self.world))
            dist.all_gather(parts, local.contiguous(), group=group)
            full = torch.cat(parts)
        if not self.uniform:
            full = full.index_select(0, self._keep_index(full.device))
        if out is not None:
            out.copy_(full)
            return out
        return full


class NcclTokenGather:
    """The token all-gather through the library's C ABI (dp_allgather_tokens,
    SURVEY §8(b)): one ncclAllGather of int32 ids per iteration on a
    communicator the library creates over NCCL (resolved at run time, the
    copy torch already loaded).  Rank 0 draws the ncclUniqueId
    (dp_nccl_unique_id) and hands it to the other ranks through the
    torch.distributed group; every rank then joins on its own device.
    Stream-ordered and CUDA-graph capturable like any NCCL collective."""

    def __init__(self, shard: BatchShard, device, group=None):
        import ctypes as C

        import torch

        from . import _native as N

        self.shard, self.device = shard, torch.device(device)
        lib = N.load()
        if not lib.dp_nccl_available():
            raise N.NativeUnavailable("dp_allgather_tokens needs libnccl.so.2")
        uid = (C.c_uint8 * 128)()
        if shard.rank == 0:
            N.check(lib.dp_nccl_unique_id(uid), "dp_nccl_unique_id")
        if shard.world > 1:
            import torch.distributed as dist

            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            C.memmove(uid, box[0], 128)
        self._comm = C.c_void_p()
        with torch.cuda.device(self.device):
            N.check(lib.dp_nccl_comm_init(C.byref(self._comm), shard.world, uid, shard.rank), "dp_nccl_comm_init")
            self._pad = torch.zeros(shard.block, dtype=torch.int32, device=self.device)
            self._full = torch.empty(shard.block * shard.world, dtype=torch.int32, device=self.device)
        self._lib, self._N = lib, N

    def __call__(self, local, out=None):
        """[rows] int32 CUDA tensor of this rank -> [B] in batch order (on the
        current stream of the plane's device)."""
        import ctypes as C

        import torch

        sh = self.shard
        if local.shape[0] != sh.rows or local.dtype != torch.int32 or local.device != self.device:
            raise ValueError(f"rank {sh.rank} gathers its {sh.rows} int32 tokens on {self.device}")
        src = local.contiguous()
        if sh.rows < sh.block:
            self._pad[: sh.rows].copy_(src)
            src = self._pad
        st = torch.cuda.current_stream(self.device).cuda_stream
        self._N.check(self._lib.dp_allgather_tokens(C.c_void_p(src.data_ptr()), C.c_void_p(self._full.data_ptr()),
                                                    sh.block, self._comm, C.c_void_p(st)), "dp_allgather_tokens")
        full = self._full if sh.uniform else self._full.index_select(0, sh._keep_index(self.device))
        if out is not None:
            out.copy_(full)
            return out
        return full

    def close(self) -> None:
        if self._comm:
            self._N.check(self._lib.dp_nccl_comm_destroy(self._comm), "dp_nccl_comm_destroy")
            self._comm = None


__all__ = ["BatchShard", "NcclTokenGather"]
