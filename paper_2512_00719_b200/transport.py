"""Batch partitioning, shard views and the decision wire format (the parts of
decplane/transport.py on the decision path).

* `partition_batch` (transport.py:133-144): contiguous row blocks per worker /
  GPU, larger first.
* `AssembledLogitsView` / `assemble_view` (transport.py:460-557): t vocab
  shards of one iteration stitched into a zero-copy column-range view.  The
  blocks' values may be host numpy arrays or CUDA tensors; the GPU samplers
  read device shards in place (`DecisionPlane.sample_sharded`).
* `DecisionBatch` frames (transport.py:173-184, :258-278): the byte-exact
  little-endian encoding decisions travel back in.  `encode_decisions`
  packs a whole device batch on the GPU (`dp_encode_decisions`, one 17-byte
  record per row) so only the wire payload crosses PCIe.
"""

from __future__ import annotations

import ctypes as C
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

from .core import LogitsShardBlock, TokenDecision

MAGIC = 0x53494D50            # "SIMP"
PROTOCOL_VERSION = 1
HEADER_LEN = 20
FRAME_DECISION_BATCH = 3
_HEADER = struct.Struct("<IHHQI")
FLAG_EOS = 0x01
FLAG_ACCEPTED_HOT = 0x02
FLAG_HAS_LOGPROB = 0x04
RECORD_BYTES = 17             # u64 seq_id, u32 token_id, u8 flags, f32 logprob


class TransportError(Exception):
    pass


class BadMagicError(TransportError):
    pass


class VersionMismatchError(TransportError):
    pass


class TruncatedPayloadError(TransportError):
    pass


class ChecksumError(TransportError):
    pass


class ProtocolError(TransportError):
    pass


class IncompleteIterationError(TransportError):
    pass


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


def shard_ranges(vocab_size: int, t: int) -> list[tuple[int, int]]:
    """Equal vocab slices of t TP ranks (the tiling AssembledLogitsView checks)."""
    if t < 1 or vocab_size % t:
        raise ValueError(f"vocabulary {vocab_size} does not split into {t} equal shards")
    w = vocab_size // t
    return [(r * w, (r + 1) * w) for r in range(t)]


# ---------------------------------------------------------------------------
# shard views


def _is_cuda(x) -> bool:
    return getattr(x, "is_cuda", False)


@dataclass
class AssembledLogitsView:
    """Logical V x |cols| view over t shard blocks, restricted to a column
    range, without copying (transport.py:460-557).  Raises
    IncompleteIterationError for mixed iterations or a broken tiling."""

    blocks: list
    col_lo: int
    col_hi: int

    def __post_init__(self):
        if not self.blocks:
            raise IncompleteIterationError("no shards supplied")
        blocks = sorted(self.blocks, key=lambda b: b.v_lo)
        it, width, lo = blocks[0].iteration_id, blocks[0].v_hi - blocks[0].v_lo, 0
        for b in blocks:
            if b.iteration_id != it:
                raise IncompleteIterationError("shards from mixed iterations")
            if b.v_lo != lo or b.v_hi - b.v_lo != width:
                raise IncompleteIterationError(f"shard tiling broken at [{b.v_lo}, {b.v_hi}), expected lo {lo}")
            lo = b.v_hi
        self.blocks = blocks
        self.width = width
        self.vocab_size = lo
        self.iteration_id = it

    @property
    def num_cols(self) -> int:
        return self.col_hi - self.col_lo

    @property
    def on_device(self) -> bool:
        return _is_cuda(self.blocks[0].values)

    def row_max(self, col: int) -> float:
        return float(self.blocks[0].row_max[self.col_lo + col])

    def total_expsum(self, col: int) -> float:
        return float(self.blocks[0].total_expsum[self.col_lo + col])

    def shard_rows(self, cols, device):
        """Per shard, a [len(cols), W] row-major tensor of the given view
        columns on `device`: views of device blocks (no copy for a contiguous
        column range), one H2D copy per shard for host blocks."""
        import torch

        cols = np.asarray(cols, dtype=np.int64) + self.col_lo
        contiguous = cols.size > 0 and np.array_equal(cols, np.arange(cols[0], cols[0] + cols.size))
        out = []
        for b in self.blocks:
            v = b.values
            if _is_cuda(v):
                rows = v.T                                     # (W, B) F-order -> [B, W] row-major
                rows = rows[int(cols[0]): int(cols[0]) + cols.size] if contiguous else \
                    rows.index_select(0, torch.as_tensor(cols, device=rows.device))
                out.append(rows if rows.device == device else rows.to(device))
            else:
                host = np.ascontiguousarray(np.asarray(v, dtype=np.float32).T[cols])
                out.append(torch.from_numpy(host).to(device, non_blocking=False))
        return out


def assemble_view(shards, col_range: tuple[int, int], expected_t: int | None = None) -> AssembledLogitsView:
    """Stitch an iteration's shard blocks into a zero-copy column-range view."""
    blocks = [getattr(s, "block", s) for s in shards]
    if expected_t is not None and len(blocks) != expected_t:
        raise IncompleteIterationError(f"have {len(blocks)} shards, expected {expected_t}")
    return AssembledLogitsView(blocks=blocks, col_lo=col_range[0], col_hi=col_range[1])


# ---------------------------------------------------------------------------
# decision batches on the wire


@dataclass
class DecisionBatch:
    iteration_id: int
    decisions: list = field(default_factory=list)


def _frame(iteration_id: int, payload: bytes) -> bytes:
    head = _HEADER.pack(MAGIC, PROTOCOL_VERSION, FRAME_DECISION_BATCH, iteration_id, len(payload))
    return head + payload + struct.pack("<I", zlib.crc32(payload) & 0xFFFFFFFF)


def encode_decision_batch(batch: DecisionBatch) -> bytes:
    """encode_frame for a DecisionBatch (transport.py:173-184)."""
    if not batch.decisions:
        return _frame(batch.iteration_id, b"")
    parts = [struct.pack("<I", len(batch.decisions))]
    for d in batch.decisions:
        fl = (FLAG_EOS if d.is_eos else 0) | (FLAG_ACCEPTED_HOT if d.accepted_hot else 0)
        if d.logprob is not None:
            fl |= FLAG_HAS_LOGPROB
        parts.append(struct.pack("<QIB", d.seq_id, d.token_id, fl))
        if d.logprob is not None:
            parts.append(struct.pack("<f", d.logprob))
    return _frame(batch.iteration_id, b"".join(parts))


def decode_decision_batch(data: bytes) -> DecisionBatch:
    """decode_frame for a DecisionBatch frame (transport.py:197-278)."""
    if len(data) < HEADER_LEN:
        raise TruncatedPayloadError("short header")
    magic, version, ftype, iteration_id, n = _HEADER.unpack_from(data, 0)
    if magic != MAGIC:
        raise BadMagicError(f"magic 0x{magic:08X}")
    if version != PROTOCOL_VERSION:
        raise VersionMismatchError(f"frame version {version}, expected {PROTOCOL_VERSION}")
    if ftype != FRAME_DECISION_BATCH:
        raise ProtocolError(f"frame type {ftype} is not a decision batch")
    if len(data) < HEADER_LEN + n + 4:
        raise TruncatedPayloadError(f"frame needs {HEADER_LEN + n + 4} bytes, have {len(data)}")
    payload = data[HEADER_LEN:HEADER_LEN + n]
    (crc,) = struct.unpack_from("<I", data, HEADER_LEN + n)
    if crc != (zlib.crc32(payload) & 0xFFFFFFFF):
        raise ChecksumError("payload CRC32 mismatch")
    if n == 0:
        return DecisionBatch(iteration_id, [])
    if n < 4:
        raise TruncatedPayloadError("payload ends at 0, need 4")
    (count,) = struct.unpack_from("<I", payload, 0)
    off, out = 4, []
    for _ in range(count):
        if off + 13 > n:
            raise TruncatedPayloadError(f"payload ends at {n}, need {off + 13}")
        seq, tok, fl = struct.unpack_from("<QIB", payload, off)
        off += 13
        lp = None
        if fl & FLAG_HAS_LOGPROB:
            if off + 4 > n:
                raise TruncatedPayloadError(f"payload ends at {n}, need {off + 4}")
            (lp,) = struct.unpack_from("<f", payload, off)
            off += 4
        out.append(TokenDecision(iteration_id, seq, tok, bool(fl & FLAG_EOS), bool(fl & FLAG_ACCEPTED_HOT), lp))
    return DecisionBatch(iteration_id, out)


def encode_decisions(plane, d, iteration_id: int, rows=None) -> bytes:
    """DecisionBatch frame for a device batch of decisions: the GPU packs the
    17-byte records (dp_encode_decisions: seq_id, token, flags with eos /
    accepted_hot / has_logprob, f32 logprob), one D2H copy of the payload,
    CRC32 on the host.  `rows` selects live rows (e.g. not retired)."""
    import torch

    from . import _native as N

    n = plane.batch
    with torch.cuda.device(plane.device):
        buf = torch.empty(4 + RECORD_BYTES * n, dtype=torch.uint8, device=plane.device)
        N.call("dp_encode_decisions", C.c_void_p(d.token.data_ptr()), C.c_void_p(d.logprob.data_ptr()),
               C.c_void_p(d.flags.data_ptr()), C.c_void_p(plane._seq_dev.data_ptr()), n,
               C.c_void_p(buf.data_ptr()), C.c_void_p(torch.cuda.current_stream(plane.device).cuda_stream))
        payload = buf.cpu().numpy()
    if rows is not None:
        rows = np.asarray(rows, dtype=np.int64)
        rec = payload[4:].reshape(n, RECORD_BYTES)[rows]
        payload = np.concatenate([np.frombuffer(struct.pack("<I", rows.size), np.uint8), rec.reshape(-1)])
    if payload.size == 4 and n == 0 or (rows is not None and rows.size == 0):
        return _frame(iteration_id, b"")
    return _frame(iteration_id, payload.tobytes())


__all__ = [
    "partition_batch", "shard_ranges", "AssembledLogitsView", "assemble_view", "DecisionBatch",
    "encode_decision_batch", "decode_decision_batch", "encode_decisions", "LogitsShardBlock",
    "TransportError", "BadMagicError", "VersionMismatchError", "TruncatedPayloadError", "ChecksumError",
    "ProtocolError", "IncompleteIterationError",
]
