"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it.  The product path (`paper_2512_00719_b200`) never imports
anything under `oracle/` and fails loudly when its CUDA library is missing.

It is a numpy restatement of the reference decision law
(`/root/reference/pkg/src/decplane`, "decplane" 0.1.0, pure Python + numpy;
numpy is the only third-party arithmetic and is not vendored — this container
has numpy 2.3.5, the reference pins only `numpy>=1.24`,
`pkg/pyproject.toml:10-12`).  Every function cites the reference file:line it
follows and uses the same numpy primitives in the same order, so on identical
inputs it is bit-identical to the reference.  That claim is pinned by
`tests/test_oracle_golden.py` against

* the reference's own golden vectors (`pkg/tests/data/rng_probes.txt`,
  copied to `tests/golden/rng_probes.txt`), and
* fixtures produced by running the reference itself in this container
  (`tests/golden/make_golden.py`, outputs `tests/golden/*.npz`).

Besides tokens, the oracle reports *boundary margins*: how close each draw,
accept test and top-p / min-p cut came to flipping.  The parity tests exempt
(and log) rows whose margin is below 1e-6, as the north-star tolerance allows.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# counter RNG  (rng.py:15-120)

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15          # rng.py:16
MULT_A = 0xBF58476D1CE4E5B9          # rng.py:17
MULT_B = 0x94D049BB133111EB          # rng.py:18
DOMAIN_SAMPLER = 0                   # rng.py:21
DOMAIN_LOGITS = 1                    # rng.py:22
DOMAIN_PERMUTE = 7                   # service.py:426
DRAWS_PER_SEQUENCE = 3               # rng.py:26


def mix(z: int) -> int:
    """SplitMix64 finalizer (rng.py:39-43)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * MULT_A) & MASK64
    z = ((z ^ (z >> 27)) * MULT_B) & MASK64
    return z ^ (z >> 31)


def hash_fields(seed: int, domain: int, iteration: int, seq: int, counter: int) -> int:
    """Five-field absorption chain (rng.py:46-52)."""
    h = mix((seed & MASK64) ^ GOLDEN)
    h = mix(h ^ (domain & MASK64))
    h = mix(h ^ (iteration & MASK64))
    h = mix(h ^ (seq & MASK64))
    h = mix(h ^ (counter & MASK64))
    return h


def to_unit(h: int) -> float:
    """Top 53 bits -> [0,1) (rng.py:55-57)."""
    return (h >> 11) * (1.0 / (1 << 53))


def draw(seed: int, iteration: int, seq: int, idx: int) -> float:
    """rng.draw (rng.py:60-63)."""
    return to_unit(hash_fields(seed, DOMAIN_SAMPLER, iteration, seq, idx))


def _mix_array(z: np.ndarray) -> np.ndarray:
    # rng.py:71-74
    z = (z ^ (z >> np.uint64(30))) * np.uint64(MULT_A)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(MULT_B)
    return z ^ (z >> np.uint64(31))


def _hash_array(seed, domain, iteration, seqs: np.ndarray, counters: np.ndarray) -> np.ndarray:
    # rng.py:77-87: scalar absorption up to the iteration, vector rounds after
    h = mix((seed & MASK64) ^ GOLDEN)
    h = mix(h ^ (domain & MASK64))
    h = mix(h ^ (iteration & MASK64))
    hv = np.full(seqs.shape, h, dtype=np.uint64)
    hv = _mix_array(hv ^ seqs.astype(np.uint64))
    return _mix_array(hv ^ counters.astype(np.uint64))


def _unit_array(h: np.ndarray) -> np.ndarray:
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))   # rng.py:90-91


def pregenerate_slice(seed: int, iteration: int, seq_ids) -> np.ndarray:
    """[n,3] uniforms (u_hot, u_accept, u_tail) per sequence (rng.py:94-113)."""
    seq = np.asarray(list(seq_ids), dtype=np.uint64)
    n = seq.shape[0]
    seqs = np.repeat(seq, DRAWS_PER_SEQUENCE)
    idxs = np.tile(np.arange(DRAWS_PER_SEQUENCE, dtype=np.uint64), n)
    return _unit_array(_hash_array(seed, DOMAIN_SAMPLER, iteration, seqs, idxs)).reshape(n, 3)


def keyed_uniform_block(seed: int, domain: int, iteration: int, seq: int, count: int) -> np.ndarray:
    """rng.keyed_uniform_block (rng.py:116-120)."""
    counters = np.arange(count, dtype=np.uint64)
    seqs = np.full(count, seq, dtype=np.uint64)
    return _unit_array(_hash_array(seed, domain, iteration, seqs, counters))


def uniforms_per_row(seeds, iteration: int, seq_ids) -> np.ndarray:
    """Per-row params.seed (service.py:760-761) -> [B,3]."""
    out = np.empty((len(seq_ids), 3), dtype=np.float64)
    for b, (s, q) in enumerate(zip(seeds, seq_ids)):
        out[b] = pregenerate_slice(int(s), iteration, [int(q)])[0]
    return out


# ---------------------------------------------------------------------------
# params + per-sequence penalty state  (core.py:23-169, penalty.py:18-78)


@dataclass
class Params:
    """core.SamplingParams field for field (core.py:23-34)."""

    temperature: float = 1.0
    top_k: int = 0
    top_p: float = 1.0
    min_p: float = 0.0
    rep_penalty: float = 1.0
    presence_penalty: float = 0.0
    frequency_penalty: float = 0.0
    seed: int = 0

    def penalties_neutral(self) -> bool:          # core.py:36-41
        return self.rep_penalty == 1.0 and self.presence_penalty == 0.0 and self.frequency_penalty == 0.0

    def filters_neutral(self, n: int) -> bool:    # core.py:43-45
        k_off = self.top_k == 0 or self.top_k >= n
        return k_off and self.top_p >= 1.0 and self.min_p == 0.0


@dataclass
class State:
    """Dense restatement of SequenceState (core.py:100-169)."""

    vocab_size: int
    prompt_mask: np.ndarray
    output_hist: np.ndarray
    output_ids: list = field(default_factory=list)
    touched_ids: list = field(default_factory=list)

    @classmethod
    def new(cls, prompt, vocab_size: int) -> "State":
        prompt = np.asarray(list(prompt), dtype=np.int64)
        hist = np.bincount(prompt, minlength=vocab_size)
        mask = hist > 0
        st = cls(vocab_size, mask, np.zeros(vocab_size, dtype=np.int32))
        st.touched_ids = [int(t) for t in np.flatnonzero(mask)]          # core.py:166-168
        return st

    def update(self, tok: int) -> None:
        """update_output_histogram (penalty.py:18-32)."""
        tok = int(tok)
        if tok < 0 or tok >= self.vocab_size:
            raise ValueError("token out of range")
        was = self.output_hist[tok] > 0
        self.output_hist[tok] += 1
        if not was:
            self.output_ids.append(tok)
            if not self.prompt_mask[tok]:
                self.touched_ids.append(tok)

    def entries(self):
        """Sparse (id, out_count) list = the device ELL row (touched set)."""
        return [(t, int(self.output_hist[t])) for t in self.touched_ids]


def penalize(x: np.ndarray, st: State, p: Params) -> np.ndarray:
    """apply_penalties (penalty.py:66-78): divisive rep on touched ids, then
    two sequential subtractions on output ids, all f64."""
    out = np.array(x, dtype=np.float64, copy=True)
    if p.penalties_neutral():
        return out
    if p.rep_penalty != 1.0:                                          # penalty.py:35-44
        ids = np.asarray(st.touched_ids, dtype=np.int64)
        out[ids] = out[ids] / p.rep_penalty
    if p.presence_penalty != 0.0 or p.frequency_penalty != 0.0:
        ids = np.asarray(st.output_ids, dtype=np.int64)
        if ids.size:
            vals = out[ids]
            vals = vals - p.presence_penalty
            vals = vals - p.frequency_penalty * st.output_hist[ids].astype(np.float64)
            out[ids] = vals
    return out


def ready_row(x_wire: np.ndarray, st: State, p: Params) -> np.ndarray:
    """ReadyColumn.full: penalize(f64(wire f32)) then /tau (service.py:236-241)."""
    r = penalize(np.asarray(x_wire, dtype=np.float32).astype(np.float64), st, p)
    if p.temperature != 1.0:
        r = r / p.temperature
    return r


# ---------------------------------------------------------------------------
# truncation-first filter + inverse-CDF draw  (filtering.py:38-162)


def top_k_ids(z: np.ndarray, k: int) -> np.ndarray:
    """_top_k_ids (filtering.py:38-58): argpartition + exact boundary-tie repair."""
    n = z.shape[0]
    if k >= n:
        return np.arange(n, dtype=np.int64)
    split = np.argpartition(z, n - k)
    selected = split[n - k:]
    boundary = z[split[n - k]]
    if int((z == boundary).sum()) == int((z[selected] == boundary).sum()):
        return np.asarray(selected, dtype=np.int64)
    greater = np.flatnonzero(z > boundary)
    ties = np.flatnonzero(z == boundary)[: k - greater.shape[0]]
    return np.concatenate([greater, ties]).astype(np.int64)


@dataclass
class Draw:
    index: int            # position inside the domain
    logprob: float
    kept: int             # surviving candidates after all filters
    margin: float         # min distance of any decision to its flip point
    topk_set: np.ndarray  # domain positions of the top-k stage (sorted asc), or None


def filter_draw(values: np.ndarray, p: Params, u: float, want_topk: bool = False) -> Draw:
    """_filter_core + filtered_draw + categorical_draw at tau_eff = 1
    (filtering.py:61-105, :124-140, :158-162; service.py:391, shvs.py:192-196)."""
    z = np.asarray(values, dtype=np.float64)
    n = z.shape[0]
    if n < 1:
        raise ValueError("empty source domain")
    k_on = p.top_k != 0 and p.top_k < n
    ids = top_k_ids(z, max(1, p.top_k)) if k_on else np.arange(n, dtype=np.int64)
    topk_set = np.sort(ids) if (want_topk and k_on) else None
    order = np.lexsort((ids, -z[ids]))                                # filtering.py:83
    ids = ids[order]
    kept = ids.shape[0]
    margin = math.inf
    w_kept = None
    if p.top_p < 1.0 or p.min_p > 0.0:
        scaled = z[ids] / 1.0
        w = np.exp(scaled - scaled[0])                                # filtering.py:90
        if p.top_p < 1.0:
            cum = np.cumsum(w)
            threshold = p.top_p * cum[-1]
            kp = int(np.searchsorted(cum, threshold, side="left")) + 1  # filtering.py:95
            kept = min(kept, kp)
            lo, hi = max(0, kp - 2), min(cum.shape[0], kp + 1)
            margin = min(margin, float(np.min(np.abs(cum[lo:hi] - threshold))) / cum[-1])
        if p.min_p > 0.0:
            floor = p.min_p * w[0]
            km = int(np.searchsorted(-w, -floor, side="right"))       # filtering.py:98
            kept = min(kept, km)
            lo, hi = max(0, km - 1), min(w.shape[0], km + 1)
            margin = min(margin, float(np.min(np.abs(w[lo:hi] - floor))))
        kept = max(1, kept)
        ids = ids[:kept]
        w_kept = w[:kept]
    truncated = z[ids]
    w = w_kept if w_kept is not None else np.exp((truncated - truncated[0]) / 1.0)   # filtering.py:137-138
    probs = w / w.sum()                                               # filtering.py:139
    cdf = np.cumsum(probs)                                            # filtering.py:160
    j = min(int(np.searchsorted(cdf, u, side="right")), cdf.shape[0] - 1)
    lo, hi = max(0, j - 1), min(cdf.shape[0], j + 1)
    margin = min(margin, float(np.min(np.abs(cdf[lo:hi] - u))))
    if j == cdf.shape[0] - 1 and cdf.shape[0] > 1:
        margin = min(margin, abs(float(cdf[-2]) - u))
    return Draw(int(ids[j]), float(np.log(probs[j])), int(kept), margin, topk_set)


class DegenerateRow(ValueError):
    pass


@dataclass
class Decision:
    token: int
    logprob: float
    accepted_hot: bool
    alpha: float
    margin: float
    ready: np.ndarray | None = None
    topk_set: np.ndarray | None = None     # token ids of the top-k stage (full path)


def sample_full_row(x_wire: np.ndarray, st: State, p: Params, u: np.ndarray,
                    keep_debug: bool = False) -> Decision:
    """Engine full path with token-id tie order everywhere, i.e.
    _Sampler("offload-truncate", HotVocab(V, arange(V))) (service.py:381-409):
    truncating rows -> _global_filter_draw(ready, tau=1, u_hot); neutral rows ->
    split_decision with the identity hot set, which is the same law with u_hot
    (alpha = 1, tail empty)."""
    ready = ready_row(x_wire, st, p)
    if not np.isfinite(ready.max()):
        raise DegenerateRow("row max is not finite")
    d = filter_draw(ready, p, float(u[0]), want_topk=keep_debug)
    return Decision(d.index, d.logprob, False, 1.0, d.margin,
                    ready if keep_debug else None, d.topk_set)


def row_summary(ready: np.ndarray):
    """shvs.row_summary (shvs.py:157-168)."""
    z = np.asarray(ready, dtype=np.float64)
    rm = float(z.max())
    if not np.isfinite(rm):
        raise DegenerateRow("row max is not finite")
    return rm, float(np.exp(z - rm).sum())


def sample_shvs_row(x_wire_by_id: np.ndarray, st: State, p: Params, u: np.ndarray,
                    hot_ids: np.ndarray, tail_ids: np.ndarray,
                    summary=None) -> Decision:
    """split_decision (shvs.py:198-255) as driven by _Sampler SHVS
    (service.py:354-380).  x_wire_by_id is the row in token-id order; the
    producer summary is row_summary over the full ready row
    (service.py:484-489) unless given."""
    ready = ready_row(x_wire_by_id, st, p)
    m, s_total = summary if summary is not None else row_summary(ready)
    hot_vals = ready[hot_ids]
    w_hot = np.exp(np.asarray(hot_vals, dtype=np.float64) - m)       # shvs.py:143-145
    hot_sum = float(w_hot.sum())
    tail_n = tail_ids.shape[0]
    if tail_n == 0:
        alpha = 1.0
    else:                                                             # shvs.py:148-154
        if not np.isfinite(s_total) or s_total <= 0.0:
            raise DegenerateRow("total weight sum unusable")
        alpha = min(hot_sum / s_total, 1.0)
    margin = math.inf
    if hot_sum > 0.0:
        d = filter_draw(hot_vals, p, float(u[0]))
        margin = d.margin
        if tail_n:
            margin = min(margin, abs(float(u[1]) - alpha))
        if float(u[1]) <= alpha:
            return Decision(int(hot_ids[d.index]), d.logprob, True, alpha, margin)
    elif tail_n == 0:
        raise DegenerateRow("hot set covers the vocabulary but has zero mass")
    tail_vals = ready[tail_ids]
    d = filter_draw(tail_vals, p, float(u[2]))
    if not np.isfinite(np.max(tail_vals)):                           # shvs.py:246-247
        raise DegenerateRow("tail has no finite candidate")
    return Decision(int(tail_ids[d.index]), d.logprob, False, alpha, min(margin, d.margin))


# ---------------------------------------------------------------------------
# hot vocabulary  (shvs.py:37-132)


def tail_ids_of(hot_ids: np.ndarray, vocab_size: int) -> np.ndarray:
    mask = np.ones(vocab_size, dtype=bool)
    mask[np.asarray(hot_ids, dtype=np.int64)] = False
    return np.flatnonzero(mask).astype(np.int64)                     # shvs.py:71-77


def build_hot_vocab(freq_trace, hot_size: int, vocab_size: int) -> np.ndarray:
    """shvs.build_hot_vocab (shvs.py:95-112): count desc, id asc."""
    counts = np.zeros(vocab_size, dtype=np.int64)
    for t, c in freq_trace:
        counts[int(t)] = int(c)
    order = np.lexsort((np.arange(vocab_size), -counts))
    return order[:hot_size].astype(np.int64)


# ---------------------------------------------------------------------------
# synthetic logits  (service.py:429-467)


def synthetic_hot_ordering(seed: int, vocab_size: int) -> np.ndarray:
    u = keyed_uniform_block(seed, DOMAIN_PERMUTE, 0, 0, vocab_size)
    return np.argsort(u, kind="stable").astype(np.int64)


class Synthetic:
    """SyntheticSource: base[rank] = -s*ln(rank+1), Gumbel noise per element."""

    def __init__(self, vocab_size: int, seed: int = 0, zipf: float = 1.2, noise: float = 0.3):
        self.v, self.seed, self.noise = vocab_size, seed, noise
        self.rank_to_token = synthetic_hot_ordering(seed, vocab_size)
        base_by_rank = -zipf * np.log(np.arange(1, vocab_size + 1, dtype=np.float64))
        self.base = np.empty(vocab_size, dtype=np.float64)
        self.base[self.rank_to_token] = base_by_rank

    def column(self, iteration: int, seq: int) -> np.ndarray:
        u = keyed_uniform_block(self.seed, DOMAIN_LOGITS, iteration, seq, self.v)
        u = np.maximum(u, 2.0 ** -60)
        return self.base + self.noise * (-np.log(-np.log(u)))

    def wire(self, iteration: int, seq_ids) -> np.ndarray:
        """[B,V] row-major f32 wire logits (make_shard_blocks cast, service.py:481)."""
        return np.stack([self.column(iteration, s) for s in seq_ids]).astype(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 -> bf16 -> f32 (what a bf16 LM head emits)."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


# ---------------------------------------------------------------------------
# batch drivers


def sample_batch(x_wire: np.ndarray, states, params, seq_ids, iteration: int,
                 path: str = "full", hot_ids=None, uniforms=None, update: bool = True):
    """Run one iteration of the decision law over a [B,V] batch (row-major,
    token-id order).  Mirrors Engine._run_worker_iteration (service.py:752-766):
    uniforms per row from params.seed, decision, then penalty update."""
    bsz, v = x_wire.shape
    if uniforms is None:
        uniforms = uniforms_per_row([pp.seed for pp in params], iteration, seq_ids)
    tail = tail_ids_of(hot_ids, v) if path == "shvs" else None
    out = []
    for b in range(bsz):
        if path == "full":
            d = sample_full_row(x_wire[b], states[b], params[b], uniforms[b])
        else:
            d = sample_shvs_row(x_wire[b], states[b], params[b], uniforms[b], hot_ids, tail)
        if update:
            states[b].update(d.token)
        out.append(d)
    return out


def partition_batch(batch_size: int, workers: int):
    """transport.partition_batch (transport.py:133-144)."""
    base, rem = divmod(batch_size, workers)
    out, lo = [], 0
    for j in range(workers):
        size = base + (1 if j < rem else 0)
        out.append((lo, lo + size))
        lo += size
    return out
