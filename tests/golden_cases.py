"""Shared helpers: rebuild the reference-run golden cases from their fixtures.

The fixture stores the reference's outputs and a sha256 of each logits matrix;
the logits themselves are regenerated with the oracle's SyntheticSource
restatement and must hash identically (so the oracle generator is pinned too).
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from oracle import decplane_oracle as O

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

KINDS = [
    dict(temperature=0.8, top_k=50, top_p=0.9, rep_penalty=1.1),
    dict(temperature=0.8, top_k=1),
    dict(temperature=1.5, top_p=0.9),
    dict(temperature=0.7, min_p=0.05),
    dict(),
    dict(temperature=0.8, top_k=20, presence_penalty=-0.4, frequency_penalty=0.2),
    dict(temperature=0.8, top_k=40, top_p=0.95, min_p=0.02, rep_penalty=0.9,
         presence_penalty=0.5, frequency_penalty=0.1),
]
C1 = dict(temperature=0.8, top_k=50, top_p=0.9, rep_penalty=1.1)
C2 = dict(temperature=0.8, top_k=50, top_p=0.9, min_p=0.05, rep_penalty=1.1,
          presence_penalty=0.5, frequency_penalty=0.1)

LONG_KINDS = [
    dict(temperature=0.8, top_k=1024, top_p=0.95, rep_penalty=1.1, presence_penalty=0.5, frequency_penalty=0.1),
    dict(temperature=0.9, top_k=5000, min_p=0.01, rep_penalty=1.2),
    dict(temperature=0.8, top_k=50, top_p=0.9, min_p=0.05, rep_penalty=1.1, presence_penalty=0.5,
         frequency_penalty=0.1),
    dict(temperature=0.7, top_p=0.9, rep_penalty=1.3, frequency_penalty=0.2),
]
HEAVY = dict(temperature=0.7, top_k=40, top_p=0.95, rep_penalty=1.3, presence_penalty=1.5, frequency_penalty=1.0)

CASES = {
    "c1_full": lambda b: C1,
    "het_full": lambda b: dict(KINDS[b % len(KINDS)], seed=b % 3),
    "het_shvs": lambda b: dict(KINDS[b % len(KINDS)], seed=b % 3),
    "shvs_accept": lambda b: dict(C2, seed=7),
    "shvs_reject": lambda b: dict(C2, seed=7),
    "shvs_neutral": lambda b: dict(seed=b),
    "c2_full": lambda b: C2,
    # round 2: the shapes and regimes the bench ships (make_golden.py --round2)
    "shvs_c2big": lambda b: dict(C2, seed=b),
    "long_full": lambda b: dict(LONG_KINDS[b % 4], seed=b),
    "long_shvs": lambda b: dict(LONG_KINDS[b % 4], seed=b),
    "heavy_shvs": lambda b: dict(HEAVY, seed=b),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class Case:
    def __init__(self, name: str):
        d = np.load(os.path.join(HERE, f"{name}.npz"))
        self.name = name
        self.meta = json.loads(str(d["meta"]))
        self.tokens = d["tokens"]
        self.logprobs = d["logprobs"]
        self.accepted = d["accepted"]
        self.hashes = [str(h) for h in d["hashes"]]
        self.prompts = d["prompts"]
        self.hot_ids = d["hot_ids"] if "hot_ids" in d else None
        self.params_of = CASES[name]
        m = self.meta
        self.vocab, self.batch, self.iters = m["vocab"], m["batch"], m["iters"]
        self.path = "shvs" if m["variant"] == "shvs" else "full"
        self._src = O.Synthetic(self.vocab, seed=m["seed"], zipf=m["zipf"], noise=m["noise"])

    def params(self):
        return [O.Params(**self.params_of(b)) for b in range(self.batch)]

    def logits(self, it: int) -> np.ndarray:
        x = self._src.wire(it, range(self.batch))
        if self.meta["bf16"]:
            x = O.bf16_round(x)
        return x

    def states(self):
        return [O.State.new(self.prompts[b], self.vocab) for b in range(self.batch)]


ALL = list(CASES)
