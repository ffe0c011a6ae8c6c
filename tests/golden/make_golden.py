"""Generate the golden fixtures by running the REFERENCE decision plane itself.

Run here (the reference is importable only in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It drives the reference's own engine pieces exactly as its harness does
(`make_shard_blocks` + `assemble_view` + `_Sampler.sample` +
`update_output_histogram`, harness.py:266-279, service.py:739-772) and freezes
tokens / logprobs / accept flags plus a sha256 of every logits matrix it fed
in.  Logits are regenerated at test time by the oracle's restatement of
SyntheticSource and checked against the stored hash, so fixtures stay small.
`/root/reference` is never read at test time.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

from decplane import rng as ref_rng
from decplane import sizing as ref_sizing
from decplane.core import SamplingParams, new_sequence_state
from decplane.filtering import build_filter_index_map, categorical_draw, subset_softmax
from decplane.penalty import update_output_histogram
from decplane.service import EngineConfig, SyntheticSource, _Sampler, make_shard_blocks
from decplane.shvs import HotVocab, analytic_shvs_distribution
from decplane.transport import assemble_view

HERE = os.path.dirname(os.path.abspath(__file__))

# the heterogeneous parameter mix of SURVEY 8(a') verification (7 kinds)
KINDS = [
    dict(temperature=0.8, top_k=50, top_p=0.9, rep_penalty=1.1),                       # C1 knobs
    dict(temperature=0.8, top_k=1),                                                    # greedy
    dict(temperature=1.5, top_p=0.9),                                                  # top-p only
    dict(temperature=0.7, min_p=0.05),                                                 # min-p only
    dict(),                                                                            # neutral
    dict(temperature=0.8, top_k=20, presence_penalty=-0.4, frequency_penalty=0.2),     # negative presence
    dict(temperature=0.8, top_k=40, top_p=0.95, min_p=0.02, rep_penalty=0.9,
         presence_penalty=0.5, frequency_penalty=0.1),                                 # rep < 1 + all filters
]

C2_PARAMS = dict(temperature=0.8, top_k=50, top_p=0.9, min_p=0.05, rep_penalty=1.1,
                 presence_penalty=0.5, frequency_penalty=0.1)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bf16_round(x):
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def prompts_for(batch, vocab, length=32):
    return [np.random.default_rng(seed=b).integers(0, vocab, size=length).tolist() for b in range(batch)]


def run(vocab, batch, iters, params_of, variant, hot_ids=None, zipf=1.2, noise=0.3, bf16=False,
        prompt_len=32, seed=0):
    """Reference engine loop over `iters` iterations; returns the fixture dict."""
    cfg = EngineConfig(vocab_size=vocab, batch_size=batch, seed=seed, zipf_exponent=zipf,
                       noise_scale=noise)
    src = SyntheticSource(cfg)
    prompts = prompts_for(batch, vocab, prompt_len)
    states = [new_sequence_state(b, prompts[b], vocab) for b in range(batch)]
    hot = HotVocab(vocab, np.arange(vocab) if hot_ids is None else hot_ids)
    sampler = _Sampler(variant, hot)
    toks = np.zeros((iters, batch), np.int64)
    lps = np.zeros((iters, batch), np.float64)
    acc = np.zeros((iters, batch), bool)
    hashes = []
    for it in range(iters):
        mat = src.matrix(it, list(range(batch)))                      # V x B f64
        wire32 = mat.astype(np.float32)
        if bf16:
            wire32 = bf16_round(wire32)
        hashes.append(sha(wire32.T.copy()))                             # [B,V] row-major
        blocks = make_shard_blocks(cfg, it, wire32.astype(np.float64), states,
                                   lambda b: SamplingParams(**params_of(b)))
        view = assemble_view(blocks, (0, batch))
        for b in range(batch):
            p = SamplingParams(**params_of(b))
            draws = ref_rng.pregenerate_slice(p.seed, it, [b])[0]
            d = sampler.sample(view, b, b, states[b], p, draws, it)
            update_output_histogram(states[b], d.token_id)
            toks[it, b], lps[it, b], acc[it, b] = d.token_id, d.logprob, d.accepted_hot
    return dict(tokens=toks, logprobs=lps, accepted=acc, hashes=np.array(hashes),
                prompts=np.array(prompts, np.int64),
                meta=json.dumps(dict(vocab=vocab, batch=batch, iters=iters, zipf=zipf, noise=noise,
                                     bf16=bf16, variant=variant, seed=seed)))


# round-2 cases: the configurations the bench ships (SHVS tail clusters at the
# real vocabulary, long penalty lists, wide top-k, a long heavy-penalty run)
LONG_KINDS = [
    dict(temperature=0.8, top_k=1024, top_p=0.95, rep_penalty=1.1, presence_penalty=0.5, frequency_penalty=0.1),
    dict(temperature=0.9, top_k=5000, min_p=0.01, rep_penalty=1.2),
    dict(temperature=0.8, top_k=50, top_p=0.9, min_p=0.05, rep_penalty=1.1, presence_penalty=0.5,
         frequency_penalty=0.1),
    dict(temperature=0.7, top_p=0.9, rep_penalty=1.3, frequency_penalty=0.2),
]
HEAVY = dict(temperature=0.7, top_k=40, top_p=0.95, rep_penalty=1.3, presence_penalty=1.5, frequency_penalty=1.0)


def main_round2():
    out = {}
    # SHVS at V=152,064 / H=4,096 with odd-ranked hot ids: ~half the rows reject,
    # more than the 74 resident tail clusters -> 4-CTA clusters loop over rows
    src = SyntheticSource(EngineConfig(vocab_size=152064, seed=0))
    hot = src.hot_ordering()[1::2][:4096].copy()
    out["shvs_c2big"] = run(152064, 160, 2, lambda b: dict(C2_PARAMS, seed=b), "shvs", hot_ids=hot)
    out["shvs_c2big"]["hot_ids"] = hot
    # 2-4k unique prompt ids per row, top-k 1024 / 5000, full path and SHVS
    out["long_full"] = run(32000, 16, 3, lambda b: dict(LONG_KINDS[b % 4], seed=b), "offload-truncate",
                           prompt_len=3500)
    src32 = SyntheticSource(EngineConfig(vocab_size=32000, seed=0))
    hot32 = src32.hot_ordering()[:2048].copy()
    out["long_shvs"] = run(32000, 16, 3, lambda b: dict(LONG_KINDS[b % 4], seed=b), "shvs", hot_ids=hot32,
                           prompt_len=3500)
    out["long_shvs"]["hot_ids"] = hot32
    # 300 iterations of heavy presence / frequency penalties on spiky rows: the
    # penalized mass leaves the producer's raw summary (summary_raw regime)
    src8 = SyntheticSource(EngineConfig(vocab_size=8192, seed=0, zipf_exponent=1.6))
    hot8 = src8.hot_ordering()[:1024].copy()
    out["heavy_shvs"] = run(8192, 8, 300, lambda b: dict(HEAVY, seed=b), "shvs", hot_ids=hot8, zipf=1.6)
    out["heavy_shvs"]["hot_ids"] = hot8
    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print(name, d["tokens"].shape, "accept", float(np.mean(d["accepted"])))


def main():
    if "--round2" in sys.argv:
        return main_round2()
    out = {}
    # (1) C1 at full size: V=32000, B=64, tau .8, k 50, p .9, rep 1.1 (BASELINE configs[0])
    c1 = dict(temperature=0.8, top_k=50, top_p=0.9, rep_penalty=1.1)
    out["c1_full"] = run(32000, 64, 3, lambda b: c1, "offload-truncate")
    # (2) heterogeneous V=2048, bf16 ties, 7 kinds, full path and SHVS H=512 (zipf .6 -> rejections)
    het = lambda b: dict(KINDS[b % len(KINDS)], seed=b % 3)
    out["het_full"] = run(2048, 40, 6, het, "offload-truncate", zipf=0.6, bf16=True)
    src = SyntheticSource(EngineConfig(vocab_size=2048, seed=0))
    hot = src.hot_ordering()[:512]
    out["het_shvs"] = run(2048, 40, 6, het, "shvs", hot_ids=hot, zipf=0.6, bf16=True)
    out["het_shvs"]["hot_ids"] = hot
    # (3) SHVS V=4096/H=512: a cold hot set forces rejections, the hot head forces accepts
    src4 = SyntheticSource(EngineConfig(vocab_size=4096, seed=0))
    order = src4.hot_ordering()
    for name, hot_ids in (("shvs_accept", order[:512]), ("shvs_reject", order[::-1][:512].copy())):
        out[name] = run(4096, 16, 3, lambda b: dict(C2_PARAMS, seed=7), "shvs", hot_ids=hot_ids)
        out[name]["hot_ids"] = hot_ids
    # (4) neutral SHVS (exactness mode) on a C3-like shape, small batch
    src3 = SyntheticSource(EngineConfig(vocab_size=8192, seed=0))
    out["shvs_neutral"] = run(8192, 8, 2, lambda b: dict(seed=b), "shvs",
                              hot_ids=src3.hot_ordering()[:1024], zipf=1.2)
    out["shvs_neutral"]["hot_ids"] = src3.hot_ordering()[:1024]
    # (5) real Qwen2.5 vocab with C2 knobs (full penalties + k/p/min-p), small batch
    out["c2_full"] = run(152064, 4, 2, lambda b: C2_PARAMS, "offload-truncate")

    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print(name, d["tokens"].shape, "accept", float(np.mean(d["accepted"])))

    # (6) SPEC hand examples evaluated by the reference
    spec = {}
    fmap, _ = build_filter_index_map(np.array([3.0, 1.0, 2.0]), SamplingParams(top_k=2))
    spec["topk_321_k2"] = sorted(int(i) for i in fmap.forward)
    fmap, _ = build_filter_index_map(np.log(np.array([0.6, 0.3, 0.1])), SamplingParams(top_p=0.7))
    spec["topp_631_p07"] = sorted(int(i) for i in fmap.forward)
    spec["draw_37_029"] = categorical_draw(np.array([0.3, 0.7]), 0.29)
    spec["draw_37_031"] = categorical_draw(np.array([0.3, 0.7]), 0.31)
    law = analytic_shvs_distribution(np.log(np.array([4.0, 2.0, 1.0, 1.0])), HotVocab(4, np.array([0, 1])),
                                     SamplingParams())
    spec["shvs_law_4211"] = law.tolist()
    spec["softmax_10"] = subset_softmax(np.array([1.0, 0.0]), 1.0).tolist()

    # (7) sizing model golden values (sizing.py:78-183)
    rs = np.random.default_rng(0)
    grid = [1, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 128256]
    rows = [np.exp(-1.2 * np.log(np.arange(1, 128257)) + 0.3 * rs.gumbel(size=128256)) for _ in range(8)]
    curve = ref_sizing.estimate_hit_ratio_curve(rows, np.arange(128256), grid)
    pts = [(h, 8.55e-6 + 1.06e-8 * h) for h in (4096, 8192, 16384, 32768)]
    c0, c, resid = ref_sizing.fit_affine_cost(pts)
    model = ref_sizing.SizingModel(c0=c0, c=c, curve=curve, vocab_size=128256)
    spec["sizing"] = dict(grid=grid, alpha_bar=curve.alpha_bar.tolist(), c0=c0, c=c,
                          hot=ref_sizing.optimal_hot_size(model),
                          cost_4096=ref_sizing.expected_cost(4096, model),
                          hot_budget=ref_sizing.optimal_hot_size(model, cycle_budget=6e-4))
    lin = ref_sizing.HitRatioCurve(np.array([1.0, 1000.0]), np.array([0.001, 1.0]))
    spec["sizing_linear"] = ref_sizing.optimal_hot_size(ref_sizing.SizingModel(0.0, 1.0, lin, 1000))
    with open(os.path.join(HERE, "spec_examples.json"), "w") as fh:
        json.dump(spec, fh, indent=1)
    print(json.dumps({k: v for k, v in spec.items() if k != "sizing"}))


if __name__ == "__main__":
    sys.exit(main())
