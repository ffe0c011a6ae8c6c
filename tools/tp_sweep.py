"""TP-sharded ingestion at C2: the full-vocabulary step over t vocab shards
read in place (dp_sample_full_sharded, one t-CTA cluster per row) against the
contiguous-row step and against stitching the shards first (torch.cat + the
contiguous step).  Llama-3 V=128,256, B=1,024 fp32, C2 knobs; CUDA-event graph
replays, inputs alternate between two batches (> L2).

    python tools/tp_sweep.py [--out profiles/r1/tp_sweep.json]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2512_00719_b200 import DecisionPlane  # noqa: E402
from paper_2512_00719_b200.synthetic import SyntheticSource  # noqa: E402


def timed(fn, steps):
    g = bench._graph(fn, steps)
    torch.cuda.synchronize()
    return bench._timed(g) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1", "tp_sweep.json"))
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    v, b = cfg["V"], cfg["B"]
    dev = torch.device("cuda")
    prompts = [np.random.default_rng(s).integers(0, v, bench.PROMPT_LEN) for s in range(b)]
    params = [bench.row_params(cfg, s) for s in range(b)]
    src = SyntheticSource(v, device=dev)
    bufs = [src.generate(i, range(b)) for i in range(2)]
    plane = DecisionPlane(v, params, prompts=prompts, device=dev, max_generated=bench.RESET_EVERY + 8)

    def contiguous(i):
        plane.sample(bufs[i & 1], i)

    rows = [dict(t=1, mode="contiguous")]
    for i in range(3):
        contiguous(i)
    rows[0]["ms"] = timed(contiguous, args.steps)
    for t in (2, 4, 8):
        w = v // t
        shards = [[x[:, s * w:(s + 1) * w].contiguous() for s in range(t)] for x in bufs]

        def sharded(i):
            plane.sample_sharded(shards[i & 1], i)

        def stitched(i):
            plane.sample(torch.cat(shards[i & 1], dim=1), i)

        plane.state.reset()
        for i in range(3):
            sharded(i)
        assert plane.last_stitched is False
        rows.append(dict(t=t, mode="in-place", ms=timed(sharded, args.steps)))
        plane.state.reset()
        for i in range(3):
            stitched(i)
        rows.append(dict(t=t, mode="stitched", ms=timed(stitched, args.steps)))
        del shards
    for r in rows:
        r["tokens_per_s"] = b / (r["ms"] / 1e3)
        print(f"t={r['t']} {r['mode']:10s} {r['ms'] * 1e3:8.1f} us  {r['tokens_per_s'] / 1e6:6.2f} M tok/s",
              flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(dict(config=cfg["name"], V=v, B=b, params=cfg["params"], rows=rows), fh, indent=1)


if __name__ == "__main__":
    main()
