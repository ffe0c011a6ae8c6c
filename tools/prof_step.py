"""Minimal driver for ncu captures: build a workload the way bench.py does and
run a few sampling steps (no graph, no timing).

    python tools/prof_step.py --config c2 --variant full|shvs --steps 3
"""

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2512_00719_b200 import DecisionPlane, HotVocab, SamplingParams  # noqa: E402
from paper_2512_00719_b200.synthetic import SyntheticSource  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--variant", default="full")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--hot", type=int, default=4096)
    ap.add_argument("--bf16", action="store_true")
    ap.add_argument("--plan-flags", type=int, default=0)
    ap.add_argument("--extra", default="", help="comma list: fused (producer-fused summary), curve (K6), "
                                                "summary (K2 penalized)")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    v, b = cfg["V"], cfg["B"]
    prompts = [np.random.default_rng(s).integers(0, v, cfg.get("prompt_len", 32)) for s in range(b)]
    src = SyntheticSource(v, device="cuda")
    hot = HotVocab(v, src.hot_ordering()[: args.hot]) if args.variant == "shvs" else None
    params = [bench.row_params(cfg, s) for s in range(b)]
    plane = DecisionPlane(v, params, prompts=prompts, hot=hot, split=args.split, kernel=args.kernel,
                          max_generated=136)
    plane.plan_flags = args.plan_flags
    perm = hot.device_maps(plane.device)[0] if hot is not None else None
    dt = torch.bfloat16 if (args.bf16 or cfg["dtype"] == "bf16") else torch.float32
    extra = set(filter(None, args.extra.split(",")))
    if "fused" in extra:
        x, summ = src.generate(0, range(b), dtype=dt, perm=perm, summary_params=plane.params_dev)
    else:
        x = src.generate(0, range(b), dtype=dt, perm=perm)
        summ = plane.producer_summary(x) if args.variant == "shvs" else None
    if "curve" in extra and hot is not None:
        plane.hot_mass_curve(x, [256, 512, 1024, 2048, 4096, 8192, 16384, 32768])
    if "summary" in extra:
        plane.row_summary(x, inv_perm=hot.device_maps(plane.device)[1] if hot is not None else None)
    for i in range(args.steps):
        if args.variant == "shvs":
            plane.sample(x, i, variant="shvs", summary=summ, summary_raw=True)
        else:
            plane.sample(x, i)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
