"""Per-phase clock profile of the sampler kernels (debug stats slots).

    python tools/phase_prof.py --variant shvs|full [--config c2] [--hot 16384]
Prints stats[0..23] averaged per decided row plus the kernel span from
globaltimer (stats[21] min start, stats[22] max end).
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_00719_b200 import DecisionPlane, HotVocab  # noqa: E402
from paper_2512_00719_b200.synthetic import SyntheticSource  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--variant", default="shvs")
ap.add_argument("--hot", type=int, default=4096)
ap.add_argument("--kernel", type=int, default=0)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--grow", type=int, default=0, help="decide (and record) this many steps first: longer penalty lists")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
v, b = cfg["V"], cfg["B"]
prompts = [np.random.default_rng(s).integers(0, v, cfg.get("prompt_len", 32)) for s in range(b)]
src = SyntheticSource(v, device="cuda")
hot = HotVocab(v, src.hot_ordering()[: args.hot]) if args.variant == "shvs" else None
plane = DecisionPlane(v, [bench.row_params(cfg, s) for s in range(b)], prompts=prompts, hot=hot,
                      kernel=args.kernel, max_generated=136)
perm = hot.device_maps(plane.device)[0] if hot is not None else None
dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
x = src.generate(0, range(b), dtype=dt, perm=perm)
summ = plane.producer_summary(x) if args.variant == "shvs" else None
for i in range(args.grow):
    if args.variant == "shvs":
        plane.sample(x, 1000 + i, variant="shvs", summary=summ, summary_raw=True)
    else:
        plane.sample(x, 1000 + i)
for i in range(args.steps):
    d = plane._outputs(True, 0)
    d.stats.zero_()
    d.stats[21] = 2 ** 62
    if args.variant == "shvs":
        d = plane.sample(x, i, variant="shvs", summary=summ, summary_raw=True, debug=True)
    else:
        d = plane.sample(x, i, debug=True)
    torch.cuda.synchronize()
    st = d.stats.cpu().numpy().astype(np.float64)
    rows = max(st[0], 1)
    span = (st[22] - st[21]) / 1e3 if st[21] < 2 ** 61 else float("nan")
    acc = float(np.mean((d.flags.cpu().numpy() & 2) != 0))
    print(f"step {i}: rows {int(st[0])} restreams {int(st[1])} cand/row {st[3] / rows:.1f} accept {acc:.4f} "
          f"span_us {span:.1f}")
    print("   cycles/row by slot:", {j: round(st[j] / rows) for j in range(4, 24) if st[j]})
    nrej = int(((d.flags.cpu().numpy() & 8) != 0).sum())
    print(f"   rejected rows {nrej}; topk slots per rejected row:",
          {j: round(st[j] / max(nrej, 1)) for j in range(12, 21) if st[j]})
