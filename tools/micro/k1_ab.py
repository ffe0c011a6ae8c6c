"""A-B of the full-path kernels at one config: K1p (persistent) vs K1
(DP_PLAN_NO_PERSIST), graph-replayed (bench-style) and single eager calls.
    python tools/micro/k1_ab.py [--config c2]"""
import argparse, json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench
from paper_2512_00719_b200 import DecisionPlane, _native as N
from paper_2512_00719_b200.synthetic import SyntheticSource

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=20)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
v, b = cfg["V"], cfg["B"]
prompts = [np.random.default_rng(s).integers(0, v, 32) for s in range(b)]
src = SyntheticSource(v, device="cuda")
dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
xs = [src.generate(i, range(b), dtype=dt) for i in range(2)]
out = {}
for name, flags in (("persist", 0), ("per_row", N.PLAN_NO_PERSIST)):
    plane = DecisionPlane(v, [bench.row_params(cfg, s) for s in range(b)], prompts=prompts, max_generated=136)
    plane._plan.flags = flags
    for upd in (False, True):
        ms = bench._graph_ms(lambda i: plane.sample(xs[i & 1], i, update=upd), args.steps)
        out[f"{name}_graph_{'upd' if upd else 'noupd'}_us"] = ms * 1e3
    st = torch.cuda.current_stream()
    evs = []
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        plane.sample(xs[i & 1], 100 + i, update=False)
        e1.record(st)
        torch.cuda.synchronize()
        evs.append(e0.elapsed_time(e1) * 1e3)
    out[f"{name}_eager_us"] = sorted(evs)[len(evs) // 2]
print(json.dumps({k: round(v_, 1) for k, v_ in out.items()}))
