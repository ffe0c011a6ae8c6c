import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2512_00719_b200 import DecisionPlane, SamplingParams
from paper_2512_00719_b200.synthetic import SyntheticSource
cfg = bench.CONFIGS["c2"]; v, b = cfg["V"], cfg["B"]
prompts = [np.random.default_rng(s).integers(0, v, 32) for s in range(b)]
plane = DecisionPlane(v, [SamplingParams(**cfg["params"])] * b, prompts=prompts, max_generated=136)
src = SyntheticSource(v, device="cuda")
x = src.generate(0, range(b))
for i in range(3):
    d = plane.sample(x, i, debug=True)
    torch.cuda.synchronize()
    print("stats", d.stats.cpu().numpy().tolist(), "flags", np.bincount(d.flags.cpu().numpy(), minlength=256).nonzero())
