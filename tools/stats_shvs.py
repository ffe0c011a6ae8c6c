import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2512_00719_b200 import DecisionPlane, SamplingParams, HotVocab
from paper_2512_00719_b200.synthetic import SyntheticSource
cfg = bench.CONFIGS["c2"]; v, b = cfg["V"], cfg["B"]
H = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
prompts = [np.random.default_rng(s).integers(0, v, 32) for s in range(b)]
src = SyntheticSource(v, device="cuda")
hot = HotVocab(v, src.hot_ordering()[:H])
plane = DecisionPlane(v, [SamplingParams(**cfg["params"])] * b, prompts=prompts, hot=hot, max_generated=136)
x = src.generate(0, range(b), perm=hot.device_maps(plane.device)[0])
summ = plane.producer_summary(x)
names = {0:"rows",3:"cands",12:"fin:hash+pen",13:"fin:raw",14:"fin:sort",15:"fin:tail",16:"fin:draw",17:"setup",18:"stream",19:"select",20:"merge"}
for i in range(3):
    d = plane.sample(x, i, variant="shvs", summary=summ, summary_raw=True, debug=True, update=False)
    torch.cuda.synchronize()
st = d.stats.cpu().numpy()
rows = max(1, st[0]) if st[0] else b
print({names.get(k, k): (int(st[k]) // 3 // b if k not in (0, 3) else int(st[k])) for k in range(24) if st[k]})
