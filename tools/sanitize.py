"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): full path, SHVS (whole and split storage), nucleus rows, the
general fallback, penalty update and reset, on a few rows.

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_00719_b200 import DecisionPlane, HotVocab, SamplingParams  # noqa: E402
from paper_2512_00719_b200.synthetic import SyntheticSource  # noqa: E402

v, b = 8192, 12
kinds = [dict(temperature=0.8, top_k=50, top_p=0.9, min_p=0.05, rep_penalty=1.1, presence_penalty=0.5,
              frequency_penalty=0.1), dict(temperature=0.7, top_p=0.9), dict(temperature=9.0),
         dict(temperature=1.0, top_k=1), dict(temperature=6.0, top_p=0.99, rep_penalty=1.2)]
params = [SamplingParams(**kinds[i % len(kinds)], seed=i) for i in range(b)]
prompts = [np.random.default_rng(i).integers(0, v, 24) for i in range(b)]
src = SyntheticSource(v, device="cuda")
plane = DecisionPlane(v, params, prompts=prompts, max_generated=16)
x = src.generate(0, range(b))
for it in range(3):
    plane.sample(x, it)
plane.state.reset()
hot = HotVocab(v, src.hot_ordering()[:2048])
plane_s = DecisionPlane(v, params, prompts=prompts, hot=hot, max_generated=16)
xs = hot.to_hot_first(x).contiguous()
summ = plane_s.producer_summary(xs)
for it in range(2):
    plane_s.sample(xs, it, variant="shvs", summary=summ, summary_raw=True)
    plane_s.sample_split(xs[:, :2048].contiguous(), xs[:, 2048:].contiguous(), 10 + it, summ, summary_raw=True)
plane_k = DecisionPlane(v, params, prompts=prompts, max_generated=16, kernel=2, hot=hot)
plane_k.sample(xs, 3, variant="shvs", summary=summ, summary_raw=True)
# TP-sharded rows: one shard per cluster rank (B < #SMs) and several shards
# per CTA (B >= #SMs), misaligned shard rows
for bt, t in ((12, 4), (160, 8)):
    vt = 8200
    pt = [SamplingParams(**kinds[i % 2 if i % 2 == 0 else 3], seed=i) for i in range(bt)]
    pr = [np.random.default_rng(i).integers(0, vt, 8) for i in range(bt)]
    plane_t = DecisionPlane(vt, pt, prompts=pr, max_generated=16)
    xt = SyntheticSource(vt, device="cuda").generate(0, range(bt))
    w = vt // t
    for it in range(2):
        plane_t.sample_sharded([xt[:, s * w:(s + 1) * w].contiguous() for s in range(t)], it)
        assert plane_t.last_stitched is False
# round 2: K1p (persistent, warp-specialised; forced on a small batch so the
# grid loops), K1h (exact-sort hot pass, every row / nucleus rows), long
# penalty lists (pen_excl instantiation + late penalized keep), the
# producer-fused summary (8-CTA clusters) and the bytes-touched counters
from paper_2512_00719_b200 import _native as N  # noqa: E402

bp = 700
pp = [SamplingParams(**kinds[0 if i % 3 else 3], seed=i) for i in range(bp)]
prp = [np.random.default_rng(i).integers(0, v, 24) for i in range(bp)]
plane_p = DecisionPlane(v, pp, prompts=prp, max_generated=16)
plane_p.plan_flags = N.PLAN_FORCE_PERSIST
plane_p._plan.flags = N.PLAN_FORCE_PERSIST
xp = src.generate(1, range(bp))
for it in range(2):
    plane_p.sample(xp, it, debug=(it == 1))
for flags in (N.PLAN_HOT_SORT_ALL, N.PLAN_HOT_SORT):
    plane_h = DecisionPlane(v, params, prompts=prompts, hot=hot, max_generated=16)
    plane_h.plan_flags = flags
    plane_h.sample(xs, 4, variant="shvs", summary=summ, summary_raw=True, debug=True)
long_prompts = [np.random.default_rng(i).integers(0, v, 600) for i in range(b)]
plane_l = DecisionPlane(v, params, prompts=long_prompts, hot=hot, max_generated=16)
for it in range(2):
    plane_l.sample(x, it)
    plane_l.sample(xs, 20 + it, variant="shvs", summary=summ, summary_raw=True)
xf, sf = src.generate(2, range(b), perm=hot.device_maps(plane_s.device)[0], summary_params=plane_s.params_dev)
plane_s.sample(xf, 30, variant="shvs", summary=sf, summary_raw=True)
torch.cuda.synchronize()
print("sanitize workload done")
