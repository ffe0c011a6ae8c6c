"""Per-row timeline of the K1 kernel (DP_TIMELINE build via DP_LIB):
row start, end of stream, end of select/merge, end of finish, SM id.
    DP_LIB=.../timeline.so python tools/micro/timeline.py [--config c2]"""
import argparse, os, sys, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench
from paper_2512_00719_b200 import DecisionPlane
from paper_2512_00719_b200.synthetic import SyntheticSource

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--out", default=None)
ap.add_argument("--grow", type=int, default=0, help="decide (and record) this many steps first: longer penalty lists")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
v, b = cfg["V"], cfg["B"]
prompts = [np.random.default_rng(s).integers(0, v, 32) for s in range(b)]
src = SyntheticSource(v, device="cuda")
plane = DecisionPlane(v, [bench.row_params(cfg, s) for s in range(b)], prompts=prompts, max_generated=136)
dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
xs = [src.generate(i, range(b), dtype=dt) for i in range(2)]
for i in range(args.grow):
    plane.sample(xs[i & 1], 1000 + i)
for i in range(4):
    d = plane.sample(xs[i & 1], i, debug=True, topk_stride=8, update=False)
torch.cuda.synchronize()
tl = d.topk_ready.cpu().numpy()[:, :5]
valid = tl[:, 3] > 0
t0 = tl[valid, 0].min()
r = (tl[:, :4] - t0) / 1e3
sm = np.nan_to_num(tl[:, 4]).astype(int)
stream = r[:, 1] - r[:, 0]; sel = r[:, 2] - r[:, 1]; fin = r[:, 3] - r[:, 2]
print(f"span {np.nanmax(r[:, 3]):.1f} us; per row: stream {np.nanmedian(stream):.1f} (p10 {np.nanpercentile(stream,10):.1f} p90 {np.nanpercentile(stream,90):.1f}) "
      f"select {np.nanmedian(sel):.1f} finish {np.nanmedian(fin):.1f} us")
if cfg.get("mix"):   # per row kind (bench.MIX index, penalties on / off)
    kind = np.arange(b) % len(bench.MIX)
    pen = (np.arange(b) // len(bench.MIX)) % 2
    ok = tl[:, 3] > 0
    for kk in range(len(bench.MIX)):
        for pp in (0, 1):
            m = ok & (kind == kk) & (pen == pp)
            if m.any():
                print(f"  kind {kk} {bench.MIX[kk]} pen {pp}: rows {m.sum()} stream {np.nanmedian(stream[m]):.1f} "
                      f"select {np.nanmedian(sel[m]):.1f} finish {np.nanmedian(fin[m]):.1f} (p90 {np.nanpercentile(fin[m], 90):.1f}) us")
    print(f"  rows without a K1 timeline (other kernels): {(~ok).sum()}")
order = np.argsort(r[:, 0])
starts = np.sort(r[valid, 0])
print("row starts (us) deciles:", np.round(np.percentile(starts, np.arange(0, 101, 10)), 1).tolist())
print("row ends (us) deciles:", np.round(np.percentile(r[valid, 3], np.arange(0, 101, 10)), 1).tolist())
# how many rows are streaming / finishing at each microsecond
grid = np.arange(0, np.nanmax(r[:, 3]) + 1, max(2.0, np.nanmax(r[:, 3]) / 200))
streaming = [(np.sum((r[:, 0] <= t) & (r[:, 1] > t))) for t in grid]
finishing = [(np.sum((r[:, 1] <= t) & (r[:, 3] > t))) for t in grid]
print("t(us) streaming finishing:")
for t, s_, f_ in zip(grid, streaming, finishing):
    print(f"  {t:6.1f} {s_:4d} {f_:4d}")
if args.out:
    np.save(args.out, tl)
