"""Per-row timeline of the SHVS tail pass (K1 kTail, DP_TIMELINE build via
DP_LIB): for every rejected row, CTA 0's row start, end of its own stream,
end of the cluster merge + select, end of the final stage (globaltimer).
    DP_LIB=.../timeline.so python tools/micro/timeline_shvs.py [--config c2] [--hot 2048]"""
import argparse, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench
from paper_2512_00719_b200 import DecisionPlane, HotVocab
from paper_2512_00719_b200.synthetic import SyntheticSource

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--hot", type=int, default=2048)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
v, b = cfg["V"], cfg["B"]
prompts = [np.random.default_rng(s).integers(0, v, 32) for s in range(b)]
src = SyntheticSource(v, device="cuda")
hot = HotVocab(v, src.hot_ordering()[: args.hot])
plane = DecisionPlane(v, [bench.row_params(cfg, s) for s in range(b)], prompts=prompts, hot=hot, max_generated=136)
perm = hot.device_maps(plane.device)[0]
dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
xs = [src.generate(i, range(b), dtype=dt, perm=perm, summary_params=plane.params_dev) for i in range(2)]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(6):
    x, summ = xs[i & 1]
    torch.cuda.synchronize()
    ev[0].record()
    d = plane.sample(x, i, variant="shvs", summary=summ, summary_raw=True, debug=True, topk_stride=8, update=False)
    ev[1].record()
    torch.cuda.synchronize()
    fl = d.flags.cpu().numpy()
    rej = np.nonzero(fl & 8)[0]
    tl = d.topk_ready.cpu().numpy()[rej, :8]
    ok = tl[:, 3] > 0
    tl = tl[ok]
    if len(tl) == 0:
        print(f"step {i}: no tail rows"); continue
    t0 = tl[:, 0].min()
    r = (tl[:, :4] - t0) / 1e3
    stream = r[:, 1] - r[:, 0]; sel = r[:, 2] - r[:, 1]; fin = r[:, 3] - r[:, 2]
    print(f"step {i}: call {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us, tail rows {len(tl)}; tail span {r[:, 3].max():.1f} us; "
          f"per row median: start {np.median(r[:, 0]):.1f} stream {np.median(stream):.1f} merge+select {np.median(sel):.1f} "
          f"finish {np.median(fin):.1f} (max {r[:, 3].max():.1f}); starts p90 {np.percentile(r[:, 0], 90):.1f}")
    print(f"   finish phases (us, median): penalties {np.median(tl[:, 5]) / 1e3:.2f} ordering {np.median(tl[:, 6]) / 1e3:.2f} "
          f"draw {np.median(tl[:, 7]) / 1e3:.2f}; rest (uniforms, record, epilogue) "
          f"{np.median(fin - (tl[:, 5] + tl[:, 6] + tl[:, 7]) / 1e3):.2f}")
