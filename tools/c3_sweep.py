"""C3: SHVS hot-vocabulary size sweep vs the full-vocabulary path, with the
measured acceptance and the paper's sizing model (BASELINE configs[2]).

    python tools/c3_sweep.py [--out profiles/r1/c3_sweep.json]

Llama-3 vocab V=128,256, B=1,024 fp32 synthetic logits (SyntheticSource
formula), C2 knobs (rep/pres/freq penalties, tau .8, top-k 50, top-p .9,
min-p .05).  For every H in the grid:
  * alpha_bar(H): mean per-row hot mass from the K6 kernel
    (sizing.estimate_hit_ratio_curve, sizing.py:78-100);
  * T_hot(H): device time of the hot path alone (every row accepted: the
    summary is scaled so alpha = 1) — the reference's measure_hot_path_cost
    (harness.py:350-376) on the GPU;
  * T(H): device time of the real SHVS step (hot pass + tail pass for the
    rejected rows + penalty update) and its acceptance rate.
(c0, c) are fitted on (H, T_hot(H)/B) (sizing.fit_affine_cost), the model
cost F(H) = c0 + c (alpha_bar H + (1 - alpha_bar)(V - H)) (Eq. 10) is
minimised by sizing.optimal_hot_size, and the full-vocabulary step is timed
for comparison.  All times are CUDA-event graph replays, inputs alternate
between two batches (> L2).
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
from paper_2512_00719_b200 import DecisionPlane, HotVocab  # noqa: E402
from paper_2512_00719_b200 import sizing  # noqa: E402
from paper_2512_00719_b200.synthetic import SyntheticSource  # noqa: E402


def timed_steps(fn, steps):
    g = bench._graph(fn, steps)
    torch.cuda.synchronize()
    return bench._timed(g) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--grid", default="1024,2048,4096,8192,12288,16384,24576,32768")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1", "c3_sweep.json"))
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    v, b = cfg["V"], cfg["B"]
    grid = [int(h) for h in args.grid.split(",")]
    dev = torch.device("cuda")
    prompts = [np.random.default_rng(s).integers(0, v, bench.PROMPT_LEN) for s in range(b)]
    params = [bench.row_params(cfg, s) for s in range(b)]
    src = SyntheticSource(v, device=dev)
    order = src.hot_ordering()

    # alpha_bar(H) on hot-first rows ordered by the largest hot set
    plane_c = DecisionPlane(v, params, prompts=prompts, hot=HotVocab(v, order[: max(grid)]), device=dev,
                            max_generated=bench.RESET_EVERY + 8)
    perm = plane_c.hot.device_maps(dev)[0]
    xs = src.generate(0, range(b), perm=perm)
    # the hit-ratio curve also needs its low end (the model interpolates it)
    cgrid = sorted(set([1, 16, 64, 256, 512] + grid))
    curve_rows = plane_c.hot_mass_curve(xs, cgrid).cpu().numpy()
    cbar = curve_rows.mean(axis=0)
    abar = np.array([cbar[cgrid.index(h)] for h in grid])
    del xs

    # full-vocabulary path
    plane_f = DecisionPlane(v, params, prompts=prompts, device=dev, max_generated=bench.RESET_EVERY + 8)
    bufs = [src.generate(i, range(b)) for i in range(2)]

    def full_step(i):
        d = plane_f.sample(bufs[i & 1], i, update=False)
        plane_f.state.update(d.token, d.flags)

    for i in range(3):
        full_step(i)
    t_full = timed_steps(full_step, args.steps)
    del bufs

    rows = []
    for h in grid:
        hot = HotVocab(v, order[:h])
        plane = DecisionPlane(v, params, prompts=prompts, hot=hot, device=dev, max_generated=bench.RESET_EVERY + 8)
        perm = hot.device_maps(dev)[0]
        hb = [src.generate(i, range(b), perm=perm) for i in range(2)]
        summ = [plane.producer_summary(x) for x in hb]
        # alpha = 1 for every row: the hot path alone (no rejections)
        forced = [(s[0], s[1] * 1e-30) for s in summ]

        def hot_only(i):
            d = plane.sample(hb[i & 1], i, variant="shvs", summary=forced[i & 1], summary_raw=False, update=False)
            plane.state.update(d.token, d.flags)

        def shvs_step(i):
            d = plane.sample(hb[i & 1], i, variant="shvs", summary=summ[i & 1], summary_raw=True, update=False)
            plane.state.update(d.token, d.flags)

        for i in range(3):
            hot_only(i)
        t_hot = timed_steps(hot_only, args.steps)
        plane.state.reset()
        for i in range(3):
            shvs_step(i)
        t_shvs = timed_steps(shvs_step, args.steps)
        d = plane.sample(hb[0], 0, variant="shvs", summary=summ[0], summary_raw=True, update=False)
        acc = float(np.mean((d.flags.cpu().numpy() & 0x02) != 0))
        rows.append(dict(H=h, alpha_bar=float(abar[grid.index(h)]), accept=acc, t_hot_ms=t_hot, t_shvs_ms=t_shvs,
                         tokens_per_s=b / (t_shvs / 1e3)))
        print(f"H={h:6d} alpha_bar={abar[grid.index(h)]:.4f} accept={acc:.4f} hot-only {t_hot * 1e3:7.1f} us "
              f"SHVS step {t_shvs * 1e3:7.1f} us", flush=True)
        del hb, plane

    # the paper's sizing model on the GPU-measured costs (seconds per row)
    c0, c, resid = sizing.fit_affine_cost([(r["H"], r["t_hot_ms"] / 1e3 / b) for r in rows])
    curve = sizing.HitRatioCurve(np.array(cgrid, np.float64), np.maximum.accumulate(cbar))
    model = sizing.SizingModel(c0=max(c0, 0.0), c=max(c, 1e-15), curve=curve, vocab_size=v)
    h_star = sizing.optimal_hot_size(model)
    best = min(rows, key=lambda r: r["t_shvs_ms"])
    out = dict(config=cfg["name"], V=v, B=b, params=cfg["params"], grid=grid, full_step_ms=t_full,
               curve=dict(grid=cgrid, alpha_bar=cbar.tolist()),
               full_tokens_per_s=b / (t_full / 1e3), sweep=rows, fit=dict(c0=c0, c=c, max_residual=resid),
               model_hot_size=h_star, model_expected_cost_s=float(sizing.expected_cost(h_star, model)),
               measured_best_H=best["H"], measured_best_ms=best["t_shvs_ms"],
               note="c0, c fitted on the GPU hot-path time per row (sizing.fit_affine_cost); H* = "
                    "sizing.optimal_hot_size over [1, V]; the tail pass on the GPU runs rejected rows in "
                    "parallel, so the model's per-token tail cost is an upper bound")
    print(json.dumps({k: out[k] for k in ("full_step_ms", "fit", "model_hot_size", "measured_best_H")}))
    print(sizing.sizing_report(model, h_star))
    # the model's pick, measured
    if h_star not in grid:
        print(f"model H* = {h_star} is not on the timing grid; nearest measured: "
              f"{min(grid, key=lambda g: abs(g - h_star))}")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
