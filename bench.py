"""Benchmark of the B200 decision plane (driver contract: one JSON line).

Default workload (N=1): BASELINE configs[1] — Qwen2.5 vocab V=152,064,
B=1,024 fp32 logits, repetition/presence/frequency penalties + top-k/top-p/
min-p, synthetic logits from the SyntheticSource formula generated on device.
A step = one pass of the hot path over the batch: dp_sample_full (fused
penalties -> tau -> top-k -> top-p -> min-p -> draw, with the penalty-state
update fused into the deciding kernel) — the reference's timed unit,
sample + update_output_histogram (harness.py:274-279).  With N GPUs each rank
runs BASELINE configs[3] (C4: V=151,936, B=8,192 split over the ranks by
partition_batch, strong scaling) and the step ends with the token-id
all-gather over NCCL, inside the timed region.  `--gpus N` without a launcher
re-execs itself under torch.distributed.run (one process per GPU).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                    [--config c2|c1|c3|c4|c5] [--variant full|shvs]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2_PARAMS = dict(temperature=0.8, top_k=50, top_p=0.9, min_p=0.05, rep_penalty=1.1,
                 presence_penalty=0.5, frequency_penalty=0.1)
C1_PARAMS = dict(temperature=0.8, top_k=50, top_p=0.9, rep_penalty=1.1)
CONFIGS = {
    "c1": dict(V=32000, B=64, dtype="f32", params=C1_PARAMS, name="llama2-32k-b64"),
    "c2": dict(V=152064, B=1024, dtype="f32", params=C2_PARAMS, name="qwen2.5-152k-b1024"),
    "c3": dict(V=128256, B=1024, dtype="f32", params=C2_PARAMS, name="llama3-128k-b1024-shvs-sweep"),
    "c4": dict(V=151936, B=8192, dtype="f32", params=C2_PARAMS, name="qwen3-151936-b8192", strong=True),
    "c5": dict(V=152064, B=16384, dtype="bf16", params=C2_PARAMS, name="qwen2.5-152k-b16384-bf16-mix",
               mix=True),
    # diagnostics (not BASELINE configs): C2 shape, one filter kind per run
    "c2p": dict(V=152064, B=1024, dtype="f32", params=dict(temperature=0.8, top_p=0.9), name="c2-top-p-only"),
    "c2m": dict(V=152064, B=1024, dtype="f32", params=dict(temperature=0.8, min_p=0.05), name="c2-min-p-only"),
    "c2n": dict(V=152064, B=1024, dtype="f32", params=dict(temperature=0.8), name="c2-neutral"),
    # C2 with 2,048-token prompts per row (~2,000 unique penalized ids: the
    # realistic serving penalty state)
    "c2long": dict(V=152064, B=1024, dtype="f32", params=C2_PARAMS, name="c2-2048-token-prompts", prompt_len=2048),
}
METRIC = "sampled tokens/s at V=152k, B=1024; achieved HBM GB/s vs B200 peak"
PROMPT_LEN = 32
RESET_EVERY = 128  # harness.py:266-269


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-exec this command under
    torch.distributed.run with N local ranks (one process per GPU, rendezvous
    on 127.0.0.1).  NCCL's INIT lines (rank / nranks of every communicator)
    go to stderr so the rank count can be checked."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:   # timed region shorter than the sampling period: one query right after it
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=10).stdout
                parts = [p.strip() for p in out.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
                    self.after = True
            except Exception:
                pass
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": reasons, "samples": len(self.samples)}
        if getattr(self, "after", False):
            out["note"] = "timed region shorter than the 50 ms sampling period: queried right after it"
        return out


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of the reference algorithm, on host cores)

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    """The unmodified reference package installed by pip --target baseline/_ref."""
    return os.path.isdir(os.path.join(REF_DIR, "decplane"))


def _ref_worker(args):
    """The reference's own sampler loop (harness.py:255-279): per iteration the
    producer make_shard_blocks (service.py:470-504, untimed like the harness),
    then per row _Sampler("offload-truncate").sample + update_output_histogram
    (timed).  Returns (rows decided, seconds inside the timed calls)."""
    x, prompts, params, seq0, seconds = args
    sys.path.insert(0, REF_DIR)
    from decplane import rng as ref_rng
    from decplane.core import SamplingParams as RP, new_sequence_state
    from decplane.penalty import update_output_histogram as ref_update
    from decplane.service import EngineConfig, _Sampler, make_shard_blocks
    from decplane.shvs import HotVocab as RHot
    from decplane.transport import assemble_view

    n, v = x.shape
    cfg = EngineConfig(vocab_size=v, batch_size=n)
    states = [new_sequence_state(seq0 + b, list(prompts[b]), v) for b in range(n)]
    p = RP(**params)
    sampler = _Sampler("offload-truncate", RHot(v, np.arange(v)))
    col_major = np.ascontiguousarray(x.T).astype(np.float64)     # (V, B) wire layout, core.py:186-199
    rows, busy, it, t_start = 0, 0.0, 0, time.perf_counter()
    while True:
        blocks = make_shard_blocks(cfg, it, col_major, states, lambda b: p)
        view = assemble_view(blocks, (0, n))
        for b in range(n):
            draws = ref_rng.pregenerate_slice(p.seed, it, [seq0 + b])[0]
            t0 = time.perf_counter()
            d = sampler.sample(view, b, seq0 + b, states[b], p, draws, it)
            ref_update(states[b], d.token_id)
            busy += time.perf_counter() - t0
            rows += 1
        it += 1
        if time.perf_counter() - t_start >= seconds:
            break
    return rows, busy


def _port_worker(args):
    """Fallback when baseline/_ref is absent: the oracle port of the same law."""
    x, prompts, params, seq0, seconds = args
    from oracle import decplane_oracle as O

    v = x.shape[1]
    states = [O.State.new(p, v) for p in prompts]
    pp = O.Params(**params)
    t0 = time.perf_counter()
    n, it = 0, 0
    while True:
        for b in range(x.shape[0]):
            u = O.pregenerate_slice(pp.seed, it, [seq0 + b])[0]
            d = O.sample_full_row(x[b], states[b], pp, u)
            states[b].update(d.token)
            n += 1
        it += 1
        if time.perf_counter() - t0 >= seconds:
            break
    return n, time.perf_counter() - t0


class CpuBaseline:
    """The reference CPU sampler timed on this host's cores: one process per
    core (the reference's m-sampler design, service.py:584-589, without the
    GIL), rows split by partition_batch (transport.py:133-144), one process
    pool reused across measurements.  Uses the unmodified reference from
    baseline/_ref when installed ("reference"), else the oracle port ("port")."""

    def __init__(self, x_rows: np.ndarray, prompts, params, cores: int | None = None):
        import multiprocessing as mp

        cores = cores or len(os.sched_getaffinity(0))
        self.kind = "reference" if reference_available() else "port"
        self.worker = _ref_worker if self.kind == "reference" else _port_worker
        idx = np.arange(x_rows.shape[0])
        parts = [idx[lo:hi] for lo, hi in _partition(x_rows.shape[0], min(cores, x_rows.shape[0]))]
        self.parts = [(x_rows[p], [prompts[i] for i in p], params, int(p[0])) for p in parts if len(p)]
        self.pool = mp.get_context("fork").Pool(len(self.parts))

    def measure(self, seconds: float):
        """(tokens/s, processes, rows decided) over about `seconds` of work."""
        res = self.pool.map(self.worker, [job + (seconds,) for job in self.parts])
        rows = sum(r[0] for r in res)
        # every process decides its rows concurrently: aggregate rate = sum of per-process rates
        rate = sum(r[0] / r[1] for r in res if r[1] > 0)
        return rate, len(self.parts), rows

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_baseline(x_rows: np.ndarray, prompts, params, seconds: float, cores: int | None = None):
    """One measurement with a fresh pool.  Returns (tokens/s, processes, rows, kind)."""
    cb = CpuBaseline(x_rows, prompts, params, cores)
    try:
        rate, procs, rows = cb.measure(seconds)
    finally:
        cb.close()
    return rate, procs, rows, cb.kind


def _partition(n, m):
    base, rem = divmod(n, m)
    out, lo = [], 0
    for j in range(m):
        hi = lo + base + (j < rem)
        out.append((lo, hi))
        lo = hi
    return out


def reference_arm(args, cfg):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import decplane_oracle as O

    v = cfg["V"]
    nrows = int(min(cfg["B"], max(64, len(os.sched_getaffinity(0)))))
    src = O.Synthetic(v)
    x = src.wire(0, range(nrows))
    prompts = [np.random.default_rng(b).integers(0, v, cfg.get("prompt_len", PROMPT_LEN)) for b in range(nrows)]
    steps = []
    # bounded: the whole --steps K --warmup W run stays within ~ref_budget
    # seconds (one process pool; every step decides each process's rows at
    # least once)
    per_step = max(0.02, min(args.ref_seconds, args.ref_budget / max(1, args.steps + args.warmup)))
    cb = CpuBaseline(x, prompts, cfg["params"])
    kind = cb.kind
    try:
        for _ in range(args.warmup):
            cb.measure(per_step)
        total_rows, total_t = 0, 0.0
        for _ in range(args.steps):
            rate, cores, rows = cb.measure(per_step)
            steps.append(rate)
            total_rows += rows
            total_t += rows / rate
    finally:
        cb.close()
    value = total_rows / total_t
    what = ("unmodified reference (baseline/_ref) _Sampler('offload-truncate').sample + "
            "update_output_histogram, producer make_shard_blocks untimed as in harness.py:255-279"
            if kind == "reference" else "oracle port of _Sampler.sample + update_output_histogram")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * cfg["B"] / value,
            "higher_is_better": True, "scaling": "strong" if cfg.get("strong") else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SyntheticSource formula, seed 0)",
            "config": {"workload": cfg["name"], "V": v, "B": cfg["B"], "params": cfg["params"]},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind,
                             "sample": f"{nrows} rows of the workload, {per_step:.2f}s per step, {what}"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm

def _graph(fn, k, join=None):
    """Capture k calls of fn() (each given its step index) into one CUDA graph;
    join() re-joins any side stream the steps forked before capture ends."""
    import torch

    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for i in range(k):
                fn(i)
            if join is not None:
                join()
    torch.cuda.current_stream().wait_stream(side)
    return g


def _timed(g, dist=None, world=1):
    """Device time of one replay (ms), barrier + synchronize on both sides, max over ranks."""
    import torch

    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(st)
    g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


SIZING_GRID = (256, 512, 1024, 2048, 4096, 8192, 16384, 32768)


def shvs_hot_size(args, plane, src, seq_ids, dev, dtype):
    """The hot size SHVS runs at: `--hot H`, or (default) the paper's sizing
    model on this workload — control.HotSizeController calibrates the hot
    path's cost on the GPU at every grid size, measures the hit-ratio curve
    of the current rows with K6 and takes sizing.optimal_hot_size (untimed
    setup, like the reference's fit-sizing step, cli.py:70-95).  Leaves the
    plane's hot set at that size."""
    import torch

    from paper_2512_00719_b200 import HotVocab
    from paper_2512_00719_b200.control import HotSizeController

    v = plane.vocab_size
    master = HotVocab(v, src.hot_ordering())
    if args.hot > 0:
        plane.set_hot(master.resize(args.hot))
        return args.hot, {"chosen_by": "--hot"}
    plane.set_hot(master.resize(4096))
    ctl = HotSizeController(plane, master, grid=SIZING_GRID)
    xm = src.generate(0, seq_ids, perm=master.device_maps(dev)[0], dtype=dtype)
    c0, c = ctl.calibrate_cost(xm)
    h = ctl.refit(xm)
    ctl.begin_iteration(0)
    del xm
    torch.cuda.empty_cache()
    curve = ctl.model.curve
    return h, {"chosen_by": "sizing model (control.HotSizeController: GPU-timed hot-path cost fit + K6 "
                            "hit-ratio curve, sizing.optimal_hot_size)",
               "grid": [int(g) for g in curve.grid], "alpha_bar": [round(float(a), 6) for a in curve.alpha_bar],
               "c0_s_per_row": c0, "c_s_per_row_token": c, "hot_size": h,
               "cost_points_s_per_row": [[int(hh), t] for hh, t in ctl.cost_points]}


def _graph_ms(fn, k):
    """Device ms per call of fn(i), k calls captured in one graph and replayed."""
    import torch

    for i in range(2):
        fn(i)
    g = _graph(fn, k)
    torch.cuda.synchronize()
    return _timed(g) / k


def measure_shvs_e2e(args, cfg, plane_kw, src, seq_ids, dev, shard, world):
    """SHVS (speculative hot-vocab sampling) on the same workload, the
    paper's decision path, at the sizing model's hot size: device step time
    (sample + penalty update, CUDA graph) and end to end with HOST-resident
    hot-first logits — the hot prefix is staged with one strided DMA,
    rejected rows' tails are read zero-copy (dp_stage_hot +
    dp_sample_shvs_split).  The producer emits the penalty-free row summary
    while it writes the logits (make_shard_blocks contract, service.py:470-504;
    dp_synth_logits' fused summary): its marginal cost over the plain producer
    is measured and added to the step ("with_summary"), and the cost of a
    separate summary pass (dp_row_summary_raw) is reported beside it."""
    import torch
    import torch.distributed as dist

    from paper_2512_00719_b200 import DecisionPlane

    v = cfg["V"]
    plane = DecisionPlane(v, **plane_kw)
    plane.plan_flags = args.plan_flags
    tdt = torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16
    h, sizing_info = shvs_hot_size(args, plane, src, seq_ids, dev, tdt)
    esz = 4 if cfg["dtype"] == "f32" else 2
    perm = plane.hot.device_maps(dev)[0]
    bufs, summ = [], []
    for i in range(2):
        x, sm = src.generate(i, seq_ids, dtype=tdt, perm=perm, summary_params=plane.params_dev)
        bufs.append(x)
        summ.append(sm)
    # producer cost: plain generator vs generator + fused summary, and a separate summary pass
    sd = torch.from_numpy(np.asarray(seq_ids, np.uint64).view(np.int64)).to(dev)
    t_plain = _graph_ms(lambda i: src.generate(i, sd, dtype=tdt, perm=perm, out=bufs[i & 1]), 10)
    t_fused = _graph_ms(lambda i: src.generate(i, sd, dtype=tdt, perm=perm, out=bufs[i & 1],
                                               summary_params=plane.params_dev, summary_out=summ[i & 1]), 10)
    t_sep = _graph_ms(lambda i: plane.producer_summary(bufs[i & 1]), 20)
    fused_extra = max(0.0, t_fused - t_plain)
    base_it = [args.warmup]

    def step(i):
        it = base_it[0] + i
        if it % RESET_EVERY == 0 and it > 0:
            plane.state.reset()
        return plane.sample(bufs[it & 1], it, variant="shvs", summary=summ[it & 1], summary_raw=True)

    for i in range(args.warmup):
        step(i - args.warmup)
    torch.cuda.synchronize()
    g = _graph(step, args.steps)
    ms = _timed(g, dist if world > 1 else None, world)
    d = plane.sample(bufs[0], 0, variant="shvs", summary=summ[0], summary_raw=True, update=False, debug=True)
    torch.cuda.synchronize()
    flags = d.flags.cpu().numpy()
    accept = float(np.mean((flags & 0x02) != 0))
    bytes_row = float(d.bytes_touched.double().mean().item())
    rows = shard.rows
    # e2e: pinned host logits -> stage hot prefix -> sample (tail zero-copy) -> D2H tokens
    host = bufs[0].cpu().pin_memory()
    sh = (summ[0][0].cpu().pin_memory(), summ[0][1].cpu().pin_memory())
    staging = torch.empty((rows, h), dtype=tdt, device=dev)
    tok_host = torch.empty(rows, dtype=torch.int32).pin_memory()
    n_e2e = max(3, min(args.steps, 20))
    st = torch.cuda.current_stream()
    for k in range(2):   # warm the path
        plane.sample_host(host, 20_000 + k, sh, staging=staging, summary_raw=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(n_e2e):
        dd = plane.sample_host(host, 10_000 + k, sh, staging=staging, summary_raw=True)
        tok_host.copy_(dd.token, non_blocking=True)
    e1.record(st)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms, ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms, ms = float(t[0]), float(t[1])
    rej = int(((dd.flags.cpu().numpy() & 0x08) != 0).sum())
    tail_bytes = rej * (v - h) * esz
    step_ms = ms / args.steps
    return {"hot_size": h, "sizing": sizing_info, "accept": accept,
            "value": shard.batch_size * args.steps / (ms / 1000.0), "ms_per_step": step_ms,
            "with_summary": {"ms_per_step": step_ms + fused_extra,
                             "value": shard.batch_size / ((step_ms + fused_extra) / 1000.0),
                             "summary": "producer-fused (dp_synth_logits emits (row_max, total_expsum) while "
                                        "writing the logits); its marginal producer cost is added"},
            "producer_ms": {"logits_only": t_plain, "logits_plus_fused_summary": t_fused,
                            "fused_summary_marginal": fused_extra, "separate_summary_pass": t_sep},
            "bytes_touched_per_row": {"measured_mean": bytes_row,
                                      "algorithmic": h * esz + (1 - accept) * (v - h) * esz,
                                      "source": "dp_debug_t.bytes_touched (kernel-counted loads per row)"},
            "e2e": {"value": shard.batch_size * n_e2e / (e2e_ms / 1000.0), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(rows * h * esz + 16 * rows + tail_bytes),
                    "d2h_bytes_per_step": int(rows * 4), "steps": n_e2e,
                    "path": "DecisionPlane.sample_host: pinned hot-first host logits, hot prefix staged "
                            "(dp_stage_hot), rejected tails read zero-copy (dp_sample_shvs_split); "
                            "h2d counts the zero-copy tail bytes of the rejected rows"}}


MIX = [  # C5: heterogeneous per-row params (BASELINE configs[4])
    dict(temperature=0.8, top_k=1),                                   # greedy
    dict(temperature=0.8, top_k=50),                                  # top-k only
    dict(temperature=0.8, top_p=0.9),                                 # top-p only
    dict(temperature=0.8, min_p=0.05),                                # min-p
    dict(C2_PARAMS),                                                  # penalties + k + p
]
PEN = dict(rep_penalty=1.1, presence_penalty=0.5, frequency_penalty=0.1)


def row_params(cfg, b):
    from paper_2512_00719_b200 import SamplingParams

    if cfg.get("mix"):
        kw = dict(MIX[b % len(MIX)])
        if (b // len(MIX)) % 2 == 1:   # penalties on / off alternate
            kw.update(PEN)
        return SamplingParams(**kw, seed=0)
    return SamplingParams(**cfg["params"], seed=0)


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL's INIT lines (rank / nranks of each communicator) on stderr, so
        # the rank count of a run can be checked from its log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    import build

    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    from paper_2512_00719_b200 import DecisionPlane, HotVocab
    from paper_2512_00719_b200.sharded import BatchShard, NcclTokenGather
    from paper_2512_00719_b200.synthetic import SyntheticSource

    v = cfg["V"]
    # C4: the global batch is fixed and split over the ranks (strong); the
    # other configs keep B rows per GPU (weak).  Rows: partition_batch blocks.
    scaling = "strong" if cfg.get("strong") else "weak"
    shard = BatchShard(cfg["B"] if scaling == "strong" else cfg["B"] * world, world, rank)
    b_local = shard.rows
    seq_ids = shard.seq_ids
    prompts = [np.random.default_rng(int(s)).integers(0, v, cfg.get("prompt_len", PROMPT_LEN)) for s in seq_ids]
    params = [row_params(cfg, int(s)) for s in seq_ids]
    src = SyntheticSource(v, device=dev)
    variant = args.variant or ("shvs" if cfg.get("mix") else "full")
    hot = None
    plane = DecisionPlane(v, params, prompts=prompts, seq_ids=seq_ids, hot=hot, device=dev,
                          max_generated=RESET_EVERY + 8, split=args.split, kernel=args.kernel)
    plane.plan_flags = args.plan_flags
    tdt = torch.float32 if cfg["dtype"] == "f32" else torch.bfloat16
    sizing_info = None
    if variant == "shvs":
        hot_size, sizing_info = shvs_hot_size(args, plane, src, seq_ids, dev, tdt)
        hot = plane.hot
    perm = hot.device_maps(dev)[0] if hot is not None else None
    # 2 x batch > L2.  SHVS: the producer emits the penalty-free row summary
    # while it writes the logits (dp_synth_logits' fused summary; the
    # sampler corrects it for the penalty list), so a step streams only the
    # hot prefix (+ tails of rejected rows)
    summaries = None
    if variant == "shvs":
        gen = [src.generate(i, seq_ids, dtype=tdt, perm=perm, summary_params=plane.params_dev) for i in range(2)]
        bufs, summaries = [g[0] for g in gen], [g[1] for g in gen]
    else:
        bufs = [src.generate(i, seq_ids, dtype=tdt, perm=perm) for i in range(2)]
    gathered = torch.empty(shard.batch_size, dtype=torch.int32, device=dev)
    tok_pp = [torch.empty(b_local, dtype=torch.int32, device=dev) for _ in range(2)]
    gstream = torch.cuda.Stream(device=dev)
    # the token all-gather through the library's C ABI (dp_allgather_tokens)
    gather = NcclTokenGather(shard, dev) if world > 1 else None
    base_it = [0]

    def sample_only(i):
        it = base_it[0] + i
        if variant == "shvs":
            return plane.sample(bufs[it & 1], it, variant="shvs", summary=summaries[it & 1], summary_raw=True,
                                update=False)
        return plane.sample(bufs[it & 1], it, update=False)

    def step(i):
        # sample + penalty update (fused into the deciding kernel: fuse_update)
        it = base_it[0] + i
        if it % RESET_EVERY == 0 and it > 0:
            plane.state.reset()
        if variant == "shvs":
            d = plane.sample(bufs[it & 1], it, variant="shvs", summary=summaries[it & 1], summary_raw=True)
        else:
            d = plane.sample(bufs[it & 1], it)
        if world > 1:
            # token-id all-gather on a side stream: it overlaps the next step's
            # sampling (the penalty update needs only the local tokens)
            cur = torch.cuda.current_stream()
            tok_pp[it & 1].copy_(d.token)
            gstream.wait_stream(cur)
            with torch.cuda.stream(gstream):
                gather(tok_pp[it & 1], out=gathered)
        return d

    def join():
        if world > 1:
            torch.cuda.current_stream().wait_stream(gstream)

    for i in range(args.warmup):                     # eager warm-up (also JIT-free: kernels are prebuilt)
        step(i)
    join()
    base_it[0] = args.warmup
    torch.cuda.synchronize()
    try:
        g = _graph(step, args.steps, join)
        graphed = True
    except Exception as exc:   # e.g. a collective that cannot be captured
        print(f"# graph capture failed ({exc}); timing eagerly", file=sys.stderr)
        graphed = False
    with ClockSampler(local) as clk:
        if graphed:
            ms = _timed(g, dist, world)
        else:
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0.record(st)
            for i in range(args.steps):
                step(i)
            join()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if world > 1:
                t = torch.tensor([ms], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
    total_tokens = shard.batch_size * args.steps
    value = total_tokens / (ms / 1000.0)

    # dominant kernel(s): the sampling launch(es) alone, graph-replayed
    kg = _graph(sample_only, args.kernel_steps)
    torch.cuda.synchronize()
    kern_ms = _timed(kg) / args.kernel_steps
    producer_ms = None
    if variant == "shvs":
        producer_ms = {"separate_summary_pass": _graph_ms(lambda i: plane.producer_summary(bufs[i & 1]), 20),
                       "note": "the timed step uses the summary the producer emitted with the logits"}
    d = sample_only(0)
    torch.cuda.synchronize()
    # kernel-counted bytes loaded per row (dp_debug_t.bytes_touched), one untimed call
    dm = plane.sample(bufs[0], 0, variant=variant, summary=summaries[0] if summaries else None,
                      summary_raw=variant == "shvs", update=False, debug=True)
    bytes_measured = float(dm.bytes_touched.double().mean().item())
    flags = d.flags.cpu().numpy()
    accept = float(np.mean((flags & 0x02) != 0)) if variant == "shvs" else None
    pen_len = plane.state.len.float().mean().item()
    esz = 4 if cfg["dtype"] == "f32" else 2
    small = 8 * pen_len + 4 + 64 + 8 + 13                # penalty list, params, seq id, outputs
    if variant == "shvs":
        # algorithmic bytes: hot prefix (H) + tail on rejection + producer summary
        h = plane.hot.size
        bytes_per_row = h * esz + (1 - accept) * (v - h) * esz + 16 + small
    else:
        bytes_per_row = v * esz + small
    achieved = bytes_per_row * b_local / (kern_ms / 1000.0) / 1e9
    peak, peak_kind = measured_peak()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic = json.load(fh).get(f"{args.config}_{variant}")
    except Exception:
        pass

    # e2e through the public API with HOST buffers: pinned logits H2D, sample,
    # token D2H, every step inside the timed region
    st = torch.cuda.current_stream()
    host = bufs[0].cpu().pin_memory()
    dbuf = torch.empty_like(bufs[0])
    tok_host = torch.empty(b_local, dtype=torch.int32).pin_memory()
    n_e2e = max(2, min(args.steps, 6))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(n_e2e):
        dbuf.copy_(host, non_blocking=True)
        if variant == "shvs":
            dd = plane.sample(dbuf, 10_000 + k, variant="shvs", summary=summaries[0], summary_raw=True)
        else:
            dd = plane.sample(dbuf, 10_000 + k)
        if world > 1:
            gather(dd.token, out=gathered)
            tok_host.copy_(gathered[shard.lo:shard.hi], non_blocking=True)
        else:
            tok_host.copy_(dd.token, non_blocking=True)
    e1.record(st)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": shard.batch_size * n_e2e / (e2e_ms / 1000.0),
           "unit": "tokens/s", "h2d_bytes_per_step": int(host.numel() * host.element_size()),
           "d2h_bytes_per_step": int(tok_host.numel() * 4), "steps": n_e2e,
           "path": "DecisionPlane.sample on pinned host logits (H2D + sample + D2H per step)"}

    shvs = None
    if variant == "full" and not args.no_shvs:
        plane_kw = dict(params=params, prompts=prompts, seq_ids=seq_ids, device=dev, max_generated=RESET_EVERY + 8)
        shvs = measure_shvs_e2e(args, cfg, plane_kw, src, seq_ids, dev, shard, world)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            nrows = int(min(b_local, max(64, len(os.sched_getaffinity(0)))))
            x_rows = bufs[0][:nrows].float().cpu().numpy()
            if hot is not None:   # back to token-id order for the reference law
                x_rows = x_rows[:, hot.inv_perm]
            rate, cores, rows, kind = cpu_baseline(x_rows, prompts[:nrows], cfg["params"], args.cpu_seconds)
            what = ("unmodified reference (baseline/_ref) _Sampler('offload-truncate').sample + "
                    "update_output_histogram" if kind == "reference" else
                    "oracle port of _Sampler.sample + update_output_histogram")
            cpu = {"value": rate, "unit": "tokens/s", "cores": cores, "kind": kind,
                   "sample": f"{nrows} rows of this workload (full-vocabulary law, same logits) looped for "
                             f"{args.cpu_seconds:.0f}s on {cores} processes ({rows} decisions), {what}"}
        # our kernels per step (ncu launch list, profiles/r1/final/launches_*.csv):
        # full = the top-k sampler (penalty update fused); SHVS = hot pass +
        # tail pass (the NCCL all-gather of N > 1 is NCCL's kernel)
        launches = {"full": 1, "shvs": 2}[variant]
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic (SyntheticSource formula on device)",
            "config": {"workload": cfg["name"], "V": v, "B_per_gpu": b_local, "variant": variant,
                       "hot_size": plane.hot.size if variant == "shvs" else None,
                       "sizing": sizing_info,
                       "params": "5-way mix" if cfg.get("mix") else cfg["params"],
                       "l2": "inputs larger than L2 (2 x batch buffers alternate)",
                       "timing": "CUDA graph of the K steps" if graphed else "eager",
                       "split": plane._plan.split, "kernel": plane._plan.kernel},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "dp_sample_full" if variant == "full" else "dp_sample_shvs",
                         "kernel_ms": kern_ms, "bytes_per_row": bytes_per_row,
                         "bytes_per_row_measured": bytes_measured,
                         "traffic_source": "profiles/traffic.json: ncu --set full dram__bytes_read.sum + "
                                           "dram__bytes_write.sum of one launch of this kernel"},
            "producer_summary_ms": producer_ms,
            "shvs_accept": accept,
            "shvs": shvs,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * launches + sum(
                1 for i in range(args.warmup, args.warmup + args.steps) if i % RESET_EVERY == 0),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        gather.close()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--kernel-steps", type=int, default=50)
    ap.add_argument("--hot", type=int, default=0,
                    help="SHVS hot-set size; 0 (default): the sizing model's choice on this workload")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c2 on one GPU, c4 (B=8,192 split over the ranks, strong scaling) on N > 1")
    ap.add_argument("--variant", default=None, choices=["full", "shvs"],
                    help="default: full (C5: shvs, the config's SHVS mix)")
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--plan-flags", type=int, default=0, help="extra DP_PLAN_* bits for every plane (A-B)")
    ap.add_argument("--kernel", type=int, default=0, help="dp_plan_t.kernel: 0 auto, 1 CTA/cluster, 2 warp-per-row")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=5.0)
    ap.add_argument("--ref-budget", type=float, default=90.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shvs", action="store_true", help="skip the SHVS sub-measurement of the full-path line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    _, world, _ = env_rank()
    if args.config is None:
        args.config = "c2" if world == 1 else "c4"
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        reference_arm(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
