"""bench.py's launcher contract on CPU: `--gpus N` without torchrun re-execs
itself under torch.distributed.run with N ranks and rank 0 alone prints one
JSON line carrying n_gpus = N (driver contract; the reference arm is the one
that runs without a GPU)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_self_launches_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--steps", "1", "--warmup", "3", "--ref-budget", "2", "--ref-seconds", "0.5"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2
    assert line["impl"] == "reference"
    assert line["scaling"] == "strong"         # N > 1 defaults to C4 (B split over the ranks)
    assert line["config"]["workload"].startswith("qwen3-151936")
