"""A-B timing of the synthetic producer: plain vs fused summary (and an
optional variant library via DP_LIB).  python tools/micro/synth_ab.py"""
import os, sys, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench
from paper_2512_00719_b200 import DecisionPlane, SamplingParams
from paper_2512_00719_b200.synthetic import SyntheticSource

v, b = 152064, 1024
dev = torch.device("cuda")
src = SyntheticSource(v, device=dev)
plane = DecisionPlane(v, [SamplingParams(temperature=0.8)] * b)
sd = torch.arange(b, dtype=torch.int64, device=dev)
out = [torch.empty((b, v), dtype=torch.float32, device=dev) for _ in range(2)]
sm = [(torch.empty(b, dtype=torch.float64, device=dev), torch.empty(b, dtype=torch.float64, device=dev)) for _ in range(2)]
t_plain = bench._graph_ms(lambda i: src.generate(i, sd, out=out[i & 1]), 10)
t_fused = bench._graph_ms(lambda i: src.generate(i, sd, out=out[i & 1], summary_params=plane.params_dev,
                                                 summary_out=sm[i & 1]), 10)
t_sep = bench._graph_ms(lambda i: plane.producer_summary(out[i & 1]), 20)
print(json.dumps(dict(lib=os.environ.get("DP_LIB", "default"), plain=t_plain, fused=t_fused, separate=t_sep)))
