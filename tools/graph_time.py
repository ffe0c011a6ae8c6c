"""Device time per dp_sample_full call, measured by replaying a CUDA graph of K calls."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2512_00719_b200 import DecisionPlane, SamplingParams
from paper_2512_00719_b200.synthetic import SyntheticSource
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]; v, b = cfg["V"], cfg["B"]
dt = torch.bfloat16 if "--bf16" in sys.argv else torch.float32
esz = 2 if dt == torch.bfloat16 else 4
for split, nt in ((1, 256), (1, 128), (2, 128)):
    prompts = [np.random.default_rng(s).integers(0, v, 32) for s in range(b)]
    plane = DecisionPlane(v, [SamplingParams(**cfg["params"])] * b, prompts=prompts, max_generated=136, split=split)
    plane._plan.reserved[0] = nt
    src = SyntheticSource(v, device="cuda")
    bufs = [src.generate(i, range(b), dtype=dt) for i in range(2)]
    K = 20
    for i in range(3):
        plane.sample(bufs[i & 1], i, update=False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(K):
                plane.sample(bufs[i & 1], 100 + i, update=False)
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"{'bf16' if esz == 2 else 'f32'} split={split} nt={nt}: {ms*1000:.1f} us/call  {v*esz*b/(ms/1e3)/1e9:.0f} GB/s", flush=True)
