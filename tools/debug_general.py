import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import decplane_oracle as O
from tests.golden_cases import Case
from paper_2512_00719_b200 import DecisionPlane, SamplingParams
case = Case(sys.argv[1] if len(sys.argv) > 1 else "het_full")
params = case.params(); states = case.states()
plane = DecisionPlane(case.vocab, [SamplingParams(**vars(p)) for p in params], prompts=[case.prompts[b] for b in range(case.batch)], max_generated=64)
x = case.logits(0)
u = O.uniforms_per_row([p.seed for p in params], 0, list(range(case.batch)))
d = plane.sample(torch.from_numpy(x).cuda(), 0, debug=True, update=False)
tok = d.token.cpu().numpy(); kept = d.kept.cpu().numpy(); mar = d.margin.cpu().numpy(); lp = d.logprob.cpu().numpy()
for b in range(case.batch):
    p = params[b]
    r = O.ready_row(x[b], states[b], p)
    dd = O.filter_draw(r, p, float(u[b, 0]))
    # oracle rank of GPU token
    order = np.lexsort((np.arange(len(r)), -r))
    rank_gpu = int(np.flatnonzero(order == tok[b])[0]) if 0 <= tok[b] < len(r) else -1
    rank_or = int(np.flatnonzero(order == dd.index)[0])
    w = np.exp(r[order] - r[order[0]]); cdf = np.cumsum(w) / w[:dd.kept].sum()
    print(b, "k=%d p=%.2f minp=%.2f" % (p.top_k, p.top_p, p.min_p), "gpu", tok[b], "kept", kept[b], "lp %.4f" % lp[b],
          "| oracle", dd.index, "kept", dd.kept, "lp %.4f" % dd.logprob, "ranks", rank_gpu, rank_or, "u %.6f" % u[b,0],
          "cdf@gpu %.6f" % (cdf[rank_gpu] if rank_gpu >= 0 else -1), "ok" if tok[b] == dd.index else "MISMATCH")
