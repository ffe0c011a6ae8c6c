"""GPU tests of the online sizing loop (control.HotSizeController) and of
the measured bytes-touched counters (the VisitCounter analogue).

* K6 along the master ordering on rows in another layout (col_of_pos) equals
  K6 on rows written in the master layout — the online loop measures the
  curve on the rows it just decided;
* calibrate -> refit -> resize lands at the next iteration boundary, and the
  acceptance window equals the accept flags of the calls observed;
* bytes touched per row (instrument.py:6-33 counts elements streamed: hot H,
  tail V - H, full V): every row reports at least the reference's count, a
  rejected SHVS row its hot prefix plus its tail, and the batch mean stays
  within the re-stream / penalty-gather slack of the algorithmic bytes.
"""

import numpy as np
import pytest

from oracle import decplane_oracle as O

pytestmark = pytest.mark.gpu

C2 = dict(temperature=0.8, top_k=50, top_p=0.9, min_p=0.05, rep_penalty=1.1, presence_penalty=0.5,
          frequency_penalty=0.1)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    import build

    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _plane(v, bsz, hot=None, params=C2):
    from paper_2512_00719_b200 import DecisionPlane, SamplingParams

    prompts = [np.random.default_rng(b).integers(0, v, 32) for b in range(bsz)]
    return DecisionPlane(v, [SamplingParams(**params, seed=b) for b in range(bsz)], prompts=prompts, hot=hot)


def test_curve_along_master_ordering_through_position_map(torch_cuda):
    torch = torch_cuda
    from paper_2512_00719_b200 import HotVocab
    from paper_2512_00719_b200.synthetic import SyntheticSource

    v, bsz = 65536, 64
    src = SyntheticSource(v, device="cuda")
    master = HotVocab(v, src.hot_ordering())
    cur = master.resize(1000)
    plane = _plane(v, bsz, hot=master)
    grid = [16, 500, 1000, 4096, 20000]
    xm = src.generate(0, range(bsz), perm=master.device_maps(plane.device)[0])
    want = plane.hot_mass_curve(xm, grid).cpu().numpy()
    plane.set_hot(cur)
    xc = src.generate(0, range(bsz), perm=cur.device_maps(plane.device)[0])
    got = plane.hot_mass_curve(xc, grid, order=master).cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=1e-8)   # K2 sums the two layouts in different orders
    # and against the oracle on one row (token-id order)
    x = xc.cpu().numpy()[:, cur.inv_perm]
    st = O.State.new(np.random.default_rng(0).integers(0, v, 32), v)
    r = O.ready_row(x[0].astype(np.float64), st, O.Params(**C2))
    p = np.exp(r - r.max())
    np.testing.assert_allclose(got[0], [p[master.hot_ids[:h]].sum() / p.sum() for h in grid], rtol=1e-6)


def test_controller_calibrates_refits_and_resizes_at_iteration_boundary(torch_cuda):
    torch = torch_cuda
    from paper_2512_00719_b200 import HotVocab
    from paper_2512_00719_b200.control import HotSizeController
    from paper_2512_00719_b200.synthetic import SyntheticSource

    v, bsz = 152064, 256
    src = SyntheticSource(v, device="cuda")
    master = HotVocab(v, src.hot_ordering())
    plane = _plane(v, bsz, hot=master.resize(8192))
    ctl = HotSizeController(plane, master, grid=(512, 1024, 2048, 4096, 8192, 16384), every=3)
    xm = src.generate(0, range(bsz), perm=master.device_maps(plane.device)[0])
    c0, c = ctl.calibrate_cost(xm)
    assert c0 >= 0 and c > 0 and len(ctl.cost_points) == 6
    assert plane.hot.size == 8192                       # calibration leaves the hot set alone
    h_star = ctl.refit(src.generate(0, range(bsz), perm=plane.hot.device_maps(plane.device)[0]))
    assert 1 <= h_star <= v and ctl.pending == h_star
    assert plane.hot.size == 8192                       # parked, not applied mid-iteration
    flags = []
    for it in range(6):
        hot = ctl.begin_iteration(it)
        if it == 0:
            assert hot.size == h_star and ctl.history == [(0, h_star)]
        x, summ = src.generate(it, range(bsz), perm=hot.device_maps(plane.device)[0],
                               summary_params=plane.params_dev)
        d = plane.sample(x, it, variant="shvs", summary=summ, summary_raw=True)
        flags.append(d.flags.cpu().numpy().copy())
        ctl.end_iteration(it, d, logits=x)
    assert ctl.pending is not None or ctl.history[-1][0] > 0   # refits every 3 iterations
    window = np.concatenate(flags[-len(ctl._acc):])
    assert abs(ctl.acceptance_rate() - np.mean((window & 2) != 0)) < 1e-12
    assert "hot_size:" in ctl.report()


@pytest.mark.parametrize("bf16", [False, True])
def test_bytes_touched_per_row(torch_cuda, bf16):
    torch = torch_cuda
    from paper_2512_00719_b200 import HotVocab
    from paper_2512_00719_b200.synthetic import SyntheticSource

    v, bsz, h = 152064, 512, 1024
    esz = 2 if bf16 else 4
    dt = torch.bfloat16 if bf16 else torch.float32
    src = SyntheticSource(v, device="cuda")
    hot = HotVocab(v, src.hot_ordering()[:h])
    plane = _plane(v, bsz, hot=hot)
    plen = plane.state.len.cpu().numpy().astype(np.int64)
    # full path: >= V elements per row (instrument.py: visits V), < 2 passes
    x = src.generate(0, range(bsz), dtype=dt)
    d = plane.sample(x, 0, debug=True, update=False)
    bt = d.bytes_touched.cpu().numpy()
    assert (bt >= v * esz).all() and (bt <= 2 * v * esz + plen * esz).all()
    # SHVS: hot prefix always, the tail only on rejection
    x, summ = src.generate(0, range(bsz), dtype=dt, perm=hot.device_maps(plane.device)[0],
                           summary_params=plane.params_dev)
    d = plane.sample(x, 0, variant="shvs", summary=summ, summary_raw=True, debug=True, update=False)
    bt = d.bytes_touched.cpu().numpy()
    fl = d.flags.cpu().numpy()
    rej = (fl & 0x08) != 0
    assert rej.any() and (~rej).any()
    assert (bt[~rej] >= h * esz).all() and (bt[~rej] <= 3 * h * esz + plen[~rej] * esz).all()
    assert (bt[rej] >= v * esz).all()
    algo = h * esz + rej.mean() * (v - h) * esz
    assert algo <= bt.mean() <= 1.5 * algo + plen.mean() * esz * 3
    print(f"SHVS bytes/row: measured {bt.mean():.0f}, algorithmic {algo:.0f}, reject {rej.mean():.3f}")


def test_eos_retirement_compacts_rows_and_keeps_decisions(torch_cuda):
    """service.py:709-714: rows whose token is an EOS id leave the batch at
    the iteration boundary.  The compacted plane keeps each surviving row's
    seq_id, params and penalty list, so its next decisions equal those of a
    plane that never retired anyone (uniforms are keyed by seq_id)."""
    torch = torch_cuda
    from paper_2512_00719_b200 import DecisionPlane, SamplingParams, _native as N
    from paper_2512_00719_b200.synthetic import SyntheticSource

    v, bsz = 4096, 64
    prompts = [np.random.default_rng(b).integers(0, v, 16) for b in range(bsz)]
    params = [SamplingParams(**C2, seed=b) for b in range(bsz)]
    a = DecisionPlane(v, params, prompts=prompts, seq_ids=np.arange(100, 100 + bsz))
    ref = DecisionPlane(v, params, prompts=prompts, seq_ids=np.arange(100, 100 + bsz))
    src = SyntheticSource(v, device="cuda")
    x0 = src.generate(0, range(100, 100 + bsz))
    d = a.sample(x0, 0)
    r0 = ref.sample(x0, 0)
    tok0 = d.token.cpu().numpy()
    eos = {int(tok0[3]), int(tok0[10])}
    kept = a.retire_finished(d, eos)
    fl = d.flags.cpu().numpy()
    assert all(bool(fl[b] & N.FLAG_EOS) == (int(tok0[b]) in eos) for b in range(bsz))
    assert 3 not in kept and 10 not in kept and a.batch == kept.size
    assert np.array_equal(a.seq_ids, np.arange(100, 100 + bsz)[kept])
    x1 = src.generate(1, range(100, 100 + bsz))
    d1 = a.sample(x1[torch.from_numpy(kept).cuda()].contiguous(), 1)
    r1 = ref.sample(x1, 1)
    assert np.array_equal(d1.token.cpu().numpy(), r1.token.cpu().numpy()[kept])
    rows_a, rows_r = a.state.rows(), ref.state.rows()
    for i, b in enumerate(kept):
        assert np.array_equal(rows_a[i][0], rows_r[b][0]) and np.array_equal(rows_a[i][1], rows_r[b][1])
    # max_tokens: everything retires once the generated length is reached
    assert a.retire_finished(d1, max_tokens=2).size == 0 and a.batch == 0
