"""CPU-only tests: the C-ABI library builds and exports every declared symbol,
and the host-side logic (params, hot vocab, partitioning, sizing) matches the
reference semantics.  No kernel is launched here."""

import json
import os
import re

import numpy as np
import pytest

from oracle import decplane_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import build

    build.build()
    from paper_2512_00719_b200 import _native as N

    return N.load()


def test_library_exports_every_header_symbol(lib):
    header = open(os.path.join(ROOT, "include", "decplane_b200.h")).read()
    declared = set(re.findall(r"^DP_API\s+[\w\s\*]+?\b(dp_\w+)\(", header, flags=re.M))
    assert {"dp_sample_full", "dp_sample_shvs", "dp_row_summary", "dp_penalty_update"} <= declared
    for name in declared:
        assert hasattr(lib, name), name
    from paper_2512_00719_b200 import _native as N

    assert set(N.EXPORTS) == declared
    assert lib.dp_version() >= 100


def test_struct_layouts_match_header():
    import ctypes as C

    from paper_2512_00719_b200 import _native as N

    assert C.sizeof(N.Params) == 64
    assert N.Params.top_p.offset == 16 and N.Params.seed.offset == 56
    assert C.sizeof(N.Penalty) == 48 and N.Penalty.max_len.offset == 40
    assert C.sizeof(N.Plan) == 48 and N.Plan.workspace.offset == 32 and N.Plan.workspace_len.offset == 40


def test_library_rejects_bad_arguments_without_gpu(lib):
    # argument validation happens before any CUDA call
    import ctypes as C

    from paper_2512_00719_b200 import _native as N

    st = lib.dp_sample_full(None, 0, 1, 10, 10, None, None, None, None, 0, None, None, None, None, None, None)
    assert st == N.DP_ERR_ARG
    assert b"null" in lib.dp_last_error()
    pen = N.Penalty(1, 1, 1, 1, 4, 99, 0, 0)
    st = lib.dp_sample_full(C.c_void_p(1), 0, 1, 10, 10, C.c_void_p(1), C.byref(pen), None, C.c_void_p(1), 0,
                            C.c_void_p(1), C.c_void_p(1), C.c_void_p(1), None, None, None)
    assert st == N.DP_ERR_ARG and b"penalty" in lib.dp_last_error()
    st = lib.dp_sample_full(C.c_void_p(1), 5, 1, 10, 10, C.c_void_p(1), C.byref(pen), None, C.c_void_p(1), 0,
                            C.c_void_p(1), C.c_void_p(1), C.c_void_p(1), None, None, None)
    assert st == N.DP_ERR_UNSUPPORTED


def test_sharded_entry_checks_tiling_without_gpu(lib):
    """dp_sample_full_sharded refuses what AssembledLogitsView refuses
    (transport.py:474-489: unequal widths / broken tiling), before any CUDA call."""
    import ctypes as C

    from paper_2512_00719_b200 import _native as N

    one = C.c_void_p(1)
    pen = N.Penalty(1, 1, 1, 1, 4, 12, 0, 0)

    def call(ptrs, t, v, ld):
        arr = (C.c_void_p * max(len(ptrs), 1))(*ptrs)
        return lib.dp_sample_full_sharded(arr, t, 0, 1, v, ld, one, C.byref(pen), None, one, 0, one, one, one,
                                          None, None, None)

    assert call([1, 1], 2, 13, 7) == N.DP_ERR_ARG and b"tile" in lib.dp_last_error()    # 13 % 2 != 0
    assert call([1, 1], 2, 12, 5) == N.DP_ERR_ARG                                        # ld < V / t
    assert call([1] * 9, 9, 18, 2) == N.DP_ERR_ARG and b"shard count" in lib.dp_last_error()
    assert call([1, 0], 2, 12, 6) == N.DP_ERR_ARG and b"null shard" in lib.dp_last_error()
    # valid tiling but no plan bounds: rows may lack top-k -> the caller stitches
    assert call([1, 1], 2, 12, 6) == N.DP_ERR_UNSUPPORTED and b"stitch" in lib.dp_last_error()


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2512_00719_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f


def test_validate_params_mirrors_reference():
    from paper_2512_00719_b200 import SamplingParams, validate_params

    assert validate_params(SamplingParams(), 100) == []
    assert validate_params(SamplingParams(temperature=0.0), 10) == ["temperature must be positive"]
    assert validate_params(SamplingParams(top_k=11), 10) == ["top_k exceeds vocabulary"]
    errs = validate_params(SamplingParams(temperature=-1, top_p=0, min_p=1, rep_penalty=0, seed=-1), 10)
    assert len(errs) == 5
    assert SamplingParams(top_k=5).filters_neutral(5) and not SamplingParams(top_k=4).filters_neutral(5)
    assert SamplingParams().penalties_neutral()


def test_hot_vocab_layout_and_reference_tie_rules():
    from paper_2512_00719_b200 import HotVocab, build_hot_vocab

    assert build_hot_vocab([(0, 5), (1, 1), (2, 9), (3, 1)], 2, 4).hot_ids.tolist() == [2, 0]
    assert build_hot_vocab([(0, 1), (1, 1), (2, 1)], 2, 3).hot_ids.tolist() == [0, 1]
    hv = HotVocab(10, [7, 2, 5])
    assert hv.tail_ids.tolist() == [0, 1, 3, 4, 6, 8, 9]
    assert hv.perm.tolist() == [7, 2, 5, 0, 1, 3, 4, 6, 8, 9]
    assert (hv.perm[hv.inv_perm] == np.arange(10)).all()
    assert hv.resize(2).hot_ids.tolist() == [7, 2]
    with pytest.raises(ValueError):
        HotVocab(4, [1, 1])


def test_hot_vocab_trace_roundtrip(tmp_path):
    from paper_2512_00719_b200 import build_hot_vocab, load_hot_vocab_trace, save_hot_vocab_trace

    trace = [(3, 10), (1, 10), (0, 4), (2, 1)]
    p = tmp_path / "hot.tsv"
    save_hot_vocab_trace(p, trace)
    back = load_hot_vocab_trace(p)
    assert back == [(1, 10), (3, 10), (0, 4), (2, 1)]
    assert build_hot_vocab(back, 3, 4).hot_ids.tolist() == [1, 3, 0]


def test_partition_batch_matches_reference():
    from paper_2512_00719_b200 import partition_batch

    for b in (1, 7, 64, 1000, 8192):
        for w in (1, 2, 3, 8):
            assert partition_batch(b, w) == O.partition_batch(b, w)


def test_sizing_matches_reference_golden(golden_dir):
    from paper_2512_00719_b200 import sizing

    spec = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    s = spec["sizing"]
    curve = sizing.HitRatioCurve(s["grid"], s["alpha_bar"])
    pts = [(h, 8.55e-6 + 1.06e-8 * h) for h in (4096, 8192, 16384, 32768)]
    c0, c, _ = sizing.fit_affine_cost(pts)
    assert abs(c0 - s["c0"]) <= 1e-12 * abs(s["c0"]) + 1e-18 and abs(c - s["c"]) <= 1e-12 * s["c"]
    model = sizing.SizingModel(c0, c, curve, 128256)
    assert sizing.optimal_hot_size(model) == s["hot"]
    assert sizing.expected_cost(4096, model) == pytest.approx(s["cost_4096"], rel=1e-12)
    assert sizing.optimal_hot_size(model, cycle_budget=6e-4) == s["hot_budget"]
    lin = sizing.HitRatioCurve([1.0, 1000.0], [0.001, 1.0])
    assert sizing.optimal_hot_size(sizing.SizingModel(0.0, 1.0, lin, 1000)) == spec["sizing_linear"] == 500


def test_synthetic_hot_ordering_matches_oracle():
    from paper_2512_00719_b200.synthetic import hot_ordering

    for v in (16, 2048, 32000):
        np.testing.assert_array_equal(hot_ordering(0, v), O.synthetic_hot_ordering(0, v))
        np.testing.assert_array_equal(hot_ordering(5, v), O.synthetic_hot_ordering(5, v))


def test_collective_entry_points_resolve_nccl(lib):
    """dp_allgather_tokens' NCCL is found at run time (no GPU needed to draw a
    unique id); bad arguments fail with DP_ERR_ARG before touching NCCL."""
    import ctypes as C

    from paper_2512_00719_b200 import _native as N

    assert lib.dp_nccl_available() == 1
    uid = (C.c_uint8 * 128)()
    assert lib.dp_nccl_unique_id(uid) == N.DP_OK
    assert any(bytes(uid))
    assert lib.dp_allgather_tokens(None, None, 4, None, None) == N.DP_ERR_ARG
    assert lib.dp_allgather_tokens(None, None, 0, C.c_void_p(1), None) == N.DP_OK


def test_hot_size_controller_boundary_logic_on_cpu():
    """control.HotSizeController's host logic (service.py:602-610 apply_control
    + run_iteration): a requested size is validated now and applied only at the
    next iteration boundary; the acceptance window averages the observed
    calls.  A stand-in plane (no kernels) carries the hot set."""
    import torch

    from paper_2512_00719_b200.control import HotSizeController
    from paper_2512_00719_b200.shvs import HotVocab

    class Plane:
        vocab_size, batch = 64, 4

        def __init__(self):
            self.hot = None

        def set_hot(self, hot):
            self.hot = hot

    class D:
        def __init__(self, flags):
            self.flags = torch.tensor(flags, dtype=torch.uint8)

    plane = Plane()
    master = HotVocab(64, np.arange(64)[::-1].copy())
    ctl = HotSizeController(plane, master, grid=(8, 16, 32), window=8)
    with pytest.raises(ValueError):
        ctl.request(0)
    with pytest.raises(ValueError):
        ctl.request(65)
    with pytest.raises(ValueError):
        ctl.begin_iteration(0)          # no hot set yet
    ctl.request(16)
    assert plane.hot is None            # parked until the boundary
    hot = ctl.begin_iteration(3)
    assert hot.size == 16 and list(hot.hot_ids) == list(master.hot_ids[:16]) and ctl.history == [(3, 16)]
    assert ctl.begin_iteration(4) is hot and ctl.history == [(3, 16)]
    for fl in ([2, 0, 2, 2], [0, 0, 2, 0], [2, 2, 2, 2]):
        ctl.end_iteration(0, D(fl))     # no logits: observe only
    # window of 8 decisions = the last two calls
    assert abs(ctl.acceptance_rate() - 5 / 8) < 1e-12
    with pytest.raises(ValueError):
        ctl.refit(None)                 # no cost model yet


def test_hot_size_controller_curve_spans_one_to_v():
    """The controller's hit-ratio curve carries H = 1 and H = V like
    fit-sizing's `sorted(set(grid + [1, V]))` (cli.py:88).  Without the H = 1
    point np.interp holds alpha flat below the first grid size, and with a
    dominant fixed cost c0 (C1 on a B200) Eq. 10's argmin lands on H = 1.  A
    stand-in plane returns a known per-row curve (no kernels)."""
    import torch

    from paper_2512_00719_b200 import sizing
    from paper_2512_00719_b200.control import HotSizeController
    from paper_2512_00719_b200.shvs import HotVocab

    v, bsz = 32000, 4

    def alpha(h):   # hot mass of the first h ids: 0.30 at h = 1, 0.95 at 256, 1 at V
        return min(1.0, 0.30 + 0.65 * np.log(h) / np.log(256)) if h < v else 1.0

    class Plane:
        vocab_size, batch = v, bsz

        def __init__(self):
            self.hot = None
            self.asked = None

        def set_hot(self, hot):
            self.hot = hot

        def hot_mass_curve(self, logits, grid, summary=None, order=None):
            self.asked = list(grid)
            return torch.tensor([[alpha(h) for h in grid]] * bsz, dtype=torch.float64)

    plane = Plane()
    master = HotVocab(v, np.arange(v))
    # C1's fitted constants (bench_c1.jsonl): c0 = 5.7e-7 s per row, c = 5.0e-12 s per row-token
    ctl = HotSizeController(plane, master, grid=(256, 512, 1024, 2048, 4096, 8192, 16384), cost=(5.7e-7, 5.0e-12))
    h = ctl.refit(None)
    assert plane.asked[0] == 1 and 256 in plane.asked
    assert list(ctl.model.curve.grid[[0, -1]]) == [1.0, float(v)]
    assert abs(ctl.model.curve.value(1.0) - alpha(1)) < 1e-12
    assert h > 1
    assert h == sizing.optimal_hot_size(ctl.model)


def test_product_fails_loudly_without_library_or_device(tmp_path, monkeypatch):
    """No CPU fallback: a missing library raises NativeUnavailable at load,
    and a DecisionPlane without a CUDA sm_100 device raises it at
    construction (this container has no GPU)."""
    import torch

    from paper_2512_00719_b200 import DecisionPlane, SamplingParams, _native

    monkeypatch.setattr(_native, "_lib", None)   # as in a fresh process (another test may have loaded it)
    with pytest.raises(_native.NativeUnavailable):
        _native.load(str(tmp_path / "missing.so"))
    monkeypatch.undo()
    if not torch.cuda.is_available():
        with pytest.raises(_native.NativeUnavailable):
            DecisionPlane(64, [SamplingParams(top_k=4, seed=0)], device="cuda:0")
