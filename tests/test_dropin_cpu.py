"""CPU tests of the drop-in host surface: the SequenceState mirror and
update_output_histogram, the DecisionBatch wire format, shard views and the
growable penalty table's capacity logic.  Where the unmodified reference is
installed (baseline/_ref, `pip install --target`) the mirror is
compared with it object for object; no kernel is launched here."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "decplane")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF)
    import decplane.core as core
    import decplane.penalty as penalty
    import decplane.transport as transport

    return core, penalty, transport


def _history(seed, v, n):
    rs = np.random.default_rng(seed)
    hot = rs.integers(0, v, 12)
    return [int(hot[rs.integers(0, 12)]) if rs.random() < 0.6 else int(rs.integers(0, v)) for _ in range(n)]


def test_sequence_state_matches_reference(ref):
    core, penalty, _ = ref
    from paper_2512_00719_b200 import new_sequence_state, update_output_histogram
    from paper_2512_00719_b200.core import sparse_entries

    v = 500
    for seed in range(5):
        prompt = np.random.default_rng(100 + seed).integers(0, v, 40).tolist()
        a = new_sequence_state(7, prompt, v, max_generated=64)
        b = core.new_sequence_state(7, prompt, v, max_generated=64)
        for tok in _history(seed, v, 64):
            update_output_histogram(a, tok)
            penalty.update_output_histogram(b, tok)
        for f in ("prompt_hist", "output_hist", "prompt_mask", "output_mask"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
        assert a.generated_len == b.generated_len == 64
        np.testing.assert_array_equal(a.history(), b.history())
        np.testing.assert_array_equal(a.output_id_view(), b.output_id_view())
        np.testing.assert_array_equal(a.touched_id_view(), b.touched_id_view())
        a.check_consistency()
        # both raise when the append buffer is full (core.py:90-92)
        with pytest.raises(OverflowError):
            update_output_histogram(a, 0)
        with pytest.raises(OverflowError):
            penalty.update_output_histogram(b, 0)
        # the device-table row built from either object is the same
        for x, y in zip(sparse_entries(a), sparse_entries(b)):
            np.testing.assert_array_equal(x, y)


def test_update_rejects_out_of_range_token():
    from paper_2512_00719_b200 import RangeError, new_sequence_state, update_output_histogram

    st = new_sequence_state(0, [1, 2], 10)
    with pytest.raises(RangeError):
        update_output_histogram(st, 10)
    with pytest.raises(RangeError):
        new_sequence_state(0, [11], 10)


def test_decision_batch_wire_bytes_match_reference(ref):
    _, _, transport = ref
    from paper_2512_00719_b200 import TokenDecision
    from paper_2512_00719_b200 import transport as T

    decs = [TokenDecision(9, 100 + i, 7 * i, i % 3 == 0, i % 2 == 1, -0.25 * i) for i in range(6)]
    ours = T.encode_decision_batch(T.DecisionBatch(9, decs))
    theirs = transport.encode_frame(transport.DecisionBatch(9, decs))
    assert ours == theirs
    assert T.encode_decision_batch(T.DecisionBatch(3, [])) == transport.encode_frame(transport.DecisionBatch(3, []))
    back = T.decode_decision_batch(ours)
    assert [(d.seq_id, d.token_id, d.is_eos, d.accepted_hot) for d in back.decisions] == \
           [(d.seq_id, d.token_id, d.is_eos, d.accepted_hot) for d in decs]
    with pytest.raises(T.ChecksumError):
        T.decode_decision_batch(ours[:-1] + bytes([ours[-1] ^ 1]))
    with pytest.raises(T.TruncatedPayloadError):
        T.decode_decision_batch(ours[:30])


def test_assemble_view_checks_tiling_and_reads_columns():
    from paper_2512_00719_b200 import LogitsShardBlock, assemble_view
    from paper_2512_00719_b200.transport import IncompleteIterationError

    v, b = 12, 5
    x = np.arange(v * b, dtype=np.float32).reshape(b, v)
    blocks = [LogitsShardBlock(0, r, lo, lo + 4, np.asfortranarray(x[:, lo:lo + 4].T), np.zeros(b), np.ones(b), 3)
              for r, lo in enumerate((0, 4, 8))]
    view = assemble_view(blocks[::-1], (1, 4))
    assert view.vocab_size == v and view.num_cols == 3
    rows = view.shard_rows([0, 2], "cpu")
    np.testing.assert_array_equal(np.concatenate([r.numpy() for r in rows], axis=1), x[[1, 3]])
    with pytest.raises(IncompleteIterationError):
        assemble_view(blocks[:1] + blocks[2:], (0, b))
    bad = LogitsShardBlock(1, 2, 8, 12, blocks[2].values, np.zeros(b), np.ones(b), 3)
    with pytest.raises(IncompleteIterationError):
        assemble_view(blocks[:2] + [bad], (0, b))


def test_penalty_table_grows_and_overflows_like_the_reference():
    """Host capacity logic of the device table (no kernel): the bound passed
    to the kernels is exact, the table doubles before it could overflow, and
    recording past max_generated raises OverflowError (core.py:90-92)."""
    from paper_2512_00719_b200.penalty import PenaltyState

    st = PenaltyState([[1, 2, 3], [4]], 5000, device="cpu", max_generated=600)
    assert st.cap == 3 + 256 and st.bound == 3
    caps = []
    for i in range(600):
        nat = st.prepare(True)
        assert nat.max_len == 3 + i + 1 <= st.cap
        st.committed(True)
        caps.append(st.cap)
    assert sorted(set(caps)) == [259, 518, 603]      # doubling, then the logical limit
    assert PenaltyState([[1, 2, 3]], 100, device="cpu").cap == 100   # never beyond V unique ids
    with pytest.raises(OverflowError):
        st.prepare(True)
    st.recorded = 0
    assert st.prepare(False).max_len == 3
