"""SURVEY 8(f) row 4, CPU side: the oracle restatement of hitrate.py is pinned
bit-for-bit to the reference's own rates (tests/golden/gen_golden.py:
gen_hitrate), plus the reference's known-answer and property tests
(pkg/tests/test_hitrate.py) restated, and the host-side argument checks."""
import numpy as np
import pytest

from conftest import golden
from oracle import hitrate as O


def _golden_sequences():
    d = golden("hitrate_rows.npz")
    out = []
    for i in range(int(d["nseq"])):
        lens = d[f"lens_{i}"]
        rows = np.split(d[f"rows_{i}"], np.cumsum(lens)[:-1])
        out.append((rows, d[f"topk_{i}"], d[f"evict_{i}"]))
    return d["ks"], out


def test_oracle_bit_exact_vs_reference():
    ks, seqs = _golden_sequences()
    for rows, topk, evict in seqs:
        for j, k in enumerate(ks):
            np.testing.assert_array_equal(O.topk_hitrate(rows, int(k)), topk[j])
            np.testing.assert_array_equal(O.eviction_hitrate(rows, int(k)), evict[j])


def test_pairwise_sum_is_numpys(rng):
    for n in (0, 1, 7, 8, 9, 127, 128, 129, 1000, 5000):
        a = rng.random(n)
        assert O.pairwise_sum(a) == float(np.sum(a))


def test_known_answers():  # pkg/tests/test_hitrate.py:17-39
    assert O.topk_hitrate([np.array([0.7, 0.2, 0.1])], 1)[0] == pytest.approx(0.7)
    assert O.topk_hitrate([np.array([0.7, 0.2, 0.1])], 2)[0] == pytest.approx(0.9)
    rows = [np.full(5, 0.2)] * 3
    assert np.allclose(O.topk_hitrate(rows, 100), 1.0)
    assert np.allclose(O.eviction_hitrate(rows, 100), 1.0)
    assert (O.topk_hitrate(rows, 0) == 0.0).all()
    with pytest.raises(ValueError):
        O.topk_hitrate([np.array([1.0])], -1)
    with pytest.raises(ValueError):
        O.eviction_hitrate([np.array([1.0])], -1)


def test_topk_dominates_eviction(rng):  # pkg/tests/test_hitrate.py:41-75
    for _ in range(5):
        rows = []
        for t in range(6):
            x = rng.random(20 + t)
            rows.append(x / x.sum())
        prev = None
        for k in range(0, 30, 3):
            tk, ev = O.topk_hitrate(rows, k), O.eviction_hitrate(rows, k)
            assert (ev <= tk + 1e-12).all()
            if prev is not None:
                assert (tk >= prev - 1e-12).all()
            prev = tk


def test_device_api_argument_errors():
    from paper_2503_16163_b200 import hitrate as H
    with pytest.raises(ValueError):
        H.topk_hitrate([np.array([1.0])], -1)
    with pytest.raises(ValueError):
        H.eviction_hitrate([np.array([1.0])], -2)
    assert H.topk_hitrate([], 3).size == 0
    with pytest.raises(ValueError):
        H.AttentionTrace()
