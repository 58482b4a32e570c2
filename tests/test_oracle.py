"""Pin the numpy oracle against fixtures produced by the reference itself
(tests/golden/gen_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import golden
from oracle import restate as R


def _groups(q):
    vals, off = q["values"], q["offsets"]
    return [vals[off[i]:off[i + 1]] for i in range(len(off) - 1)]


@pytest.mark.parametrize("bits", [1, 2, 4])
def test_quantizer_matches_reference_bit_exact(bits):
    q = golden("quant_groups.npz")
    groups = _groups(q)
    poff = q[f"b{bits}_poff"]
    codes_all, deq_all, packed_all = [], [], []
    for i, g in enumerate(groups):
        z, s = R.quant_params(g[None], bits)
        assert z[0] == q[f"b{bits}_zero"][i]
        assert s[0] == q[f"b{bits}_scale"][i]
        assert z.astype(np.float16).view(np.uint16)[0] == q[f"b{bits}_zero16"][i]
        assert s.astype(np.float16).view(np.uint16)[0] == q[f"b{bits}_scale16"][i]
        c = R.quantize(g[None], z, s, bits)
        codes_all.append(c[0])
        deq_all.append(R.dequantize(c, z, s)[0])
        p = R.pack_groups(c, bits)[0]
        assert p.tobytes() == q[f"b{bits}_packed"][poff[i]:poff[i + 1]].tobytes()
        assert np.array_equal(R.unpack_groups(p[None], g.size, bits)[0], c[0])
        packed_all.append(p)
    assert np.array_equal(np.concatenate(codes_all), q[f"b{bits}_codes"])
    assert np.array_equal(np.concatenate(deq_all).view(np.uint32),
                          q[f"b{bits}_deq"].view(np.uint32))


def test_packing_kats():
    # test_quant.py:111-116
    assert R.pack_groups(np.array([[3, 0, 1, 2]]), 2)[0].tolist() == [0x93]
    assert R.pack_groups(np.array([[1, 0, 0, 0, 0, 0, 0, 1]]), 1)[0].tolist() == [0x81]


def test_frontier_rule():
    assert R.frontier(1024, 32, 32) == 992
    assert R.frontier(4096, 32, 32) == 4064
    assert R.frontier(96, 64, 32) == 32       # test_kvcache.py:58-65
    assert R.frontier(95, 64, 32) == 0
    assert R.frontier(10, 64, 32) == 0


@pytest.mark.parametrize("tag", ["b2_d128", "b1_d128", "b4_d128", "b16_d128",
                                 "b2_d10_g4", "b1_d8_g4", "b2_d128_g64", "b1_d128_g64"])
def test_snapshot_and_materialize_match_reference(tag):
    c = golden(f"cache_{tag}.npz")
    K, V, bits, g, r = c["K"], c["V"], int(c["bits"]), int(c["g"]), int(c["r"])
    f = R.frontier(K.shape[0], r, g)
    assert f == int(c["frontier"])
    if bits != 16:
        exp = R.normative_export(K, V, f, bits, g)
        assert np.array_equal(exp["key_codes"], c["key_codes"])
        assert np.array_equal(exp["key_zero"].view(np.uint16), c["key_zero16"])
        assert np.array_equal(exp["key_scale"].view(np.uint16), c["key_scale16"])
        assert np.array_equal(exp["val_codes"], c["val_codes"])
        assert np.array_equal(exp["val_zero"].view(np.uint16), c["val_zero16"])
        assert np.array_equal(exp["val_scale"].view(np.uint16), c["val_scale16"])
    mk, mv = R.materialize_all(K, V, f, bits, g, [int(p) for p in c["pins"]])
    assert np.array_equal(mk.view(np.uint32), c["mat_k"].view(np.uint32))
    assert np.array_equal(mv.view(np.uint32), c["mat_v"].view(np.uint32))


@pytest.mark.parametrize("tag", ["mha_b2", "gqa_b1", "mha_b16", "gqa4_b2", "gqa_b2_g64"])
def test_decode_layer_matches_reference(tag):
    z = golden(f"decode_{tag}.npz")
    bits, g, r, k, Hq = (int(z[x]) for x in ("bits", "g", "r", "k", "Hq"))
    K0, V0 = z["K0"], z["V0"]
    st = R.LayerState(K0.shape[1], K0.shape[2], bits, g, r, k)
    st.extend(K0, V0)
    pre = R.predecode_layer(st, z["pre_q"], z["pre_k"], z["pre_v"])
    np.testing.assert_allclose(pre["out"], z["pre_out"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(pre["agg"][0], z["pre_agg"], rtol=1e-5, atol=1e-7)
    assert pre["picked"][0] == tuple(z["pre_picked"].tolist())
    st.pinned[0] = pre["picked"][0]
    for i in range(int(z["steps"])):
        res = R.decode_layer(st, z["q"][i], z["k_new"][i], z["v_new"][i])
        np.testing.assert_allclose(res["out"], z["out"][i], rtol=1e-5, atol=1e-6)
        n = st.n - 1
        np.testing.assert_allclose(res["agg"][0], z["agg"][i][:n], rtol=1e-5, atol=1e-7)
        np.testing.assert_allclose(res["pinned_mass"], z["pinned_mass"][i], rtol=1e-5, atol=1e-7)
        exp_pick = tuple(p for p in z["picked"][i].tolist() if p >= 0)
        assert res["picked"][0] == exp_pick
        assert res["new"][0] == [p for p in z["new"][i].tolist() if p >= 0]
        st.pinned[0] = res["picked"][0]


def test_select_topk_kats():
    # test_engine.py:55-76
    assert R.select_topk(np.array([0.1, 0.9, 0.5]), 2, range(3)) == (1, 2)
    assert R.select_topk(np.array([0.5, 0.5, 0.5]), 2, range(3)) == (0, 1)
    assert R.select_topk(np.array([1.0]), 0, range(1)) == ()
    assert R.select_topk(np.array([]), 3, []) == ()
    assert R.select_topk(np.array([0.3, 0.1, 0.2]), 10, [0, 2]) == (0, 2)


def test_memory_ratio_table():
    # test_acceptance.py:45-58
    for length, bits, g, ratio in [(4096, 2, 32, 0.22), (4096, 2, 64, 0.19),
                                   (32768, 2, 32, 0.19), (32768, 1, 64, 0.10),
                                   (8192, 1, 32, 0.14), (8192, 2, 64, 0.17)]:
        assert R.memory_ratio(bits, g, length, 128) == ratio


def test_quantizer_kats():
    # test_quant.py:10-24 (params), 35-59 (codes, clamp, degenerate), 63-72 (levels, round trip)
    z, s = R.quant_params(np.array([[0.0, 0.3, 1.0]]), 1)
    assert (z[0], s[0]) == (0.25, 0.5)
    z, s = R.quant_params(np.array([[0.0, 1.0, 2.0, 3.0]]), 2)
    assert (z[0], s[0]) == (0.0, 1.0)
    z, s = R.quant_params(np.array([[7.0, 7.0, 7.0]]), 2)
    assert (z[0], s[0]) == (7.0, 0.0)
    g = np.array([[0.0, 0.3, 0.5, 1.0]])
    assert R.quantize(g, *R.quant_params(g, 1), 1)[0].tolist() == [0, 0, 1, 1]   # boundary maps up
    g = np.array([[0.0, 1.0, 2.0, 3.0]])
    zs = R.quant_params(g, 2)
    c = R.quantize(g, *zs, 2)
    assert c[0].tolist() == [0, 1, 2, 3]
    assert R.dequantize(c, *zs)[0].tolist() == [0.0, 1.0, 2.0, 3.0]
    g = np.array([[3.0, 3.0]])
    zs = R.quant_params(g, 2)
    assert R.quantize(g, *zs, 2)[0].tolist() == [0, 0]
    assert R.dequantize(R.quantize(g, *zs, 2), *zs)[0].tolist() == [3.0, 3.0]
    rng = np.random.default_rng(0)
    for _ in range(200):
        g = (rng.standard_normal(int(rng.integers(2, 40))) * rng.uniform(0.1, 10))[None]
        for bits in (1, 2, 4):
            c = R.quantize(g, *R.quant_params(g, bits), bits)
            assert c.min() >= 0 and c.max() <= (1 << bits) - 1
    g = np.concatenate([[0.0, 1.0], rng.random(14)])[None]
    zs = R.quant_params(g, 1)
    assert set(np.unique(R.dequantize(R.quantize(g, *zs, 1), *zs))) <= {np.float32(0.25), np.float32(0.75)}
