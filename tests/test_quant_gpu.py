"""K1 quantizer + K6 append/migration + parity readers, on the device, against
fixtures produced by the reference (bit-exact) and the pinned oracle."""
import numpy as np
import pytest

from conftest import golden
from oracle import restate as R
from oracle.synth import make_kv

pytestmark = pytest.mark.gpu

TAGS = ["b2_d128", "b1_d128", "b4_d128", "b16_d128", "b2_d10_g4", "b1_d8_g4", "b2_d128_g64", "b1_d128_g64"]


def _cache(c, mode, batch=1):
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache
    K, V = c["K"], c["V"]
    n, H, d = K.shape
    budget = CacheBudget(bits=int(c["bits"]), group_size=int(c["g"]), residual=int(c["r"]),
                         prefetch_k=int(c["k"]), context_length=max(256, n + 8))
    cache = DeviceTwoTierCache(1, H, d, budget, batch=batch)
    if mode == "prefill":
        cache.prefill(0, np.broadcast_to(K, (batch,) + K.shape), np.broadcast_to(V, (batch,) + V.shape))
    else:
        for i in range(n):
            cache.append_verified(0, np.broadcast_to(K[i], (batch, H, d)), np.broadcast_to(V[i], (batch, H, d)))
    return cache


@pytest.mark.parametrize("mode", ["prefill", "append"])
@pytest.mark.parametrize("tag", TAGS)
def test_packed_tier_bit_exact_vs_reference_snapshot(tag, mode):
    c = golden(f"cache_{tag}.npz")
    cache = _cache(c, mode)
    f = int(c["frontier"])
    assert cache.quantized_frontier(0) == f
    assert cache.length(0) == c["K"].shape[0]
    if int(c["bits"]) != 16:
        e = cache.export_packed(0)
        assert np.array_equal(e["key_codes"], c["key_codes"])
        assert np.array_equal(e["key_zero"].view(np.uint16), c["key_zero16"])
        assert np.array_equal(e["key_scale"].view(np.uint16), c["key_scale16"])
        assert np.array_equal(e["val_codes"], c["val_codes"])
        assert np.array_equal(e["val_zero"].view(np.uint16), c["val_zero16"])
        assert np.array_equal(e["val_scale"].view(np.uint16), c["val_scale16"])
    cache.pin(0, [int(p) for p in c["pins"]])
    assert cache.pinned_positions(0) == tuple(sorted(int(p) for p in c["pins"]))
    for h in range(c["K"].shape[1]):
        mk, mv = cache.materialize(0, h)
        assert np.array_equal(mk.view(np.uint32), c["mat_k"][:, h].view(np.uint32)), f"keys head {h}"
        assert np.array_equal(mv.view(np.uint32), c["mat_v"][:, h].view(np.uint32)), f"values head {h}"
    cache.close()


def test_snapshot_dict_matches_reference_format():
    c = golden("cache_b2_d10_g4.npz")
    cache = _cache(c, "append")
    snap = cache.snapshot()
    layer = snap["layers"][0]
    assert layer["quantized_frontier"] == int(c["frontier"])
    blk = layer["blocks"][1]
    head = blk["heads"][2]
    grp = head["key_groups"][7]
    assert set(grp) == {"codes", "count", "bits", "zero_fp16", "scale_fp16"}
    assert bytes.fromhex(grp["codes"]) == c["key_codes"][1, 2, 7].tobytes()[:1]
    assert int.from_bytes(bytes.fromhex(grp["zero_fp16"]), "little") == c["key_zero16"][1, 2, 7]
    assert [len(r) for r in head["value_rows"]] == [3] * 4   # 4+4+2 channels, ragged
    cache.close()


def test_batch_sequences_are_independent():
    rng = np.random.default_rng(3)
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache
    K, V = make_kv(rng, 300, 2, 128)
    K2, V2 = make_kv(rng, 300, 2, 128)
    budget = CacheBudget(bits=2, group_size=32, residual=32, prefetch_k=8, context_length=512)
    cache = DeviceTwoTierCache(1, 2, 128, budget, batch=2)
    cache.prefill(0, np.stack([K, K2]), np.stack([V, V2]))
    f = R.frontier(300, 32, 32)
    for seq, (k, v) in enumerate([(K, V), (K2, V2)]):
        e = cache.export_packed(0, seq)
        o = R.normative_export(k, v, f, 2, 32)
        assert np.array_equal(e["key_codes"], o["key_codes"])
        assert np.array_equal(e["val_codes"], o["val_codes"])
        mk, _ = R.materialize_all(k, v, f, 2, 32)
        dk, _ = cache.materialize(0, 1, seq)
        assert np.array_equal(dk, mk[:, 1])
    cache.close()


def test_migrate_and_pin_errors():
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache
    rng = np.random.default_rng(4)
    cache = DeviceTwoTierCache(1, 2, 8, CacheBudget(bits=2, group_size=4, residual=4, prefetch_k=2,
                                                    context_length=64))
    with pytest.raises(ValueError):
        cache.migrate_residual(0)          # kvcache.py:175-177
    K, V = make_kv(rng, 16, 2, 8)
    for i in range(16):
        cache.append_verified(0, K[i], V[i])
    with pytest.raises(ValueError):
        cache.pin(0, [0, 1, 2])            # larger than the prefetch budget
    with pytest.raises(ValueError):
        cache.pin(0, [cache.quantized_frontier(0)])   # residual window
    with pytest.raises(ValueError):
        cache.slow_fetch(0, [16])
    k, v, nbytes = cache.slow_fetch(0, [3, 0, 7])
    assert np.array_equal(k[0], K[3]) and np.array_equal(v[2], V[7])
    assert nbytes == cache.row_bytes(3)
    cache.pin(0, [0, 1])
    cache.pin(0, [2])
    assert cache.pinned_positions(0) == (2,)
    cache.pin(0, [])
    assert cache.pinned_positions(0) == ()
    cache.close()


def test_full_size_c2_layer_properties():
    """C2 geometry (b=16, ctx 32k, 32 heads, 2-bit): sampled blocks bit-exact
    vs the oracle, frontier rule, slow tier round trip."""
    import torch
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache
    b, n, H, d = 16, 32768, 32, 128
    gen = torch.Generator(device="cuda").manual_seed(0)
    K = (torch.randn((b, n, H, d), device="cuda", generator=gen) +
         2 * torch.randn((1, 1, H, d), device="cuda", generator=gen)).to(torch.bfloat16)
    V = torch.randn((b, n, H, d), device="cuda", generator=gen).to(torch.bfloat16)
    budget = CacheBudget(bits=2, group_size=32, residual=64, prefetch_k=64, context_length=n + 64)
    cache = DeviceTwoTierCache(1, H, d, budget, batch=b)
    cache.prefill(0, K, V)
    f = R.frontier(n, 64, 32)
    assert cache.quantized_frontier(0) == f and cache.length(0) == n
    seq = 11
    e = cache.export_packed(0, seq)
    rng = np.random.default_rng(0)
    Ks = K[seq].float().cpu().numpy()
    Vs = V[seq].float().cpu().numpy()
    for blk in rng.choice(f // 32, size=8, replace=False):
        s = slice(blk * 32, blk * 32 + 32)
        o = R.normative_export(Ks[s], Vs[s], 32, 2, 32)
        assert np.array_equal(e["key_codes"][blk], o["key_codes"][0])
        assert np.array_equal(e["key_scale"][blk].view(np.uint16), o["key_scale"][0].view(np.uint16))
        assert np.array_equal(e["val_codes"][s], o["val_codes"])
        assert np.array_equal(e["val_zero"][s].view(np.uint16), o["val_zero"].view(np.uint16))
    k, v, _ = cache.slow_fetch(0, [0, 12345, n - 1], seq)
    assert np.array_equal(k, Ks[[0, 12345, n - 1]])
    cache.close()


@pytest.mark.parametrize("bits", [1, 2])
def test_fast_quantizer_tie_heavy_bit_exact(bits):
    """Fast-layout K1 (d=128, g=32) on integer-grid rows: (x - z)/s lands
    exactly on the 0.5 / 1.5 / 2.5 rounding boundaries for many elements, so
    the float64 fallback of the fp32 code path (and rint's half-even) is
    exercised; codes and fp16 params must equal the oracle bit for bit."""
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache
    rng = np.random.default_rng(40 + bits)
    n, H, d = 32 * 24 + 70, 2, 128
    K = rng.integers(-3, 4, size=(n, H, d)).astype(np.float32) * 0.5      # grid of 0.5: ranges of 1..3
    V = rng.integers(0, 7, size=(n, H, d)).astype(np.float32) * 0.25
    K[:, :, 5] = 1.0          # a degenerate key channel (scale 0)
    V[7, 1, 32:64] = -2.0     # a degenerate value group
    budget = CacheBudget(bits=bits, group_size=32, residual=64, prefetch_k=16, context_length=n + 8)
    cache = DeviceTwoTierCache(1, H, d, budget)
    cache.prefill(0, K[None], V[None])
    f = R.frontier(n, 64, 32)
    e = cache.export_packed(0)
    o = R.normative_export(K[:f], V[:f], f, bits, 32)
    for key in ("key_codes", "val_codes"):
        assert np.array_equal(e[key], o[key]), key
    for key in ("key_zero", "key_scale", "val_zero", "val_scale"):
        assert np.array_equal(e[key].view(np.uint16), o[key].view(np.uint16)), key
    cache.close()
