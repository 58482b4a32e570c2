"""Regression tests for the round-1 advisor findings:

- export right after a decode step whose append triggers a migration (the
  migration runs on the layer's copy stream; export must wait for it);
- odd group sizes on the generic quantizer (float64 param slots must stay
  8-byte aligned);
- select_topk with -0.0 scores (the reference treats -0.0 == 0.0);
- the adapter decoding past max_len / context_length like the reference."""
import numpy as np
import pytest

from oracle import restate as R
from oracle.synth import make_kv, make_queries, make_step_kv

pytestmark = pytest.mark.gpu


def test_export_after_decode_triggered_migration():
    """n0 = 1023, r = 64, g = 32: residual = 95 = r + g - 1, so the first decode
    step's append migrates one block (f: 928 -> 960) on the copy stream.  The
    export issued right after decode_layer (no host sync) must see it."""
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder
    rng = np.random.default_rng(3)
    b, n0, H, Hq, d, bits, g, r, k = 4, 1023, 8, 32, 128, 2, 32, 64, 64
    KV = [make_kv(rng, n0, H, d) for _ in range(b)]
    budget = CacheBudget(bits=bits, group_size=g, residual=r, prefetch_k=k, context_length=n0 + 8)
    cache = DeviceTwoTierCache(1, H, d, budget, batch=b, q_heads=Hq)
    cache.prefill(0, np.stack([x[0] for x in KV]), np.stack([x[1] for x in KV]))
    assert cache.quantized_frontier(0) == 928
    dec = SpeculativeLayerDecoder(cache)
    q = np.stack([make_queries(rng, 1, Hq, d) for _ in range(b)])
    kn, vn = zip(*[make_step_kv(rng, 1, H, d) for _ in range(b)])
    dec.predecode_layer(0, q, np.stack(kn), np.stack(vn))
    q2 = np.stack([make_queries(rng, 2, Hq, d) for _ in range(b)])
    kn, vn = zip(*[make_step_kv(rng, 2, H, d) for _ in range(b)])
    dec.decode_layer(0, 1, q2, np.stack(kn), np.stack(vn))
    for s in (b - 1, 0):
        e = cache.export_packed(0, seq=s)         # no synchronize in between
        assert e["frontier"] == 960
        K = np.concatenate([KV[s][0], kn[s][:1]])
        V = np.concatenate([KV[s][1], vn[s][:1]])
        ref = R.normative_export(K, V, 960, bits, g)
        for key in ("key_codes", "val_codes"):
            assert np.array_equal(e[key], ref[key]), key
        for key in ("key_zero", "key_scale", "val_zero", "val_scale"):
            assert np.array_equal(e[key].view(np.uint16), ref[key].view(np.uint16)), key
    cache.close()


@pytest.mark.parametrize("mode", ["prefill", "append"])
@pytest.mark.parametrize("g,d,bits", [(5, 8, 2), (3, 10, 1), (7, 14, 4)])
def test_odd_group_size_generic_quantizer(g, d, bits, mode):
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache
    rng = np.random.default_rng(g * 100 + d)
    n, H, r = 61, 2, 4
    K, V = make_kv(rng, n, H, d)
    budget = CacheBudget(bits=bits, group_size=g, residual=r, prefetch_k=4, context_length=n + 8)
    cache = DeviceTwoTierCache(1, H, d, budget)
    if mode == "prefill":
        cache.prefill(0, K[None], V[None])
    else:
        for i in range(n):
            cache.append_verified(0, K[i][None], V[i][None])
    f = R.frontier(n, r, g)
    assert cache.quantized_frontier(0) == f
    e = cache.export_packed(0)
    ref = R.normative_export(K, V, f, bits, g)
    for key in ("key_codes", "val_codes"):
        assert np.array_equal(e[key], ref[key]), key
    for key in ("key_zero", "key_scale", "val_zero", "val_scale"):
        assert np.array_equal(e[key].view(np.uint16), ref[key].view(np.uint16)), key
    Kt, Vt = R.materialize_all(K, V, f, bits, g)
    for h in range(H):
        mk, mv = cache.materialize(0, h)
        assert np.array_equal(mk, Kt[:, h]) and np.array_equal(mv, Vt[:, h])
    cache.close()


def test_select_topk_negative_zero():
    from paper_2503_16163_b200 import select_topk
    s = np.array([0.0, -0.0, 0.5, -0.0, 0.0], np.float32)
    assert select_topk(s, 2) == R.select_topk(s, 2, range(5)) == (0, 2)
    assert select_topk(s, 4) == R.select_topk(s, 4, range(5)) == (0, 1, 2, 3)


def test_adapter_decodes_past_max_len():
    """The reference decodes past max_len and context_length (engine.py:286-339
    has no length check); so must the adapter."""
    from types import SimpleNamespace

    from conftest import golden
    from paper_2503_16163_b200 import CacheBudget, ChannelModel
    from paper_2503_16163_b200.adapter import generate
    z = golden("adapter_b2.npz")
    cfg = SimpleNamespace(**{k[4:]: int(z[k]) for k in z.files if k.startswith("cfg_") and k != "cfg_rope_base"})
    cfg.rope_base = float(z["cfg_rope_base"])
    layers = [SimpleNamespace(**{nm: z[f"w_{i}_{nm}"] for nm in
                                 ("wq", "wk", "wv", "wo", "attn_norm", "ffn_norm", "w1", "w2")})
              for i in range(cfg.layers)]
    w = SimpleNamespace(embedding=z["w_embedding"], layers=layers, final_norm=z["w_final_norm"],
                        head=z["w_head"])
    prompt = [int(t) % cfg.vocab for t in range(1, 41)]
    cfg.max_len = 48
    budget = CacheBudget(bits=2, group_size=8, residual=8, prefetch_k=8, context_length=48)
    res = generate(cfg, w, prompt, 20, budget, ChannelModel(bandwidth=1e6))   # 40 + 20 > 48
    assert len(res.tokens) == 21


def test_debug_and_measurement_entry_points():
    """Round-2 C ABI additions: the fp32 debug output (off -> ValueError), the
    prefetch wall-time union and the host-link peak probe."""
    import ctypes

    import torch
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder, _lib
    rng = np.random.default_rng(8)
    K, V = make_kv(rng, 600, 2, 128)
    cache = DeviceTwoTierCache(1, 2, 128, CacheBudget(bits=2, group_size=32, residual=64, prefetch_k=32,
                                                      context_length=640), q_heads=8)
    cache.prefill(0, K[None], V[None])
    dec = SpeculativeLayerDecoder(cache)
    with pytest.raises(ValueError):
        dec.debug_out_f32(0, 1)                    # not enabled
    dec.debug_output_f32(True)
    q = make_queries(rng, 1, 8, 128)
    kn, vn = make_step_kv(rng, 1, 2, 128)
    out = dec.predecode_layer(0, q[None], kn[None], vn[None])
    o32 = dec.debug_out_f32(0, 1)
    assert torch.equal(out.float(), o32.to(torch.bfloat16).float())
    cache.profile(True)
    q2 = make_queries(rng, 2, 8, 128)
    kn, vn = make_step_kv(rng, 2, 2, 128)
    dec.decode_layer(0, 1, q2[None], kn[None], vn[None])
    prof = cache.profile(False)
    wall = _lib.lib().spc_profile_prefetch_wall_ms(cache.handle)
    assert 0.0 <= wall <= prof["prefetch_ms"] + 1e-6
    cache.close()
    dma, zc = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.lib().spc_h2d_peak(0, 64 << 20, ctypes.byref(dma), ctypes.byref(zc)))
    assert 1.0 < dma.value < 200.0 and 1.0 < zc.value < 200.0
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().spc_h2d_peak(0, 1000, ctypes.byref(dma), ctypes.byref(zc)))
