"""the full decoder step around the hot path (decoder.py,
csrc/layer.cu).

Kernel checks against torch fp32 formulas of the reference's numerics
(numerics.py:42-78, engine.py:35-36): bf16 outputs within one bf16 ulp, the
fp32 residual update and the argmax (ties -> lowest index) exact.  Stack check:
DecoderStack (cuBLAS bf16 GEMMs + fused kernels + spc_decode_layer) against a
torch emulation with the same rounding points on a twin cache.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ULP = 2.0 ** -7  # one bf16 ulp, relative


def _lib():
    from paper_2503_16163_b200 import _lib
    return _lib


def _st():
    import torch
    return torch.cuda.current_stream().cuda_stream


def _rms(x, gain, eps=1e-6):
    import torch
    return x * gain / torch.sqrt(torch.mean(x * x, dim=-1, keepdim=True) + eps)


def test_add_rmsnorm():
    import torch
    L = _lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    for rows, hidden, with_delta in [(32, 4096, True), (7, 264, False), (1, 8, True)]:
        x = torch.randn(rows, hidden, device="cuda", generator=g) * 3
        d = torch.randn(rows, hidden, device="cuda", generator=g).bfloat16()
        gain = torch.rand(hidden, device="cuda", generator=g) + 0.5
        out = torch.empty(rows, hidden, dtype=torch.bfloat16, device="cuda")
        x0 = x.clone()
        L.check(L.lib().spc_add_rmsnorm(x.data_ptr(), d.data_ptr() if with_delta else None, gain.data_ptr(),
                                        out.data_ptr(), rows, hidden, 1e-6, _st()))
        xe = x0 + d.float() if with_delta else x0
        assert torch.equal(x, xe)
        torch.testing.assert_close(out.float(), _rms(xe, gain), rtol=ULP, atol=1e-6)
    with pytest.raises(ValueError, match="multiple of 8"):
        L.check(L.lib().spc_add_rmsnorm(x.data_ptr(), None, gain.data_ptr(), out.data_ptr(), 1, 12, 1e-6, _st()))


def test_qkv_rope():
    import torch
    L = _lib()
    rows, Hq, Hkv, d, base = 6, 4, 2, 128, 10000.0
    g = torch.Generator(device="cuda").manual_seed(1)
    qkv = torch.randn(rows, (Hq + 2 * Hkv) * d, device="cuda", generator=g).bfloat16()
    pos = torch.tensor([0, 1, 5, 4095, 32767, 131071], dtype=torch.int32, device="cuda")
    q = torch.empty(rows, Hq, d, dtype=torch.bfloat16, device="cuda")
    k = torch.empty(rows, Hkv, d, dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    tab = torch.empty(rows, d, dtype=torch.float32, device="cuda")
    L.check(L.lib().spc_rope_table(pos.data_ptr(), rows, d, base, tab.data_ptr(), _st()))
    L.check(L.lib().spc_qkv_rope(qkv.data_ptr(), tab.data_ptr(), rows, Hq, Hkv, d, q.data_ptr(),
                                 k.data_ptr(), v.data_ptr(), _st()))
    src = qkv.float().cpu().numpy().reshape(rows, Hq + 2 * Hkv, d)
    idx = np.arange(d // 2, dtype=np.float64)
    ang = pos.cpu().numpy().astype(np.float64)[:, None] * base ** (-2.0 * idx / d)   # numerics.py:62
    cos, sin = np.cos(ang).astype(np.float32)[:, None], np.sin(ang).astype(np.float32)[:, None]
    x0, x1 = src[..., 0::2], src[..., 1::2]
    rot = np.empty_like(src)
    rot[..., 0::2] = x0 * cos - x1 * sin
    rot[..., 1::2] = x0 * sin + x1 * cos
    tc = tab.cpu().numpy().reshape(rows, d // 2, 2)
    np.testing.assert_allclose(tc[..., 0], cos[:, 0], rtol=0, atol=2e-7)
    np.testing.assert_allclose(tc[..., 1], sin[:, 0], rtol=0, atol=2e-7)
    torch.testing.assert_close(q.float().cpu(), torch.from_numpy(rot[:, :Hq]), rtol=ULP, atol=1e-5)
    torch.testing.assert_close(k.float().cpu(), torch.from_numpy(rot[:, Hq:Hq + Hkv]), rtol=ULP, atol=1e-5)
    assert torch.equal(v.float().cpu(), torch.from_numpy(src[:, Hq + Hkv:]))


def test_silu_and_argmax():
    import torch
    L = _lib()
    g = torch.Generator(device="cuda").manual_seed(2)
    a = (torch.randn(64, 1000, device="cuda", generator=g) * 4).bfloat16()
    ref = torch.nn.functional.silu(a.float())
    L.check(L.lib().spc_silu(a.data_ptr(), a.numel(), _st()))
    torch.testing.assert_close(a.float(), ref, rtol=ULP, atol=1e-6)
    # argmax with planted ties (lowest index wins, numerics.py:73-78)
    x = torch.randn(9, 32000, device="cuda", generator=g).bfloat16()
    x[1, [7, 900, 31999]] = 50.0
    x[2, [31998, 31999]] = 60.0
    x[3] = 0.0
    out = torch.empty(9, dtype=torch.int32, device="cuda")
    L.check(L.lib().spc_argmax_rows(x.data_ptr(), 9, 32000, out.data_ptr(), _st()))
    exp = np.argmax(x.float().cpu().numpy(), axis=1)
    assert out.cpu().numpy().tolist() == exp.tolist()
    assert out[1].item() == 7 and out[2].item() == 31998 and out[3].item() == 0


def _emulate(cfg, W, dec, rows, step, tokens, pos):
    """Torch fp32 with bf16 rounding at the stack's rounding points."""
    import torch
    bf = lambda t: t.bfloat16().float()
    B = rows if step is None else rows // 2
    x = W.emb[tokens.reshape(-1).long()].float()
    d, Hq, Hkv = cfg.head_dim, cfg.q_heads, cfg.kv_heads
    idx = torch.arange(d // 2, dtype=torch.float64, device="cuda")
    ang = pos.double()[:, None] * cfg.rope_base ** (-2.0 * idx / d)
    cos, sin = torch.cos(ang).float()[:, None], torch.sin(ang).float()[:, None]

    def rope(t):
        o = torch.empty_like(t)
        o[..., 0::2] = t[..., 0::2] * cos - t[..., 1::2] * sin
        o[..., 1::2] = t[..., 0::2] * sin + t[..., 1::2] * cos
        return bf(o)

    delta = None
    for layer, lw in enumerate(W.layers):
        if delta is not None:
            x = x + delta
        xn = bf(_rms(x, lw["attn_norm"]))
        qkv = bf(xn @ lw["wqkv"].float().t())
        q = rope(qkv[:, :Hq * d].reshape(rows, Hq, d))
        k = rope(qkv[:, Hq * d:(Hq + Hkv) * d].reshape(rows, Hkv, d))
        v = qkv[:, (Hq + Hkv) * d:].reshape(rows, Hkv, d)
        r = 1 if step is None else 2
        q, k, v = (t.reshape(B, r, -1, d).bfloat16() for t in (q, k, v))
        if step is None:
            out = dec.predecode_layer(layer, q, k, v)
        else:
            out = dec.decode_layer(layer, step, q, k, v).out
        delta = bf(out.float().reshape(rows, -1) @ lw["wo"].float().t())
        x = x + delta
        xn = bf(_rms(x, lw["ffn_norm"]))
        h = bf(xn @ lw["w1"].float().t())
        h = bf(h / (1 + torch.exp(-h)))
        delta = bf(h @ lw["w2"].float().t())
    x = x + delta
    return bf(bf(_rms(x, W.final_norm)) @ W.head.float().t())


def test_stack_matches_emulation():
    import torch
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder
    from paper_2503_16163_b200.decoder import DecoderStack, stack_from_reference
    from paper_2503_16163_b200.weights import DecoderConfig, init_decoder
    torch.backends.cuda.matmul.allow_tf32 = False
    rc = DecoderConfig(layers=2, q_heads=8, kv_heads=2, head_dim=128, vocab=512, hidden=256, ffn=512, seed=4)
    cfg, W = stack_from_reference(rc, init_decoder(rc))
    B, n0 = 3, 400
    budget = CacheBudget(bits=2, group_size=32, residual=64, prefetch_k=16, context_length=1024)
    caches = [DeviceTwoTierCache(cfg.layers, cfg.kv_heads, cfg.head_dim, budget, batch=B, q_heads=cfg.q_heads)
              for _ in range(2)]
    g = torch.Generator(device="cuda").manual_seed(5)
    for layer in range(cfg.layers):
        K = torch.randn(B, n0, cfg.kv_heads, cfg.head_dim, device="cuda", generator=g).bfloat16()
        V = torch.randn(B, n0, cfg.kv_heads, cfg.head_dim, device="cuda", generator=g).bfloat16()
        for c in caches:
            c.prefill(layer, K, V)
    stack, dec = DecoderStack(cfg, W, caches[0]), SpeculativeLayerDecoder(caches[1])
    tok = torch.randint(0, cfg.vocab, (B,), device="cuda", generator=g)
    pos = torch.full((B,), n0, dtype=torch.int32, device="cuda")
    got = stack.predecode(tok, pos).clone()
    ref = _emulate(cfg, W, dec, B, None, tok, pos)
    torch.testing.assert_close(stack.logits[:B].float(), ref, rtol=3e-2, atol=3e-2 * ref.abs().max().item())
    spec = got.long()
    ver = torch.randint(0, cfg.vocab, (B,), device="cuda", generator=g)
    for step in range(1, 4):
        toks = torch.stack([ver, spec], dim=1)
        nxt = stack.decode_step(step, toks, pos).clone()
        p2 = torch.stack([pos, pos + 1], dim=1).reshape(-1)
        ref = _emulate(cfg, W, dec, 2 * B, step, toks, p2)
        lg = stack.logits.float()
        torch.testing.assert_close(lg, ref, rtol=3e-2, atol=3e-2 * ref.abs().max().item())
        top2 = torch.topk(ref, 2, dim=1).values
        clear = (top2[:, 0] - top2[:, 1]) > 0.05 * ref.abs().max()
        assert torch.equal(nxt.reshape(-1)[clear].long(), ref.argmax(dim=1)[clear])
        assert nxt.reshape(-1).cpu().numpy().tolist() == np.argmax(lg.cpu().numpy(), axis=1).tolist()
        ver, spec, pos = nxt[:, 0].long(), nxt[:, 1].long(), pos + 1
    for c in caches:
        c.close()
