"""Step graphs (spc_graph_begin / spc_graph_launch, decode.step_graph): the
decode calls of a step captured and replayed as one CUDA graph must give the
eager calls' results bit for bit -- outputs, pinned mass, tickets and the
packed tier -- across steps whose shape changes (migrations every g steps
re-instantiate the graph, the other steps update it in place).  Also the
protocol: nothing but spc_decode_layer between begin and launch."""
import numpy as np
import pytest

from oracle.synth import make_kv, make_queries, make_step_kv

pytestmark = pytest.mark.gpu


def _setup(rng_seed, layers, b, H, Hq, n0, bits):
    import torch
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder
    rng = np.random.default_rng(rng_seed)
    d, g, r, k = 128, 32, 64, 32
    budget = CacheBudget(bits=bits, group_size=g, residual=r, prefetch_k=k, context_length=n0 + 80)
    cache = DeviceTwoTierCache(layers, H, d, budget, batch=b, q_heads=Hq)
    for layer in range(layers):
        KV = [make_kv(rng, n0, H, d) for _ in range(b)]
        cache.prefill(layer, np.stack([x[0] for x in KV]), np.stack([x[1] for x in KV]))
    dec = SpeculativeLayerDecoder(cache)
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda:0").to(torch.bfloat16)
    for layer in range(layers):
        q = np.stack([make_queries(rng, 1, Hq, d) for _ in range(b)])
        kn, vn = zip(*[make_step_kv(rng, 1, H, d) for _ in range(b)])
        dec.predecode_layer(layer, bf(q), bf(np.stack(kn)), bf(np.stack(vn)))
    return cache, dec, rng, bf


@pytest.mark.parametrize("bits,H,Hq", [(2, 4, 4), (1, 2, 8)])
def test_step_graph_equals_eager(bits, H, Hq):
    import torch
    layers, b, n0, d, steps = 2, 2, 600, 128, 40
    ca, da, rng, bf = _setup(5, layers, b, H, Hq, n0, bits)
    cb, db, _, _ = _setup(5, layers, b, H, Hq, n0, bits)
    ins = []
    for t in range(steps):
        per = []
        for layer in range(layers):
            q = np.stack([make_queries(rng, 2, Hq, d) for _ in range(b)])
            kn, vn = zip(*[make_step_kv(rng, 2, H, d) for _ in range(b)])
            per.append((bf(q), bf(np.stack(kn)), bf(np.stack(vn))))
        ins.append(per)
    outs_a = [[torch.empty((b, 2, Hq, d), dtype=torch.bfloat16, device="cuda:0") for _ in range(layers)]
              for _ in range(steps)]
    outs_b = [[torch.empty_like(o) for o in row] for row in outs_a]
    pm_a = [[torch.empty((b, Hq), dtype=torch.float32, device="cuda:0") for _ in range(layers)] for _ in range(steps)]
    pm_b = [[torch.empty_like(p) for p in row] for row in pm_a]
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for t in range(steps):
            for layer in range(layers):
                da.decode_layer(layer, t + 1, *ins[t][layer], out=outs_a[t][layer], pinned_mass=pm_a[t][layer])
            with db.step_graph():
                for layer in range(layers):
                    db.decode_layer(layer, t + 1, *ins[t][layer], out=outs_b[t][layer], pinned_mass=pm_b[t][layer])
    torch.cuda.synchronize()
    for t in range(steps):
        for layer in range(layers):
            assert torch.equal(outs_a[t][layer].view(torch.int16), outs_b[t][layer].view(torch.int16)), (t, layer)
            assert torch.equal(pm_a[t][layer].view(torch.int32), pm_b[t][layer].view(torch.int32)), (t, layer)
    for layer in range(layers):
        pa, na = da.ticket(layer)
        pb, nb = db.ticket(layer)
        assert torch.equal(pa, pb) and torch.equal(na, nb)
        assert ca.quantized_frontier(layer) == cb.quantized_frontier(layer) > n0 - 64 - 32
        for s in range(b):
            ea, eb = ca.export_packed(layer, seq=s), cb.export_packed(layer, seq=s)
            for key in ("key_codes", "val_codes", "key_zero", "key_scale", "val_zero", "val_scale"):
                assert np.array_equal(np.asarray(ea[key]).view(np.uint8), np.asarray(eb[key]).view(np.uint8)), key
    inst, upd = db.graph_stats()
    assert inst >= 2 and upd >= steps // 2, (inst, upd)   # migrations re-instantiate, the rest update
    # an eager step after graph steps still orders behind them
    with torch.cuda.stream(side):
        q, kn, vn = ins[-1][0]
        o1 = da.decode_layer(0, steps + 1, q, kn, vn).out
        o2 = db.decode_layer(0, steps + 1, q, kn, vn).out
    torch.cuda.synchronize()
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
    ca.close()
    cb.close()


def test_step_graph_protocol():
    import torch
    from paper_2503_16163_b200 import ProtocolError, _lib
    cache, dec, rng, bf = _setup(9, 1, 1, 2, 2, 300, 2)
    side = torch.cuda.Stream()
    q = bf(np.stack([make_queries(rng, 2, 2, 128)]))
    kn, vn = make_step_kv(rng, 2, 2, 128)
    kn, vn = bf(kn[None]), bf(vn[None])
    out = torch.empty((1, 2, 2, 128), dtype=torch.bfloat16, device="cuda:0")
    pm = torch.empty((1, 2), dtype=torch.float32, device="cuda:0")
    with torch.cuda.stream(side):
        with pytest.raises(ProtocolError):
            with dec.step_graph():
                dec.decode_layer(0, 1, q, kn, vn, out=out, pinned_mass=pm)
                _lib.check(_lib.lib().spc_migrate(cache.handle, 0, side.cuda_stream))  # not allowed here
    cache.close()
    # the legacy default stream cannot be captured
    cache, dec, rng, bf = _setup(9, 1, 1, 2, 2, 300, 2)
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().spc_graph_begin(cache.handle, 0))
    cache.close()
