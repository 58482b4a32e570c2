"""KV-head sharding of the decode hot path (shard.py) on the device.

Two ranks (spawned processes, gloo process group -- the box has one GPU, so
both ranks share cuda:0; on a multi-GPU box the same code runs one rank per
GPU over NCCL) each own half of the kv heads of every sequence.  With
layer-scope top-k the partial aggregates are summed across ranks on the
cache's copy stream (spc_set_agg_reduce / spc_agg_buffer / spc_finish_layer)
before the selection.  Every rank must reproduce the single-process run: its
heads' outputs and pinned mass, the summed aggregate, and the same ticket
(picked positions, new-pin counts) at every step.  kv_head scope runs with no
exchange at all.
"""
import os
import socket

import numpy as np
import pytest

from oracle import restate as R
from oracle.synth import make_kv, make_queries, make_step_kv

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(cfg, steps):
    b, n0, H, Hq, d = cfg["b"], cfg["n0"], cfg["H"], cfg["Hq"], cfg["d"]
    rng = np.random.default_rng(cfg["seed"])
    KV = [make_kv(rng, n0, H, d) for _ in range(b)]
    K = np.stack([x[0] for x in KV])
    V = np.stack([x[1] for x in KV])
    pre = (np.stack([make_queries(rng, 1, Hq, d) for _ in range(b)]),
           *map(np.stack, zip(*[make_step_kv(rng, 1, H, d) for _ in range(b)])))
    q = np.stack([make_queries(rng, 2, Hq, d) for _ in range(b)])
    dec = []
    for _ in range(steps):
        kn, vn = zip(*[make_step_kv(rng, 2, H, d) for _ in range(b)])
        dec.append((q, np.stack(kn), np.stack(vn)))
        q = R.bf16_round((q + 0.3 * rng.standard_normal(q.shape)).astype(np.float32))
    return K, V, pre, dec


def _run(cfg, rank, world, steps=3, reduce=None):
    """Predecode + `steps` decode steps on this rank's head shard; returns
    per-step (out, pinned_mass, agg, picked, new_count) as numpy."""
    import torch
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder
    from paper_2503_16163_b200.shard import head_shard
    sh = head_shard(cfg["H"], cfg["Hq"], rank, world)
    K, V, pre, dec_in = _inputs(cfg, steps)
    budget = CacheBudget(bits=cfg["bits"], group_size=32, residual=64, prefetch_k=cfg["k"],
                         context_length=cfg["n0"] + steps + 8)
    cache = DeviceTwoTierCache(1, sh.kv_heads, cfg["d"], budget, batch=cfg["b"], q_heads=sh.q_heads,
                               topk_scope=cfg["scope"])
    cache.prefill(0, sh.slice_kv(K), sh.slice_kv(V))
    dec = SpeculativeLayerDecoder(cache, agg_reduce=reduce)
    res = []
    o = dec.predecode_layer(0, sh.slice_q(pre[0]), sh.slice_kv(pre[1]), sh.slice_kv(pre[2]))
    picked, newc = dec.ticket(0)
    res.append((o.float().cpu().numpy(), None, dec.debug_agg(0).cpu().numpy(), picked.cpu().numpy(),
                newc.cpu().numpy()))
    for t, (q, kn, vn) in enumerate(dec_in, start=1):
        r = dec.decode_layer(0, t, sh.slice_q(q), sh.slice_kv(kn), sh.slice_kv(vn))
        picked, newc = dec.ticket(0)
        torch.cuda.synchronize()
        res.append((r.out.float().cpu().numpy(), r.pinned_mass.cpu().numpy(),
                    dec.debug_agg(0).cpu().numpy(), picked.cpu().numpy(), newc.cpu().numpy()))
    f = cache.quantized_frontier(0)
    cache.close()
    return res, f


def _worker(rank, port, cfg, out_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2503_16163_b200.shard import allreduce_sum
        reduce = allreduce_sum() if cfg["scope"] == "layer" else None
        res, _ = _run(cfg, rank, WORLD, reduce=reduce)
        out_q.put((rank, res))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _sharded(cfg):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, cfg, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=400) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.timeout(600)
@pytest.mark.parametrize("bits,scope", [(2, "layer"), (1, "layer"), (2, "kv_head")])
def test_head_sharded_decode_matches_single_process(bits, scope):
    cfg = dict(seed=11 + bits, b=2, n0=1500, H=4, Hq=8, d=128, bits=bits, k=32, scope=scope)
    full, f = _run(cfg, 0, 1)
    shards = _sharded(cfg)
    from paper_2503_16163_b200.shard import head_shard
    for rank, res in shards.items():
        sh = head_shard(cfg["H"], cfg["Hq"], rank, WORLD)
        for step, ((o, pm, agg, picked, newc), (fo, fpm, fagg, fpicked, fnewc)) in enumerate(zip(res, full)):
            fo = fo[:, :, sh.q_lo:sh.q_hi]
            err = np.abs(o - fo).max() / np.abs(fo).max()
            assert err <= 8e-3, (rank, step, err)  # one bf16 ulp: split plans differ with the head count
            if pm is not None:
                np.testing.assert_allclose(pm, fpm[:, sh.q_lo:sh.q_hi], rtol=1e-5, atol=1e-7)
            if scope == "layer":  # the reduced aggregate equals the all-head one up to reassociation
                np.testing.assert_allclose(agg[..., :f], fagg[..., :f], rtol=1e-5, atol=1e-9)
                np.testing.assert_array_equal(picked, fpicked)
                np.testing.assert_array_equal(newc, fnewc)
            else:  # kv_head scope: this rank's units are the full run's units [kv_lo, kv_hi)
                np.testing.assert_allclose(agg[..., :f], fagg[:, sh.kv_lo:sh.kv_hi, :f], rtol=1e-6, atol=1e-9)
                np.testing.assert_array_equal(picked, fpicked[:, sh.kv_lo:sh.kv_hi])
                np.testing.assert_array_equal(newc, fnewc[:, sh.kv_lo:sh.kv_hi])


def test_agg_reduce_protocol():
    """Until spc_finish_layer, the layer's ticket is not readable and the next
    step is refused (ProtocolError); the reduction hook runs once per layer call."""
    import torch
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder
    from paper_2503_16163_b200 import _lib
    from paper_2503_16163_b200.transfer import ProtocolError
    cfg = dict(seed=5, b=1, n0=400, H=2, Hq=4, d=128, bits=2, k=16, scope="layer")
    K, V, pre, dec_in = _inputs(cfg, 1)
    budget = CacheBudget(bits=2, group_size=32, residual=64, prefetch_k=16, context_length=500)
    cache = DeviceTwoTierCache(1, 2, 128, budget, batch=1, q_heads=4)
    cache.prefill(0, K, V)
    calls = []

    def double(t):  # a 2-rank all-reduce of equal partials
        calls.append(t.numel())
        t.mul_(2.0)

    dec = SpeculativeLayerDecoder(cache, agg_reduce=double)
    dec.predecode_layer(0, *pre)
    assert len(calls) == 1
    lib = _lib.lib()  # raw C calls: decode without the decoder's finish hook
    q, kn, vn = (torch.as_tensor(x).to("cuda:0", torch.bfloat16).contiguous() for x in dec_in[0])
    out = torch.empty_like(q)
    pm = torch.empty((1, 4), dtype=torch.float32, device="cuda:0")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.spc_decode_layer(cache.handle, 0, 1, q.data_ptr(), kn.data_ptr(), vn.data_ptr(),
                                    out.data_ptr(), pm.data_ptr(), s))
    with pytest.raises(ProtocolError):
        dec.ticket(0)
    with pytest.raises(ProtocolError):
        _lib.check(lib.spc_decode_layer(cache.handle, 0, 2, q.data_ptr(), kn.data_ptr(), vn.data_ptr(),
                                        out.data_ptr(), pm.data_ptr(), s))
    _lib.check(lib.spc_finish_layer(cache.handle, 0))
    with pytest.raises(ProtocolError):
        _lib.check(lib.spc_finish_layer(cache.handle, 0))
    picked, newc = dec.ticket(0)
    torch.cuda.synchronize()
    assert (picked >= 0).sum().item() == 16
    cache.close()


# ---- the full decoder step with head-sharded attention + all-gather of the outputs ----
def _stack_run(rank, world, group=None):
    """Predecode + 3 decode steps of a 2-layer GQA model (8 q / 2 kv heads) with
    fixed token inputs; returns the logits of every call (numpy)."""
    import torch
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache
    from paper_2503_16163_b200.decoder import DecoderStack, stack_from_reference
    from paper_2503_16163_b200.shard import head_shard
    from paper_2503_16163_b200.weights import DecoderConfig, init_decoder
    torch.backends.cuda.matmul.allow_tf32 = False
    rc = DecoderConfig(layers=2, q_heads=8, kv_heads=2, head_dim=128, vocab=512, hidden=256, ffn=512, seed=4)
    cfg, W = stack_from_reference(rc, init_decoder(rc))
    sh = head_shard(cfg.kv_heads, cfg.q_heads, rank, world) if world > 1 else None
    B, n0 = 3, 400
    budget = CacheBudget(bits=2, group_size=32, residual=64, prefetch_k=16, context_length=1024)
    kvh, qh = (sh.kv_heads, sh.q_heads) if sh else (cfg.kv_heads, cfg.q_heads)
    cache = DeviceTwoTierCache(cfg.layers, kvh, cfg.head_dim, budget, batch=B, q_heads=qh)
    g = torch.Generator(device="cuda").manual_seed(5)
    for layer in range(cfg.layers):
        K = torch.randn(B, n0, cfg.kv_heads, cfg.head_dim, device="cuda", generator=g).bfloat16()
        V = torch.randn(B, n0, cfg.kv_heads, cfg.head_dim, device="cuda", generator=g).bfloat16()
        if sh:
            K, V = sh.slice_kv(K).contiguous(), sh.slice_kv(V).contiguous()
        cache.prefill(layer, K, V)
    stack = DecoderStack(cfg, W, cache, shard=sh, group=group)
    tok = torch.randint(0, cfg.vocab, (B,), device="cuda", generator=g)
    pos = torch.full((B,), n0, dtype=torch.int32, device="cuda")
    stack.predecode(tok, pos)
    logits = [stack.logits[:B].float().cpu().numpy()]
    for step in range(1, 4):
        toks = torch.randint(0, cfg.vocab, (B, 2), device="cuda", generator=g)
        stack.decode_step(step, toks, pos)
        logits.append(stack.logits.float().cpu().numpy())
        pos = pos + 1
    cache.close()
    return logits


def _stack_worker(rank, port, out_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        out_q.put((rank, _stack_run(rank, WORLD)))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_head_sharded_decoder_stack_matches_single_process():
    """Each rank projects and attends its heads; the all-gathered outputs feed a
    replicated Wo / FFN / head, so every rank's logits match the single-GPU stack."""
    import torch.multiprocessing as mp
    full = _stack_run(0, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stack_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=400) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, ref in enumerate(full):
        np.testing.assert_array_equal(got[0][i], got[1][i])        # replicated after the all-gather
        scale = np.abs(ref).max()
        assert np.abs(got[0][i] - ref).max() <= 2e-2 * scale, (i, np.abs(got[0][i] - ref).max() / scale)
