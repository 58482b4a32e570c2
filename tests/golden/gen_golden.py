"""Generate golden fixtures by running the REFERENCE itself (read-only import
from /root/reference/pkg/src).  Run once in the build container:

    python tests/golden/gen_golden.py

The fixtures are committed; nothing at test/bench time reads /root/reference.

Files
-----
quant_groups.npz   quantizer known-answer vectors: reference quant_params,
                   quantize_group, pack_codes, dequantize_group and the fp16
                   snapshot params for random / dyadic / degenerate / tie groups
                   (quant.py:59-160).
cache_<tag>.npz    a TwoTierCache filled with bf16-representable rows: the
                   reference snapshot() parsed into normative arrays, plus
                   materialize() for every head after pin() (kvcache.py).
decode_<tag>.npz   the per-layer body of SpeculativeDecoder.decode_step
                   (engine.py:299-321) replayed with reference objects for a
                   few steps, after predecode (engine.py:245-268).
adapter_<tag>.npz  reference generate() token streams (bf16 hot-path boundary).
report_toy.spkc    reference `gen-weights --seed 2` weight file (model.py
                   init_decoder + save_weights).
report_<tag>.json  reference experiments.run_decode() reports on that file
                   (bf16 hot-path boundary), plus the arguments used.
hitrate_rows.npz   random attention-trace sequences (flat, peaky, tied and
                   growing rows) with the reference topk_hitrate /
                   eviction_hitrate over a k sweep (hitrate.py:34-77).
hitrate_report.json reference experiments.hitrate_experiment() on
                   report_toy.spkc (FullCacheDecoder trace, experiments.py:100-137).

    python tests/golden/gen_golden.py [report]   # only the listed groups
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from speckv import engine, quant  # noqa: E402
from speckv.kvcache import CacheBudget, TwoTierCache  # noqa: E402
from speckv.model import DecoderConfig  # noqa: E402
from speckv.transfer import ChannelModel, PrefetchTicket, SimulatedChannel  # noqa: E402

from oracle.restate import bf16_round  # noqa: E402
from oracle.synth import make_kv, make_queries, make_step_kv  # noqa: E402


def gen_quant_groups():
    rng = np.random.default_rng(20250316)
    groups = []
    for size in (1, 2, 3, 4, 7, 16, 31, 32, 33, 64):
        for _ in range(6):
            groups.append((rng.standard_normal(size) * rng.uniform(0.01, 10)
                           + rng.normal(0, 3)).astype(np.float32))
    # bf16-representable groups (what the device sees)
    for _ in range(40):
        groups.append(bf16_round(rng.standard_normal(32).astype(np.float32) * 3 + 1))
    # dyadic groups: exact midpoint / threshold arithmetic (test_acceptance.py:36-42)
    for _ in range(40):
        vals = rng.integers(-4 * 64, 4 * 64, size=int(rng.integers(2, 33)))
        if vals.max() == vals.min():
            vals[0] += 64
        groups.append((vals.astype(np.float64) / 64).astype(np.float32))
    # degenerate and known-answer groups (test_quant.py)
    groups += [np.full(32, 3.0, np.float32), np.full(5, -7.25, np.float32),
               np.array([0.0, 0.3, 0.5, 1.0], np.float32),
               np.array([0.0, 1.0, 2.0, 3.0], np.float32),
               np.array([0.0, 0.3, 1.0], np.float32),
               np.array([0.0, 0.5, 1.0, 1.5], np.float32),
               # exact half-way points for 2-bit rint ties: (x-lo)/s = k+0.5
               np.array([0.0, 0.5, 1.5, 2.5, 3.0], np.float32),
               np.array([1e-30, 1.0, 3.0e-30, 0.5], np.float32),
               np.array([65504.0, -65504.0, 1.0], np.float32),
               np.array([1 + 2**-11 + 2**-20, 1.0, 3.0], np.float32)]
    out = {}
    values, offsets = [], [0]
    for g in groups:
        values.append(g)
        offsets.append(offsets[-1] + g.size)
    out["values"] = np.concatenate(values).astype(np.float32)
    out["offsets"] = np.asarray(offsets, np.int64)
    for bits in (1, 2, 4):
        codes, zeros, scales, z16, s16, packed, poff, deq = [], [], [], [], [], [], [0], []
        for g in groups:
            pg = quant.PackedGroup.from_values(g, bits)
            snap = pg.snapshot()
            c = quant.quantize_group(g, pg.params)
            codes.append(c)
            zeros.append(pg.params.zero)
            scales.append(pg.params.scale)
            z16.append(int.from_bytes(bytes.fromhex(snap["zero_fp16"]), "little"))
            s16.append(int.from_bytes(bytes.fromhex(snap["scale_fp16"]), "little"))
            packed.append(np.frombuffer(pg.codes, np.uint8))
            poff.append(poff[-1] + len(pg.codes))
            deq.append(pg.dequantize())
        out[f"b{bits}_codes"] = np.concatenate(codes).astype(np.uint8)
        out[f"b{bits}_zero"] = np.asarray(zeros, np.float64)
        out[f"b{bits}_scale"] = np.asarray(scales, np.float64)
        out[f"b{bits}_zero16"] = np.asarray(z16, np.uint16)
        out[f"b{bits}_scale16"] = np.asarray(s16, np.uint16)
        out[f"b{bits}_packed"] = np.concatenate(packed).astype(np.uint8)
        out[f"b{bits}_poff"] = np.asarray(poff, np.int64)
        out[f"b{bits}_deq"] = np.concatenate(deq).astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "quant_groups.npz"), **out)


def parse_snapshot(snap, layer, H, d, g, bits):
    """Reference snapshot dict -> normative arrays (same form as
    oracle.restate.normative_export)."""
    blocks = snap["layers"][layer]["blocks"]
    nb = len(blocks)
    f = snap["layers"][layer]["quantized_frontier"]
    nbytes = (g * bits + 7) // 8
    nchunk = (d + g - 1) // g
    kc = np.zeros((nb, H, d, nbytes), np.uint8)
    kz = np.zeros((nb, H, d), np.uint16)
    ks = np.zeros((nb, H, d), np.uint16)
    vc = np.zeros((f, H, nchunk, nbytes), np.uint8)
    vz = np.zeros((f, H, nchunk), np.uint16)
    vs = np.zeros((f, H, nchunk), np.uint16)
    for b, blk in enumerate(blocks):
        for h, head in enumerate(blk["heads"]):
            for c, grp in enumerate(head["key_groups"]):
                raw = bytes.fromhex(grp["codes"])
                kc[b, h, c, :len(raw)] = np.frombuffer(raw, np.uint8)
                kz[b, h, c] = int.from_bytes(bytes.fromhex(grp["zero_fp16"]), "little")
                ks[b, h, c] = int.from_bytes(bytes.fromhex(grp["scale_fp16"]), "little")
            for t, row in enumerate(head["value_rows"]):
                for j, grp in enumerate(row):
                    raw = bytes.fromhex(grp["codes"])
                    vc[b * g + t, h, j, :len(raw)] = np.frombuffer(raw, np.uint8)
                    vz[b * g + t, h, j] = int.from_bytes(bytes.fromhex(grp["zero_fp16"]), "little")
                    vs[b * g + t, h, j] = int.from_bytes(bytes.fromhex(grp["scale_fp16"]), "little")
    return dict(frontier=np.int64(f), key_codes=kc, key_zero16=kz, key_scale16=ks,
                val_codes=vc, val_zero16=vz, val_scale16=vs)


def gen_cache(tag, bits, H, d, g, r, k, n, pins, seed):
    rng = np.random.default_rng(seed)
    K, V = make_kv(rng, n, H, d)
    # force degenerate key groups (constant channel over a block) and a
    # constant value group, to exercise scale == 0
    if n >= 2 * g:
        K[g:2 * g, 0, 3] = K[g, 0, 3]
        V[5, H - 1, :min(g, d)] = V[5, H - 1, 0]
    cache = TwoTierCache(1, H, d, CacheBudget(bits=bits, group_size=g, residual=r,
                                             prefetch_k=k, context_length=4096))
    for i in range(n):
        cache.append_verified(0, K[i], V[i])
    cache.pin(0, pins)
    out = {"K": K, "V": V, "pins": np.asarray(pins, np.int64),
           "bits": np.int64(bits), "g": np.int64(g), "r": np.int64(r), "k": np.int64(k)}
    if bits != 16:
        out.update(parse_snapshot(cache.snapshot(), 0, H, d, g, bits))
    else:
        out["frontier"] = np.int64(cache.quantized_frontier(0))
    mk, mv = zip(*[cache.materialize(0, h) for h in range(H)])
    out["mat_k"] = np.stack(mk, 1)
    out["mat_v"] = np.stack(mv, 1)
    np.savez_compressed(os.path.join(HERE, f"cache_{tag}.npz"), **out)


def gen_decode(tag, bits, Hq, H, d, g, r, k, n0, steps, seed, tau=1.0):
    """Replay engine.py:245-268 (predecode) and :299-321 (decode_step's
    layer body) on reference objects with synthetic post-RoPE q/k/v."""
    rng = np.random.default_rng(seed)
    cfg = DecoderConfig(layers=1, q_heads=Hq, kv_heads=H, head_dim=d, max_len=65536)
    budget = CacheBudget(bits=bits, group_size=g, residual=r, prefetch_k=k,
                         context_length=max(4096, n0 + steps + 4))
    cache = TwoTierCache(1, H, d, budget)
    chan = SimulatedChannel(cache, ChannelModel())
    K, V = make_kv(rng, n0, H, d)
    for i in range(n0):
        cache.append_verified(0, K[i], V[i])
    prev = ()
    rec = {"K0": K, "V0": V, "bits": np.int64(bits), "g": np.int64(g), "r": np.int64(r),
           "k": np.int64(k), "Hq": np.int64(Hq), "steps": np.int64(steps)}

    # predecode (engine.py:245-268)
    q = make_queries(rng, 1, Hq, d, tau)
    kn, vn = make_step_kv(rng, 1, H, d)
    keys, vals = [], []
    for h in range(H):
        mk, mv = cache.materialize(0, h)
        keys.append(np.concatenate([mk, kn[:, h, :]], 0))
        vals.append(np.concatenate([mv, vn[:, h, :]], 0))
    n_cached = keys[0].shape[0] - 1
    out, probs = engine._attend(cfg, q, keys, vals, np.ones((1, n_cached + 1), bool))
    agg = np.sum([a[0, :n_cached] for a in probs], axis=0)
    picked = engine.select_topk(agg, k, cache.packed_positions(0))
    chan.schedule_prefetch(PrefetchTicket(0, 0, picked, cache.row_bytes(len(picked))))
    rec.update(pre_q=q, pre_k=kn, pre_v=vn, pre_out=out.reshape(1, Hq, d), pre_agg=agg,
               pre_picked=np.asarray(picked, np.int64))
    prev = picked

    # decode steps; q drifts so pins are partly reused
    qs, ks_, vs_, outs, aggs, pickeds, news, masses = [], [], [], [], [], [], [], []
    qcur = make_queries(rng, 2, Hq, d, tau)
    for step in range(1, steps + 1):
        pos, kp, vp = chan.await_layer(step, 0)
        cache.pin(0, pos, kp, vp)
        q = qcur
        kn, vn = make_step_kv(rng, 2, H, d)
        keys, vals = [], []
        for h in range(H):
            mk, mv = cache.materialize(0, h)
            keys.append(np.concatenate([mk, kn[:, h, :]], 0))
            vals.append(np.concatenate([mv, vn[:, h, :]], 0))
        n_cached = keys[0].shape[0] - 2
        mask = np.ones((2, n_cached + 2), bool)
        mask[0, n_cached + 1] = False
        out, probs = engine._attend(cfg, q, keys, vals, mask)
        pinned = list(cache.pinned_positions(0))
        mass = [float(a[0, pinned].sum()) if pinned else 0.0 for a in probs]
        agg = np.sum([a[1, :n_cached] for a in probs], axis=0)
        picked = engine.select_topk(agg, k, cache.packed_positions(0))
        new = [p for p in picked if p not in set(prev)]
        chan.schedule_prefetch(PrefetchTicket(step, 0, picked, cache.row_bytes(len(new))))
        prev = picked
        cache.append_verified(0, kn[0], vn[0])
        qs.append(q); ks_.append(kn); vs_.append(vn); outs.append(out.reshape(2, Hq, d))
        aggs.append(np.pad(agg, (0, steps + 1 - step)))
        pk = np.full(k, -1, np.int64); pk[:len(picked)] = picked; pickeds.append(pk)
        nw = np.full(k, -1, np.int64); nw[:len(new)] = new; news.append(nw)
        masses.append(mass)
        qcur = bf16_round(q + 0.3 * rng.standard_normal(q.shape).astype(np.float32))
    rec.update(q=np.stack(qs), k_new=np.stack(ks_), v_new=np.stack(vs_), out=np.stack(outs),
               agg=np.stack(aggs), picked=np.stack(pickeds), new=np.stack(news),
               pinned_mass=np.asarray(masses))
    np.savez_compressed(os.path.join(HERE, f"decode_{tag}.npz"), **rec)


def gen_adapter(tag, bits, g, r, k, L, prompt_len, steps, seed):
    """Reference generate() (engine.py:342-386) with the hot-path boundary in
    bf16: q/k/v rounded after _qkv, attention outputs rounded after _attend --
    exactly what the device path receives and returns."""
    from speckv.model import init_decoder
    from speckv import engine as E
    cfg = DecoderConfig(seed=seed)
    w = init_decoder(cfg)
    orig_qkv, orig_attend = E._qkv, E._attend

    def qkv16(c, lw, x, positions):
        q, k_, v = orig_qkv(c, lw, x, positions)
        return bf16_round(q), bf16_round(k_), bf16_round(v)

    def attend16(c, q, keys, vals, mask):
        out, probs = orig_attend(c, q, keys, vals, mask)
        return bf16_round(out), probs

    E._qkv, E._attend = qkv16, attend16
    try:
        prompt = [int(t) for t in np.random.default_rng(seed + 100).integers(0, cfg.vocab, prompt_len)]
        budget = CacheBudget(bits=bits, group_size=g, residual=r, prefetch_k=k, context_length=L)
        res = E.generate(cfg, w, prompt, steps, budget, ChannelModel(bandwidth=1e6),
                         compute_time_per_step=1e-3)
        base_tokens, base_logits, _ = E.FullCacheDecoder(cfg, w).generate(prompt, steps)
    finally:
        E._qkv, E._attend = orig_qkv, orig_attend
    rec = {"seed": np.int64(seed), "bits": np.int64(bits), "g": np.int64(g), "r": np.int64(r),
           "k": np.int64(k), "L": np.int64(L), "prompt": np.asarray(prompt, np.int64),
           "steps": np.int64(steps), "tokens": np.asarray(res.tokens, np.int64),
           "logits": np.stack(res.logits), "base_tokens": np.asarray(base_tokens, np.int64),
           "pinned_mass": np.asarray([m.pinned_mass for m in res.metrics]),
           "bytes": np.asarray([m.bytes_fetched for m in res.metrics], np.int64),
           "new_pins": np.asarray([m.new_pins for m in res.metrics], np.int64),
           "hit": np.asarray([m.speculative_hit for m in res.metrics]),
           "overlapped": np.asarray([r_["overlapped_s"] for r_ in res.latency_rows]),
           "total_seconds": np.float64(res.total_seconds),
           "w_embedding": w.embedding, "w_final_norm": w.final_norm, "w_head": w.head}
    for i, lw in enumerate(w.layers):
        for name in ("wq", "wk", "wv", "wo", "attn_norm", "ffn_norm", "w1", "w2"):
            rec[f"w_{i}_{name}"] = getattr(lw, name)
    for name in ("layers", "q_heads", "kv_heads", "head_dim", "vocab", "hidden", "ffn", "max_len"):
        rec[f"cfg_{name}"] = np.int64(getattr(cfg, name))
    rec["cfg_rope_base"] = np.float64(cfg.rope_base)
    np.savez_compressed(os.path.join(HERE, f"adapter_{tag}.npz"), **rec)


def gen_report():
    """experiments.run_decode (experiments.py:46-97) on a reference-written
    weight file, with the same bf16 hot-path boundary as gen_adapter."""
    import json
    from speckv import experiments as X
    from speckv import model as M
    from speckv import engine as E
    wpath = os.path.join(HERE, "report_toy.spkc")
    cfg = M.DecoderConfig(seed=2)
    M.save_weights(wpath, cfg, M.init_decoder(cfg))
    orig_qkv, orig_attend = E._qkv, E._attend

    def qkv16(c, lw, x, positions):
        q, k_, v = orig_qkv(c, lw, x, positions)
        return bf16_round(q), bf16_round(k_), bf16_round(v)

    def attend16(c, q, keys, vals, mask):
        out, probs = orig_attend(c, q, keys, vals, mask)
        return bf16_round(out), probs

    cases = {
        "b1": dict(prompt=None, prompt_len=12, steps=6, bits=1, group_size=4, k=4, residual=4,
                   bandwidth=16e9, alpha=5.0, overhead=0.0, compute_s=0.0, mode="sim", seed=0),
        "b2_seed9": dict(prompt=None, prompt_len=12, steps=8, bits=2, group_size=4, k=6, residual=4,
                         bandwidth=8e9, alpha=3.0, overhead=1e-6, compute_s=2e-6, mode="sim", seed=9),
        "b2_prompt": dict(prompt=[1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18], prompt_len=32,
                          steps=5, bits=2, group_size=4, k=4, residual=4, bandwidth=16e9, alpha=5.0,
                          overhead=0.0, compute_s=1e-3, mode="thread", seed=0),
    }
    E._qkv, E._attend = qkv16, attend16
    try:
        for tag, args in cases.items():
            rep = X.run_decode(weights_path="report_toy.spkc", max_len=4096, **{**args})  # noqa
            with open(os.path.join(HERE, f"report_{tag}.json"), "w") as fh:
                json.dump({"args": args, "report": rep}, fh, indent=1)
    finally:
        E._qkv, E._attend = orig_qkv, orig_attend


def gen_hitrate():
    """hitrate.py on synthetic traces + experiments.hitrate_experiment."""
    import json
    from speckv import experiments as X
    from speckv import hitrate as Hr
    rng = np.random.default_rng(11)
    seqs = []
    for kind in ("flat", "peaky", "tied", "sparse", "short"):
        n0 = {"short": 1, "sparse": 40}.get(kind, 150)
        steps = 9
        rows = []
        for t in range(steps):
            n = n0 + t
            if kind == "flat":
                x = rng.random(n).astype(np.float32)
            elif kind == "peaky":
                x = np.exp(3.0 * rng.standard_normal(n)).astype(np.float32)
            elif kind == "tied":
                x = rng.integers(1, 4, n).astype(np.float32)
            elif kind == "sparse":
                x = np.where(rng.random(n) < 0.3, rng.random(n), 0.0).astype(np.float32)
                x[0] = 1.0
            else:
                x = rng.random(n).astype(np.float32)
            rows.append((x / x.sum(dtype=np.float32)).astype(np.float32))
        seqs.append(rows)
    ks = [0, 1, 2, 3, 5, 16, 64, 1000]
    rec = {"ks": np.asarray(ks, np.int64), "nseq": np.int64(len(seqs))}
    for i, rows in enumerate(seqs):
        rec[f"lens_{i}"] = np.asarray([r.size for r in rows], np.int64)
        rec[f"rows_{i}"] = np.concatenate(rows)
        rec[f"topk_{i}"] = np.stack([Hr.topk_hitrate(rows, k) for k in ks])
        rec[f"evict_{i}"] = np.stack([Hr.eviction_hitrate(rows, k) for k in ks])
    np.savez_compressed(os.path.join(HERE, "hitrate_rows.npz"), **rec)
    args = dict(prompt=None, prompt_len=12, steps=6, k_sweep=[1, 4, 16, 64], seed=0)
    rep = X.hitrate_experiment(weights_path="report_toy.spkc", max_len=4096, **args)
    with open(os.path.join(HERE, "hitrate_report.json"), "w") as fh:
        json.dump({"args": args, "report": rep}, fh, indent=1)


def gen_g64():
    """g=64 (the paper's Table 4 group size): the fast layout's two-record groups."""
    gen_cache("b2_d128_g64", 2, 2, 128, 64, 64, 8, 330, [0, 5, 100, 200], seed=21)
    gen_cache("b1_d128_g64", 1, 2, 128, 64, 64, 8, 330, [3, 64, 191], seed=22)
    gen_decode("gqa_b2_g64", 2, 8, 2, 128, 64, 64, 16, 400, 3, seed=23)


if __name__ == "__main__" and len(sys.argv) > 1:
    os.chdir(HERE)
    for name in sys.argv[1:]:
        globals()["gen_" + name]()
    sys.exit(0)

if __name__ == "__main__":
    gen_quant_groups()
    gen_cache("b2_d128", 2, 2, 128, 32, 32, 8, 200, [0, 5, 37, 100], seed=1)
    gen_cache("b1_d128", 1, 2, 128, 32, 32, 8, 200, [3, 64, 127], seed=2)
    gen_cache("b4_d128", 4, 2, 128, 32, 32, 8, 200, [31, 32], seed=3)
    gen_cache("b16_d128", 16, 2, 128, 32, 32, 8, 200, [10], seed=4)
    gen_cache("b2_d10_g4", 2, 3, 10, 4, 3, 4, 19, [2, 9], seed=5)   # ragged value groups
    gen_cache("b1_d8_g4", 1, 2, 8, 4, 4, 4, 40, [1, 5, 20], seed=6)
    gen_decode("mha_b2", 2, 4, 4, 128, 32, 32, 16, 300, 4, seed=7)
    gen_decode("gqa_b1", 1, 8, 2, 128, 32, 32, 16, 300, 4, seed=8, tau=3.0)
    gen_decode("mha_b16", 16, 4, 4, 128, 32, 32, 16, 200, 3, seed=9)
    gen_decode("gqa4_b2", 2, 8, 2, 128, 32, 64, 32, 700, 5, seed=10)
    gen_adapter("b2", 2, 4, 4, 4, 4096, 12, 10, seed=3)
    gen_adapter("b1", 1, 4, 4, 4, 4096, 20, 10, seed=4)
    gen_adapter("b16_exact", 16, 4, 8, 1024, 1024, 32, 16, seed=5)
    os.chdir(HERE)
    gen_report()
    gen_hitrate()
    print("golden fixtures written to", HERE)
