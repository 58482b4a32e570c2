#!/usr/bin/env python
"""Build container only (needs /root/reference): time the UNMODIFIED reference's
per-layer decode step at BASELINE config 1 (C1: 1 layer, 32 heads x d128, ctx
4096, 2-bit, k=64, r=32, batch 1) by replaying engine.py:300-321 on a real
TwoTierCache (SURVEY 8(d) "CPU reference timing", mode (i)), and the oracle
port on the same inputs for the port/reference speed ratio.  Writes
profiles/r2_reference_c1_timing.json.

The reference is pure Python and does not exist on the GPU box, so this is
the only place it can be timed; bench.py's reference arm runs the port."""
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    from speckv import engine, kvcache, model
    from speckv.kvcache import CacheBudget, TwoTierCache

    from oracle import restate as R
    from oracle.synth import make_kv, make_queries, make_step_kv
    H, Hq, d, n, bits, g, r, k = 32, 32, 128, 4096, 2, 32, 32, 64
    rng = np.random.default_rng(0)
    K, V = make_kv(rng, n, H, d)
    q = make_queries(rng, 2, Hq, d)
    kn, vn = make_step_kv(rng, 2, H, d)
    budget = CacheBudget(bits=bits, group_size=g, residual=r, prefetch_k=k, context_length=n)
    cache = TwoTierCache(1, H, d, budget)
    t0 = time.perf_counter()
    for i in range(n):
        cache.append_verified(0, K[i], V[i])
    prefill_s = time.perf_counter() - t0
    cfg = model.DecoderConfig(layers=1, q_heads=Hq, kv_heads=H, head_dim=d, vocab=64, hidden=64, ffn=64,
                              max_len=n + 8)
    # engine.py:300-321 on the real cache (no ticket pins: predecode-like first step)
    t0 = time.perf_counter()
    keys, vals = [], []
    for h in range(H):
        mk, mv = cache.materialize(0, h)
        keys.append(np.concatenate([mk, kn[:, h, :]], 0))
        vals.append(np.concatenate([mv, vn[:, h, :]], 0))
    t_mat = time.perf_counter() - t0
    n_cached = keys[0].shape[0] - 2
    mask = np.ones((2, n_cached + 2), dtype=bool)
    mask[0, n_cached + 1] = False
    t1 = time.perf_counter()
    out, probs = engine._attend(cfg, q, keys, vals, mask)
    t_att = time.perf_counter() - t1
    agg = np.sum([a[1, :n_cached] for a in probs], axis=0)
    t2 = time.perf_counter()
    picked = engine.select_topk(agg, k, cache.packed_positions(0))
    t_sel = time.perf_counter() - t2
    ref_step = time.perf_counter() - t0
    # the oracle port on the same inputs
    st = R.LayerState(H, d, bits, g, r, k)
    st.extend(K, V)
    st._sync_packed()
    t3 = time.perf_counter()
    o = R.decode_layer(st, q, kn, vn, append=False)
    port_step = time.perf_counter() - t3
    assert set(o["picked"][0]) == set(picked)
    np.testing.assert_allclose(o["out"].reshape(2, -1), out, rtol=1e-4, atol=1e-5)
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": i.get("internal_api"), "threads": i.get("num_threads")} for i in threadpool_info()]
    except Exception:
        blas = None
    cpu = None
    with open("/proc/cpuinfo") as fh:
        for line in fh:
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    rec = {"what": "unmodified reference (speckv) C1 decode-layer step, engine.py:300-321 replayed on a real "
                   "TwoTierCache, vs the oracle port (oracle/restate.py) on the same inputs; build container",
           "config": "C1: 1 layer, 32 heads x d128, ctx 4096, 2-bit (g32, r32), k64, batch 1",
           "reference_step_s": ref_step, "reference_materialize_s": t_mat, "reference_attend_s": t_att,
           "reference_select_s": t_sel, "reference_prefill_append_s": prefill_s,
           "port_step_s": port_step, "port_speedup_over_reference": ref_step / port_step,
           "reference_tokens_per_s": 1.0 / ref_step, "port_tokens_per_s": 1.0 / port_step,
           "same_topk": True, "cpu": cpu, "nproc": os.cpu_count(), "blas": blas,
           "python": platform.python_version(), "numpy": np.__version__}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r2_reference_c1_timing.json"), "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
