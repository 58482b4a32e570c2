#!/usr/bin/env python
"""A/B timing of the K2 attend kernel between library builds on one box.

  python tools/ab_k2.py --config c3 --libs libA.so libB.so [--rounds 2]

Each (round, lib) runs in a fresh subprocess (SPC_LIB_PATH=lib) that builds a
one-layer cache at the config's geometry, warms up, and reports the mean K2
launch time over --steps decode steps (library CUDA-event profiling).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(config, steps, heads=0, batch=0):
    import torch

    import bench
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder
    cfg = dict(bench.CONFIGS[config])
    cfg["layers"] = 1
    if heads:  # e.g. one rank's share of a head-sharded config: --heads 1 --batch 32 (C4 over 8)
        g = cfg["q_heads"] // cfg["kv_heads"]
        cfg["kv_heads"], cfg["q_heads"] = heads, heads * g
    if batch:
        cfg["batch"] = batch
    dev = "cuda:0"
    budget = CacheBudget(bits=cfg["bits"], group_size=cfg["group"], residual=cfg["residual"],
                         prefetch_k=cfg["topk"], context_length=cfg["ctx"] + steps + 80)
    cache = DeviceTwoTierCache(1, cfg["kv_heads"], cfg["head_dim"], budget, batch=cfg["batch"],
                               q_heads=cfg["q_heads"], host_layers=1)
    q, kn, vn, s0 = bench.make_inputs(cfg, steps + 6, dev, 1, seed=3)
    bench.prefill_cache(cache, cfg, 1, s0, dev, seed=4)
    dec = SpeculativeLayerDecoder(cache)
    dec.predecode_layer(0, q[0, 0][:, :1], kn[0, 0][:, :1], vn[0, 0][:, :1])
    for t in range(1, 5):
        dec.decode_layer(0, t, q[t, 0], kn[t, 0], vn[t, 0])
    cache.profile(True)
    for t in range(5, 5 + steps):
        dec.decode_layer(0, t, q[t, 0], kn[t, 0], vn[t, 0])
    p = cache.profile(False)
    print(json.dumps({"k2_ms": p["attn_ms"] / max(1, p["attn_launches"]), "n": p["attn_launches"]}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--libs", nargs="+")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--heads", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    a = ap.parse_args()
    if a.child:
        return child(a.config, a.steps, a.heads, a.batch)
    for r in range(a.rounds):
        for lib in a.libs:
            env = dict(os.environ, SPC_LIB_PATH=os.path.abspath(lib))
            out = subprocess.run([sys.executable, __file__, "--child", "--config", a.config, "--steps",
                                  str(a.steps), "--heads", str(a.heads), "--batch", str(a.batch)], env=env, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(f"round {r} {os.path.basename(lib)}: {line}", flush=True)


if __name__ == "__main__":
    main()
