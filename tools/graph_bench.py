#!/usr/bin/env python
"""Eager vs step-graph decode (spc_graph_begin / spc_graph_launch) at a bench
config: the same cache geometry, data and stream; device time per step with
CUDA events over --steps steps after --warmup (each arm its own cache, built
identically), and the host time per step (wall clock of issuing the steps).

  python tools/graph_bench.py --config c1 --steps 200
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def arm(cfg, graph, steps, warmup, dev):
    import torch

    import bench
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder, _lib
    hl = bench.plan_host_layers(cfg, 1)
    total = warmup + steps + 1
    budget = CacheBudget(bits=cfg["bits"], group_size=cfg["group"], residual=cfg["residual"],
                         prefetch_k=cfg["topk"], context_length=cfg["ctx"] + 64 + total + 8)
    cache = DeviceTwoTierCache(cfg["layers"], cfg["kv_heads"], cfg["head_dim"], budget, batch=cfg["batch"],
                               q_heads=cfg["q_heads"], host_layers=hl)
    dec = SpeculativeLayerDecoder(cache)
    q, kn, vn, s0 = bench.make_inputs(cfg, total, dev, hl, seed=1)
    bench.prefill_cache(cache, cfg, hl, s0, dev, seed=2)
    L = cfg["layers"]
    out = torch.empty((L, cfg["batch"], 2, cfg["q_heads"], cfg["head_dim"]), dtype=torch.bfloat16, device=dev)
    pm = torch.empty((L, cfg["batch"], cfg["q_heads"]), dtype=torch.float32, device=dev)
    lib, h = _lib.lib(), cache.handle
    side = torch.cuda.Stream(dev)
    st = side.cuda_stream
    with torch.cuda.stream(side):
        for layer in range(L):
            dec.predecode_layer(layer, q[0, layer][:, :1], kn[0, layer][:, :1], vn[0, layer][:, :1])

    def step(t):
        if graph:
            _lib.check(lib.spc_graph_begin(h, st))
        for layer in range(L):
            _lib.check(lib.spc_decode_layer(h, layer, t, q[t, layer].data_ptr(), kn[t, layer].data_ptr(),
                                            vn[t, layer].data_ptr(), out[layer].data_ptr(), pm[layer].data_ptr(),
                                            st))
        if graph:
            _lib.check(lib.spc_graph_launch(h, st))

    t = 1
    for _ in range(warmup):
        step(t)
        t += 1
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(side)
    w0 = time.perf_counter()
    for _ in range(steps):
        step(t)
        t += 1
    host_s = time.perf_counter() - w0
    e1.record(side)
    torch.cuda.synchronize(dev)
    res = {"graph": graph, "device_ms_per_step": e0.elapsed_time(e1) / steps,
           "host_issue_ms_per_step": 1e3 * host_s / steps}
    if graph:
        res["instantiations"], res["updates"] = dec.graph_stats()
    res["tokens_per_s"] = cfg["batch"] / (res["device_ms_per_step"] / 1e3)
    cache.close()
    return res


def main():
    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=2)
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS[a.config])
    rows = []
    for r in range(a.rounds):
        for g in (False, True):
            x = arm(cfg, g, a.steps, a.warmup, "cuda:0")
            x["round"] = r
            rows.append(x)
            print(json.dumps(x), flush=True)
    best = {g: min(x["device_ms_per_step"] for x in rows if x["graph"] == g) for g in (False, True)}
    print(json.dumps({"config": a.config, "steps": a.steps, "eager_ms": best[False], "graph_ms": best[True],
                      "speedup": best[False] / best[True]}))


if __name__ == "__main__":
    main()
