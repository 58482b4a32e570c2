#!/usr/bin/env python
"""Kernel timeline of the hot-path decode step (bench.py's loop) via
torch.profiler (CUPTI): for every K2 launch of one profiled step, its duration
and which other kernels overlapped it (and for how long).  Answers "why is K2
slower in the 32-layer loop than alone".  Writes gpurun_out/timeline_<cfg>.json.

  python tools/timeline_hotpath.py --config c4 --heads 1 --batch 32   # C4 rank share
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder, _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--heads", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS[a.config])
    if a.heads:
        g = cfg["q_heads"] // cfg["kv_heads"]
        cfg["kv_heads"], cfg["q_heads"] = a.heads, a.heads * g
    if a.batch:
        cfg["batch"] = a.batch
    dev = "cuda:0"
    hl = bench.plan_host_layers(cfg, 1)
    W = 4
    budget = CacheBudget(bits=cfg["bits"], group_size=cfg["group"], residual=cfg["residual"],
                         prefetch_k=cfg["topk"], context_length=cfg["ctx"] + 64 + W + a.steps + 8)
    cache = DeviceTwoTierCache(cfg["layers"], cfg["kv_heads"], cfg["head_dim"], budget, batch=cfg["batch"],
                               q_heads=cfg["q_heads"], host_layers=hl)
    dec = SpeculativeLayerDecoder(cache)
    q, kn, vn, s0 = bench.make_inputs(cfg, W + a.steps + 1, dev, hl, seed=1)
    bench.prefill_cache(cache, cfg, hl, s0, dev, seed=2)
    L = cfg["layers"]
    out = torch.empty((L, cfg["batch"], 2, cfg["q_heads"], cfg["head_dim"]), dtype=torch.bfloat16, device=dev)
    pm = torch.empty((L, cfg["batch"], cfg["q_heads"]), dtype=torch.float32, device=dev)
    lib, h = _lib.lib(), cache.handle
    stream = torch.cuda.current_stream().cuda_stream
    for layer in range(L):
        dec.predecode_layer(layer, q[0, layer][:, :1], kn[0, layer][:, :1], vn[0, layer][:, :1])

    def step(t):
        for layer in range(L):
            _lib.check(lib.spc_decode_layer(h, layer, t, q[t, layer].data_ptr(), kn[t, layer].data_ptr(),
                                            vn[t, layer].data_ptr(), out[layer].data_ptr(), pm[layer].data_ptr(),
                                            stream))

    t = 1
    for _ in range(W):
        step(t)
        t += 1
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            step(t)
            t += 1
        torch.cuda.synchronize()
    path = os.path.join(ROOT, "gpurun_out", f"trace_{a.config}.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    prof.export_chrome_trace(path)
    with open(path) as fh:
        ev = [e for e in json.load(fh)["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    k2 = [e for e in ev if "k_attend_fast" in e["name"]]
    short = lambda n: n.split("(")[0].replace("void ", "").replace("spc::", "").replace("<unnamed>::", "")
    rows, overlap_tot = [], collections.Counter()
    for e in k2[-L:]:  # the last profiled step
        s0, s1 = e["ts"], e["ts"] + e["dur"]
        ov = collections.Counter()
        for o in ev:
            if o is e or "k_attend_fast" in o["name"]:
                continue
            lo, hi = max(s0, o["ts"]), min(s1, o["ts"] + o["dur"])
            if hi > lo:
                ov[short(o["name"])] += hi - lo
        for k, v in ov.items():
            overlap_tot[k] += v
        rows.append({"k2_us": e["dur"], "overlap_us": dict(ov)})
    durs = [r["k2_us"] for r in rows]
    res = {"config": a.config, "heads": a.heads, "batch": cfg["batch"], "k2_us_mean": sum(durs) / len(durs),
           "k2_us_min": min(durs), "k2_us_max": max(durs),
           "overlap_us_per_k2": {k: v / len(rows) for k, v in overlap_tot.most_common()},
           "per_layer": rows}
    print(json.dumps({k: v for k, v in res.items() if k != "per_layer"}, indent=1))
    with open(os.path.join(ROOT, "gpurun_out", f"timeline_{a.config}.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    cache.close()


if __name__ == "__main__":
    main()
