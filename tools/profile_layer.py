#!/usr/bin/env python
"""Single-layer driver for ncu: one decode layer at a BASELINE geometry.

  ncu --set full -k regex:k_attend_fast -s 2 -c 1 -o gpurun_out/prof \
      python tools/profile_layer.py --config c2 --steps 4

Builds a 1-layer DeviceTwoTierCache with the config's (batch, heads, ctx,
bits), prefills synthetic bf16 KV, predecodes and runs `--steps` decode steps.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--impl", default="auto")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--ctx", type=int, default=0)
    ap.add_argument("--heads", type=int, default=0)
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    if args.batch:
        cfg["batch"] = args.batch
    if args.ctx:
        cfg["ctx"] = args.ctx
    if args.heads:
        g = cfg["q_heads"] // cfg["kv_heads"]
        cfg["kv_heads"], cfg["q_heads"] = args.heads, args.heads * g
    cfg["layers"] = 1
    dev = "cuda:0"
    budget = CacheBudget(bits=cfg["bits"], group_size=cfg["group"], residual=cfg["residual"],
                         prefetch_k=cfg["topk"], context_length=cfg["ctx"] + args.steps + 64)
    cache = DeviceTwoTierCache(1, cfg["kv_heads"], cfg["head_dim"], budget, batch=cfg["batch"],
                               q_heads=cfg["q_heads"], host_layers=1)
    cache.set_attend_impl(args.impl)
    q, k_new, v_new, s0 = bench.make_inputs(cfg, args.steps + 1, dev, 1, seed=5)
    bench.prefill_cache(cache, cfg, 1, s0, dev, seed=6)
    dec = SpeculativeLayerDecoder(cache)
    dec.predecode_layer(0, q[0, 0][:, :1], k_new[0, 0][:, :1], v_new[0, 0][:, :1])
    for t in range(1, args.steps + 1):
        dec.decode_layer(0, t, q[t, 0], k_new[t, 0], v_new[t, 0])
    torch.cuda.synchronize()
    print("ok", cache.length(0), cache.quantized_frontier(0))
    cache.close()


if __name__ == "__main__":
    main()
