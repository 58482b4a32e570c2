#!/usr/bin/env python
"""Kernel timeline of the full-decoder step (bench.py --full-decoder) via
torch.profiler (CUPTI): per-kernel totals per step, per-stream busy time and
compute-stream idle gaps.  Writes gpurun_out/full_decoder_trace.json.

  python tools/profile_full_decoder.py [--config c2] [--steps 3]
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
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache
    from paper_2503_16163_b200.decoder import DecoderStack, StackConfig, random_stack

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0)
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    if args.batch:
        cfg["batch"] = args.batch
    hidden, ffn, vocab = bench.MODEL_SHAPES[args.config]
    sc = StackConfig(layers=cfg["layers"], q_heads=cfg["q_heads"], kv_heads=cfg["kv_heads"],
                     head_dim=cfg["head_dim"], hidden=hidden, ffn=ffn, vocab=vocab)
    dev = "cuda:0"
    hl = bench.plan_host_layers(cfg, 1)
    budget = CacheBudget(bits=cfg["bits"], group_size=cfg["group"], residual=cfg["residual"],
                         prefetch_k=cfg["topk"], context_length=cfg["ctx"] + 64 + args.steps + 8)
    cache = DeviceTwoTierCache(cfg["layers"], cfg["kv_heads"], cfg["head_dim"], budget, batch=cfg["batch"],
                               q_heads=cfg["q_heads"], host_layers=hl)
    s0 = torch.randn((hl, cfg["batch"], cfg["q_heads"], cfg["head_dim"]), device=dev).bfloat16()
    bench.prefill_cache(cache, cfg, hl, s0, dev, seed=99)
    stack = DecoderStack(sc, random_stack(sc, dev), cache)
    B, n = cfg["batch"], cfg["ctx"]
    tok0 = torch.randint(0, vocab, (B,), device=dev)
    pos = torch.full((B,), n, dtype=torch.int32, device=dev)
    toks = torch.stack([tok0.int(), stack.predecode(tok0, pos).clone()], 1)
    step = 1
    for _ in range(4):
        toks = stack.decode_step(step, toks, pos + step - 1).clone()
        step += 1
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(args.steps):
            toks = stack.decode_step(step, toks, pos + step - 1).clone()
            step += 1
        torch.cuda.synchronize()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", "full_decoder_trace.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    streams = collections.defaultdict(list)
    for e in ev:
        name = e["name"]
        short = name.replace("(anonymous namespace)::", "").split("(")[0][:70]
        tot[short] += e["dur"]
        cnt[short] += 1
        streams[e["args"].get("stream", e.get("tid"))].append((e["ts"], e["ts"] + e["dur"], short))
    print(f"per-step kernel time (us), {args.steps} steps:")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
        print(f"  {v / args.steps:10.1f}  x{cnt[k] / args.steps:6.1f}  {k}")
    t0 = min(s for v in streams.values() for s, _, _ in v)
    t1 = max(e for v in streams.values() for _, e, _ in v)
    print(f"window {(t1 - t0) / args.steps:.1f} us/step")
    for sid, v in streams.items():
        v.sort()
        busy = sum(e - s for s, e, _ in v)
        gaps = collections.defaultdict(float)
        for (s0_, e0_, n0_), (s1_, e1_, n1_) in zip(v, v[1:]):
            if s1_ > e0_:
                gaps[f"{n0_[:30]} -> {n1_[:30]}"] += s1_ - e0_
        print(f"stream {sid}: {len(v) / args.steps:.0f} kernels/step, busy {busy / args.steps:.1f} us/step")
        for k, g in sorted(gaps.items(), key=lambda kv: -kv[1])[:8]:
            print(f"    gap {g / args.steps:9.1f} us/step  {k}")
    cache.close()


if __name__ == "__main__":
    main()
