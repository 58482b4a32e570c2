#!/usr/bin/env python
"""BASELINE.json configs[4] -- kernel sweep: ctx 4k-256k x top-k 16-512 x 1/2-bit.

One decode layer (MHA 32 heads x d128, g32, r64, bf16 I/O) per point, batch
scaled so every point streams ~0.5M tokens per head; W warm-up + K timed
decode steps with the library's live CUDA-event profiling.  Reports per point:
  K2 (attend) achieved GB/s = algorithmic bytes per launch / avg launch time,
  fraction of the measured HBM peak, and K5 (PCIe prefetch) GB/s = bytes the
  gathers moved / their kernel time.

  python tools/sweep.py [--quick] [--group 64] [--ctx ...] [--topk ...] > gpurun_out/sweep.jsonl
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def point(bits, ctx, k, steps=10, warmup=3, group=32):
    import torch

    import bench
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder, _lib

    batch = max(1, min(16, (1 << 19) // ctx))
    cfg = dict(workload=f"sweep bits={bits} ctx={ctx} k={k}", layers=1, batch=batch, kv_heads=32,
               q_heads=32, head_dim=128, ctx=ctx, bits=bits, group=group, residual=64, topk=k)
    dev = "cuda:0"
    budget = CacheBudget(bits=bits, group_size=group, residual=64, prefetch_k=k,
                         context_length=ctx + steps + warmup + 64)
    cache = DeviceTwoTierCache(1, 32, 128, budget, batch=batch, q_heads=32, host_layers=1)
    q, kn, vn, s0 = bench.make_inputs(cfg, steps + warmup + 1, dev, 1, seed=7)
    bench.prefill_cache(cache, cfg, 1, s0, dev, seed=8)
    dec = SpeculativeLayerDecoder(cache)
    dec.predecode_layer(0, q[0, 0][:, :1], kn[0, 0][:, :1], vn[0, 0][:, :1])
    lib, h = _lib.lib(), cache.handle

    def prof(enable):
        am, al, sm, sl, nl = (ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(),
                              ctypes.c_int64(), ctypes.c_int64())
        _lib.check(lib.spc_profile(h, enable, ctypes.byref(am), ctypes.byref(al), ctypes.byref(sm),
                                   ctypes.byref(sl), ctypes.byref(nl)))
        return am.value, al.value

    t = 1
    for _ in range(warmup):
        dec.decode_layer(0, t, q[t, 0], kn[t, 0], vn[t, 0])
        t += 1
    n, f = cache.length(0), cache.quantized_frontier(0)
    torch.cuda.synchronize()
    prof(1)
    for _ in range(steps):
        dec.decode_layer(0, t, q[t, 0], kn[t, 0], vn[t, 0])
        t += 1
    attn_ms, attn_n = prof(0)
    pf_ms, pf_bytes = lib.spc_profile_prefetch_ms(h), int(lib.spc_profile_prefetch_bytes(h))
    ab = bench.algorithmic_bytes_per_layer(cfg, n + steps // 2, f, k)
    avg = attn_ms / max(1, attn_n)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    out = {"bits": bits, "group": group, "kernel": "fast" if cache.fast_path else "generic",
           "ctx": ctx, "topk": k, "batch": batch,
           "k2_ms": avg, "k2_gbs": ab["hbm"] / avg / 1e6, "k2_frac_hbm": ab["hbm"] / avg / 1e6 / peaks["hbm_gbs"],
           "k2_algorithmic_bytes": ab["hbm"],
           "prefetch_bytes_per_step": pf_bytes / steps, "prefetch_ms_per_step": pf_ms / steps,
           "prefetch_gbs": (pf_bytes / 1e9) / max(1e-9, pf_ms / 1e3),
           "new_pin_fraction": pf_bytes / steps / max(1, batch * k * cache.row_bytes(1))}
    cache.close()
    del q, kn, vn
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--group", type=int, default=32, help="quantization group size g (paper Table 4: 64)")
    ap.add_argument("--ctx", type=int, nargs="*", help="override the context list")
    ap.add_argument("--topk", type=int, nargs="*", help="override the top-k list")
    args = ap.parse_args()
    ctxs = args.ctx or ([4096, 32768, 131072] if args.quick else [4096, 16384, 65536, 131072, 262144])
    ks = args.topk or ([16, 128, 512] if args.quick else [16, 64, 256, 512])
    for bits in (2, 1):
        for ctx in ctxs:
            for k in ks:
                print(json.dumps(point(bits, ctx, k, group=args.group)), flush=True)


if __name__ == "__main__":
    main()
