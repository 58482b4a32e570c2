"""Child process of tests/test_fold_gpu.py and tools/split_precision.py (not a
test module): one predecode of a long-context geometry on cuda:0, the kernel's
fp32 output checked against the oracle per q head.  The K2 split count is read
once per process (SPC_NSPLIT), hence a process per case.  Prints one JSON line.

Data as tests/test_bench_geometry_gpu.py: K = N(0,1) + a per-(head, channel)
offset, 256 needles along the query, V = N(0,1) -- zero-mean values, so the
output is a small random walk and accumulation bias shows up relative to it.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NEEDLES = 256


def run(b, H, Hq, n0, bits, k, seqs):
    import numpy as np
    import torch

    from oracle import restate as R
    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder
    d, g, r, G = 128, 32, 64, Hq // H
    dev = "cuda:0"
    gen = torch.Generator(device=dev).manual_seed(2024)
    bf = lambda x: x.to(torch.bfloat16)
    q = bf(torch.randn((b, 1, Hq, d), device=dev, generator=gen))
    _ = bf(torch.randn((b, 1, Hq, d), device=dev, generator=gen))
    K = torch.randn((b, n0, H, d), device=dev, generator=gen)
    K += 2.0 * torch.randn((1, 1, H, d), device=dev, generator=gen)
    qdir = q[:, 0].float().view(b, H, G, d).mean(2)
    pos = torch.randint(0, n0 - r - g, (b, NEEDLES, H), device=dev, generator=gen)
    bi = torch.arange(b, device=dev)[:, None, None].expand_as(pos)
    hi = torch.arange(H, device=dev)[None, None, :].expand_as(pos)
    K[bi, pos, hi] += 0.5 * qdir[bi, hi]
    K = bf(K)
    V = bf(torch.randn((b, n0, H, d), device=dev, generator=gen))
    budget = CacheBudget(bits=bits, group_size=g, residual=r, prefetch_k=k, context_length=n0 + 16)
    cache = DeviceTwoTierCache(1, H, d, budget, batch=b, q_heads=Hq, host_layers=0)
    assert cache.fast_path
    cache.prefill(0, K, V)
    dec = SpeculativeLayerDecoder(cache)
    dec.debug_output_f32(True)
    kn = bf(torch.randn((b, 1, H, d), device=dev, generator=gen))
    vn = bf(torch.randn((b, 1, H, d), device=dev, generator=gen))
    dec.predecode_layer(0, q, kn, vn)
    o32 = dec.debug_out_f32(0, 1).cpu().numpy()
    f32 = lambda x: x.float().cpu().numpy()
    res = {"geometry": dict(b=b, H=H, Hq=Hq, n0=n0, bits=bits, k=k),
           "nsplit_env": os.environ.get("SPC_NSPLIT", "model"), "per_seq": {}}
    for s in seqs:
        st = R.LayerState(H, d, bits, g, r, k, "layer")
        st.extend(f32(K[s]), f32(V[s]))
        o = R.predecode_layer(st, f32(q[s]), f32(kn[s]), f32(vn[s]))["out"]
        errs = [float(np.linalg.norm(o32[s][0, h] - o[0, h]) / np.linalg.norm(o[0, h])) for h in range(Hq)]
        # the error's component along the reference output (a scale error)
        par = [float(np.dot(o32[s][0, h] - o[0, h], o[0, h]) / np.dot(o[0, h], o[0, h])) for h in range(Hq)]
        res["per_seq"][s] = {"rel_err": errs, "scale_err": par}
    res["max_rel_err"] = max(max(v["rel_err"]) for v in res["per_seq"].values())
    cache.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    for name, dflt in (("b", 2), ("H", 4), ("Hq", 4), ("n0", 131072), ("bits", 1), ("k", 64)):
        ap.add_argument("--" + name, type=int, default=dflt)
    ap.add_argument("--seqs", default="0")
    a = ap.parse_args()
    print(json.dumps(run(a.b, a.H, a.Hq, a.n0, a.bits, a.k, [int(s) for s in a.seqs.split(",")])))


if __name__ == "__main__":
    main()
