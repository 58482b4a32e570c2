#!/usr/bin/env python
"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum
--clock-control none --csv --log-file X.csv python bench.py ...`): per-kernel
count / total / average, and the serialised per-layer-step share of the decode
kernels (the launches of spc_decode_layer: K2 attend, K3 combine / agg, K4
top-k, K5 prefetch, K6 appends).  Times under ncu are cold-cache and
serialised, so only the shares are comparable with the bench's live numbers.

  python tools/launch_summary.py gpurun_out/launches.csv > profiles/<name>.txt
"""
import collections
import csv
import re
import sys

DECODE = ("k_attend_fast", "k_attend_generic", "k_combine", "k_agg", "k_topk", "k_prefetch",
          "k_ring_append", "k_host_append")


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name[:60]


def main(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("==")) if r]
    hdr = rows[0]
    iK, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[iM] != "gpu__time_duration.sum":
            continue
        k = short(r[iK])
        tot[k] += float(r[iV].replace(",", "")) / 1e3  # ns -> us
        cnt[k] += 1
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"{k:60s} n={cnt[k]:5d} total={tot[k] / 1e3:10.3f} ms avg={tot[k] / cnt[k]:10.2f} us")
    # per layer-step: the attend kernel's launch count is the number of layer-steps
    att = [k for k in tot if "k_attend_fast" in k or "k_attend_generic" in k]
    steps = sum(cnt[k] for k in att)
    if not steps:
        return
    dec = {k: tot[k] / steps for k in tot if any(d in k for d in DECODE)}
    s = sum(dec.values())
    print(f"\nper layer-step ({steps} layer-steps incl. predecode), serialised decode kernels: {s:.1f} us")
    for k in sorted(dec, key=lambda x: -dec[x]):
        print(f"  {k:60s} {dec[k]:9.1f} us ({dec[k] / s * 100:5.1f}%)")


if __name__ == "__main__":
    main(sys.argv[1])
