#!/usr/bin/env python
"""CPU: SASS opcode histogram of a kernel's hot loop from an .ncu-rep source page.

Instructions executed at least --min times (e.g. once per 32-token block) are
the loop body; prints the opcode histogram per loop iteration and, with
--dump, the loop's instructions with their executed counts.

  python tools/ncu_loop_sass.py rep.ncu-rep --iters 262144 [--dump]"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--iters", type=float, required=True, help="loop iterations (warp-blocks) per launch")
    ap.add_argument("--min-frac", type=float, default=0.5)
    ap.add_argument("--dump", action="store_true")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    ie, src = h.index("Instructions Executed"), h.index("Source")
    hist, tot, body = collections.Counter(), 0.0, []
    for r in rows[hdr + 1:]:
        if len(r) <= ie:
            continue
        try:
            n = float(r[ie])
        except ValueError:
            continue
        if n < a.min_frac * a.iters:
            continue
        op = r[src].strip().split()
        if not op:
            continue
        o = op[0] if not op[0].startswith("@") else op[1]
        o = o.split(".")[0]
        hist[o] += n / a.iters
        tot += n / a.iters
        body.append((r[0], n / a.iters, r[src].strip()))
    print(f"loop instructions per iteration: {tot:.1f}")
    for o, n in hist.most_common(40):
        print(f"  {o:10s} {n:7.1f}")
    if a.dump:
        for addr, n, s in body:
            print(f"{addr}  {n:5.2f}  {s}")


if __name__ == "__main__":
    main()
