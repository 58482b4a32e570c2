#!/usr/bin/env python
"""CPU: per-CUDA-source-line warp-instructions and stall samples of a kernel
from an .ncu-rep (source page, cuda+sass view), normalised per loop
iteration (one 32-token block per warp).  Inlined helpers are attributed to
their own definition lines.

  python tools/ncu_lines_per_block.py rep.ncu-rep --iters 262016 [--min 0.5]"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--iters", type=float, required=True)
    ap.add_argument("--min", type=float, default=0.5, help="print lines with >= this many instructions per block")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, tot_i, tot_s, rows = "?", 0.0, 0.0, []
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] in ("File Name", "File Path"):
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if len(r) < 65 or not r[0].isdigit():
            continue
        m = r[-61:]  # metric columns (a source line with quotes can split into extra fields)
        try:
            inst, samp = float(m[3]), float(m[0])
        except ValueError:
            continue
        tot_i += inst
        tot_s += samp
        rows.append((fname, int(r[0]), inst / a.iters, samp, ",".join(r[1:len(r) - 63]).strip()[:90]))
    print("total: %.1f warp-instructions per block, %d samples" % (tot_i / a.iters, tot_s))
    for f, ln, ipb, s, src in rows:
        if ipb >= a.min:
            print("%-18s %5d %7.1f %6.1f%%  %s" % (f, ln, ipb, 100.0 * s / max(1.0, tot_s), src))


if __name__ == "__main__":
    main()
