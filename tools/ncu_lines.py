#!/usr/bin/env python
"""CPU: per-source-line instruction counts and stall samples of one kernel in an
.ncu-rep (captured with --import-source on, built with -lineinfo).

  python tools/ncu_lines.py rep.ncu-rep [--per N] [--top 40]

--per divides the executed warp-instruction counts (e.g. by the number of
32-token blocks of the launch, to read instructions per block)."""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--per", type=float, default=1.0)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hdr]
    ie = h.index("Instructions Executed")
    samp = h.index("Warp Stall Sampling (All Samples)")
    lines, cur = [], None
    total = 0
    for r in rows[hdr + 1:]:
        if len(r) <= ie:
            continue
        if r[0]:
            # the source text may contain unescaped quotes: index the metrics from the right
            k = len(r) - len(h)
            try:
                n = float(r[ie + k])
                s = float(r[samp + k]) if r[samp + k] not in ("", "-") else 0.0
            except ValueError:
                continue
            lines.append((n, s, r[0], ",".join(r[1:2 + k]).strip()[:90]))
            total += n
    lines.sort(reverse=True)
    tot_s = sum(x[1] for x in lines)
    print(f"total warp instructions {total:.0f} ({total / a.per:.1f} per unit); samples {tot_s:.0f}")
    for n, s, ln, src in lines[:a.top]:
        print(f"{n / a.per:9.1f} {100 * n / total:5.1f}%  smp {100 * s / max(1, tot_s):5.1f}%  L{ln:>5}  {src}")


if __name__ == "__main__":
    main()
