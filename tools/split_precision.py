#!/usr/bin/env python
"""fp32 output error of one predecode vs the oracle as a function of the K2
split count (run once per SPC_NSPLIT value: the split count is read once per
process).  Geometry and data as tests/test_bench_geometry_gpu.py; the work is
tests/precision_child.py.

  for s in 4 8 16 32; do SPC_NSPLIT=$s python tools/split_precision.py --case c4_share8; done
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    from precision_child import run
    from test_bench_geometry_gpu import CASES

    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="c4_share8")
    ap.add_argument("--seqs", default="0,31")
    a = ap.parse_args()
    c = CASES[a.case]
    res = run(c["b"], c["H"], c["Hq"], c["n0"], c["bits"], c["k"], [int(s) for s in a.seqs.split(",")])
    res["case"] = a.case
    print(json.dumps(res))


if __name__ == "__main__":
    main()
