"""K2 accumulator fold (attend_mma.cu, SPC_K2_FOLD): long per-warp block runs.

mma.sync's fp32 accumulation truncates toward the accumulator's magnitude; the
value sum's unsigned-code part and zero-point part grow linearly over a warp's
blocks and cancel in the output, so without the fold the output error grows
with the blocks per warp (2.6e-3 at 64, 1.1e-2 at 256 -- profiles/r2_35_fold.json).
Each case forces 4 splits of a 128k context (SPC_NSPLIT=4: 1024 blocks per
split, 128 per warp, the folding instantiation) in a child process and bounds
the fp32 output per q head by the decode contract's 2e-3 against the oracle.
MHA rows take the PG layout (NR <= 2), GQA-4 rows the cooperative-decode one."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("H,Hq,bits", [(4, 4, 1), (4, 4, 2), (1, 4, 1), (1, 4, 2)])
def test_long_warp_runs_within_contract(H, Hq, bits):
    env = dict(os.environ, SPC_NSPLIT="4")
    out = subprocess.run([sys.executable, os.path.join(HERE, "precision_child.py"), "--b", "2", "--H", str(H),
                          "--Hq", str(Hq), "--bits", str(bits), "--n0", "131072", "--seqs", "1"],
                         env=env, capture_output=True, text=True, timeout=540)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["max_rel_err"] <= 2e-3, res["max_rel_err"]
