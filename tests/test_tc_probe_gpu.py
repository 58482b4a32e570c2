"""The tcgen05 A/B probe of K2's score phase (tools/tc_probe.cu, DESIGN.md §3
"Measured A/B, tcgen05 against mma.sync") stays numerically checked: both
variants -- mma.sync and tcgen05 with the A operand and the accumulators in
TMEM -- must match the host fp64 scores of the first 64 blocks.  The probe is
measurement tooling, not the product path; this keeps its numbers honest."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_tc_probe_variants_match_fp64(tmp_path):
    exe = tmp_path / "tc_probe"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                    os.path.join(ROOT, "tools", "tc_probe.cu"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "4096"], capture_output=True, text=True, timeout=300, check=True).stdout
    lines = [json.loads(x) for x in out.splitlines() if x.startswith("{")]
    assert len(lines) == 3 and any("tcgen05" in d["variant"] for d in lines)
    for d in lines:
        # scores up to ~1.3e2 from 128-term sums of ~22-bit B products: 1e-5 of the range
        assert d["max_abs_err_vs_fp64"] <= 1e-5 * d["ref_max"] + 1e-3, d
