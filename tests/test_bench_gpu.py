"""bench.py's multi-rank launcher end to end on the device: `--gpus 2` outside
torchrun relaunches itself with two ranks (here both on cuda:0 over gloo,
SPC_BENCH_BACKEND=gloo; on an 8-GPU box one rank per GPU over NCCL), splits
the 8 KV heads of the C3-shaped `tiny` config over the ranks, all-reduces each
layer's partial top-k aggregate, and rank 0 prints one JSON line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(900)
def test_bench_two_ranks_head_sharded():
    env = dict(os.environ, SPC_BENCH_BACKEND="gloo", PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "tiny",
                          "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--host-layers", "1"],
                         capture_output=True, text=True, timeout=800, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 8
    assert d["scaling"] == "strong"
    assert d["rank_share"]["kv_heads"] == 4 and d["rank_share"]["q_heads"] == 16 and d["rank_share"]["batch"] == 8
    assert "kv-heads x2" in d["config"]["parallelism"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


@pytest.mark.timeout(600)
def test_bench_step_graphs():
    """`--graph`: every step (and every e2e step with its host copies) as one
    CUDA graph; the line carries the graph stats and the eager pass's timings."""
    env = dict(os.environ, PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--graph",
                          "--steps", "20", "--warmup", "3", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=500, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    inst, upd = d["graph"]["instantiations_updates"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["roofline"]["frac"] > 0
    assert 1 <= inst <= 8 and upd >= 30, (inst, upd)
