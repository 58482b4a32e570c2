"""Multi-process (gloo, world size 2) coverage of the N>1 path on CPU.

bench.py shards the decode by sequence with no data-path collective: each
rank owns its sequences' caches.  These tests check, with the oracle as the
compute stand-in, that (1) per-rank sharded decode results equal a
single-process run (the path is exchange-free under sequence sharding, incl.
the layer-scope top-k), and (2) the timing/aggregation helpers of bench.py
reduce with MAX over ranks and count whole-job tokens.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restate as R
from oracle.synth import make_kv, make_queries, make_step_kv

WORLD = 2
CFG = dict(n0=300, H=2, Hq=4, d=16, bits=2, g=8, r=8, k=6, seqs=4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _seq_inputs(seq):
    rng = np.random.default_rng(100 + seq)
    K, V = make_kv(rng, CFG["n0"], CFG["H"], CFG["d"])
    q = make_queries(rng, 2, CFG["Hq"], CFG["d"])
    kn, vn = make_step_kv(rng, 2, CFG["H"], CFG["d"])
    return K, V, q, kn, vn


def _decode_seq(seq):
    K, V, q, kn, vn = _seq_inputs(seq)
    st = R.LayerState(CFG["H"], CFG["d"], CFG["bits"], CFG["g"], CFG["r"], CFG["k"])
    st.extend(K, V)
    res = R.decode_layer(st, q, kn, vn)
    picked = np.full(CFG["k"], -1, np.int64)
    picked[:len(res["picked"][0])] = res["picked"][0]
    return res["out"].astype(np.float32), picked


def _worker(rank, port, out_q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    mine = list(range(rank, CFG["seqs"], WORLD))            # sequence sharding
    outs = {s: _decode_seq(s) for s in mine}
    gathered = [None] * WORLD
    dist.all_gather_object(gathered, outs)
    # bench.py aggregation: MAX of per-rank elapsed, whole-job tokens
    import bench
    elapsed = torch.tensor([10.0 + rank], dtype=torch.float64)
    mx = bench.reduce_max(elapsed.item())
    tokens = bench.whole_job_tokens(batch=len(mine), steps=5, world=WORLD)
    if rank == 0:
        merged = {}
        for g in gathered:
            merged.update(g)
        out_q.put((merged, mx, tokens))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sequence_sharding_is_exchange_free_and_max_reduced():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    merged, mx, tokens = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert mx == 11.0
    assert tokens == 2 * 5 * WORLD
    for s in range(CFG["seqs"]):
        out, picked = _decode_seq(s)
        np.testing.assert_array_equal(merged[s][0], out)
        np.testing.assert_array_equal(merged[s][1], picked)


def test_plan_host_layers():
    import bench
    cfg = dict(bench.CONFIGS["c2"])
    slab = 2 * cfg["batch"] * (cfg["ctx"] + 256) * cfg["kv_heads"] * cfg["head_dim"] * 2
    # 196 GB box, 1 rank: largest divisor of 32 layers within 45% of available
    hl = bench.plan_host_layers(cfg, 1, avail=196 << 30)
    assert cfg["layers"] % hl == 0 and hl * slab <= 0.45 * (196 << 30)
    assert bench.plan_host_layers(cfg, 8, avail=196 << 30) == 1
    assert bench.plan_host_layers(cfg, 1, avail=4 << 40) == 32


# ---- KV-head sharding (shard.py): layer-scope top-k needs the agg all-reduce ----
HCFG = dict(n0=300, H=4, Hq=8, d=16, bits=2, g=8, r=8, k=6)


def _head_inputs():
    rng = np.random.default_rng(7)
    K, V = make_kv(rng, HCFG["n0"], HCFG["H"], HCFG["d"])
    q = make_queries(rng, 2, HCFG["Hq"], HCFG["d"])
    kn, vn = make_step_kv(rng, 2, HCFG["H"], HCFG["d"])
    return K, V, q, kn, vn


def _head_decode(rank, world):
    from paper_2503_16163_b200.shard import head_shard
    sh = head_shard(HCFG["H"], HCFG["Hq"], rank, world)
    K, V, q, kn, vn = _head_inputs()
    st = R.LayerState(sh.kv_heads, HCFG["d"], HCFG["bits"], HCFG["g"], HCFG["r"], HCFG["k"])
    st.extend(sh.slice_kv(K), sh.slice_kv(V))
    res = R.decode_layer(st, sh.slice_q(q), sh.slice_kv(kn), sh.slice_kv(vn))
    return res, st.f


def _head_worker(rank, port, out_q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2503_16163_b200.shard import allreduce_sum
    res, f = _head_decode(rank, WORLD)
    agg = torch.from_numpy(np.ascontiguousarray(res["agg"][0], np.float32))   # this rank's partial
    allreduce_sum()(agg)
    picked = R.select_topk(agg.numpy(), HCFG["k"], range(f))
    out_q.put((rank, res["out"], agg.numpy(), picked))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_head_sharding_layer_scope_allreduce():
    """Each rank attends its half of the kv heads; the summed partial
    aggregates select the same top-k as the single-process layer (engine.py:317)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_head_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict((r, rest) for r, *rest in (q.get(timeout=240) for _ in range(WORLD)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full, f = _head_decode(0, 1)
    from paper_2503_16163_b200.shard import head_shard
    for rank, (out, agg, picked) in got.items():
        sh = head_shard(HCFG["H"], HCFG["Hq"], rank, WORLD)
        np.testing.assert_array_equal(out, full["out"][:, sh.q_lo:sh.q_hi])
        np.testing.assert_allclose(agg, full["agg"][0], rtol=1e-6, atol=1e-9)
        assert picked == full["picked"][0]


def test_head_shard_ranges():
    from paper_2503_16163_b200.shard import head_shard
    shards = [head_shard(8, 32, r, 4) for r in range(4)]
    assert [(s.kv_lo, s.kv_hi, s.q_lo, s.q_hi) for s in shards] == [
        (0, 2, 0, 8), (2, 4, 8, 16), (4, 6, 16, 24), (6, 8, 24, 32)]
    assert all(s.q_heads == 4 * s.kv_heads for s in shards)   # GQA groups stay whole
    with pytest.raises(ValueError):
        head_shard(8, 32, 0, 3)      # heads run out -> shard by sequence instead
    with pytest.raises(ValueError):
        head_shard(8, 32, 4, 4)


# ---- the bench launcher and the (KV head x sequence) partition (bench.py --gpus N) ----
def test_plan_partition_heads_then_batch():
    from paper_2503_16163_b200.shard import plan_partition
    # C3: 8 KV heads over 2/4/8 ranks -> pure head sharding, global batch 8 on every rank
    for n in (2, 4, 8):
        parts = [plan_partition(8, 32, 8, r, n) for r in range(n)]
        assert all(p.head_groups == n and p.batch_groups == 1 and p.batch == 8 for p in parts)
        assert sorted((p.heads.kv_lo, p.heads.kv_hi) for p in parts) == [(i * 8 // n, (i + 1) * 8 // n)
                                                                       for i in range(n)]
        assert all(p.agg_group == list(range(n)) for p in parts)
    # heads run out: 16 ranks over 8 KV heads -> 2 batch slices of 16 sequences (C4's batch 32)
    parts = [plan_partition(8, 32, 32, r, 16) for r in range(16)]
    assert {(p.head_groups, p.batch_groups) for p in parts} == {(8, 2)}
    assert parts[3].seq_lo == 0 and parts[11].seq_lo == 16 and parts[11].heads.kv_lo == 3
    assert parts[11].agg_group == list(range(8, 16))
    # 3 ranks, 8 heads: gcd 1 -> batch sharding; C3's batch 8 does not split over 3
    with pytest.raises(ValueError):
        plan_partition(8, 32, 8, 0, 3)
    assert plan_partition(8, 32, 6, 2, 3).seq_lo == 4
    assert plan_partition(32, 32, 16, 1, 2, "seq").heads.kv_heads == 32


def _dry(args):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args, capture_output=True, text=True,
                         timeout=240, cwd="/tmp", env=dict(os.environ, PYTHONPATH=root))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.timeout(300)
def test_bench_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun relaunches itself with 2 ranks
    (torch.distributed.run); rank 0 alone prints the JSON line."""
    d = _dry(["--gpus", "2", "--config", "c3", "--dry-run"])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 8
    assert [r["kv"] for r in d["ranks"]] == [[0, 4], [4, 8]]
    assert all(r["seqs"] == [0, 8] and r["agg_group"] == [0, 1] for r in d["ranks"])


@pytest.mark.timeout(300)
def test_reference_arm_config_matches_gpu_arm():
    """Both arms print the same `config` object for the same workload."""
    import argparse
    import bench
    args = argparse.Namespace(shard="auto", share=0, gpus=2)
    a = bench.workload_config(dict(bench.CONFIGS["c3"]), 2, args)
    d = _dry(["--gpus", "2", "--config", "c3", "--dry-run"])
    assert a == d["config"]


def test_ctx128k_companion_summary(monkeypatch):
    """The default single-GPU bench line carries the metric's 128k half: a C3
    child run whose JSON line is summarised into `ctx_128k` (or the reason it
    is missing); the child itself is told not to recurse."""
    import argparse
    import json
    import subprocess
    import bench
    seen = {}
    child = {"config": {"workload": "C3: ..."}, "value": 596.0, "unit": "tokens/s", "ms_per_step": 13.4,
             "steps": 10, "warmup": 3, "e2e": {"value": 611.0},
             "roofline": {"achieved": 1320.0, "peak": 6500.0, "frac": 0.2, "traffic": 6.6e8,
                          "avg_launch_ms": 0.41, "kernel_share_of_step": 0.98},
             "prefetch": {"exposed_fraction": 0.006, "h2d_gbs": 35.5, "h2d_frac": 0.64},
             "gpu_launches": 1920, "clocks": {"sm_mhz": 1965.0}, "topk_parity": {"band": 1e-4}}

    def fake_run(cmd, **kw):
        seen["cmd"] = cmd
        return subprocess.CompletedProcess(cmd, 0, stdout="[log]\n" + json.dumps(child) + "\n", stderr="")

    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    s = bench.run_ctx128k_companion(argparse.Namespace(steps=10, warmup=3))
    assert "--no-ctx128k" in seen["cmd"] and seen["cmd"][seen["cmd"].index("--config") + 1] == "c3"
    assert s["value"] == 596.0 and s["e2e"] == 611.0 and s["roofline"]["frac"] == 0.2
    assert s["prefetch"]["h2d_frac"] == 0.64 and s["steps"] == 10

    def failing_run(cmd, **kw):
        return subprocess.CompletedProcess(cmd, 1, stdout="", stderr="CUDA out of memory")

    monkeypatch.setattr(bench.subprocess, "run", failing_run)
    s = bench.run_ctx128k_companion(argparse.Namespace(steps=10, warmup=3))
    assert "unavailable" in s and "out of memory" in s["unavailable"]
