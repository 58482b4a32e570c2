#!/usr/bin/env python
"""bench.py -- SpeCache dual-token decode on B200 (BASELINE.json metric).

One step = one dual-token decode step (engine.py:286-339's per-layer body,
hot path only: K2 attend over the 1/2-bit tier + pinned/residual/in-step rows,
K3 combine + cross-head aggregate, K4 top-k + pin diff, K5 PCIe prefetch of new
pins, K6 append) over ALL layers of the model for the whole batch.  Tokens per
step = batch (row 0 emits one verified token per sequence, engine.py:172).

Default workload: BASELINE.json configs[1] ("c2"): LLaMA-2-7B-shaped 32-layer
decode, MHA 32 heads x d=128, ctx 32k, batch 16, 2-bit KV (g=32, r=64),
top-k 64, one B200.  Inputs are synthetic (seeded, bf16), post-RoPE q/k/v
(the projections around the hot path are out of scope).  Per-step data
(~52 GB of low-bit KV) is far larger than L2 (126 MB), so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c1]
  python bench.py --impl reference ...     # CPU reference arm (oracle port)

Multi-GPU (torchrun, one rank per GPU): the path shards by sequence with no
data-path collective -- every rank runs its own batch (weak scaling); NCCL is
used only for the barrier and the max-over-ranks timing.  `--shard heads`
instead splits the config's KV heads over the ranks (strong scaling, the
north star's partitioning): each layer's partial top-k aggregate is summed
across ranks by an NCCL all-reduce on the cache's copy stream (shard.py).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1] -- the metric's single-GPU configuration
    "c2": dict(workload="C2: LLaMA-2-7B-shaped 32-layer SpeCache decode, MHA 32 heads x d128, "
                        "ctx 32k, batch 16, 2-bit KV (g32, r64), top-k 64",
               layers=32, batch=16, kv_heads=32, q_heads=32, head_dim=128, ctx=32768, bits=2,
               group=32, residual=64, topk=64),
    # BASELINE.json configs[2] per GPU
    "c3": dict(workload="C3: Mistral-7B-shaped GQA (8 KV heads) 32-layer decode, ctx 128k, batch 8, "
                        "1-bit KV (g32, r64), top-k 128",
               layers=32, batch=8, kv_heads=8, q_heads=32, head_dim=128, ctx=131072, bits=1,
               group=32, residual=64, topk=128),
    # BASELINE.json configs[3], one rank's share: global batch 32 over 8 GPUs -> 4
    # sequences per rank (sequence sharding); `--gpus 8` under torchrun is C4 itself
    "c4": dict(workload="C4: LLaMA-3-8B-shaped GQA (8 KV heads) 32-layer decode, ctx 128k, global batch 32 "
                        "over 8 GPUs (4 per rank), 1-bit KV (g32, r64), top-k 256, full bf16 cache in pinned host",
               layers=32, batch=4, kv_heads=8, q_heads=32, head_dim=128, ctx=131072, bits=1,
               group=32, residual=64, topk=256),
    # C3's geometry at 2 bits (not a BASELINE config): the 2-bit x 8-row K2 instantiation
    "c3b2": dict(workload="C3 geometry at 2-bit: Mistral-7B-shaped GQA (8 KV heads) 32-layer decode, ctx 128k, "
                          "batch 8, 2-bit KV (g32, r64), top-k 128",
                 layers=32, batch=8, kv_heads=8, q_heads=32, head_dim=128, ctx=131072, bits=2,
                 group=32, residual=64, topk=128),
    # BASELINE.json configs[0] (parity config; launch-bound)
    "c1": dict(workload="C1: single-layer SpeCache decode, 32 heads x d128, ctx 4096, 2-bit KV, "
                        "top-k 64, residual 32, batch 1",
               layers=1, batch=1, kv_heads=32, q_heads=32, head_dim=128, ctx=4096, bits=2,
               group=32, residual=32, topk=64),
}
METRIC = "decode tokens/s at 32k/128k ctx (device-timed), HBM & H2D roofline fraction"
NEEDLES = 256        # planted high-score keys per (seq, kv head): peaky attention
DRIFT = 0.3          # q_{t+1} = bf16(q_t + DRIFT * N(0,1))


# -------------------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    return rank, world, local, local_world


def reduce_max(value: float, device=None) -> float:
    """Max over ranks (the timing rule: a multi-GPU number is the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_tokens(batch: int, steps: int, world: int) -> int:
    """Every rank decodes its own `batch` sequences (sequence sharding, weak
    scaling); one verified token per sequence per step (engine.py:172)."""
    return batch * steps * world


def measure_h2d_peak(device, nbytes: int = 256 << 20, reps: int = 5) -> float:
    """Host-link roofline for K5: best pinned-host -> device cudaMemcpy of one
    large buffer, GB/s (CUDA events).  Measured outside any timed region."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(reps):
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize(device)
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    del src, dst
    return best


def mem_available_bytes() -> int:
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 64 << 30


def plan_host_layers(cfg: dict, local_world: int, avail: int | None = None, frac: float = 0.45) -> int:
    """Distinct pinned-host slow-tier slabs per rank: the largest divisor of
    `layers` whose slabs fit in `frac` of the host's available memory shared by
    the ranks on this node.  Layers l and l' with l == l' (mod host_layers) are
    fed identical KV, so the aliased slab is exact for both."""
    avail = mem_available_bytes() if avail is None else avail
    slab = 2 * cfg["batch"] * (cfg["ctx"] + 256) * cfg["kv_heads"] * cfg["head_dim"] * 2
    budget = frac * avail / max(1, local_world)
    best = 1
    for hl in range(1, cfg["layers"] + 1):
        if cfg["layers"] % hl == 0 and hl * slab <= budget:
            best = hl
    return best


def algorithmic_bytes_per_layer(cfg: dict, n: int, f: int, npin: int) -> dict:
    """HBM = sum over (seq, kv head) of [f*b_tok + n_pin*4d +
    (n-f)*4d + 2*4d] + q in + O out; b_tok = d(B/4 + 8/g) (fp16/bf16 params)."""
    d, B, g = cfg["head_dim"], cfg["bits"], cfg["group"]
    b_tok = d * (B / 4 + 8 / g)
    units = cfg["batch"] * cfg["kv_heads"]
    kv = units * (f * b_tok + npin * 4 * d + (n - f) * 4 * d + 2 * 4 * d)
    qo = cfg["batch"] * 2 * cfg["q_heads"] * d * 2 * 2
    return {"hbm": kv + qo, "flops": 8 * cfg["batch"] * cfg["q_heads"] * n * d, "b_tok": b_tok}


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML in a
    thread every 10 ms, so a ~0.2 s timed region still gets ~20 samples; the
    nvidia-smi CLI is the fallback when pynvml is missing)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []   # (sm_mhz, max_mhz, {reason names})
        self.proc = None
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx),
                                          {n for n, b in zip(self.NAMES, bits) if rs & b}))
                    except Exception:
                        pass
                    self.stop.wait(0.01)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) == 7 and p[0].replace(".", "").isdigit():
                self.rows.append((float(p[0]), float(p[1]) if p[1].replace(".", "").isdigit() else 0.0,
                                  {self.NAMES[i] for i in range(4) if p[3 + i] == "Active"}))

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif self.thread:
            self.thread.join(timeout=1)

    def summary(self) -> dict:
        sm = sorted(r[0] for r in self.rows)
        mx = [r[1] for r in self.rows if r[1] > 0]
        reasons = sorted(set().union(*[r[2] for r in self.rows])) if self.rows else []
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self.proc is None else "nvidia-smi"}


# -------------------------------------------------------------------------------------
def cpu_reference_sample(cfg: dict, threads: int, units: int, seed: int = 0) -> dict:
    """Time the CPU reference path (oracle port of engine.py:299-321: dequantize
    every packed group, attend both rows, aggregate, select_topk) on `units`
    (layer, seq) units of `cfg`, `threads` at a time.  Returns tokens/s
    extrapolated to the full step (layers x batch units per `batch` tokens)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from oracle import restate as R
    from oracle.synth import make_kv, make_queries, make_step_kv

    H, Hq, d, n = cfg["kv_heads"], cfg["q_heads"], cfg["head_dim"], cfg["ctx"]

    def prep(i):
        rng = np.random.default_rng(seed + i)
        st = R.LayerState(H, d, cfg["bits"], cfg["group"], cfg["residual"], cfg["topk"])
        K, V = make_kv(rng, n, H, d)
        st.extend(K, V)
        st._sync_packed()  # prefill quantization is not part of the decode step
        q = make_queries(rng, 2, Hq, d)
        kn, vn = make_step_kv(rng, 2, H, d)
        return st, q, kn, vn

    def run(args):
        st, q, kn, vn = args
        t0 = time.perf_counter()
        R.decode_layer(st, q, kn, vn, append=False)
        return time.perf_counter() - t0

    with ThreadPoolExecutor(max(1, min(8, threads))) as ex:
        work = list(ex.map(prep, range(units)))
    with ThreadPoolExecutor(threads) as ex:
        t0 = time.perf_counter()
        per_unit = list(ex.map(run, work))
        wall = time.perf_counter() - t0
    units_per_step = cfg["layers"] * cfg["batch"]
    step_s = units_per_step * wall / units
    return {"value": cfg["batch"] / step_s, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"{units} of {units_per_step} (layer, seq) decode units of {cfg['workload'][:2]} "
                      f"(n={n}), {threads} threads, wall {wall:.2f}s, "
                      f"median unit {sorted(per_unit)[len(per_unit) // 2]:.2f}s; "
                      f"tokens/s extrapolated to the full step"}


def run_reference_arm(args, cfg):
    rank, world, _, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    units = threads
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(cfg, threads, units, seed=1000 * i)
        if i >= args.warmup:
            vals.append(r)
    value = sum(v["value"] for v in vals) / len(vals)
    base = vals[-1]
    base["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * cfg["batch"] / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["workload"], "global_batch": cfg["batch"], "seq_len": cfg["ctx"],
                       "parallelism": "cpu threads"},
            "cpu_baseline": base,
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------------------------------
def make_inputs(cfg, steps, device, host_layers, seed):
    """Per-step q / k_new / v_new for every layer, resident in HBM, plus the
    initial query direction per layer (for the needles)."""
    import torch
    b, H, Hq, d, L = cfg["batch"], cfg["kv_heads"], cfg["q_heads"], cfg["head_dim"], cfg["layers"]
    gen = torch.Generator(device=device).manual_seed(seed)
    # q stream per layer: s(t+1) = bf16(s(t) + DRIFT*N); row0(t) = s(t), row1(t) = s(t+1)
    s = torch.randn((L, b, Hq, d), device=device, generator=gen).to(torch.bfloat16)
    s0 = s.clone()
    qs = []
    for _ in range(steps + 1):
        qs.append(s)
        s = (s.float() + DRIFT * torch.randn(s.shape, device=device, generator=gen)).to(torch.bfloat16)
    q = torch.stack([torch.stack([qs[t], qs[t + 1]], dim=2) for t in range(steps)])  # [T, L, b, 2, Hq, d]
    kv = torch.randn((2, steps, host_layers, b, 2, H, d), device=device, generator=gen).to(torch.bfloat16)
    idx = torch.arange(L, device=device) % host_layers
    k_new = kv[0][:, idx].contiguous()  # layers aliased mod host_layers carry identical KV
    v_new = kv[1][:, idx].contiguous()
    return q.contiguous(), k_new, v_new, s0


def prefill_cache(cache, cfg, host_layers, s0, device, seed):
    """Synthetic prompt KV per distinct slab, quantized into every layer that
    aliases it.  K = N(0,1) + per-(head, channel) offset N(0,2^2); V = N(0,1);
    NEEDLES keys per (seq, head) get += 0.5 * the layer's initial query."""
    import torch
    b, H, Hq, d, n = cfg["batch"], cfg["kv_heads"], cfg["q_heads"], cfg["head_dim"], cfg["ctx"]
    G = Hq // H
    for j in range(host_layers):
        gen = torch.Generator(device=device).manual_seed(seed + 7919 * j)
        K = torch.randn((b, n, H, d), device=device, generator=gen)
        K += 2.0 * torch.randn((1, 1, H, d), device=device, generator=gen)
        qdir = s0[j].float().view(b, H, G, d).mean(2)  # [b, H, d]
        pos = torch.randint(0, n - cfg["residual"] - cfg["group"], (b, NEEDLES, H), device=device,
                            generator=gen)
        bi = torch.arange(b, device=device)[:, None, None].expand_as(pos)
        hi = torch.arange(H, device=device)[None, None, :].expand_as(pos)
        K[bi, pos, hi] += 0.5 * qdir[bi, hi]
        Kb = K.to(torch.bfloat16)
        del K
        Vb = torch.randn((b, n, H, d), device=device, generator=gen).to(torch.bfloat16)
        for layer in range(j, cfg["layers"], host_layers):
            cache.prefill(layer, Kb, Vb)
        del Kb, Vb
        torch.cuda.synchronize(device)


def agg_reducer(cache, layers, device):
    """Per-layer cross-rank sum of the partial top-k aggregate for a KV-head
    sharded cache (shard.py): NCCL all-reduce on the layer's copy stream, then
    the rest of the ticket (spc_finish_layer).  Views and streams are built once."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2503_16163_b200 import _lib
    from paper_2503_16163_b200.decode import _device_f32
    lib, h = _lib.lib(), cache.handle
    views = []
    for layer in range(layers):
        ptr, count, st = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_void_p()
        _lib.check(lib.spc_agg_buffer(h, layer, ctypes.byref(ptr), ctypes.byref(count), ctypes.byref(st)))
        views.append((_device_f32(ptr.value, count.value, device), torch.cuda.ExternalStream(st.value, device=device)))

    def reduce(layer):
        v, s = views[layer]
        with torch.cuda.stream(s):
            dist.all_reduce(v)
        _lib.check(lib.spc_finish_layer(h, layer))

    return reduce


def run_gpu_arm(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder
    from paper_2503_16163_b200 import _lib

    rank, world, local, local_world = dist_env()
    torch.cuda.set_device(local)
    device = f"cuda:{local}"
    heads = args.shard == "heads"
    if world > 1 or heads:  # head sharding reduces the aggregate even at N=1 (a 1-rank NCCL group)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        dist.init_process_group("nccl", device_id=torch.device(device), rank=rank, world_size=world)
    if heads:
        from paper_2503_16163_b200.shard import head_shard
        sh = head_shard(cfg["kv_heads"], cfg["q_heads"], rank, world)
        cfg = dict(cfg, kv_heads=sh.kv_heads, q_heads=sh.q_heads)

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        cpu_base = cpu_reference_sample(cfg, threads, threads)

    W, K = args.warmup, args.steps
    total_steps = 2 * (W + K)  # device-timed pass + end-to-end pass
    host_layers = args.host_layers or plan_host_layers(cfg, local_world)
    budget = CacheBudget(bits=cfg["bits"], group_size=cfg["group"], residual=cfg["residual"],
                         prefetch_k=cfg["topk"], context_length=cfg["ctx"] + total_steps + 64)
    t_setup = time.perf_counter()
    cache = DeviceTwoTierCache(cfg["layers"], cfg["kv_heads"], cfg["head_dim"], budget,
                               batch=cfg["batch"], q_heads=cfg["q_heads"], device=local,
                               host_layers=host_layers)
    reduce_layer = None
    if heads:
        from paper_2503_16163_b200.shard import allreduce_sum
        dec = SpeculativeLayerDecoder(cache, agg_reduce=allreduce_sum())
        reduce_layer = agg_reducer(cache, cfg["layers"], device)
    else:
        dec = SpeculativeLayerDecoder(cache)
    q, k_new, v_new, s0 = make_inputs(cfg, total_steps + 1, device, host_layers, seed=1234 + rank)
    prefill_cache(cache, cfg, host_layers, s0, device, seed=99 + rank)
    L = cfg["layers"]
    out = torch.empty((L, cfg["batch"], 2, cfg["q_heads"], cfg["head_dim"]), dtype=torch.bfloat16,
                      device=device)
    pm = torch.empty((L, cfg["batch"], cfg["q_heads"]), dtype=torch.float32, device=device)
    lib, h = _lib.lib(), cache.handle
    stream = torch.cuda.current_stream(device).cuda_stream

    def step_device(t, qt, kt, vt):
        for layer in range(L):
            _lib.check(lib.spc_decode_layer(h, layer, t, qt[layer].data_ptr(), kt[layer].data_ptr(),
                                            vt[layer].data_ptr(), out[layer].data_ptr(),
                                            pm[layer].data_ptr(), stream))
            if reduce_layer:
                reduce_layer(layer)

    # predecode (Alg. 2): first tickets
    for layer in range(L):
        dec.predecode_layer(layer, q[0, layer][:, :1], k_new[0, layer][:, :1], v_new[0, layer][:, :1])
    torch.cuda.synchronize(device)
    setup_s = time.perf_counter() - t_setup
    h2d_peak = measure_h2d_peak(device)

    import ctypes
    def profile(enable):
        am, al, sm, sl, nl = (ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(),
                              ctypes.c_int64(), ctypes.c_int64())
        _lib.check(lib.spc_profile(h, enable, ctypes.byref(am), ctypes.byref(al), ctypes.byref(sm),
                                   ctypes.byref(sl), ctypes.byref(nl)))
        return am.value, al.value, sm.value, sl.value, nl.value

    t = 1
    for _ in range(W):
        step_device(t, q[t], k_new[t], v_new[t])
        t += 1
    n_mid = cache.length(0)
    f_mid = cache.quantized_frontier(0)
    # new-pin statistics over the timed region
    picked0, newc0 = dec.ticket(0)
    torch.cuda.synchronize(device)
    profile(1)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    newpins = []
    with ClockSampler(local) as clocks:
        ev0.record()
        for _ in range(K):
            step_device(t, q[t], k_new[t], v_new[t])
            t += 1
        ev1.record()
        torch.cuda.synchronize(device)
    elapsed_ms = ev0.elapsed_time(ev1)
    attn_ms, attn_n, sel_ms, sel_n, launches = profile(0)
    wait_ms = lib.spc_profile_wait_ms(h)
    pf_ms = lib.spc_profile_prefetch_ms(h)
    pf_bytes = int(lib.spc_profile_prefetch_bytes(h))
    _, newc = dec.ticket(L // 2)
    npin = int((picked0 >= 0).sum().item()) // max(1, cfg["batch"])
    new_frac = float(newc.float().mean().item()) / max(1, cfg["topk"])
    elapsed_ms = reduce_max(elapsed_ms, device)
    if world > 1:
        dist.barrier()

    # ---- end-to-end: host buffers in, host results out, copies inside the region ----
    # inputs staged per step in pinned host memory before the region; the
    # region copies them H2D, runs the step, and reads the results back
    e2e_in = [(q[i].cpu().pin_memory(), k_new[i].cpu().pin_memory(), v_new[i].cpu().pin_memory())
              for i in range(t, t + W + K)]
    o_h = torch.empty_like(out, device="cpu").pin_memory()
    pm_h = torch.empty_like(pm, device="cpu").pin_memory()
    q_d, k_d, v_d = torch.empty_like(q[0]), torch.empty_like(k_new[0]), torch.empty_like(v_new[0])

    # layer-pipelined: layer l+1's inputs copy H2D on one copy stream while layer
    # l decodes, and layer l's outputs copy D2H on another; the step ends when
    # its last results are on the host (the compute stream waits for them)
    comp = torch.cuda.current_stream(device)
    cs_in, cs_out = torch.cuda.Stream(device), torch.cuda.Stream(device)

    GRP = 8  # layers per copy group: one H2D and one D2H per group keeps the host-side cost low

    def step_e2e(i, tt):
        qh, kh, vh = e2e_in[i]
        groups = [(g0, min(L, g0 + GRP)) for g0 in range(0, L, GRP)]
        ev_in = [torch.cuda.Event() for _ in groups]
        cs_in.wait_stream(comp)  # the previous step is done with q_d / k_d / v_d
        with torch.cuda.stream(cs_in):
            for gi, (g0, g1) in enumerate(groups):
                q_d[g0:g1].copy_(qh[g0:g1], non_blocking=True)
                k_d[g0:g1].copy_(kh[g0:g1], non_blocking=True)
                v_d[g0:g1].copy_(vh[g0:g1], non_blocking=True)
                ev_in[gi].record(cs_in)
        for gi, (g0, g1) in enumerate(groups):
            comp.wait_event(ev_in[gi])
            for layer in range(g0, g1):
                _lib.check(lib.spc_decode_layer(h, layer, tt, q_d[layer].data_ptr(), k_d[layer].data_ptr(),
                                                v_d[layer].data_ptr(), out[layer].data_ptr(),
                                                pm[layer].data_ptr(), stream))
                if reduce_layer:
                    reduce_layer(layer)
            ev = torch.cuda.Event()
            ev.record(comp)
            cs_out.wait_event(ev)
            with torch.cuda.stream(cs_out):
                o_h[g0:g1].copy_(out[g0:g1], non_blocking=True)
                pm_h[g0:g1].copy_(pm[g0:g1], non_blocking=True)
        comp.wait_stream(cs_out)

    for i in range(W):
        step_e2e(i, t)
        t += 1
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    w0 = time.perf_counter()
    for i in range(W, W + K):
        step_e2e(i, t)
        t += 1
    torch.cuda.synchronize(device)
    e2e_s = time.perf_counter() - w0
    e2e_s = reduce_max(e2e_s, device)
    h2d = (q_d.numel() + k_d.numel() + v_d.numel()) * 2
    d2h = o_h.numel() * 2 + pm_h.numel() * 4

    ms_per_step = elapsed_ms / K
    tokens = cfg["batch"] * K if heads else whole_job_tokens(cfg["batch"], K, world)
    value = tokens / (elapsed_ms / 1e3)
    ab = algorithmic_bytes_per_layer(cfg, n_mid + K // 2, f_mid, npin)
    attn_avg_ms = attn_ms / max(1, attn_n)
    achieved = ab["hbm"] / (attn_avg_ms / 1e3) / 1e9
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
        peak, peak_src = float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh).get(args.config)
            if tr and tr.get("kernel_impl") == ("fast" if cache.fast_path else "generic"):
                traffic = tr["bytes_per_launch"]
    except (OSError, ValueError):
        pass
    h2d_pf = pf_bytes / K  # measured: new pins x row bytes, summed over the timed steps
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if heads else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded; peaky: %d needle keys per "
        "(seq, kv head), q drift sigma %.1f)" % (NEEDLES, DRIFT),
        "config": {"workload": cfg["workload"], "global_batch": cfg["batch"] * (1 if heads else world),
                   "seq_len": cfg["ctx"], "layers": cfg["layers"],
                   "parallelism": (f"kv-heads x{world} ({cfg['kv_heads']} kv / {cfg['q_heads']} q heads per rank; "
                                   "per-layer NCCL all-reduce of the top-k aggregate on the copy stream)") if heads
                   else f"replicas-by-sequence x{world} (no collective)",
                   "bits": cfg["bits"], "topk": cfg["topk"], "l2": "no flush: per-step KV traffic "
                   "%.1f GB >> 126 MB L2" % (ab["hbm"] * cfg["layers"] / 1e9),
                   "host_layers": host_layers, "attention_impl": "fast" if cache.fast_path else "generic"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "K2 attend (per layer launch, all sequences)",
                     "algorithmic_bytes_per_launch": ab["hbm"], "avg_launch_ms": attn_avg_ms,
                     "launches": attn_n, "kernel_share_of_step": attn_ms / max(1e-9, elapsed_ms)},
        "prefetch": {"new_pin_fraction": h2d_pf / max(1, cfg["topk"] * cfg["batch"] * cfg["layers"] * cache.row_bytes(1)),
                     "h2d_bytes_per_step": h2d_pf,
                     "exposed_ms_per_step": wait_ms / K, "exposed_fraction": wait_ms / max(1e-9, elapsed_ms),
                     "copy_stream_ms_per_step": sel_ms / K, "prefetch_kernel_ms_per_step": pf_ms / K,
                     "h2d_gbs": (h2d_pf / 1e9) / max(1e-9, pf_ms / K / 1e3),
                     "h2d_peak_gbs": h2d_peak,
                     "h2d_frac": (h2d_pf / 1e9) / max(1e-9, pf_ms / K / 1e3) / max(1e-9, h2d_peak),
                     "h2d_peak_how": "best of 5 pinned-host -> device copies of 256 MiB (CUDA events), same process"},
        "e2e": {"value": tokens / e2e_s,
                "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "how": "through spc_decode_layer (C ABI) with pinned host inputs/outputs; per group of 8 "
                       "layers, H2D of its q/k/v and D2H of its outputs on two copy streams overlapping the "
                       "other groups' decode; wall clock around synchronize, max over ranks"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "setup_s": setup_s,
        "cpu_baseline": cpu_base,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    cache.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


# model shapes around the hot path for --full-decoder (hidden, ffn, vocab); random-init weights
MODEL_SHAPES = {"c2": (4096, 11008, 32000),   # LLaMA-2-7B (two-matrix SiLU FFN, engine.py:66-68)
                "c3": (4096, 14336, 32000),   # Mistral-7B
                "c1": (4096, 11008, 32000)}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def run_full_decoder(args, cfg):
    """the whole model step around the hot path (decoder.py):
    RMSNorm / QKV GEMM / RoPE / spc_decode_layer / Wo / FFN per layer, logits and
    argmax for both rows, next tokens fed back on the device.  Random-init bf16
    weights of the named architecture; the prompt KV is synthetic (prefill_cache).
    Host slabs are aliased mod host_layers as in the hot-path bench: aliased
    layers share (and overwrite) one slow-tier slab, which keeps the PCIe
    traffic and timing identical but makes prefetched row CONTENT approximate."""
    import torch
    import torch.distributed as dist

    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache
    from paper_2503_16163_b200.decoder import DecoderStack, StackConfig, random_stack

    rank, world, local, local_world = dist_env()
    torch.cuda.set_device(local)
    device = f"cuda:{local}"
    heads = args.shard == "heads"
    if world > 1 or heads:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        dist.init_process_group("nccl", device_id=torch.device(device), rank=rank, world_size=world)
    hidden, ffn, vocab = MODEL_SHAPES[args.config]
    sh = None
    if heads:  # attention heads split over the ranks, outputs all-gathered before Wo (decoder.py)
        from paper_2503_16163_b200.shard import head_shard
        sh = head_shard(cfg["kv_heads"], cfg["q_heads"], rank, world)
    sc = StackConfig(layers=cfg["layers"], q_heads=cfg["q_heads"], kv_heads=cfg["kv_heads"],
                     head_dim=cfg["head_dim"], hidden=hidden, ffn=ffn, vocab=vocab)
    W, K = args.warmup, args.steps
    host_layers = args.host_layers or plan_host_layers(cfg, local_world)
    budget = CacheBudget(bits=cfg["bits"], group_size=cfg["group"], residual=cfg["residual"],
                         prefetch_k=cfg["topk"], context_length=cfg["ctx"] + W + K + 64)
    lcfg = dict(cfg, kv_heads=sh.kv_heads, q_heads=sh.q_heads) if sh else cfg   # this rank's heads
    cache = DeviceTwoTierCache(cfg["layers"], lcfg["kv_heads"], cfg["head_dim"], budget, batch=cfg["batch"],
                               q_heads=lcfg["q_heads"], device=local, host_layers=host_layers)
    s0 = torch.randn((host_layers, cfg["batch"], lcfg["q_heads"], cfg["head_dim"]), device=device).to(
        torch.bfloat16)
    prefill_cache(cache, lcfg, host_layers, s0, device, seed=99 + rank)
    # head sharding: every rank holds the same (replicated) weights
    weights = random_stack(sc, device, seed=7 + (0 if sh else rank))
    stack = DecoderStack(sc, weights, cache, shard=sh)
    B, n = cfg["batch"], cfg["ctx"]
    gen = torch.Generator(device=device).manual_seed(5 + rank)
    tok0 = torch.randint(0, vocab, (B,), device=device, generator=gen)
    pos = torch.full((B,), n, dtype=torch.int32, device=device)
    spec = stack.predecode(tok0, pos).clone()
    toks = torch.stack([tok0.to(torch.int32), spec], dim=1)
    step = 1
    for _ in range(W):
        toks = stack.decode_step(step, toks, pos + step - 1).clone()
        step += 1
    prof0 = cache.profile(True)
    del prof0
    stack.launches = 0
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record()
        for _ in range(K):
            toks = stack.decode_step(step, toks, pos + step - 1).clone()
            step += 1
        e1.record()
        torch.cuda.synchronize(device)
    elapsed_ms = reduce_max(e0.elapsed_time(e1), device)
    prof = cache.profile(False)
    ms_per_step = elapsed_ms / K
    tokens = B * K if heads else whole_job_tokens(B, K, world)
    value = tokens / (elapsed_ms / 1e3)
    f = cache.quantized_frontier(0)
    nn = cache.length(0)
    kv_bytes = algorithmic_bytes_per_layer(lcfg, nn - K // 2, f, cfg["topk"])["hbm"] * cfg["layers"]
    wbytes = sc.weight_bytes()
    achieved = (kv_bytes + wbytes) / (ms_per_step / 1e3) / 1e9
    peak, peak_src = hbm_peak()
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if heads else "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic prompt KV + random-init weights; tokens fed back on device",
        "config": {"workload": cfg["workload"] + f"; FULL DECODER (hidden {hidden}, ffn {ffn}, vocab {vocab})",
                   "global_batch": B * (1 if heads else world), "seq_len": n, "layers": cfg["layers"],
                   "parallelism": (f"kv-heads x{world} (attention outputs all-gathered before Wo; Wo/FFN/head "
                                   "replicated; agg all-reduce per layer)") if heads
                   else f"replicas-by-sequence x{world} (no collective)", "host_layers": host_layers,
                   "l2": "no flush: weights %.1f GB + KV %.1f GB per step >> L2" % (wbytes / 1e9, kv_bytes / 1e9)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_source": peak_src, "kernel": "whole step (KV + weights)",
                     "algorithmic_bytes_per_step": kv_bytes + wbytes, "weight_bytes_per_step": wbytes,
                     "kv_bytes_per_step": kv_bytes},
        "breakdown_ms_per_step": {"attend_k2": prof["attn_ms"] / K,
                                  "rest_of_step": ms_per_step - prof["attn_ms"] / K,
                                  "weights_at_peak": wbytes / peak / 1e6,
                                  "exposed_prefetch": prof["wait_ms"] / K,
                                  "prefetch_kernels": prof["prefetch_ms"] / K},
        "h2d_bytes_per_step": prof["prefetch_bytes"] / K,
        "gpu_launches": prof["launches"] + stack.launches,
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    cache.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--host-layers", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="seq", choices=["seq", "heads"],
                    help="multi-GPU partition: by sequence (no collective; default) or by KV head "
                         "(layer-scope top-k: per-layer NCCL all-reduce of the aggregate on the copy stream)")
    ap.add_argument("--full-decoder", action="store_true",
                    help="time the whole model step around the hot path (SURVEY 8(f) row 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    if args.full_decoder:
        return run_full_decoder(args, cfg)
    return run_gpu_arm(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
