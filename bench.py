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

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c1]
  python bench.py --impl reference ...     # CPU reference arm (oracle port)

Multi-GPU: one rank per GPU over NCCL.  Under torchrun the ranks come from the
environment; `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks.  The config's GLOBAL batch is partitioned
(shard.plan_partition, the north star's rule): by KV head first, by sequence
where the heads run out (strong scaling, `--shard auto`, the default).  The
ranks that share a batch slice sum each layer's partial top-k aggregate with
an NCCL all-reduce on the cache's copy stream (engine.py:317 couples all
heads of a sequence); nothing else crosses ranks.  `--shard replicas` runs the
whole config on every rank (weak scaling, no collective).  `--share N` runs
rank 0's share of an N-way partition alone on one GPU (e.g. C4's 8-GPU rank).
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
    # BASELINE.json configs[3]: global batch 32, 8 GPUs (`--gpus 8`: one KV head per
    # rank); `--share 8` runs one rank's share (1 KV head x 32 sequences) on one GPU
    "c4": dict(workload="C4: LLaMA-3-8B-shaped GQA (8 KV heads) 32-layer decode, ctx 128k, global batch 32, "
                        "1-bit KV (g32, r64), top-k 256, full bf16 cache in pinned host",
               layers=32, batch=32, kv_heads=8, q_heads=32, head_dim=128, ctx=131072, bits=1,
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
    # launcher tests only (not a BASELINE config): C3's shape at 4k context, 2 layers
    "tiny": dict(workload="tiny: C3-shaped GQA (8 KV heads), 2 layers, ctx 4096, batch 8, 1-bit KV, top-k 128 "
                          "(launcher test config)",
                 layers=2, batch=8, kv_heads=8, q_heads=32, head_dim=128, ctx=4096, bits=1,
                 group=32, residual=64, topk=128),
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


def measure_h2d_peak(device, nbytes: int = 256 << 20) -> dict:
    """Host-link roofline for K5 (spc_h2d_peak): best of 5 pinned-host -> device
    transfers of one 256 MiB buffer, by DMA (cudaMemcpyAsync) and by a
    zero-copy read kernel (K5's own mechanism); the peak is the better of the
    two.  Measured outside any timed region."""
    import ctypes

    import torch

    from paper_2503_16163_b200 import _lib
    dma, zc = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.lib().spc_h2d_peak(torch.device(device).index or 0, nbytes, ctypes.byref(dma),
                                       ctypes.byref(zc)))
    return {"dma_gbs": dma.value, "zero_copy_gbs": zc.value, "peak_gbs": max(dma.value, zc.value)}


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
def cpu_info() -> dict:
    """Host CPU model, visible cores and numpy's BLAS thread pool."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": i.get("internal_api"), "threads": i.get("num_threads")} for i in threadpool_info()]
    except Exception:
        pass
    return {"model": model, "cpus": os.cpu_count(), "blas": blas}


class CpuSample:
    """The CPU reference path (oracle port of engine.py:299-321: dequantize every
    packed group, attend both rows, aggregate, select_topk) on a bounded sample
    of `units` (layer, seq) decode units of `cfg`, prepared once (prefill
    quantization is not part of the decode step) and timed `threads` at a time.

    One sample = one pass over the units; a full decode step is
    layers x batch units for `batch` tokens, so the sample's tokens/s
    equivalent is units / layers / wall."""

    def __init__(self, cfg: dict, units: int, seed: int = 0):
        import numpy as np
        from concurrent.futures import ThreadPoolExecutor

        from oracle import restate as R
        from oracle.synth import make_kv, make_queries, make_step_kv
        self.cfg, self.units = cfg, units
        H, Hq, d, n = cfg["kv_heads"], cfg["q_heads"], cfg["head_dim"], cfg["ctx"]

        def prep(i):
            rng = np.random.default_rng(seed + i)
            st = R.LayerState(H, d, cfg["bits"], cfg["group"], cfg["residual"], cfg["topk"])
            K, V = make_kv(rng, n, H, d)
            st.extend(K, V)
            st._sync_packed()
            q = make_queries(rng, 2, Hq, d)
            kn, vn = make_step_kv(rng, 2, H, d)
            return st, q, kn, vn

        with ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1))) as ex:
            self.work = list(ex.map(prep, range(units)))

    def _run(self, w):
        from oracle import restate as R
        st, q, kn, vn = w
        t0 = time.perf_counter()
        R.decode_layer(st, q, kn, vn, append=False)
        return time.perf_counter() - t0

    def time(self, threads: int) -> dict:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            t0 = time.perf_counter()
            per_unit = list(ex.map(self._run, self.work))
            wall = time.perf_counter() - t0
        return {"wall_s": wall, "median_unit_s": sorted(per_unit)[len(per_unit) // 2],
                "tokens_per_s": self.units / self.cfg["layers"] / wall}

    def single_core(self) -> dict:
        """One unit on one thread with the BLAS pool limited to 1."""
        try:
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                s = self._run(self.work[0])
        except ImportError:
            s = self._run(self.work[0])
        return {"unit_s": s, "tokens_per_s": 1.0 / self.cfg["layers"] / s}


def cpu_reference_sample(cfg: dict, threads: int, units: int, seed: int = 0, single: bool = True) -> dict:
    """cpu_baseline for the GPU arm: one timed sample (see CpuSample)."""
    smp = CpuSample(cfg, units, seed)
    r = smp.time(threads)
    one = smp.single_core() if single else None
    full = cfg["layers"] * cfg["batch"]
    return {"value": r["tokens_per_s"], "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"{units} of {full} (layer, seq) decode units of {cfg['workload'][:2]} (n={cfg['ctx']}), "
                      f"{threads} threads, wall {r['wall_s']:.2f}s, median unit {r['median_unit_s']:.2f}s; "
                      f"tokens/s = units / layers / wall",
            "single_core": one, "cpu": cpu_info(),
            "note": "oracle/restate.py: vectorised numpy restatement of the reference's per-layer decode "
                    "(the reference itself is pure Python and does not travel to the GPU box; its own "
                    "timing in the build container is profiles/r2_reference_c1_timing.json)"}


def workload_config(cfg: dict, world: int, args, part=None) -> dict:
    """The `config` object both arms print (same workload, same keys)."""
    d, B, g = cfg["head_dim"], cfg["bits"], cfg["group"]
    kv_gb = cfg["layers"] * cfg["batch"] * cfg["kv_heads"] * cfg["ctx"] * d * (B / 4 + 8 / g) / 1e9
    if args.shard == "replicas":
        par = f"replicas x{world}: the whole config on every rank (no collective)"
        gb = cfg["batch"] * world
    else:
        if part is None:
            from paper_2503_16163_b200.shard import plan_partition
            part = plan_partition(cfg["kv_heads"], cfg["q_heads"], cfg["batch"], 0, max(world, args.share or 1),
                                  args.shard)
        par = part.describe()
        if part.head_groups > 1:
            par += "; per-layer NCCL all-reduce of the top-k aggregate over each batch slice's ranks"
        if args.share and world == 1 and args.share > 1:
            par = f"rank 0 of {args.share} alone on 1 GPU: " + par
        gb = cfg["batch"]
    return {"workload": cfg["workload"], "global_batch": gb, "seq_len": cfg["ctx"], "layers": cfg["layers"],
            "bits": cfg["bits"], "group": g, "residual": cfg["residual"], "topk": cfg["topk"],
            "kv_heads": cfg["kv_heads"], "q_heads": cfg["q_heads"], "head_dim": d, "parallelism": par,
            "l2": "no flush: per-step low-bit KV %.1f GB >> 126 MB L2" % kv_gb}


def run_reference_arm(args, cfg):
    """`--impl reference`: the CPU reference path (oracle port) on this box's
    host cores, rank 0 only.  Each step is one bounded sample (CpuSample) of
    the workload; ms_per_step is that sample's real wall time and value its
    tokens/s equivalent, so `steps x ms_per_step` is the time actually spent."""
    rank, world, _, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    units = max(1, min(threads, 16))
    smp = CpuSample(cfg, units)
    vals = []
    for i in range(args.warmup + args.steps):
        r = smp.time(threads)
        if i >= args.warmup:
            vals.append(r)
    one = smp.single_core()
    wall = sum(v["wall_s"] for v in vals)
    value = units * len(vals) / cfg["layers"] / wall
    full = cfg["layers"] * cfg["batch"]
    base = {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"each step: {units} of {full} (layer, seq) decode units of {cfg['workload'][:2]} "
                      f"(n={cfg['ctx']}) on {threads} threads; tokens/s = units / layers / wall",
            "units_per_step": units, "full_step_units": full, "timed_wall_s": wall,
            "single_core": one, "cpu": cpu_info()}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * wall / len(vals), "higher_is_better": True,
            "scaling": "weak" if args.shard == "replicas" else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded)", "config": workload_config(cfg, args.gpus, args),
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


TIE_BAND = 1e-4   # documented near-tie band of the top-k parity contract


def topk_band_population(dec, layer: int, cfg: dict) -> dict:
    """Live, after the timed region: for `layer`'s last ticket, the positions
    outside the picked set whose aggregate lies within TIE_BAND of the k-th
    picked value (the only places a top-k set may differ from the reference's),
    summed over sequences and units."""
    import torch
    agg = dec.debug_agg(layer)
    picked, _ = dec.ticket(layer)
    f = dec.cache.quantized_frontier(layer)
    agg = agg[..., :f]
    sel = picked.long()
    valid = sel >= 0
    vals = torch.gather(agg, -1, sel.clamp(min=0))
    kth = torch.where(valid, vals, torch.full_like(vals, float("inf"))).min(-1).values
    # outside the picked set: invalid (-1) picks point at a padding column f
    mask = torch.ones(agg.shape[:-1] + (f + 1,), dtype=torch.bool, device=agg.device)
    mask.scatter_(-1, torch.where(valid, sel, torch.full_like(sel, f)), False)
    near = ((agg >= kth[..., None] * (1 - TIE_BAND)) & mask[..., :f]).sum().item()
    return {"band_positions_outside_set": int(near), "units": int(agg.shape[0] * agg.shape[1]),
            "layer": layer}


def parity_record(config: str) -> dict:
    """The oracle parity run at this config's geometry (tests/test_bench_geometry_gpu.py),
    as committed under profiles/: top-k band swaps and worst per-head error."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_parity_bench_geometry.json")) as fh:
            d = json.load(fh)
    except (OSError, ValueError):
        return {}
    rec = d.get({"c4": "c4_share8"}.get(config, config))
    if not rec:
        return {}
    return {"oracle_check": "tests/test_bench_geometry_gpu.py (profiles/r2_parity_bench_geometry.json)",
            "oracle_band_swaps": rec.get("topk_band_swaps"),
            "oracle_worst_head_rel_err_fp32": rec.get("worst_head_rel_err_fp32")}


def agg_reducer(cache, layers, device, group=None):
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
            dist.all_reduce(v, group=group)
        _lib.check(lib.spc_finish_layer(h, layer))

    return reduce


def run_gpu_arm(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2503_16163_b200 import CacheBudget, DeviceTwoTierCache, SpeculativeLayerDecoder
    from paper_2503_16163_b200 import _lib

    rank, world, local, local_world = dist_env()
    device, group, part, lcfg, reduce_agg = setup_ranks(args, cfg)
    if args.graph and reduce_agg:
        raise SystemExit("--graph does not combine with the cross-rank aggregate reduction (--shard heads)")

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        cpu_base = cpu_reference_sample(cfg, threads, max(1, min(threads, 16)))
    gcfg, cfg = cfg, lcfg   # gcfg: the global workload; cfg: this rank's share
    if args.compute_priority:
        # the decode loop's stream above the library's selection streams (lowest priority)
        torch.cuda.set_stream(torch.cuda.Stream(device, priority=args.compute_priority))

    W, K = args.warmup, args.steps
    if args.graph and not args.compute_priority:
        torch.cuda.set_stream(torch.cuda.Stream(device))  # the legacy default stream cannot be captured
    # device-timed pass + end-to-end pass (+ the eager profiled pass of --graph)
    total_steps = (3 if args.graph else 2) * (W + K)
    host_layers = args.host_layers or plan_host_layers(cfg, local_world)
    budget = CacheBudget(bits=cfg["bits"], group_size=cfg["group"], residual=cfg["residual"],
                         prefetch_k=cfg["topk"], context_length=cfg["ctx"] + total_steps + 64)
    t_setup = time.perf_counter()
    cache = DeviceTwoTierCache(cfg["layers"], cfg["kv_heads"], cfg["head_dim"], budget,
                               batch=cfg["batch"], q_heads=cfg["q_heads"], device=torch.device(device).index,
                               host_layers=host_layers)
    if args.pf_inflight:
        cache.set_prefetch_inflight(args.pf_inflight)
    if args.agg_mode != "spill":
        cache.set_agg_mode(args.agg_mode)
    reduce_layer = None
    if reduce_agg:
        from paper_2503_16163_b200.shard import allreduce_sum
        dec = SpeculativeLayerDecoder(cache, agg_reduce=allreduce_sum(group))
        reduce_layer = agg_reducer(cache, cfg["layers"], device, group)
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

    def step_device(t, qt, kt, vt, graph=False):
        if graph:
            _lib.check(lib.spc_graph_begin(h, stream))
        for layer in range(L):
            _lib.check(lib.spc_decode_layer(h, layer, t, qt[layer].data_ptr(), kt[layer].data_ptr(),
                                            vt[layer].data_ptr(), out[layer].data_ptr(),
                                            pm[layer].data_ptr(), stream))
            if reduce_layer:
                reduce_layer(layer)
        if graph:
            _lib.check(lib.spc_graph_launch(h, stream))

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
    if args.graph:
        # K2 / prefetch event timings need the eager path (profiling events
        # cannot sit inside a step graph): one profiled eager pass first
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        for _ in range(K):
            step_device(t, q[t], k_new[t], v_new[t])
            t += 1
        eb.record()
        torch.cuda.synchronize(device)
        prof_eager = profile(0)
        eager_ms = ea.elapsed_time(eb)
        for _ in range(W):
            step_device(t, q[t], k_new[t], v_new[t], graph=True)
            t += 1
        torch.cuda.synchronize(device)
    with ClockSampler(torch.device(device).index) as clocks:
        ev0.record()
        for _ in range(K):
            step_device(t, q[t], k_new[t], v_new[t], graph=args.graph)
            t += 1
        ev1.record()
        torch.cuda.synchronize(device)
    elapsed_ms = ev0.elapsed_time(ev1)
    attn_ms, attn_n, sel_ms, sel_n, launches = prof_eager if args.graph else profile(0)
    prof_ms = eager_ms if args.graph else elapsed_ms  # the pass the event timings come from
    wait_ms = lib.spc_profile_wait_ms(h)
    pf_ms = lib.spc_profile_prefetch_ms(h)
    pf_wall_ms = lib.spc_profile_prefetch_wall_ms(h)
    pf_bytes = int(lib.spc_profile_prefetch_bytes(h))
    _, newc = dec.ticket(L // 2)
    band = topk_band_population(dec, 0, cfg)
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
    # two buffer sets: step i+1's inputs copy in while step i decodes, and step
    # i's results copy out while step i+1 decodes (each set is reused two steps later)
    o_h = [torch.empty_like(out, device="cpu").pin_memory() for _ in range(2)]
    pm_h = [torch.empty_like(pm, device="cpu").pin_memory() for _ in range(2)]
    q_d = [torch.empty_like(q[0]) for _ in range(2)]
    k_d = [torch.empty_like(k_new[0]) for _ in range(2)]
    v_d = [torch.empty_like(v_new[0]) for _ in range(2)]
    o_d = [out, torch.empty_like(out)]
    pm_d = [pm, torch.empty_like(pm)]

    # layer-pipelined: layer group g+1's inputs copy H2D on one copy stream while
    # group g decodes, and group g's outputs copy D2H on another
    comp = torch.cuda.current_stream(device)
    cs_in, cs_out = torch.cuda.Stream(device), torch.cuda.Stream(device)
    done_in = [None, None]   # compute finished reading input set s (event)
    done_out = [None, None]  # output set s copied to the host (event)

    GRP = 8  # layers per copy group: one H2D and one D2H per group keeps the host-side cost low

    def step_e2e(i, tt):
        sb = i & 1
        qh, kh, vh = e2e_in[i]
        groups = [(g0, min(L, g0 + GRP)) for g0 in range(0, L, GRP)]
        ev_in = [torch.cuda.Event() for _ in groups]
        if done_in[sb] is not None:
            cs_in.wait_event(done_in[sb])  # step i-2 is done with this input set
        with torch.cuda.stream(cs_in):
            for gi, (g0, g1) in enumerate(groups):
                q_d[sb][g0:g1].copy_(qh[g0:g1], non_blocking=True)
                k_d[sb][g0:g1].copy_(kh[g0:g1], non_blocking=True)
                v_d[sb][g0:g1].copy_(vh[g0:g1], non_blocking=True)
                ev_in[gi].record(cs_in)
        if done_out[sb] is not None:
            comp.wait_event(done_out[sb])  # step i-2's results are on the host
        for gi, (g0, g1) in enumerate(groups):
            comp.wait_event(ev_in[gi])
            for layer in range(g0, g1):
                _lib.check(lib.spc_decode_layer(h, layer, tt, q_d[sb][layer].data_ptr(), k_d[sb][layer].data_ptr(),
                                                v_d[sb][layer].data_ptr(), o_d[sb][layer].data_ptr(),
                                                pm_d[sb][layer].data_ptr(), stream))
                if reduce_layer:
                    reduce_layer(layer)
            ev = torch.cuda.Event()
            ev.record(comp)
            cs_out.wait_event(ev)
            with torch.cuda.stream(cs_out):
                o_h[sb][g0:g1].copy_(o_d[sb][g0:g1], non_blocking=True)
                pm_h[sb][g0:g1].copy_(pm_d[sb][g0:g1], non_blocking=True)
        done_in[sb] = torch.cuda.Event()
        done_in[sb].record(comp)
        done_out[sb] = torch.cuda.Event()
        done_out[sb].record(cs_out)

    if args.graph:
        # one packed transfer each way per step: q|k|v in, out|pinned_mass out
        def packed(shapes_dtypes, dev):
            sizes = [int(np.prod(sh)) * torch.empty((), dtype=dt).element_size() for sh, dt in shapes_dtypes]
            buf = torch.empty(sum(sizes), dtype=torch.uint8, device=dev)
            views, o = [], 0
            for (sh, dt), n in zip(shapes_dtypes, sizes):
                views.append(buf[o:o + n].view(dt).view(sh))
                o += n
            return buf, views
        in_spec = [(tuple(q[0].shape), torch.bfloat16), (tuple(k_new[0].shape), torch.bfloat16),
                   (tuple(v_new[0].shape), torch.bfloat16)]
        in_dev, (qg, kg, vg) = packed(in_spec, device)
        out_dev, (og, pmg) = packed([(tuple(out.shape), torch.bfloat16), (tuple(pm.shape), torch.float32)], device)
        out_host = torch.empty(out_dev.numel(), dtype=torch.uint8).pin_memory()
        g_in = []
        for i in range(len(e2e_in)):
            hb, (hq, hk, hv) = packed(in_spec, "cpu")
            hq.copy_(e2e_in[i][0]), hk.copy_(e2e_in[i][1]), hv.copy_(e2e_in[i][2])
            g_in.append(hb.pin_memory())

    def step_e2e_graph(i, tt):
        # one graph per step: H2D of the step's inputs, the layers, D2H of the results
        _lib.check(lib.spc_graph_begin(h, stream))
        _lib.check(lib.spc_copy_async(in_dev.data_ptr(), g_in[i].data_ptr(), in_dev.numel(), stream))
        for layer in range(L):
            _lib.check(lib.spc_decode_layer(h, layer, tt, qg[layer].data_ptr(), kg[layer].data_ptr(),
                                            vg[layer].data_ptr(), og[layer].data_ptr(), pmg[layer].data_ptr(),
                                            stream))
        _lib.check(lib.spc_copy_async(out_host.data_ptr(), out_dev.data_ptr(), out_dev.numel(), stream))
        _lib.check(lib.spc_graph_launch(h, stream))

    run_e2e = step_e2e_graph if args.graph else step_e2e
    for i in range(W):
        run_e2e(i, t)
        t += 1
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    w0 = time.perf_counter()
    for i in range(W, W + K):
        run_e2e(i, t)
        t += 1
    torch.cuda.synchronize(device)
    e2e_s = time.perf_counter() - w0
    e2e_s = reduce_max(e2e_s, device)
    h2d = (q_d[0].numel() + k_d[0].numel() + v_d[0].numel()) * 2
    d2h = o_h[0].numel() * 2 + pm_h[0].numel() * 4

    ms_per_step = elapsed_ms / K
    # strong partition: the ranks together decode the global batch per step;
    # replicas: every rank its own copy of the config (weak scaling)
    tokens = whole_job_tokens(gcfg["batch"], K, world) if args.shard == "replicas" else gcfg["batch"] * K
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
        "scaling": "weak" if args.shard == "replicas" else "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded; peaky: %d needle keys per "
        "(seq, kv head), q drift sigma %.1f)" % (NEEDLES, DRIFT),
        "config": workload_config(gcfg, world, args, part),
        "rank_share": {"kv_heads": cfg["kv_heads"], "q_heads": cfg["q_heads"], "batch": cfg["batch"],
                       "host_layers": host_layers, "attention_impl": "fast" if cache.fast_path else "generic",
                       "prefetch_inflight_bytes": args.pf_inflight or None, "agg_mode": args.agg_mode,
                       "host_slabs_note": "layers l, l' with l = l' mod host_layers share one pinned slow-tier "
                                          "slab and are fed identical KV (host RAM); PCIe bytes unchanged"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "K2 attend (per layer launch, all sequences)",
                     "algorithmic_bytes_per_launch": ab["hbm"], "avg_launch_ms": attn_avg_ms,
                     "launches": attn_n, "kernel_share_of_step": attn_ms / max(1e-9, prof_ms)},
        "prefetch": {"new_pin_fraction": h2d_pf / max(1, cfg["topk"] * cfg["batch"] * cfg["layers"] * cache.row_bytes(1)),
                     "h2d_bytes_per_step": h2d_pf,
                     "exposed_ms_per_step": wait_ms / K, "exposed_fraction": wait_ms / max(1e-9, prof_ms),
                     "copy_stream_ms_per_step": sel_ms / K, "prefetch_kernel_ms_per_step": pf_ms / K,
                     "prefetch_wall_ms_per_step": pf_wall_ms / K,
                     "h2d_gbs": (h2d_pf / 1e9) / max(1e-9, pf_wall_ms / K / 1e3),
                     "h2d_peak_gbs": h2d_peak["peak_gbs"], "h2d_peak_dma_gbs": h2d_peak["dma_gbs"],
                     "h2d_peak_zero_copy_gbs": h2d_peak["zero_copy_gbs"],
                     "h2d_frac": (h2d_pf / 1e9) / max(1e-9, pf_wall_ms / K / 1e3) / max(1e-9, h2d_peak["peak_gbs"]),
                     "h2d_how": "bytes = new pins x row bytes; time = union of the K5 kernel intervals on the two "
                                "copy streams (CUDA events); peak = best of 5 transfers of 256 MiB from pinned host "
                                "memory, DMA and zero-copy kernel, same process"},
        "e2e": {"value": tokens / e2e_s,
                "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "how": ("one step graph per step (spc_graph_begin / spc_graph_launch) holding the H2D of the "
                        "step's q/k/v from pinned host memory (spc_copy_async), every layer's spc_decode_layer and "
                        "the D2H of its outputs; wall clock around synchronize, max over ranks") if args.graph else
                       ("through spc_decode_layer (C ABI) with pinned host inputs/outputs; per group of 8 "
                        "layers, H2D of its q/k/v and D2H of its outputs on two copy streams overlapping the "
                        "other groups' decode, two buffer sets so consecutive steps' copies overlap too; "
                        "wall clock around synchronize, max over ranks")},
        "gpu_launches": launches,
        **({"graph": {"step_graphs": True, "instantiations_updates": dec.graph_stats(),
                      "eager_ms_per_step": eager_ms / K,
                      "timings_from": "roofline, prefetch and gpu_launches from an eager profiled pass of the "
                                      "same K steps (profiling events cannot sit inside a step graph)"}}
           if args.graph else {}),
        "clocks": clocks.summary(),
        "topk_parity": {"band": TIE_BAND, **band, **parity_record(args.config)},
        "setup_s": setup_s,
        "cpu_baseline": cpu_base,
    }
    if rank == 0:
        if getattr(args, "ctx128k", None) is not None:
            line["ctx_128k"] = args.ctx128k
        print(json.dumps(line), flush=True)
    cache.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def run_ctx128k_companion(args) -> dict:
    """The metric's 128k half in the default (driver-run) line: the same bench
    at C3 (BASELINE configs[2] on one GPU: GQA 8 KV heads, 128k, batch 8,
    1-bit, k128) in a child process, run BEFORE the headline config so each
    process owns the GPU and the pinned host memory alone.  Returns a compact
    summary of the child's JSON line (or the reason it is missing)."""
    cmd = [sys.executable, os.path.abspath(__file__), "--config", "c3", "--steps", str(args.steps),
           "--warmup", str(args.warmup), "--no-cpu-baseline", "--no-ctx128k"]
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        lines = [x for x in res.stdout.splitlines() if x.startswith("{")]
        if res.returncode != 0 or not lines:
            return {"unavailable": "C3 child exited %d: %s" % (res.returncode, res.stderr.strip()[-300:])}
        d = json.loads(lines[-1])
    except (subprocess.TimeoutExpired, ValueError, OSError) as e:
        return {"unavailable": "C3 child failed: %r" % (e,)}
    rf, pf = d.get("roofline", {}), d.get("prefetch", {})
    return {"workload": d["config"]["workload"], "value": d["value"], "unit": d["unit"],
            "ms_per_step": d["ms_per_step"], "steps": d["steps"], "warmup": d["warmup"],
            "e2e": d.get("e2e", {}).get("value"),
            "roofline": {k: rf.get(k) for k in ("achieved", "peak", "frac", "traffic", "avg_launch_ms",
                                                  "kernel_share_of_step")},
            "prefetch": {k: pf.get(k) for k in ("exposed_fraction", "h2d_gbs", "h2d_frac")},
            "gpu_launches": d.get("gpu_launches"), "clocks": d.get("clocks"),
            "topk_parity": d.get("topk_parity"),
            "how": "bench.py --config c3 in a child process before the headline run, same steps/warmup"}


def setup_ranks(args, cfg):
    """Device, process group and this rank's share of the partition.

    Returns (device, agg_group, partition, rank_cfg, reduce_agg).  NCCL by
    default (SPC_BENCH_BACKEND=gloo for two ranks sharing one GPU in tests);
    rank r uses GPU LOCAL_RANK mod the visible device count."""
    import torch
    import torch.distributed as dist

    from paper_2503_16163_b200.shard import plan_partition
    rank, world, local, _ = dist_env()
    ndev = max(1, torch.cuda.device_count())
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    device = f"cuda:{dev_index}"
    part, lcfg, group, reduce_agg = None, dict(cfg), None, False
    if args.shard != "replicas":
        share = args.share if (world == 1 and args.share) else world
        part = plan_partition(cfg["kv_heads"], cfg["q_heads"], cfg["batch"], rank if world > 1 else 0, share,
                              args.shard)
        lcfg = dict(cfg, kv_heads=part.heads.kv_heads, q_heads=part.heads.q_heads, batch=part.batch)
        # the agg all-reduce: across the head groups of a batch slice; `--shard heads`
        # at N=1 exercises it as a 1-rank group
        reduce_agg = (world > 1 and part.head_groups > 1) or (world == 1 and args.shard == "heads" and share == 1)
    if world > 1 or reduce_agg:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        backend = os.environ.get("SPC_BENCH_BACKEND", "nccl")
        kw = {"device_id": torch.device(device)} if backend == "nccl" else {}
        dist.init_process_group(backend, rank=rank, world_size=world, **kw)
        if reduce_agg and part is not None and part.batch_groups > 1:
            for ranks in part.all_agg_groups():   # every rank creates every group, in order
                g = dist.new_group(ranks)
                if rank in ranks:
                    group = g
    return device, group, part, lcfg, reduce_agg


def relaunch_under_torchrun(argv, nproc: int) -> int:
    """`--gpus N` outside torchrun: re-run this script with N ranks
    (torch.distributed.run, 127.0.0.1 rendezvous); rank 0's JSON line passes
    through on stdout."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)
    print(f"[bench] relaunching under torchrun: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


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
    heads = args.shard == "heads" or (args.shard == "auto" and world > 1)
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


def run_dry(args, cfg):
    """The launcher and partition logic on CPU (gloo): every rank reports its
    share; rank 0 prints one JSON line with the partition."""
    import torch.distributed as dist

    from paper_2503_16163_b200.shard import plan_partition
    rank, world, _, _ = dist_env()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    part = plan_partition(cfg["kv_heads"], cfg["q_heads"], cfg["batch"], rank, world,
                          "seq" if args.shard == "replicas" else args.shard)
    mine = {"rank": rank, "kv": [part.heads.kv_lo, part.heads.kv_hi], "q": [part.heads.q_lo, part.heads.q_hi],
            "seqs": [part.seq_lo, part.seq_hi], "agg_group": part.agg_group}
    shares = [None] * world
    if world > 1:
        dist.all_gather_object(shares, mine)
        dist.destroy_process_group()
    else:
        shares = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "config": workload_config(cfg, world, args, part),
                          "ranks": shares}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--host-layers", type=int, default=0)
    ap.add_argument("--agg-mode", default="spill", choices=["spill", "recompute"],
                    help="top-k aggregate: spill the speculative logits (default) or recompute them (K3r)")
    ap.add_argument("--compute-priority", type=int, default=0,
                    help="CUDA stream priority of the decode loop (negative = higher; 0 = default stream priority)")
    ap.add_argument("--pf-inflight", type=int, default=0,
                    help="PCIe gather bytes in flight (spc_set_prefetch_inflight; 0 = library default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ctx128k", action="store_true",
                    help="skip the C3 (128k) companion measurement of the default single-GPU run")
    ap.add_argument("--graph", action="store_true",
                    help="issue each step as one CUDA graph (spc_graph_begin/launch), the e2e pass with its "
                         "host copies inside; K2/prefetch timings then come from an eager profiled pass")
    ap.add_argument("--shard", default="auto", choices=["auto", "heads", "seq", "replicas"],
                    help="multi-GPU partition of the global batch: auto = by KV head, then by sequence "
                         "where heads run out (default, the north star's rule); heads; seq; or replicas "
                         "(whole config on every rank, weak scaling)")
    ap.add_argument("--share", type=int, default=0,
                    help="run rank 0's share of an N-way partition alone on one GPU")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without a GPU: init the process group (gloo), print the partition")
    ap.add_argument("--full-decoder", action="store_true",
                    help="time the whole model step around the hot path (SURVEY 8(f) row 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        return relaunch_under_torchrun(sys.argv[1:], args.gpus)
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    if args.dry_run:
        return run_dry(args, cfg)
    if args.full_decoder:
        return run_full_decoder(args, cfg)
    args.ctx128k = None
    if (args.config == "c2" and not args.no_ctx128k and "WORLD_SIZE" not in os.environ and args.gpus == 1
            and not args.share and not args.graph):
        args.ctx128k = run_ctx128k_companion(args)
    return run_gpu_arm(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
