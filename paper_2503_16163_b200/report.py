"""`run_decode` report on the device.

Same arguments and the same report as the reference's experiment harness
(src/speckv/experiments.py:46-97): {experiment, config, rows, summary} with
the same snake_case keys in the same order and the same 9-digit rounding, so
`json.dumps(report, indent=2)` is byte-stable across identical invocations
and diffable against a reference report.  The token loop is
DeviceSpeculativeDecoder (adapter.py) over the B200 cache.

clock="logical" (default) keeps the reference's transfer model
(transfer.py:58-112, the ChannelModel arguments); clock="measured" puts
CUDA-event timings of every step into compute_s / transfer_s / overlapped_s /
serialized_s (adapter.py docstring) and adds config["clock"] = "measured".
"""
from __future__ import annotations

import numpy as np

from .budget import CacheBudget, memory_ratio
from .transfer import ChannelModel
from .weights import load_weights, with_runtime

__all__ = ["run_decode", "make_prompt", "decode_report"]


def make_prompt(vocab: int, length: int, seed: int) -> list[int]:
    """experiments.py:37-40: default_rng(seed).integers(0, vocab, length)."""
    return [int(t) for t in np.random.default_rng(seed).integers(0, vocab, size=length)]


def _round(x: float, digits: int = 9) -> float:
    return float(round(float(x), digits))


def decode_report(result, config: dict, bits: int, group_size: int, residual: int, k: int,
                  max_len: int) -> dict:
    """Assemble the report from a GenerateResult (experiments.py:67-97)."""
    by_step = {row["step"]: row for row in result.latency_rows}
    rows = []
    for m in result.metrics:
        lat = by_step[m.step]
        rows.append({
            "step": m.step, "token": m.token, "speculative_hit": m.speculative_hit,
            "pinned_mass": _round(m.pinned_mass), "bytes_fetched": m.bytes_fetched,
            "new_pins": m.new_pins, "compute_s": _round(lat["compute_s"]),
            "transfer_s": _round(lat["transfer_s"]), "overlapped_s": _round(lat["overlapped_s"]),
            "serialized_s": _round(lat["serialized_s"]),
        })
    n = len(result.metrics)
    summary = {
        "tokens": result.tokens,
        "speculative_hit_rate": _round(sum(1 for m in result.metrics if m.speculative_hit) / n),
        "mean_pinned_mass": _round(float(np.mean([m.pinned_mass for m in result.metrics]))),
        "bytes_fetched_total": int(sum(m.bytes_fetched for m in result.metrics)),
        "overlapped_total_s": _round(sum(r["overlapped_s"] for r in result.latency_rows)),
        "serialized_total_s": _round(sum(r["serialized_s"] for r in result.latency_rows)),
        "memory_ratio": memory_ratio(bits, group_size, max_len, residual + k),
    }
    return {"experiment": "decode", "config": config, "rows": rows, "summary": summary}


def run_decode(weights_path: str, prompt: list[int] | None, prompt_len: int, steps: int, bits: int,
               group_size: int, k: int, residual: int, bandwidth: float, alpha: float,
               overhead: float, compute_s: float, mode: str, seed: int, max_len: int = 4096,
               clock: str = "logical", device: int = 0) -> dict:
    """experiments.py:46-97 with the decode on the B200."""
    from .adapter import generate
    cfg, weights = load_weights(weights_path)
    cfg = with_runtime(cfg, max_len=max_len)
    if prompt is None:
        prompt = make_prompt(cfg.vocab, prompt_len, seed)
    budget = CacheBudget(bits=bits, group_size=group_size, residual=residual, prefetch_k=k,
                         context_length=max_len)
    channel = ChannelModel(bandwidth=bandwidth, scatter_penalty=alpha, fixed_overhead=overhead)
    result = generate(cfg, weights, prompt, steps, budget, channel, mode=mode,
                      compute_time_per_step=compute_s, device=device, clock=clock)
    config = {"weights_path": weights_path, "prompt_len": len(prompt), "steps": steps, "bits": bits,
              "group_size": group_size, "k": k, "residual": residual, "bandwidth": bandwidth,
              "alpha": alpha, "overhead": overhead, "compute_s": compute_s, "mode": mode, "seed": seed}
    if clock != "logical":
        config["clock"] = clock
    return decode_report(result, config, bits, group_size, residual, k, max_len)
