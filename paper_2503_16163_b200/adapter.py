"""DeviceSpeculativeDecoder -- drop-in for the reference's token loop
(SpeculativeDecoder / generate, engine.py:186-386) with the SpeCache hot path
on the B200 (DeviceTwoTierCache + SpeculativeLayerDecoder).

This is the SURVEY.md 8(f) "next" row 2: it closes the loop from prompt to
tokens so the object-level API of the reference can be driven on the device.
The toy model around the hot path (RMSNorm, projections, RoPE, SiLU FFN,
logits; engine.py:35-72, numerics.py:42-78) runs as plain fp32 PyTorch on the
same GPU -- it is plumbing around the path, not part of it.  The hot-path
boundary is bf16: q/k/v enter the cache and the attention as bf16, attention
outputs leave as bf16 (the C ABI contract).

Same constructor arguments, phase rules (ProtocolError), StepMetrics and
GenerateResult fields as the reference.  The latency rows use the reference's
logical-clock model (transfer.py:58-112) by default; clock="measured"
replaces it with CUDA-event timings of each step on the device (SURVEY 8(f)
row 3): overlapped_s = the step's device time on the compute stream (exposed
prefetch waits included), transfer_s = the step's PCIe gather kernels,
compute_s = overlapped_s minus the exposed waits, serialized_s = compute_s +
transfer_s.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .budget import CacheBudget
from .cache import DeviceTwoTierCache
from .decode import SpeculativeLayerDecoder, StepMetrics
from .toymodel import ToyModel
from .transfer import ChannelModel, ProtocolError, step_latency, transfer_time

__all__ = ["DeviceSpeculativeDecoder", "GenerateResult", "generate"]


@dataclass
class GenerateResult:
    """engine.py:175-183."""
    tokens: list
    logits: list
    metrics: list
    latency_rows: list
    prefill_seconds: float
    total_seconds: float
    decoder: "DeviceSpeculativeDecoder" = None


class DeviceSpeculativeDecoder(ToyModel):
    """engine.py:186-339 on the device cache.  `config` / `weights` are the
    reference's DecoderConfig / Weights (or any objects with the same fields)."""

    def __init__(self, config, weights, budget: CacheBudget, channel_model: ChannelModel | None = None,
                 mode: str = "sim", compute_time_per_step: float = 0.0, prefill_time: float = 0.0,
                 device: int = 0, clock: str = "logical", capacity: int | None = None):
        import dataclasses

        import torch
        if mode not in ("sim", "thread"):
            raise ValueError("mode must be 'sim' or 'thread'")
        if clock not in ("logical", "measured"):
            raise ValueError("clock must be 'logical' or 'measured'")
        self.clock_mode = clock
        self._measured: dict[int, dict] = {}
        self._ev = None
        ToyModel.__init__(self, config, weights, device)
        self.budget = budget
        # The reference decodes past context_length and max_len (context_length
        # only feeds memory_ratio, kvcache.py:55-63; decode_step has no length
        # check, engine.py:286-339).  The device cache is sized by `capacity`
        # (default: max(context_length, max_len) + 1024 positions); self.budget
        # keeps the caller's budget.
        cap = capacity if capacity is not None else max(budget.context_length, config.max_len) + 1024
        dev_budget = dataclasses.replace(budget, context_length=max(cap, budget.context_length))
        self.cache = DeviceTwoTierCache(config.layers, config.kv_heads, config.head_dim, dev_budget,
                                        q_heads=config.q_heads, device=device)
        self.layer_dec = SpeculativeLayerDecoder(self.cache)
        self.channel_model = channel_model or ChannelModel()
        self.compute_time_per_step = compute_time_per_step
        self.prefill_time = prefill_time
        self.clock = 0.0
        self._step_seconds: dict[int, float] = {}
        self._phase = "init"
        self._step = 0
        self._pos = 0
        self._verified = None
        self._speculative = None
        self.predecode_bytes = 0
        self.predecode_new_pins = 0
        self.last_logits = None

    def close(self) -> None:
        self.cache.close()

    def _qkv(self, lw, x, positions):
        """engine.py:39-48, then rounded to bf16 at the hot-path boundary."""
        import torch
        q, k, v = self._qkv_f32(lw, x, positions)
        bf = lambda t: t.to(torch.bfloat16)
        return bf(q), bf(k), bf(v)

    # -- phases (engine.py:220-339) --------------------------------------------------------
    def prefill(self, prompt) -> int:
        import torch
        if self._phase != "init":
            raise ProtocolError("prefill may only run once")
        cfg = self.config
        prompt = [int(t) for t in prompt]
        if not prompt:
            raise ValueError("prompt must be nonempty")
        if len(prompt) > cfg.max_len:
            raise ValueError("prompt longer than the configured max length")
        n = len(prompt)
        x = self.emb[prompt].clone()
        mask = torch.tril(torch.ones((n, n), dtype=torch.bool, device=self.dev))
        scale = np.float32(cfg.head_dim ** -0.5)
        for layer, lw in enumerate(self.lw):
            q, k, v = self._qkv(lw, x, range(n))
            self.cache.prefill(layer, k[None], v[None])  # Alg. 1: slow tier + bulk quantization
            # full-precision causal attention over the local prompt KV (engine.py:236-238)
            qf, kf, vf = q.float(), k.float(), v.float()
            outs = []
            for hq in range(cfg.q_heads):
                hk = hq // (cfg.q_heads // cfg.kv_heads)
                s = (qf[:, hq, :] @ kf[:, hk, :].T) * float(scale)
                s = torch.where(mask, s, torch.tensor(-math.inf, device=self.dev))
                a = torch.softmax(s, dim=-1)
                outs.append(a @ vf[:, hk, :])
            att = torch.cat(outs, dim=1).to(torch.bfloat16).float()
            x = self._ffn(lw, x + att @ lw["wo"])
        self._pos = n
        self._verified = int(torch.argmax(self._logits(x[-1:])[0]))
        self._phase = "prefilled"
        return self._verified

    def _ticket_bytes(self, layer: int) -> tuple[int, int]:
        _, newc = self.layer_dec.ticket(layer)
        new = int(newc.sum().item())
        return self.cache.row_bytes(new), new

    def predecode(self) -> int:
        import torch
        if self._phase != "prefilled":
            raise ProtocolError("predecode requires a completed prefill")
        p = self._pos
        self._measure_begin()
        x = self.emb[[self._verified]].clone()
        for layer, lw in enumerate(self.lw):
            q, k, v = self._qkv(lw, x, [p])
            out = self.layer_dec.predecode_layer(layer, q[None], k[None], v[None])
            nbytes, new = self._ticket_bytes(layer)
            self.predecode_bytes += nbytes
            self.predecode_new_pins += new
            self._charge(0, nbytes)
            x = self._ffn(lw, x + out[0].reshape(1, -1).float() @ lw["wo"])
        self._speculative = int(torch.argmax(self._logits(x)[0]))
        self._measure_end(0)
        self._phase = "decoding"
        self._step = 1
        return self._speculative

    def decode_step(self):
        import torch
        if self._phase != "decoding":
            raise ProtocolError("decode_step requires predecode first")
        p = self._pos
        self._measure_begin()
        x = self.emb[[self._verified, self._speculative]].clone()
        pin_mass, bytes_fetched, new_pins = [], 0, 0
        for layer, lw in enumerate(self.lw):
            q, k, v = self._qkv(lw, x, (p, p + 1))
            res = self.layer_dec.decode_layer(layer, self._step, q[None], k[None], v[None])
            pin_mass.append(res.pinned_mass[0].double().cpu().numpy())
            nbytes, new = self._ticket_bytes(layer)
            bytes_fetched += nbytes
            new_pins += new
            self._charge(self._step, nbytes)
            x = self._ffn(lw, x + res.out[0].reshape(2, -1).float() @ lw["wo"])
        logits = self._logits(x)
        verified_next = int(torch.argmax(logits[0]))
        speculative_next = int(torch.argmax(logits[1]))
        self._measure_end(self._step)
        metrics = StepMetrics(step=self._step, token=verified_next,
                              speculative_hit=bool(verified_next == self._speculative),
                              pinned_mass=float(np.mean(np.concatenate(pin_mass))),
                              bytes_fetched=bytes_fetched, new_pins=new_pins)
        self.last_logits = logits.cpu().numpy()
        self._verified, self._speculative = verified_next, speculative_next
        self._pos = p + 1
        self._step += 1
        return verified_next, metrics

    # -- logical clock (transfer.py:90-112), the reference's report model --------------
    def _charge(self, step: int, nbytes: int) -> None:
        if nbytes > 0:
            self._step_seconds[step] = self._step_seconds.get(step, 0.0) + transfer_time(
                nbytes, self.channel_model, contiguous=False)

    def step_transfer_seconds(self, step: int) -> float:
        if self.clock_mode == "measured":
            return self._measured.get(step, {}).get("transfer_s", 0.0)
        return self._step_seconds.get(step, 0.0)

    def end_step(self, step: int, compute_s: float) -> float:
        overlapped = step_latency(compute_s, self.step_transfer_seconds(step), overlapped=True)
        self.clock += overlapped
        return overlapped

    # -- measured clock (CUDA events + the library's per-launch event pairs) -------------
    def _measure_begin(self) -> None:
        if self.clock_mode != "measured":
            return
        import torch
        self.cache.profile(True)  # drain + reset, record events for this step
        self._ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        self._ev[0].record()

    def _measure_end(self, step: int) -> None:
        if self.clock_mode != "measured":
            return
        self._ev[1].record()
        prof = self.cache.profile(False)  # synchronizes the device
        step_s = self._ev[0].elapsed_time(self._ev[1]) / 1e3
        compute = max(0.0, step_s - prof["wait_ms"] / 1e3)
        transfer = prof["prefetch_ms"] / 1e3
        self._measured[step] = {"compute_s": compute, "transfer_s": transfer, "overlapped_s": step_s,
                                "serialized_s": compute + transfer, "h2d_bytes": prof["prefetch_bytes"],
                                "attn_s": prof["attn_ms"] / 1e3}

    def latency_row(self, step: int, compute_s: float) -> dict:
        """One report row's timing fields (engine.py:361-381), advancing the clock."""
        if self.clock_mode == "measured":
            m = self._measured[step]
            self.clock += m["overlapped_s"]
            return {"compute_s": m["compute_s"], "transfer_s": m["transfer_s"],
                    "overlapped_s": m["overlapped_s"], "serialized_s": m["serialized_s"]}
        t = self.step_transfer_seconds(step)
        return {"compute_s": compute_s, "transfer_s": t, "overlapped_s": self.end_step(step, compute_s),
                "serialized_s": step_latency(compute_s, t, overlapped=False)}


def generate(config, weights, prompt, steps: int, budget: CacheBudget,
             channel_model: ChannelModel | None = None, mode: str = "sim",
             compute_time_per_step: float = 0.0, prefill_time: float = 0.0,
             device: int = 0, clock: str = "logical") -> GenerateResult:
    """engine.py:342-386 on the device (clock: see the module docstring)."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    prompt = list(prompt)
    dec = DeviceSpeculativeDecoder(config, weights, budget, channel_model, mode,
                                   compute_time_per_step, prefill_time, device, clock,
                                   capacity=max(budget.context_length, len(prompt) + steps + 2))
    try:
        tokens = [dec.prefill(prompt)]
        dec.predecode()
        compute_s = compute_time_per_step
        rows = [{"step": 0, **dec.latency_row(0, compute_s),
                 "bytes": dec.predecode_bytes, "new_pins": dec.predecode_new_pins}]
        logits, metrics = [], []
        for _ in range(steps):
            step_idx = dec._step
            token, m = dec.decode_step()
            tokens.append(token)
            logits.append(dec.last_logits[0])
            metrics.append(m)
            rows.append({"step": step_idx, **dec.latency_row(step_idx, compute_s),
                         "bytes": m.bytes_fetched, "new_pins": m.new_pins})
        return GenerateResult(tokens=tokens, logits=logits, metrics=metrics, latency_rows=rows,
                              prefill_seconds=prefill_time, total_seconds=prefill_time + dec.clock,
                              decoder=dec)
    finally:
        dec.close()
