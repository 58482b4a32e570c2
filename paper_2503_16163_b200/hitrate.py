"""Hit-rate study on the device.

The reference's analysis path -- a full-cache decode that records every
attention probability row (FullCacheDecoder, engine.py:86-160), the
AttentionTrace container and the two retention curves (hitrate.py:17-77), and
hitrate_experiment (experiments.py:100-137) -- with the trace resident in HBM
and the attention, the row checks and both curves computed by the CUDA kernels
of csrc/hitrate.cu (spc_full_attend, spc_trace_row_sums, spc_topk_hitrate,
spc_eviction_hitrate).  Rates are bit-identical to hitrate.py on the same
rows; see the kernel file for how the reference's float64 summation orders are
reproduced.

Layout: a trace is a device fp32 tensor data[nseq][steps][max_len] plus
lens[steps] (row t of every sequence has lens[t] valid entries); sequence
s = layer * q_heads + head, the order of AttentionTrace.sequences().
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .toymodel import ToyModel

__all__ = ["AttentionTrace", "topk_hitrate", "eviction_hitrate", "DeviceFullCacheDecoder",
           "hitrate_experiment"]


def _stream_ptr():
    import torch
    return torch.cuda.current_stream().cuda_stream


class AttentionTrace:
    """hitrate.py:17-31.  `rows[layer][head][query_step]` -> 1-d probability
    row (host arrays, as the reference), or a device tensor `data` of shape
    [nseq, steps, max_len] with `lens` (one length per step)."""

    def __init__(self, rows=None, *, data=None, lens=None, device: int = 0):
        import torch
        if data is None:
            if rows is None:
                raise ValueError("AttentionTrace needs rows or data")
            seqs = [seq for per_layer in rows for seq in per_layer]
            steps = len(seqs[0]) if seqs else 0
            if any(len(s) != steps for s in seqs):
                raise ValueError("every sequence of a trace must have the same number of query steps")
            lens = [int(np.asarray(r).size) for r in seqs[0]] if seqs else []
            for s in seqs:
                if [int(np.asarray(r).size) for r in s] != lens:
                    raise ValueError("trace rows of one query step must have equal lengths")
            L = max(lens) if lens else 0
            host = np.zeros((len(seqs), steps, max(L, 1)), np.float32)
            for i, s in enumerate(seqs):
                for t, r in enumerate(s):
                    host[i, t, :lens[t]] = np.asarray(r, np.float32)
            data = torch.as_tensor(host, device=f"cuda:{device}")
            self.layers = len(rows)
        else:
            self.layers = None
            if data.dim() != 3 or data.dtype != torch.float32 or not data.is_cuda:
                raise ValueError("trace data must be a [nseq, steps, max_len] float32 CUDA tensor")
        self.data = data.contiguous()
        self.lens = [int(x) for x in lens]
        if len(self.lens) != self.data.shape[1]:
            raise ValueError("lens must have one entry per query step")
        if self.lens and max(self.lens) > self.data.shape[2]:
            raise ValueError("a row length exceeds the trace's max_len")
        self._lens_dev = torch.as_tensor(np.asarray(self.lens or [0], np.int32), device=self.data.device)

    @property
    def nseq(self) -> int:
        return int(self.data.shape[0])

    @property
    def steps(self) -> int:
        return int(self.data.shape[1])

    @property
    def max_len(self) -> int:
        return max(self.lens) if self.lens else 0

    def _args(self):
        S, T, L = self.data.shape
        return (self.data.data_ptr(), T * L, L, self._lens_dev.data_ptr(), S, T, self.max_len)

    def sequences(self):
        """hitrate.py:23-25: host copies, one list of rows per (layer, head)."""
        host = self.data.cpu().numpy()
        for s in range(self.nseq):
            yield [host[s, t, :self.lens[t]].copy() for t in range(self.steps)]

    def row_sums(self) -> np.ndarray:
        """float32 np.sum of every row, [nseq, steps] (device)."""
        import torch
        out = torch.empty((self.nseq, self.steps), dtype=torch.float64, device=self.data.device)
        if self.nseq and self.steps:
            _lib.check(_lib.lib().spc_trace_row_sums(*self._args(), out.data_ptr(), _stream_ptr()))
        return out.cpu().numpy()

    def validate(self, tol: float = 1e-6) -> None:
        """hitrate.py:27-31."""
        if (np.abs(self.row_sums() - 1.0) > tol).any():
            raise ValueError("attention trace row does not sum to 1")

    def _rates(self, fn: str, k: int) -> np.ndarray:
        import torch
        if k < 0:
            raise ValueError("k must be >= 0")
        out = torch.empty((self.nseq, self.steps), dtype=torch.float64, device=self.data.device)
        if self.nseq and self.steps:
            _lib.check(getattr(_lib.lib(), fn)(*self._args(), int(k), out.data_ptr(), _stream_ptr()))
        return out.cpu().numpy()

    def topk_hitrates(self, k: int) -> np.ndarray:
        """topk_hitrate of every sequence, [nseq, steps]."""
        return self._rates("spc_topk_hitrate", k)

    def eviction_hitrates(self, k: int) -> np.ndarray:
        """eviction_hitrate of every sequence, [nseq, steps]."""
        return self._rates("spc_eviction_hitrate", k)


def _one_sequence(rows) -> AttentionTrace:
    return AttentionTrace([[list(rows)]])


def topk_hitrate(rows, k: int) -> np.ndarray:
    """hitrate.py:34-43: per query, the probability mass of the k largest
    entries of its row.  `rows` is one sequence (list of 1-d rows)."""
    if k < 0:
        raise ValueError("k must be >= 0")
    rows = list(rows)
    if not rows:
        return np.asarray([], np.float64)
    return _one_sequence(rows).topk_hitrates(k)[0]


def eviction_hitrate(rows, k: int) -> np.ndarray:
    """hitrate.py:46-77: greedy budget-k eviction driven by cumulative
    renormalised attention scores; the rate of query t is the full-row mass of
    the set retained after it."""
    if k < 0:
        raise ValueError("k must be >= 0")
    rows = list(rows)
    if not rows:
        return np.asarray([], np.float64)
    return _one_sequence(rows).eviction_hitrates(k)[0]


class DeviceFullCacheDecoder(ToyModel):
    """engine.py:86-160 on the GPU: greedy decode over an uncompressed fp32
    cache; decode-step attention is spc_full_attend, which writes each q head's
    probability row straight into the device trace."""

    def __init__(self, config, weights, device: int = 0):
        import torch
        super().__init__(config, weights, device)
        L = config.max_len
        self.K = torch.zeros((config.layers, L, config.kv_heads, config.head_dim), dtype=torch.float32,
                             device=self.dev)
        self.V = torch.zeros_like(self.K)
        self._pos = 0
        self._scale = float(np.float32(config.head_dim ** -0.5))
        self._scratch = None

    def prefill(self, prompt) -> int:
        """engine.py:101-121 (full-precision causal attention over the prompt)."""
        import math
        import torch
        cfg = self.config
        prompt = [int(t) for t in prompt]
        if not prompt:
            raise ValueError("prompt must be nonempty")
        if len(prompt) > cfg.max_len:
            raise ValueError("prompt longer than the configured max length")
        n = len(prompt)
        x = self.emb[prompt].clone()
        mask = torch.tril(torch.ones((n, n), dtype=torch.bool, device=self.dev))
        for layer, lw in enumerate(self.lw):
            q, k, v = self._qkv_f32(lw, x, range(n))
            self.K[layer, :n], self.V[layer, :n] = k, v
            outs = []
            for hq in range(cfg.q_heads):
                hk = hq // (cfg.q_heads // cfg.kv_heads)
                s = (q[:, hq, :] @ k[:, hk, :].T) * self._scale
                s = torch.where(mask, s, torch.tensor(-math.inf, device=self.dev))
                outs.append(torch.softmax(s, dim=-1) @ v[:, hk, :])
            x = self._ffn(lw, x + torch.cat(outs, dim=1) @ lw["wo"])
        self._pos = n
        return int(torch.argmax(self._logits(x[-1:])[0]))

    def step(self, token: int, trace_rows=None):
        """engine.py:123-141.  trace_rows: a device [layers * q_heads, >= p+1]
        fp32 view receiving this step's probability rows (or None)."""
        import torch
        cfg = self.config
        p = self._pos
        if p + 1 > cfg.max_len:
            raise ValueError("context exceeds the configured max length")
        x = self.emb[[int(token)]].clone()
        lib, st = _lib.lib(), _stream_ptr()
        if trace_rows is None:
            if self._scratch is None:
                self._scratch = torch.empty((cfg.q_heads, cfg.max_len), dtype=torch.float32, device=self.dev)
        for layer, lw in enumerate(self.lw):
            q, k, v = self._qkv_f32(lw, x, [p])
            self.K[layer, p], self.V[layer, p] = k[0], v[0]
            out = torch.empty((cfg.q_heads, cfg.head_dim), dtype=torch.float32, device=self.dev)
            if trace_rows is None:
                probs, ld = self._scratch, self._scratch.stride(0)
            else:
                probs = trace_rows[layer * cfg.q_heads:(layer + 1) * cfg.q_heads]
                ld = probs.stride(0)
            qc = q[0].contiguous()
            _lib.check(lib.spc_full_attend(qc.data_ptr(), self.K[layer].data_ptr(), self.V[layer].data_ptr(),
                                           p + 1, cfg.q_heads, cfg.kv_heads, cfg.head_dim, self._scale,
                                           out.data_ptr(), probs.data_ptr(), ld, st))
            x = self._ffn(lw, x + out.reshape(1, -1) @ lw["wo"])
        self._pos = p + 1
        logits = self._logits(x)[0]
        return int(torch.argmax(logits)), logits

    def generate(self, prompt, steps: int, record_trace: bool = False):
        """engine.py:143-160.  Returns (tokens, per-step logits, trace) where the
        trace is a device AttentionTrace (None unless record_trace)."""
        import torch
        cfg = self.config
        t = self.prefill(prompt)
        tokens, logits_list = [t], []
        data = None
        if record_trace:
            L = self._pos + steps
            data = torch.zeros((cfg.layers * cfg.q_heads, steps, L), dtype=torch.float32, device=self.dev)
        lens = []
        for s in range(steps):
            lens.append(self._pos + 1)
            t, logits = self.step(t, data[:, s] if record_trace else None)
            tokens.append(t)
            logits_list.append(logits.cpu().numpy())
        trace = AttentionTrace(data=data, lens=lens) if record_trace else None
        return tokens, logits_list, trace


def _round(x: float, digits: int = 9) -> float:
    return float(round(float(x), digits))


def hitrate_experiment(weights_path: str, prompt: list[int] | None, prompt_len: int, steps: int,
                       k_sweep: list[int], seed: int, max_len: int = 4096, device: int = 0) -> dict:
    """experiments.py:100-137 on the device: traced full-cache decode, then
    both hit-rate curves over the k sweep, per query and as means."""
    from .report import make_prompt
    from .weights import load_weights, with_runtime
    config, weights = load_weights(weights_path)
    config = with_runtime(config, max_len=max_len)
    if prompt is None:
        prompt = make_prompt(config.vocab, prompt_len, seed)
    dec = DeviceFullCacheDecoder(config, weights, device=device)
    _, _, trace = dec.generate(prompt, steps, record_trace=True)
    trace.validate()
    report_rows, summary_topk, summary_evict = [], [], []
    for k in k_sweep:
        topk_by_query = np.mean(trace.topk_hitrates(k), axis=0)
        evict_by_query = np.mean(trace.eviction_hitrates(k), axis=0)
        for q in range(len(topk_by_query)):
            report_rows.append({"k": int(k), "query_step": q, "topk_rate": _round(topk_by_query[q]),
                                "eviction_rate": _round(evict_by_query[q])})
        summary_topk.append(_round(float(np.mean(topk_by_query))))
        summary_evict.append(_round(float(np.mean(evict_by_query))))
    return {
        "experiment": "hitrate",
        "config": {"weights_path": weights_path, "prompt_len": len(prompt), "steps": steps,
                   "k_sweep": [int(k) for k in k_sweep], "seed": seed},
        "rows": report_rows,
        "summary": {"k_sweep": [int(k) for k in k_sweep], "topk_mean": summary_topk,
                    "eviction_mean": summary_evict},
    }
