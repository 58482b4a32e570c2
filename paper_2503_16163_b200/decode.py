"""The dual-token decode step of SpeCache, one layer at a time, on the device.

Reference: SpeculativeDecoder.predecode (engine.py:245-268) and the per-layer
body of SpeculativeDecoder.decode_step (engine.py:299-321), fed post-RoPE
q/k/v.  The projections, FFN and logits around it are outside the hot path;
callers hand in q [batch, rows, q_heads, d] and k_new/v_new
[batch, rows, kv_heads, d] (rows = 1 predecode, 2 decode: row 0 verified at
position n, row 1 speculative at n+1).

Per call the library launches, on the caller's stream: K2 attention over the
packed low-bit tier + pinned/residual/in-step rows, K3 combine + cross-head
aggregate; on its copy stream K4 top-k + pin diff and K5 the PCIe prefetch of
the new pins (the ticket); then K6 append of row 0.  The next decode_layer of
the same layer waits on that ticket's event (await_layer).
"""
from __future__ import annotations

import contextlib

from dataclasses import dataclass

import numpy as np

from . import _lib
from .cache import DeviceTwoTierCache, current_stream, to_device_bf16

__all__ = ["LayerResult", "StepMetrics", "SpeculativeLayerDecoder", "select_topk"]


@dataclass
class StepMetrics:
    """engine.py:164-172."""
    step: int
    token: int
    speculative_hit: bool
    pinned_mass: float
    bytes_fetched: int
    new_pins: int
    tokens_emitted: int = 1


@dataclass
class LayerResult:
    out: "object"          # torch bf16 [batch, rows, q_heads, d]
    pinned_mass: "object"  # torch fp32 [batch, q_heads] (decode only)


class SpeculativeLayerDecoder:
    """Drives one DeviceTwoTierCache through predecode / decode steps.

    Phase rules follow the reference state machine (engine.py:221-222,
    247-248, 288-289) per layer; ticket rules follow transfer.py:84-100 and are
    enforced by the C library (ProtocolError)."""

    def __init__(self, cache: DeviceTwoTierCache, agg_reduce=None):
        """agg_reduce: for a KV-head-sharded cache with layer-scope top-k
        (shard.py), a callable that sums a device fp32 tensor in place across
        ranks (e.g. ``shard.allreduce_sum()``).  It is called on the cache's
        copy stream after each layer's partial aggregate, before the top-k."""
        self.cache = cache
        self._dev = cache._torch_device
        self._agg_reduce = agg_reduce
        if agg_reduce is not None:
            _lib.check(_lib.lib().spc_set_agg_reduce(cache.handle, 1))

    def _finish(self, layer: int) -> None:
        """Cross-rank sum of the partial aggregate, then the rest of the ticket."""
        if self._agg_reduce is None:
            return
        import ctypes

        import torch
        lib = _lib.lib()
        ptr, count, stream = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_void_p()
        _lib.check(lib.spc_agg_buffer(self.cache.handle, layer, ctypes.byref(ptr), ctypes.byref(count),
                                      ctypes.byref(stream)))
        view = _device_f32(ptr.value, count.value, self._dev)
        with torch.cuda.stream(torch.cuda.ExternalStream(stream.value, device=self._dev)):
            self._agg_reduce(view)
        _lib.check(lib.spc_finish_layer(self.cache.handle, layer))

    def _inputs(self, q, k_new, v_new, rows):
        c = self.cache
        q = to_device_bf16(q, self._dev)
        k = to_device_bf16(k_new, self._dev)
        v = to_device_bf16(v_new, self._dev)
        if q.dim() == 3:
            q, k, v = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
        if tuple(q.shape) != (c.batch, rows, c.q_heads, c.head_dim):
            raise ValueError(f"q must be [batch, {rows}, q_heads, head_dim]")
        if tuple(k.shape) != (c.batch, rows, c.kv_heads, c.head_dim) or k.shape != v.shape:
            raise ValueError(f"k_new/v_new must be [batch, {rows}, kv_heads, head_dim]")
        return q, k, v

    def predecode_layer(self, layer: int, q, k_new, v_new, out=None):
        import torch
        c = self.cache
        q, k, v = self._inputs(q, k_new, v_new, 1)
        if out is None:
            out = torch.empty_like(q)
        _lib.check(_lib.lib().spc_predecode_layer(c.handle, layer, q.data_ptr(), k.data_ptr(),
                                                  v.data_ptr(), out.data_ptr(),
                                                  current_stream(self._dev)))
        self._keep = (q, k, v)
        self._finish(layer)
        return out

    def decode_layer(self, layer: int, step: int, q, k_new, v_new, out=None,
                     pinned_mass=None) -> LayerResult:
        import torch
        c = self.cache
        q, k, v = self._inputs(q, k_new, v_new, 2)
        if out is None:
            out = torch.empty_like(q)
        if pinned_mass is None:
            pinned_mass = torch.empty((c.batch, c.q_heads), dtype=torch.float32, device=self._dev)
        _lib.check(_lib.lib().spc_decode_layer(c.handle, layer, step, q.data_ptr(), k.data_ptr(),
                                               v.data_ptr(), out.data_ptr(), pinned_mass.data_ptr(),
                                               current_stream(self._dev)))
        self._keep = (q, k, v)
        self._finish(layer)
        return LayerResult(out, pinned_mass)

    @contextlib.contextmanager
    def step_graph(self):
        """Capture the decode_layer calls inside the block and launch them as one
        CUDA graph at its end (spc_graph_begin / spc_graph_launch): one graph
        launch per step instead of the per-layer kernels and cross-stream
        events.  The current stream must not be the legacy default stream;
        inputs must be device bf16 tensors and out / pinned_mass preallocated
        (nothing may allocate or copy from the host while capturing)."""
        lib, h = _lib.lib(), self.cache.handle
        s = current_stream(self._dev)
        _lib.check(lib.spc_graph_begin(h, s))
        try:
            yield self
        except BaseException:
            lib.spc_graph_abort(h)
            raise
        _lib.check(lib.spc_graph_launch(h, s))

    def graph_stats(self):
        """(instantiations, in-place updates) of the step graph."""
        import ctypes
        i, u = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().spc_graph_stats(self.cache.handle, ctypes.byref(i), ctypes.byref(u)))
        return i.value, u.value

    def ticket(self, layer: int):
        """(picked int32 [batch, units, k] ascending -1 padded, new_count int32 [batch, units])
        of the last ticket issued for ``layer``."""
        import torch
        c = self.cache
        picked = torch.empty((c.batch, c.units, c.budget.prefetch_k), dtype=torch.int32, device=self._dev)
        newc = torch.empty((c.batch, c.units), dtype=torch.int32, device=self._dev)
        _lib.check(_lib.lib().spc_ticket(c.handle, layer, picked.data_ptr(), newc.data_ptr(),
                                         current_stream(self._dev)))
        return picked, newc

    def debug_agg(self, layer: int):
        import torch
        c = self.cache
        L = _capacity(c)
        agg = torch.empty((c.batch, c.units, L), dtype=torch.float32, device=self._dev)
        _lib.check(_lib.lib().spc_debug_agg(c.handle, layer, agg.data_ptr(), current_stream(self._dev)))
        return agg

    def debug_output_f32(self, enable: bool = True) -> None:
        """Keep each layer's fp32 attention output (before the bf16 rounding) for parity tests."""
        _lib.check(_lib.lib().spc_debug_output_f32(self.cache.handle, int(enable)))

    def debug_out_f32(self, layer: int, rows: int):
        """The last fp32 output of `layer`: [batch, rows, q_heads, head_dim]."""
        import torch
        c = self.cache
        buf = torch.empty((c.batch, 2, c.q_heads, c.head_dim), dtype=torch.float32, device=self._dev)
        _lib.check(_lib.lib().spc_debug_out_f32(c.handle, layer, buf.data_ptr(), current_stream(self._dev)))
        return buf.view(-1)[:c.batch * rows * c.q_heads * c.head_dim].view(c.batch, rows, c.q_heads, c.head_dim)


class _CudaArray:
    """__cuda_array_interface__ over library-owned device memory (zero copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def _device_f32(ptr: int, count: int, device):
    import torch
    return torch.as_tensor(_CudaArray(ptr, count), device=device)


def _capacity(c: DeviceTwoTierCache) -> int:
    g = c.budget.group_size
    lcm = g
    while lcm % 32:
        lcm += g
    L = c.budget.context_length
    return (L + lcm - 1) // lcm * lcm


def select_topk(scores, k: int, eligible=None, device: int = 0) -> tuple:
    """Device select_topk (engine.py:75-84) for eligible = range(n) (the
    packed-positions domain): k highest, ties to the lower position, sorted."""
    import torch
    # + 0.0 turns -0.0 into +0.0: the radix select orders raw fp32 bit patterns,
    # and the reference treats -0.0 == 0.0 (stable argsort, engine.py:82)
    s = torch.as_tensor(np.asarray(scores, np.float32), device=f"cuda:{device}") + 0.0
    n = s.numel() if eligible is None else len(eligible)
    if eligible is not None and list(eligible) != list(range(n)):
        raise ValueError("device select_topk supports eligible = range(n)")
    if k <= 0 or n == 0:
        return ()
    if bool((s[:n] < 0).any()):
        raise ValueError("device select_topk expects non-negative scores (probability mass)")
    out = torch.empty(k, dtype=torch.int32, device=s.device)
    with torch.cuda.device(s.device):
        _lib.check(_lib.lib().spc_select_topk(s.data_ptr(), n, k, out.data_ptr(),
                                              current_stream(s.device)))
    return tuple(int(p) for p in out.cpu().tolist() if p >= 0)
