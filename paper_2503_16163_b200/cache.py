"""DeviceTwoTierCache -- the reference's TwoTierCache (kvcache.py:112-281),
batched over lockstep sequences and resident on a B200.

Fast tier in HBM: 1/2/4-bit packed codes + bf16 (min, max) group params,
residual window ring, pinned full-precision slot pool.  Slow tier: every
verified row, bf16, in pinned (page-locked, device-mapped) host memory.
All work runs in libspecache.so (csrc/); this class only marshals tensors and
mirrors the reference's method names, argument meaning and errors.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .budget import CacheBudget, frontier

__all__ = ["DeviceTwoTierCache", "to_device_bf16", "current_stream"]

_SCOPES = {"layer": 0, "kv_head": 1}


def _torch():
    import torch
    return torch


def current_stream(device) -> int:
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


def to_device_bf16(x, device):
    """numpy / torch -> contiguous bf16 CUDA tensor (float32 -> bf16 is RN-even,
    identical to oracle.restate.bf16_round)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.bfloat16)
    else:
        a = np.ascontiguousarray(np.asarray(x, np.float32))
        if not a.flags.writeable:  # e.g. np.broadcast_to views: torch wants a writable buffer
            a = a.copy()
        t = torch.from_numpy(a).to(device=device, dtype=torch.bfloat16)
    return t.contiguous()


class DeviceTwoTierCache:
    """TwoTierCache on the device.

    Parameters mirror ``TwoTierCache(layers, kv_heads, head_dim, budget)``; the
    extra keywords are the B200 batching/placement knobs:
    batch (lockstep sequences), q_heads (GQA width, default kv_heads),
    device, topk_scope ("layer" = reference, "kv_head" = per-KV-head sets),
    host_layers (distinct pinned-host slabs, default 0 = one per layer; a
    smaller value aliases layer l onto slab l % host_layers, which is only
    correct when the aliased layers are fed identical KV -- a benchmarking knob
    for host-memory budgets, see include/specache.h).
    """

    def __init__(self, layers: int, kv_heads: int, head_dim: int, budget: CacheBudget, *,
                 batch: int = 1, q_heads: int | None = None, device: int = 0,
                 topk_scope: str = "layer", host_layers: int = 0):
        if layers <= 0 or kv_heads <= 0 or head_dim <= 0:
            raise ValueError("layers, kv_heads and head_dim must be positive")
        if topk_scope not in _SCOPES:
            raise ValueError("topk_scope must be 'layer' or 'kv_head'")
        self.layers, self.kv_heads, self.head_dim = layers, kv_heads, head_dim
        self.budget = budget
        self.batch = batch
        self.q_heads = q_heads or kv_heads
        self.device = device
        self.topk_scope = topk_scope
        self.units = 1 if topk_scope == "layer" else kv_heads
        self.heads_per_unit = kv_heads if topk_scope == "layer" else 1
        dims = _lib.SpcDims(layers, batch, kv_heads, self.q_heads, head_dim, budget.bits,
                            budget.group_size, budget.residual, budget.prefetch_k,
                            budget.context_length, _SCOPES[topk_scope], host_layers)
        self._h = ctypes.c_void_p()
        _lib.check(_lib.lib().spc_cache_create(ctypes.byref(dims), device, ctypes.byref(self._h)))
        self._torch_device = f"cuda:{device}"

    # -- lifetime ----------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.lib().spc_cache_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def _stream(self) -> int:
        return current_stream(self._torch_device)

    @property
    def fast_path(self) -> bool:
        return bool(_lib.lib().spc_cache_fast_path(self._h))

    def set_attend_impl(self, impl: str) -> None:
        """'auto' | 'generic' (exact float64 dequant) | 'fast' (tensor cores)."""
        _lib.check(_lib.lib().spc_set_attend_impl(self._h, {"auto": 0, "generic": 1, "fast": 2}[impl]))

    def set_agg_mode(self, mode: str) -> None:
        """Top-k aggregate: 'spill' (default) or 'recompute' (SURVEY hard part (b))."""
        if mode not in ("spill", "recompute"):
            raise ValueError("agg mode must be 'spill' or 'recompute'")
        _lib.check(_lib.lib().spc_set_agg_mode(self._h, 0 if mode == "spill" else 1))

    def set_prefetch_inflight(self, nbytes: int) -> None:
        """K5 sysmem bytes in flight over the batch (0 = default 256 KiB)."""
        _lib.check(_lib.lib().spc_set_prefetch_inflight(self._h, int(nbytes)))

    def profile(self, enable: bool) -> dict:
        """Collect (and reset) the library's CUDA-event timings since the last
        call, then switch event recording on/off for what follows.  Synchronizes
        the device.  ms fields: attn = K2 launches, copy = copy-stream work per
        layer (agg .. host append), wait = exposed prefetch waits on the compute
        stream, prefetch = PCIe gather kernels; prefetch_bytes = rows moved."""
        import ctypes as C
        lib = _lib.lib()
        am, al, sm, sl, nl = C.c_double(), C.c_int64(), C.c_double(), C.c_int64(), C.c_int64()
        _lib.check(lib.spc_profile(self._h, int(bool(enable)), C.byref(am), C.byref(al), C.byref(sm),
                                   C.byref(sl), C.byref(nl)))
        return {"attn_ms": am.value, "attn_launches": al.value, "copy_ms": sm.value,
                "copy_launches": sl.value, "launches": nl.value,
                "wait_ms": float(lib.spc_profile_wait_ms(self._h)),
                "prefetch_ms": float(lib.spc_profile_prefetch_ms(self._h)),
                "prefetch_bytes": int(lib.spc_profile_prefetch_bytes(self._h))}

    @property
    def device_bytes(self) -> int:
        return int(_lib.lib().spc_device_bytes(self._h))

    @property
    def host_bytes(self) -> int:
        return int(_lib.lib().spc_host_bytes(self._h))

    # -- bookkeeping (kvcache.py:133-150) ------------------------------------------
    def length(self, layer: int) -> int:
        self._check_layer(layer)
        return int(_lib.lib().spc_length(self._h, layer))

    def quantized_frontier(self, layer: int) -> int:
        self._check_layer(layer)
        return int(_lib.lib().spc_frontier(self._h, layer))

    def packed_positions(self, layer: int) -> range:
        return range(self.quantized_frontier(layer))

    def residual_positions(self, layer: int) -> range:
        return range(self.quantized_frontier(layer), self.length(layer))

    def pinned_positions(self, layer: int, seq: int = 0, unit: int = 0) -> tuple:
        torch = _torch()
        self._check_layer(layer)
        ptr = ctypes.c_void_p()
        _lib.check(_lib.lib().spc_pin_state(self._h, layer, ctypes.byref(ptr)))
        n = self.batch * self.units * self.budget.prefetch_k
        torch.cuda.synchronize(self._torch_device)
        arr = _device_to_numpy(ptr.value, n * 4, np.int32, self._torch_device)
        arr = arr.reshape(self.batch, self.units, -1)[seq, unit]
        return tuple(sorted(int(p) for p in arr if p >= 0))

    def row_bytes(self, positions: int) -> int:
        # 16-bit accounting, key + value rows (kvcache.py:148-150)
        return positions * 2 * self.head_dim * 2 * self.kv_heads

    def _check_layer(self, layer: int) -> None:
        if not 0 <= layer < self.layers:
            raise ValueError("layer out of range")

    # -- writes ---------------------------------------------------------------------
    def prefill(self, layer: int, K, V) -> None:
        """Bulk form of n x append_verified (engine.py:234-235): K, V
        [batch, n, kv_heads, head_dim] (numpy float32 or torch)."""
        k = to_device_bf16(K, self._torch_device)
        v = to_device_bf16(V, self._torch_device)
        if k.dim() == 3:
            k, v = k.unsqueeze(0), v.unsqueeze(0)
        want = (self.batch, k.shape[1], self.kv_heads, self.head_dim)
        if tuple(k.shape) != want or tuple(v.shape) != want:
            raise ValueError(f"prefill rows must have shape {want}")
        _lib.check(_lib.lib().spc_prefill(self._h, layer, k.data_ptr(), v.data_ptr(), k.shape[1],
                                          self._stream()))
        self._keepalive = (k, v)

    def append_verified(self, layer: int, k_rows, v_rows) -> None:
        """kvcache.py:162-171: rows (kv_heads, head_dim) for batch 1, or
        (batch, kv_heads, head_dim)."""
        self._check_layer(layer)
        k = to_device_bf16(k_rows, self._torch_device)
        v = to_device_bf16(v_rows, self._torch_device)
        want = (self.kv_heads, self.head_dim)
        if k.dim() == 2:
            k, v = k.unsqueeze(0), v.unsqueeze(0)
        if tuple(k.shape[1:]) != want or tuple(v.shape[1:]) != want or k.shape[0] != self.batch:
            raise ValueError(f"rows must have shape {want}")
        _lib.check(_lib.lib().spc_append(self._h, layer, k.data_ptr(), v.data_ptr(), 0, self._stream()))
        self._keepalive = (k, v)

    def migrate_residual(self, layer: int) -> None:
        self._check_layer(layer)
        _lib.check(_lib.lib().spc_migrate(self._h, layer, self._stream()))

    def pin(self, layer: int, positions, k_rows=None, v_rows=None, seq: int = 0, unit: int = 0) -> None:
        """kvcache.py:194-218: replace the pinned set of (seq, unit); rows default
        to a slow-tier fetch.  Explicit rows: (len(positions), heads_per_unit, d)."""
        self._check_layer(layer)
        positions = [int(p) for p in positions]
        if len(positions) > self.budget.prefetch_k:
            raise ValueError("pinned set larger than the prefetch budget")
        pos = (ctypes.c_int32 * max(1, len(positions)))(*positions)
        kp = vp = None
        if k_rows is not None and v_rows is not None:
            k = to_device_bf16(k_rows, self._torch_device)
            v = to_device_bf16(v_rows, self._torch_device)
            if tuple(k.shape) != (len(positions), self.heads_per_unit, self.head_dim):
                raise ValueError("pin rows shape mismatch")
            order = np.argsort(positions, kind="stable")
            k, v = k[order].contiguous(), v[order].contiguous()
            kp, vp = k.data_ptr(), v.data_ptr()
            self._keepalive = (k, v)
        _lib.check(_lib.lib().spc_pin(self._h, layer, seq, unit, pos, len(positions), kp, vp,
                                      self._stream()))

    # -- reads ------------------------------------------------------------------------
    def materialize(self, layer: int, head: int, seq: int = 0):
        """kvcache.py:222-243, bit-identical float32: (keys, values) [n, d] numpy."""
        torch = _torch()
        n = self.length(layer)
        keys = torch.empty((max(n, 1), self.head_dim), dtype=torch.float32, device=self._torch_device)
        vals = torch.empty_like(keys)
        _lib.check(_lib.lib().spc_materialize(self._h, layer, seq, head, keys.data_ptr(),
                                              vals.data_ptr(), self._stream()))
        return keys[:n].cpu().numpy(), vals[:n].cpu().numpy()

    def slow_fetch(self, layer: int, positions, seq: int = 0):
        """kvcache.py:245-259: exact rows (npos, kv_heads, d) float32 + bytes."""
        positions = [int(p) for p in positions]
        npos = len(positions)
        shape = (npos, self.kv_heads, self.head_dim)
        k = np.zeros(shape, np.uint16)
        v = np.zeros(shape, np.uint16)
        pos = (ctypes.c_int32 * max(1, npos))(*positions)
        _lib.check(_lib.lib().spc_slow_fetch(self._h, layer, seq, pos, npos, k.ctypes.data, v.ctypes.data))
        return _bf16_to_f32(k), _bf16_to_f32(v), self.row_bytes(npos)

    def slow_rows(self, layer: int, head: int, seq: int = 0):
        n = self.length(layer)
        k, v, _ = self.slow_fetch(layer, range(n), seq)
        return k[:, head, :], v[:, head, :]

    def export_packed(self, layer: int, seq: int = 0) -> dict:
        """Normative packed arrays of one (layer, seq) (see oracle.restate.normative_export)."""
        torch = _torch()
        g, bits, d, H = self.budget.group_size, self.budget.bits, self.head_dim, self.kv_heads
        f = self.quantized_frontier(layer)
        nb, nch = (g * bits + 7) // 8, (d + g - 1) // g
        dev = self._torch_device
        kc = torch.zeros((max(f // g, 1), H, d, nb), dtype=torch.uint8, device=dev)
        kz = torch.zeros((max(f // g, 1), H, d), dtype=torch.int16, device=dev)
        ks = torch.zeros_like(kz)
        vc = torch.zeros((max(f, 1), H, nch, nb), dtype=torch.uint8, device=dev)
        vz = torch.zeros((max(f, 1), H, nch), dtype=torch.int16, device=dev)
        vs = torch.zeros_like(vz)
        _lib.check(_lib.lib().spc_export_packed(self._h, layer, seq, kc.data_ptr(), kz.data_ptr(),
                                                ks.data_ptr(), vc.data_ptr(), vz.data_ptr(),
                                                vs.data_ptr(), self._stream()))
        cut = lambda t, m: t[:m].cpu().numpy()
        return {"frontier": f,
                "key_codes": cut(kc, f // g), "key_zero": cut(kz, f // g).view(np.float16),
                "key_scale": cut(ks, f // g).view(np.float16), "val_codes": cut(vc, f),
                "val_zero": cut(vz, f).view(np.float16), "val_scale": cut(vs, f).view(np.float16)}

    def snapshot(self, seq: int = 0) -> dict:
        """Fast-tier dump in the reference's normative dict form
        (kvcache.py:270-281, quant.py:150-160) for one sequence."""
        layers = []
        g, bits, d = self.budget.group_size, self.budget.bits, self.head_dim
        for layer in range(self.layers):
            f = self.quantized_frontier(layer)
            blocks = []
            if bits == 16:
                K, V, _ = self.slow_fetch(layer, range(f), seq)
                for b0 in range(0, f, g):
                    heads = [{"keys_fp16": K[b0:b0 + g, h].astype(np.float16).tobytes().hex(),
                              "values_fp16": V[b0:b0 + g, h].astype(np.float16).tobytes().hex()}
                             for h in range(self.kv_heads)]
                    blocks.append({"start": b0, "count": g, "bits": bits, "heads": heads})
            else:
                e = self.export_packed(layer, seq)
                for bi in range(f // g):
                    heads = []
                    for h in range(self.kv_heads):
                        kg = [_group_dict(e["key_codes"][bi, h, c], g, bits, e["key_zero"][bi, h, c],
                                          e["key_scale"][bi, h, c]) for c in range(d)]
                        vr = []
                        for t in range(bi * g, bi * g + g):
                            row = []
                            for j in range((d + g - 1) // g):
                                cnt = min(d, (j + 1) * g) - j * g
                                row.append(_group_dict(e["val_codes"][t, h, j], cnt, bits,
                                                       e["val_zero"][t, h, j], e["val_scale"][t, h, j]))
                            vr.append(row)
                        heads.append({"key_groups": kg, "value_rows": vr})
                    blocks.append({"start": bi * g, "count": g, "bits": bits, "heads": heads})
            layers.append({"layer": layer, "quantized_frontier": f, "blocks": blocks})
        return {"layers": layers}


def _group_dict(codes: np.ndarray, count: int, bits: int, z16, s16) -> dict:
    nb = (count * bits + 7) // 8
    return {"codes": bytes(codes[:nb]).hex(), "count": int(count), "bits": bits,
            "zero_fp16": np.float16(z16).tobytes().hex(), "scale_fp16": np.float16(s16).tobytes().hex()}


def _bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def _device_to_numpy(ptr: int, nbytes: int, dtype, device) -> np.ndarray:
    """Copy a raw device allocation (owned by the library) to host."""
    torch = _torch()

    class _Holder:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_Holder(), device=device).cpu().numpy().view(dtype)


def frontier_of(n: int, budget: CacheBudget) -> int:
    return frontier(n, budget.residual, budget.group_size)
