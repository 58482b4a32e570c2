"""fp32 toy decoder pieces on the GPU (engine.py:35-72, numerics.py:42-78).

Plumbing around the hot path, shared by the drop-in token loop
(adapter.DeviceSpeculativeDecoder) and the full-cache trace source of the
hit-rate study (hitrate.DeviceFullCacheDecoder).  Plain fp32 PyTorch on the
device with TF32 off, like the reference's numpy fp32; RoPE angles in fp64
(numerics.py:62).
"""
from __future__ import annotations

import numpy as np

_LAYER_FIELDS = ("wq", "wk", "wv", "wo", "attn_norm", "ffn_norm", "w1", "w2")


class ToyModel:
    def __init__(self, config, weights, device: int = 0):
        import torch
        torch.backends.cuda.matmul.allow_tf32 = False  # fp32 model math, as the reference
        self.config = config
        self.dev = f"cuda:{device}"
        T = lambda a: torch.as_tensor(np.asarray(a, np.float32), device=self.dev)
        self.emb = T(weights.embedding)
        self.lw = [{k: T(getattr(lw, k)) for k in _LAYER_FIELDS} for lw in weights.layers]
        self.final_norm, self.head = T(weights.final_norm), T(weights.head)
        d = config.head_dim
        idx = np.arange(d // 2, dtype=np.float64)
        self._inv_freq = config.rope_base ** (-2.0 * idx / d)

    def _rmsnorm(self, x, gain, eps=1e-6):
        import torch
        ms = torch.mean(x * x, dim=-1, keepdim=True)
        return x * gain / torch.sqrt(ms + eps)

    def _rope(self, x, positions):
        import torch
        ang = np.outer(np.asarray(positions, np.float64), self._inv_freq)  # float64 like numerics.py:62
        cos = torch.as_tensor(np.cos(ang).astype(np.float32), device=self.dev)[:, None, :]
        sin = torch.as_tensor(np.sin(ang).astype(np.float32), device=self.dev)[:, None, :]
        x0, x1 = x[..., 0::2], x[..., 1::2]
        out = torch.empty_like(x)
        out[..., 0::2] = x0 * cos - x1 * sin
        out[..., 1::2] = x0 * sin + x1 * cos
        return out

    def _qkv_f32(self, lw, x, positions):
        """engine.py:39-48 in fp32."""
        cfg = self.config
        n = x.shape[0]
        xn = self._rmsnorm(x, lw["attn_norm"])
        q = (xn @ lw["wq"]).reshape(n, cfg.q_heads, cfg.head_dim)
        k = (xn @ lw["wk"]).reshape(n, cfg.kv_heads, cfg.head_dim)
        v = (xn @ lw["wv"]).reshape(n, cfg.kv_heads, cfg.head_dim)
        return self._rope(q, positions), self._rope(k, positions), v

    def _ffn(self, lw, x):
        import torch
        xn = self._rmsnorm(x, lw["ffn_norm"])
        g = xn @ lw["w1"]
        return x + (g / (1.0 + torch.exp(-g))) @ lw["w2"]

    def _logits(self, x):
        return self._rmsnorm(x, self.final_norm) @ self.head
