"""Seeded synthetic inputs -- TEST INFRASTRUCTURE ONLY.

Every tensor is rounded to bf16 and returned as float32 so the bf16 device
path and the float32 reference see identical numbers.
  K = N(0,1) + per-(kv head, channel) offset N(0, 2^2)  (channel outliers)
  V = N(0,1)
  q = tau * N(0,1); optional planted "needle" keys K[i] += 0.5*q_spec
  drift: q_{t+1} = bf16(q_t + sigma*N(0,1))
"""
from __future__ import annotations

import numpy as np

from .restate import bf16_round

__all__ = ["make_kv", "make_queries", "make_step_kv"]


def make_kv(rng: np.random.Generator, n: int, kv_heads: int, head_dim: int,
            offset_std: float = 2.0):
    off = rng.normal(0.0, offset_std, size=(1, kv_heads, head_dim)).astype(np.float32)
    K = rng.standard_normal((n, kv_heads, head_dim)).astype(np.float32) + off
    V = rng.standard_normal((n, kv_heads, head_dim)).astype(np.float32)
    return bf16_round(K), bf16_round(V)


def make_queries(rng: np.random.Generator, rows: int, q_heads: int, head_dim: int,
                 tau: float = 1.0):
    return bf16_round((rng.standard_normal((rows, q_heads, head_dim)) * tau).astype(np.float32))


def make_step_kv(rng: np.random.Generator, rows: int, kv_heads: int, head_dim: int):
    k = rng.standard_normal((rows, kv_heads, head_dim)).astype(np.float32)
    v = rng.standard_normal((rows, kv_heads, head_dim)).astype(np.float32)
    return bf16_round(k), bf16_round(v)
