"""Vectorised numpy restatement of the reference decode hot path.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Every function cites
the reference code it restates; paths are relative to
``/root/reference/pkg/src/speckv``.  Parity is pinned against fixtures made by
the reference itself (``tests/golden/``), checked in ``tests/test_oracle.py``.

Conventions
-----------
* Rows are float32 (the reference stores ``np.float32`` copies,
  ``kvcache.py:152-158``).  Callers feed bf16-representable values so the
  device (bf16 I/O) and this oracle see identical inputs.
* A "layer state" is the per-(layer, sequence) cache of the reference's
  ``TwoTierCache``: all appended rows ``K, V [n, Hkv, d]`` (the slow tier),
  the quantized frontier ``f`` and the pinned set.  The packed tier is a pure
  function of ``K[:f], V[:f]`` (blocks are quantized once, never rewritten,
  ``kvcache.py:173-192``), so it is recomputed on demand.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "FULL_PRECISION_BITS", "frontier", "quant_params", "quantize", "dequantize",
    "pack_groups", "unpack_groups", "quantize_keys_block", "quantize_values",
    "normative_export", "materialize_all", "masked_softmax_rows", "attend",
    "select_topk", "LayerState", "decode_layer", "predecode_layer",
    "row_bytes", "memory_ratio", "bf16_round",
]

FULL_PRECISION_BITS = 16
_SUPPORTED_BITS = (1, 2, 4)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (RN-even) and return float32.

    Synthetic inputs are made bf16-representable so the bf16 device path and
    the float32 reference see the same numbers.
    """
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return rounded.astype(np.uint32).view(np.float32).reshape(a.shape)


def frontier(n: int, residual: int, group: int) -> int:
    """Quantized frontier after n appends.

    ``append_verified`` migrates the oldest g residual rows whenever the
    residual reaches r + g (``kvcache.py:162-171``), so f(n) = g*floor((n-r)/g)
    for n >= r, else 0.
    """
    if n < residual:
        return 0
    return group * ((n - residual) // group)


def row_bytes(positions: int, head_dim: int, kv_heads: int) -> int:
    """16-bit accounting of a K+V fetch (``kvcache.py:148-150``)."""
    return positions * 2 * head_dim * 2 * kv_heads


def memory_ratio(bits: int, group_size: float, context_length: int, resident_extra: int) -> float:
    """``kvcache.py:55-63`` (half-up rounding to 2 decimals)."""
    import math
    from decimal import ROUND_HALF_UP, Decimal
    raw = bits / 16.0 + (0.0 if math.isinf(group_size) else 2.0 / group_size)
    raw += resident_extra / context_length
    return float(Decimal(repr(raw)).quantize(Decimal("0.01"), rounding=ROUND_HALF_UP))


# -- quantizer (quant.py) ---------------------------------------------------

def quant_params(groups: np.ndarray, bits: int):
    """Per-group (zero, scale) in float64 over the last axis (``quant.py:59-73``).

    B=1: zero=(3lo+hi)/4, scale=(hi-lo)/2 (Eq. 3); B>=2: zero=lo,
    scale=(hi-lo)/(2^B-1) (Eq. 2).
    """
    if bits not in _SUPPORTED_BITS:
        raise ValueError(f"unsupported bit width {bits!r}")
    g = np.asarray(groups, dtype=np.float64)
    if g.shape[-1] == 0:
        raise ValueError("cannot quantize an empty group")
    lo = g.min(axis=-1)
    hi = g.max(axis=-1)
    if bits == 1:
        zero = (3.0 * lo + hi) / 4.0
        scale = (hi - lo) / 2.0
    else:
        zero = lo
        scale = (hi - lo) / float((1 << bits) - 1)
    return zero, scale


def quantize(groups: np.ndarray, zero: np.ndarray, scale: np.ndarray, bits: int) -> np.ndarray:
    """Integer codes (``quant.py:76-87``): degenerate (scale==0) -> 0; B=1
    threshold ``x >= zero + scale/2``; B>=2 ``clip(rint((x-zero)/scale))``
    (round-half-even)."""
    x = np.asarray(groups, dtype=np.float64)
    z = np.asarray(zero)[..., None]
    s = np.asarray(scale)[..., None]
    deg = (np.asarray(scale) == 0.0)[..., None]
    if bits == 1:
        codes = (x >= z + s / 2.0).astype(np.float64)
    else:
        top = (1 << bits) - 1
        with np.errstate(divide="ignore", invalid="ignore"):
            codes = np.clip(np.rint((x - z) / s), 0, top)
    codes = np.where(deg, 0.0, codes)
    return codes.astype(np.uint8)


def dequantize(codes: np.ndarray, zero: np.ndarray, scale: np.ndarray) -> np.ndarray:
    """``float32(code*scale + zero)`` with float64 multiply then add
    (``quant.py:90-93``)."""
    return (np.asarray(codes).astype(np.float64) * np.asarray(scale)[..., None]
            + np.asarray(zero)[..., None]).astype(np.float32)


def pack_groups(codes: np.ndarray, bits: int) -> np.ndarray:
    """LSB-first packing of each last-axis group (``quant.py:96-109``):
    code i occupies bits [iB, (i+1)B).  Returns uint8 [..., ceil(G*B/8)]."""
    codes = np.asarray(codes, dtype=np.uint8)
    G = codes.shape[-1]
    per = 8 // bits
    nb = (G + per - 1) // per
    pad = np.zeros(codes.shape[:-1] + (nb * per,), dtype=np.uint16)
    pad[..., :G] = codes
    pad = pad.reshape(codes.shape[:-1] + (nb, per))
    shifts = (np.arange(per) * bits).astype(np.uint16)
    return (pad << shifts).sum(axis=-1).astype(np.uint8)


def unpack_groups(packed: np.ndarray, count: int, bits: int) -> np.ndarray:
    """Inverse of :func:`pack_groups` (``quant.py:112-123``)."""
    raw = np.asarray(packed, dtype=np.uint8)
    per = 8 // bits
    shifts = (np.arange(per) * bits).astype(np.uint8)
    mask = (1 << bits) - 1
    codes = ((raw[..., None] >> shifts) & mask).reshape(raw.shape[:-1] + (-1,))
    return codes[..., :count].astype(np.uint8)


def quantize_keys_block(kblocks: np.ndarray, bits: int):
    """Key layout (``quant.py:163-174`` via ``kvcache.py:184-188``): one group
    per (block, head, channel) spanning the block's g tokens.

    kblocks: [nb, g, H, d] float32 -> (codes [nb,H,d,g], zero, scale [nb,H,d]).
    """
    groups = np.ascontiguousarray(np.asarray(kblocks, np.float32).transpose(0, 2, 3, 1))
    z, s = quant_params(groups, bits)
    return quantize(groups, z, s, bits), z, s


def quantize_values(v: np.ndarray, bits: int, group: int):
    """Value layout (``quant.py:177-190`` via ``kvcache.py:189-190``): per
    token, groups of ``group`` consecutive channels (last group may be ragged).

    v: [f, H, d] -> list over chunks j of (codes [f,H,len_j], zero, scale [f,H]).
    """
    v = np.asarray(v, np.float32)
    d = v.shape[-1]
    out = []
    for j0 in range(0, d, group):
        chunk = v[..., j0:j0 + group]
        z, s = quant_params(chunk, bits)
        out.append((quantize(chunk, z, s, bits), z, s))
    return out


def normative_export(K: np.ndarray, V: np.ndarray, f: int, bits: int, group: int):
    """Normative packed form of the fast tier of one layer (what
    ``TwoTierCache.snapshot`` serialises, ``kvcache.py:270-281``,
    ``quant.py:150-160``), as arrays:

    key_codes  uint8 [nb, H, d, ceil(gB/8)]  key_zero/key_scale fp16 [nb, H, d]
    val_codes  uint8 [f, H, nchunk, ceil(gB/8)] (ragged chunks padded with 0)
    val_zero/val_scale fp16 [f, H, nchunk]
    fp16 params are the *direct* float64 -> float16 conversion (np.float16).
    """
    H, d = K.shape[1], K.shape[2]
    nb = f // group
    kc, kz, ks = quantize_keys_block(K[:f].reshape(nb, group, H, d), bits)
    chunks = quantize_values(V[:f], bits, group)
    nchunk = len(chunks)
    nbytes = (group * bits + 7) // 8
    val_codes = np.zeros((f, H, nchunk, nbytes), np.uint8)
    val_zero = np.zeros((f, H, nchunk), np.float16)
    val_scale = np.zeros((f, H, nchunk), np.float16)
    for j, (c, z, s) in enumerate(chunks):
        p = pack_groups(c, bits)
        val_codes[:, :, j, :p.shape[-1]] = p
        val_zero[:, :, j] = z.astype(np.float16)
        val_scale[:, :, j] = s.astype(np.float16)
    return {
        "key_codes": pack_groups(kc, bits), "key_zero": kz.astype(np.float16),
        "key_scale": ks.astype(np.float16), "val_codes": val_codes,
        "val_zero": val_zero, "val_scale": val_scale,
    }


def materialize_all(K: np.ndarray, V: np.ndarray, f: int, bits: int, group: int,
                    pinned=()):
    """Effective fast-tier K, V for every head (``kvcache.py:222-243``):
    dequantized packed [0,f), pinned positions overridden with the exact rows,
    residual [f,n) verbatim.  16-bit tier keeps float32 copies
    (``kvcache.py:82-90,185-187``).  Returns float32 [n, H, d] twice."""
    K = np.asarray(K, np.float32)
    V = np.asarray(V, np.float32)
    Kt = K.copy()
    Vt = V.copy()
    if f and bits != FULL_PRECISION_BITS:
        n, H, d = K.shape
        nb = f // group
        kc, kz, ks = quantize_keys_block(K[:f].reshape(nb, group, H, d), bits)
        Kt[:f] = dequantize(kc, kz, ks).transpose(0, 3, 1, 2).reshape(f, H, d)
        j0 = 0
        for c, z, s in quantize_values(V[:f], bits, group):
            w = c.shape[-1]
            Vt[:f, :, j0:j0 + w] = dequantize(c, z, s)
            j0 += w
    for p in pinned:
        Kt[p] = K[p]
        Vt[p] = V[p]
    return Kt, Vt


# -- attention + selection (numerics.py, engine.py) -------------------------

def masked_softmax_rows(scores: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """``numerics.py:24-39``."""
    scores = np.asarray(scores, dtype=np.float32)
    mask = np.asarray(mask, dtype=bool)
    if mask.shape != scores.shape:
        raise ValueError("mask shape must equal scores shape")
    if not mask.any(axis=-1).all():
        raise ValueError("softmax row with every cell masked")
    shifted = np.where(mask, scores, -np.inf)
    shifted = shifted - shifted.max(axis=-1, keepdims=True)
    expd = np.where(mask, np.exp(shifted), 0.0).astype(np.float32)
    return expd / expd.sum(axis=-1, keepdims=True)


def attend(q: np.ndarray, keys_by_head, values_by_head, mask: np.ndarray, group: int):
    """Grouped-query attention (``engine.py:51-63``): q head j reads kv head
    j // group; S = (q K^T) * float32(d^-0.5); A = masked softmax; O = A V.
    Returns (O [rows, Hq*d], list of per-q-head A [rows, n])."""
    q = np.asarray(q, np.float32)
    d = q.shape[-1]
    scale = np.float32(d ** -0.5)
    outs, probs = [], []
    for hq in range(q.shape[1]):
        hk = hq // group
        scores = (q[:, hq, :] @ np.asarray(keys_by_head[hk], np.float32).T) * scale
        a = masked_softmax_rows(scores, mask)
        outs.append(a @ np.asarray(values_by_head[hk], np.float32))
        probs.append(a)
    return np.concatenate(outs, axis=1), probs


def select_topk(scores: np.ndarray, k: int, eligible) -> tuple:
    """``engine.py:75-84``: k highest of float64(scores) over the eligible
    positions; ties to the lower position; sorted result."""
    eligible = np.asarray(sorted(int(p) for p in eligible), dtype=np.int64)
    if k <= 0 or eligible.size == 0:
        return ()
    sub = np.asarray(scores, dtype=np.float64)[eligible]
    order = np.argsort(-sub, kind="stable")
    picked = eligible[order[: min(k, eligible.size)]]
    return tuple(sorted(int(p) for p in picked))


class LayerState:
    """One (layer, sequence) of the reference ``TwoTierCache`` in array form.

    ``append``/``extend`` follow ``append_verified``/``migrate_residual``
    (``kvcache.py:162-192``): blocks crossing the frontier are quantized once
    and their codes + float64 params are kept (the reference's ``_PackedBlock``
    list); ``materialize_head`` dequantizes them every call like
    ``materialize`` (``kvcache.py:222-243``).  ``pinned`` follows ``pin``
    (``kvcache.py:194-218``, whole-set replacement): a dict unit -> sorted
    tuple, unit 0 for the reference's per-layer scope, or the kv head for the
    per-(kv-head) extension.
    """

    def __init__(self, kv_heads: int, head_dim: int, bits: int, group: int,
                 residual: int, prefetch_k: int, scope: str = "layer"):
        self.H, self.d = kv_heads, head_dim
        self.bits, self.g, self.r, self.k = bits, group, residual, prefetch_k
        self.scope = scope
        self.K = np.zeros((0, kv_heads, head_dim), np.float32)
        self.V = np.zeros((0, kv_heads, head_dim), np.float32)
        nunits = 1 if scope == "layer" else kv_heads
        self.pinned = {u: () for u in range(nunits)}
        self._pf = 0            # frontier covered by the stored codes
        self._kq = []           # per block batch: (codes [nb,H,d,g], zero, scale [nb,H,d])
        self._vq = []           # per token batch: list over chunks of (codes, zero, scale)

    @property
    def n(self) -> int:
        return self.K.shape[0]

    @property
    def f(self) -> int:
        return frontier(self.n, self.r, self.g)

    def append(self, k_rows: np.ndarray, v_rows: np.ndarray) -> None:
        self.K = np.concatenate([self.K, np.asarray(k_rows, np.float32)[None]], 0)
        self.V = np.concatenate([self.V, np.asarray(v_rows, np.float32)[None]], 0)

    def extend(self, K: np.ndarray, V: np.ndarray) -> None:
        self.K = np.concatenate([self.K, np.asarray(K, np.float32)], 0)
        self.V = np.concatenate([self.V, np.asarray(V, np.float32)], 0)

    def unit_of(self, head: int) -> int:
        return 0 if self.scope == "layer" else head

    def _sync_packed(self) -> None:
        f = self.f
        if self.bits == FULL_PRECISION_BITS or f <= self._pf:
            return
        a, g, H, d = self._pf, self.g, self.H, self.d
        nb = (f - a) // g
        self._kq.append(quantize_keys_block(self.K[a:f].reshape(nb, g, H, d), self.bits))
        self._vq.append(quantize_values(self.V[a:f], self.bits, g))
        self._pf = f

    def materialize_head(self, h: int):
        """Effective K, V [n, d] float32 of kv head h (kvcache.py:222-243)."""
        self._sync_packed()
        f = self.f
        Kt = self.K[:, h, :].copy()
        Vt = self.V[:, h, :].copy()
        if self.bits != FULL_PRECISION_BITS and f:
            pos = 0
            for (kc, kz, ks), vchunks in zip(self._kq, self._vq):
                nb = kc.shape[0]
                rows = nb * self.g
                Kt[pos:pos + rows] = dequantize(kc[:, h], kz[:, h], ks[:, h]).transpose(0, 2, 1).reshape(rows, self.d)
                j0 = 0
                for c, z, sc in vchunks:
                    w = c.shape[-1]
                    Vt[pos:pos + rows, j0:j0 + w] = dequantize(c[:, h], z[:, h], sc[:, h])
                    j0 += w
                pos += rows
            for p in self.pinned[self.unit_of(h)]:
                Kt[p] = self.K[p, h]
                Vt[p] = self.V[p, h]
        return Kt, Vt

    def materialize(self):
        """Per-head effective K, V: lists over kv heads of [n, d]."""
        ks, vs = zip(*[self.materialize_head(h) for h in range(self.H)])
        return list(ks), list(vs)


def _agg_by_unit(probs, row: int, n: int, group: int, scope: str, kv_heads: int):
    if scope == "layer":
        # engine.py:317 / :262 -- sum over ALL q heads of the layer.
        return [np.sum([a[row, :n] for a in probs], axis=0)]
    return [np.sum([probs[j][row, :n] for j in range(h * group, (h + 1) * group)], axis=0)
            for h in range(kv_heads)]


def _attend_streaming(state: LayerState, q: np.ndarray, k_new: np.ndarray, v_new: np.ndarray,
                      mask: np.ndarray):
    """``attend`` over [materialize(h) ; in-step rows], one kv head at a time
    (same float32 arithmetic as engine.py:51-63, bounded memory)."""
    Hq, d = q.shape[1], q.shape[2]
    group = Hq // state.H
    scale = np.float32(d ** -0.5)
    outs, probs = [None] * Hq, [None] * Hq
    for h in range(state.H):
        mk, mv = state.materialize_head(h)
        keys = np.concatenate([mk, k_new[:, h, :]], 0)
        vals = np.concatenate([mv, v_new[:, h, :]], 0)
        for hq in range(h * group, (h + 1) * group):
            scores = (q[:, hq, :] @ keys.T) * scale
            a = masked_softmax_rows(scores, mask)
            outs[hq] = a @ vals
            probs[hq] = a
    return np.concatenate(outs, axis=1), probs


def decode_layer(state: LayerState, q: np.ndarray, k_new: np.ndarray, v_new: np.ndarray,
                 append: bool = True):
    """One layer of ``SpeculativeDecoder.decode_step`` (``engine.py:299-321``)
    for one sequence, with the pins already applied (the awaited ticket).

    q [2,Hq,d]; k_new, v_new [2,Hkv,d].  Returns a dict with out [2,Hq,d],
    probs (per q head), agg (per unit), picked (per unit), new (per unit),
    pinned_mass [Hq].  Appends row 0 when ``append`` (``engine.py:321``).
    """
    q = np.asarray(q, np.float32)
    Hq, d = q.shape[1], q.shape[2]
    group = Hq // state.H
    n, f = state.n, state.f
    mask = np.ones((2, n + 2), dtype=bool)
    mask[0, n + 1] = False  # engine.py:310
    out, probs = _attend_streaming(state, q, k_new, v_new, mask)
    pinned_mass = np.zeros(Hq, np.float64)
    for j, a in enumerate(probs):  # engine.py:314-316
        pins = list(state.pinned[state.unit_of(j // group)])
        pinned_mass[j] = float(a[0, pins].sum()) if pins else 0.0
    aggs = _agg_by_unit(probs, 1, n, group, state.scope, state.H)
    picked, new = [], []
    for u, agg in enumerate(aggs):  # engine.py:270-284
        sel = select_topk(agg, state.k, range(f))
        prev = set(state.pinned[u])
        picked.append(sel)
        new.append([p for p in sel if p not in prev])
    if append:
        state.append(k_new[0], v_new[0])
    return {"out": out.reshape(2, Hq, d), "probs": probs, "agg": aggs,
            "picked": picked, "new": new, "pinned_mass": pinned_mass}


def predecode_layer(state: LayerState, q: np.ndarray, k_new: np.ndarray, v_new: np.ndarray):
    """One layer of ``SpeculativeDecoder.predecode`` (``engine.py:245-268``):
    single row at position n against the fast tier plus its own KV, agg from
    row 0, no append."""
    q = np.asarray(q, np.float32)
    Hq, d = q.shape[1], q.shape[2]
    group = Hq // state.H
    n, f = state.n, state.f
    mask = np.ones((1, n + 1), dtype=bool)
    out, probs = _attend_streaming(state, q, k_new, v_new, mask)
    aggs = _agg_by_unit(probs, 0, n, group, state.scope, state.H)
    picked, new = [], []
    for u, agg in enumerate(aggs):
        sel = select_topk(agg, state.k, range(f))
        prev = set(state.pinned[u])
        picked.append(sel)
        new.append([p for p in sel if p not in prev])
    return {"out": out.reshape(1, Hq, d), "probs": probs, "agg": aggs,
            "picked": picked, "new": new}
