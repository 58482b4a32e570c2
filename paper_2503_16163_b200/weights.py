"""Toy-decoder configuration and the reference's weight file.

The report/CLI layer (report.py, cli.py) takes the same weight files as the
reference's `speckv decode WEIGHTS` (src/speckv/model.py:1-8 states the
normative layout), so a file written by either side loads in the other:

  b"SPKC" | u32 version=1 | u32 layers, q_heads, kv_heads, head_dim, vocab,
  hidden, ffn, seed | little-endian float32 arrays: embedding (vocab, hidden);
  per layer wq (hidden, Hq*d), wk, wv (hidden, Hkv*d), wo (Hq*d, hidden),
  attn_norm, ffn_norm (hidden,), w1 (hidden, ffn), w2 (ffn, hidden);
  final_norm (hidden,); head (hidden, vocab).

`init_decoder` draws the same seeded parameters as model.py:73-97 (one
default_rng(seed) stream, N(0,1)*std cast to float32, in file order), so
`gen-weights` output is byte-identical to the reference's.  Host-side
plumbing only: the model around the hot path is not part of the path.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field, replace

import numpy as np

__all__ = ["DecoderConfig", "LayerWeights", "Weights", "init_decoder", "save_weights",
           "load_weights", "with_runtime", "MAGIC", "FORMAT_VERSION"]

MAGIC = b"SPKC"
FORMAT_VERSION = 1
_HEADER = struct.Struct("<9I")
_LAYER_FIELDS = ("wq", "wk", "wv", "wo", "attn_norm", "ffn_norm", "w1", "w2")


@dataclass(frozen=True)
class DecoderConfig:
    """model.py:22-49 -- same fields, defaults and validation messages."""
    layers: int = 2
    q_heads: int = 4
    kv_heads: int = 2
    head_dim: int = 8
    vocab: int = 64
    hidden: int = 32
    ffn: int = 64
    rope_base: float = 10000.0
    seed: int = 0
    max_len: int = 1024

    def __post_init__(self) -> None:
        for name in ("layers", "q_heads", "kv_heads", "head_dim", "vocab", "hidden", "ffn", "max_len"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.q_heads % self.kv_heads:
            raise ValueError("q_heads must be divisible by kv_heads")
        if self.head_dim % 2:
            raise ValueError("head_dim must be even (rotary pairs)")

    @property
    def group(self) -> int:
        return self.q_heads // self.kv_heads


@dataclass
class LayerWeights:
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    attn_norm: np.ndarray
    ffn_norm: np.ndarray
    w1: np.ndarray
    w2: np.ndarray


@dataclass
class Weights:
    embedding: np.ndarray
    layers: list = field(default_factory=list)
    final_norm: np.ndarray = None
    head: np.ndarray = None


def _shapes(cfg: DecoderConfig):
    """(name, shape) in file order (model.py:100-111)."""
    h, qd, kd = cfg.hidden, cfg.q_heads * cfg.head_dim, cfg.kv_heads * cfg.head_dim
    yield "embedding", (cfg.vocab, h)
    per_layer = {"wq": (h, qd), "wk": (h, kd), "wv": (h, kd), "wo": (qd, h), "attn_norm": (h,),
                 "ffn_norm": (h,), "w1": (h, cfg.ffn), "w2": (cfg.ffn, h)}
    for i in range(cfg.layers):
        for n in _LAYER_FIELDS:
            yield (i, n), per_layer[n]
    yield "final_norm", (h,)
    yield "head", (h, cfg.vocab)


def _std(cfg: DecoderConfig, name) -> float | None:
    """Init std per tensor (model.py:79-96); None = ones (norm gains)."""
    n = name[1] if isinstance(name, tuple) else name
    h, qd = cfg.hidden, cfg.q_heads * cfg.head_dim
    return {"embedding": 1.0, "wq": h ** -0.5, "wk": h ** -0.5, "wv": h ** -0.5, "wo": qd ** -0.5,
            "w1": h ** -0.5, "w2": cfg.ffn ** -0.5, "head": h ** -0.5}.get(n)


def _assemble(cfg: DecoderConfig, arrays: dict) -> Weights:
    w = Weights(embedding=arrays["embedding"], final_norm=arrays["final_norm"], head=arrays["head"])
    w.layers = [LayerWeights(**{n: arrays[(i, n)] for n in _LAYER_FIELDS}) for i in range(cfg.layers)]
    return w


def _arrays(w: Weights):
    yield w.embedding
    for lw in w.layers:
        for n in _LAYER_FIELDS:
            yield getattr(lw, n)
    yield w.final_norm
    yield w.head


def init_decoder(cfg: DecoderConfig) -> Weights:
    """Seeded parameters, bitwise identical to model.py:73-97 for equal seeds."""
    rng = np.random.default_rng(cfg.seed)
    arrays = {}
    for name, shape in _shapes(cfg):
        std = _std(cfg, name)
        arrays[name] = (np.ones(shape, np.float32) if std is None
                        else (rng.standard_normal(shape) * std).astype(np.float32))
    return _assemble(cfg, arrays)


def save_weights(path: str, cfg: DecoderConfig, w: Weights) -> int:
    """model.py:114-125: write the file, return its byte count."""
    blob = MAGIC + _HEADER.pack(FORMAT_VERSION, cfg.layers, cfg.q_heads, cfg.kv_heads, cfg.head_dim,
                                cfg.vocab, cfg.hidden, cfg.ffn, cfg.seed)
    blob += b"".join(np.ascontiguousarray(a, dtype="<f4").tobytes() for a in _arrays(w))
    with open(path, "wb") as fh:
        fh.write(blob)
    return len(blob)


def load_weights(path: str) -> tuple[DecoderConfig, Weights]:
    """model.py:128-163, same error messages."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != MAGIC:
        raise ValueError("not a weight file: bad magic")
    version, *dims = _HEADER.unpack_from(blob, 4)
    if version != FORMAT_VERSION:
        raise ValueError(f"unsupported weight format version {version}")
    layers, q_heads, kv_heads, head_dim, vocab, hidden, ffn, seed = dims
    cfg = DecoderConfig(layers=layers, q_heads=q_heads, kv_heads=kv_heads, head_dim=head_dim,
                        vocab=vocab, hidden=hidden, ffn=ffn, seed=seed)
    off = 4 + _HEADER.size
    arrays = {}
    for name, shape in _shapes(cfg):
        n = int(np.prod(shape))
        if off + 4 * n > len(blob):
            raise ValueError("weight file has trailing or missing bytes")
        arrays[name] = np.frombuffer(blob, "<f4", n, off).reshape(shape).astype(np.float32)
        off += 4 * n
    if off != len(blob):
        raise ValueError("weight file has trailing or missing bytes")
    return cfg, _assemble(cfg, arrays)


def with_runtime(cfg: DecoderConfig, **overrides) -> DecoderConfig:
    """model.py:166-168: runtime-only settings (max_len, rope_base)."""
    return replace(cfg, **overrides)
