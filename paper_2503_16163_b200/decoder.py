"""Full decoder step around the hot path.

The reference's per-layer body (engine.py:286-325: _qkv -> attend -> Wo ->
residual -> _ffn, then _logits / argmax for both rows) at real model sizes on
the B200, so tokens/s can be timed with the weight traffic included:

  add_rmsnorm (fused residual add + RMSNorm, layer.cu)
  -> x @ Wqkv (one cuBLAS bf16 GEMM for Wq|Wk|Wv)
  -> spc_qkv_rope (split + RoPE from a once-per-step spc_rope_table, layer.cu)
  -> spc_decode_layer (the hot path: K2 attend + K3/K4/K5 on the copy stream)
  -> o @ Wo -> add_rmsnorm -> x @ W1 -> spc_silu -> @ W2
  ... -> final add_rmsnorm -> x @ head -> spc_argmax_rows (both rows).

Residual stream fp32; GEMM operands bf16 with fp32 accumulation (cuBLAS);
weights stored [out, in] so every GEMM is x @ W^T.  Batch sharding (bench.py)
keeps this exchange-free, so there is no all-gather on this path.

KV-head sharding (``shard=HeadShard``, shard.py; SURVEY 8(e) collective (3)):
the rank projects and attends only its heads (its rows of Wq|Wk|Wv, its cache
shard), the per-head attention outputs are all-gathered across ranks (NCCL
over NVLink on a multi-GPU box) into the head order Wo expects, and Wo, the
FFN and the logits run replicated.  Layer-scope top-k reduces the partial
aggregates as in decode.SpeculativeLayerDecoder.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from .cache import DeviceTwoTierCache, current_stream

__all__ = ["StackConfig", "StackWeights", "random_stack", "stack_from_reference", "DecoderStack",
           "LLAMA2_7B"]


@dataclass(frozen=True)
class StackConfig:
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int
    hidden: int
    ffn: int
    vocab: int
    rope_base: float = 10000.0
    eps: float = 1e-6

    @property
    def qkv_width(self) -> int:
        return (self.q_heads + 2 * self.kv_heads) * self.head_dim

    def weight_bytes(self) -> int:
        """bf16 bytes one decode step streams (all layers + head; the embedding
        gather touches only 2*batch rows)."""
        h, qd = self.hidden, self.q_heads * self.head_dim
        per_layer = h * self.qkv_width + qd * h + 2 * h * self.ffn
        return 2 * (self.layers * per_layer + h * self.vocab)


# LLaMA-2-7B shape with the reference's two-matrix SiLU FFN (engine.py:66-68)
LLAMA2_7B = StackConfig(layers=32, q_heads=32, kv_heads=32, head_dim=128, hidden=4096, ffn=11008,
                        vocab=32000)


@dataclass
class StackWeights:
    emb: object           # bf16 [vocab, hidden]
    layers: list          # dicts: wqkv [qkv_width, h], wo [h, Hq*d], w1 [ffn, h], w2 [h, ffn] bf16;
    final_norm: object    #        attn_norm / ffn_norm fp32 [h]
    head: object          # bf16 [vocab, hidden]


def random_stack(cfg: StackConfig, device="cuda:0", seed: int = 0) -> StackWeights:
    """Random-init weights of the architecture (the reference's stds,
    model.py:79-96), drawn on the device."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    h, qd, kd = cfg.hidden, cfg.q_heads * cfg.head_dim, cfg.kv_heads * cfg.head_dim

    def rnd(shape, std):
        return (torch.randn(shape, generator=g, device=device, dtype=torch.float32) * std).to(torch.bfloat16)

    ones = lambda: torch.ones(h, dtype=torch.float32, device=device)
    layers = []
    for _ in range(cfg.layers):
        layers.append({"wqkv": rnd((qd + 2 * kd, h), h ** -0.5), "wo": rnd((h, qd), qd ** -0.5),
                       "w1": rnd((cfg.ffn, h), h ** -0.5), "w2": rnd((h, cfg.ffn), cfg.ffn ** -0.5),
                       "attn_norm": ones(), "ffn_norm": ones()})
    return StackWeights(emb=rnd((cfg.vocab, h), 1.0), layers=layers, final_norm=ones(),
                        head=rnd((cfg.vocab, h), h ** -0.5))


def stack_from_reference(cfg, weights, device="cuda:0") -> tuple[StackConfig, StackWeights]:
    """A reference DecoderConfig / Weights (model.py, [in, out] fp32) on the device."""
    import numpy as np
    import torch
    bf = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float32), device=device).to(torch.bfloat16)
    f32 = lambda a: torch.as_tensor(np.asarray(a, np.float32), device=device)
    sc = StackConfig(layers=cfg.layers, q_heads=cfg.q_heads, kv_heads=cfg.kv_heads, head_dim=cfg.head_dim,
                     hidden=cfg.hidden, ffn=cfg.ffn, vocab=cfg.vocab, rope_base=float(cfg.rope_base))
    layers = [{"wqkv": bf(np.concatenate([lw.wq, lw.wk, lw.wv], axis=1).T), "wo": bf(lw.wo.T),
               "w1": bf(lw.w1.T), "w2": bf(lw.w2.T), "attn_norm": f32(lw.attn_norm),
               "ffn_norm": f32(lw.ffn_norm)} for lw in weights.layers]
    return sc, StackWeights(emb=bf(weights.embedding), layers=layers, final_norm=f32(weights.final_norm),
                            head=bf(weights.head.T))


def _shard_weights(cfg: StackConfig, w: StackWeights, sh) -> StackWeights:
    """Rows of Wq|Wk|Wv for this rank's q and kv heads; everything else shared."""
    import torch
    d, qd, kd = cfg.head_dim, cfg.q_heads * cfg.head_dim, cfg.kv_heads * cfg.head_dim
    layers = []
    for lw in w.layers:
        wq, wk, wv = lw["wqkv"][:qd], lw["wqkv"][qd:qd + kd], lw["wqkv"][qd + kd:]
        wqkv = torch.cat([wq[sh.q_lo * d:sh.q_hi * d], wk[sh.kv_lo * d:sh.kv_hi * d],
                          wv[sh.kv_lo * d:sh.kv_hi * d]]).contiguous()
        layers.append({**lw, "wqkv": wqkv})
    return StackWeights(emb=w.emb, layers=layers, final_norm=w.final_norm, head=w.head)


class DecoderStack:
    """Decode steps of the whole model over a DeviceTwoTierCache (one per
    batch of sequences).  Preallocated buffers, no host syncs inside a step."""

    def __init__(self, cfg: StackConfig, weights: StackWeights, cache: DeviceTwoTierCache,
                 shard=None, group=None):
        import torch
        self.shard, self.group = shard, group
        self.full_q_heads = cfg.q_heads
        if shard is not None:  # this rank's heads; weights arrive whole and are sliced here
            weights = _shard_weights(cfg, weights, shard)
            cfg = StackConfig(**{**cfg.__dict__, "q_heads": shard.q_heads, "kv_heads": shard.kv_heads})
        if (cache.layers, cache.kv_heads, cache.head_dim, cache.q_heads) != (
                cfg.layers, cfg.kv_heads, cfg.head_dim, cfg.q_heads):
            raise ValueError("cache geometry does not match the decoder")
        if cfg.hidden % 8 or cfg.ffn % 8:
            raise ValueError("hidden and ffn must be multiples of 8")
        self.cfg, self.w, self.cache = cfg, weights, cache
        # the GEMMs and small kernels are latency-sensitive to queued sysmem reads:
        # run the PCIe gather at 128 KiB in flight (measured: C2 step -20%)
        cache.set_prefetch_inflight(128 << 10)
        dev = cache._torch_device
        self.dev = dev
        B = cache.batch
        R = 2 * B
        bf, f32, i32 = torch.bfloat16, torch.float32, torch.int32
        e = lambda *s, dt=bf: torch.empty(s, dtype=dt, device=dev)
        self.x = e(R, cfg.hidden, dt=f32)
        self.xn = e(R, cfg.hidden)
        self.qkv = e(R, cfg.qkv_width)
        self.q = e(B, 2, cfg.q_heads, cfg.head_dim)
        self.k = e(B, 2, cfg.kv_heads, cfg.head_dim)
        self.v = e(B, 2, cfg.kv_heads, cfg.head_dim)
        self.attn = e(B, 2, cfg.q_heads, cfg.head_dim)
        self.delta = e(R, cfg.hidden)
        self.g = e(R, cfg.ffn)
        self.logits = e(R, cfg.vocab)
        self.next = e(R, dt=i32)
        self.pos = e(R, dt=i32)
        self.rope = e(R, cfg.head_dim, dt=f32)  # (cos, sin) per (row, pair)
        self.pinned_mass = e(B, cfg.q_heads, dt=f32)
        if shard is not None:
            W = shard.world
            self.attn_all = e(W, R, cfg.q_heads * cfg.head_dim)            # all-gather target
            self.attn_cat = e(R, self.full_q_heads * cfg.head_dim)         # [row][rank][head][d]
            self._agg = None
            if cache.topk_scope == "layer":
                from .decode import SpeculativeLayerDecoder
                from .shard import allreduce_sum
                self._agg = SpeculativeLayerDecoder(cache, agg_reduce=allreduce_sum(group))
        self.launches = 0  # kernels + GEMMs this object issued outside spc_decode_layer

    def _layers(self, rows: int, step: int | None) -> None:
        """All layers over the first `rows` rows (2B decode, B predecode)."""
        import torch
        cfg, lib, st = self.cfg, _lib.lib(), current_stream(self.dev)
        h = self.cache.handle
        x, xn, qkv, delta, g = self.x[:rows], self.xn[:rows], self.qkv[:rows], self.delta[:rows], self.g[:rows]
        q = self.q.view(-1)[: rows * cfg.q_heads * cfg.head_dim]
        k = self.k.view(-1)[: rows * cfg.kv_heads * cfg.head_dim]
        v = self.v.view(-1)[: rows * cfg.kv_heads * cfg.head_dim]
        attn = self.attn.view(-1)[: rows * cfg.q_heads * cfg.head_dim]
        _lib.check(lib.spc_rope_table(self.pos.data_ptr(), rows, cfg.head_dim, cfg.rope_base,
                                      self.rope.data_ptr(), st))
        for layer, lw in enumerate(self.w.layers):
            _lib.check(lib.spc_add_rmsnorm(x.data_ptr(), delta.data_ptr() if layer else None,
                                           lw["attn_norm"].data_ptr(), xn.data_ptr(), rows, cfg.hidden,
                                           cfg.eps, st))
            torch.matmul(xn, lw["wqkv"].t(), out=qkv)
            _lib.check(lib.spc_qkv_rope(qkv.data_ptr(), self.rope.data_ptr(), rows, cfg.q_heads, cfg.kv_heads,
                                        cfg.head_dim, q.data_ptr(), k.data_ptr(), v.data_ptr(), st))
            if step is None:
                _lib.check(lib.spc_predecode_layer(h, layer, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                   attn.data_ptr(), st))
            else:
                _lib.check(lib.spc_decode_layer(h, layer, step, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                attn.data_ptr(), self.pinned_mass.data_ptr(), st))
            if self.shard is not None:
                if self._agg is not None:
                    self._agg._finish(layer)
                torch.matmul(self._gather_heads(attn, rows), lw["wo"].t(), out=delta)
            else:
                torch.matmul(attn.view(rows, -1), lw["wo"].t(), out=delta)
            _lib.check(lib.spc_add_rmsnorm(x.data_ptr(), delta.data_ptr(), lw["ffn_norm"].data_ptr(),
                                           xn.data_ptr(), rows, cfg.hidden, cfg.eps, st))
            torch.matmul(xn, lw["w1"].t(), out=g)
            _lib.check(lib.spc_silu(g.data_ptr(), g.numel(), st))
            torch.matmul(g, lw["w2"].t(), out=delta)
        _lib.check(lib.spc_add_rmsnorm(x.data_ptr(), delta.data_ptr(), self.w.final_norm.data_ptr(),
                                       xn.data_ptr(), rows, cfg.hidden, cfg.eps, st))
        logits = self.logits[:rows]
        torch.matmul(xn, self.w.head.t(), out=logits)
        _lib.check(lib.spc_argmax_rows(logits.data_ptr(), rows, cfg.vocab, self.next.data_ptr(), st))
        self.launches += len(self.w.layers) * 8 + 4

    def _gather_heads(self, attn, rows: int):
        """All-gather of the per-head attention outputs of every rank, laid out
        [row][all q heads][d] for Wo (ranks own contiguous head ranges)."""
        import torch
        import torch.distributed as dist
        W = self.shard.world
        src = attn.view(rows, -1)
        dst = self.attn_all[:, :rows]
        if W == 1:
            dst[0].copy_(src)
        elif dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(dst, src, group=self.group)
        else:  # gloo (CPU-side / single-GPU multi-process tests)
            dist.all_gather(list(dst.unbind(0)), src.contiguous(), group=self.group)
        cat = self.attn_cat[:rows]
        cat.view(rows, W, -1).copy_(dst.transpose(0, 1))
        return cat

    def _embed(self, tokens, rows: int) -> None:
        import torch
        torch.index_select(self.w.emb, 0, tokens.reshape(-1)[:rows].to(torch.int64), out=self.xn[:rows])
        self.x[:rows].copy_(self.xn[:rows])
        self.launches += 2

    def predecode(self, tokens, positions):
        """Alg. 2 over the model: tokens [B] (verified T1), positions [B] (= n).
        Returns next tokens [B] int32 (device)."""
        import torch
        B = self.cache.batch
        self.pos[:B].copy_(torch.as_tensor(positions, device=self.dev).to(torch.int32).reshape(B))
        self._embed(torch.as_tensor(tokens, device=self.dev), B)
        self._layers(B, None)
        return self.next[:B]

    def decode_step(self, step: int, tokens, positions):
        """One dual-token step: tokens [B, 2] (verified, speculative) at
        positions [B] (verified position p; speculative p + 1).  Returns
        next tokens [B, 2] int32 (device): row 0 = verified next, row 1 =
        speculative next (engine.py:323-331)."""
        import torch
        B = self.cache.batch
        p = torch.as_tensor(positions, device=self.dev).to(torch.int32).reshape(B, 1)
        self.pos.view(B, 2).copy_(torch.cat([p, p + 1], dim=1))
        self._embed(torch.as_tensor(tokens, device=self.dev), 2 * B)
        self._layers(2 * B, step)
        return self.next.view(B, 2)
