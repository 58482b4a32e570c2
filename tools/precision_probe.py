#!/usr/bin/env python
"""Why K2 keeps the f16 hi+lo split of both B operands.

Emulates, in float64 numpy, single-f16 B operands (no lo part) for the score
MMA (B = Q*s per key channel) and for the value MMA (B = P*s per value group),
on 2-bit and 1-bit KIVI-quantized synthetic data (4096 tokens, d=128, g=32,
32 planted needle keys, q scale tau), and reports the output error against the
exact dequantized attention: before and after the bf16 output rounding, the
latter measured like tests/test_decode_gpu.py (norm-relative vs the
bf16-rounded reference, bar 2e-3).

  python tools/precision_probe.py
"""
import numpy as np


def bf16(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).bfloat16().float().numpy().astype(np.float64)


def f16(x):
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float64)


def quant(x, axis, bits):
    lo, hi = x.min(axis, keepdims=True), x.max(axis, keepdims=True)
    if bits == 2:
        z, s = lo, (hi - lo) / 3
        c = np.clip(np.rint((x - z) / np.where(s == 0, 1, s)), 0, 3)
    else:
        z, s = (3 * lo + hi) / 4, (hi - lo) / 2
        c = (x >= z + s / 2).astype(np.float64)
    return c, z, s


def main():
    rng = np.random.default_rng(0)
    n, d = 4096, 128
    sc = d ** -0.5 * np.log2(np.e)
    print("bits tau | keys hi-only: pre / after bf16 | values hi-only: pre / after bf16")
    for bits in (2, 1):
        for tau in (1.0, 3.0):
            worst = np.zeros(4)
            for _ in range(6):
                K = bf16(rng.standard_normal((n, d)) + rng.normal(0, 2, (1, d)))
                V = bf16(rng.standard_normal((n, d)))
                q = bf16(rng.standard_normal(d) * tau)
                K[rng.choice(n, 32, replace=False)] += 0.5 * q
                kc, kz, ks = quant(K.reshape(n // 32, 32, d), 1, bits)      # per-channel key groups
                vc, vz, vs = quant(V.reshape(n, 4, 32), 2, bits)            # per-token value groups
                Kq = (kc * ks + kz).reshape(n, d)
                Vq = (vc * vs + vz).reshape(n, d)
                S = (Kq @ q) * sc
                S_hi = ((kc * f16(q * ks * sc)).sum(-1) + (q * kz * sc).sum(-1)).reshape(n)

                def attend(S, hi_values):
                    P = np.exp2(S - S.max())
                    if not hi_values:
                        return (P @ Vq) / P.sum()
                    Ps = P[:, None, None] * vs
                    return ((P[:, None, None] * vz).sum(0) + (vc * f16(Ps)).sum(0)).reshape(d) / P.sum()

                O = attend(S, False)
                for i, got in enumerate((attend(S_hi, False), attend(S, True))):
                    pre = np.linalg.norm(got - O) / np.linalg.norm(O)
                    post = np.linalg.norm(bf16(got) - bf16(O)) / np.linalg.norm(bf16(O))
                    worst[2 * i] = max(worst[2 * i], pre)
                    worst[2 * i + 1] = max(worst[2 * i + 1], post)
            print(f"{bits}    {tau:.0f}   | {worst[0]:.2e} / {worst[1]:.2e}          | "
                  f"{worst[2]:.2e} / {worst[3]:.2e}")


def score_error_sources():
    """Score (log2 units) error against exact float64 arithmetic on a 32-token
    2-bit key block with channel offsets N(0, 2^2): the reference's own fp32
    path (q . K~ then * float32(d^-1/2)) vs K2's two terms -- the fp32 zero-point
    sum C_j (4-term lane partials + a 32-lane tree) and the f16 hi+lo key B
    operand.  All three are of the same order, so K2 differs from the reference
    by about as much as the reference differs from exact arithmetic."""
    rng = np.random.default_rng(0)
    d = 128
    f32 = np.float32
    e_ref = e_c = e_b = 0.0
    for _ in range(50):
        off = rng.normal(0, 2, d)
        K = (rng.standard_normal((32, d)) + off).astype(np.float32)
        q = (rng.standard_normal(d) * 1.5).astype(np.float32)
        lo, hi = K.min(0).astype(np.float64), K.max(0).astype(np.float64)
        z, s = lo, (hi - lo) / 3
        codes = np.clip(np.rint((K - z) / np.where(s == 0, 1, s)), 0, 3)
        Kq = codes * s + z
        sc = d ** -0.5 * np.log2(np.e)
        exact = Kq @ (q.astype(np.float64) * sc)
        Kq32 = Kq.astype(np.float32)
        ref = np.array([np.dot(q, Kq32[t]) for t in range(32)], dtype=np.float32) * f32(d ** -0.5)
        e_ref = max(e_ref, np.abs(ref.astype(np.float64) * np.log2(np.e) - exact).max())
        Qf = (q * f32(sc)).astype(np.float32)
        parts = (Qf * z.astype(np.float32)).astype(np.float32).reshape(32, 4).sum(1, dtype=np.float32)
        while parts.size > 1:
            parts = (parts[0::2] + parts[1::2]).astype(np.float32)
        e_c = max(e_c, abs(float(parts[0]) - float((Qf.astype(np.float64) * z).sum())))
        w = Qf.astype(np.float64) * s
        hi16 = f16(w)
        e_b = max(e_b, np.abs(codes @ (hi16 + f16(w - hi16)) - codes @ w).max())
    print(f"score error vs exact: reference fp32 {e_ref:.2e}; K2 zero-point sum {e_c:.2e}, hi/lo operand {e_b:.2e}")


if __name__ == "__main__":
    main()
    score_error_sources()
