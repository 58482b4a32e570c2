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


if __name__ == "__main__":
    main()
