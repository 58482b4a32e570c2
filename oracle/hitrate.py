"""Restatement of the reference hit-rate study -- TEST INFRASTRUCTURE ONLY
(see ``oracle/__init__.py``).  Follows ``hitrate.py`` (paths relative to
``/root/reference/pkg/src/speckv``) operation for operation, including the
float64 summation orders, so it is bit-identical to the reference; pinned by
``tests/test_hitrate.py`` against ``tests/golden/hitrate_rows.npz``.
"""
from __future__ import annotations

import numpy as np

__all__ = ["topk_hitrate", "eviction_hitrate", "pairwise_sum"]


def pairwise_sum(a) -> float:
    """numpy's float64 pairwise summation (the reduction np.sum uses): leaves
    of <= 128 elements with 8 strided accumulators, split at n/2 rounded down
    to a multiple of 8."""
    n = len(a)
    if n < 8:
        res = 0.0
        for v in a:
            res += float(v)
        return res
    if n <= 128:
        r = [float(a[j]) for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for j in range(i, n):
            res += float(a[j])
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


def topk_hitrate(rows, k: int) -> np.ndarray:
    """hitrate.py:34-43: mass of the k largest entries, summed descending."""
    if k < 0:
        raise ValueError("k must be >= 0")
    out = []
    for row in rows:
        row = np.asarray(row, dtype=np.float64)
        take = min(k, row.size)
        top = np.sort(row)[::-1][:take]
        out.append(pairwise_sum(top))
    return np.asarray(out)


def eviction_hitrate(rows, k: int) -> np.ndarray:
    """hitrate.py:46-77.  Candidates stay in ascending position order, so the
    victims of one query are the (len - k) smallest (cumulative, position)
    keys -- the reference's repeated min() -- and mass / rate are
    left-to-right float64 sums over that order."""
    if k < 0:
        raise ValueError("k must be >= 0")
    pos = np.zeros(0, np.int64)
    cum = np.zeros(0, np.float64)
    seen = 0
    out = []
    for row in rows:
        row = np.asarray(row, dtype=np.float64)
        new = np.arange(seen, row.size, dtype=np.int64)
        pos = np.concatenate([pos, new])
        cum = np.concatenate([cum, np.zeros(new.size)])
        seen = max(seen, row.size)
        mass = 0.0
        for i in pos:
            mass += row[i]
        if mass > 0:
            cum = cum + row[pos] / mass
        if pos.size > k:
            order = np.lexsort((pos, cum))        # ascending (cum, position)
            keep = np.sort(order[pos.size - k:])  # survivors, back in position order
            pos, cum = pos[keep], cum[keep]
        rate = 0.0
        for i in pos:
            rate += row[i]
        out.append(float(rate))
    return np.asarray(out)
