"""Layout-blind tensor equivalence (host side; used only for detect_waste's 1%
output rule on boundary tensors, detect.py:55-69).

Restates the reference's criterion (tensor_equiv.py:118-294): two tensors are
equivalent when their element counts match, their Frobenius norms agree, and
the multiset of singular-value spectra of all non-trivial unfoldings of the
smaller-order tensor embeds injectively into the other's with every matched
pair within epsilon (relative L2 distance); the score is the bottleneck
distance of the best embedding.  Spectra come from LAPACK SVD here rather than
the reference's one-sided Jacobi (agreement ~1e-15 relative).  This is tiny
dense work on host snapshots (order <= 8), not on the GPU hot path.
"""

from __future__ import annotations

import math
from typing import Optional

import numpy as np

SPECTRUM_FLOOR = 1e-12
ORDER_CAP = 8
_NORM_FLOOR = 1e-30


def _arr(t) -> np.ndarray:
    if isinstance(t, np.ndarray):
        return np.asarray(t, dtype=np.float64)
    return np.asarray(t.values, dtype=np.float64).reshape(tuple(t.shape))


def _spectrum(mat: np.ndarray) -> np.ndarray:
    s = np.linalg.svd(mat, compute_uv=False)
    s = np.sort(s)[::-1]
    return s[s >= SPECTRUM_FLOOR]


def spectra(t) -> list[np.ndarray]:
    a = _arr(t)
    r = a.ndim
    if r > ORDER_CAP:
        raise ValueError(f"tensor order {r} exceeds the cap of {ORDER_CAP}")
    if r == 1:
        return [np.array([math.sqrt(float(a @ a))])]
    out = []
    for mask in range(1, (1 << r) - 1):
        rows = [m for m in range(r) if mask >> m & 1]
        cols = [m for m in range(r) if not mask >> m & 1]
        nr = int(np.prod([a.shape[m] for m in rows]))
        out.append(_spectrum(a.transpose(rows + cols).reshape(nr, -1)))
    return out


def _distance(x: np.ndarray, y: np.ndarray) -> float:
    n = max(len(x), len(y))
    if n == 0:
        return 0.0
    xp = np.zeros(n)
    yp = np.zeros(n)
    xp[:len(x)] = x
    yp[:len(y)] = y
    denom = max(min(math.sqrt(float(x @ x)), math.sqrt(float(y @ y))), _NORM_FLOOR)
    return math.sqrt(float(((xp - yp) ** 2).sum())) / denom


def _matching_ok(dist: np.ndarray, limit: float) -> bool:
    """Kuhn augmenting paths: can every row take a distinct column within limit?"""
    n_rows, n_cols = dist.shape
    owner = [-1] * n_cols

    def augment(i, seen):
        for j in range(n_cols):
            if dist[i, j] <= limit and not seen[j]:
                seen[j] = True
                if owner[j] < 0 or augment(owner[j], seen):
                    owner[j] = i
                    return True
        return False

    return all(augment(i, [False] * n_cols) for i in range(n_rows))


def tensors_equivalent(a, b, epsilon: float = 1e-3) -> tuple[bool, float]:
    if epsilon <= 0:
        raise ValueError("epsilon must be positive")
    xa, xb = _arr(a), _arr(b)
    if xa.size != xb.size:
        return False, math.inf
    na, nb = float(np.sqrt(np.sum(xa * xa))), float(np.sqrt(np.sum(xb * xb)))
    nd = abs(na - nb) / max(min(na, nb), _NORM_FLOOR)
    if nd > epsilon:
        return False, math.inf
    if xa.ndim == 1 or xb.ndim == 1:
        return nd <= epsilon, nd
    sa, sb = spectra(xa), spectra(xb)
    small, large = (sa, sb) if len(sa) <= len(sb) else (sb, sa)
    if not small:
        return True, 0.0
    dist = np.array([[_distance(x, y) for y in large] for x in small])
    levels = sorted({float(d) for d in dist.ravel() if d <= epsilon})
    if not levels or not _matching_ok(dist, levels[-1]):
        return False, math.inf
    lo, hi = 0, len(levels) - 1
    while lo < hi:
        mid = (lo + hi) // 2
        if _matching_ok(dist, levels[mid]):
            hi = mid
        else:
            lo = mid + 1
    return True, levels[lo]


def boundary_rel_diff(boundary_right, trace_a, trace_b, limit: float = 0.01) -> float:
    """detect._boundary_rel_diff (detect.py:55-69): worst boundary-tensor diff."""
    from .trace_model import elementwise_rel_diff

    worst = 0.0
    for ta, tb in boundary_right:
        sa, sb = trace_a.snapshot(ta), trace_b.snapshot(tb)
        if tuple(sa.shape) == tuple(sb.shape):
            d = elementwise_rel_diff(sa, sb)
            if d > limit:
                d = min(d, tensors_equivalent(sa, sb, 1.0)[1])
        else:
            d = tensors_equivalent(sa, sb, 1.0)[1]
        worst = max(worst, d)
    return worst
