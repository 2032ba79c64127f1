"""Oracle for the tensor-equivalence path -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

A numpy restatement of the reference's one-sided Jacobi singular values
(tensor_equiv.py:113-159: round-robin rounds from tensor_equiv.py:85-99, the
off-diagonal measure of :102-110, tolerance 1e-14, 60 sweeps), invariant sets
(:162-180), spectrum distance (:183-194), bottleneck embedding (:197-242) and
the decision of tensors_equivalent (:245-294), plus the match prefilter
(subgraph_match.py:128-145).  Pinned against the reference's own outputs in
tests/golden/tensors.json.gz (tests/test_oracle_tensor.py); the device path
(csrc/tensor.cu) is checked against it on adversarial inputs the reference's
corpus lacks.
"""

from __future__ import annotations

import math

import numpy as np

TOL = 1e-14
SWEEPS = 60
FLOOR = 1e-12
NORM_FLOOR = 1e-30


def rounds(n: int) -> list:
    """Circle-method schedule: position 0 fixed, the rest rotate right one
    place per round; an odd n gets a bye."""
    players = list(range(n)) + ([-1] if n % 2 else [])
    k = len(players)
    out = []
    for _ in range(k - 1):
        out.append([(min(players[i], players[k - 1 - i]), max(players[i], players[k - 1 - i]))
                    for i in range(k // 2) if players[i] >= 0 and players[k - 1 - i] >= 0])
        players = [players[0], players[-1]] + players[1:-1]
    return out


def _offdiag(a: np.ndarray) -> float:
    g = a.T @ a
    d = np.sqrt(np.clip(np.diag(g), 0.0, None))
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.abs(g) / np.outer(d, d)
    np.fill_diagonal(r, 0.0)
    return float(np.nan_to_num(r, nan=0.0).max())


def singular_values(mat) -> list:
    a = np.array(mat, dtype=np.float64)
    if a.shape[1] > a.shape[0]:
        a = a.T.copy()
    if a.shape[1] == 1:
        vals = [math.sqrt(float(a[:, 0] @ a[:, 0]))]
    else:
        sched = rounds(a.shape[1])
        for _ in range(SWEEPS):
            if _offdiag(a) <= TOL:
                break
            for pairs in sched:
                ps = np.array([p for p, _ in pairs])
                qs = np.array([q for _, q in pairs])
                cp, cq = a[:, ps], a[:, qs]
                al = (cp * cp).sum(0)
                be = (cq * cq).sum(0)
                ga = (cp * cq).sum(0)
                scale = np.sqrt(np.clip(al * be, 0.0, None))
                act = np.abs(ga) > TOL * np.where(scale > 0, scale, 1.0)
                if not act.any():
                    continue
                zeta = np.zeros_like(ga)
                zeta[act] = (be[act] - al[act]) / (2.0 * ga[act])
                t = np.zeros_like(ga)
                t[act] = np.sign(zeta[act]) / (np.abs(zeta[act]) + np.sqrt(1.0 + zeta[act] ** 2))
                t[act & (zeta == 0.0)] = 1.0
                c = 1.0 / np.sqrt(1.0 + t * t)
                s = c * t
                a[:, ps] = cp * c - cq * s
                a[:, qs] = cp * s + cq * c
        vals = np.sqrt((a * a).sum(0)).tolist()
    vals = sorted(vals, reverse=True)
    while vals and vals[-1] < FLOOR:
        vals.pop()
    return vals


def invariant_set(x) -> list:
    x = np.asarray(x, dtype=np.float64)
    r = x.ndim
    if r == 1:
        return [[math.sqrt(float(x @ x))]]
    out = []
    for mask in range(1, (1 << r) - 1):
        g = [m for m in range(r) if mask >> m & 1]
        c = [m for m in range(r) if not mask >> m & 1]
        out.append(singular_values(x.transpose(g + c).reshape(int(np.prod([x.shape[m] for m in g])), -1)))
    return out


def distance(a, b) -> float:
    n = max(len(a), len(b))
    if n == 0:
        return 0.0
    d = sum(((a[i] if i < len(a) else 0.0) - (b[i] if i < len(b) else 0.0)) ** 2 for i in range(n))
    na, nb = math.sqrt(sum(v * v for v in a)), math.sqrt(sum(v * v for v in b))
    return math.sqrt(d) / max(min(na, nb), NORM_FLOOR)


def _perfect(dist, limit) -> bool:
    n_large = len(dist[0]) if dist else 0
    adj = [[j for j in range(n_large) if row[j] <= limit] for row in dist]
    owner = [None] * n_large

    def aug(i, seen):
        for j in adj[i]:
            if j not in seen:
                seen.add(j)
                if owner[j] is None or aug(owner[j], seen):
                    owner[j] = i
                    return True
        return False

    return all(aug(i, set()) for i in range(len(dist)))


def embed(small, large, eps):
    if not small:
        return 0.0
    dist = [[distance(x, y) for y in large] for x in small]
    levels = sorted({d for row in dist for d in row if d <= eps})
    if not levels or not _perfect(dist, levels[-1]):
        return None
    lo, hi = 0, len(levels) - 1
    while lo < hi:
        mid = (lo + hi) // 2
        if _perfect(dist, levels[mid]):
            hi = mid
        else:
            lo = mid + 1
    return levels[lo]


def equivalent(a, b, eps=1e-3):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.size != b.size:
        return False, math.inf
    na, nb = math.sqrt(float(a.ravel() @ a.ravel())), math.sqrt(float(b.ravel() @ b.ravel()))
    nd = abs(na - nb) / max(min(na, nb), NORM_FLOOR)
    if nd > eps:
        return False, math.inf
    if a.ndim == 1 or b.ndim == 1:
        return nd <= eps, nd
    sa, sb = invariant_set(a), invariant_set(b)
    small, large = (sa, sb) if len(sa) <= len(sb) else (sb, sa)
    w = embed(small, large, eps)
    return (False, math.inf) if w is None else (True, w)


def prefilter(counts_a, counts_b, norms_a, norms_b, eps) -> list:
    """(a, b) index pairs surviving counts + per-run norm gaps, row-major;
    norms_* are [runs][n] arrays of sqrt(sum(v*v))."""
    out = []
    for a in range(len(counts_a)):
        for b in range(len(counts_b)):
            if counts_a[a] != counts_b[b]:
                continue
            ok = True
            for ra, rb in zip(norms_a, norms_b):
                x, y = ra[a], rb[b]
                if not abs(x - y) <= eps * max(min(x, y), 1e-30):
                    ok = False
                    break
            if ok:
                out.append((a, b))
    return out


def py_norm(values) -> float:
    """The prefilter norm exactly as the reference computes it (CPython sum)."""
    return math.sqrt(sum(v * v for v in values))
