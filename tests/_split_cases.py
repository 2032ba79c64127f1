"""Seeded overlapping interval sets for the overlap-split tests (shared by the
CPU oracle tests and the GPU parity tests)."""
import numpy as np


def signal(rng, n, kind):
    ts = np.cumsum(rng.integers(1, 60, size=n)).astype(np.int64) + 1000
    w = rng.uniform(50.0, 700.0, size=n)
    span_hi = int(ts[-1] + rng.integers(1, 40)) if kind == "step" else int(ts[-1])
    return ts, w, span_hi


def overlapping(rng, ts, span_hi, m, streams=4):
    """m intervals from `streams` independent back-to-back streams (concurrent
    kernels), plus nested, duplicated, abutting and zero-length ones."""
    lo_all, hi_all = [], []
    t0, t1 = int(ts[0]), int(span_hi)
    per = max(m // (streams + 1), 1)
    for _ in range(streams):
        d = rng.integers(1, max(2, (t1 - t0) // per), size=per)
        st = t0 + rng.integers(0, max(1, (t1 - t0) // 4)) + np.concatenate([[0], np.cumsum(d)[:-1]])
        en = st + rng.integers(0, 3 * d.max() + 1, size=per)
        ok = en <= t1
        lo_all.append(st[ok]); hi_all.append(en[ok])
    lo = np.concatenate(lo_all); hi = np.concatenate(hi_all)
    k = len(lo)
    extra_lo = rng.integers(t0, t1, size=max(m - k, 4))
    extra_hi = np.minimum(extra_lo + rng.integers(0, 500, size=extra_lo.size), t1)
    lo = np.concatenate([lo, extra_lo, lo[:3], [t0, t0, t1]]).astype(np.int64)
    hi = np.concatenate([hi, extra_hi, hi[:3], [t0, t1, t1]]).astype(np.int64)  # duplicates, empty, full span
    perm = rng.permutation(lo.size)
    return lo[perm], hi[perm]


def disjoint(rng, ts, span_hi, m):
    t0, t1 = int(ts[0]), int(span_hi)
    cuts = np.sort(rng.choice(np.arange(t0, t1 + 1), size=2 * m, replace=False))
    lo, hi = cuts[0::2], cuts[1::2]
    hi = np.where(rng.random(m) < 0.3, np.minimum(lo + 0, hi), hi)  # some empty
    abut = rng.random(m - 1) < 0.3   # some abutting: hi[i] == lo[i+1]
    hi[:-1] = np.where(abut, lo[1:], hi[:-1])
    return lo.astype(np.int64), hi.astype(np.int64)
