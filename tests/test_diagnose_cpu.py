"""Host side of the batched classifier (paper_2512_08365_b200/diagnose.py)
against the reference's golden categories: the program-model probe and the
LCS alignment need no device."""

import itertools
import random

import pytest

from _classify_cases import cases, traces
from paper_2512_08365_b200 import diagnose as dg


def _lcs_len(a, b):
    n, m = len(a), len(b)
    t = [[0] * (m + 1) for _ in range(n + 1)]
    for i in range(n - 1, -1, -1):
        for j in range(m - 1, -1, -1):
            t[i][j] = 1 + t[i + 1][j + 1] if a[i] == b[j] else max(t[i + 1][j], t[i][j + 1])
    return t[0][0]


def test_golden_corpus_covers_every_category():
    cats = {f[4] for c in cases().values() for f in c["findings"] if f[2] == "waste"}
    assert {"redundant", "misconfiguration", "api_misuse"} <= cats


@pytest.mark.parametrize("name", sorted(cases()))
def test_misconfiguration_probe_matches_reference(name):
    """Every finding the reference calls misconfiguration carries a config
    diagnosis; every api_misuse finding does not (redundant ones are decided
    before the probe runs)."""
    ta, tb = traces(name)
    for na, nb, verdict, _, cat, _ in cases()[name]["findings"]:
        if verdict != "waste" or cat == "redundant":
            continue
        assert dg._config_diagnosis(na, nb, ta, tb) == (cat == "misconfiguration"), (na, nb, cat)


def test_lcs_alignment_is_a_longest_common_subsequence():
    rng = random.Random(7)
    for _ in range(300):
        a = [rng.choice("abcd") for _ in range(rng.randrange(0, 9))]
        b = [rng.choice("abcd") for _ in range(rng.randrange(0, 9))]
        ma, mb = dg._lcs_matched(a, b)
        assert len(ma) == len(mb) == _lcs_len(a, b)
        pa, pb = sorted(ma), sorted(mb)
        assert all(a[i] == b[j] for i, j in zip(pa, pb))


def test_lcs_tie_rule_prefers_skipping_a():
    # dp[i+1][j] >= dp[i][j+1] skips a's element first (diagnose.py:219-222)
    ma, mb = dg._lcs_matched(["x", "y"], ["y", "x"])
    assert (ma, mb) == ({1}, {0})


def test_deviation_rules():
    assert dg._deviation(["f", "g", "h"], ["f", "g", "k"]) == 2
    assert dg._deviation(["f", "g"], ["f", "g", "k"]) is None
    with pytest.raises(dg.DisjointCallPathsError):
        dg._deviation(["f"], ["g"])
    with pytest.raises(dg.DiagnoseError):
        dg._deviation([], ["g"])


def test_kernelless_pair_raises_like_reference():
    name = next(iter(sorted(cases())))
    ta, tb = traces(name)
    empty = [o.op_id for o in ta.operators if not o.kernel_ids]
    empty_b = [o.op_id for o in tb.operators if not o.kernel_ids]
    for a, b in itertools.product(empty[:1], empty_b[:1]):
        with pytest.raises(dg.DiagnoseError):
            dg._config_diagnosis([a], [b], ta, tb)


def _walk_loop(o_s, o_e, entry, k_s, k_e):
    """diagnose.py:376-385 literally, per op."""
    lo, hi, own = [], [], []
    for i in range(len(o_s)):
        busy = sorted((int(s), int(e)) for s, e, x in zip(k_s, k_e, entry) if x == i)
        cur = int(o_s[i])
        for s, e in busy + [(int(o_e[i]), int(o_e[i]))]:
            if s > cur:
                lo.append(cur)
                hi.append(s)
                own.append(i)
            cur = max(cur, e)
    return lo, hi, own


@pytest.mark.parametrize("lift", [True, False])
def test_gap_walk_matches_reference_loop(lift):
    import numpy as np
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.integers(1, 6))
        o_s = np.sort(rng.integers(0, 1000, n))
        o_e = o_s + rng.integers(0, 300, n)
        rows = [(i, int(s), int(s + rng.integers(1, 80))) for i in range(n)
                for s in rng.integers(o_s[i], o_e[i] + 1, int(rng.integers(0, 5)))]
        rows = [r for r in rows if r[2] <= o_e[r[0]]]
        rng.shuffle(rows)
        entry = np.array([r[0] for r in rows], dtype=np.int64)
        k_s = np.array([r[1] for r in rows], dtype=np.int64)
        k_e = np.array([r[2] for r in rows], dtype=np.int64)
        lo, hi, own = dg.gap_walk(o_s, o_e, entry, k_s, k_e, lift=lift)
        want = _walk_loop(o_s, o_e, entry, k_s, k_e)
        assert (lo.tolist(), hi.tolist(), own.tolist()) == want
