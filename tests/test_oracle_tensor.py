"""The tensor-equivalence oracle pinned to the reference's outputs, and the
host logic of tensor_match (graph view, topological ranks)."""

import numpy as np
import pytest

from _tensor_cases import data, names, random_tensors, traces
from oracle import tensor_equiv as ot
from paper_2512_08365_b200 import tensor_match as tm


def _close(a, b, rel=1e-12):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert abs(x - y) <= rel * max(abs(x), abs(y), 1e-300) + 1e-300, (x, y)


def test_round_robin_schedule_covers_every_pair_once():
    for n in range(2, 12):
        seen = [p for r in ot.rounds(n) for p in r]
        assert sorted(seen) == [(p, q) for p in range(n) for q in range(p + 1, n)]
        for r in ot.rounds(n):
            cols = [c for p in r for c in p]
            assert len(cols) == len(set(cols))


def test_oracle_invariant_sets_match_reference():
    for x, want in random_tensors():
        got = ot.invariant_set(x)
        assert len(got) == len(want)
        for g, w in zip(got, want):
            _close(g, w, 1e-12)


@pytest.mark.parametrize("name", names())
def test_oracle_prefilter_and_scores_match_reference(name):
    ta, tb = traces(name)
    A, B = tm._GraphView(ta), tm._GraphView(tb)
    runs = max(min(ta.run_count, tb.run_count), 1)
    ca = [len(ta.snapshot(t).values) for t in A.ids]
    cb = [len(tb.snapshot(t).values) for t in B.ids]
    na = [[ot.py_norm(ta.snapshot(t, r).values) for t in A.ids] for r in range(runs)]
    nb = [[ot.py_norm(tb.snapshot(t, r).values) for t in B.ids] for r in range(runs)]
    cand = ot.prefilter(ca, cb, na, nb, 1e-3)
    g = data()["match"][name]
    assert len(cand) == g["candidate_pairs"]
    want = {(a, b): s for a, b, s in g["pairs"]}
    for a, b in cand:
        key = (A.ids[a], B.ids[b])
        if key in want:
            worst = 0.0
            for r in range(runs):
                sa, sb = ta.snapshot(key[0], r), tb.snapshot(key[1], r)
                eq, s = ot.equivalent(np.reshape(sa.values, sa.shape), np.reshape(sb.values, sb.shape))
                assert eq
                worst = max(worst, s)
            assert worst == pytest.approx(want[key], rel=1e-6, abs=1e-12)


def test_topological_ranks_from_traces_match_compgraph_order():
    ta, _ = traces("tf32_misconfig")
    v = tm._GraphView(ta)
    assert v.rank[tm.SOURCE] == 0
    assert v.rank[tm.SINK] == len(v.rank) - 1
    ops = [o.op_id for o in ta.operators]
    # a chain: ranks follow the dependency order
    for op in ta.operators:
        for t in op.input_tensor_ids:
            p = v.producer[t]
            assert v.rank[p] < v.rank[op.op_id]
    assert set(ops) <= set(v.rank)
