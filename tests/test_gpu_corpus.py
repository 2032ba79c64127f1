"""Corpus mode: pipeline.analyze_corpus over several trace
pairs -- per pair the same ledgers / join / report order as the single-pair
``analyze`` (its top-k, n_waste and exact wasted joules), and the corpus
top-k equal to a full host sort of every pair's findings on the report key
(detect.py:263-266: wasted desc, nodes_a asc, then corpus order -- pair,
finding -- as a stable sort of the concatenated corpus)."""

from dataclasses import replace

import numpy as np
import pytest
import torch

from paper_2512_08365_b200 import synth
from paper_2512_08365_b200.pipeline import analyze, analyze_corpus

pytestmark = pytest.mark.gpu


def _corpus(n_pairs, n_ops):
    base = synth.scaled(synth.CONFIGS["C5"], n_ops)
    return [synth.make_pair(replace(base, seed=base.seed + i)) for i in range(n_pairs)]


def test_corpus_matches_single_pairs_and_full_sort():
    pairs = _corpus(5, 20_000)
    k = 50
    ca = analyze_corpus(pairs, k=k)
    all_keys = []
    for i, (a, b) in enumerate(pairs):
        single = analyze(a, b, k=k)
        ps = ca.pairs[i]
        assert ps.join.P == single.join.P
        torch.testing.assert_close(ps.join.order, single.join.order, rtol=0, atol=0)
        assert ps.n_waste == single.join.n_waste
        assert ps.wasted_joules == single.join.wasted_joules
        assert ps.total_a == single.ledger_a.total_joules and ps.total_b == single.ledger_b.total_joules
        jd = ps.join
        f = torch.arange(jd.P, device=jd.columns.key_hi.device)
        tie = jd.pair_of(f)[0]
        if jd.columns.tie_rank is not None:
            tie = torch.where(tie >= 0, jd.columns.tie_rank[tie.clamp(min=0)], tie)
        lo = ~(((tie + 1) << 32) | f)
        all_keys.append(np.stack([jd.columns.key_hi[:jd.P].cpu().numpy().view(np.uint64),
                                  lo.cpu().numpy().view(np.uint64),
                                  np.full(jd.P, i, dtype=np.uint64), f.cpu().numpy().view(np.uint64)]))
    kk = np.concatenate(all_keys, axis=1)
    sel = np.lexsort((kk[3], kk[2], ~(kk[1] >> np.uint64(32)), ~kk[0]))[:k]
    want = [(int(kk[2][j]), int(kk[3][j])) for j in sel]
    assert ca.top == want
    rows = ca.findings([(a, b) for a, b in pairs], classify=False)
    assert [r[0] for r in rows] == [p for p, _ in want]
    ws = [wf.wasted_joules for _, wf in rows]
    assert ws == sorted(ws, reverse=True) or rows[0][1].verdict != "waste"


def test_corpus_of_one_pair_and_empty_k():
    pairs = _corpus(1, 5_000)
    ca = analyze_corpus(pairs, k=10)
    assert len(ca.top) == 10 and all(p == 0 for p, _ in ca.top)
    single = analyze(*pairs[0], k=10)
    assert [f for _, f in ca.top] == single.join.order.cpu().tolist()
