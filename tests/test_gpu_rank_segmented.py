"""Segmented top-k (csrc/diff.cu dw_rank_segmented): the report
order of every trace pair of a corpus in one call.  Each segment must equal
the oracle's order of that segment alone (oracle.rank: the reference's
sorted(key=(verdict != waste, -wasted, nodes_a)), detect.py:263-266) and its
exact waste sum; empty segments, segments shorter than k, heavy ties and the
join's implicit low key (tie rank / B-only numbering) included."""

import numpy as np
import pytest
import torch

import oracle
from paper_2512_08365_b200 import detect as D

pytestmark = pytest.mark.gpu


def _segment(rng, P, ties):
    wasted = rng.exponential(1.0, size=P)
    if ties:
        wasted = np.round(wasted, 1)
        wasted[rng.random(P) < 0.3] = 0.0
    verdict = rng.choice([0, 1, 2], size=P, p=[0.7, 0.2, 0.1]).astype(np.int8)
    tie = rng.integers(0, P // 3 + 1, size=P)
    bits = wasted.view(np.uint64) & np.uint64(0x7FFFFFFFFFFFFFFF)
    hi = bits | ((verdict == 2).astype(np.uint64) << np.uint64(63))
    lo = ~(((tie.astype(np.uint64) + np.uint64(1)) << np.uint64(32)) | np.arange(P, dtype=np.uint64))
    return wasted, verdict, tie, hi, lo


@pytest.mark.parametrize("k", [1, 100, 4000])
def test_segments_match_oracle(k):
    rng = np.random.default_rng(k)
    sizes = [0, 5, 1000, 250_000, 1_000_000, 37, 120_000]
    dev = torch.device("cuda")
    segs, refs = [], []
    for i, P in enumerate(sizes):
        wasted, verdict, tie, hi, lo = _segment(rng, P, ties=i % 2 == 1)
        refs.append((oracle.rank(verdict, wasted, tie) if P else np.zeros(0, dtype=np.int64), wasted, verdict))
        segs.append((torch.from_numpy(hi.view(np.int64)).to(dev), torch.from_numpy(lo.view(np.int64)).to(dev),
                     None, 0))
    order, summary = D.rank_order_segmented(segs, k)
    order, summary = order.cpu().numpy(), summary.cpu().numpy()
    for i, (ref, wasted, verdict) in enumerate(refs):
        n = min(k, sizes[i])
        np.testing.assert_array_equal(order[i, :n], ref[:n], err_msg=f"segment {i}")
        assert (order[i, n:] == -1).all()
        assert summary[i, 0] == (verdict == 2).sum()
        assert summary[i, 1] == (oracle.fx_sum(wasted[verdict == 2]) if sizes[i] else 0.0)
        assert summary[i, 2] == sizes[i]


def test_segments_equal_single_rank_with_join_numbering():
    """Implicit low keys (no key_lo column): A findings tie on their op's id
    rank, B-only findings after n_a sort first among equal keys."""
    rng = np.random.default_rng(7)
    dev = torch.device("cuda")
    segs, singles = [], []
    for P, n_a in ((300_000, 250_000), (50_000, 50_000), (10, 3)):
        wasted, verdict, _, hi, _ = _segment(rng, P, ties=True)
        rank = torch.from_numpy(rng.permutation(n_a).astype(np.int64)).to(dev)
        khi = torch.from_numpy(hi.view(np.int64)).to(dev)
        segs.append((khi, None, rank, n_a))
        singles.append(D.rank_order(khi, None, min(100, P), tie_rank=rank, n_a=n_a))
    order, summary = D.rank_order_segmented(segs, 100)
    for i, (o1, s1) in enumerate(singles):
        n = o1.numel()
        torch.testing.assert_close(order[i, :n], o1, rtol=0, atol=0)
        torch.testing.assert_close(summary[i, :3], s1[:3], rtol=0, atol=0)


def test_segmented_rejects_large_k():
    dev = torch.device("cuda")
    hi = torch.zeros(10, dtype=torch.int64, device=dev)
    from paper_2512_08365_b200._native import NativeError
    with pytest.raises(NativeError):
        D.rank_order_segmented([(hi, None, None, 10)], 9000)
