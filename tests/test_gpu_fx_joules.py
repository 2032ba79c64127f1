"""Exact joule sums (dw_fx_sum_exact / fx_sum_kernel, dw_rank's waste sum):
every value converts to 2^-64 J fixed point rounded half to even, whichever of
fx_joules' three paths (|x| < 0.5, [0.5, 2^10), beyond) it takes.  Checked one
value at a time against exact rational arithmetic at the path boundaries,
ties, subnormals and negatives, and as sums against the oracle's fx_sum."""

from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
from paper_2512_08365_b200 import detect as D
from paper_2512_08365_b200.shard import _fx_exact

pytestmark = pytest.mark.gpu

TWO64 = 2 ** 64


def _edge_values():
    v = [0.0, -0.0, 5e-324, 2.0 ** -1022, 2.0 ** -64, 2.0 ** -65, 3 * 2.0 ** -66, 1.5 * 2.0 ** -64,
         2.5 * 2.0 ** -64, 0.5, np.nextafter(0.5, 0), np.nextafter(0.5, 1), 1024.0, np.nextafter(1024.0, 0),
         np.nextafter(1024.0, 2048), 1.0, 0.1, 0.3, 123.456, 1e6, 3.0e15, 2.0 ** 62, 1.0 - 2.0 ** -53]
    v += [-x for x in v if x > 0]
    rng = np.random.default_rng(5)
    v += list(rng.uniform(0, 1, 200) * 10.0 ** rng.integers(-20, 12, 200))
    return [float(x) for x in v]


def _exact(x: float) -> int:
    return round(Fraction(x) * TWO64)  # Fraction rounds half to even


def _as_int(pair) -> int:
    lo, hi = (int(t) & (TWO64 - 1) for t in pair)
    v = (hi << 64) | lo
    return v - (1 << 128) if v >> 127 else v


@pytest.mark.parametrize("x", _edge_values())
def test_single_value_rounds_half_even(x):
    got = _as_int(_fx_exact(torch.tensor([x], dtype=torch.float64, device="cuda")).cpu().tolist())
    assert got == _exact(x)


def test_sums_equal_oracle_across_paths():
    rng = np.random.default_rng(11)
    for n in (1, 1000, 300_001, 4_000_000):
        x = rng.uniform(0, 1, n) * 10.0 ** rng.integers(-6, 6, n)
        x[rng.random(n) < 0.01] *= -1
        got = _as_int(_fx_exact(torch.from_numpy(x).cuda()).cpu().tolist())
        if n <= 1000:
            assert got == sum(_exact(float(t)) for t in x)
        assert float(Fraction(got, TWO64)) == oracle.fx_sum(x)


def test_waste_sum_and_histogram_across_paths():
    """dw_rank's waste pass: exact wasted sum and waste count whatever the
    magnitudes (all three conversion paths), and the first-digit histogram's
    warp-aggregated counts leave the top-k order intact."""
    rng = np.random.default_rng(12)
    for P, spread, k in ((5000, 0, 100), (1_000_003, 6, 1000), (2_000_000, 0, 100)):
        wasted = rng.exponential(1.0, size=P) * (10.0 ** rng.integers(-spread, spread + 1, P) if spread else 1.0)
        verdict = rng.choice([0, 1, 2], size=P, p=[0.5, 0.2, 0.3]).astype(np.int8)
        tie = rng.integers(0, P // 2, size=P)
        order_ref = oracle.rank(verdict, wasted, tie)
        bits = wasted.view(np.uint64) & np.uint64(0x7FFFFFFFFFFFFFFF)
        hi = bits | ((verdict == 2).astype(np.uint64) << np.uint64(63))
        lo = ~(((tie.astype(np.uint64) + np.uint64(1)) << np.uint64(32)) | np.arange(P, dtype=np.uint64))
        order, summary = D.rank_order(torch.from_numpy(hi.view(np.int64)).cuda(),
                                      torch.from_numpy(lo.view(np.int64)).cuda(), k)
        np.testing.assert_array_equal(order.cpu().numpy(), order_ref[:k])
        s = summary.cpu().numpy()
        assert s[0] == (verdict == 2).sum()
        assert s[1] == oracle.fx_sum(wasted[verdict == 2])
