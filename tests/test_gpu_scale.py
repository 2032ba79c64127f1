"""Parity at the benchmarked scales.

The headline numbers come from bench.py's C4 step: both ledgers (trapezoid
over the given power samples, summation="exact"), the signature join with
its finding columns, and the ranked top-k.  These tests run that same path at
the full C2 (1M ops per trace) and C3 (10M ops, four concurrent streams)
sizes and on a 5M-op pair drawn from the C4 distribution, and compare every
stage with the CPU oracle (oracle/dw_oracle.c) on the same inputs:

  * ledgers: bit-identical to the oracle's MODE_EXACT (summation="exact") and
    MODE_DEVICE (summation="reference"); within 1e-12 relative of the
    reference-order sums (MODE_REFERENCE) -- the north star's bar is 1e-6;
  * join: match_a / b_only bit-identical (multi-bucket partner staging: at
    these sizes the pairing runs over 1-10 of its 1M-op buckets);
  * findings: every column bit-identical, the top-k report order identical,
    the waste count and the exact wasted sum identical;
  * pipeline.analyze (the bench's public entry point, key-only findings):
    the same top-k findings, totals and wasted joules.
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

from paper_2512_08365_b200 import build_ledger, join_diff, synth  # noqa: E402
from paper_2512_08365_b200.pipeline import analyze  # noqa: E402


def oracle_join(ca, cb, ja, jb, theta, k):
    """The oracle's join + detect + report order over the same columns
    (vectorised CSR, as bench.py's cpu_step builds it)."""
    sig_a = ca.host("op_sig").view(np.uint64)
    sig_b = cb.host("op_sig").view(np.uint64)
    ma, mb = oracle.join(sig_a, sig_b)
    na = len(ma)
    b_only = np.nonzero(mb < 0)[0]
    off_a = np.concatenate([np.arange(na + 1), np.full(len(b_only), na)]).astype(np.int64)
    mem_a = np.arange(na, dtype=np.int32)
    has_b = (ma >= 0).astype(np.int64)
    off_b = np.concatenate([[0], np.cumsum(has_b), has_b.sum() + np.arange(1, len(b_only) + 1)]).astype(np.int64)
    mem_b = np.concatenate([ma[ma >= 0], b_only]).astype(np.int32)
    d = oracle.detect(off_a, mem_a, off_b, mem_b, ja, jb, ca.host("op_start"), ca.host("op_end"),
                      cb.host("op_start"), cb.host("op_end"), None, theta)
    tie = np.concatenate([np.arange(na) + 1, np.zeros(len(b_only), dtype=np.int64)])
    order = oracle.rank(d["verdict"], d["wasted"], tie)[:k]
    return ma, b_only, d, order


def oracle_ledger(c, mode):
    return oracle.ledger("linear", c.host("ts"), c.host("watts"), None, c.host("op_start"), c.host("op_end"),
                         c.host("k_start"), c.host("k_end"), mode)


def check_ledger(c, led, mode):
    po, pk, total, idle = oracle_ledger(c, mode)
    np.testing.assert_array_equal(led.per_operator.array(), po)
    np.testing.assert_array_equal(led.per_kernel.array(), pk)
    assert led.total_joules == total
    assert led.idle_joules == idle
    return po, pk


def run_scale(cfg, theta=0.10, k=1000, reference_too=False):
    ca, cb = synth.make_pair(cfg)
    la = build_ledger(ca, method="samples", summation="exact")
    lb = build_ledger(cb, method="samples", summation="exact")
    ja, _ = check_ledger(ca, la, oracle.MODE_EXACT)
    jb, _ = check_ledger(cb, lb, oracle.MODE_EXACT)
    # the exact sums against the reference's own sequential order
    ref_a = oracle_ledger(ca, oracle.MODE_REFERENCE)
    np.testing.assert_allclose(ja, ref_a[0], rtol=1e-12, atol=1e-300)
    if reference_too:
        rl = build_ledger(ca, method="samples")
        check_ledger(ca, rl, oracle.MODE_DEVICE)
    jd = join_diff(ca, cb, la, lb, theta, k)
    ma, b_only, d, order = oracle_join(ca, cb, ja, jb, theta, k)
    np.testing.assert_array_equal(jd.match_a.cpu().numpy(), ma)
    np.testing.assert_array_equal(jd.b_only.cpu().numpy(), b_only)
    h = jd.columns.host()
    P = jd.P
    assert P == len(ma) + len(b_only)
    np.testing.assert_array_equal(h["energy_a"][:P], d["energy"][:, 0])
    np.testing.assert_array_equal(h["energy_b"][:P], d["energy"][:, 1])
    np.testing.assert_array_equal(h["ratio"][:P], d["ratio"])
    np.testing.assert_array_equal(h["verdict"][:P], d["verdict"])
    np.testing.assert_array_equal(h["side"][:P], d["side"])
    np.testing.assert_array_equal(h["wasted"][:P], d["wasted"])
    np.testing.assert_array_equal(jd.order.cpu().numpy(), order)
    waste = d["verdict"] == oracle.VERDICT_WASTE
    assert jd.n_waste == int(waste.sum()) > 0
    assert jd.wasted_joules == oracle.fx_sum(d["wasted"][waste])
    # the bench's public entry point (lean keys) gives the same report
    res = analyze(ca, cb, "samples", theta, k)
    assert res.join.order.cpu().numpy().tolist() == order.tolist()
    assert (res.join.n_waste, res.join.wasted_joules) == (jd.n_waste, jd.wasted_joules)
    assert res.report.total_a == la.total_joules and res.report.total_b == lb.total_joules
    top = res.report.findings
    assert [f.wasted_joules for f in top] == d["wasted"][order].tolist()
    assert [f.energy_a for f in top] == d["energy"][order, 0].tolist()
    return jd


def test_scale_C2_full():
    """C2 at full size: 1M ops per trace (decode-shaped), two join buckets."""
    jd = run_scale(synth.CONFIGS["C2"], reference_too=True)
    assert jd.n_a == 1_000_000


def test_scale_C3_full():
    """C3 at full size: 10M ops per trace on four concurrent streams
    (overlapping kernels), ten join buckets."""
    jd = run_scale(synth.CONFIGS["C3"], k=500)
    assert jd.n_a == 10_000_000


def test_scale_C4_distribution_5M():
    """A 5M-op / 50M-sample pair drawn from the C4 distribution (the bench's
    workload shape, 1/20 of its size)."""
    jd = run_scale(synth.scaled(synth.CONFIGS["C4"], 5_000_000, 50_000_000), k=2000)
    assert jd.n_a == 5_000_000


def test_scale_C3_split_vs_oracle():
    """C3's overlap-split ledger (concurrent kernels share the power) at 2M
    ops: bit-identical to the oracle's dwo_split."""
    ca, _ = synth.make_pair(synth.scaled(synth.CONFIGS["C3"], 2_000_000))
    led = build_ledger(ca, method="samples", overlap="split")
    ts, w = ca.host("ts"), ca.host("watts")
    np.testing.assert_array_equal(led.per_kernel.array(),
                                  oracle.split("linear", ts, w, None, ca.host("k_start"), ca.host("k_end")))
    np.testing.assert_array_equal(led.per_operator.array(),
                                  oracle.split("linear", ts, w, None, ca.host("op_start"), ca.host("op_end")))
