"""GPU parity of the overlap-split mode (csrc/split.cu) against the CPU
oracle's restatement (oracle/dw_oracle.c dwo_split): bit-exact.  The mode has
no reference function; it must equal the compat path whenever
nothing overlaps, which is pinned against the reference's golden vectors."""
import numpy as np
import pytest

import oracle
from _split_cases import disjoint, overlapping, signal

pytestmark = pytest.mark.gpu

dw = pytest.importorskip("paper_2512_08365_b200")
from paper_2512_08365_b200 import PowerSignal, SignalError, TraceColumns, build_ledger  # noqa: E402
from paper_2512_08365_b200 import energy as E  # noqa: E402


def _sig(ts, w, span_hi, kind):
    return PowerSignal.from_columns(ts, w, span_hi if kind == "step" else None, kind)


def test_split_g1_example():
    ts, w = np.array([0, 100]), np.array([100.0, 300.0])
    got = E.integrate_split(_sig(ts, w, 150, "step"), np.array([0, 50]), np.array([100, 150])).cpu().numpy()
    np.testing.assert_array_equal(got, oracle.split("step", ts, w, 150, np.array([0, 50]), np.array([100, 150])))
    np.testing.assert_allclose(got, [0.0075, 0.0175], rtol=1e-15)


@pytest.mark.parametrize("kind", ["step", "linear"])
@pytest.mark.parametrize("seed,n,m", [(1, 50, 20), (2, 3000, 800), (3, 40000, 20000), (4, 5, 30)])
def test_split_bit_exact_vs_oracle(kind, seed, n, m):
    rng = np.random.default_rng(seed)
    ts, w, span_hi = signal(rng, n, kind)
    lo, hi = overlapping(rng, ts, span_hi, m)
    got = E.integrate_split(_sig(ts, w, span_hi, kind), lo, hi).cpu().numpy()
    np.testing.assert_array_equal(got, oracle.split(kind, ts, w, span_hi, lo, hi))


@pytest.mark.parametrize("kind", ["step", "linear"])
def test_split_equals_compat_without_overlap(kind):
    rng = np.random.default_rng(21)
    ts, w, span_hi = signal(rng, 20000, kind)
    lo, hi = disjoint(rng, ts, span_hi, 3000)
    sig = _sig(ts, w, span_hi, kind)
    np.testing.assert_array_equal(E.integrate_split(sig, lo, hi).cpu().numpy(),
                                  E.integrate_many(sig, lo, hi).cpu().numpy())


def test_split_long_slices_use_the_device_definition():
    """Slices spanning more than DW_DIRECT_MAX segments go through the exact
    fixed-point path, exactly as the oracle's MODE_DEVICE restates it."""
    rng = np.random.default_rng(5)
    ts, w, span_hi = signal(rng, 5000, "step")
    lo = np.array([ts[10], ts[100], ts[50]]); hi = np.array([ts[2000], ts[4000], ts[60]])
    got = E.integrate_split(_sig(ts, w, span_hi, "step"), lo, hi).cpu().numpy()
    np.testing.assert_array_equal(got, oracle.split("step", ts, w, span_hi, lo, hi))


def test_split_out_of_span_raises():
    ts, w = np.array([10, 20, 30]), np.array([1.0, 2.0, 3.0])
    with pytest.raises(SignalError, match="outside"):
        E.integrate_split(_sig(ts, w, 40, "step"), np.array([12, 0]), np.array([15, 100]))


@pytest.mark.parametrize("kind", ["ground_truth", "samples"])
def test_split_ledger_c3_shape(kind):
    """A C3-shaped trace (4 concurrent streams): split ledger vs the oracle,
    and operators + idle == total with no double counting."""
    from paper_2512_08365_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["C3"], 20000)
    ca, _ = synth.make_pair(cfg)
    led = build_ledger(ca, method=kind, overlap="split")
    comp = build_ledger(ca, method=kind)
    ts, w = ca.host("ts"), ca.host("watts")
    k = "step" if kind == "ground_truth" else "linear"
    span_hi = ca.signal_span()[1] if k == "step" else None
    np.testing.assert_array_equal(led.per_operator.array(),
                                  oracle.split(k, ts, w, span_hi, ca.host("op_start"), ca.host("op_end")))
    np.testing.assert_array_equal(led.per_kernel.array(),
                                  oracle.split(k, ts, w, span_hi, ca.host("k_start"), ca.host("k_end")))
    assert led.total_joules == comp.total_joules
    assert led.operator_total() <= led.total_joules * (1 + 1e-12)
    assert comp.operator_total() > led.operator_total()  # compat double-counts concurrent streams
    assert led.operator_total() + led.idle_joules == pytest.approx(led.total_joules, rel=1e-12)
