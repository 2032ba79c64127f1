"""GPU parity: libdwb200 attribution vs the reference's golden vectors and the
CPU oracle.  Bit-exact wherever the interval spans <= DW_DIRECT_MAX segments
(the reference's own sequential fp64 sum); the fixed-point path for longer
intervals is bit-exact against the oracle's MODE_DEVICE and within 1e-12
relative of the reference."""
import json

import numpy as np
import pytest
import torch

import oracle
from conftest import GOLDEN, load_scenario, scenario_names

pytestmark = pytest.mark.gpu

dw = pytest.importorskip("paper_2512_08365_b200")
from paper_2512_08365_b200 import PowerSignal, SignalError, TraceColumns, build_ledger  # noqa: E402
from paper_2512_08365_b200 import energy as E  # noqa: E402
from paper_2512_08365_b200.trace_model import TraceError  # noqa: E402


def _signals(g, with_span):
    for s in range(len(g["sig_off"]) - 1):
        sl = slice(g["sig_off"][s], g["sig_off"][s + 1])
        iv = slice(g["iv_off"][s], g["iv_off"][s + 1])
        span_hi = int(g["span"][s][1]) if with_span else None
        yield g["ts"][sl], g["watts"][sl], span_hi, g["lo"][iv], g["hi"][iv], g["joules"][iv]


def _nseg(ts, lo, hi):
    a = np.searchsorted(ts, lo, side="right") - 1
    b = np.searchsorted(ts, hi, side="left") - 1
    return np.where(hi > lo, b - a + 1, 0)


def test_step_golden(golden_step):
    for ts, w, span_hi, lo, hi, ref in _signals(golden_step, True):
        sig = PowerSignal.from_columns(ts, w, span_hi, "step")
        got = E.integrate_many(sig, lo, hi).cpu().numpy()
        short = _nseg(ts, lo, hi) <= oracle.DW_DIRECT_MAX
        np.testing.assert_array_equal(got[short], ref[short])
        np.testing.assert_allclose(got[~short], ref[~short], rtol=1e-12, atol=0)
        np.testing.assert_array_equal(
            got, oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_DEVICE))


def test_linear_golden(golden_linear):
    for ts, w, _, lo, hi, ref in _signals(golden_linear, False):
        sig = PowerSignal.from_columns(ts, w, kind="linear")
        got = E.integrate_many(sig, lo, hi).cpu().numpy()
        dev = oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_DEVICE)
        np.testing.assert_array_equal(got, dev)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-300)


def _cols(sc, side):
    return TraceColumns.from_arrays(
        sc[f"{side}_ts"], sc[f"{side}_watts"], sc[f"{side}_op_start"], sc[f"{side}_op_end"],
        sc[f"{side}_k_start"], sc[f"{side}_k_end"], sc[f"{side}_k_op"],
        trace_end=int(max(sc[f"{side}_span"][1] - 1, sc[f"{side}_ts"][-1])),
        op_ids=[str(x) for x in sc[f"{side}_op_ids"]], k_ids=[str(x) for x in sc[f"{side}_k_ids"]])


@pytest.mark.parametrize("name", scenario_names())
def test_ledger_golden(name):
    sc = load_scenario(name)
    for side in ("a", "b"):
        cols = _cols(sc, side)
        assert cols.signal_span()[1] == sc[f"{side}_span"][1]
        led = build_ledger(cols)
        np.testing.assert_array_equal(led.per_operator.array(), sc[f"gt_{side}_per_op"])
        np.testing.assert_array_equal(led.per_kernel.array(), sc[f"gt_{side}_per_k"])
        total, idle = sc[f"gt_{side}_total_idle"]
        assert led.total_joules == pytest.approx(total, rel=1e-12, abs=0)
        assert abs(led.idle_joules - idle) <= 1e-12 * total
        for tag, period, delay in (("s40", 40_000, 200_000), ("s1", 1_000, 0)):
            if f"{tag}_{side}_per_op" not in sc:
                continue
            view = E.sampled_view(cols, period, delay, 0)
            np.testing.assert_array_equal(E._host(view._ts), sc[f"{tag}_{side}_view_ts"])
            np.testing.assert_array_equal(E._host(view._w), sc[f"{tag}_{side}_view_watts"])
            led = build_ledger(cols, method="sampled", period_us=period, delay_us=delay, seed=0)
            np.testing.assert_array_equal(led.per_operator.array(), sc[f"{tag}_{side}_per_op"])
            np.testing.assert_array_equal(led.per_kernel.array(), sc[f"{tag}_{side}_per_k"])
            total, idle = sc[f"{tag}_{side}_total_idle"]
            assert led.total_joules == pytest.approx(total, rel=1e-12, abs=0)
            assert abs(led.idle_joules - idle) <= 1e-12 * total


def test_error_messages_match_reference():
    with open(GOLDEN / "errors.json") as fh:
        msgs = json.load(fh)
    sig = PowerSignal(segments=((10, 100, 50.0), (100, 150, 70.0)))
    for name, iv in (("outside_lo", (0, 100)), ("outside_hi", (20, 151)), ("reversed", (60, 50))):
        with pytest.raises(SignalError) as ei:
            E.integrate(sig, iv)
        assert str(ei.value) == msgs[name]
    with pytest.raises(SignalError) as ei:
        PowerSignal().span()
    assert str(ei.value) == msgs["empty"]


def test_ledger_reports_first_bad_interval_in_reference_order():
    ts = np.array([100, 200, 300], dtype=np.int64)
    w = np.array([10.0, 20.0, 30.0])
    # op 1's kernel is bad, op 2 is bad: the kernel (visited first) is reported
    cols = TraceColumns.from_arrays(ts, w, np.array([100, 150, 250]), np.array([140, 260, 290]),
                                    np.array([110, 149, 255]), np.array([120, 160, 280]),
                                    np.array([0, 1, 2], dtype=np.int32), trace_end=300)
    led = build_ledger(cols)
    assert led.per_operator.array().shape == (3,)
    bad = TraceColumns.from_arrays(ts, w, np.array([100, 150, 250]), np.array([140, 260, 240]),
                                   np.array([110, 90, 255]), np.array([120, 160, 280]),
                                   np.array([0, 1, 2], dtype=np.int32), trace_end=300)
    with pytest.raises(SignalError, match=r"interval \[90,160\] outside signal span \[100,301\]"):
        build_ledger(bad)
    bad2 = TraceColumns.from_arrays(ts, w, np.array([100, 150, 250]), np.array([140, 140, 290]),
                                    np.array([110, 150, 255]), np.array([120, 160, 280]),
                                    np.array([0, 1, 2], dtype=np.int32), trace_end=300)
    with pytest.raises(SignalError, match="interval end precedes start"):
        build_ledger(bad2)


def test_power_order_validated():
    ts = np.array([100, 200, 200, 300], dtype=np.int64)
    cols = TraceColumns.from_arrays(ts, np.ones(4), np.array([100]), np.array([150]))
    with pytest.raises(TraceError, match="strictly increasing"):
        build_ledger(cols, validate_order=True)


def _random_case(seed, S, n, max_len, dense=False):
    rng = np.random.default_rng(seed)
    gaps = rng.integers(1, 4 if dense else 300, size=S)
    ts = np.cumsum(gaps).astype(np.int64)
    w = rng.uniform(50, 900, size=S)
    span_hi = int(ts[-1]) + int(rng.integers(1, 500))
    lo = np.sort(rng.integers(ts[0], span_hi, size=n))
    ln = (rng.pareto(1.2, size=n) * max_len / 20).astype(np.int64)
    hi = np.minimum(lo + ln, span_hi)
    return ts, w, span_hi, lo, hi


@pytest.mark.parametrize("seed,S,n,max_len", [(1, 300_000, 200_000, 3000), (2, 2_000_001, 500_000, 40_000),
                                              (3, 5000, 100_000, 100)])
def test_random_step_vs_oracle(seed, S, n, max_len):
    ts, w, span_hi, lo, hi = _random_case(seed, S, n, max_len)
    sig = PowerSignal.from_columns(ts, w, span_hi, "step")
    got = E.integrate_many(sig, lo, hi).cpu().numpy()
    np.testing.assert_array_equal(got, oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_DEVICE))
    ref = oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_REFERENCE)
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=0)


@pytest.mark.parametrize("seed,S,n,max_len", [(4, 300_000, 200_000, 3000), (5, 1_000_003, 300_000, 20_000)])
def test_random_linear_vs_oracle(seed, S, n, max_len):
    ts, w, span_hi, lo, hi = _random_case(seed, S, n, max_len)
    hi = np.minimum(hi, ts[-1])
    lo = np.minimum(lo, hi)
    sig = PowerSignal.from_columns(ts, w, kind="linear")
    got = E.integrate_many(sig, lo, hi).cpu().numpy()
    np.testing.assert_array_equal(got, oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_DEVICE))


def test_linear_total_device_definition():
    ts, w, span_hi, lo, hi = _random_case(9, 300_000, 1000, 500)
    sig = E.PowerSignal.from_columns(ts, w, kind="linear")
    cols = TraceColumns.from_arrays(ts, w, np.minimum(lo, ts[-1]), np.minimum(hi, ts[-1]),
                                    trace_end=int(ts[-1]))
    led = build_ledger(cols, method="ground_truth")
    assert led.total_joules == oracle.total_device("step", ts, w, int(ts[-1]) + 1)
    from paper_2512_08365_b200.energy import _run_ledger
    _, _, st = _run_ledger(cols, sig, False)
    assert st.totals[0] == oracle.total_device("linear", ts, w)
    ref = oracle.integrate_linear(ts, w, [ts[0]], [ts[-1]], oracle.MODE_REFERENCE)[0]
    assert st.totals[0] == pytest.approx(ref, rel=1e-12)


def test_unsorted_sets_match_sorted():
    ts, w, span_hi, lo, hi = _random_case(7, 100_000, 50_000, 2000)
    perm = np.random.default_rng(0).permutation(lo.size)
    sig = PowerSignal.from_columns(ts, w, span_hi, "step")
    a = E.integrate_many(sig, lo, hi).cpu().numpy()
    b = E.integrate_many(sig, lo[perm], hi[perm]).cpu().numpy()
    np.testing.assert_array_equal(a[perm], b)


def test_ledger_total_long_and_idle():
    ts, w, span_hi, lo, hi = _random_case(8, 200_000, 20_000, 500)
    cols = TraceColumns.from_arrays(ts, w, lo, hi, trace_end=span_hi - 1)
    led = build_ledger(cols)
    assert led.total_joules == oracle.total_device("step", ts, w, cols.signal_span()[1])
    sh = cols.signal_span()[1]
    ref_total = oracle.integrate_step(ts, w, sh, [ts[0]], [sh], oracle.MODE_REFERENCE)[0]
    assert led.total_joules == pytest.approx(ref_total, rel=1e-12)
    assert led.operator_total() == oracle.fx_sum(led.per_operator.array())
    assert led.idle_joules == max(led.total_joules - led.operator_total(), 0.0)


def test_ledger_of_loaded_trace_file_matches_golden():
    from paper_2512_08365_b200 import load_trace
    tr = load_trace(str(GOLDEN / "traces" / "tf32_misconfig" / "trace_a.jsonl"))
    led = build_ledger(tr)
    sc = load_scenario("preset_tf32_misconfig")
    want = dict(zip((str(x) for x in sc["a_op_ids"]), sc["gt_a_per_op"]))
    assert {k: led.per_operator[k] for k in want} == want


def test_config1_golden():
    """BASELINE config 1 (10,142 ops per side): ground truth ledgers bit-exact,
    the 1 kHz sampled view and its first 500 op / kernel integrals bit-exact."""
    sc = load_scenario("cfg1")
    for side in ("a", "b"):
        cols = _cols(sc, side)
        led = build_ledger(cols)
        np.testing.assert_array_equal(led.per_operator.array(), sc[f"gt_{side}_per_op"])
        np.testing.assert_array_equal(led.per_kernel.array(), sc[f"gt_{side}_per_k"])
        total, idle = sc[f"gt_{side}_total_idle"]
        assert led.total_joules == pytest.approx(total, rel=1e-12)
        assert abs(led.idle_joules - idle) <= 1e-12 * total
        view = E.sampled_view(cols, 1_000, 0, 0)
        np.testing.assert_array_equal(E._host(view._ts), sc[f"s1_{side}_view_ts"])
        np.testing.assert_array_equal(E._host(view._w), sc[f"s1_{side}_view_watts"])
        lin = build_ledger(cols, method="sampled", period_us=1_000, delay_us=0)
        np.testing.assert_array_equal(lin.per_operator.array()[:500], sc[f"s1_{side}_per_op500"])
        np.testing.assert_array_equal(lin.per_kernel.array()[:500], sc[f"s1_{side}_per_k500"])


# ------------------------------------------------- summation="exact" (DW_SUM_EXACT)
# Every interval is the exact sum of its pieces rounded to 2^-40 W*us, rounded
# once: bit-identical to the oracle's MODE_EXACT, within a few ulps of the
# reference's sequential sums (tolerance 1e-12 relative here; the north star
# asks 1e-6).  Each piece is rounded to 2^-40 W*us, so an interval's absolute
# error is at most (pieces / 2) * 2^-40 W*us = pieces * 4.5e-19 J: EXACT_ATOL
# covers intervals of up to ~200 pieces whose energy is too small for the
# relative bar (below ~1e-4 J the quantum dominates 1e-12 relative).
EXACT_ATOL = 1e-16  # J


@pytest.mark.parametrize("seed,S,n,max_len", [(11, 300_000, 200_000, 3000), (12, 2_000_001, 500_000, 40_000),
                                              (13, 5000, 100_000, 100)])
def test_exact_step_vs_oracle(seed, S, n, max_len):
    ts, w, span_hi, lo, hi = _random_case(seed, S, n, max_len)
    sig = PowerSignal.from_columns(ts, w, span_hi, "step")
    got = E.integrate_many(sig, lo, hi, summation="exact").cpu().numpy()
    np.testing.assert_array_equal(got, oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_EXACT))
    ref = oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_REFERENCE)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=EXACT_ATOL)


@pytest.mark.parametrize("seed,S,n,max_len", [(14, 300_000, 200_000, 3000), (15, 1_000_003, 300_000, 20_000)])
def test_exact_linear_vs_oracle(seed, S, n, max_len):
    ts, w, span_hi, lo, hi = _random_case(seed, S, n, max_len)
    hi = np.minimum(hi, ts[-1])
    lo = np.minimum(lo, hi)
    sig = PowerSignal.from_columns(ts, w, kind="linear")
    got = E.integrate_many(sig, lo, hi, summation="exact").cpu().numpy()
    np.testing.assert_array_equal(got, oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_EXACT))
    ref = oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_REFERENCE)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=EXACT_ATOL)


def test_exact_golden_vectors(golden_step, golden_linear):
    for ts, w, span_hi, lo, hi, ref in _signals(golden_step, True):
        got = E.integrate_many(PowerSignal.from_columns(ts, w, span_hi, "step"), lo, hi, summation="exact")
        got = got.cpu().numpy()
        np.testing.assert_array_equal(got, oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_EXACT))
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=EXACT_ATOL)
    for ts, w, _, lo, hi, ref in _signals(golden_linear, False):
        got = E.integrate_many(PowerSignal.from_columns(ts, w, kind="linear"), lo, hi, summation="exact")
        got = got.cpu().numpy()
        np.testing.assert_array_equal(got, oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_EXACT))
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=EXACT_ATOL)


@pytest.mark.parametrize("name", ["preset_tf32_misconfig", "preset_join_redundant", "fuzz_00", "cfg1"])
def test_exact_ledger_golden(name):
    sc = load_scenario(name)
    for side in ("a", "b"):
        cols = _cols(sc, side)
        led = build_ledger(cols, summation="exact")
        np.testing.assert_allclose(led.per_operator.array(), sc[f"gt_{side}_per_op"], rtol=1e-12, atol=EXACT_ATOL)
        np.testing.assert_allclose(led.per_kernel.array(), sc[f"gt_{side}_per_k"], rtol=1e-12, atol=EXACT_ATOL)
        ts, w = cols.host("ts"), cols.host("watts")
        span_hi = cols.signal_span()[1]
        po, pk, total, idle = oracle.ledger("step", ts, w, span_hi, cols.host("op_start"), cols.host("op_end"),
                                            cols.host("k_start"), cols.host("k_end"), oracle.MODE_EXACT)
        np.testing.assert_array_equal(led.per_operator.array(), po)
        np.testing.assert_array_equal(led.per_kernel.array(), pk)
        assert led.total_joules == total
        assert led.idle_joules == idle
        assert led.total_joules == pytest.approx(sc[f"gt_{side}_total_idle"][0], rel=1e-12)


def _wide_case(seed, kind):
    """Timestamps with gaps of more than 2^32 us (tile windows too wide for
    32-bit offsets: the kernels' int64 branch) between dense runs."""
    rng = np.random.default_rng(seed)
    gaps = rng.integers(1, 400, size=60_000)
    gaps[rng.integers(0, gaps.size, size=25)] = (1 << 32) + rng.integers(0, 1 << 20, size=25)
    ts = np.cumsum(gaps).astype(np.int64)
    w = rng.uniform(0.001, 2.0, size=ts.size)  # small watts: long gaps stay within the term range
    span_hi = int(ts[-1]) + 7
    top = span_hi if kind == "step" else int(ts[-1])
    lo = np.sort(rng.integers(ts[0], top, size=20_000))
    hi = np.minimum(lo + rng.integers(0, 3000, size=lo.size), top)
    # some intervals across a wide gap
    k = rng.integers(0, ts.size - 2, size=200)
    lo2, hi2 = ts[k] + 1, np.minimum(ts[k + 2] - 1, top)
    lo = np.concatenate([lo, np.minimum(lo2, hi2)])
    hi = np.concatenate([hi, hi2])
    o = np.argsort(lo, kind="stable")
    return ts, w, span_hi, lo[o], hi[o]


@pytest.mark.parametrize("summation,mode", [("reference", oracle.MODE_DEVICE), ("exact", oracle.MODE_EXACT)])
@pytest.mark.parametrize("kind", ["step", "linear"])
def test_wide_windows(kind, summation, mode):
    """Windows spanning >= 2^32 us take the int64 path (attribute.cu 'wide')."""
    ts, w, span_hi, lo, hi = _wide_case(31, kind)
    if kind == "step":
        got = E.integrate_many(PowerSignal.from_columns(ts, w, span_hi, "step"), lo, hi, summation=summation)
        want = oracle.integrate_step(ts, w, span_hi, lo, hi, mode)
        ref = oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_REFERENCE)
    else:
        got = E.integrate_many(PowerSignal.from_columns(ts, w, kind="linear"), lo, hi, summation=summation)
        want = oracle.integrate_linear(ts, w, lo, hi, mode)
        ref = oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_REFERENCE)
    got = got.cpu().numpy()
    np.testing.assert_array_equal(got, want)
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-300)


@pytest.mark.parametrize("kind", ["step", "linear"])
def test_exact_huge_pieces_take_the_long_path(kind):
    """Pieces above 2^23 W*us (beyond the two-instruction rounding) and
    intervals whose bound exceeds the 64-bit window prefix go through the
    int128 long-interval kernel: still the oracle's MODE_EXACT bit for bit."""
    rng = np.random.default_rng(5)
    ts = np.cumsum(rng.integers(1, 50_000, size=40_000)).astype(np.int64)
    w = rng.uniform(1.0, 1500.0, size=ts.size)
    span_hi = int(ts[-1]) + 3
    top = span_hi if kind == "step" else int(ts[-1])
    lo = np.sort(rng.integers(ts[0], top, size=30_000))
    hi = np.minimum(lo + rng.integers(0, 200_000, size=lo.size), top)
    if kind == "step":
        got = E.integrate_many(PowerSignal.from_columns(ts, w, span_hi, "step"), lo, hi, summation="exact")
        want = oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_EXACT)
    else:
        got = E.integrate_many(PowerSignal.from_columns(ts, w, kind="linear"), lo, hi, summation="exact")
        want = oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_EXACT)
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def test_exact_ledger_total_and_idle():
    ts, w, span_hi, lo, hi = _random_case(18, 200_000, 20_000, 500)
    cols = TraceColumns.from_arrays(ts, w, lo, hi, trace_end=span_hi - 1)
    led = build_ledger(cols, summation="exact")
    sh = cols.signal_span()[1]
    assert led.total_joules == oracle.total_device("step", ts, w, sh, exact=True)
    assert led.operator_total() == oracle.fx_sum(led.per_operator.array())
    assert led.idle_joules == max(led.total_joules - led.operator_total(), 0.0)
    ref = build_ledger(cols)  # the long span total is the same exact sum in both modes
    assert led.total_joules == ref.total_joules


def test_mean_power_matches_reference_rule():
    """mean_power (energy.py:133-137): integrate * 1e6 / (hi - lo); 0 for an
    empty or reversed interval; errors as integrate."""
    sig = PowerSignal(segments=((0, 5000, 100.0), (5000, 10000, 300.0)))
    assert E.mean_power(sig, (0, 10000)) == 2.0 * 1e6 / 10000
    assert E.mean_power(sig, (0, 5000)) == 100.0
    assert E.mean_power(sig, (7000, 7000)) == 0.0
    assert E.mean_power(sig, (7000, 6000)) == 0.0
    with pytest.raises(SignalError, match="outside"):
        E.mean_power(sig, (0, 10001))
    rng = np.random.default_rng(3)
    ts = np.cumsum(rng.integers(1, 300, size=5000)).astype(np.int64)
    w = rng.uniform(50, 700, size=ts.size)
    lin = PowerSignal.from_columns(ts, w, kind="linear")
    for lo, hi in ((int(ts[10]) + 3, int(ts[400]) - 1), (int(ts[0]), int(ts[-1]))):
        j = oracle.integrate_linear(ts, w, [lo], [hi], oracle.MODE_DEVICE)[0]
        assert E.mean_power(lin, (lo, hi)) == j * 1e6 / (hi - lo)


def test_analyze_raises_ledger_errors_first():
    """pipeline.analyze launches both ledgers and the pairing before it reads
    any ledger status: a data error still comes from trace A before trace B,
    and before the pairing's own errors (no signatures here)."""
    from paper_2512_08365_b200.pipeline import analyze
    ts = np.array([100, 200, 300], dtype=np.int64)
    w = np.array([10.0, 20.0, 30.0])

    def cols(k_start):
        return TraceColumns.from_arrays(ts, w, np.array([100, 150, 250]), np.array([140, 260, 290]),
                                        np.array(k_start), np.array([120, 160, 280]),
                                        np.array([0, 1, 2], dtype=np.int32), trace_end=300)
    good, bad_a, bad_b = cols([110, 150, 255]), cols([110, 90, 255]), cols([110, 150, 20])
    with pytest.raises(SignalError, match=r"interval \[90,160\]"):
        analyze(bad_a, bad_b)
    with pytest.raises(SignalError, match=r"interval \[20,280\]"):
        analyze(good, bad_b)
    with pytest.raises(ValueError, match="signatures"):
        analyze(good, good)
