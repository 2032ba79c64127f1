"""Pin the CPU oracle (oracle/dw_oracle.c) to the reference's own outputs.

Golden vectors were recorded by running the reference package
(tests/golden/make_golden.py); every comparison in MODE_REFERENCE is bit-exact
because the oracle performs the reference's arithmetic in the reference's order.
"""
import numpy as np
import pytest

import oracle
from conftest import GOLDEN, load_scenario, pair_tuples, scenario_names


def _nsegs_step(ts, span_hi, lo, hi):
    a = np.searchsorted(ts, lo, side="right") - 1
    b = np.searchsorted(ts, hi, side="left") - 1
    return np.where(hi > lo, b - a + 1, 0)


def _signals(g, with_span):
    for s in range(len(g["sig_off"]) - 1):
        ts = g["ts"][g["sig_off"][s]:g["sig_off"][s + 1]]
        w = g["watts"][g["sig_off"][s]:g["sig_off"][s + 1]]
        sl = slice(g["iv_off"][s], g["iv_off"][s + 1])
        span_hi = g["span"][s][1] if with_span else None
        yield ts, w, span_hi, g["lo"][sl], g["hi"][sl], g["joules"][sl]


def test_step_oracle_bit_exact_vs_reference(golden_step):
    n = 0
    for ts, w, span_hi, lo, hi, ref in _signals(golden_step, True):
        got = oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_REFERENCE)
        np.testing.assert_array_equal(got, ref)
        n += len(lo)
    assert n > 500


def test_step_device_mode_within_1e12(golden_step):
    long_seen = 0
    for ts, w, span_hi, lo, hi, ref in _signals(golden_step, True):
        got = oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_DEVICE)
        nseg = _nsegs_step(ts, span_hi, lo, hi)
        short = nseg <= oracle.DW_DIRECT_MAX
        np.testing.assert_array_equal(got[short], ref[short])
        np.testing.assert_allclose(got[~short], ref[~short], rtol=1e-12, atol=0)
        long_seen += int((~short).sum())
    assert long_seen > 20  # the fixed-point path is exercised


def test_linear_oracle_bit_exact_vs_reference(golden_linear):
    for ts, w, _, lo, hi, ref in _signals(golden_linear, False):
        got = oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_REFERENCE)
        np.testing.assert_array_equal(got, ref)


def test_linear_device_mode_within_1e12(golden_linear):
    for ts, w, _, lo, hi, ref in _signals(golden_linear, False):
        got = oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_DEVICE)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-300)


def test_fixed_point_roundtrip():
    rng = np.random.default_rng(1)
    x = rng.uniform(0, 1e3, size=1000) * 10.0 ** rng.integers(-3, 12, size=1000)
    # a single value survives the q() / rounding round trip to 2^-32 W*us
    for v in x[:200]:
        got = oracle.fx_sum(np.array([v]))
        assert got == v  # 2^-64 J resolution: exact for these magnitudes
    s = oracle.fx_sum(x)
    assert s == pytest.approx(float(np.sum(x)), rel=1e-13)
    assert s == oracle.py_sum(x) or abs(s - oracle.py_sum(x)) <= 2 * np.spacing(s)


def test_py_sum_is_cpython_sum():
    rng = np.random.default_rng(7)
    for _ in range(2000):
        x = rng.uniform(0, 1, size=int(rng.integers(1, 40))) * 10.0 ** rng.integers(-8, 8)
        assert oracle.py_sum(x) == sum(x.tolist())


@pytest.mark.parametrize("name", scenario_names())
def test_ledger_bit_exact_vs_reference(name):
    sc = load_scenario(name)
    for side in ("a", "b"):
        per_op, per_k, total, idle = oracle.ledger(
            "step", sc[f"{side}_ts"], sc[f"{side}_watts"], sc[f"{side}_span"][1],
            sc[f"{side}_op_start"], sc[f"{side}_op_end"], sc[f"{side}_k_start"],
            sc[f"{side}_k_end"])
        np.testing.assert_array_equal(per_op, sc[f"gt_{side}_per_op"])
        np.testing.assert_array_equal(per_k, sc[f"gt_{side}_per_k"])
        assert (total, idle) == tuple(sc[f"gt_{side}_total_idle"])
        for tag in ("s40", "s1"):
            if f"{tag}_{side}_per_op" not in sc:
                continue
            per_op, per_k, total, idle = oracle.ledger(
                "linear", sc[f"{tag}_{side}_view_ts"], sc[f"{tag}_{side}_view_watts"], None,
                sc[f"{side}_op_start"], sc[f"{side}_op_end"], sc[f"{side}_k_start"],
                sc[f"{side}_k_end"])
            np.testing.assert_array_equal(per_op, sc[f"{tag}_{side}_per_op"])
            np.testing.assert_array_equal(per_k, sc[f"{tag}_{side}_per_k"])
            assert (total, idle) == tuple(sc[f"{tag}_{side}_total_idle"])


@pytest.mark.parametrize("name", scenario_names())
@pytest.mark.parametrize("tag,theta", [("det10", 0.10), ("det05", 0.05)])
def test_detect_and_rank_bit_exact_vs_reference(name, tag, theta):
    sc = load_scenario(name)
    d = oracle.detect(sc["pair_off_a"], sc["pair_mem_a"], sc["pair_off_b"], sc["pair_mem_b"],
                      sc["gt_a_per_op"], sc["gt_b_per_op"], sc["a_op_start"], sc["a_op_end"],
                      sc["b_op_start"], sc["b_op_end"], sc["pair_out_diff"], theta)
    np.testing.assert_array_equal(d["energy"], sc[f"{tag}_energy"])
    np.testing.assert_array_equal(d["ratio"], sc[f"{tag}_ratio"])
    np.testing.assert_array_equal(d["lat"], sc[f"{tag}_lat"])
    np.testing.assert_array_equal(d["verdict"], sc[f"{tag}_verdict"])
    np.testing.assert_array_equal(d["side"], sc[f"{tag}_side"])
    np.testing.assert_array_equal(d["wasted"], sc[f"{tag}_wasted"])
    np.testing.assert_array_equal(d["informational"], sc[f"{tag}_info"])
    tie = oracle.tuple_rank(pair_tuples(sc, "a"))
    order = oracle.rank(d["verdict"], d["wasted"], tie)
    np.testing.assert_array_equal(order, sc[f"{tag}_rank"])
    waste = [float(d["wasted"][i]) for i in order if d["verdict"][i] == oracle.VERDICT_WASTE]
    wasted = oracle.py_sum(waste) if waste else 0
    total_a, total_b, ref_wasted, ref_pct = sc[f"{tag}_report"]
    assert wasted == ref_wasted
    ineff = max(total_a, total_b)
    assert (wasted / ineff if ineff > 0 else 0.0) == ref_pct


def test_detect_threshold_rejected():
    with pytest.raises(ValueError, match="threshold"):
        oracle.detect([0], [], [0], [], [], [], [], [], [], [], None, 0.0)


def test_occurrence_and_join_definition():
    sig_a = np.array([5, 7, 5, 5, 9], dtype=np.uint64)
    sig_b = np.array([7, 5, 5, 11, 5, 5], dtype=np.uint64)
    np.testing.assert_array_equal(oracle.occurrence(sig_a), [0, 0, 1, 2, 0])
    ma, mb = oracle.join(sig_a, sig_b)
    np.testing.assert_array_equal(ma, [1, 0, 2, 4, -1])
    np.testing.assert_array_equal(mb, [1, 0, 2, -1, 3, -1])


# ------------------------------------------------ overlap split (G1) oracle

def test_split_g1_example():
    """ops [0,100) and [50,150) over 100 W then 300 W.  Compat
    double-counts (0.01 + 0.02 > 0.025 J total); split shares the overlap."""
    ts, w = np.array([0, 100]), np.array([100.0, 300.0])
    lo, hi = np.array([0, 50]), np.array([100, 150])
    np.testing.assert_array_equal(oracle.integrate_step(ts, w, 150, lo, hi, oracle.MODE_DEVICE), [0.01, 0.02])
    got = oracle.split("step", ts, w, 150, lo, hi)
    np.testing.assert_allclose(got, [0.0075, 0.0175], rtol=1e-15)
    assert got.sum() == pytest.approx(0.025, rel=1e-15)


@pytest.mark.parametrize("kind", ["step", "linear"])
def test_split_equals_compat_without_overlap(kind):
    from _split_cases import disjoint, signal
    rng = np.random.default_rng(7 if kind == "step" else 8)
    ts, w, span_hi = signal(rng, 3000, kind)
    lo, hi = disjoint(rng, ts, span_hi, 400)
    comp = (oracle.integrate_step(ts, w, span_hi, lo, hi, oracle.MODE_DEVICE) if kind == "step"
            else oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_DEVICE))
    np.testing.assert_array_equal(oracle.split(kind, ts, w, span_hi, lo, hi), comp)


@pytest.mark.parametrize("kind", ["step", "linear"])
def test_split_conserves_union_energy(kind):
    """Shares add up to the energy of the union of the set's intervals."""
    from _split_cases import overlapping, signal
    rng = np.random.default_rng(11)
    ts, w, span_hi = signal(rng, 2000, kind)
    lo, hi = overlapping(rng, ts, span_hi, 600)
    got = oracle.split(kind, ts, w, span_hi, lo, hi)
    order = np.argsort(lo, kind="stable")
    ulo, uhi = [], []
    for a, b in zip(lo[order], hi[order]):
        if b <= a:
            continue
        if ulo and a <= uhi[-1]:
            uhi[-1] = max(uhi[-1], b)
        else:
            ulo.append(a); uhi.append(b)
    f = (lambda x, y: oracle.integrate_step(ts, w, span_hi, x, y, oracle.MODE_DEVICE)) if kind == "step" \
        else (lambda x, y: oracle.integrate_linear(ts, w, x, y, oracle.MODE_DEVICE))
    union = f(np.array(ulo), np.array(uhi)).sum()
    assert got.sum() == pytest.approx(union, rel=1e-9)
    assert np.all(got >= 0)


# --------------------------------------------- replay estimator (golden)

def _replay_cases():
    import json
    z = np.load(GOLDEN / "replay.npz")
    settings = json.loads(str(z["settings"]))
    for c in z["cases"]:
        for tag, kw in settings:
            yield str(c), tag, kw


@pytest.mark.parametrize("case,tag,kw", list(_replay_cases()))
def test_replay_oracle_bit_exact_vs_reference(case, tag, kw):
    z = np.load(GOLDEN / "replay.npz")
    ts, w, span = z[f"{case}_ts"], z[f"{case}_watts"], z[f"{case}_span"]
    kw = {"repeat": 1000, "period_us": 40_000, "delay_us": 200_000, "seed": 0, **kw}
    watts, joules = oracle.replay(ts, w, span[1], z[f"{case}_op_start"], z[f"{case}_op_end"], **kw)
    np.testing.assert_array_equal(joules, z[f"{case}_{tag}_per_op"])
    kdur = z[f"{case}_k_end"] - z[f"{case}_k_start"]
    np.testing.assert_array_equal(watts[z[f"{case}_k_op"]] * kdur / 1_000_000, z[f"{case}_{tag}_per_k"])
