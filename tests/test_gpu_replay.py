"""GPU replay estimator (csrc/replay.cu) vs the reference's own replay
ledgers (tests/golden/replay.npz, recorded from diffwatt.energy.build_ledger
(method="replay")) -- bit-exact -- and vs the CPU oracle at larger sizes."""
import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

dw = pytest.importorskip("paper_2512_08365_b200")
from paper_2512_08365_b200 import SignalError, TraceColumns, build_ledger, replay_estimate  # noqa: E402


def _cases():
    z = np.load(GOLDEN / "replay.npz")
    for c in z["cases"]:
        for tag, kw in json.loads(str(z["settings"])):
            yield str(c), tag, kw


def _cols(z, c):
    return TraceColumns.from_arrays(z[f"{c}_ts"], z[f"{c}_watts"], z[f"{c}_op_start"], z[f"{c}_op_end"],
                                    z[f"{c}_k_start"], z[f"{c}_k_end"], z[f"{c}_k_op"],
                                    trace_end=int(max(z[f"{c}_span"][1] - 1, z[f"{c}_ts"][-1])),
                                    op_ids=[str(x) for x in z[f"{c}_op_ids"]],
                                    k_ids=[str(x) for x in z[f"{c}_k_ids"]])


@pytest.mark.parametrize("case,tag,kw", list(_cases()))
def test_replay_ledger_bit_exact_vs_reference(case, tag, kw):
    z = np.load(GOLDEN / "replay.npz")
    cols = _cols(z, case)
    assert cols.signal_span()[1] == z[f"{case}_span"][1]
    led = build_ledger(cols, method="replay", **kw)
    np.testing.assert_array_equal(led.per_operator.array(), z[f"{case}_{tag}_per_op"])
    np.testing.assert_array_equal(led.per_kernel.array(), z[f"{case}_{tag}_per_k"])
    total, idle = z[f"{case}_{tag}_total_idle"]
    assert led.total_joules == pytest.approx(total, rel=1e-12, abs=0)
    assert abs(led.idle_joules - idle) <= 1e-12 * total


def test_replay_estimate_api():
    z = np.load(GOLDEN / "replay.npz")
    cols = _cols(z, "demo")
    oid = str(z["demo_op_ids"][2])
    est = replay_estimate(cols, oid, seed=0)
    assert est.joules == z["demo_d_per_op"][2]
    assert est.repeat == 1000 and est.samples_used > 0
    with pytest.raises(KeyError):
        replay_estimate(cols, "nope")
    with pytest.raises(SignalError, match="repeat"):
        replay_estimate(cols, oid, repeat=0)


def test_replay_requires_kernels():
    z = np.load(GOLDEN / "replay.npz")
    c = "demo"
    keep = z[f"{c}_k_op"] != 0  # op 0 loses its kernels
    cols = TraceColumns.from_arrays(z[f"{c}_ts"], z[f"{c}_watts"], z[f"{c}_op_start"], z[f"{c}_op_end"],
                                    z[f"{c}_k_start"][keep], z[f"{c}_k_end"][keep], z[f"{c}_k_op"][keep],
                                    trace_end=int(max(z[f"{c}_span"][1] - 1, z[f"{c}_ts"][-1])),
                                    op_ids=[str(x) for x in z[f"{c}_op_ids"]])
    with pytest.raises(SignalError, match="no kernels"):
        build_ledger(cols, method="replay")


@pytest.mark.parametrize("kw", [dict(), dict(repeat=37, period_us=700, delay_us=90, seed=3),
                                dict(delay_us=0, period_us=1000, repeat=200)])
def test_replay_vs_oracle_at_scale(kw):
    """A C2-shaped trace (thousands of ops): bit-exact against the oracle."""
    from paper_2512_08365_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["C2"], 20_000)
    a, _ = synth.make_pair(cfg)
    led = build_ledger(a, method="replay", **kw)
    args = {"repeat": 1000, "period_us": 40_000, "delay_us": 200_000, "seed": 0, **kw}
    watts, joules = oracle.replay(a.host("ts"), a.host("watts"), a.signal_span()[1], a.host("op_start"),
                                  a.host("op_end"), **args)
    np.testing.assert_array_equal(led.per_operator.array(), joules)
    kdur = a.host("k_end") - a.host("k_start")
    np.testing.assert_array_equal(led.per_kernel.array(), watts[a.host("k_op")] * kdur / 1_000_000)
