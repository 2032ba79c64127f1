"""Host-side logic (CPU): ranking tie-break, signatures, the dict views over
device columns, the synthetic generators' invariants and the CPU baseline path."""
import numpy as np
import pytest
import torch

import oracle
from paper_2512_08365_b200 import synth
from paper_2512_08365_b200.detect import tuple_rank
from paper_2512_08365_b200.energy import JoulesView
from paper_2512_08365_b200.join import signature_of


def test_tuple_rank_is_python_tuple_order():
    tuples = [("b",), ("a", "c"), (), ("a",), ("a", "c"), ("a", "b"), ("b",)]
    r = tuple_rank(tuples)
    order = sorted(range(len(tuples)), key=lambda i: (tuples[i], i))
    assert sorted(range(len(tuples)), key=lambda i: (r[i], i)) == order
    assert r[1] == r[4] and r[0] == r[6] and r[2] == 0
    np.testing.assert_array_equal(r, oracle.tuple_rank(tuples))


def test_signature_is_deterministic_and_field_sensitive():
    s = signature_of("aten::mm", (64, 32))
    assert s == signature_of("aten::mm", (64, 32))
    others = {signature_of("aten::mm", (64, 33)), signature_of("aten::bmm", (64, 32)),
              signature_of("aten::mm", (64, 32), "bfloat16"), signature_of("aten::mm", (64, 32), callsite="x")}
    assert s not in others and len(others) == 4
    assert 0 <= s < 2 ** 64


def test_joules_view_is_a_read_only_mapping():
    t = torch.tensor([1.5, 2.5, 3.0], dtype=torch.float64)
    v = JoulesView(["x", "y", "z"], t)
    assert list(v) == ["x", "y", "z"] and len(v) == 3
    assert v["y"] == 2.5 and "z" in v and "w" not in v
    assert dict(v) == {"x": 1.5, "y": 2.5, "z": 3.0}
    assert v == {"x": 1.5, "y": 2.5, "z": 3.0}
    assert sum(v.values()) == 7.0
    anon = JoulesView(None, t, "k")
    assert list(anon) == ["k0", "k1", "k2"] and anon["k2"] == 3.0


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4"])
def test_synthetic_pairs_are_well_formed(cfg):
    a, b = synth.make_pair(synth.scaled(synth.CONFIGS[cfg], 4000), device="cpu")
    for c in (a, b):
        assert bool((c.ts[1:] > c.ts[:-1]).all())
        assert int(c.ts[-1]) == c.trace_end or int(c.ts[-1]) <= c.trace_end
        ko = c.k_op.long()
        assert bool((c.k_start >= c.op_start[ko]).all() and (c.k_end <= c.op_end[ko]).all())
        assert bool((c.k_end > c.k_start).all()) and bool((c.op_end >= c.op_start).all())
        assert c.ops_sorted
        assert int(c.op_end.max()) <= int(c.ts[-1])  # samples cover every interval
    assert b.n_ops >= a.n_ops  # B = A + inserted operators
    # deterministic per seed
    a2, _ = synth.make_pair(synth.scaled(synth.CONFIGS[cfg], 4000), device="cpu")
    assert torch.equal(a.ts, a2.ts) and torch.equal(a.op_sig, a2.op_sig)


def test_cpu_baseline_step_runs():
    import argparse
    import bench
    args = argparse.Namespace(config="C4", method="samples", k=10, cpu_sample_ops=5000)
    r = bench.cpu_baseline(args)
    assert r["value"] > 0 and r["kind"] == "port" and r["cores"] >= 1


@pytest.mark.parametrize("theta", [0.10, 0.05, 1.0])
def test_host_judge_equals_oracle_detect(theta):
    """detect.judge (the host twin of the device verdict, used for the key-only
    join's top-k rows) against the oracle's detect on single-op pairs,
    including ties, zero energies, one-sided pairs and latency edges."""
    import numpy as np
    import oracle
    from paper_2512_08365_b200.detect import SIDES, VERDICTS, judge
    rng = np.random.default_rng(int(theta * 100))
    P = 3000
    ja = rng.uniform(0, 2, P)
    jb = ja * rng.choice([1.0, 1.04, 1.06, 1.11, 0.9, 0.5, 2.0], P)
    ja[::17] = 0.0
    jb[::23] = 0.0
    la = rng.integers(0, 1000, P)
    lb = la + rng.integers(-20, 20, P)
    lb = np.maximum(lb, 0)
    off = np.arange(P + 1)
    mem = np.arange(P, dtype=np.int32)
    zeros = np.zeros(P, dtype=np.int64)
    d = oracle.detect(off, mem, off, mem, ja, jb, zeros, la, zeros, lb, None, theta)
    for i in range(P):
        ratio, wasted, verdict, side, info = judge(float(ja[i]), float(jb[i]), int(la[i]), int(lb[i]), 0.0, theta)
        assert ratio == d["ratio"][i] or (np.isinf(ratio) and np.isinf(d["ratio"][i]))
        assert wasted == d["wasted"][i]
        assert VERDICTS.index(verdict) == d["verdict"][i]
        assert SIDES.index(side) == d["side"][i]
        assert info == d["informational"][i]
