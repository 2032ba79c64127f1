"""Time-window sharding (paper_2512_08365_b200/shard.py):
every rank of the multi-GPU decomposition run in one process on one GPU
(loopback collectives) must reproduce the one-GPU ledger and join bit for
bit -- including intervals longer than DW_DIRECT_MAX that cross window edges
(K7 exact partial sums) and the totals (exact sums of per-rank shares)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

dw = pytest.importorskip("paper_2512_08365_b200")
from paper_2512_08365_b200 import TraceColumns, build_ledger, shard, synth  # noqa: E402
from paper_2512_08365_b200.join import join_diff  # noqa: E402


def _check_ledger(cols, method, world):
    full = build_ledger(cols, method=method)
    kind = "step" if method == "ground_truth" else "linear"
    parts = shard.sharded_ledger_loopback(cols, kind, world)
    op, k = shard.gather_ledger(parts, cols.n_ops, cols.n_kernels)
    np.testing.assert_array_equal(op.cpu().numpy(), full.per_operator.array())
    np.testing.assert_array_equal(k.cpu().numpy(), full.per_kernel.array())
    for p in parts:
        assert p.total_joules == full.total_joules
        assert p.op_total == full.operator_total()
        assert p.idle_joules == full.idle_joules
    return full, parts


@pytest.mark.parametrize("method", ["samples", "ground_truth"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_ledger_c4_shape(method, world):
    cfg = synth.scaled(synth.CONFIGS["C4"], 100_000)
    a, _ = synth.make_pair(cfg)
    _check_ledger(a, method, world)


def _long_crossing_trace(kind_seed):
    """Short ops plus long ones spanning several windows (crossing intervals)."""
    rng = np.random.default_rng(kind_seed)
    S = 40_000
    ts = (np.cumsum(rng.integers(50, 150, size=S)) + 10_000).astype(np.int64)
    w = rng.uniform(75.0, 700.0, size=S)
    t0, t1 = int(ts[0]), int(ts[-1])
    lo = np.sort(rng.integers(t0, t1 - 10_000, size=3000))
    hi = lo + rng.integers(0, 8000, size=3000)
    # long ones: thousands of samples, across window edges
    llo = rng.integers(t0, t0 + (t1 - t0) // 3, size=40)
    lhi = np.minimum(llo + rng.integers(400_000, 2_500_000, size=40), t1)
    lo, hi = np.concatenate([lo, llo]), np.concatenate([hi, lhi])
    o = np.argsort(lo, kind="stable")
    lo, hi = lo[o].astype(np.int64), hi[o].astype(np.int64)
    # kernels: pieces of the ops (some long too)
    klo = lo + (hi - lo) // 4
    khi = hi - (hi - lo) // 4
    return TraceColumns.from_arrays(ts, w, lo, hi, klo, khi, np.arange(len(lo), dtype=np.int32))


@pytest.mark.parametrize("method", ["samples", "ground_truth"])
@pytest.mark.parametrize("world", [2, 4, 7])
def test_sharded_ledger_long_crossing(method, world):
    cols = _long_crossing_trace(3)
    full, parts = _check_ledger(cols, method, world)
    s = torch.cuda.synchronize()
    # the case actually exercised crossing intervals
    inps = [shard.rank_inputs(cols, "step" if method == "ground_truth" else "linear", wd)
            for wd in shard.plan(cols.n_power, world, "step" if method == "ground_truth" else "linear")]
    assert sum(int(shard.crossing(i).shape[0]) for i in inps) > 0


def test_sharded_ledger_error_order():
    """The first invalid interval in build_ledger order raises, as unsharded."""
    from paper_2512_08365_b200 import SignalError
    cols = _long_crossing_trace(4)
    op_end = cols.op_end.copy()
    op_end[2000] = cols.ts[-1] + 10**9  # outside the span, owned by a middle rank
    bad = TraceColumns.from_arrays(cols.ts, cols.watts, cols.op_start, op_end, cols.k_start, cols.k_end,
                                   cols.k_op, trace_end=int(cols.ts[-1]))
    with pytest.raises(SignalError, match="outside"):
        shard.sharded_ledger_loopback(bad, "linear", 4)


@pytest.mark.parametrize("world", [2, 3, 6])
def test_sharded_join_matches_one_gpu(world):
    cfg = synth.scaled(synth.CONFIGS["C4"], 60_000)
    a, b = synth.make_pair(cfg)
    la, lb = build_ledger(a, method="samples"), build_ledger(b, method="samples")
    jd = join_diff(a, b, la, lb, 0.10, 50, full_columns=False, epw=False)
    top = jd.top_findings(a, b)
    ia, ib = jd.pair_of(jd.order)
    pa = shard.sharded_ledger_loopback(a, "linear", world)
    pb = shard.sharded_ledger_loopback(b, "linear", world)
    As = [shard.shard_ops(a, p, True) for p in pa]
    Bs = [shard.shard_ops(b, p, False) for p in pb]
    res = shard.sharded_join_loopback(As, Bs, a.n_ops, 0.10, 50)
    assert res.P == jd.P
    assert res.n_waste == jd.n_waste
    assert res.wasted_joules == jd.wasted_joules
    assert [r[0] for r in res.top] == ia.cpu().tolist()
    assert [r[1] for r in res.top] == ib.cpu().tolist()
    assert [r[7] for r in res.top] == [f.wasted_joules for f in top]
    assert [r[2] for r in res.top] == [f.energy_a for f in top]
