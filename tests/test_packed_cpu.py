"""Packed columnar trace files (columns.pack / save_packed / load_packed) on
the host: the uint32 deltas and durations round-trip exactly, the span is
preserved, and traces that cannot be packed are refused."""
import numpy as np
import pytest

from paper_2512_08365_b200.columns import TraceColumns, load_packed, pack, save_packed


def _cols(seed=0, n=5000, m=400):
    rng = np.random.default_rng(seed)
    ts = (np.cumsum(rng.integers(1, 5000, size=n)) + 10**12).astype(np.int64)  # large absolute times
    w = rng.uniform(50, 700, size=n)
    st = np.sort(rng.integers(ts[0], ts[-1] - 10**6, size=m))
    en = st + rng.integers(0, 10**6, size=m)
    kst = np.sort(np.concatenate([st, st + 1]))
    ken = kst + rng.integers(1, 1000, size=kst.size)
    sig = rng.integers(0, 2**63, size=m, dtype=np.int64).view(np.uint64)
    return TraceColumns.from_arrays(ts, w, st, en, kst, ken, np.repeat(np.arange(m, dtype=np.int32), 2),
                                    op_sig=sig)


def test_roundtrip(tmp_path):
    c = _cols()
    save_packed(c, tmp_path / "t.dwc")
    p = load_packed(tmp_path / "t.dwc")
    dec = lambda base, d: base + np.cumsum(np.asarray(d).view(np.uint32).astype(np.int64))  # noqa: E731
    np.testing.assert_array_equal(dec(p.ts_base, p.ts), c.ts)
    np.testing.assert_array_equal(np.asarray(p.watts), c.watts)
    np.testing.assert_array_equal(dec(p.op_start_base, p.op_start), c.op_start)
    np.testing.assert_array_equal(dec(p.op_start_base, p.op_start) + np.asarray(p.op_end).view(np.uint32),
                                  c.op_end)
    np.testing.assert_array_equal(dec(p.k_start_base, p.k_start) + np.asarray(p.k_end).view(np.uint32), c.k_end)
    np.testing.assert_array_equal(np.asarray(p.op_sig), c.op_sig)
    np.testing.assert_array_equal(np.asarray(p.k_op), c.k_op)
    assert p.signal_span() == c.signal_span()
    assert p.n_power == c.n_power and p.n_ops == c.n_ops and p.n_kernels == c.n_kernels


def test_host_bytes_shrink():
    c = _cols()
    p = pack(c)
    full = c.ts.nbytes + c.watts.nbytes + c.op_start.nbytes * 2 + c.k_start.nbytes * 2 + c.op_sig.nbytes
    assert p.host_bytes < 0.8 * full


@pytest.mark.parametrize("mutate", ["unsorted_ts", "huge_gap", "negative_duration"])
def test_unpackable_refused(mutate):
    c = _cols()
    ts, en = c.ts.copy(), c.op_end.copy()
    if mutate == "unsorted_ts":
        ts[10], ts[11] = ts[11], ts[10]
    elif mutate == "huge_gap":
        ts[100:] += 1 << 33
    else:
        en[5] = c.op_start[5] - 1
    bad = TraceColumns.from_arrays(ts, c.watts, c.op_start, en, c.k_start, c.k_end, c.k_op)
    with pytest.raises(ValueError):
        pack(bad)
