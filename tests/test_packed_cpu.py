"""Packed columnar trace files (columns.pack / save_packed / load_packed) on
the host: the 16/32-bit deltas and durations and the decimal watts codes
round-trip exactly, the span is preserved, and traces that cannot be packed
are refused."""
import numpy as np
import pytest

from paper_2512_08365_b200.columns import TraceColumns, decimal_code, load_packed, pack, save_packed


def _u(d):
    d = np.asarray(d)
    return d.view(np.uint16 if d.itemsize == 2 else np.uint32).astype(np.int64)


def _round9(x):
    return np.array([float(f"{v:.9g}") for v in x])


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
    dec = lambda base, d: base + np.cumsum(_u(d))  # noqa: E731
    np.testing.assert_array_equal(dec(p.ts_base, p.ts), c.ts)
    assert p.watts_p0 is None  # uniform draws are not 9-digit decimals: f64 column
    np.testing.assert_array_equal(np.asarray(p.watts), c.watts)
    np.testing.assert_array_equal(dec(p.op_start_base, p.op_start), c.op_start)
    np.testing.assert_array_equal(dec(p.op_start_base, p.op_start) + _u(p.op_end), c.op_end)
    np.testing.assert_array_equal(dec(p.k_start_base, p.k_start) + _u(p.k_end), c.k_end)
    assert np.asarray(p.ts).itemsize == 2 and np.asarray(p.op_end).itemsize == 4  # narrowest width per column
    np.testing.assert_array_equal(np.asarray(p.op_sig_dict)[_fields(p.op_sig, p.sig_bits, c.n_ops)], c.op_sig)
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


def _decode(p0, code):
    code = np.asarray(code).view(np.uint32)
    m = (code & 0x3FFFFFFF).astype(np.float64)
    pw = p0 + (code >> 30).astype(np.int64)
    return np.where(pw >= 0, m / 10.0 ** np.abs(pw), m * 10.0 ** np.abs(pw))


def test_decimal_watts_roundtrip(tmp_path):
    rng = np.random.default_rng(3)
    w = _round9(np.concatenate([rng.uniform(50, 700, 3000), rng.uniform(1.0, 9.9, 100), [75.0, 0.0, 999.0]]))
    p0, code = decimal_code(w)
    np.testing.assert_array_equal(_decode(p0, code), w)
    c = _cols()
    c = TraceColumns.from_arrays(c.ts[:w.size], w, c.op_start[:10], c.op_end[:10], c.k_start[:20], c.k_end[:20],
                                 c.k_op[:20])
    save_packed(c, tmp_path / "d.dwc")
    p = load_packed(tmp_path / "d.dwc")
    assert p.watts_p0 == p0
    np.testing.assert_array_equal(_decode(p.watts_p0, p.watts), w)


def test_non_decimal_watts_stay_f64():
    assert decimal_code(np.array([1.0 / 3.0, 2.0])) is None
    assert decimal_code(np.array([-1.0])) is None
    assert decimal_code(np.array([np.nan])) is None


def _fields(words, width, n):
    w = np.asarray(words).view(np.uint32).astype(np.uint64)
    bit = np.arange(n, dtype=np.int64) * width
    k = bit >> 5
    win = w[k] | (w[k + 1] << np.uint64(32))
    return ((win >> (bit & 31).astype(np.uint64)) & np.uint64((1 << width) - 1)).astype(np.int64)


def _unbits(base, bias, width, words, n):
    w = np.asarray(words).view(np.uint32).astype(np.uint64)
    i = np.arange(1, n, dtype=np.int64)
    bit = i * width
    k = bit >> 5
    win = w[k] | (w[k + 1] << np.uint64(32))
    f = ((win >> (bit & 31).astype(np.uint64)) & np.uint64((1 << width) - 1)).astype(np.int64)
    return base + np.concatenate([[0], np.cumsum(bias + f)])


def test_regular_clock_ts_bit_packed(tmp_path):
    """A sampling clock with jitter: bit-packed deltas (7 bits here);
    signatures as a dictionary + 16-bit codes."""
    rng = np.random.default_rng(5)
    ts = (10**9 + np.cumsum(160 + rng.integers(-40, 41, size=5000))).astype(np.int64)
    sig = rng.integers(0, 300, size=50).astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    st = np.sort(rng.integers(ts[0], ts[-1] - 1000, size=50))
    c = TraceColumns.from_arrays(ts, np.full(5000, 75.0), st, st + 100, op_sig=sig)
    for p in (pack(c), None):
        if p is None:
            save_packed(c, tmp_path / "r.dwc")
            p = load_packed(tmp_path / "r.dwc")
        assert p.ts_bits == 7 and p.n_power == ts.size
        np.testing.assert_array_equal(_unbits(p.ts_base, p.ts_bias, p.ts_bits, p.ts, ts.size), ts)
        assert p.sig_bits is not None and p.sig_bits <= 9  # < 300 distinct signatures
        np.testing.assert_array_equal(np.asarray(p.op_sig_dict)[_fields(p.op_sig, p.sig_bits, sig.size)], sig)
        assert p.signal_span() == c.signal_span()


@pytest.mark.parametrize("spread", [0, 1, 2, 3, 31, 32, 255, 4095, 32767])
def test_bitfields_roundtrip_every_width(spread):
    """_bitfields packs v - min(v) in bit_length(spread) bits (at least 1),
    fields straddling 32-bit words included; torch and numpy agree."""
    import torch
    from paper_2512_08365_b200.columns import _bitfields
    rng = np.random.default_rng(spread)
    v = 1000 + rng.integers(0, spread + 1, size=4097)
    v[0], v[-1] = 1000, 1000 + spread
    lo, width, words = _bitfields(v, 15)
    assert lo == 1000 and width == max(1, spread.bit_length())
    np.testing.assert_array_equal(_fields(words, width, v.size) + lo, v)
    lo_t, width_t, words_t = _bitfields(torch.from_numpy(v), 15)
    assert (lo_t, width_t) == (lo, width)
    np.testing.assert_array_equal(words_t.numpy().view(np.uint32), words)


def test_bitfields_refuse_wide_spreads():
    from paper_2512_08365_b200.columns import _bitfields, _bitpack
    assert _bitfields(np.array([0, 1 << 15]), 15) is None
    assert _bitpack(np.array([5, 3])) is None          # a negative delta: not sorted
    assert _bitpack(np.array([7])) is None             # fewer than two samples


def test_run_coded_watts(tmp_path):
    """Watts that repeat (a meter read faster than it updates) travel as a
    change bitmap plus one code per change (columns.rep_code); the host
    decode of the file's columns gives every sample back."""
    from paper_2512_08365_b200.columns import rep_code
    rng = np.random.default_rng(5)
    c = _cols()
    n = c.n_power
    runs = rng.integers(1, 12, size=n)
    w = _round9(np.repeat(rng.uniform(50, 700, n), runs)[:n])
    c = TraceColumns.from_arrays(c.ts, w, c.op_start, c.op_end, c.k_start, c.k_end, c.k_op)
    p = pack(c)
    assert p.watts_rep is not None and np.asarray(p.watts).size < n / 2
    assert pack(c, runs=False).watts_rep is None
    save_packed(c, tmp_path / "r.dwc")
    q = load_packed(tmp_path / "r.dwc")
    for x in (p, q):
        bits = np.unpackbits(np.asarray(x.watts_rep).view(np.uint8), bitorder="little")[:n].astype(bool)
        assert bits[0]
        codes = np.asarray(x.watts)
        if x.watts_bits is not None:  # bit-packed codes: bias + fields (columns._pack_codes)
            codes = (x.watts_bits[1] + _fields(codes, x.watts_bits[0], int(bits.sum()))).astype(np.uint32)
        np.testing.assert_array_equal(_decode(x.watts_p0, codes)[np.cumsum(bits) - 1], w)
    assert q.host_bytes == p.host_bytes < pack(c, runs=False).host_bytes
    # no repeats: plain codes
    assert rep_code(np.arange(1000, dtype=np.uint32)) is None


def _ungrid(base, bias, width, words, n, step):
    i = np.arange(n, dtype=np.int64)
    return base + i * (step >> 32) + ((i * (step & 0xFFFFFFFF)) >> 32) + bias + _fields(words, width, n)


@pytest.mark.parametrize("jitter,period", [(0.3, 50.0), (0.45, 1000.0), (0.1, 7.3), (0.49, 123456.7)])
def test_grid_coded_clock(tmp_path, jitter, period):
    """A clock read at nominal instants i * period with up to +-jitter periods
    of read jitter (synth._power): residuals from the line through the first
    and last sample need one bit fewer than the deltas, so pack() grid-codes
    them; the host restatement of dw_unpack_grid and the .dwc round trip give
    the timestamps back exactly."""
    rng = np.random.default_rng(int(period))
    n = 20001
    x = np.arange(n) + (2 * rng.random(n) - 1) * jitter
    x[0], x[-1] = 0, n - 1
    ts = (10**11 + np.floor(x * period)).astype(np.int64)
    assert (np.diff(ts) > 0).all()
    st = np.sort(rng.integers(ts[0], ts[-1] - 10, size=40))
    c = TraceColumns.from_arrays(ts, np.full(n, 75.0), st, st + 5)
    dpk = pack(c, grid_ts=False)
    for p in (pack(c), None):
        if p is None:
            save_packed(c, tmp_path / "g.dwc")
            p = load_packed(tmp_path / "g.dwc")
        assert p.ts_step is not None and p.ts_bits < (dpk.ts_bits or 8 * np.asarray(dpk.ts).itemsize)
        np.testing.assert_array_equal(_ungrid(p.ts_base, p.ts_bias, p.ts_bits, np.asarray(p.ts), n, p.ts_step), ts)
        assert p.signal_span() == c.signal_span()


def test_grid_not_chosen_for_random_walk_clock():
    """Deltas with independent noise (a drifting clock): the residuals from
    the line grow like a random walk, so pack() keeps the delta coding."""
    rng = np.random.default_rng(3)
    ts = (10**9 + np.cumsum(160 + rng.integers(-40, 41, size=100_000))).astype(np.int64)
    p = pack(TraceColumns.from_arrays(ts, np.full(ts.size, 75.0), ts[:1], ts[:1] + 1))
    assert p.ts_step is None and p.ts_bits == 7
