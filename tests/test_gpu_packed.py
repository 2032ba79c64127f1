"""Packed columns (16/32-bit deltas / durations, 9-digit decimal watts codes,
csrc/pack.cu): device decode is exact, and every result computed from a packed trace equals the unpacked
one; the .dwc file round-trips."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

dw = pytest.importorskip("paper_2512_08365_b200")
from paper_2512_08365_b200 import build_ledger, synth  # noqa: E402
from paper_2512_08365_b200.columns import load_packed, pack, save_packed  # noqa: E402
from paper_2512_08365_b200.pipeline import analyze  # noqa: E402


def test_decode_exact_and_ledger_identical(tmp_path):
    cfg = synth.scaled(synth.CONFIGS["C4"], 50_000)
    a, b = synth.make_pair(cfg)
    p = pack(a)
    assert p.watts_p0 is not None  # synthetic watts are at the format's 9-digit precision
    assert p.ts_bits is not None and 6 <= p.ts_bits <= 8  # C4's jittered clock: 7-bit ts deltas
    from dataclasses import replace
    regular = pack(synth.make_pair(replace(cfg, jitter=0.0))[0])
    assert regular.ts_bits == 1  # a regular clock packs to 1-bit deltas
    assert set(p.iv_bits) == {"op_start", "op_end", "k_start", "k_end"}  # bit-packed intervals
    assert p.op_sig_dict is not None and p.sig_bits is not None
    for n in ("ts", "watts", "op_start", "op_end", "k_start", "k_end", "op_sig"):
        assert torch.equal(p.device(n), a.device(n)), n
    assert p.signal_span() == a.signal_span()
    la, lp = build_ledger(a, method="samples"), build_ledger(p, method="samples")
    assert torch.equal(la.per_operator.tensor, lp.per_operator.tensor)
    assert torch.equal(la.per_kernel.tensor, lp.per_kernel.tensor)
    assert la.total_joules == lp.total_joules
    # file round trip, pinned host columns, full analysis
    save_packed(a, tmp_path / "a.dwc")
    save_packed(b, tmp_path / "b.dwc")
    ha, hb = load_packed(tmp_path / "a.dwc", pin=True), load_packed(tmp_path / "b.dwc", pin=True)
    ra = analyze(a, b, "samples", 0.10, 20)
    rp = analyze(ha, hb, "samples", 0.10, 20)
    assert rp.report.wasted_joules == ra.report.wasted_joules
    assert [f.wasted_joules for f in rp.report.findings] == [f.wasted_joules for f in ra.report.findings]
    assert [f.pair for f in rp.report.findings] == [f.pair for f in ra.report.findings]
    assert [f.category for f in rp.report.findings] == [f.category for f in ra.report.findings]
    # the shipped host form carries no owner column: classification by containment
    from paper_2512_08365_b200.columns import PackedColumns
    bare = [PackedColumns(q.ts_base, q.ts, q.watts, q.op_start_base, q.op_start, q.op_end, q.k_start_base,
                          q.k_start, q.k_end, q.trace_end, op_sig=q.op_sig, watts_p0=q.watts_p0, ts_bias=q.ts_bias,
                          op_sig_dict=q.op_sig_dict, ts_bits=q.ts_bits, ts_step=q.ts_step, watts_bits=q.watts_bits, n_power=q.n_power,
                          ts_last=q._ts_last, iv_bits=q.iv_bits, n_ops=q.n_ops, n_kernels=q.n_kernels,
                          sig_bits=q.sig_bits, watts_rep=q.watts_rep)
            for q in (ha, hb)]
    rb = analyze(bare[0], bare[1], "samples", 0.10, 20)
    assert [f.category for f in rb.report.findings] == [f.category for f in ra.report.findings]
    assert rb.report.wasted_joules == ra.report.wasted_joules


def test_pack_rejects_unsorted():
    ts = np.array([1, 5, 3])
    from paper_2512_08365_b200.columns import TraceColumns
    c = TraceColumns.from_arrays(ts, np.ones(3), np.array([1]), np.array([2]))
    with pytest.raises(ValueError):
        pack(c)


@pytest.mark.parametrize("jitter", [0, 1, 3, 17, 100])
def test_bit_packed_timestamps_decode_exactly(jitter):
    """dw_unpack_bits: widths 1..8, fields crossing 32-bit word boundaries."""
    from paper_2512_08365_b200.columns import TraceColumns
    g = torch.Generator().manual_seed(jitter)
    n = 300_001
    d = 160 + torch.randint(-jitter, jitter + 1, (n,), generator=g) if jitter else torch.full((n,), 160)
    ts = (10**12 + torch.cumsum(d, 0)).to(torch.int64)
    c = TraceColumns.from_arrays(ts.numpy(), np.full(n, 75.0), np.array([int(ts[3])]), np.array([int(ts[9])]))
    p = pack(c)
    assert p.ts_bits is not None and p.ts_bits <= 8
    assert torch.equal(p.device("ts").cpu(), ts)
    assert p.signal_span() == c.signal_span()


@pytest.mark.parametrize("spread", [0, 1, 7, 200, 4095, 32000])
def test_bit_packed_intervals_decode_exactly(spread):
    """dw_unpack_bits + dw_unpack_bits_dur on interval columns of every width."""
    from paper_2512_08365_b200.columns import TraceColumns
    rng = np.random.default_rng(spread + 1)
    n = 200_003
    st = 10**9 + np.cumsum(rng.integers(50, 51 + spread, size=n)).astype(np.int64)
    en = st + rng.integers(3, 4 + spread, size=n)
    ts = np.arange(st[0] - 100, en.max() + 1000, 997, dtype=np.int64)
    c = TraceColumns.from_arrays(ts, np.full(ts.size, 75.0), st, en, st, en, np.arange(n, dtype=np.int32))
    p = pack(c)
    assert {"op_start", "op_end", "k_start", "k_end"} <= set(p.iv_bits)
    for name in ("op_start", "op_end", "k_start", "k_end"):
        assert torch.equal(p.device(name).cpu(), torch.from_numpy(c.host(name))), name
    assert p.n_ops == n and p.n_kernels == n


@pytest.mark.parametrize("n,maxrun", [(1, 1), (33, 3), (100_003, 9), (1_000_000, 1), (2_500_017, 40)])
def test_run_coded_watts_decode_exactly(n, maxrun):
    """dw_unpack_decimal_rep: the change bitmap's prefix counts across words,
    warps and blocks (32768 samples each); ragged tails; runs of one sample
    (a code per sample) and long runs."""
    from paper_2512_08365_b200 import _native
    from paper_2512_08365_b200.columns import decimal_code
    rng = np.random.default_rng(n)
    runs = rng.integers(1, maxrun + 1, size=n)
    vals = np.round(rng.uniform(1.0, 900.0, size=n), 3)
    w = np.repeat(vals, runs)[:n]
    p0, code = decimal_code(w)
    new = np.ones(n, dtype=bool)
    new[1:] = code[1:] != code[:-1]
    words = np.packbits(np.concatenate([new, np.zeros((-n) % 32, dtype=bool)]), bitorder="little").view(np.uint32)
    dev = torch.device("cuda")
    d_code = torch.from_numpy(code[new].view(np.int32)).to(dev)
    d_rep = torch.from_numpy(words.view(np.int32)).to(dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    L = _native.lib()
    ws = torch.empty(L.dw_unpack_decimal_rep_workspace_size(n), dtype=torch.uint8, device=dev)
    _native.check(L.dw_unpack_decimal_rep(_native.ptr(d_code), _native.ptr(d_rep), n, p0, _native.ptr(out),
                                          ws.data_ptr(), ws.numel(), _native.stream_handle()), "rep")
    np.testing.assert_array_equal(out.cpu().numpy(), w)
    assert L.dw_unpack_decimal_rep(_native.ptr(d_code), _native.ptr(d_rep), n, p0, _native.ptr(out),
                                   ws.data_ptr(), 8, _native.stream_handle()) == _native.DW_E_WORKSPACE


def test_run_coded_trace_analysis_identical():
    """The C4-shaped synthetic power repeats ~80% of samples: it travels
    run-coded, decodes to the same column, and the pinned-host analysis is
    identical to the device-resident one."""
    cfg = synth.scaled(synth.CONFIGS["C4"], 200_000)
    a, b = synth.make_pair(cfg)
    p = pack(a)
    assert p.watts_rep is not None
    assert p.watts.numel() < 0.4 * a.n_power
    assert torch.equal(p.device("watts"), a.device("watts"))
    pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)  # noqa: E731
    from paper_2512_08365_b200.columns import PackedColumns
    hosts = []
    for c in (a, b):
        q = pack(c)
        hosts.append(PackedColumns(q.ts_base, pin(q.ts), pin(q.watts), q.op_start_base, pin(q.op_start),
                                   pin(q.op_end), q.k_start_base, pin(q.k_start), pin(q.k_end), q.trace_end,
                                   op_sig=pin(q.op_sig), watts_p0=q.watts_p0, ts_bias=q.ts_bias,
                                   op_sig_dict=pin(q.op_sig_dict), ts_bits=q.ts_bits, ts_step=q.ts_step, watts_bits=q.watts_bits, n_power=q.n_power,
                                   ts_last=q._ts_last, iv_bits=q.iv_bits, n_ops=q.n_ops, n_kernels=q.n_kernels,
                                   sig_bits=q.sig_bits, watts_rep=pin(q.watts_rep)))
    ra = analyze(a, b, "samples", 0.10, 20)
    rh = analyze(hosts[0], hosts[1], "samples", 0.10, 20, copy_stream=torch.cuda.Stream())
    assert rh.report.total_a == ra.report.total_a and rh.report.total_b == ra.report.total_b
    assert rh.report.wasted_joules == ra.report.wasted_joules
    assert [f.pair for f in rh.report.findings] == [f.pair for f in ra.report.findings]
    # a run-coded column without its bitmap is refused, not misread
    bad = PackedColumns(p.ts_base, p.ts, p.watts, p.op_start_base, p.op_start, p.op_end, p.k_start_base, p.k_start,
                        p.k_end, p.trace_end, op_sig=p.op_sig, watts_p0=p.watts_p0, ts_bias=p.ts_bias,
                        op_sig_dict=p.op_sig_dict, ts_bits=p.ts_bits, ts_step=p.ts_step, n_power=p.n_power,
                        ts_last=p._ts_last,
                        iv_bits=p.iv_bits, n_ops=p.n_ops, n_kernels=p.n_kernels, sig_bits=p.sig_bits)
    with pytest.raises(ValueError):
        bad.device("watts")


@pytest.mark.parametrize("jitter,period,n", [(0.3, 50.0, 300_001), (0.49, 1000.0, 1_000_003), (0.1, 7.3, 3),
                                             (0.45, 123456.7, 70_000), (0.0, 3.0, 200_000)])
def test_grid_coded_timestamps_decode_exactly(jitter, period, n):
    """dw_unpack_grid: residuals from the clock's line (any width the packer
    picks, fields crossing 32-bit words) decode to the exact timestamps, and
    pack() picks them only when narrower than the deltas."""
    from paper_2512_08365_b200.columns import TraceColumns
    rng = np.random.default_rng(n)
    x = np.arange(n) + (2 * rng.random(n) - 1) * jitter
    x[0], x[-1] = 0, n - 1
    ts = (10**12 + np.floor(x * period)).astype(np.int64)
    c = TraceColumns.from_arrays(ts, np.full(n, 75.0), ts[:1], ts[:1] + 1)
    p = pack(c)
    d = pack(c, grid_ts=False)
    if p.ts_step is not None:
        assert p.ts_bits < (d.ts_bits or 8 * np.asarray(d.ts).itemsize)
    assert np.array_equal(p.device("ts").cpu().numpy(), ts)
    assert p.signal_span() == c.signal_span()


def test_c4_clock_is_grid_coded():
    """C4's jittered clock (synth._power): grid-coded in one bit fewer than
    its deltas, and the device packer (torch path) agrees with the host one."""
    cfg = synth.scaled(synth.CONFIGS["C4"], 50_000)
    a, _ = synth.make_pair(cfg)
    p = pack(a)
    d = pack(a, grid_ts=False)
    assert p.ts_step is not None and p.ts_bits == d.ts_bits - 1
    assert torch.equal(p.device("ts"), a.device("ts"))
    ts_host = a.host("ts")
    q = pack(type(a).from_arrays(ts_host, a.host("watts"), a.host("op_start")[:1], a.host("op_end")[:1]))
    assert (q.ts_step, q.ts_bias, q.ts_bits) == (p.ts_step, p.ts_bias, p.ts_bits)
    assert np.array_equal(np.asarray(q.ts).view(np.uint32), np.asarray(p.ts.cpu() if isinstance(p.ts, torch.Tensor)
                                                                         else p.ts).view(np.uint32))


@pytest.mark.parametrize("kind", ["c4", "milliwatts", "mixed_decades"])
def test_bit_packed_watts_codes_decode_exactly(kind):
    """dw_unpack_decimal_rep_bits: run-coded watts whose stored codes are
    bit-packed after stripping their shared decimal zeros -- C4's 6-decimal
    kernel watts (30 bits), integer-milliwatt NVML readings (p0 lowered by 3,
    ~20 bits), values across decades (several exponents j) -- decode to the
    exact doubles, and the .dwc file round-trips them."""
    from paper_2512_08365_b200.columns import TraceColumns
    from paper_2512_08365_b200.synth import round9
    rng = np.random.default_rng(len(kind))
    n = 400_003
    ts = (10**9 + np.arange(n) * 100).astype(np.int64)
    runs = np.repeat(np.arange(n // 5 + 1), 5)[:n]
    if kind == "c4":
        vals = round9(torch.from_numpy(rng.uniform(150.0, 700.0, n // 5 + 1))).numpy()
    elif kind == "milliwatts":
        vals = rng.integers(60_000, 1_000_000, n // 5 + 1) / 1000.0
    else:
        vals = round9(torch.from_numpy(rng.uniform(5.0, 60.0, n // 5 + 1))).numpy()  # j in {0, 1}: 31 bits
    w = vals[runs]
    c = TraceColumns.from_arrays(ts, w, ts[:1], ts[:1] + 10)
    p = pack(c)
    assert p.watts_rep is not None and p.watts_bits is not None
    if kind == "milliwatts":
        assert p.watts_bits[0] <= 20
    if kind == "c4":
        assert p.watts_bits[0] == 30
    if kind == "mixed_decades":  # two exponents j: the j bit is inside the packed spread
        assert p.watts_bits[0] == 31
    assert np.array_equal(p.device("watts").cpu().numpy(), w)
    import tempfile, os
    with tempfile.TemporaryDirectory() as d:
        save_packed(c, os.path.join(d, "w.dwc"))
        q = load_packed(os.path.join(d, "w.dwc"))
        assert q.watts_bits == p.watts_bits and q.watts_p0 == p.watts_p0
        assert np.array_equal(q.device("watts").cpu().numpy(), w)
