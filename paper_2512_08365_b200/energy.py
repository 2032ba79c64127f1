"""Energy attribution -- drop-in for the reference's ``diffwatt.energy``.

Same names, signatures, return types and exceptions as
/root/reference/pkg/src/diffwatt/energy.py; the per-interval integration runs
in libdwb200 on the GPU (csrc/attribute.cu), never on the host:

    integrate(signal, (lo, hi))        energy.py:90-105   -> dw_attribute
    build_ledger(trace, method, ...)   energy.py:280-331  -> dw_ledger
    PowerSignal.value_at for sampling  energy.py:57-66    -> dw_step_value_at

Numerics: intervals covering <= DW_DIRECT_MAX (256) power segments get the
reference's own sequential fp64 sum, bit for bit; longer ones (and the ledger
total) get an exact fixed-point sum rounded once, within 1e-12
relative of the reference's sequential sum.
"""

from __future__ import annotations

import ctypes
from collections.abc import Mapping
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np
import torch

from . import _native
from .columns import PackedColumns, TraceColumns, synthetic_id, synthetic_ids
from .trace_model import OperatorEvent, PowerSample, Trace

US_PER_S = 1_000_000

DEFAULT_SAMPLER_PERIOD_US = 40_000  # 25 Hz (energy.py:23)
DEFAULT_SAMPLER_DELAY_US = 200_000  # energy.py:24
DEFAULT_REPLAY_REPEAT = 1000
REPLAY_MARGIN = 0.10

IDLE_OP = "idle"

METHODS = ("ground_truth", "sampled", "replay")
# Extension for traces whose power records are already high-rate meter
# samples (the scale configs): integrate them with the sampled branch's
# trapezoid (energy.py:108-130) as given, without re-sampling.
EXTRA_METHODS = ("samples",)


class SignalError(ValueError):
    pass


# ----------------------------------------------------------------- signals


class PowerSignal:
    """Piecewise-constant ground truth, or a sampled view of one.

    Constructor-compatible with the reference dataclass (energy.py:37-82):
    ``PowerSignal(segments=...)`` / ``PowerSignal(samples=..., period_us=, delay_us=)``.
    Internally it is columnar: ``ts``/``watts`` arrays plus ``span_hi`` (step)
    -- see ``from_columns``.
    """

    __slots__ = ("_ts", "_w", "_span_hi", "_kind", "period_us", "delay_us", "_segments",
                 "_samples", "_dev", "_first")

    def __init__(self, segments=(), samples=(), period_us=None, delay_us=None):
        self.period_us = period_us
        self.delay_us = delay_us
        self._segments = tuple(segments) if segments else ()
        self._samples = tuple(samples) if samples else ()
        self._dev = {}
        self._first = None
        if self._segments:
            self._kind = _native.DW_SIGNAL_STEP
            ts, w = [], []
            prev_end = None
            for s, e, watts in self._segments:
                if prev_end is not None and s != prev_end:
                    if s < prev_end:
                        raise SignalError("overlapping ground-truth segments are not supported")
                    ts.append(prev_end)  # a gap integrates to nothing: hold 0 W
                    w.append(0.0)
                ts.append(int(s))
                w.append(float(watts))
                prev_end = int(e)
            self._ts = np.asarray(ts, dtype=np.int64)
            self._w = np.asarray(w, dtype=np.float64)
            self._span_hi = int(self._segments[-1][1])
        elif self._samples:
            self._kind = _native.DW_SIGNAL_LINEAR
            self._ts = np.fromiter((s.timestamp for s in self._samples), dtype=np.int64,
                                   count=len(self._samples))
            self._w = np.fromiter((s.watts for s in self._samples), dtype=np.float64,
                                  count=len(self._samples))
            self._span_hi = int(self._ts[-1])
        else:
            self._kind = None
            self._ts = self._w = None
            self._span_hi = None

    @classmethod
    def from_columns(cls, ts, watts, span_hi=None, kind="step", period_us=None,
                     delay_us=None, first=None) -> "PowerSignal":
        """A signal over existing arrays (numpy or CUDA tensors): ``kind="step"``
        takes breakpoints ts with the last segment ending at ``span_hi``;
        ``kind="linear"`` takes samples (``span_hi``, when given, is their last
        timestamp).  ``first``: ts[0] when the caller knows it (no device read)."""
        sig = cls.__new__(cls)
        sig.period_us, sig.delay_us = period_us, delay_us
        sig._segments = None
        sig._samples = None
        sig._dev = {}
        sig._ts, sig._w = ts, watts
        sig._first = None if first is None else int(first)
        if kind == "step":
            sig._kind = _native.DW_SIGNAL_STEP
            sig._span_hi = int(span_hi)
        else:
            sig._kind = _native.DW_SIGNAL_LINEAR
            if span_hi is None:
                span_hi = ts[-1].item() if isinstance(ts, torch.Tensor) else ts[-1]
            sig._span_hi = int(span_hi)
        return sig

    # reference fields, materialised lazily
    @property
    def segments(self) -> tuple:
        if self._segments is None:
            if self._kind != _native.DW_SIGNAL_STEP:
                self._segments = ()
            else:
                ts = _host(self._ts)
                w = _host(self._w)
                ends = np.append(ts[1:], self._span_hi)
                self._segments = tuple(zip(ts.tolist(), ends.tolist(), w.tolist()))
        return self._segments

    @property
    def samples(self) -> tuple:
        if self._samples is None:
            if self._kind != _native.DW_SIGNAL_LINEAR:
                self._samples = ()
            else:
                self._samples = tuple(PowerSample(timestamp=t, watts=w) for t, w in
                                      zip(_host(self._ts).tolist(), _host(self._w).tolist()))
        return self._samples

    @property
    def is_ground_truth(self) -> bool:
        return self._kind == _native.DW_SIGNAL_STEP

    def __len__(self) -> int:
        return 0 if self._ts is None else int(self._ts.shape[0])

    def span(self) -> tuple[int, int]:
        if self._kind is None or len(self) == 0:
            raise SignalError("empty power signal")
        first = getattr(self, "_first", None)
        if first is None:
            first = self._ts[0].item() if isinstance(self._ts, torch.Tensor) else self._ts[0]
            self._first = int(first)
        return int(first), int(self._span_hi)

    def value_at(self, t_us: float) -> float:
        """Ground-truth value at a time point, clamped to the signal span
        (energy.py:57-66); evaluated on the device."""
        if not self.is_ground_truth:
            raise SignalError("value_at requires the ground-truth form")
        return float(_value_at(self, np.asarray([t_us], dtype=np.float64))[0])

    def __eq__(self, other) -> bool:
        if not isinstance(other, PowerSignal):
            return NotImplemented
        return (self._kind == other._kind and self.segments == other.segments
                and self.samples == other.samples and self.period_us == other.period_us
                and self.delay_us == other.delay_us)

    def __repr__(self) -> str:
        kind = {0: "step", 1: "linear"}.get(self._kind, "empty")
        return f"PowerSignal({kind}, n={len(self)}, span_hi={self._span_hi})"

    # device residency
    def _device(self):
        dev = _native.device()
        key = dev.index
        if key not in self._dev:
            self._dev[key] = (_to_dev(self._ts, torch.int64, dev), _to_dev(self._w, torch.float64, dev))
        return self._dev[key]

    def _c_signal(self, validate_order=False, summation: str = "reference") -> tuple:
        ts_d, w_d = self._device()
        sig = _native.Signal(ts_d.data_ptr(), w_d.data_ptr(), int(ts_d.numel()),
                             int(self._span_hi), int(self._kind), 1 if validate_order else 0,
                             _sum_mode(summation), 0)
        return sig, (ts_d, w_d)


SUMMATIONS = ("reference", "exact")


def _sum_mode(summation: str) -> int:
    """dw_signal_t.sum_mode of a summation name (include/dwb200.h):
    "reference" -- the reference's own sequential fp64 sum for intervals of
    up to DW_DIRECT_MAX pieces (bit-identical to energy.integrate), exact
    fixed point beyond; "exact" -- every interval as the exact sum of its
    pieces rounded to 2^-40 W*us, rounded once (deterministic, independent of
    how the device groups the pieces, within a few ulps of the reference)."""
    if summation not in SUMMATIONS:
        raise ValueError(f"unknown summation {summation!r}")
    return _native.SUM_EXACT if summation == "exact" else _native.SUM_REFERENCE


def _host(a):
    if isinstance(a, torch.Tensor):
        return a.cpu().numpy()
    return np.asarray(a)


def _to_dev(a, dtype, dev):
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)


def _value_at(sig: PowerSignal, t: np.ndarray) -> np.ndarray:
    dev = _native.device()
    csig, keep = sig._c_signal()
    t_d = torch.from_numpy(np.ascontiguousarray(t, dtype=np.float64)).to(dev)
    out = torch.empty_like(t_d)
    rc = _native.lib().dw_step_value_at(ctypes.byref(csig), _native.ptr(t_d), t_d.numel(),
                                        _native.ptr(out), _native.stream_handle())
    _native.check(rc, "dw_step_value_at")
    return out.cpu().numpy()


def ground_truth_signal(trace) -> PowerSignal:
    """PowerSignal.from_breakpoints over the trace's power records (energy.py:85-87)."""
    cols = TraceColumns.from_trace(trace)
    if cols.n_power == 0:
        raise SignalError("trace carries no power records")
    _, span_hi = cols.signal_span()
    if isinstance(cols, PackedColumns):  # host columns hold codes: the decoded device columns
        return PowerSignal.from_columns(cols.device("ts"), cols.device("watts"), span_hi, "step")
    return PowerSignal.from_columns(cols.ts, cols.watts, span_hi, "step")


# ----------------------------------------------------------------- integrate


def _raise_interval_error(lo: int, hi: int, span: tuple[int, int]):
    if hi < lo:
        raise SignalError("interval end precedes start")
    raise SignalError(f"interval [{lo},{hi}] outside signal span [{span[0]},{span[1]}]")


def integrate_many(signal: PowerSignal, lo, hi, summation: str = "reference") -> torch.Tensor:
    """Joules for many intervals at once (device tensor out).  Errors follow
    the reference: the first invalid interval raises SignalError.
    ``summation``: see ``_sum_mode``."""
    if signal._kind is None or len(signal) == 0:
        raise SignalError("empty power signal")
    dev = _native.device()
    lo_d = _to_dev(lo, torch.int64, dev).reshape(-1)
    hi_d = _to_dev(hi, torch.int64, dev).reshape(-1)
    out = torch.empty(lo_d.numel(), dtype=torch.float64, device=dev)
    sorted_ = bool(lo_d.numel() < 2 or bool((lo_d[1:] >= lo_d[:-1]).all().item()))
    iset = _native.IntervalSet(_native.ptr(lo_d), _native.ptr(hi_d), lo_d.numel(),
                               _native.ptr(out), 1 if sorted_ else 0, 0)
    csig, keep = signal._c_signal(summation=summation)
    sizes = (ctypes.c_int64 * 1)(lo_d.numel())
    L = _native.lib()
    nbytes = L.dw_attribute_workspace_size(csig.n, sizes, 1)
    ws = _native.Workspace.get(nbytes)
    stream = _native.stream_handle()
    _native.check(L.dw_attribute(ctypes.byref(csig), ctypes.byref(iset), 1, ws.data_ptr(),
                                 ws.numel(), stream), "dw_attribute")
    st = _native.Status()
    L.dw_status(ws.data_ptr(), stream, ctypes.byref(st))
    if st.bad_index[0] >= 0:
        k = st.bad_index[0]
        _raise_interval_error(int(lo_d[k].item()), int(hi_d[k].item()), signal.span())
    return out


def integrate_split(signal: PowerSignal, lo, hi) -> torch.Tensor:
    """Overlap-split joules of one interval set (device tensor out): the
    signal's power divided equally among the set's intervals active at each
    instant (the reference has no such mode, it
    gives every interval the full signal -- SURVEY.md G1).  Equal to
    ``integrate_many`` when no two intervals overlap.  Errors as
    ``integrate_many``."""
    if signal._kind is None or len(signal) == 0:
        raise SignalError("empty power signal")
    dev = _native.device()
    lo_d = _to_dev(lo, torch.int64, dev).reshape(-1)
    hi_d = _to_dev(hi, torch.int64, dev).reshape(-1)
    out = torch.empty(lo_d.numel(), dtype=torch.float64, device=dev)
    iset = _native.IntervalSet(_native.ptr(lo_d), _native.ptr(hi_d), lo_d.numel(), _native.ptr(out), 0, 0)
    csig, keep = signal._c_signal()
    L = _native.lib()
    ws = _native.Workspace.get(L.dw_attribute_split_workspace_size(csig.n, lo_d.numel()))
    stream = _native.stream_handle()
    _native.check(L.dw_attribute_split(ctypes.byref(csig), ctypes.byref(iset), ws.data_ptr(), ws.numel(),
                                       stream), "dw_attribute_split")
    st = _native.Status()
    L.dw_status(ws.data_ptr(), stream, ctypes.byref(st))
    if st.order_index >= 0:
        from .trace_model import TraceError
        raise TraceError("power samples must be strictly increasing in timestamp")
    if st.bad_index[0] >= 0:
        k = st.bad_index[0]
        _raise_interval_error(int(lo_d[k].item()), int(hi_d[k].item()), signal.span())
    return out


def integrate(signal: PowerSignal, interval: tuple[int, int]) -> float:
    """Joules over ``interval``; exact for ground truth, trapezoidal for samples
    (energy.py:90-105)."""
    if not isinstance(signal, PowerSignal):
        signal = _coerce_signal(signal)
    lo, hi = interval
    if hi < lo:
        raise SignalError("interval end precedes start")
    start, end = signal.span()
    if lo < start or hi > end:
        raise SignalError(f"interval [{lo},{hi}] outside signal span [{start},{end}]")
    return float(integrate_many(signal, np.array([lo]), np.array([hi]))[0].item())


def _coerce_signal(sig) -> PowerSignal:
    """Accept the reference's PowerSignal dataclass too."""
    segs = getattr(sig, "segments", ())
    samples = getattr(sig, "samples", ())
    return PowerSignal(segments=segs, samples=samples, period_us=getattr(sig, "period_us", None),
                       delay_us=getattr(sig, "delay_us", None))


def mean_power(signal: PowerSignal, interval: tuple[int, int]) -> float:
    lo, hi = interval
    if hi <= lo:
        return 0.0
    return integrate(signal, interval) * US_PER_S / (hi - lo)


# ----------------------------------------------------------------- sampler


def _sample_times(start: int, end: int, period_us: int) -> np.ndarray:
    k = (end - start) // period_us
    return start + period_us * np.arange(1, k + 1, dtype=np.int64)


def sample_signal(truth: PowerSignal, period_us: int = DEFAULT_SAMPLER_PERIOD_US,
                  delay_us: int = DEFAULT_SAMPLER_DELAY_US, seed: int = 0) -> PowerSignal:
    """Vendor-counter emulation (energy.py:144-172): samples every ``period_us``
    reading the truth at (t - delay), delay ~ U[0.5, 1.5] x ``delay_us`` drawn
    from numpy's PCG64 exactly as the reference draws it (one vectorised draw
    equals the reference's per-sample scalar draws).  The reads run on the GPU."""
    if not truth.is_ground_truth:
        raise SignalError("sample_signal requires a ground-truth signal")
    if period_us <= 0:
        raise SignalError("sampler period must be positive")
    rng = np.random.default_rng(seed)
    start, end = truth.span()
    times = _sample_times(start, end, period_us)
    if times.size == 0:
        times = np.array([end], dtype=np.int64)
    if delay_us:
        delays = rng.uniform(0.5 * delay_us, 1.5 * delay_us, size=times.size)
        query = times.astype(np.float64) - delays
    else:
        query = times.astype(np.float64)
    watts = _value_at(truth, query)
    return PowerSignal.from_columns(times, watts, kind="linear", period_us=period_us,
                                    delay_us=delay_us)


def sampled_view(trace, period_us: int = DEFAULT_SAMPLER_PERIOD_US,
                 delay_us: int = DEFAULT_SAMPLER_DELAY_US, seed: int = 0) -> PowerSignal:
    """sample_signal anchored at the span ends (energy.py:175-189)."""
    truth = ground_truth_signal(trace)
    sig = sample_signal(truth, period_us, delay_us, seed)
    start, end = truth.span()
    ts = _host(sig._ts)
    w = _host(sig._w)
    if ts[0] > start:
        ts = np.concatenate([[start], ts])
        w = np.concatenate([[w[0]], w])
    if ts[-1] < end:
        ts = np.concatenate([ts, [end]])
        w = np.concatenate([w, [w[-1]]])
    return PowerSignal.from_columns(ts.astype(np.int64), w.astype(np.float64), kind="linear",
                                    period_us=period_us, delay_us=delay_us)


# ----------------------------------------------------------------- ledger


class JoulesView(Mapping):
    """Read-only ``dict[str, float]`` view over a joules column (the
    reference's per_operator / per_kernel dicts, energy.py:268-269), in the
    reference's insertion order.  Values stay in HBM until first read."""

    def __init__(self, ids: Optional[Sequence[str]], joules: torch.Tensor, prefix: str = "op"):
        self._ids = ids
        self._dev = joules
        self._host = None
        self._index = None
        self._prefix = prefix

    @property
    def tensor(self) -> torch.Tensor:
        return self._dev

    def array(self) -> np.ndarray:
        if self._host is None:
            self._host = self._dev.cpu().numpy()
        return self._host

    def _id(self, i: int) -> str:
        return self._ids[i] if self._ids is not None else synthetic_id(self._prefix, i, len(self))

    def _idx(self):
        if self._index is None:
            n = len(self)
            if self._ids is not None:
                self._index = {k: i for i, k in enumerate(self._ids)}
            else:
                self._index = {k: i for i, k in enumerate(synthetic_ids(self._prefix, n))}
        return self._index

    def __getitem__(self, key):
        return float(self.array()[self._idx()[key]])

    def __iter__(self):
        if self._ids is not None:
            return iter(self._ids)
        return iter(synthetic_ids(self._prefix, len(self)))

    def __len__(self):
        return int(self._dev.numel())

    def __contains__(self, key):
        return key in self._idx()

    def values(self):
        return self.array().tolist()

    def items(self):
        return zip(iter(self), self.array().tolist())

    def __repr__(self):
        return f"JoulesView(n={len(self)})"

    def __eq__(self, other):
        if isinstance(other, Mapping):
            return dict(self.items()) == dict(other.items())
        return NotImplemented


@dataclass(frozen=True)
class EnergyLedger:
    """Per-kernel / per-operator joules plus the idle pseudo-operator
    (energy.py:263-277)."""

    method: str
    per_kernel: Mapping[str, float]
    per_operator: Mapping[str, float]
    idle_joules: float
    total_joules: float
    op_total: Optional[float] = None  # exact device sum (operator_total)

    def operator_total(self) -> float:
        if self.op_total is not None:
            return self.op_total
        return sum(self.per_operator.values())

    def subgraph_joules(self, op_ids: Iterable[str]) -> float:
        return sum(self.per_operator[o] for o in op_ids)

    def operator_tensor(self) -> Optional[torch.Tensor]:
        return getattr(self.per_operator, "tensor", None)

    def kernel_tensor(self) -> Optional[torch.Tensor]:
        return getattr(self.per_kernel, "tensor", None)


class _PendingStatus:
    """A ledger's status block read in two steps (dw_status_copy now,
    dw_status_decode when needed), so the next launches queue before the host
    waits for this one."""

    def __init__(self, ws: torch.Tensor, stream):
        L = _native.lib()
        self.host = torch.empty(_native.DW_STATUS_BYTES, dtype=torch.uint8, pin_memory=True)
        _native.check(L.dw_status_copy(ws.data_ptr(), self.host.data_ptr(), stream), "dw_status_copy")
        self.done = torch.cuda.Event()
        self.done.record()

    def result(self):
        self.done.synchronize()
        st = _native.Status()
        _native.lib().dw_status_decode(self.host.data_ptr(), ctypes.byref(st))
        return st


def _run_ledger(cols: TraceColumns, sig: PowerSignal, validate_order: bool, summation: str = "reference",
                defer: bool = False):
    """dw_ledger on the device; returns (per_op, per_k, status) -- with
    ``defer`` the status as a _PendingStatus (read later)."""
    dev = _native.device()
    L = _native.lib()
    op_s, op_e = cols.device("op_start"), cols.device("op_end")
    k_s, k_e = cols.device("k_start"), cols.device("k_end")
    per_op = torch.empty(cols.n_ops, dtype=torch.float64, device=dev)
    per_k = torch.empty(cols.n_kernels, dtype=torch.float64, device=dev)
    ops = _native.IntervalSet(_native.ptr(op_s), _native.ptr(op_e), cols.n_ops,
                              _native.ptr(per_op), 1 if cols.ops_sorted else 0, 0)
    kers = _native.IntervalSet(_native.ptr(k_s), _native.ptr(k_e), cols.n_kernels,
                               _native.ptr(per_k), 1 if cols.kernels_sorted else 0, 0)
    csig, keep = sig._c_signal(validate_order, summation)
    sizes = (ctypes.c_int64 * 2)(cols.n_ops, cols.n_kernels)
    nbytes = L.dw_attribute_workspace_size(csig.n, sizes, 2)
    ws = _native.Workspace.get(nbytes)
    stream = _native.stream_handle()
    _native.check(L.dw_ledger(ctypes.byref(csig), ctypes.byref(ops), ctypes.byref(kers),
                              ws.data_ptr(), ws.numel(), stream), "dw_ledger")
    if defer:
        return per_op, per_k, _PendingStatus(ws, stream)
    st = _native.Status()
    L.dw_status(ws.data_ptr(), stream, ctypes.byref(st))
    return per_op, per_k, st


def _raise_ledger_errors(cols: TraceColumns, st, span):
    """First failing interval in build_ledger's iteration order (op, then its
    kernels; energy.py:305-316) raises the reference's SignalError.  ``span``:
    the signal's span, or a callable returning it (read only on an error)."""
    if st.order_index >= 0:
        from .trace_model import TraceError
        raise TraceError("power samples must be strictly increasing in timestamp")
    for j in (0, 1):
        if st.unsorted_index[j] >= 0:
            raise RuntimeError("internal: interval set flagged sorted is not sorted")
    bad_op, bad_k = st.bad_index[0], st.bad_index[1]
    if bad_op < 0 and bad_k < 0:
        return
    owner = None
    if bad_k >= 0:
        k_op = cols.k_op
        owner = int(k_op[bad_k].item() if isinstance(k_op, torch.Tensor) else k_op[bad_k]) \
            if k_op is not None else bad_k
    if bad_op >= 0 and (owner is None or bad_op <= owner):
        lo, hi = _read_pair(cols, "op_start", "op_end", bad_op)
    else:
        lo, hi = _read_pair(cols, "k_start", "k_end", bad_k)
    _raise_interval_error(lo, hi, span() if callable(span) else span)


def _read_pair(cols, a, b, i):
    x, y = getattr(cols, a), getattr(cols, b)
    if isinstance(x, torch.Tensor):
        return int(x[i].item()), int(y[i].item())
    return int(x[i]), int(y[i])


# ------------------------------------------------------------------ replay


@dataclass(frozen=True)
class ReplayEstimate:
    op_id: str
    watts: float
    joules: float
    repeat: int
    samples_used: int


def _sampler_delays(n: int, delay_us: int, seed: int) -> np.ndarray:
    """The delayed sampler's per-sample delays (energy.py:160-165): every
    replay restarts the seeded numpy stream, so one array serves all ops
    (rng.uniform(a, b, size=n) draws exactly what n scalar calls draw)."""
    if not delay_us:
        return np.zeros(max(n, 1))
    return np.random.default_rng(seed).uniform(0.5 * delay_us, 1.5 * delay_us, size=max(n, 1))


def _replay_device(truth: PowerSignal, starts, ends, repeat, period_us, delay_us, seed):
    """dw_replay over operators [starts, ends): (watts, joules) device tensors."""
    dev = _native.device()
    s_d = _to_dev(starts, torch.int64, dev).reshape(-1)
    e_d = _to_dev(ends, torch.int64, dev).reshape(-1)
    n = int(s_d.numel())
    dmax = int((e_d - s_d).max().item()) if n else 0
    delays = torch.from_numpy(_sampler_delays(repeat * dmax // period_us + 2, delay_us, seed)).to(dev)
    watts = torch.empty(n, dtype=torch.float64, device=dev)
    joules = torch.empty(n, dtype=torch.float64, device=dev)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    csig, keep = truth._c_signal()
    L = _native.lib()
    _native.check(L.dw_replay(ctypes.byref(csig), _native.ptr(s_d), _native.ptr(e_d), n, int(repeat),
                              int(period_us), _native.ptr(delays), int(delays.numel()), _native.ptr(watts),
                              _native.ptr(joules), _native.ptr(bad), _native.stream_handle()), "dw_replay")
    b = int(bad.item())
    if 0 <= b < (1 << 62):
        raise SignalError("sample_signal requires a ground-truth signal")
    return watts, joules


def _kernel_owners(cols: TraceColumns) -> torch.Tensor:
    """Owning operator of every kernel (device int64).  From ``k_op`` when the
    columns carry it; otherwise (packed columns ship none) by containment,
    which is exact when operators are sorted and pairwise disjoint and
    kernels sorted, since every kernel lies inside its owner (the trace
    validation, trace_model.py:529-540).  Anything else raises."""
    if cols.k_op is not None:
        return cols.device("k_op").to(torch.int64)
    s, e = cols.device("op_start"), cols.device("op_end")
    ks, ke = cols.device("k_start"), cols.device("k_end")
    ok = bool(s.numel()) and cols.ops_sorted and cols.kernels_sorted and (
        s.numel() < 2 or bool((s[1:] >= e[:-1]).all().item()))
    if ok:
        own = torch.searchsorted(s, ks, right=True) - 1
        oc = own.clamp(min=0)
        ok = bool(((own >= 0) & (ks >= s[oc]) & (ke <= e[oc])).all().item())
    if not ok:
        raise ValueError("replay needs each kernel's operator: the columns carry no k_op and the "
                         "kernels are not contained in sorted, disjoint operators")
    return own


def _replay_checks(cols: TraceColumns, repeat: int, first_op: int = 0) -> None:
    """replay_estimate's argument errors in build_ledger's op order
    (energy.py:227-230): an op without kernels, then repeat < 1.  The
    kernel-less scan runs on the device (one scatter, one reduction)."""
    n = cols.n_ops - first_op
    first_missing = None
    if n > 0:
        dev = _native.device()
        has = torch.zeros(cols.n_ops, dtype=torch.bool, device=dev)
        if cols.n_kernels:
            has[_kernel_owners(cols)] = True
        miss = ~has[first_op:]
        if bool(miss.any().item()):
            first_missing = int(torch.argmax(miss.to(torch.int8)).item()) + first_op
    if first_missing == first_op:
        oid = cols.op_ids[first_missing] if cols.op_ids is not None else synthetic_id("op", first_missing, cols.n_ops)
        raise SignalError(f"operator {oid!r} launched no kernels; nothing to replay")
    if repeat < 1:
        raise SignalError("repeat must be >= 1")
    if first_missing is not None:
        oid = cols.op_ids[first_missing] if cols.op_ids is not None else synthetic_id("op", first_missing, cols.n_ops)
        raise SignalError(f"operator {oid!r} launched no kernels; nothing to replay")


def _replay_ledger(cols: TraceColumns, truth: PowerSignal, repeat, period_us, delay_us, seed) -> EnergyLedger:
    """build_ledger(method="replay") (energy.py:306-311, 318-319): per-op
    replay estimates, kernels at their op's steady watts, total = the ground
    truth over the span, idle = max(total - sum, 0)."""
    _replay_checks(cols, repeat)
    cols.wait_ready()
    tsig = PowerSignal.from_columns(cols.device("ts"), cols.device("watts"), truth._span_hi, "step")
    watts, per_op = _replay_device(tsig, cols.device("op_start"), cols.device("op_end"), repeat, period_us,
                                   delay_us, seed)
    k_op = _kernel_owners(cols) if cols.n_kernels else None
    kdur = (cols.device("k_end") - cols.device("k_start")).to(torch.float64)
    # tensor / tensor: an IEEE division per element (a scalar divisor may be
    # turned into a reciprocal multiply)
    per_k = torch.div(watts[k_op] * kdur, torch.full_like(kdur, float(US_PER_S))) if cols.n_kernels else kdur
    empty = cols.device("op_start")[:0]
    totals = _span_total(tsig, empty)
    op_total = _fx_sum(per_op)
    return EnergyLedger(method="replay", per_kernel=JoulesView(cols.k_ids, per_k, "k"),
                        per_operator=JoulesView(cols.op_ids, per_op, "op"),
                        idle_joules=max(totals - op_total, 0.0), total_joules=totals, op_total=op_total)


def _span_total(sig: PowerSignal, empty: torch.Tensor) -> float:
    """The ledger total over the whole span (dw_ledger with no intervals)."""
    L = _native.lib()
    e = _native.IntervalSet(_native.ptr(empty), _native.ptr(empty), 0, 0, 1, 0)
    csig, keep = sig._c_signal()
    sizes = (ctypes.c_int64 * 2)(0, 0)
    ws = _native.Workspace.get(L.dw_attribute_workspace_size(csig.n, sizes, 2))
    stream = _native.stream_handle()
    _native.check(L.dw_ledger(ctypes.byref(csig), ctypes.byref(e), ctypes.byref(e), ws.data_ptr(), ws.numel(),
                              stream), "dw_ledger")
    st = _native.Status()
    L.dw_status(ws.data_ptr(), stream, ctypes.byref(st))
    return float(st.totals[0])


def replay_estimate(trace, op_id: str, repeat: int = DEFAULT_REPLAY_REPEAT,
                    period_us: int = DEFAULT_SAMPLER_PERIOD_US, delay_us: int = DEFAULT_SAMPLER_DELAY_US,
                    seed: int = 0) -> ReplayEstimate:
    """Estimate one operator's steady power by replaying it back to back
    (energy.py:208-256) -- the replay kernel on one operator."""
    cols = TraceColumns.from_trace(trace)
    ids = list(cols.op_ids) if cols.op_ids is not None else synthetic_ids("op", cols.n_ops)
    try:
        i = ids.index(op_id)
    except ValueError:
        raise KeyError(op_id) from None
    k_op = cols.k_op.cpu().numpy() if isinstance(cols.k_op, torch.Tensor) else np.asarray(
        cols.k_op if cols.k_op is not None else [], dtype=np.int64)
    if not np.any(k_op == i):
        raise SignalError(f"operator {op_id!r} launched no kernels; nothing to replay")
    if repeat < 1:
        raise SignalError("repeat must be >= 1")
    truth = ground_truth_signal(cols)
    tsig = PowerSignal.from_columns(cols.device("ts"), cols.device("watts"), truth._span_hi, "step")
    lo, hi = int(_host(cols.op_start)[i]), int(_host(cols.op_end)[i])
    watts, joules = _replay_device(tsig, np.array([lo]), np.array([hi]), repeat, period_us, delay_us, seed)
    # samples used: the mid-window reads (energy.py:245-248)
    ts = _host(cols.ts)
    d = hi - lo
    a = max(int(np.searchsorted(ts, lo, side="right")) - 1, 0)
    b = int(np.searchsorted(ts, hi, side="left")) - 1
    p0s = max(int(ts[a]), lo) - lo
    seg_end_b = int(ts[b + 1]) if b + 1 < len(ts) else truth._span_hi
    ple = min(seg_end_b, hi) - lo
    sr, er = p0s, (repeat - 1) * d + ple
    total = float(repeat * d)
    lo_m, hi_m = 0.1 * total, (1.0 - 0.1) * total
    t = np.arange(sr + period_us, er + 1, period_us, dtype=np.int64) if er >= sr + period_us else np.array([er])
    used = int(np.count_nonzero((lo_m <= t) & (t <= hi_m))) or int(t.size)
    return ReplayEstimate(op_id=op_id, watts=float(watts.item()), joules=float(joules.item()), repeat=repeat,
                          samples_used=used)


def _split_ledger(method: str, cols: TraceColumns, signal: PowerSignal, st) -> EnergyLedger:
    """Split-mode ledger: the compat pass above validated the intervals and
    integrated the span (total); here each set is split among its concurrently
    active intervals and idle = max(total - exact sum of operators, 0)."""
    per_op = integrate_split(signal, cols.device("op_start"), cols.device("op_end"))
    per_k = integrate_split(signal, cols.device("k_start"), cols.device("k_end"))
    op_total = _fx_sum(per_op)
    total = float(st.totals[0])
    return EnergyLedger(method=method, per_kernel=JoulesView(cols.k_ids, per_k, "k"),
                        per_operator=JoulesView(cols.op_ids, per_op, "op"),
                        idle_joules=max(total - op_total, 0.0), total_joules=total, op_total=op_total)


def _fx_sum(x: torch.Tensor) -> float:
    L = _native.lib()
    out = torch.zeros(1, dtype=torch.float64, device=x.device)
    ws = _native.Workspace.get(L.dw_fx_sum_workspace_size(x.numel()))
    _native.check(L.dw_fx_sum(_native.ptr(x), x.numel(), _native.ptr(out), ws.data_ptr(), ws.numel(),
                              _native.stream_handle()), "dw_fx_sum")
    return float(out.item())


def build_ledger(trace, method: str = "ground_truth",
                 period_us: int = DEFAULT_SAMPLER_PERIOD_US,
                 delay_us: int = DEFAULT_SAMPLER_DELAY_US, repeat: int = DEFAULT_REPLAY_REPEAT,
                 seed: int = 0, validate_order: bool = False, overlap: str = "compat",
                 summation: str = "reference") -> EnergyLedger:
    """Attribute energy to kernels and operators (energy.py:280-331).

    ``summation="reference"`` (default) sums each interval's pieces in the
    reference's order (bit-identical to energy.integrate up to DW_DIRECT_MAX
    pieces); ``summation="exact"`` sums them exactly in fixed point and
    rounds once -- the scale path's mode (pipeline.analyze, bench.py), within
    a few ulps of the reference and bit-identical to the oracle's MODE_EXACT.

    ``overlap="compat"`` (default) is the reference: every interval gets the
    full signal over its span.  ``overlap="split"`` divides the power among
    concurrently active operators (and, separately, kernels) -- see
    ``integrate_split``; idle is then the energy outside every operator.

    ``trace`` is a reference-style Trace (the reference's own objects work) or a
    TraceColumns.  Gaps between kernels inside an operator's interval go to the
    operator; gaps between operators go to ``idle``.
    """
    return _begin_ledger(trace, method, period_us, delay_us, repeat, seed, validate_order, overlap,
                         summation)()


def _begin_ledger(trace, method="ground_truth", period_us=DEFAULT_SAMPLER_PERIOD_US,
                  delay_us=DEFAULT_SAMPLER_DELAY_US, repeat=DEFAULT_REPLAY_REPEAT, seed=0,
                  validate_order=False, overlap="compat", summation="reference"):
    """build_ledger in two halves: the launches now, then a callable that
    waits for the status, raises build_ledger's errors (same order: the
    argument checks here, the data errors in the callable) and returns the
    EnergyLedger.  pipeline.analyze launches both traces' ledgers before it
    waits for either."""
    if method not in METHODS and method not in EXTRA_METHODS:
        raise ValueError(f"unknown energy method {method!r}")
    if overlap not in ("compat", "split"):
        raise ValueError(f"unknown overlap mode {overlap!r}")
    _sum_mode(summation)
    cols = TraceColumns.from_trace(trace)
    if method == "samples":
        if cols.n_power == 0:
            raise SignalError("trace carries no power records")
        cols.wait_ready()
        first, last = cols._first_last_ts()
        signal = PowerSignal.from_columns(cols.device("ts"), cols.device("watts"), span_hi=last, kind="linear",
                                          first=first)
        return _finish_ledger(method, cols, signal, signal.span, overlap,
                              _run_ledger(cols, signal, validate_order, summation, defer=True))
    truth = ground_truth_signal(cols)
    if method == "replay":
        led = _replay_ledger(cols, truth, repeat, period_us, delay_us, seed)
        return lambda: led
    if method == "ground_truth":
        cols.wait_ready()
        signal = PowerSignal.from_columns(cols.device("ts"), cols.device("watts"),
                                          truth._span_hi, "step")
    else:
        signal = sampled_view(cols, period_us, delay_us, seed)
    return _finish_ledger(method, cols, signal, truth.span(), overlap,
                          _run_ledger(cols, signal, validate_order, summation, defer=True))


def _finish_ledger(method, cols, signal, span, overlap, launched):
    per_op, per_k, pending = launched
    if overlap == "split":
        # checked and split now, not when the ledger is read: the split
        # integrals queued early overlap whatever the caller does next
        st = pending.result()
        _raise_ledger_errors(cols, st, span)
        led = _split_ledger(method, cols, signal, st)
        return lambda: led

    def finish() -> EnergyLedger:
        st = pending.result()
        _raise_ledger_errors(cols, st, span)
        return EnergyLedger(method=method, per_kernel=JoulesView(cols.k_ids, per_k, "k"),
                            per_operator=JoulesView(cols.op_ids, per_op, "op"),
                            idle_joules=float(st.totals[2]), total_joules=float(st.totals[0]),
                            op_total=float(st.totals[1]))
    return finish
