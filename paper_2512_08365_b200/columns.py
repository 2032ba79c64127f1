"""Columnar (SoA) trace buffers -- the ingestion side of the hot path.

The reference keeps a trace as frozen dataclasses (trace_model.py:241-314) and
walks them per interval.  Here a trace becomes flat columns (DESIGN.md "Data
layout"):

    power    ts int64[S] (strictly increasing), watts f64[S]
    ops      start, end int64[N]          (trace order)
    kernels  start, end int64[K], op int32[K]   (flattened in op.kernel_ids order,
                                                 i.e. build_ledger's iteration order)

plus optional per-op columns for the signature join (sig u64, work f64, rank
int64).  Columns are numpy on the host and move to HBM once (``device()``);
scale workloads can be constructed directly from device tensors.
"""

from __future__ import annotations

import math
import weakref
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native


def synthetic_id(prefix: str, i: int, n: int) -> str:
    """Name of item ``i`` of ``n`` in columns that carry no ids: zero-padded to
    the width of ``n - 1``, so lexicographic order (the report's nodes_a
    tie-break, detect.py:263-266) equals index order.  Every view of such
    columns (ledgers, detect, join findings, diagnosis) uses this name."""
    return f"{prefix}{i:0{len(str(max(n - 1, 0)))}d}"


def synthetic_ids(prefix: str, n: int) -> list:
    w = len(str(max(n - 1, 0)))
    return [f"{prefix}{i:0{w}d}" for i in range(n)]


def _np_i64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def _is_sorted(a) -> bool:
    if isinstance(a, torch.Tensor):
        return bool(a.numel() < 2 or bool((a[1:] >= a[:-1]).all().item()))
    return bool(a.shape[0] < 2 or np.all(a[1:] >= a[:-1]))


@dataclass
class TraceColumns:
    ts: object                  # int64[S]   numpy or torch (cuda)
    watts: object               # f64[S]
    trace_end: int              # Trace.span_us()[1] (trace_model.py:307-314)
    op_start: object            # int64[N]
    op_end: object              # int64[N]
    k_start: object             # int64[K]
    k_end: object               # int64[K]
    k_op: object = None         # int32[K] owner op index
    op_ids: Optional[Sequence[str]] = None
    k_ids: Optional[Sequence[str]] = None
    op_names: Optional[Sequence[str]] = None
    k_names: Optional[Sequence[str]] = None   # kernel names, k_* row order (diagnosis)
    op_sig: object = None       # uint64[N] signature hash (join)
    op_work: object = None      # f64[N] useful work per op (join)
    op_rank: object = None      # int64[N] lexicographic rank of op ids
    ops_sorted: Optional[bool] = None
    kernels_sorted: Optional[bool] = None
    _dev: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        if self.ops_sorted is None:
            self.ops_sorted = _is_sorted(self.op_start)
        if self.kernels_sorted is None:
            self.kernels_sorted = _is_sorted(self.k_start)

    # ------------------------------------------------------------ sizes
    @property
    def n_power(self) -> int:
        return int(self.ts.shape[0])

    @property
    def n_ops(self) -> int:
        return int(self.op_start.shape[0])

    @property
    def n_kernels(self) -> int:
        return int(self.k_start.shape[0])

    def signal_span(self) -> tuple[int, int]:
        """Ground-truth span: (first power ts, max(trace end, last ts + 1))
        -- PowerSignal.from_breakpoints (energy.py:68-82)."""
        first, last = self._first_last_ts()
        return first, max(int(self.trace_end), last + 1)

    def _first_last_ts(self) -> tuple[int, int]:
        if "first_last" not in self._dev:
            if isinstance(self.ts, torch.Tensor):
                fl = torch.stack([self.ts[0], self.ts[-1]]).cpu().tolist()
            else:
                fl = [int(self.ts[0]), int(self.ts[-1])]
            self._dev["first_last"] = (int(fl[0]), int(fl[1]))
        return self._dev["first_last"]

    # ------------------------------------------------------------ device
    def device(self, name: str) -> torch.Tensor:
        """The column ``name`` resident in HBM on the current CUDA device."""
        dev = _native.device()
        key = (name, dev.index)
        t = self._dev.get(key)
        if t is None:
            src = getattr(self, name)
            if src is None:
                return None
            if isinstance(src, torch.Tensor):
                t = src.to(dev, non_blocking=True).contiguous()
            else:
                t = torch.from_numpy(np.ascontiguousarray(src)).to(dev, non_blocking=True)
            self._dev[key] = t
        return t

    HOT = ("ts", "watts", "op_start", "op_end", "k_start", "k_end", "op_sig")

    def prefetch(self, stream: "torch.cuda.Stream", names=HOT,
                 decode_stream: "torch.cuda.Stream | None" = None) -> "torch.cuda.Event":
        """Start the host->HBM copies of ``names`` on ``stream`` (pinned host
        buffers copy asynchronously); later device() calls on another stream
        wait for them (``wait_ready``, or the returned event).  Unpacked
        columns need no decode (``decode_stream`` is for PackedColumns)."""
        dev = _native.device()
        with torch.cuda.stream(stream):
            for n in names:
                if getattr(self, n) is not None:
                    self.device(n)
            ev = torch.cuda.Event()
            ev.record(stream)
        self._dev["__ready__"] = ev
        return ev

    def wait_ready(self) -> None:
        ev = self._dev.pop("__ready__", None)
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def drop_device(self) -> None:
        """Forget the HBM copies (the next device() call copies again)."""
        for k in [k for k in self._dev if isinstance(k, tuple)]:
            del self._dev[k]

    def host(self, name: str) -> np.ndarray:
        src = getattr(self, name)
        if isinstance(src, torch.Tensor):
            return src.cpu().numpy()
        return src

    # ------------------------------------------------------------ builders
    @classmethod
    def from_arrays(cls, ts, watts, op_start, op_end, k_start=None, k_end=None, k_op=None,
                    trace_end=None, **kw) -> "TraceColumns":
        """Columns from arrays (numpy or torch).  ``trace_end`` defaults to the
        max over all timestamps, as Trace.span_us() computes it."""
        if k_start is None:
            k_start = np.zeros(0, dtype=np.int64) if not isinstance(op_start, torch.Tensor) \
                else op_start.new_zeros(0)
            k_end = k_start
        if trace_end is None:
            parts = []
            for a in (ts, op_end, k_end):
                if a is None or a.shape[0] == 0:
                    continue
                parts.append(int(a.max().item() if isinstance(a, torch.Tensor) else a.max()))
            trace_end = max(parts) if parts else 0
        return cls(ts=ts, watts=watts, trace_end=int(trace_end), op_start=op_start,
                   op_end=op_end, k_start=k_start, k_end=k_end, k_op=k_op, **kw)

    @classmethod
    def from_trace(cls, trace) -> "TraceColumns":
        """Columns of a reference-style ``Trace`` (the reference's own objects
        or paper_2512_08365_b200.trace_model.Trace).  Cached per trace object."""
        if isinstance(trace, TraceColumns):
            return trace
        cached = _CACHE.get(id(trace))
        if cached is not None and cached[0]() is trace:
            return cached[1]
        power = trace.power
        ts = np.fromiter((p.timestamp for p in power), dtype=np.int64, count=len(power))
        watts = np.fromiter((p.watts for p in power), dtype=np.float64, count=len(power))
        ops = trace.operators
        n = len(ops)
        op_start = np.fromiter((o.start for o in ops), dtype=np.int64, count=n)
        op_end = np.fromiter((o.end for o in ops), dtype=np.int64, count=n)
        k_ids, k_names, k_start, k_end, k_op = [], [], [], [], []
        kernels = trace.kernels
        for i, o in enumerate(ops):
            for kid in o.kernel_ids:
                k = kernels[kid]
                k_ids.append(kid)
                k_names.append(k.kernel_name)
                k_start.append(k.start)
                k_end.append(k.end)
                k_op.append(i)
        k_start = np.asarray(k_start, dtype=np.int64)
        k_end = np.asarray(k_end, dtype=np.int64)
        # Trace.span_us (trace_model.py:307-314) covers every kernel, owned or not
        ends = [int(ts.max()) if ts.size else None, int(op_end.max()) if n else None,
                int(op_start.max()) if n else None]
        ends += [max((k.end for k in kernels.values()), default=None),
                 max((k.start for k in kernels.values()), default=None)]
        ends = [e for e in ends if e is not None]
        cols = cls(ts=ts, watts=watts, trace_end=max(ends) if ends else 0, op_start=op_start,
                   op_end=op_end, k_start=k_start, k_end=k_end,
                   k_op=np.asarray(k_op, dtype=np.int32), op_ids=[o.op_id for o in ops],
                   k_ids=k_ids, op_names=[o.op_name for o in ops], k_names=k_names)
        try:
            _CACHE[id(trace)] = (weakref.ref(trace), cols)
            while len(_CACHE) > _CACHE_MAX:
                _CACHE.pop(next(iter(_CACHE)))
        except TypeError:
            pass
        return cols


_CACHE: dict = {}
_CACHE_MAX = 32


# ------------------------------------------------------------- packed columns


def _unsigned(d):
    """int64 values of a 16/32-bit unsigned column held in a signed or
    unsigned container (torch or numpy)."""
    if isinstance(d, torch.Tensor):
        mask = 0xFFFF if d.element_size() == 2 else 0xFFFFFFFF
        return d.to(torch.int64) & mask
    d = np.asarray(d)
    return d.view(np.uint16 if d.itemsize == 2 else np.uint32).astype(np.int64)


class PackedColumns(TraceColumns):
    """A trace whose sorted timestamp columns travel as deltas, whose interval
    ends travel as durations and whose watts travel as 9-digit decimal codes
    (DESIGN.md "packed columns").

    Each delta / duration column is 16-bit when every value fits, else 32-bit;
    watts are uint32 codes (``watts_p0`` set, ``dw_unpack_decimal``) when every
    sample is a 9-significant-digit decimal -- the trace format's on-disk
    precision (trace_model.py:63-65) -- else f64.  At C4: host bytes per
    sample 16 -> 6, per interval 16 -> 4.  The host->HBM copy bounds the
    end-to-end path, so this is what a deployment ships (and what
    ``save_packed`` writes).  ``device(name)`` decodes on the GPU (one scan
    per timestamp column, one pass for the watts) and caches the full columns.
    Host attributes: ``ts``/``op_start``/``k_start`` hold the deltas (``*_base``
    the first value), ``op_end``/``k_end`` the durations.
    """

    PACKED = ("ts", "op_start", "k_start")

    def __init__(self, ts_base, ts_delta, watts, op_base, op_delta, op_dur, k_base, k_delta, k_dur,
                 trace_end, k_op=None, op_sig=None, watts_p0=None, ts_bias=0, op_sig_dict=None,
                 ts_bits=None, n_power=None, ts_last=None, iv_bits=None, n_ops=None, n_kernels=None,
                 sig_bits=None, watts_rep=None, ts_step=None, watts_bits=None, **kw):
        super().__init__(ts=ts_delta, watts=watts, trace_end=int(trace_end), op_start=op_delta, op_end=op_dur,
                         k_start=k_delta, k_end=k_dur, k_op=k_op, op_sig=op_sig, ops_sorted=True,
                         kernels_sorted=True, **kw)
        self.ts_base, self.op_start_base, self.k_start_base = int(ts_base), int(op_base), int(k_base)
        self.watts_p0 = None if watts_p0 is None else int(watts_p0)
        # run-coded watts: bitmap of the samples carrying a new code (u32
        # words); ``watts`` then holds those samples' codes only
        self.watts_rep = watts_rep
        if watts_rep is not None and self.watts_p0 is None:
            raise ValueError("run-coded watts need decimal codes (watts_p0)")
        # run-coded watts whose stored codes are bit-packed: (width, bias)
        self.watts_bits = None if watts_bits is None else (int(watts_bits[0]), int(watts_bits[1]))
        if self.watts_bits is not None and watts_rep is None:
            raise ValueError("bit-packed watts codes are run-coded (watts_rep)")
        self.ts_bias = int(ts_bias)          # int8 / bit-packed ts deltas: delta = ts_bias + code
        self.op_sig_dict = op_sig_dict       # op_sig holds u16/u32 codes into this u64 dictionary
        self.ts_bits = None if ts_bits is None else int(ts_bits)  # ts holds bit-packed 32-bit words
        # grid-coded timestamps (ts_bits set): fields are residuals from
        # ts_base + floor(i * ts_step / 2^32) instead of deltas (dw_unpack_grid)
        self.ts_step = None if ts_step is None else int(ts_step)
        if self.ts_step is not None and self.ts_bits is None:
            raise ValueError("grid-coded timestamps are bit-packed (ts_bits)")
        if self.ts_bits is not None:
            self._n_power, self._ts_last = int(n_power), int(ts_last)
            self._dev["first_last"] = (self.ts_base, self._ts_last)
        # bit-packed interval columns: name -> (width, bias); op_start / k_start
        # hold packed deltas, op_end / k_end packed durations
        self.iv_bits = dict(iv_bits or {})
        self.sig_bits = None if sig_bits is None else int(sig_bits)  # op_sig: bit-packed dictionary codes
        self._n_ops = None if n_ops is None else int(n_ops)
        self._n_kernels = None if n_kernels is None else int(n_kernels)

    @property
    def n_power(self) -> int:
        return self._n_power if self.ts_bits is not None else super().n_power

    @property
    def n_ops(self) -> int:
        return self._n_ops if "op_start" in self.iv_bits else super().n_ops

    @property
    def n_kernels(self) -> int:
        return self._n_kernels if "k_start" in self.iv_bits else super().n_kernels
        self._first_last = None

    def _first_last_ts(self) -> tuple[int, int]:
        if "first_last" not in self._dev:
            t = self.ts
            if (t.element_size() if isinstance(t, torch.Tensor) else np.asarray(t).itemsize) == 1:
                dd = (t.to(torch.int64) if isinstance(t, torch.Tensor) else np.asarray(t).astype(np.int64)) \
                    + self.ts_bias  # biased int8 deltas
                dd[0] = 0
            else:
                dd = _unsigned(t)
            last = self.ts_base + int(dd.sum())
            first = self.ts_base + int(dd[0])
            self._dev["first_last"] = (first, last)
        return self._dev["first_last"]

    def _staged(self, name, dev):
        """The packed column in HBM: staged by prefetch(), else copied now."""
        t = self._dev.pop(("raw", name, dev.index), None)
        return t if t is not None else self._raw(name).to(dev, non_blocking=True)

    def prefetch(self, stream: "torch.cuda.Stream", names=TraceColumns.HOT,
                 decode_stream: "torch.cuda.Stream | None" = None) -> "torch.cuda.Event":
        """All host->HBM copies of ``names`` first (event ``copied``), then the
        decodes: a copy queued behind this one (another trace) waits for the
        transfers only.  With ``decode_stream`` each column decodes there as
        soon as its own transfer has landed, under the transfers after it."""
        dev = _native.device()
        raw = {"op_end": "op_start", "k_end": "k_start"}
        groups = []
        with torch.cuda.stream(stream):
            for n in names:
                staged = []
                # companions travel with their column: a decode never issues a
                # copy of its own (it would queue behind every transfer
                # already waiting on the copy engine)
                for m in (n, {"op_start": "op_end", "k_start": "k_end", "watts": "watts_rep",
                              "op_sig": "op_sig_dict"}.get(n), raw.get(n)):
                    if m is None or getattr(self, m) is None or (m, dev.index) in self._dev \
                            or ("raw", m, dev.index) in self._dev:
                        continue
                    t = self._raw(m).to(dev, non_blocking=True)
                    self._dev[("raw", m, dev.index)] = t
                    staged.append(t)
                if decode_stream is not None:
                    ev = None
                    if staged:
                        ev = torch.cuda.Event()
                        ev.record(stream)
                    groups.append((n, ev, staged))
            copied = torch.cuda.Event()
            copied.record(stream)
        self.copied = copied
        if decode_stream is None:
            return super().prefetch(stream, names)
        with torch.cuda.stream(decode_stream):
            for n, ev, staged in groups:
                if ev is not None:
                    decode_stream.wait_event(ev)  # this column's transfer only
                for t in staged:  # allocated on the copy stream, read on the decode stream
                    t.record_stream(decode_stream)
                if getattr(self, n) is not None:
                    self.device(n)
            ready = torch.cuda.Event()
            ready.record(decode_stream)
        self._dev["__ready__"] = ready
        return ready

    def _raw(self, name):
        src = getattr(self, name)
        if name == "op_sig_dict" and not isinstance(src, torch.Tensor):
            return torch.from_numpy(np.ascontiguousarray(np.asarray(src).view(np.int64)))
        if isinstance(src, torch.Tensor):
            return src
        a = np.ascontiguousarray(src)
        if a.dtype in (np.uint16, np.uint32):  # same bits in the signed type torch handles everywhere
            a = a.view(np.int16 if a.itemsize == 2 else np.int32)
        return torch.from_numpy(a)

    def device(self, name: str) -> torch.Tensor:
        if name == "watts" and self.watts_p0 is not None:
            return self._device_watts()
        if name == "op_sig" and self.op_sig_dict is not None:
            return self._device_sig()
        if name not in ("ts", "op_start", "op_end", "k_start", "k_end"):
            return super().device(name)
        dev = _native.device()
        key = (name, dev.index)
        t = self._dev.get(key)
        if t is not None:
            return t
        base_name = {"op_end": "op_start", "k_end": "k_start"}.get(name, name)
        delta = self._staged(base_name, dev)
        dur_name = {"op_start": "op_end", "k_start": "k_end"}.get(base_name)
        dur = self._staged(dur_name, dev) if dur_name is not None else None
        end = dur  # placeholder: decoded ends are allocated by the branch that fills them
        base = {"ts": self.ts_base, "op_start": self.op_start_base, "k_start": self.k_start_base}[base_name]
        L = _native.lib()
        bias = self.ts_bias if base_name == "ts" else 0
        if base_name == "ts" and self.ts_bits is not None:
            n = self._n_power
            out = torch.empty(n, dtype=torch.int64, device=dev)
            ws = _native.Workspace.get(L.dw_unpack_workspace_size(n))
            if self.ts_step is not None:
                _native.check(L.dw_unpack_grid(_native.ptr(delta), self.ts_bits, bias, n, base, self.ts_step,
                                               _native.ptr(out), _native.stream_handle()), "dw_unpack_grid")
            else:
                _native.check(L.dw_unpack_bits(_native.ptr(delta), self.ts_bits, bias, n, base, _native.ptr(out),
                                               ws.data_ptr(), ws.numel(), _native.stream_handle()), "dw_unpack_bits")
            self._dev[("ts", dev.index)] = out
            return out
        if base_name in self.iv_bits:
            n = self._n_ops if base_name == "op_start" else self._n_kernels
            out = torch.empty(n, dtype=torch.int64, device=dev)
            ws = _native.Workspace.get(L.dw_unpack_workspace_size(n))
            w, b = self.iv_bits[base_name]
            wd, bd = self.iv_bits[dur_name] if end is not None else (1, 0)
            if end is not None:
                end = torch.empty(n, dtype=torch.int64, device=dev)
            # starts and ends in one pass
            _native.check(L.dw_unpack_bits_w(_native.ptr(delta), w, b, n, base, _native.ptr(out),
                                             _native.ptr(dur) if end is not None else None, wd, bd, _native.ptr(end),
                                             ws.data_ptr(), ws.numel(), _native.stream_handle()), "dw_unpack_bits_w")
            self._dev[(base_name, dev.index)] = out
            if end is not None:
                self._dev[(dur_name, dev.index)] = end
            return self._dev[key]
        n = int(delta.numel())
        out = torch.empty(n, dtype=torch.int64, device=dev)
        end = torch.empty(n, dtype=torch.int64, device=dev) if dur is not None else None
        ws = _native.Workspace.get(L.dw_unpack_workspace_size(n))
        _native.check(L.dw_unpack_deltas_w(_native.ptr(delta), delta.element_size(), bias, n, base, _native.ptr(out),
                                           _native.ptr(dur) if end is not None else None,
                                           dur.element_size() if end is not None else 4, _native.ptr(end),
                                           ws.data_ptr(), ws.numel(), _native.stream_handle()),
                      "dw_unpack_deltas_w")
        self._dev[(base_name, dev.index)] = out
        if end is not None:
            self._dev[(dur_name, dev.index)] = end
        return self._dev[key]

    def _device_watts(self) -> torch.Tensor:
        dev = _native.device()
        key = ("watts", dev.index)
        t = self._dev.get(key)
        if t is None:
            code = self._staged("watts", dev)
            L = _native.lib()
            if self.watts_rep is not None:  # run-coded: one code per change
                n = self.n_power
                bits = self._staged("watts_rep", dev)
                if bits.numel() != (n + 31) // 32:
                    raise ValueError(f"watts_rep: {bits.numel()} words for {n} samples")
                t = torch.empty(n, dtype=torch.float64, device=dev)
                ws = _native.Workspace.get(L.dw_unpack_decimal_rep_workspace_size(n))
                if self.watts_bits is not None:  # the stored codes bit-packed
                    wd, wb = self.watts_bits
                    _native.check(L.dw_unpack_decimal_rep_bits(_native.ptr(code), wd, wb, _native.ptr(bits), n,
                                                               self.watts_p0, _native.ptr(t), ws.data_ptr(),
                                                               ws.numel(), _native.stream_handle()),
                                  "dw_unpack_decimal_rep_bits")
                else:
                    _native.check(L.dw_unpack_decimal_rep(_native.ptr(code), _native.ptr(bits), n, self.watts_p0,
                                                          _native.ptr(t), ws.data_ptr(), ws.numel(),
                                                          _native.stream_handle()), "dw_unpack_decimal_rep")
            else:
                if code.numel() != self.n_power:
                    raise ValueError(f"watts: {code.numel()} codes for {self.n_power} samples")
                t = torch.empty(code.numel(), dtype=torch.float64, device=dev)
                _native.check(L.dw_unpack_decimal(_native.ptr(code), code.numel(), self.watts_p0,
                                                  _native.ptr(t), _native.stream_handle()), "dw_unpack_decimal")
            self._dev[key] = t
        return t

    def _device_sig(self) -> torch.Tensor:
        dev = _native.device()
        key = ("op_sig", dev.index)
        t = self._dev.get(key)
        if t is None:
            code = self._staged("op_sig", dev)
            d = self._staged("op_sig_dict", dev)
            if self.sig_bits is not None:
                t = torch.empty(self.n_ops, dtype=torch.int64, device=dev)
                _native.check(_native.lib().dw_unpack_dict_bits(_native.ptr(d), _native.ptr(code), self.sig_bits,
                                                                self.n_ops, _native.ptr(t), _native.stream_handle()),
                              "dw_unpack_dict_bits")
            else:
                t = torch.empty(code.numel(), dtype=torch.int64, device=dev)
                _native.check(_native.lib().dw_unpack_dict(_native.ptr(d), _native.ptr(code), code.element_size(),
                                                           code.numel(), _native.ptr(t), _native.stream_handle()),
                              "dw_unpack_dict")
            self._dev[key] = t
        return t

    def host(self, name: str) -> np.ndarray:
        if name in ("ts", "op_start", "op_end", "k_start", "k_end") or (name == "watts" and self.watts_p0 is not None) \
                or (name == "op_sig" and self.op_sig_dict is not None):
            return self.device(name).cpu().numpy()
        return super().host(name)

    @property
    def host_bytes(self) -> int:
        """Bytes the hot columns occupy on the host (what crosses PCIe)."""
        def nb(a):
            return int(a.numel() * a.element_size()) if isinstance(a, torch.Tensor) else int(np.asarray(a).nbytes)
        cols = [getattr(self, n) for n in ("ts", "watts", "op_start", "op_end", "k_start", "k_end", "op_sig")]
        return sum(nb(a) for a in cols + [self.op_sig_dict, self.watts_rep] if a is not None)


def _narrow(d, what: str):
    """Unsigned 16-bit container when every value fits, else 32-bit (torch:
    int16/int32 holding the bit patterns; numpy: uint16/uint32)."""
    if isinstance(d, torch.Tensor):
        if d.numel() and (bool((d < 0).any()) or bool((d > 0xFFFFFFFF).any())):
            raise ValueError(f"{what} -- cannot pack")
        if d.numel() == 0 or int(d.max().item()) <= 0xFFFF:
            return torch.where(d >= 0x8000, d - 0x10000, d).to(torch.int16)
        return torch.where(d >= 0x80000000, d - 0x100000000, d).to(torch.int32)
    if d.size and ((d < 0).any() or (d > 0xFFFFFFFF).any()):
        raise ValueError(f"{what} -- cannot pack")
    return d.astype(np.uint16 if (d.size == 0 or d.max() <= 0xFFFF) else np.uint32)


def _deltas(x, what: str):
    """(base, deltas) of a sorted int64 column (numpy or torch)."""
    if isinstance(x, torch.Tensor):
        if x.numel() == 0:
            return 0, torch.zeros(0, dtype=torch.int16, device=x.device)
        d = torch.empty_like(x)
        d[0] = 0
        d[1:] = x[1:] - x[:-1]
        return int(x[0].item()), _narrow(d, f"{what}: not sorted, or a gap of 2^32 us or more")
    x = np.asarray(x, dtype=np.int64)
    if x.size == 0:
        return 0, np.zeros(0, dtype=np.uint16)
    return int(x[0]), _narrow(np.diff(x, prepend=x[0]), f"{what}: not sorted, or a gap of 2^32 us or more")


def _ts_deltas(x, what: str):
    """(base, bias, deltas) of the power timestamps: biased int8 when every
    delta after the first lies within 127 of the midpoint (a regular sampling
    clock with jitter), else as _deltas."""
    base, d = _deltas(x, what)
    n = int(d.shape[0])
    if n < 2:
        return base, 0, d
    full = _unsigned(d)
    tail = full[1:]
    lo, hi = (int(tail.min().item()), int(tail.max().item())) if isinstance(tail, torch.Tensor) else \
        (int(tail.min()), int(tail.max()))
    if hi - lo > 255:
        return base, 0, d
    bias = (lo + hi + 1) // 2
    code = full - bias
    if isinstance(code, torch.Tensor):
        code[0] = 0
        return base, bias, code.to(torch.int8)
    code[0] = 0
    return base, bias, code.astype(np.int8)


def _bitfields(v, max_width: int):
    """(bias, width, words) packing every element of a non-negative-spread
    int64 vector as v - min(v) in the fewest bits (<= max_width), little-endian
    in 32-bit words plus one padding word; None if the spread needs more."""
    is_t = isinstance(v, torch.Tensor)
    n = int(v.shape[0])
    if n == 0:
        return None
    lo, hi = (int(v.min().item()), int(v.max().item())) if is_t else (int(v.min()), int(v.max()))
    width = max(1, (hi - lo).bit_length())
    if width > max_width:
        return None
    nwords = (n * width + 31) // 32 + 1
    if is_t:
        f = v - lo
        bit = torch.arange(n, dtype=torch.int64, device=v.device) * width
        k, sh = bit >> 5, bit & 31
        words = torch.zeros(nwords, dtype=torch.int64, device=v.device)
        words.index_add_(0, k, (f << sh) & 0xFFFFFFFF)  # disjoint bit fields: add == or
        words.index_add_(0, k + 1, f >> (32 - sh))
        words = torch.where(words >= 0x80000000, words - 0x100000000, words).to(torch.int32)
    else:
        f = np.asarray(v, dtype=np.int64) - lo
        bit = np.arange(n, dtype=np.int64) * width
        k, sh = bit >> 5, bit & 31
        words = np.zeros(nwords, dtype=np.int64)
        np.add.at(words, k, (f << sh) & 0xFFFFFFFF)
        np.add.at(words, k + 1, f >> (32 - sh))
        words = words.astype(np.uint32)
    return lo, width, words


def _bitpack(x, max_width: int = 8):
    """(base, bias, width, words) of a sorted column whose deltas after the
    first spread at most 2^max_width - 1 (e.g. a regular sampling clock), else
    None: field i = delta_i - bias (field 0 unused), decoded by dw_unpack_bits."""
    is_t = isinstance(x, torch.Tensor)
    n = int(x.shape[0])
    if n < 2:
        return None
    d = (x[1:] - x[:-1]) if is_t else np.diff(np.asarray(x, dtype=np.int64))
    if (bool((d < 0).any()) if is_t else bool((d < 0).any())):
        return None
    lo = int(d.min().item()) if is_t else int(d.min())
    full = torch.cat([d.new_full((1,), lo), d]) if is_t else np.concatenate([[lo], d])
    packed = _bitfields(full, max_width)
    if packed is None:
        return None
    base = int(x[0].item()) if is_t else int(np.asarray(x)[0])
    return base, packed[0], packed[1], packed[2]


def _gridpack(x, max_width: int):
    """(base, bias, width, words, step_fx) of a sorted column as residuals
    from the line through its first and last values (a clock with a nominal
    period: a jittered clock's residuals span half its deltas' range), in at
    most max_width bits, else None.  Decoded by dw_unpack_grid."""
    is_t = isinstance(x, torch.Tensor)
    n = int(x.shape[0])
    if n < 3 or n >= (1 << 31) or max_width < 1:
        return None
    base = int(x[0].item()) if is_t else int(np.asarray(x)[0])
    last = int(x[-1].item()) if is_t else int(np.asarray(x)[-1])
    if last < base:
        return None
    step_fx = ((last - base) << 32) // (n - 1)
    if step_fx >> 63 or (step_fx >> 32) * (n - 1) >= (1 << 62):
        return None
    r = x.to(torch.int64).clone() if is_t else np.array(x, dtype=np.int64)
    C = 1 << 26  # residuals chunk by chunk: no n-long temporaries beyond r
    for c0 in range(0, n, C):
        c1 = min(n, c0 + C)
        i = torch.arange(c0, c1, dtype=torch.int64, device=x.device) if is_t else np.arange(c0, c1, dtype=np.int64)
        r[c0:c1] -= base + i * (step_fx >> 32) + ((i * (step_fx & 0xFFFFFFFF)) >> 32)
    packed = _bitfields(r, max_width)
    del r
    if packed is None:
        return None
    return base, packed[0], packed[1], packed[2], step_fx


def _sig_dict(sig):
    """(dictionary u64, codes u16/u32) of the signature column when it has at
    most 2^32 distinct values (it has ~1e6 at C4), else None."""
    if sig is None:
        return None
    if isinstance(sig, torch.Tensor):
        if sig.numel() == 0:
            return None
        uniq, inv = torch.unique(sig, return_inverse=True)
        if uniq.numel() > 0x7FFFFFFF:
            return None
        code = inv.to(torch.int16) if uniq.numel() <= 0x7FFF else inv.to(torch.int32)
        return uniq, code
    a = np.asarray(sig)
    if a.size == 0:
        return None
    uniq, inv = np.unique(a, return_inverse=True)
    code = inv.astype(np.uint16) if uniq.size <= 0xFFFF else inv.astype(np.uint32)
    return uniq, code


def _durations(start, end, what: str):
    if isinstance(start, torch.Tensor):
        return _narrow(end - start, f"{what}: negative or >= 2^32 us durations")
    dur = np.asarray(end, dtype=np.int64) - np.asarray(start, dtype=np.int64)
    return _narrow(dur, f"{what}: negative or >= 2^32 us durations")


_M_LIMIT = 1 << 30


def decimal_code(w):
    """(p0, uint32 codes) encoding every watts value exactly as m * 10^-(p0+j)
    (m < 2^30, j < 4; decoded by one correctly rounded IEEE operation, as
    dw_unpack_decimal does), or None when some value is not such a decimal.
    Works on numpy or torch (cuda) columns."""
    is_t = isinstance(w, torch.Tensor)
    n = int(w.numel() if is_t else np.asarray(w).size)
    if n == 0:
        return None
    if is_t:
        pos = w[w > 0]
        if bool((w < 0).any()) or not bool(torch.isfinite(w).all()):
            return None
        top = float(pos.max().item()) if pos.numel() else 1.0
    else:
        w = np.asarray(w, dtype=np.float64)
        if (w < 0).any() or not np.isfinite(w).all():
            return None
        top = float(w.max()) if (w > 0).any() else 1.0
    p0 = 8 - int(math.floor(math.log10(top)))
    p0 = max(-22, min(p0, 19))
    lib = torch if is_t else np
    code = None
    done = lib.zeros_like(w, dtype=lib.bool) if is_t else np.zeros(n, dtype=bool)
    out = (torch.zeros(n, dtype=torch.int64, device=w.device) if is_t else np.zeros(n, dtype=np.int64))
    for j in range(4):
        p = p0 + j
        scale = 10.0 ** abs(p)
        m = lib.round(w * scale) if p >= 0 else lib.round(w / scale)
        if is_t:
            sc = torch.full_like(w, scale)
            back = torch.div(m, sc) if p >= 0 else m * sc
        else:
            back = m / scale if p >= 0 else m * scale
        ok = (m >= 0) & (m < _M_LIMIT) & (back == w) & ~done
        mi = m.to(torch.int64) if is_t else m.astype(np.int64)
        out = lib.where(ok, mi | (j << 30), out)
        done = done | ok
    if not bool(done.all()):
        return None
    code = (torch.where(out >= 0x80000000, out - 0x100000000, out).to(torch.int32) if is_t
            else out.astype(np.uint32))
    return p0, code


_REP_CHUNK = 1 << 26


def rep_code(code):
    """Run-code a column of decimal codes: (bitmap words u32 -- bit i set when
    sample i's code differs from sample i-1's, bit 0 always --, the codes of
    those samples), or None when that is not at least a quarter smaller.
    numpy or torch (device columns are coded in chunks of 2^26 samples)."""
    is_t = isinstance(code, torch.Tensor)
    n = int(code.numel() if is_t else np.asarray(code).size)
    if n < 64:
        return None
    if not is_t:
        c = np.asarray(code)
        new = np.empty(n, dtype=bool)
        new[0] = True
        np.not_equal(c[1:], c[:-1], out=new[1:])
        m = int(new.sum())
        if 4 * m + 4 * ((n + 31) // 32) > 3 * n:
            return None
        words = np.packbits(np.concatenate([new, np.zeros((-n) % 32, dtype=bool)]), bitorder="little").view(np.uint32)
        return words, c[new]
    new = torch.empty(n, dtype=torch.bool, device=code.device)
    new[0] = True
    torch.ne(code[1:], code[:-1], out=new[1:])
    m = int(new.sum().item())
    if 4 * m + 4 * ((n + 31) // 32) > 3 * n:
        return None
    nw = (n + 31) // 32
    words = torch.empty(nw, dtype=torch.int32, device=code.device)
    shifts = torch.arange(32, dtype=torch.int64, device=code.device)
    for w0 in range(0, nw, _REP_CHUNK // 32):
        w1 = min(w0 + _REP_CHUNK // 32, nw)
        b = new[32 * w0: min(32 * w1, n)].to(torch.int64)
        if b.numel() < 32 * (w1 - w0):
            b = torch.cat([b, b.new_zeros(32 * (w1 - w0) - b.numel())])
        v = (b.view(-1, 32) << shifts).sum(1)
        words[w0:w1] = torch.where(v >= 0x80000000, v - 0x100000000, v).to(torch.int32)
    return words, code[new]


def _pack_codes(code, p0: int):
    """(p0', (width, bias), words) for a run-coded column's stored decimal
    codes: the decimal zeros every mantissa shares stripped (p0 lowered by as
    many, never below 0: the decode divides by 10^(p0'+j) as before, the same
    correctly rounded double) and the codes bit-packed in the bits their
    spread needs -- or None unless that is narrower than 32 bits."""
    is_t = isinstance(code, torch.Tensor)
    c = (code.to(torch.int64) & 0xFFFFFFFF) if is_t else np.asarray(code).astype(np.int64)
    if c.shape[0] == 0:
        return None
    m, j = c & 0x3FFFFFFF, c >> 30
    z = 0
    while z < p0 and bool(((m % 10 ** (z + 1)) == 0).all()):
        z += 1
    if z:
        c = (m // 10 ** z) | (j << 30)
    packed = _bitfields(c, 31)
    if packed is None:
        return None
    bias, width, words = packed
    return p0 - z, (width, bias), words


def pack(cols: TraceColumns, decimal: bool = True, runs: bool = True, grid_ts: bool = True) -> PackedColumns:
    """Packed form of a trace with sorted power, operator and kernel starts
    (ValueError otherwise -- keep such traces unpacked).  Works on host or
    device columns; the result lives where the input does."""
    bits = _bitpack(cols.ts)
    if bits is not None:
        tb, tbias, twidth, td = bits
        dwidth = twidth
    else:
        tb, tbias, td = _ts_deltas(cols.ts, "power timestamps")
        twidth = None
        dwidth = 8 * (td.element_size() if isinstance(td, torch.Tensor) else np.asarray(td).itemsize)
    tlast = int(cols.ts[-1].item()) if isinstance(cols.ts, torch.Tensor) else int(np.asarray(cols.ts)[-1])
    grid = _gridpack(cols.ts, dwidth - 1) if grid_ts else None
    tstep = None
    if grid is not None:  # residuals from the clock's line: fewer bits than its deltas
        tb, tbias, twidth, td, tstep = grid
    elif twidth is None:
        tlast = None
    ob, od = _deltas(cols.op_start, "operator starts")
    kb, kd = _deltas(cols.k_start, "kernel starts")
    o_dur = _durations(cols.op_start, cols.op_end, "operators")
    k_dur = _durations(cols.k_start, cols.k_end, "kernels")
    # narrower still: bit-pack interval deltas / durations whose spread needs <= 15 bits
    iv_bits = {}
    for sname, ename, start, end in (("op_start", "op_end", cols.op_start, cols.op_end),
                                     ("k_start", "k_end", cols.k_start, cols.k_end)):
        sp = _bitpack(start, 15)
        dp = _bitfields(end - start if isinstance(start, torch.Tensor) else
                        np.asarray(end, dtype=np.int64) - np.asarray(start, dtype=np.int64), 15) \
            if sp is not None else None
        if sp is not None and dp is not None:
            iv_bits[sname] = (sp[2], sp[1])
            iv_bits[ename] = (dp[1], dp[0])
            if sname == "op_start":
                ob, od, o_dur = sp[0], sp[3], dp[2]
            else:
                kb, kd, k_dur = sp[0], sp[3], dp[2]
    dec = decimal_code(cols.watts) if decimal else None
    watts, p0 = (cols.watts, None) if dec is None else (dec[1], dec[0])
    rc = rep_code(watts) if dec is not None and runs else None
    watts_rep = watts_bits = None
    if rc is not None:
        watts_rep, watts = rc
        wp = _pack_codes(watts, p0)
        if wp is not None:
            p0, watts_bits, watts = wp
    sd = _sig_dict(cols.op_sig)
    sig, sig_dict = (cols.op_sig, None) if sd is None else (sd[1], sd[0])
    sig_bits = None
    if sd is not None:
        codes = sd[1].to(torch.int64) if isinstance(sd[1], torch.Tensor) else np.asarray(sd[1], dtype=np.int64)
        width = max(1, (int(sd[0].shape[0]) - 1).bit_length())
        if width < 8 * (sd[1].element_size() if isinstance(sd[1], torch.Tensor) else sd[1].itemsize):
            packed = _bitfields(codes - 0, 32)  # codes start at 0: bias 0 unless code 0 is absent
            if packed is not None and packed[0] == 0 and packed[1] <= width:
                sig, sig_bits = packed[2], packed[1]
    return PackedColumns(tb, td, watts, ob, od, o_dur, kb, kd, k_dur, cols.trace_end,
                         k_op=cols.k_op, op_sig=sig, watts_p0=p0, ts_bias=tbias, op_sig_dict=sig_dict,
                         ts_bits=twidth, n_power=cols.n_power, ts_last=tlast, iv_bits=iv_bits,
                         n_ops=cols.n_ops, n_kernels=cols.n_kernels, sig_bits=sig_bits, watts_rep=watts_rep,
                         ts_step=tstep, watts_bits=watts_bits, op_ids=cols.op_ids, k_ids=cols.k_ids, op_names=cols.op_names, op_work=cols.op_work,
                         op_rank=cols.op_rank)


def save_packed(cols: TraceColumns, path) -> None:
    """The packed columnar trace file (``*.dwc``): one JSON header line, then
    every column's raw little-endian bytes, 64-byte aligned.  Columns only --
    ids, names and tensors stay in the JSONL trace (trace_model.save_trace)."""
    import json
    pc = cols if isinstance(cols, PackedColumns) else pack(cols)
    arrays = {}
    for n in ("ts", "watts", "watts_rep", "op_start", "op_end", "k_start", "k_end", "k_op", "op_sig", "op_sig_dict",
              "op_work"):
        a = getattr(pc, n)
        if a is None:
            continue
        a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
        coded = n in ("op_start", "op_end", "k_start", "k_end") or (n == "ts" and a.itemsize > 1) or \
            n in pc.iv_bits or (n == "op_sig" and pc.sig_bits is not None) or \
            (n == "ts" and pc.ts_bits is not None) or \
            (n == "watts" and pc.watts_p0 is not None) or (n == "op_sig" and pc.op_sig_dict is not None) or \
            n == "watts_rep"
        if coded:
            a = a.view(np.uint16 if a.itemsize == 2 else np.uint32)
        arrays[n] = np.ascontiguousarray(a)
    meta = {"format": "dwc", "version": 2, "trace_end": pc.trace_end, "ts_base": pc.ts_base,
            "op_base": pc.op_start_base, "k_base": pc.k_start_base, "watts_p0": pc.watts_p0,
            "ts_bias": pc.ts_bias, "ts_bits": pc.ts_bits, "n_power": pc.n_power,
            "ts_last": pc._ts_last if pc.ts_bits is not None else None, "ts_step": pc.ts_step,
            "watts_bits": list(pc.watts_bits) if pc.watts_bits is not None else None,
            "iv_bits": {k: list(v) for k, v in pc.iv_bits.items()}, "n_ops": pc.n_ops, "n_kernels": pc.n_kernels,
            "sig_bits": pc.sig_bits, "watts_rep": pc.watts_rep is not None,
            "columns": {}}
    off = 0
    for n, a in arrays.items():
        meta["columns"][n] = {"dtype": a.dtype.str, "n": int(a.shape[0]), "offset": off}
        off += (a.nbytes + 63) & ~63
    head = json.dumps(meta).encode() + b"\n"
    pad = (-len(head)) % 64
    with open(path, "wb") as fh:
        fh.write(head + b" " * pad)
        for n, a in arrays.items():
            fh.write(a.tobytes())
            fh.write(b"\0" * ((-a.nbytes) % 64))


def load_packed(path, pin: bool = False) -> PackedColumns:
    """Memory-map a ``*.dwc`` file (optionally copying it into pinned host
    memory for asynchronous host->HBM transfers)."""
    import json
    with open(path, "rb") as fh:
        head = fh.readline()
    meta = json.loads(head)
    if meta.get("format") != "dwc" or meta.get("version") not in (1, 2):
        raise ValueError(f"{path}: not a dwc v1/v2 file")
    start = (len(head) + 63) & ~63
    raw = np.memmap(path, dtype=np.uint8, mode="r")
    cols = {}
    for n, c in meta["columns"].items():
        dt = np.dtype(c["dtype"])
        a = raw[start + c["offset"]: start + c["offset"] + c["n"] * dt.itemsize].view(dt)
        t = torch.from_numpy(np.array(a)) if pin else a
        if pin:
            t = t.pin_memory()
        cols[n] = t
    def as_signed(x):  # torch has no uint16/uint32 storage for these: same bits, signed view
        if isinstance(x, torch.Tensor) and x.dtype in (torch.uint16, torch.uint32):
            return x.view(torch.int16 if x.element_size() == 2 else torch.int32)
        return x
    p0 = meta.get("watts_p0")
    sig_dict = cols.get("op_sig_dict")
    sig = cols.get("op_sig")
    return PackedColumns(meta["ts_base"], as_signed(cols["ts"]), as_signed(cols["watts"]) if p0 is not None
                         else cols["watts"], meta["op_base"], as_signed(cols["op_start"]), as_signed(cols["op_end"]),
                         meta["k_base"], as_signed(cols["k_start"]), as_signed(cols["k_end"]), meta["trace_end"],
                         k_op=cols.get("k_op"), op_sig=as_signed(sig) if sig_dict is not None else sig,
                         op_work=cols.get("op_work"), watts_p0=p0, ts_bias=meta.get("ts_bias", 0),
                         op_sig_dict=sig_dict, ts_bits=meta.get("ts_bits"), n_power=meta.get("n_power"),
                         ts_last=meta.get("ts_last"), iv_bits={k: tuple(v) for k, v in meta.get("iv_bits", {}).items()},
                         n_ops=meta.get("n_ops"), n_kernels=meta.get("n_kernels"), sig_bits=meta.get("sig_bits"),
                         watts_rep=as_signed(cols["watts_rep"]) if meta.get("watts_rep") else None,
                         ts_step=meta.get("ts_step"), watts_bits=meta.get("watts_bits"))
