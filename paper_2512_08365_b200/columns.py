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

import weakref
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native


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

    def prefetch(self, stream: "torch.cuda.Stream", names=HOT) -> None:
        """Start the host->HBM copies of ``names`` on ``stream`` (pinned host
        buffers copy asynchronously); later device() calls on another stream
        wait for them."""
        dev = _native.device()
        with torch.cuda.stream(stream):
            for n in names:
                if getattr(self, n) is not None:
                    self.device(n)
            ev = torch.cuda.Event()
            ev.record(stream)
        self._dev["__ready__"] = ev

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
        k_ids, k_start, k_end, k_op = [], [], [], []
        kernels = trace.kernels
        for i, o in enumerate(ops):
            for kid in o.kernel_ids:
                k = kernels[kid]
                k_ids.append(kid)
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
                   k_ids=k_ids, op_names=[o.op_name for o in ops])
        try:
            _CACHE[id(trace)] = (weakref.ref(trace), cols)
            while len(_CACHE) > _CACHE_MAX:
                _CACHE.pop(next(iter(_CACHE)))
        except TypeError:
            pass
        return cols


_CACHE: dict = {}
_CACHE_MAX = 32
