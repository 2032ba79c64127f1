"""CPU oracle for the Magneton/diffwatt hot path -- TEST INFRASTRUCTURE ONLY.

This package is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  ``paper_2512_08365_b200`` never does, and
its CUDA path fails loudly instead of falling back here.

It wraps ``oracle/libdw_oracle.so`` (built from ``dw_oracle.c`` by
``oracle/Makefile``), a C restatement of the reference functions named in that
file's header, each pinned against the golden vectors recorded from the
reference itself (``tests/golden``, made by ``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = _HERE / "libdw_oracle.so"
_lib = None

MODE_REFERENCE = 0  # sequential fp64 sum for every interval (the reference's arithmetic)
MODE_DEVICE = 1     # the GPU's reference-order mode: sequential <= DW_DIRECT_MAX segments, exact fixed point above
MODE_EXACT = 2      # the GPU's exact mode (summation="exact"): every interval as the exact fixed-point sum of its pieces

DW_DIRECT_MAX = 256

VERDICT_BELOW, VERDICT_TRADEOFF, VERDICT_WASTE = 0, 1, 2


def build() -> Path:
    src = _HERE / "dw_oracle.c"
    if not _LIB.exists() or _LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(_LIB))
        _lib.dwo_fx_sum.restype = ctypes.c_double
        _lib.dwo_py_sum.restype = ctypes.c_double
        _lib.dwo_total_device.restype = ctypes.c_double
        _lib.dwo_total_device_mode.restype = ctypes.c_double
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:
    lib().dwo_set_threads(ctypes.c_int(n))


def num_threads() -> int:
    return int(lib().dwo_num_threads())


class OracleError(ValueError):
    def __init__(self, code: int, index: int):
        super().__init__(f"oracle error {code} at {index}")
        self.code = code
        self.index = index


def integrate_step(ts, watts, span_hi, lo, hi, mode=MODE_REFERENCE):
    ts = np.ascontiguousarray(ts, dtype=np.int64)
    watts = np.ascontiguousarray(watts, dtype=np.float64)
    lo = np.ascontiguousarray(lo, dtype=np.int64)
    hi = np.ascontiguousarray(hi, dtype=np.int64)
    out = np.empty(lo.shape[0], dtype=np.float64)
    bad = ctypes.c_int64(-1)
    rc = lib().dwo_integrate_step(_p(ts), _p(watts), ctypes.c_int64(ts.shape[0]),
                                  ctypes.c_int64(int(span_hi)), _p(lo), _p(hi),
                                  ctypes.c_int64(lo.shape[0]), _p(out), ctypes.c_int(mode),
                                  ctypes.byref(bad))
    if rc:
        raise OracleError(rc, bad.value)
    return out


def integrate_linear(ts, watts, lo, hi, mode=MODE_REFERENCE):
    ts = np.ascontiguousarray(ts, dtype=np.int64)
    watts = np.ascontiguousarray(watts, dtype=np.float64)
    lo = np.ascontiguousarray(lo, dtype=np.int64)
    hi = np.ascontiguousarray(hi, dtype=np.int64)
    out = np.empty(lo.shape[0], dtype=np.float64)
    bad = ctypes.c_int64(-1)
    rc = lib().dwo_integrate_linear(_p(ts), _p(watts), ctypes.c_int64(ts.shape[0]), _p(lo),
                                    _p(hi), ctypes.c_int64(lo.shape[0]), _p(out),
                                    ctypes.c_int(mode), ctypes.byref(bad))
    if rc:
        raise OracleError(rc, bad.value)
    return out


def split(kind, ts, watts, span_hi, lo, hi):
    """Overlap-split joules of one interval set (the builder's G1 definition,
    dw_oracle.c dwo_split): power divided equally among the set's intervals
    active at each instant; equals the compat integral when nothing overlaps."""
    ts = np.ascontiguousarray(ts, dtype=np.int64)
    watts = np.ascontiguousarray(watts, dtype=np.float64)
    lo = np.ascontiguousarray(lo, dtype=np.int64)
    hi = np.ascontiguousarray(hi, dtype=np.int64)
    out = np.empty(lo.shape[0], dtype=np.float64)
    bad = ctypes.c_int64(-1)
    rc = lib().dwo_split(ctypes.c_int(0 if kind == "step" else 1), _p(ts), _p(watts),
                         ctypes.c_int64(ts.shape[0]), ctypes.c_int64(int(span_hi or 0)), _p(lo), _p(hi),
                         ctypes.c_int64(lo.shape[0]), _p(out), ctypes.byref(bad))
    if rc:
        raise OracleError(rc, bad.value)
    return out


def replay_delays(n: int, delay_us: int, seed: int) -> np.ndarray:
    """The sampler's per-sample delays (energy.py:160-165): a fresh numpy
    PCG64 stream per call, uniform in [0.5, 1.5] x delay_us; zeros without
    delay.  rng.uniform(a, b, size=n) equals n scalar draws."""
    if not delay_us:
        return np.zeros(max(n, 1))
    rng = np.random.default_rng(seed)
    return rng.uniform(0.5 * delay_us, 1.5 * delay_us, size=max(n, 1))


def replay(ts, watts, span_hi, op_start, op_end, repeat=1000, period_us=40_000, delay_us=200_000, seed=0):
    """replay_estimate restated for every operator (energy.py:196-256):
    (watts, joules) per op."""
    ts = np.ascontiguousarray(ts, dtype=np.int64)
    watts = np.ascontiguousarray(watts, dtype=np.float64)
    op_start = np.ascontiguousarray(op_start, dtype=np.int64)
    op_end = np.ascontiguousarray(op_end, dtype=np.int64)
    dmax = int((op_end - op_start).max()) if op_start.size else 0
    delays = replay_delays(repeat * dmax // period_us + 2, delay_us, seed)
    w_out = np.empty(op_start.shape[0])
    j_out = np.empty(op_start.shape[0])
    bad = ctypes.c_int64(-1)
    rc = lib().dwo_replay(_p(ts), _p(watts), ctypes.c_int64(ts.shape[0]), ctypes.c_int64(int(span_hi)),
                          _p(op_start), _p(op_end), ctypes.c_int64(op_start.shape[0]), ctypes.c_int64(repeat),
                          ctypes.c_int64(period_us), _p(delays), ctypes.c_int64(delays.shape[0]), _p(w_out),
                          _p(j_out), ctypes.byref(bad))
    if rc:
        raise OracleError(rc, bad.value)
    return w_out, j_out


def total_device(kind, ts, watts, span_hi=None, exact: bool = False) -> float:
    """The ledger total over the whole span under the device's definition
    (``exact``: the DW_SUM_EXACT mode's)."""
    ts = np.ascontiguousarray(ts, dtype=np.int64)
    watts = np.ascontiguousarray(watts, dtype=np.float64)
    return float(lib().dwo_total_device_mode(ctypes.c_int(0 if kind == "step" else 1), _p(ts), _p(watts),
                                             ctypes.c_int64(ts.shape[0]),
                                             ctypes.c_int64(int(span_hi) if span_hi is not None else 0),
                                             ctypes.c_int(1 if exact else 0)))


def fx_sum(x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().dwo_fx_sum(_p(x), ctypes.c_int64(x.shape[0])))


def py_sum(x) -> float:
    """CPython 3.12 ``sum()`` of floats (Neumaier), as the reference's sums run."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().dwo_py_sum(_p(x), ctypes.c_int64(x.shape[0])))


def ledger(kind, ts, watts, span_hi, op_start, op_end, k_start, k_end, mode=MODE_REFERENCE):
    """build_ledger restated (energy.py:280-331): per-op, per-kernel, total, idle.
    ``kind`` is "step" (ground truth) or "linear" (a sampled view)."""
    if kind == "step":
        f = lambda lo, hi: integrate_step(ts, watts, span_hi, lo, hi, mode)  # noqa: E731
        span = (int(ts[0]), int(span_hi))
    else:
        f = lambda lo, hi: integrate_linear(ts, watts, lo, hi, mode)  # noqa: E731
        span = (int(ts[0]), int(ts[-1]))
    per_op = f(op_start, op_end)
    per_k = f(k_start, k_end)
    if mode in (MODE_DEVICE, MODE_EXACT):
        total = total_device(kind, ts, watts, span_hi, exact=mode == MODE_EXACT)
    else:
        total = float(f(np.array([span[0]]), np.array([span[1]]))[0])
    op_total = py_sum(per_op) if mode == MODE_REFERENCE else fx_sum(per_op)
    return per_op, per_k, total, max(total - op_total, 0.0)


def detect(off_a, mem_a, off_b, mem_b, joules_a, joules_b, start_a, end_a, start_b, end_b,
           out_diff, threshold):
    P = len(off_a) - 1
    c = lambda a, t: np.ascontiguousarray(a, dtype=t)  # noqa: E731
    off_a, off_b = c(off_a, np.int64), c(off_b, np.int64)
    mem_a, mem_b = c(mem_a, np.int32), c(mem_b, np.int32)
    joules_a, joules_b = c(joules_a, np.float64), c(joules_b, np.float64)
    start_a, end_a = c(start_a, np.int64), c(end_a, np.int64)
    start_b, end_b = c(start_b, np.int64), c(end_b, np.int64)
    out_diff = c(out_diff if out_diff is not None else np.zeros(P), np.float64)
    energy = np.empty((P, 2))
    ratio = np.empty(P)
    lat = np.empty((P, 2), dtype=np.int64)
    verdict = np.empty(P, dtype=np.int8)
    side = np.empty(P, dtype=np.int8)
    wasted = np.empty(P)
    info = np.empty(P, dtype=np.int8)
    rc = lib().dwo_detect(ctypes.c_int64(P), _p(off_a), _p(mem_a), _p(off_b), _p(mem_b),
                          _p(joules_a), _p(joules_b), _p(start_a), _p(end_a), _p(start_b),
                          _p(end_b), _p(out_diff), ctypes.c_double(threshold), _p(energy),
                          _p(ratio), _p(lat), _p(verdict), _p(side), _p(wasted), _p(info))
    if rc:
        raise ValueError("threshold must be in (0, 1]")
    return dict(energy=energy, ratio=ratio, lat=lat, verdict=verdict, side=side,
                wasted=wasted, informational=info.astype(bool))


def rank(verdict, wasted, tie):
    verdict = np.ascontiguousarray(verdict, dtype=np.int8)
    wasted = np.ascontiguousarray(wasted, dtype=np.float64)
    tie = np.ascontiguousarray(tie, dtype=np.int64)
    order = np.empty(verdict.shape[0], dtype=np.int64)
    lib().dwo_rank(ctypes.c_int64(verdict.shape[0]), _p(verdict), _p(wasted), _p(tie), _p(order))
    return order


def occurrence(sig):
    sig = np.ascontiguousarray(sig, dtype=np.uint64)
    occ = np.empty(sig.shape[0], dtype=np.int64)
    lib().dwo_occurrence(_p(sig), ctypes.c_int64(sig.shape[0]), _p(occ))
    return occ


def join(sig_a, sig_b):
    sig_a = np.ascontiguousarray(sig_a, dtype=np.uint64)
    sig_b = np.ascontiguousarray(sig_b, dtype=np.uint64)
    ma = np.empty(sig_a.shape[0], dtype=np.int64)
    mb = np.empty(sig_b.shape[0], dtype=np.int64)
    lib().dwo_join(_p(sig_a), ctypes.c_int64(sig_a.shape[0]), _p(sig_b),
                   ctypes.c_int64(sig_b.shape[0]), _p(ma), _p(mb))
    return ma, mb


def tuple_rank(tuples):
    """Rank of each tuple under Python tuple ordering (equal tuples share a
    rank) -- the nodes_a tie-break of detect.report (detect.py:263-266)."""
    order = sorted(range(len(tuples)), key=lambda i: tuples[i])
    tie = np.empty(len(tuples), dtype=np.int64)
    r = -1
    prev = object()
    for i in order:
        if tuples[i] != prev:
            r += 1
            prev = tuples[i]
        tie[i] = r
    return tie
