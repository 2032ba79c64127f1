"""JSONL trace ingestion on the GPU.

``load_columns(path)`` reads a trace file straight into device columns: the
raw bytes go to HBM once and csrc/ingest.cu parses every line in its own
thread.  The fast path takes the canonical form ``trace_to_lines`` writes
(compact separators, fixed key order) for the power, op and kernel records of
traces without tensor snapshots -- the scale traces -- and validates them on
the device (power order, interval rules, unique ids and correlation ids,
kernel ownership and containment).  Anything else -- tensors, a program
model, another key order, escapes, numbers the exact fast decimal conversion
cannot take, or any violation -- loads through the reference-compatible
loader (``trace_model.load_trace``), which also raises the reference's exact
error.  Either way the result equals ``TraceColumns.from_trace(load_trace(path))``.
"""

from __future__ import annotations

import json
from collections.abc import Sequence

import numpy as np
import torch

from . import _native
from .columns import TraceColumns
from .trace_model import SCHEMA_VERSION, load_trace

L_EMPTY, L_POWER, L_OP, L_KERNEL, L_OTHER = 0, 1, 2, 3, 4
_IG_BYTES = 256


class StrView(Sequence):
    """Strings as (offset, length) spans of the file bytes, decoded on demand
    (a Python list of 1e8 ids would cost more than the whole parse)."""

    def __init__(self, raw: np.ndarray, off: np.ndarray, length: np.ndarray):
        self.raw, self.off, self.len = raw, off, length

    def __len__(self):
        return int(self.off.shape[0])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        o, n = int(self.off[i]), int(self.len[i])
        return self.raw[o:o + n].tobytes().decode("ascii")

    def index(self, value, *args):
        b = np.frombuffer(value.encode(), dtype=np.uint8)
        cand = np.nonzero(self.len == b.size)[0]
        for i in cand:
            o = int(self.off[i])
            if np.array_equal(self.raw[o:o + b.size], b):
                return int(i)
        raise ValueError(f"{value!r} is not in the view")


def _python_path(path) -> TraceColumns:
    tr = load_trace(str(path))
    cols = TraceColumns.from_trace(tr)
    cols.header, cols.config, cols.loaded_by = tr.header, dict(tr.config), "python"
    return cols


def load_columns(path) -> TraceColumns:
    """Device columns of the trace at ``path`` (see the module docstring)."""
    raw = np.fromfile(str(path), dtype=np.uint8)
    if raw.size == 0:
        return _python_path(path)
    cols = _gpu_path(raw)
    return cols if cols is not None else _python_path(path)


def _gpu_path(raw: np.ndarray):
    L = _native.lib()
    dev = _native.device()
    st = _native.stream_handle()
    p = _native.ptr
    n = int(raw.size)
    buf = torch.from_numpy(raw).to(dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    nth = (n + _IG_BYTES - 1) // _IG_BYTES
    counts = torch.empty(nth, dtype=torch.int64, device=dev)
    _native.check(L.dw_ig_nl_count(p(buf), n, p(counts), p(flags), st), "dw_ig_nl_count")
    offs = torch.cumsum(counts, 0) - counts
    nnl = int(counts.sum().item())
    tail = raw[-1] != ord("\n")
    ends = torch.empty(nnl + int(tail), dtype=torch.int64, device=dev)
    _native.check(L.dw_ig_nl_write(p(buf), n, p(offs), p(ends), st), "dw_ig_nl_write")
    if tail:
        ends[-1] = n
    nlines = int(ends.numel())
    ltype = torch.empty(nlines, dtype=torch.uint8, device=dev)
    _native.check(L.dw_ig_classify(p(buf), n, p(ends), nlines, p(ltype), p(flags), st), "dw_ig_classify")
    if int(flags.item()):
        return None
    # the few other records (header, config) are read on the host
    other = torch.nonzero(ltype == L_OTHER).flatten()
    nonempty = torch.nonzero(ltype != L_EMPTY).flatten()
    if nonempty.numel() == 0 or other.numel() == 0 or int(nonempty[0]) != int(other[0]):
        return None  # the first record must be the header
    ends_h = ends.cpu().numpy()
    header, config = None, {}
    for i in other.cpu().tolist():
        a = 0 if i == 0 else int(ends_h[i - 1]) + 1
        try:
            rec = json.loads(raw[a:int(ends_h[i])].tobytes().decode("ascii"))
        except (ValueError, UnicodeDecodeError):
            return None
        kind = rec.get("type") if isinstance(rec, dict) else None
        if header is None:
            if kind != "header" or set(rec) != {"type", "schema_version", "system", "workload", "seed"}:
                return None
            v, seed = rec["schema_version"], rec["seed"]
            if type(v) is not int or v != SCHEMA_VERSION or type(seed) is not int:
                return None
            from .trace_model import TraceHeader
            header = TraceHeader(v, str(rec["system"]), str(rec["workload"]), seed)
        elif kind == "config" and "key" in rec:
            config[str(rec["key"])] = rec.get("value")
        else:
            return None  # a second header, a program model, block traces, ...
    lines = {t: torch.nonzero(ltype == t).flatten() for t in (L_POWER, L_OP, L_KERNEL)}
    npw, nop, nk = (int(lines[t].numel()) for t in (L_POWER, L_OP, L_KERNEL))
    i64 = lambda m: torch.empty(m, dtype=torch.int64, device=dev)  # noqa: E731
    i32 = lambda m: torch.empty(m, dtype=torch.int32, device=dev)  # noqa: E731
    ts, watts = i64(npw), torch.empty(npw, dtype=torch.float64, device=dev)
    _native.check(L.dw_ig_parse_power(p(buf), p(ends), p(lines[L_POWER]), npw, p(ts), p(watts), p(flags), st),
                  "dw_ig_parse_power")
    o_id, o_idl, o_nm, o_nml, o_klf, o_klc, o_s, o_e = i64(nop), i32(nop), i64(nop), i32(nop), i64(nop), i32(nop), \
        i64(nop), i64(nop)
    _native.check(L.dw_ig_parse_op(p(buf), p(ends), p(lines[L_OP]), nop, p(o_id), p(o_idl), p(o_nm), p(o_nml),
                                   p(o_klf), p(o_klc), p(o_s), p(o_e), p(flags), st), "dw_ig_parse_op")
    k_id, k_idl, k_nm, k_nml, k_corr, k_s, k_e = i64(nk), i32(nk), i64(nk), i32(nk), i64(nk), i64(nk), i64(nk)
    _native.check(L.dw_ig_parse_kernel(p(buf), p(ends), p(lines[L_KERNEL]), nk, p(k_id), p(k_idl), p(k_nm),
                                       p(k_nml), p(k_corr), p(k_s), p(k_e), p(flags), st), "dw_ig_parse_kernel")
    if int(flags.item()) or npw == 0:
        return None
    if npw > 1 and not bool((ts[1:] > ts[:-1]).all()):
        return None  # power samples must be strictly increasing
    # unique ids (sorted 64-bit hashes; any equal pair goes to the Python path)
    def hashes(off, ln, m):
        h = torch.empty(m, dtype=torch.int64, device=dev)
        idx = torch.empty(m, dtype=torch.int32, device=dev)
        _native.check(L.dw_ig_hash(p(buf), p(off), p(ln), m, p(h), p(idx), st), "dw_ig_hash")
        hs, order = torch.sort(h ^ torch.iinfo(torch.int64).min)  # unsigned order
        return hs ^ torch.iinfo(torch.int64).min, idx[order]
    if nop:
        oh, _ = hashes(o_id, o_idl, nop)
        if nop > 1 and bool((oh[1:] == oh[:-1]).any()):
            return None
    kh, kidx = hashes(k_id, k_idl, nk) if nk else (i64(0), i32(0))
    if nk > 1 and bool((kh[1:] == kh[:-1]).any()):
        return None
    if nk > 1:
        cs = torch.sort(k_corr).values
        if bool((cs[1:] == cs[:-1]).any()):
            return None  # correlation_id values must be unique per launch
    # kernels flattened in op.kernel_ids order (build_ledger's iteration order)
    kl_base = torch.cumsum(o_klc.to(torch.int64), 0) - o_klc.to(torch.int64)
    ne = int(o_klc.to(torch.int64).sum().item()) if nop else 0
    if ne != nk:
        return None  # some kernel is not launched by exactly one operator
    fk_s, fk_e, fk_op, fk_k = i64(ne), i64(ne), i32(ne), i64(ne)
    owner = torch.zeros(max(nk, 1), dtype=torch.int32, device=dev)
    _native.check(L.dw_ig_kernel_lists(p(buf), nop, p(o_klf), p(o_klc), p(kl_base), p(o_s), p(o_e), p(kh),
                                       p(kidx), nk, p(k_id), p(k_idl), p(k_s), p(k_e), p(fk_s), p(fk_e), p(fk_op),
                                       p(fk_k), p(owner), p(flags), st), "dw_ig_kernel_lists")
    if int(flags.item()) or (nk and not bool((owner[:nk] == 1).all())):
        return None
    # Trace.span_us (trace_model.py:307-314): every timestamp of the trace
    parts = [ts.max()]
    if nop:
        parts += [o_e.max(), o_s.max()]
    if nk:
        parts += [k_e.max(), k_s.max()]
    trace_end = int(torch.stack(parts).max().item())
    h = lambda t: t.cpu().numpy()  # noqa: E731
    k_id_h, k_idl_h, fk_k_h = h(k_id), h(k_idl), h(fk_k)
    cols = TraceColumns(ts=ts, watts=watts, trace_end=trace_end, op_start=o_s, op_end=o_e, k_start=fk_s,
                        k_end=fk_e, k_op=fk_op, op_ids=StrView(raw, h(o_id), h(o_idl)),
                        k_ids=StrView(raw, k_id_h[fk_k_h], k_idl_h[fk_k_h]),
                        op_names=StrView(raw, h(o_nm), h(o_nml)),
                        k_names=StrView(raw, h(k_nm)[fk_k_h], h(k_nml)[fk_k_h]))
    cols.header, cols.config, cols.loaded_by = header, config, "gpu"
    return cols
