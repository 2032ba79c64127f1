"""JSONL trace ingestion on the GPU.

``load_columns(path)`` reads a trace file straight into device columns: the
raw bytes go to HBM once and csrc/ingest.cu parses every line in its own
thread.  The device takes the canonical form ``trace_to_lines`` writes
(compact separators, fixed key order) of the power, op and kernel records and
validates them (power order, interval rules, unique ids and correlation ids,
kernel ownership and containment).  Only the other records -- header,
config, tensor snapshots, program model, block traces -- are decoded on the
host (json, line by line), and the rules that tie operators to them (every
referenced tensor exists, no in-place ids, one producer per tensor, an
acyclic operator graph, the program-model rules) run there on the device
parse's tensor-list spans.  Operator-id ranks (the report's nodes_a
tie-break) are computed on the device at ingest (``id_ranks``).  A file the
device cannot take -- another key order, escapes, numbers the exact fast
decimal conversion cannot take -- or any violation loads through the
reference-compatible loader (``trace_model.load_trace``), which raises the
reference's exact error.  Either way the columns equal
``TraceColumns.from_trace(load_trace(path))``.
"""

from __future__ import annotations

import json
from collections.abc import Sequence

import numpy as np
import torch

from . import _native
from .columns import TraceColumns
from .trace_model import SCHEMA_VERSION, TraceError, _Loader, load_trace

L_EMPTY, L_POWER, L_OP, L_KERNEL, L_OTHER = 0, 1, 2, 3, 4


def _fallback():
    """The device path declines the file (the reference loader takes it);
    DWB200_INGEST_DEBUG=1 says where."""
    import os
    if os.environ.get("DWB200_INGEST_DEBUG"):
        import inspect
        import sys
        print(f"ingest: device path declined at ingest.py:{inspect.currentframe().f_back.f_lineno}",
              file=sys.stderr)
    return None
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
    cols.tensors, cols.progmodel, cols.blocktraces = tr.tensors, tr.progmodel, tr.blocktraces
    cols.op_tensors = [(o.input_tensor_ids, o.output_tensor_ids) for o in tr.operators] \
        if any(o.input_tensor_ids or o.output_tensor_ids for o in tr.operators) else None
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
        return _fallback()
    # the other records (header, config, tensors, program model, block traces) are read on the host
    other = torch.nonzero(ltype == L_OTHER).flatten()
    nonempty = torch.nonzero(ltype != L_EMPTY).flatten()
    if nonempty.numel() == 0 or other.numel() == 0 or int(nonempty[0]) != int(other[0]):
        return _fallback()  # the first record must be the header
    ends_h = ends.cpu().numpy()
    # header, config, tensors, program model, block traces: the loader decodes
    # them (and validates what concerns them alone); power / op / kernel stay
    # on the device
    host = _Loader()
    try:
        for i in other.cpu().tolist():
            a = 0 if i == 0 else int(ends_h[i - 1]) + 1
            host.feed(i + 1, raw[a:int(ends_h[i])].tobytes().decode("utf-8"))
    except (ValueError, UnicodeDecodeError, TraceError, AttributeError, TypeError, KeyError):
        return _fallback()
    if host.header is None or host.ops or host.kernels or host.power:
        return _fallback()  # op / kernel / power records off the device's canonical form
    header, config = host.header, dict(host.config)
    lines = {t: torch.nonzero(ltype == t).flatten() for t in (L_POWER, L_OP, L_KERNEL)}
    npw, nop, nk = (int(lines[t].numel()) for t in (L_POWER, L_OP, L_KERNEL))
    i64 = lambda m: torch.empty(m, dtype=torch.int64, device=dev)  # noqa: E731
    i32 = lambda m: torch.empty(m, dtype=torch.int32, device=dev)  # noqa: E731
    ts, watts = i64(npw), torch.empty(npw, dtype=torch.float64, device=dev)
    _native.check(L.dw_ig_parse_power(p(buf), p(ends), p(lines[L_POWER]), npw, p(ts), p(watts), p(flags), st),
                  "dw_ig_parse_power")
    o_id, o_idl, o_nm, o_nml, o_klf, o_klc, o_s, o_e = i64(nop), i32(nop), i64(nop), i32(nop), i64(nop), i32(nop), \
        i64(nop), i64(nop)
    tl_off, tl_len = i64(2 * nop), i32(2 * nop)
    _native.check(L.dw_ig_parse_op(p(buf), p(ends), p(lines[L_OP]), nop, p(o_id), p(o_idl), p(o_nm), p(o_nml),
                                   p(o_klf), p(o_klc), p(o_s), p(o_e), p(tl_off), p(tl_len), p(flags), st),
                  "dw_ig_parse_op")
    k_id, k_idl, k_nm, k_nml, k_corr, k_s, k_e = i64(nk), i32(nk), i64(nk), i32(nk), i64(nk), i64(nk), i64(nk)
    _native.check(L.dw_ig_parse_kernel(p(buf), p(ends), p(lines[L_KERNEL]), nk, p(k_id), p(k_idl), p(k_nm),
                                       p(k_nml), p(k_corr), p(k_s), p(k_e), p(flags), st), "dw_ig_parse_kernel")
    if npw == 0:
        return _fallback()
    # the device checks, read back together (one synchronisation): parse flags,
    # power order, unique op / kernel ids (sorted 64-bit hashes: any equal pair
    # goes to the Python path), unique correlation ids, one owner per kernel
    def hashes(off, ln, m):
        h = torch.empty(m, dtype=torch.int64, device=dev)
        idx = torch.empty(m, dtype=torch.int32, device=dev)
        _native.check(L.dw_ig_hash(p(buf), p(off), p(ln), m, p(h), p(idx), st), "dw_ig_hash")
        hs, order = torch.sort(h ^ torch.iinfo(torch.int64).min)  # unsigned order
        return hs ^ torch.iinfo(torch.int64).min, idx[order]

    def dup(sorted_vals):
        return (sorted_vals[1:] == sorted_vals[:-1]).any() if sorted_vals.numel() > 1 else no

    no = torch.zeros((), dtype=torch.bool, device=dev)
    oh = hashes(o_id, o_idl, nop)[0] if nop else i64(0)
    kh, kidx = hashes(k_id, k_idl, nk) if nk else (i64(0), i32(0))
    o_klc64 = o_klc.to(torch.int64)
    checks = torch.stack([flags.reshape(()).to(torch.int64),
                          ((ts[1:] <= ts[:-1]).any() if npw > 1 else no).to(torch.int64),
                          dup(oh).to(torch.int64), dup(kh).to(torch.int64),
                          dup(torch.sort(k_corr).values if nk > 1 else k_corr).to(torch.int64),
                          o_klc64.sum() if nop else torch.zeros((), dtype=torch.int64, device=dev)]).cpu().tolist()
    bad_flags, bad_order, dup_op, dup_k, dup_corr, ne = checks
    if bad_flags or bad_order or dup_op or dup_k or dup_corr:
        return _fallback()  # order / duplicate ids / correlation ids: the Python path raises
    # kernels flattened in op.kernel_ids order (build_ledger's iteration order)
    kl_base = torch.cumsum(o_klc64, 0) - o_klc64
    if ne != nk:
        return _fallback()  # some kernel is not launched by exactly one operator
    fk_s, fk_e, fk_op, fk_k = i64(ne), i64(ne), i32(ne), i64(ne)
    owner = torch.zeros(max(nk, 1), dtype=torch.int32, device=dev)
    _native.check(L.dw_ig_kernel_lists(p(buf), nop, p(o_klf), p(o_klc), p(kl_base), p(o_s), p(o_e), p(kh),
                                       p(kidx), nk, p(k_id), p(k_idl), p(k_s), p(k_e), p(fk_s), p(fk_e), p(fk_op),
                                       p(fk_k), p(owner), p(flags), st), "dw_ig_kernel_lists")
    # Trace.span_us (trace_model.py:307-314): every timestamp of the trace
    parts = [ts.max()]
    if nop:
        parts += [o_e.max(), o_s.max()]
    if nk:
        parts += [k_e.max(), k_s.max()]
    tail = torch.stack([flags.reshape(()).to(torch.int64),
                        ((owner[:nk] != 1).any() if nk else no).to(torch.int64),
                        torch.stack(parts).max()]).cpu().tolist()
    if tail[0] or tail[1]:
        return _fallback()
    trace_end = int(tail[2])
    h = lambda t: t.cpu().numpy()  # noqa: E731
    k_id_h, k_idl_h, fk_k_h = h(k_id), h(k_idl), h(fk_k)
    cols = TraceColumns(ts=ts, watts=watts, trace_end=trace_end, op_start=o_s, op_end=o_e, k_start=fk_s,
                        k_end=fk_e, k_op=fk_op, op_ids=StrView(raw, h(o_id), h(o_idl)),
                        k_ids=StrView(raw, k_id_h[fk_k_h], k_idl_h[fk_k_h]),
                        op_names=StrView(raw, h(o_nm), h(o_nml)),
                        k_names=StrView(raw, h(k_nm)[fk_k_h], h(k_nml)[fk_k_h]))
    extra = _host_records(host, raw, tl_off, tl_len, nop)
    if extra is None:
        return _fallback()
    cols.header, cols.config, cols.loaded_by = header, config, "gpu"
    cols.tensors, cols.progmodel, cols.blocktraces, cols.op_tensors = extra
    if nop:
        cols.op_rank = id_ranks(buf, o_id, o_idl)
    return cols


def _host_records(host: _Loader, raw: np.ndarray, tl_off: torch.Tensor, tl_len: torch.Tensor, nop: int):
    """The rules that tie operators to the host-decoded records
    (trace_model.py:511-586 as restated in trace_model._Checks): the loader's
    own checks on its records, then every tensor id an operator references
    exists, no id is both input and output of one operator, one producer per
    tensor, and an acyclic operator graph.  Returns (tensors, progmodel,
    blocktraces, per-op (inputs, outputs) or None) or None on any violation
    (the reference loader then raises the exact error)."""
    try:
        part = host.finish()  # tensors' run rules, program-model rules (no ops / kernels / power here)
    except TraceError:
        return _fallback()
    lens = tl_len.view(-1, 2) if nop else tl_len
    if not nop or not bool((lens > 2).any()):  # no operator references a tensor
        return part.tensors, part.progmodel, part.blocktraces, None
    offs, ln = tl_off.view(-1, 2).cpu().numpy(), lens.cpu().numpy()

    def strs(o, n):
        if n <= 2:
            return ()
        return tuple(raw[o + 2:o + n - 2].tobytes().decode("ascii").split('","'))
    io = [(strs(offs[i, 0], ln[i, 0]), strs(offs[i, 1], ln[i, 1])) for i in range(nop)]
    known = part.tensors.keys()
    made_by: dict = {}
    for i, (ins, outs) in enumerate(io):
        if not (set(ins) <= known and set(outs) <= known) or set(ins) & set(outs):
            return _fallback()
        for t in outs:
            if t in made_by:
                return _fallback()
            made_by[t] = i
    # acyclic: Kahn's peel over operator indices
    from collections import deque
    succ = [[] for _ in range(nop)]
    indeg = [0] * nop
    for i, (ins, _) in enumerate(io):
        for t in ins:
            j = made_by.get(t)
            if j is not None:
                succ[j].append(i)
                indeg[i] += 1
    q = deque(i for i in range(nop) if indeg[i] == 0)
    peeled = 0
    while q:
        i = q.popleft()
        peeled += 1
        for n in succ[i]:
            indeg[n] -= 1
            if indeg[n] == 0:
                q.append(n)
    if peeled != nop:
        return _fallback()
    return part.tensors, part.progmodel, part.blocktraces, io


def id_ranks(buf: torch.Tensor, off: torch.Tensor, length: torch.Tensor) -> torch.Tensor:
    """Lexicographic rank of byte-string ids (Python str order for ASCII ids:
    a shorter id sorts before its extensions) on the device: each id as
    big-endian 8-byte words (zero padded, dw_ig_id_words), stable sorts from
    the last word to the first, then the inverse permutation.  ``buf`` holds
    the bytes (device uint8); ids are spans (off, length).  Equal ids share
    no rank guarantee (ids are unique where this is used)."""
    L = _native.lib()
    p = _native.ptr
    n = int(off.numel())
    dev = buf.device
    if n == 0:
        return torch.empty(0, dtype=torch.int64, device=dev)
    nw = (int(length.max().item()) + 7) // 8
    order = torch.arange(n, dtype=torch.int64, device=dev)
    words = torch.empty(n, dtype=torch.int64, device=dev)
    flip = torch.iinfo(torch.int64).min
    for w in range(nw - 1, -1, -1):
        _native.check(L.dw_ig_id_words(p(buf), p(off), p(length), n, w, p(words), _native.stream_handle()),
                      "dw_ig_id_words")
        key = (words ^ flip)[order]  # unsigned order as signed
        order = order[torch.sort(key, stable=True).indices]
    rank = torch.empty(n, dtype=torch.int64, device=dev)
    rank[order] = torch.arange(n, dtype=torch.int64, device=dev)
    return rank
