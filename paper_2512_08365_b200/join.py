"""Scale path of the differential diff: signature hash-join + deltas + ranked
top-k, all on the device (csrc/diff.cu ``dw_join_diff`` and ``dw_rank``).

The reference pairs operators through SVD tensor matching and dominator cuts
(subgraph_match.py:322-422), a sequential graph algorithm.  At 1e8 operators
the north star replaces that pairing with a join on operator signatures, which
the reference does not define; the definition used here
(DESIGN.md "signature join"):

  * signature = 64-bit hash of (op name, layout-blind input shapes = element
    counts, dtype, call site / config key).  Reference-style traces carry no
    dtype or call site; they hash as "float64" and "".
  * an operator's key is (signature, k) where k counts earlier operators of the
    same signature in trace order (the k-th occurrence);
  * equal keys pair up; unmatched operators become one-sided findings whose
    other side is empty (energy 0, latency 0), judged by the reference's rule.

Findings are numbered: A's operators in order (matched or A-only), then B-only
operators in B order.  Ranking and verdicts follow detect.py exactly, with
nodes_a = (op_id,) or () for B-only findings.
"""

from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native
from .columns import TraceColumns, synthetic_id, synthetic_ids
from .detect import (DEFAULT_THRESHOLD, SIDES, VERDICT_WASTE, VERDICTS, FindingColumns,
                     Report, SubgraphPair, WasteFinding, judge, rank_order)
from .energy import EnergyLedger


def signature_of(op_name: str, shapes: Sequence[int] = (), dtype: str = "float64",
                 callsite: str = "") -> int:
    """64-bit signature of one operator (blake2b of the canonical fields)."""
    text = "\x1f".join([op_name, ",".join(str(int(s)) for s in shapes), dtype, callsite])
    return int.from_bytes(hashlib.blake2b(text.encode(), digest_size=8).digest(), "little")


def trace_signatures(trace) -> np.ndarray:
    """Signatures of a reference-style Trace's operators (op name + element
    counts of its input tensors, in order)."""
    out = np.empty(len(trace.operators), dtype=np.uint64)
    tensors = getattr(trace, "tensors", {}) or {}
    for i, op in enumerate(trace.operators):
        shapes = []
        for t in op.input_tensor_ids:
            snaps = tensors.get(t)
            shapes.append(int(np.prod(snaps[0].shape)) if snaps else 0)
        out[i] = signature_of(op.op_name, shapes)
    return out


def _sig_tensor(cols: TraceColumns, trace, dev) -> torch.Tensor:
    if cols.op_sig is None:
        if trace is None or isinstance(trace, TraceColumns):
            if cols.op_names is None:
                raise ValueError("no operator signatures: give op_sig or op_names")
            sig = np.array([signature_of(n) for n in cols.op_names], dtype=np.uint64)
        else:
            sig = trace_signatures(trace)
        cols.op_sig = sig
    s = cols.device("op_sig")
    return s if s.dtype == torch.int64 else s.view(torch.int64)


def _ranks(cols: TraceColumns, dev) -> Optional[torch.Tensor]:
    """Lexicographic rank of op ids (nodes_a tie-break); identity when ids are
    absent (synthetic ids are zero-padded, so rank == index)."""
    if cols.op_rank is not None:
        return cols.device("op_rank")
    if cols.op_ids is None:
        return None
    # ids from the Python loader: their UTF-8 bytes (byte order = str order)
    # ranked on the device, as ingest does for files it parses
    from .ingest import id_ranks
    enc = [str(x).encode("utf-8") for x in cols.op_ids]
    lens = np.fromiter((len(e) for e in enc), dtype=np.int64, count=len(enc))
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]) if len(enc) else np.zeros(0, dtype=np.int64)
    buf = torch.from_numpy(np.frombuffer(b"".join(enc) or b"\0", dtype=np.uint8).copy()).to(dev)
    cols.op_rank = id_ranks(buf, torch.from_numpy(offs.astype(np.int64)).to(dev),
                            torch.from_numpy(lens.astype(np.int32)).to(dev))
    return cols.device("op_rank")


def _ledger_joules(cols: TraceColumns, led: EnergyLedger, dev) -> torch.Tensor:
    """The ledger's operator joules in ``cols``' operator order.  The device
    column is used as is only when it belongs to these columns (same length,
    same op ids in the same order); otherwise it is rebuilt by id, so a ledger
    of other columns can never be read out of bounds or misattributed."""
    j = led.operator_tensor()
    per = led.per_operator
    ids = cols.op_ids
    if j is not None and j.numel() == cols.n_ops:
        own = getattr(per, "_ids", None)
        if ids is None and own is None:
            return j
        if ids is not None and own is not None and (own is ids or list(own) == list(ids)):
            return j
    if ids is None:
        ids = synthetic_ids("op", cols.n_ops)
    if len(per) != len(ids):
        raise ValueError(f"ledger has {len(per)} operators, the trace {len(ids)}")
    return torch.tensor([float(per[o]) for o in ids], dtype=torch.float64, device=dev)


@dataclass
class JoinDiff:
    """Device-resident result of dw_join_diff (+ dw_rank).  Finding f < n_a is
    A op f (paired with match_a[f] or A-only); finding n_a + r is B-only op
    b_only[r]."""

    P: int
    n_a: int
    n_matched: int
    n_a_only: int
    n_b_only: int
    columns: FindingColumns
    match_a: torch.Tensor        # int32 [n_a]
    b_only: torch.Tensor         # int32 [n_b_only]
    epw_a: Optional[torch.Tensor]
    epw_b: Optional[torch.Tensor]
    order: Optional[torch.Tensor]  # top-k finding indices, report order (None: ranked elsewhere)
    n_waste: int
    wasted_joules: float         # exact sum over all waste findings
    ja: Optional[torch.Tensor] = None    # operator joules of A / B (for lean columns)
    jb: Optional[torch.Tensor] = None
    threshold: float = DEFAULT_THRESHOLD
    rows_host: Optional[np.ndarray] = None  # dw_topk_rows of ``order``, read back with the counts

    def pair_of(self, f: torch.Tensor):
        """(A op, B op) of findings f (device tensors; -1 on an empty side)."""
        is_a = f < self.n_a
        ia = torch.where(is_a, f, torch.full_like(f, -1))
        fa = f.clamp(max=max(self.n_a - 1, 0))
        fb = (f - self.n_a).clamp(min=0, max=max(self.n_b_only - 1, 0))
        ma = self.match_a[fa].to(torch.int64) if self.n_a else torch.full_like(f, -1)
        bo = self.b_only[fb].to(torch.int64) if self.n_b_only else torch.full_like(f, -1)
        ib = torch.where(is_a, ma, bo)
        return ia, ib

    def _top_lean(self, cols_a, cols_b, classify, trace_a, trace_b, idx) -> list[WasteFinding]:
        """top_findings for lean joins (no per-finding verdict columns): the
        k rows' operators, joules and latencies in one device gather
        (dw_topk_rows) and one copy; verdicts on the host with the device's
        rule (judge)."""
        k = int(idx.numel())
        if idx is self.order and self.rows_host is not None:
            h = self.rows_host  # gathered by join_diff right after the rank
        else:
            out = torch.empty((6, max(k, 1)), dtype=torch.int64, device=idx.device)
            _topk_rows(idx, k, self, cols_a, cols_b, out)
            h = out[:, :k].cpu().numpy()
        ia, ib, la, lb = h[0], h[1], h[2], h[3]
        ea, eb = h[4].view(np.float64), h[5].view(np.float64)
        return self._rows(cols_a, cols_b, classify, trace_a, trace_b, ia, ib, ea, eb, la, lb, None)

    def top_findings(self, cols_a: TraceColumns, cols_b: TraceColumns, classify: bool = True,
                     trace_a=None, trace_b=None, idx: Optional[torch.Tensor] = None) -> list[WasteFinding]:
        """Materialise the top-k findings (report order) as reference-style
        WasteFinding objects; columns not written by the join are gathered from
        the ledgers on the device for these k rows only.  Waste findings are
        classified as detect_waste does (diagnose.classify_pairs; the trace
        objects, when given, enable the program-model probe)."""
        idx = self.order if idx is None else idx
        c = self.columns
        if c.ratio is None and c.energy_a is None and c.latency_a is None and self.ja is not None:
            return self._top_lean(cols_a, cols_b, classify, trace_a, trace_b, idx)
        ia_d, ib_d = self.pair_of(idx)
        has_a, has_b = ia_d >= 0, ib_d >= 0
        ia_c, ib_c = ia_d.clamp(min=0), ib_d.clamp(min=0)

        def pick(name, fallback):
            t = getattr(c, name)
            return t[idx] if t is not None else fallback()

        zero_f = torch.zeros((), dtype=torch.float64, device=idx.device)
        zero_i = torch.zeros((), dtype=torch.int64, device=idx.device)
        # every column of the k rows in two device tensors: two D2H copies
        keys_only = c.ratio is None
        fl = [pick("energy_a", lambda: torch.where(has_a, self.ja[ia_c], zero_f)),
              pick("energy_b", lambda: torch.where(has_b, self.jb[ib_c], zero_f))]
        if not keys_only:
            fl += [c.ratio[idx], c.wasted[idx]]
        fcols = torch.stack(fl).cpu().numpy()
        il = [pick("latency_a", lambda: torch.where(
                  has_a, cols_a.device("op_end")[ia_c] - cols_a.device("op_start")[ia_c], zero_i)),
              pick("latency_b", lambda: torch.where(
                  has_b, cols_b.device("op_end")[ib_c] - cols_b.device("op_start")[ib_c], zero_i)),
              ia_d, ib_d]
        if not keys_only:
            il += [c.verdict[idx].to(torch.int64), c.side[idx].to(torch.int64),
                   c.informational[idx].to(torch.int64)]
        icols = torch.stack(il).cpu().numpy()
        ea, eb = fcols[0], fcols[1]
        la, lb = icols[0], icols[1]
        ia, ib = icols[2], icols[3]
        h = None if keys_only else {"ratio": fcols[2], "wasted": fcols[3], "verdict": icols[4],
                                    "side": icols[5], "informational": icols[6]}
        return self._rows(cols_a, cols_b, classify, trace_a, trace_b, ia, ib, ea, eb, la, lb, h)

    def _rows(self, cols_a, cols_b, classify, trace_a, trace_b, ia, ib, ea, eb, la, lb, h) -> list[WasteFinding]:
        """WasteFinding rows from the k rows' columns; ``h`` None: the verdict
        columns derived on the host with the device's rule (judge)."""
        ia, ib = np.asarray(ia).tolist(), np.asarray(ib).tolist()
        ea, eb = np.asarray(ea, dtype=np.float64).tolist(), np.asarray(eb, dtype=np.float64).tolist()
        la, lb = np.asarray(la).tolist(), np.asarray(lb).tolist()
        k = len(ia)
        if h is None:  # the k rows' verdicts on the host, as the device computed them for all
            rows = [judge(ea[r], eb[r], la[r], lb[r], 0.0, self.threshold) for r in range(k)]
            ratio = [x[0] for x in rows]
            wasted = [x[1] for x in rows]
            verdict = [x[2] for x in rows]
            side = [x[3] for x in rows]
            info = [bool(x[4]) for x in rows]
        else:
            ratio, wasted = np.asarray(h["ratio"]).tolist(), np.asarray(h["wasted"]).tolist()
            verdict = [VERDICTS[v] for v in np.asarray(h["verdict"]).tolist()]
            side = [SIDES[v] for v in np.asarray(h["side"]).tolist()]
            info = [bool(v) for v in np.asarray(h["informational"]).tolist()]

        def namer(cols):
            ids = cols.op_ids
            if ids is not None:
                return lambda i: ids[i]
            w = len(str(max(cols.n_ops - 1, 0)))  # synthetic_id's zero padding
            return lambda i: f"op{i:0{w}d}"
        name_a, name_b = namer(cols_a), namer(cols_b)
        cats = ["unknown"] * k
        waste = [r for r in range(k) if verdict[r] == VERDICT_WASTE]
        if classify and waste:
            from .diagnose import classify_pairs
            got = classify_pairs(cols_a, cols_b, [side[r] for r in waste], np.asarray([ia[r] for r in waste]),
                                 np.asarray([ib[r] for r in waste]), trace_a, trace_b)
            for r, c in zip(waste, got):
                cats[r] = c
        return [WasteFinding(
            pair=SubgraphPair(nodes_a=(name_a(ia[r]),) if ia[r] >= 0 else (),
                              nodes_b=(name_b(ib[r]),) if ib[r] >= 0 else ()),
            energy_a=ea[r], energy_b=eb[r], energy_ratio=ratio[r], latency_a=la[r], latency_b=lb[r],
            output_rel_diff=0.0, verdict=verdict[r], category=cats[r], wasteful_side=side[r],
            wasted_joules=wasted[r], informational=info[r]) for r in range(k)]


DEFAULT_MAX_DISTINCT = 1 << 20


@dataclass
class JoinPrep:
    """The pairing of two traces' operators (dw_join_prepare): it needs only
    the signatures, so it can run on its own stream while the ledgers that
    supply the joules are still computing.  Holds its workspace until
    ``join_diff(..., prep=)`` writes the findings."""

    ca: TraceColumns
    cb: TraceColumns
    keep: list
    match_a: torch.Tensor
    b_only: torch.Tensor
    n_b_only: int
    ws: torch.Tensor
    max_distinct: int


def _topk_rows(idx, k, jd, cols_a, cols_b, out) -> None:
    """dw_topk_rows: the k rows' ops, latencies and joules into out [6, k]."""
    p = _native.ptr
    o = idx.contiguous()
    _native.check(_native.lib().dw_topk_rows(
        p(o), k, jd.n_a, p(jd.match_a), p(jd.b_only), p(jd.ja), p(jd.jb),
        p(cols_a.device("op_start")), p(cols_a.device("op_end")), p(cols_b.device("op_start")),
        p(cols_b.device("op_end")), p(out), _native.stream_handle()), "dw_topk_rows")


def _side(cols, trace, joules, work, rank, dev):
    p = _native.ptr
    sig = _sig_tensor(cols, trace, dev)
    s, e = cols.device("op_start"), cols.device("op_end")
    return _native.JoinSide(p(sig), p(s), p(e), p(joules), p(work), p(rank), cols.n_ops), [sig, s, e]


def join_prepare(trace_a, trace_b, *, max_distinct: int = DEFAULT_MAX_DISTINCT, stream=None) -> JoinPrep:
    """Pair the operators of two traces by (signature, occurrence) on the
    device (the first half of ``join_diff``)."""
    dev = _native.device()
    ca, cb = TraceColumns.from_trace(trace_a), TraceColumns.from_trace(trace_b)
    sa, ka = _side(ca, trace_a, None, None, None, dev)
    sb, kb = _side(cb, trace_b, None, None, None, dev)
    na, nb = ca.n_ops, cb.n_ops
    match_a = torch.empty(max(na, 1), dtype=torch.int32, device=dev)
    bonly_t = torch.empty(max(nb, 1), dtype=torch.int32, device=dev)
    L = _native.lib()
    p = _native.ptr
    md = int(min(max_distinct, na + nb)) if max_distinct else 0
    nbo = ctypes.c_int64(0)
    while True:
        ws = torch.empty(int(L.dw_join_workspace_size(na, nb, md)), dtype=torch.uint8, device=dev)
        rc = L.dw_join_prepare(ctypes.byref(sa), ctypes.byref(sb), md, p(match_a), p(bonly_t), ctypes.byref(nbo),
                               ws.data_ptr(), ws.numel(), _native.stream_handle(stream))
        if rc == _native.DW_E_WORKSPACE and md and md < na + nb:
            md = min(4 * md, na + nb)  # more distinct signatures than the table held
            continue
        break
    _native.check(rc, "dw_join_prepare")
    return JoinPrep(ca, cb, ka + kb, match_a, bonly_t, int(nbo.value), ws, md)


def join_diff(trace_a, trace_b, ledger_a: EnergyLedger, ledger_b: EnergyLedger,
              threshold: float = DEFAULT_THRESHOLD, k: int = 100, *, full_columns: bool = True,
              epw: bool = True, work_a=None, work_b=None, stream=None,
              max_distinct: int = DEFAULT_MAX_DISTINCT, prep: Optional[JoinPrep] = None,
              columns: Optional[Sequence[str]] = None, ranked: bool = True) -> JoinDiff:
    """Signature-join diff of two traces with their ledgers; top-k ranked.
    ``prep``: the pairing already made by ``join_prepare`` (same traces).
    ``ranked=False``: no ranking here (``order`` None, n_waste / wasted_joules
    0) -- a corpus ranks all its pairs at once (``pipeline.analyze_corpus``)."""
    if ledger_a.method != ledger_b.method:
        raise ValueError(f"ledger method mismatch: {ledger_a.method!r} vs {ledger_b.method!r}")
    if not 0 < threshold <= 1:
        raise ValueError("threshold must be in (0, 1]")
    dev = _native.device()
    if prep is None:
        prep = join_prepare(trace_a, trace_b, max_distinct=max_distinct, stream=stream)
    ca, cb = prep.ca, prep.cb
    sides, keep = [], []
    for cols, trace, led, work in ((ca, trace_a, ledger_a, work_a), (cb, trace_b, ledger_b, work_b)):
        j = _ledger_joules(cols, led, dev)
        w = None
        if work is not None:
            w = work if isinstance(work, torch.Tensor) else torch.as_tensor(work, dtype=torch.float64)
            w = w.to(device=dev, dtype=torch.float64).reshape(-1)
        elif cols.op_work is not None:
            w = cols.device("op_work")
        if w is not None and w.numel() != cols.n_ops:
            raise ValueError(f"work column has {w.numel()} entries for {cols.n_ops} operators")
        rank = _ranks(cols, dev) if cols is ca else None
        side, kk = _side(cols, trace, j, w, rank, dev)
        sides.append(side)
        keep += [j, w, rank] + kk
    na, nb = ca.n_ops, cb.n_ops
    Pmax = na + nb
    rank_a = keep[2]
    fc = FindingColumns(Pmax, dev, full=full_columns, columns=columns, key_lo=False, tie_rank=rank_a, n_a=na)
    epw_a = torch.empty(Pmax, dtype=torch.float64, device=dev) if epw else None
    epw_b = torch.empty(Pmax, dtype=torch.float64, device=dev) if epw else None
    na_ = na + prep.n_b_only
    kk = min(k, na_)
    # one device buffer, one read-back: counts [4], rank summary [4] (f64
    # bits), and -- lean columns -- the top-k report rows [6, k]
    hb = torch.empty(8 + 6 * max(kk, 1), dtype=torch.int64, device=dev)
    count = hb[:4]  # written whole by dw_join_findings
    L = _native.lib()
    fs = fc.c_struct()
    p = _native.ptr
    _native.check(L.dw_join_findings(ctypes.byref(sides[0]), ctypes.byref(sides[1]), prep.max_distinct,
                                     float(threshold), ctypes.byref(fs), p(prep.match_a), p(prep.b_only),
                                     prep.n_b_only, p(epw_a), p(epw_b), p(count), prep.ws.data_ptr(),
                                     prep.ws.numel(), _native.stream_handle(stream)), "dw_join_findings")
    P = na_
    jd = JoinDiff(P=P, n_a=na, n_matched=0, n_a_only=0, n_b_only=prep.n_b_only, columns=fc,
                  match_a=prep.match_a[:na], b_only=prep.b_only[:prep.n_b_only], epw_a=epw_a, epw_b=epw_b,
                  order=None, n_waste=0, wasted_joules=0.0, ja=keep[0], jb=keep[6], threshold=float(threshold))
    lean = fc.ratio is None and fc.energy_a is None and fc.latency_a is None
    if ranked:
        summary = hb[4:8].view(torch.float64)
        summary.zero_()
        jd.order, _ = rank_order(fc.key_hi[:P], None, kk, tie_rank=rank_a, n_a=na, summary=summary)
        if lean and kk:
            _topk_rows(jd.order, kk, jd, ca, cb, hb[8:].view(6, kk))
        h = hb.cpu().numpy()
        sm = h[4:8].view(np.float64)
        jd.n_waste, jd.wasted_joules = int(sm[0]), float(sm[1])
        if lean and kk:
            jd.rows_host = h[8:].reshape(6, kk)
    else:
        h = hb[:4].cpu().numpy()
    P2, matched, a_only, b_only = (int(x) for x in h[:4])
    if P2 != P or b_only != prep.n_b_only:
        raise RuntimeError(f"internal: join counted {P2} findings ({b_only} B-only), expected {P}")
    jd.n_matched, jd.n_a_only = matched, a_only
    return jd


def join_report(trace_a, trace_b, ledger_a: EnergyLedger, ledger_b: EnergyLedger,
                threshold: float = DEFAULT_THRESHOLD, k: int = 100) -> tuple[Report, JoinDiff]:
    """A reference-shaped Report holding the top-k findings of the join diff;
    wasted_joules / end_to_end_waste_pct cover every waste finding."""
    jd = join_diff(trace_a, trace_b, ledger_a, ledger_b, threshold, k)
    ca, cb = TraceColumns.from_trace(trace_a), TraceColumns.from_trace(trace_b)
    top = jd.top_findings(ca, cb, trace_a=None if isinstance(trace_a, TraceColumns) else trace_a,
                          trace_b=None if isinstance(trace_b, TraceColumns) else trace_b)
    ineff = max(ledger_a.total_joules, ledger_b.total_joules)
    pct = jd.wasted_joules / ineff if ineff > 0 else 0.0
    rep = Report(findings=tuple(top), total_a=ledger_a.total_joules, total_b=ledger_b.total_joules,
                 wasted_joules=jd.wasted_joules, end_to_end_waste_pct=pct, method=ledger_a.method,
                 threshold=threshold)
    return rep, jd
