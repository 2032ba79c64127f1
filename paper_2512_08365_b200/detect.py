"""Waste detection and report ranking -- drop-in for ``diffwatt.detect``.

``detect_waste`` and ``report`` keep the reference's names, signatures, return
types and errors (detect.py:72-130, 256-278).  The per-pair arithmetic (member
sums, latency, ratio, verdict, wasted joules, ranking key) runs in
csrc/diff.cu (``dw_detect_pairs``) and the report order comes from the device
ranking (``dw_rank``); the host only builds the CSR member lists, evaluates the
boundary-tensor output rule (tensor snapshots live on the host) and
materialises the findings.

Category: like the reference, every waste finding is classified
(detect.py:127-128, 137-172) -- here in one batch (``diagnose.classify_findings``:
one device integral launch for all forced gaps).  ``classify=fn`` substitutes a
per-finding function (e.g. the reference's own ``diffwatt.detect.classify``),
``classify=False`` skips the step and leaves "unknown".
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native
from .energy import EnergyLedger
from .columns import TraceColumns, synthetic_id, synthetic_ids
from .tensor_equiv import boundary_rel_diff

DEFAULT_THRESHOLD = 0.10
THRESHOLD_FLOOR = 0.05
LATENCY_SLACK = 1.01
OUTPUT_DIFF_LIMIT = 0.01

VERDICT_WASTE = "waste"
VERDICT_TRADEOFF = "tradeoff"
VERDICT_BELOW = "below_threshold"

VERDICTS = (VERDICT_BELOW, VERDICT_TRADEOFF, VERDICT_WASTE)  # device codes 0, 1, 2
SIDES = ("-", "A", "B")


@dataclass(frozen=True)
class SubgraphPair:
    """Field-compatible with the reference's SubgraphPair (subgraph_match.py:66-76)."""

    nodes_a: tuple[str, ...]
    nodes_b: tuple[str, ...]
    boundary_left: tuple[tuple[str, str], ...] = ()
    boundary_right: tuple[tuple[str, str], ...] = ()
    depth: int = 0
    coarse: bool = False

    def size(self) -> int:
        return max(len(self.nodes_a), len(self.nodes_b))


@dataclass(frozen=True)
class WasteFinding:
    pair: object
    energy_a: float
    energy_b: float
    energy_ratio: float
    latency_a: int
    latency_b: int
    output_rel_diff: float
    verdict: str
    category: str
    wasteful_side: str
    wasted_joules: float
    informational: bool


class FindingColumns:
    """Device columns of a batch of findings (one dw_findings_t).  ``columns``
    selects which optional columns are written (the ranking keys always are)."""

    ALL = ("energy_a", "energy_b", "ratio", "wasted", "latency_a", "latency_b", "verdict", "side",
           "informational", "delta_e", "delta_t", "epw_ratio")
    LEAN = ("ratio", "wasted", "verdict", "side", "informational")
    KEYS = ("key_hi",)  # the ranking key only: every other column is derived for the top-k rows
    # the differential output of the north star (3): energy and time deltas and the
    # energy-per-useful-work ratio per pair, plus the ranking key (32 B per finding)
    DELTAS = ("delta_e", "delta_t", "epw_ratio")

    def __init__(self, P: int, dev, full: bool = True, columns=None, key_lo: bool = True,
                 tie_rank=None, n_a: int = 0):
        cols = self.ALL if (columns is None and full) else (columns or self.LEAN)
        self.tie_rank, self.n_a = tie_rank, n_a
        types = {"energy_a": torch.float64, "energy_b": torch.float64, "ratio": torch.float64,
                 "wasted": torch.float64, "latency_a": torch.int64, "latency_b": torch.int64,
                 "verdict": torch.int8, "side": torch.int8, "informational": torch.int8,
                 "delta_e": torch.float64, "delta_t": torch.int64, "epw_ratio": torch.float64}
        self.P = P
        self.key_hi = torch.empty(P, dtype=torch.int64, device=dev)
        self.key_lo = torch.empty(P, dtype=torch.int64, device=dev) if key_lo else None
        for name in self.ALL:
            setattr(self, name, torch.empty(P, dtype=types[name], device=dev) if name in cols else None)

    def c_struct(self) -> _native.Findings:
        p = _native.ptr
        return _native.Findings(p(self.energy_a), p(self.energy_b), p(self.ratio),
                                p(self.latency_a), p(self.latency_b), p(self.verdict),
                                p(self.side), p(self.informational), p(self.wasted),
                                p(self.key_hi), p(self.key_lo), p(self.tie_rank), int(self.n_a),
                                p(self.delta_e), p(self.delta_t), p(self.epw_ratio))

    def host(self, idx=None) -> dict:
        names = self.ALL
        out = {}
        for n in names:
            t = getattr(self, n)
            if t is None:
                continue
            if idx is not None:
                t = t[idx]
            out[n] = t.cpu().numpy()
        return out


def judge(ea: float, eb: float, la: int, lb: int, out_diff: float, threshold: float) -> tuple:
    """One pair's (ratio, wasted, verdict, side, informational), detect.py:93-126
    -- the host twin of csrc/diff.cu judge() (same IEEE operations)."""
    high, low = (ea, eb) if ea >= eb else (eb, ea)
    if high == low:
        ratio, side = 1.0, "-"
    else:
        ratio = high / low if low > 0 else float("inf")
        side = "A" if ea > eb else "B"
    if ratio >= 1.0 + threshold:
        eff, ineff = (lb, la) if side == "A" else (la, lb)
        verdict = VERDICT_WASTE if (float(eff) <= LATENCY_SLACK * float(ineff) and
                                    out_diff <= OUTPUT_DIFF_LIMIT) else VERDICT_TRADEOFF
    else:
        verdict = VERDICT_BELOW
    info = verdict == VERDICT_BELOW and ratio >= 1.0 + THRESHOLD_FLOOR
    return ratio, high - low, verdict, side, info


def _check_args(ledger_a, ledger_b, threshold):
    if ledger_a.method != ledger_b.method:
        raise ValueError(f"ledger method mismatch: {ledger_a.method!r} vs {ledger_b.method!r}")
    if not 0 < threshold <= 1:
        raise ValueError("threshold must be in (0, 1]")


def _op_columns(trace, ledger, dev):
    """(op index by id, joules, start, end) of one trace, joules in the ledger's
    op order (which is the trace's op order for ledgers built here)."""
    cols = TraceColumns.from_trace(trace)
    ids = cols.op_ids if cols.op_ids is not None else synthetic_ids("op", cols.n_ops)
    index = {o: i for i, o in enumerate(ids)}
    jt = ledger.operator_tensor() if isinstance(ledger, EnergyLedger) else None
    if jt is None or jt.numel() != len(ids) or list(ledger.per_operator) != list(ids):
        per = ledger.per_operator
        jt = torch.tensor([float(per[o]) for o in ids], dtype=torch.float64)
    return index, jt.to(dev), cols.device("op_start"), cols.device("op_end")


def _csr(pairs, attr, index):
    off = np.zeros(len(pairs) + 1, dtype=np.int64)
    mem = []
    for p, pair in enumerate(pairs):
        nodes = getattr(pair, attr)
        mem.extend(index[o] for o in nodes)  # KeyError for unknown ops, as the reference
        off[p + 1] = len(mem)
    return off, np.asarray(mem, dtype=np.int32)


def tuple_rank(tuples) -> np.ndarray:
    """Rank under Python tuple ordering (equal tuples share a rank)."""
    order = sorted(range(len(tuples)), key=lambda i: tuples[i])
    tie = np.empty(len(tuples), dtype=np.int64)
    r, prev = -1, object()
    for i in order:
        if tuples[i] != prev:
            r += 1
            prev = tuples[i]
        tie[i] = r
    return tie


def detect_waste(pairs: Sequence, ledger_a: EnergyLedger, ledger_b: EnergyLedger,
                 threshold: float = DEFAULT_THRESHOLD, *, trace_a, trace_b,
                 output_diff: Optional[Sequence[float]] = None,
                 classify=None) -> list[WasteFinding]:
    """One finding per subgraph pair; the higher-energy side is the suspect
    (detect.py:72-130)."""
    _check_args(ledger_a, ledger_b, threshold)
    pairs = list(pairs)
    P = len(pairs)
    if P == 0:
        return []
    dev = _native.device()
    idx_a, ja, sa, ea = _op_columns(trace_a, ledger_a, dev)
    idx_b, jb, sb, eb = _op_columns(trace_b, ledger_b, dev)
    off_a, mem_a = _csr(pairs, "nodes_a", idx_a)
    off_b, mem_b = _csr(pairs, "nodes_b", idx_b)
    if output_diff is None:
        output_diff = [boundary_rel_diff(getattr(p, "boundary_right", ()), trace_a, trace_b)
                       for p in pairs]
    od = torch.tensor(np.asarray(output_diff, dtype=np.float64), device=dev)
    tie = torch.from_numpy(tuple_rank([tuple(p.nodes_a) for p in pairs])).to(dev)
    t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    d_off_a, d_mem_a, d_off_b, d_mem_b = t(off_a), t(mem_a), t(off_b), t(mem_b)
    fc = FindingColumns(P, dev)
    fs = fc.c_struct()
    p = _native.ptr
    rc = _native.lib().dw_detect_pairs(P, p(d_off_a), p(d_mem_a), p(d_off_b), p(d_mem_b), p(ja),
                                       p(jb), p(sa), p(ea), p(sb), p(eb), p(od), p(tie),
                                       float(threshold), ctypes.byref(fs), _native.stream_handle())
    _native.check(rc, "dw_detect_pairs")
    h = fc.host()
    findings = []
    for i, pair in enumerate(pairs):
        f = WasteFinding(
            pair=pair, energy_a=float(h["energy_a"][i]), energy_b=float(h["energy_b"][i]),
            energy_ratio=float(h["ratio"][i]), latency_a=int(h["latency_a"][i]),
            latency_b=int(h["latency_b"][i]), output_rel_diff=float(output_diff[i]),
            verdict=VERDICTS[h["verdict"][i]], category="unknown",
            wasteful_side=SIDES[h["side"][i]], wasted_joules=float(h["wasted"][i]),
            informational=bool(h["informational"][i]))
        if callable(classify) and f.verdict == VERDICT_WASTE:
            f = WasteFinding(**{**f.__dict__, "category": classify(f, trace_a, trace_b)})
        findings.append(f)
    if classify is None:
        from .diagnose import classify_findings
        cats = classify_findings(findings, trace_a, trace_b)
        findings = [f if c == f.category else WasteFinding(**{**f.__dict__, "category": c})
                    for f, c in zip(findings, cats)]
    return findings


def classify(finding: WasteFinding, trace_a, trace_b) -> str:
    """Category of one waste finding (detect.py:137-172); the batched rule is
    `diagnose.classify_findings`."""
    from .diagnose import classify as _classify
    return _classify(finding, trace_a, trace_b)


# ----------------------------------------------------------------- report


@dataclass(frozen=True)
class Report:
    findings: tuple
    total_a: float
    total_b: float
    wasted_joules: float
    end_to_end_waste_pct: float
    method: str
    threshold: float

    def waste_findings(self) -> tuple:
        return tuple(f for f in self.findings if f.verdict == VERDICT_WASTE)

    def to_dict(self) -> dict:
        return {
            "schema_version": 1,
            "method": self.method,
            "threshold": self.threshold,
            "total_joules_a": self.total_a,
            "total_joules_b": self.total_b,
            "wasted_joules": self.wasted_joules,
            "end_to_end_waste_pct": self.end_to_end_waste_pct,
            "findings": [
                {
                    "nodes_a": list(f.pair.nodes_a),
                    "nodes_b": list(f.pair.nodes_b),
                    "energy_a": f.energy_a,
                    "energy_b": f.energy_b,
                    "energy_ratio": f.energy_ratio,
                    "latency_a": f.latency_a,
                    "latency_b": f.latency_b,
                    "output_rel_diff": f.output_rel_diff,
                    "verdict": f.verdict,
                    "category": f.category,
                    "wasteful_side": f.wasteful_side,
                    "wasted_joules": f.wasted_joules,
                    "informational": f.informational,
                }
                for f in self.findings
            ],
        }

    def tsv_lines(self) -> list[str]:
        lines = ["rank\tverdict\tcategory\tside\twasted_joules\tenergy_a\tenergy_b"
                 "\tratio\tlatency_a_us\tlatency_b_us\toutput_rel_diff\tnodes_a\tnodes_b"]
        for i, f in enumerate(self.findings, start=1):
            lines.append(
                f"{i}\t{f.verdict}\t{f.category}\t{f.wasteful_side}"
                f"\t{f.wasted_joules:.6f}\t{f.energy_a:.6f}\t{f.energy_b:.6f}"
                f"\t{f.energy_ratio:.4f}\t{f.latency_a}\t{f.latency_b}"
                f"\t{f.output_rel_diff:.6f}"
                f"\t{'+'.join(f.pair.nodes_a) or '-'}\t{'+'.join(f.pair.nodes_b) or '-'}")
        return lines

    def summary_text(self) -> str:
        lines = [
            f"differential energy report (method={self.method}, threshold={self.threshold:.2f})",
            f"  total energy: A={self.total_a:.3f} J  B={self.total_b:.3f} J",
            f"  wasted: {self.wasted_joules:.3f} J "
            f"({100.0 * self.end_to_end_waste_pct:.2f}% of the inefficient side)",
        ]
        wastes = self.waste_findings()
        if not wastes:
            lines.append("  no software energy waste detected")
        for f in wastes:
            lines.append(
                f"  [{f.category}] side {f.wasteful_side} wastes {f.wasted_joules:.3f} J "
                f"(x{f.energy_ratio:.2f}) in {'+'.join(f.pair.nodes_a) or '-'} vs "
                f"{'+'.join(f.pair.nodes_b) or '-'}")
        return "\n".join(lines)


def _host_keys(findings) -> tuple[np.ndarray, np.ndarray]:
    """The device ranking key of reference-style findings (same encoding as
    csrc/diff.cu key_hi / key_lo)."""
    P = len(findings)
    wasted = np.array([f.wasted_joules for f in findings], dtype=np.float64)
    bits = wasted.view(np.uint64) & np.uint64(0x7FFFFFFFFFFFFFFF)
    waste = np.array([f.verdict == VERDICT_WASTE for f in findings], dtype=np.uint64)
    hi = bits | (waste << np.uint64(63))
    tie = tuple_rank([tuple(f.pair.nodes_a) for f in findings]).astype(np.uint64)
    lo = ~(((tie + np.uint64(1)) << np.uint64(32)) | (np.arange(P, dtype=np.uint64) & np.uint64(0xFFFFFFFF)))
    return hi.view(np.int64), lo.view(np.int64)


def rank_order(key_hi: torch.Tensor, key_lo: Optional[torch.Tensor], k: int, tie_rank=None,
               n_a: int = 0, summary: Optional[torch.Tensor] = None):
    """Indices of the k best findings (report order) and the device summary
    {n_waste, wasted_joules (exact sum), P} -- dw_rank.  Without key_lo the low
    key follows the join numbering (tie_rank / n_a).  ``summary``: a zeroed
    f64 [4] device tensor to write it into (else one is allocated)."""
    dev = _native.device()
    P = int(key_hi.numel())
    L = _native.lib()
    nbytes = L.dw_rank_workspace_size(P, k)
    ws = _native.Workspace.get(nbytes)
    order = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
    if summary is None:
        summary = torch.zeros(4, dtype=torch.float64, device=dev)
    fs = _native.Findings(None, None, None, None, None, None, None, None, None,
                          _native.ptr(key_hi), _native.ptr(key_lo), _native.ptr(tie_rank), int(n_a))
    rc = L.dw_rank(P, ctypes.byref(fs), int(k), _native.ptr(order), _native.ptr(summary),
                   ws.data_ptr(), ws.numel(), _native.stream_handle())
    _native.check(rc, "dw_rank")
    return order[:k], summary


def rank_order_segmented(segments: Sequence, k: int):
    """Report order of many finding sets in one call (dw_rank_segmented, the
    segmented top-k of a corpus: one segment per trace pair).  ``segments``:
    (key_hi, key_lo or None, tie_rank or None, n_a) per segment, as
    ``rank_order`` takes them.  Returns (order [S, k] int64 with -1 past a
    segment's P, summary [S, 4] {n_waste, wasted_joules, P, 0}), both device
    tensors; segment i equals ``rank_order`` of segment i alone."""
    dev = _native.device()
    segs = list(segments)
    S = len(segs)
    arr = (_native.RankSegment * max(S, 1))()
    keep = []
    for i, (hi, lo, tie, n_a) in enumerate(segs):
        arr[i] = _native.RankSegment(_native.ptr(hi), _native.ptr(lo), _native.ptr(tie), int(n_a),
                                     int(hi.numel()))
        keep += [hi, lo, tie]
    L = _native.lib()
    ws = _native.Workspace.get(L.dw_rank_segmented_workspace_size(S, k))
    order = torch.full((max(S, 1), max(k, 1)), -1, dtype=torch.int64, device=dev)
    summary = torch.zeros((max(S, 1), 4), dtype=torch.float64, device=dev)
    rc = L.dw_rank_segmented(arr, S, int(k), _native.ptr(order), _native.ptr(summary), ws.data_ptr(),
                             ws.numel(), _native.stream_handle())
    _native.check(rc, "dw_rank_segmented")
    return order[:S, :k], summary[:S]


def report(findings: Sequence[WasteFinding], ledger_a: EnergyLedger, ledger_b: EnergyLedger,
           threshold: float = DEFAULT_THRESHOLD) -> Report:
    """Machine-readable report plus human summary, ranked by wasted joules
    (detect.py:256-278).  The order is computed on the device."""
    findings = list(findings)
    if findings:
        dev = _native.device()
        hi, lo = _host_keys(findings)
        order, _ = rank_order(torch.from_numpy(hi).to(dev), torch.from_numpy(lo).to(dev),
                              len(findings))
        ranked = [findings[i] for i in order.cpu().tolist()]
    else:
        ranked = []
    # CPython sum() over the ranked waste findings, as the reference adds them
    wasted = sum(f.wasted_joules for f in ranked if f.verdict == VERDICT_WASTE)
    ineff = max(ledger_a.total_joules, ledger_b.total_joules)
    pct = wasted / ineff if ineff > 0 else 0.0
    return Report(findings=tuple(ranked), total_a=ledger_a.total_joules,
                  total_b=ledger_b.total_joules, wasted_joules=wasted,
                  end_to_end_waste_pct=pct, method=ledger_a.method, threshold=threshold)
