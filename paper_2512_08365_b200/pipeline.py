"""End-to-end differential analysis of one trace pair at scale -- the scale
counterpart of the reference's run_pipeline (cli.py:66-109) restricted to the
hot path: attribution of both traces, signature-join diff, ranked findings.

Inputs may live on the host (pinned buffers are copied to HBM asynchronously,
trace B's copy overlapping trace A's attribution) or already in HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native
from .columns import TraceColumns
from .detect import DEFAULT_THRESHOLD, FindingColumns, Report, WasteFinding, rank_order_segmented
from .energy import EnergyLedger, _begin_ledger, build_ledger

import numpy as np
from .join import JoinDiff, join_diff, join_prepare


@dataclass
class Analysis:
    ledger_a: EnergyLedger
    ledger_b: EnergyLedger
    report: Report          # top-k findings; totals and wasted cover everything
    join: JoinDiff


_DECODE_STREAMS: dict = {}


def _decode_stream() -> "torch.cuda.Stream":
    dev = torch.cuda.current_device()
    if dev not in _DECODE_STREAMS:
        _DECODE_STREAMS[dev] = torch.cuda.Stream()
    return _DECODE_STREAMS[dev]


def _ledger_errors_first(*pending) -> None:
    """A ledger's data error outranks a pairing error, as when each ledger
    was built (and checked) before the pairing started: raise it if any."""
    for f in pending:
        if f is not None:
            f()


def analyze(trace_a, trace_b, method: str = "samples", threshold: float = DEFAULT_THRESHOLD,
            k: int = 100, *, lean: bool = True, copy_stream: "torch.cuda.Stream | None" = None,
            summation: str = "exact", overlap: str = "compat") -> Analysis:
    """Ledgers for both traces, the signature-join diff and the top-k report.

    ``overlap`` ("compat" or "split"): energy.build_ledger's overlap mode.

    ``summation`` (default "exact"): how the ledgers sum each interval's
    pieces (energy.build_ledger) -- the exact fixed-point sum, the scale
    path's definition; "reference" for the reference's sequential order.

    ``lean`` (default): the join writes each finding's differential columns
    -- energy delta, time delta, energy-per-useful-work ratio (north star
    (3)) -- and its ranking key (the top-k rows' ratio / verdict / side /
    informational / wasted are derived on the host, equal to the device's);
    ``lean=False`` keeps every finding column on the device
    (``Analysis.join.columns``) plus per-side energy-per-work.

    (Running the join's pairing on a second stream beside the ledgers, with
    the tile kernel capped to fewer SMs via dw_set_attribute_sms, was measured
    slower on C4 -- 35.4 vs 34.5 ms at 12 reserved SMs, worse with more -- so
    the phases run back to back.)

    With ``copy_stream`` (host-resident inputs): A's ledger columns copy
    first (A's attribution starts as they land), then B's ledger columns on
    ``copy_stream`` (decoded on a side stream column by column as each lands,
    so B's attribution starts at B's last ledger byte), and the two signature
    columns last: B's ledger runs while the signatures cross PCIe, and only
    the pairing, the findings and the top-k trail the last byte (the pairing
    is the shorter of the two dependent chains -- with B's power columns last,
    B's whole ledger would trail it instead)."""
    ca, cb = TraceColumns.from_trace(trace_a), TraceColumns.from_trace(trace_b)
    prep = None
    sig_ready = ()
    if copy_stream is not None:
        led_cols = tuple(n for n in TraceColumns.HOT if n != "op_sig")
        a_ready = ca.prefetch(torch.cuda.current_stream(), names=led_cols)
        # B's copies queue behind A's transfers (not its decodes): concurrent
        # copies would share PCIe and delay A to the end of the transfer
        copy_stream.wait_event(getattr(ca, "copied", None) or a_ready)
        # (decoded on a side stream: a decode queued on the copy stream would
        # hold the next transfers behind A's attribution for the SMs)
        b_ready = cb.prefetch(copy_stream, names=led_cols, decode_stream=_decode_stream())
        sig_ready = (ca.prefetch(copy_stream, names=("op_sig",), decode_stream=_decode_stream()),
                     cb.prefetch(copy_stream, names=("op_sig",), decode_stream=_decode_stream()))
        # each ledger waits for its own columns only, not for the signatures
        ca._dev["__ready__"], cb._dev["__ready__"] = a_ready, b_ready
    # both ledgers and the pairing queue before the host waits on any of
    # them (build_ledger's status read deferred; errors raised A first)
    fa = _begin_ledger(ca, method=method, summation=summation, overlap=overlap)
    fb = None
    try:
        fb = _begin_ledger(cb, method=method, summation=summation, overlap=overlap)
        for ev in sig_ready:
            torch.cuda.current_stream().wait_event(ev)
        prep = join_prepare(ca, cb)
    except Exception:
        _ledger_errors_first(fa, fb)
        raise
    la, lb = fa(), fb()
    jd = join_diff(ca, cb, la, lb, threshold, k, full_columns=not lean, epw=not lean, prep=prep,
                   columns=FindingColumns.DELTAS if lean else None)
    top = jd.top_findings(ca, cb)
    ineff = max(la.total_joules, lb.total_joules)
    pct = jd.wasted_joules / ineff if ineff > 0 else 0.0
    rep = Report(findings=tuple(top), total_a=la.total_joules, total_b=lb.total_joules,
                 wasted_joules=jd.wasted_joules, end_to_end_waste_pct=pct, method=method,
                 threshold=threshold)
    return Analysis(la, lb, rep, jd)


@dataclass
class PairSummary:
    """One pair of a corpus after ``analyze_corpus``: its ledgers' totals, the
    join (device columns; ``order`` = this pair's top-k in report order) and
    its waste totals over every finding."""

    total_a: float
    total_b: float
    join: JoinDiff
    n_waste: int
    wasted_joules: float


@dataclass
class CorpusAnalysis:
    pairs: list                       # PairSummary per pair, corpus order
    order: torch.Tensor               # [S, k] per-pair top-k finding indices (-1 padded)
    top: list                         # corpus top-k: (pair index, finding index), report order

    def findings(self, columns, classify: bool = True) -> list:
        """The corpus top-k as (pair index, WasteFinding); ``columns`` =
        [(cols_a, cols_b)] per pair."""
        out = []
        by_pair: dict = {}
        for r, (i, f) in enumerate(self.top):
            by_pair.setdefault(i, []).append((r, f))
        rows: dict = {}
        for i, items in by_pair.items():
            jd = self.pairs[i].join
            idx = torch.tensor([f for _, f in items], dtype=torch.int64, device=jd.columns.key_hi.device)
            ca, cb = columns[i]
            for (r, _), wf in zip(items, jd.top_findings(ca, cb, classify=classify, idx=idx)):
                rows[r] = (i, wf)
        for r in range(len(self.top)):
            out.append(rows[r])
        return out


_CORPUS_STREAMS: dict = {}


def _corpus_stream() -> "torch.cuda.Stream":
    dev = torch.cuda.current_device()
    if dev not in _CORPUS_STREAMS:
        _CORPUS_STREAMS[dev] = torch.cuda.Stream()
    return _CORPUS_STREAMS[dev]


def analyze_corpus(pairs, method: str = "samples", threshold: float = DEFAULT_THRESHOLD, k: int = 100, *,
                   summation: str = "exact") -> CorpusAnalysis:
    """A corpus of trace pairs: per pair, both ledgers and
    the signature-join diff (differential columns + ranking key, as
    ``analyze``); then ONE segmented top-k launch sequence ranks every pair's
    findings (``dw_rank_segmented``: per-pair report order and exact waste
    sums), and the corpus top-k is the merge of the per-pair top-k lists on the
    same composite key, ties between pairs going to the earlier pair
    (detect.py:263-266 per pair).  Each pair's ledgers are released after its
    join; only the finding columns stay on the device."""
    summaries, segs = [], []
    pairs = list(pairs)
    main = torch.cuda.current_stream()
    # pairs alternate between two streams, and pair i+1's ledgers are queued
    # before the host blocks on pair i's join: the device works on one pair
    # while the host waits on (and sets up) the other -- each pair's own work
    # stays in order on its stream, and every result equals the serial loop's
    streams = [main, _corpus_stream()] if len(pairs) > 1 else [main]
    for st in streams[1:]:
        st.wait_stream(main)  # inputs made on the caller's stream

    def begin(i):
        with torch.cuda.stream(streams[i % len(streams)]):
            ca, cb = TraceColumns.from_trace(pairs[i][0]), TraceColumns.from_trace(pairs[i][1])
            fa = _begin_ledger(ca, method=method, summation=summation)
            fb = _begin_ledger(cb, method=method, summation=summation)
        return [ca, cb, fa, fb, None]

    def prepare(i, cur):
        with torch.cuda.stream(streams[i % len(streams)]):
            try:
                cur[4] = join_prepare(cur[0], cur[1])
            except Exception:
                _ledger_errors_first(cur[2], cur[3])
                raise

    def finish(i, cur):
        ca, cb, fa, fb, prep = cur
        with torch.cuda.stream(streams[i % len(streams)]):
            la, lb = fa(), fb()
            jd = join_diff(ca, cb, la, lb, threshold, k, full_columns=False, epw=False,
                           columns=FindingColumns.DELTAS, ranked=False, prep=prep)
        summaries.append(PairSummary(la.total_joules, lb.total_joules, jd, 0, 0.0))
        segs.append((jd.columns.key_hi[:jd.P], None, jd.columns.tie_rank, jd.n_a))

    if pairs:
        cur = begin(0)
        prepare(0, cur)
        for i in range(len(pairs)):
            nxt = None
            if i + 1 < len(pairs):
                try:
                    nxt = begin(i + 1)
                except Exception:
                    finish(i, cur)  # pair i's errors first, as a serial loop raises them
                    raise
            finish(i, cur)
            if nxt is not None:
                prepare(i + 1, nxt)
            cur = nxt
    for st in streams[1:]:
        main.wait_stream(st)
    order, summary = rank_order_segmented(segs, k)
    sm = summary.cpu().numpy()
    for i, ps in enumerate(summaries):
        ps.n_waste, ps.wasted_joules = int(sm[i, 0]), float(sm[i, 1])
        ps.join.n_waste, ps.join.wasted_joules = ps.n_waste, ps.wasted_joules
        n = min(k, ps.join.P)
        ps.join.order = order[i, :n]
    # corpus merge: every pair's top-k keys, ordered by (hi, lo) descending, pair ascending
    keys = []
    for i, ps in enumerate(summaries):
        o = ps.join.order
        if o.numel() == 0:
            continue
        jd = ps.join
        hi = jd.columns.key_hi[o]
        tie = jd.pair_of(o)[0]
        if jd.columns.tie_rank is not None:
            tie = torch.where(tie >= 0, jd.columns.tie_rank[tie.clamp(min=0)], tie)
        lo = ~(((tie + 1) << 32) | o)
        keys.append(torch.stack([hi, lo, torch.full_like(o, i), o]))
    top = []
    if keys:
        kk = torch.cat(keys, dim=1).cpu().numpy()
        hi_u = kk[0].view(np.uint64)
        lo_u = kk[1].view(np.uint64)
        # primary key last: hi desc, nodes_a tie asc (lo's upper half, stored
        # complemented), then corpus order (pair, finding) -- a stable sort of
        # the concatenated findings, as report() on the whole corpus would give
        sel = np.lexsort((kk[3], kk[2], ~(lo_u >> np.uint64(32)), ~hi_u))
        top = [(int(kk[2][j]), int(kk[3][j])) for j in sel[:k]]
    return CorpusAnalysis(summaries, order, top)
