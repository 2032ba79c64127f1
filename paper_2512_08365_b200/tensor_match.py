"""Cross-trace tensor matching -- drop-in for ``subgraph_match.match_tensors``
(subgraph_match.py:109-204), the tensor-equivalence prefilter + batched SVD of
SURVEY.md 8(f)4.

The reference walks every (A tensor, B tensor) pair in Python: element counts
and Frobenius norms over every run as a prefilter, then for each survivor the
multi-mode SVD invariant sets (one numpy Jacobi per unfolding), then an
injective pairing by closest topological rank.  At config 1 this stage takes
~125 s.  Here the per-element and per-pair work runs on the device
(csrc/tensor.cu):

  * every snapshot's norm (``dw_tensor_norms``, CPython's sum of squares --
    bit-identical, so the prefilter keeps exactly the reference's pairs);
  * the all-pairs prefilter (``dw_tensor_prefilter``, candidates in
    np.nonzero order);
  * one batched Jacobi launch for every unfolding of every (tensor, run) a
    candidate touches (``dw_unfold_spectra``).

The host keeps the parts that are a handful of numbers per candidate: the
bottleneck embedding, the run loop with its early exit (so ``full_checks``
counts as the reference does), the rank ordering and the greedy injective
pairing.  Graphs may be the reference's CompGraph objects or plain traces (the
producer map and topological ranks are then derived as graph.build_graph and
_topo_ranks do, graph.py:65-106, subgraph_match.py:88-106).
"""

from __future__ import annotations

import heapq
import math
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native
from .tensor_equiv import (DEFAULT_EPSILON, EMBED_MAX, ORDER_CAP, SpectraBatch, embed_injectively)

NORM_FLOOR = 1e-30

SOURCE, SINK = "__source__", "__sink__"  # graph.py:16-17


@dataclass(frozen=True)
class TensorPair:
    tensor_a: str
    tensor_b: str
    score: float
    confirmed_runs: tuple


@dataclass(frozen=True)
class TensorPairSet:
    """Injective pairing of equivalent tensors (subgraph_match.py:37-55)."""

    pairs: tuple

    def partner_of_a(self, tensor_id: str) -> Optional[str]:
        for p in self.pairs:
            if p.tensor_a == tensor_id:
                return p.tensor_b
        return None

    def by_a(self) -> dict:
        return {p.tensor_a: p.tensor_b for p in self.pairs}

    def by_b(self) -> dict:
        return {p.tensor_b: p.tensor_a for p in self.pairs}

    def __len__(self) -> int:
        return len(self.pairs)


@dataclass(frozen=True)
class MatchStats:
    candidate_pairs: int
    full_checks: int
    wall_time_s: float


# ------------------------------------------------------------------ graphs


class _GraphView:
    """What match_tensors needs of a graph: the trace, its tensor ids, each
    tensor's producer and every node's topological rank."""

    def __init__(self, g):
        if hasattr(g, "edges") and hasattr(g, "trace"):  # a reference CompGraph
            self.trace = g.trace
            self.ids = sorted(g.edges)
            self.producer = {t: g.edges[t].producer for t in self.ids}
            self.rank = _topo_ranks(list(g.nodes), g.successors)
            return
        tr = g
        self.trace = tr
        produced, consumed = {}, {}
        for op in tr.operators:
            for t in op.output_tensor_ids:
                produced[t] = op.op_id
            for t in op.input_tensor_ids:
                consumed.setdefault(t, []).append(op.op_id)
        self.ids = sorted(tr.tensors)
        self.producer = {t: produced.get(t, SOURCE) for t in self.ids}
        outs = {SOURCE: sorted(t for t in tr.tensors if t not in produced), SINK: []}
        for op in tr.operators:
            outs[op.op_id] = sorted(op.output_tensor_ids)
        cons = {t: tuple(consumed.get(t, [SINK])) for t in tr.tensors}

        def successors(n):
            seen, out = set(), []
            for t in outs.get(n, ()):
                for c in cons[t]:
                    if c not in seen:
                        seen.add(c)
                        out.append(c)
            return out

        nodes = [SOURCE] + [op.op_id for op in tr.operators] + [SINK]
        self.rank = _topo_ranks(nodes, successors)


def _topo_ranks(nodes, successors) -> dict:
    """Kahn's order, always taking the smallest ready node name
    (subgraph_match.py:88-106 keeps its ready list sorted: a min-heap)."""
    indeg = {n: 0 for n in nodes}
    for n in nodes:
        for m in successors(n):
            indeg[m] += 1
    ready = [n for n, d in indeg.items() if d == 0]
    heapq.heapify(ready)
    rank = {}
    while ready:
        n = heapq.heappop(ready)
        rank[n] = len(rank)
        for m in successors(n):
            indeg[m] -= 1
            if indeg[m] == 0:
                heapq.heappush(ready, m)
    return rank


# ------------------------------------------------------------------ device


def _pack(trace, ids, runs):
    """Flat values of every (run, tensor) snapshot, run-major; offsets; shapes."""
    snaps = [trace.snapshot(t, r) for r in range(runs) for t in ids]
    counts = np.fromiter((len(s.values) for s in snaps), dtype=np.int64, count=len(snaps))
    off = np.zeros(len(snaps) + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    vals = np.fromiter((v for s in snaps for v in s.values), dtype=np.float64, count=int(off[-1]))
    return snaps, vals, off


def _norms(vals, off, dev):
    n = off.shape[0] - 1
    d_vals = torch.from_numpy(vals).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    _native.check(_native.lib().dw_tensor_norms(_native.ptr(d_vals), _native.ptr(d_off), n, _native.ptr(out),
                                                _native.stream_handle()), "dw_tensor_norms")
    return out[:n]


def _prefilter(count_a, count_b, norm_a, norm_b, runs, eps, dev):
    na, nb = count_a.shape[0], count_b.shape[0]
    L, p, st = _native.lib(), _native.ptr, _native.stream_handle()
    ca, cb = torch.from_numpy(count_a).to(dev), torch.from_numpy(count_b).to(dev)
    rc = torch.empty(max(na, 1), dtype=torch.int64, device=dev)
    _native.check(L.dw_tensor_prefilter(0, na, nb, runs, p(ca), p(cb), p(norm_a), p(norm_b), float(eps), p(rc),
                                        None, None, None, st), "dw_tensor_prefilter")
    rc = rc[:na]
    total = int(rc.sum().item()) if na else 0
    ro = torch.cumsum(rc, 0) - rc
    pa = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    pb = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    if total:
        _native.check(L.dw_tensor_prefilter(1, na, nb, runs, p(ca), p(cb), p(norm_a), p(norm_b), float(eps), None,
                                            p(ro), p(pa), p(pb), st), "dw_tensor_prefilter")
    return pa[:total].cpu().numpy(), pb[:total].cpu().numpy()


def _slices(vals, off, idx):
    """Concatenated vals[off[i]:off[i+1]] for i in idx."""
    if idx.size == 0:
        return np.zeros(0)
    lens = off[idx + 1] - off[idx]
    starts = np.repeat(off[idx] - (np.cumsum(lens) - lens), lens)
    return vals[starts + np.arange(int(lens.sum()))]


def _small_large(batch, sa: int, sb: int):
    x, y = batch.spectra(sa), batch.spectra(sb)
    return (x, y) if len(x) <= len(y) else (y, x)


# ------------------------------------------------------------------ match


def match_tensors(gA, gB, epsilon: float = DEFAULT_EPSILON):
    """Equivalent-tensor pairing across two graphs (or traces); returns
    (TensorPairSet, MatchStats) like subgraph_match.match_tensors."""
    t0 = time.perf_counter()
    A, B = _GraphView(gA), _GraphView(gB)
    ta, tb = A.trace, B.trace
    runs = max(min(ta.run_count, tb.run_count), 1)
    dev = _native.device()
    snaps_a, vals_a, off_a = _pack(ta, A.ids, runs)
    snaps_b, vals_b, off_b = _pack(tb, B.ids, runs)
    na, nb = len(A.ids), len(B.ids)
    count_a = np.diff(off_a)[:na] if na else np.zeros(0, np.int64)
    count_b = np.diff(off_b)[:nb] if nb else np.zeros(0, np.int64)
    norm_a = _norms(vals_a, off_a, dev)
    norm_b = _norms(vals_b, off_b, dev)
    cand_a, cand_b = _prefilter(np.ascontiguousarray(count_a), np.ascontiguousarray(count_b), norm_a, norm_b,
                                runs, epsilon, dev)
    nrm_a, nrm_b = norm_a.cpu().numpy(), norm_b.cpu().numpy()

    # spectra of every (run, tensor) snapshot a candidate touches: ONE batched
    # Jacobi launch for both sides; then every (candidate, run) embedding in
    # one device launch (sets of <= 14 spectra; larger ones on the host)
    keys_a = sorted({(r, int(a)) for a in set(cand_a.tolist()) for r in range(runs)})
    keys_b = sorted({(r, int(b)) for b in set(cand_b.tolist()) for r in range(runs)})
    sel = [snaps_a[r * na + i] for r, i in keys_a] + [snaps_b[r * nb + i] for r, i in keys_b]
    pos_a = {k: j for j, k in enumerate(keys_a)}
    pos_b = {k: len(keys_a) + j for j, k in enumerate(keys_b)}
    shapes = [tuple(x.shape) if 1 < len(x.shape) <= ORDER_CAP else () for x in sel]
    base = np.concatenate([[0], np.cumsum([len(x.values) for x in sel])]).astype(np.int64)
    ka = np.array([r * na + i for r, i in keys_a], dtype=np.int64)
    kb = np.array([r * nb + i for r, i in keys_b], dtype=np.int64)
    vals = np.concatenate([_slices(vals_a, off_a, ka), _slices(vals_b, off_b, kb)])
    batch = SpectraBatch(vals, shapes, base[:-1])

    C, R = cand_a.shape[0], runs
    ja = np.empty((C, R), dtype=np.int64)
    jb = np.empty((C, R), dtype=np.int64)
    for r in range(R):
        ja[:, r] = [pos_a[(r, int(a))] for a in cand_a]
        jb[:, r] = [pos_b[(r, int(b))] for b in cand_b]
    order_a = np.array([len(x.shape) for x in sel], dtype=np.int64)
    nrm = np.concatenate([nrm_a[ka], nrm_b[kb]]) if sel else np.zeros(0)
    cnt = np.array([len(x.values) for x in sel], dtype=np.int64)
    # per (candidate, run): the norm gate and order-1 rule (tensor_equiv.py:271-283)
    xa, xb = nrm[ja], nrm[jb]
    nd = np.abs(xa - xb) / np.maximum(np.minimum(xa, xb), NORM_FLOOR)
    oa, ob = order_a[ja], order_a[jb]
    score = np.full((C, R), math.inf)
    size_ok = cnt[ja] == cnt[jb]
    gate = size_ok & ~(nd > epsilon)
    o1 = gate & ((oa == 1) | (ob == 1))
    score[o1] = nd[o1]
    # the reference builds both invariant sets before comparing: an order
    # above the cap raises whenever that (candidate, run) is reached
    big = (oa > ORDER_CAP) | (ob > ORDER_CAP)
    multi = gate & ~o1 & ~big
    dev_jobs = multi & (np.maximum(batch.set_count[ja], batch.set_count[jb]) <= EMBED_MAX)
    if dev_jobs.any():
        score[dev_jobs] = batch.embed(ja[dev_jobs], jb[dev_jobs], epsilon)

    full_checks = 0
    candidates = []
    for c in range(C):
        worst, ok = 0.0, True
        for r in range(R):
            full_checks += 1
            if big[c, r]:
                o = int(max(oa[c, r], ob[c, r]))
                raise ValueError(f"tensor order {o} exceeds the cap of {ORDER_CAP}")
            if multi[c, r] and not dev_jobs[c, r]:  # > 14 spectra per set: host embedding
                got = embed_injectively(*_small_large(batch, int(ja[c, r]), int(jb[c, r])), epsilon)
                score[c, r] = math.inf if got is None else got
            s = score[c, r]
            eq = bool(gate[c, r]) and s != math.inf if not o1[c, r] else bool(s <= epsilon)
            if not eq:
                ok = False
                break
            worst = max(worst, float(s))
        if ok:
            candidates.append((A.ids[int(cand_a[c])], B.ids[int(cand_b[c])], worst))

    ordered = sorted(candidates, key=lambda c: (abs(A.rank[A.producer[c[0]]] - B.rank[B.producer[c[1]]]),
                                                c[0], c[1]))
    used_a, used_b, pairs = set(), set(), []
    for x, y, score in ordered:
        if x in used_a or y in used_b:
            continue
        used_a.add(x)
        used_b.add(y)
        pairs.append(TensorPair(tensor_a=x, tensor_b=y, score=score, confirmed_runs=tuple(range(runs))))
    pairs.sort(key=lambda p: (p.tensor_a, p.tensor_b))
    stats = MatchStats(candidate_pairs=int(cand_a.shape[0]), full_checks=full_checks,
                       wall_time_s=time.perf_counter() - t0)
    return TensorPairSet(pairs=tuple(pairs)), stats


def prefilter_count(trace_a, trace_b, epsilon: float = DEFAULT_EPSILON) -> int:
    """Number of prefilter survivors (MatchStats.candidate_pairs) only."""
    A, B = _GraphView(trace_a), _GraphView(trace_b)
    runs = max(min(A.trace.run_count, B.trace.run_count), 1)
    dev = _native.device()
    _, va, oa = _pack(A.trace, A.ids, runs)
    _, vb, ob = _pack(B.trace, B.ids, runs)
    ca, cb = np.diff(oa)[:len(A.ids)], np.diff(ob)[:len(B.ids)]
    pa, _ = _prefilter(np.ascontiguousarray(ca), np.ascontiguousarray(cb), _norms(va, oa, dev), _norms(vb, ob, dev),
                       runs, epsilon, dev)
    return int(pa.shape[0])

