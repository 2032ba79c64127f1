"""Time-window sharding of one trace across ranks.

One process per GPU; rank g owns a contiguous, tile-aligned range of power
samples and every interval (operator or kernel) whose start falls in it.

    samples   [s_g, s_g+1) owned; the rank holds [s_g - DW_TILE, s_g+1 + H)
              (H = DW_DIRECT_MAX + 4): one whole tile before (so the local
              tile grid is the global one) and the halo after that any
              interval of <= DW_DIRECT_MAX pieces starting in the window needs
    pieces    [s_g, s_g+1) owned (the last rank: to the end of the signal)
    intervals owned by the window holding their start; computed whole when
              they end within the halo (bit-identical to one GPU: the same
              sequential sum, or the same fixed-point decomposition on the
              same tile sums); otherwise "crossing" -- necessarily longer than
              DW_DIRECT_MAX pieces -- and every rank adds the exact int128
              share of the pieces it owns (K7, csrc/attribute.cu
              window_partials_kernel).  The shares are all-gathered and summed
              exactly, then rounded once: the one-GPU value bit for bit.
    totals    ledger total = exact sum of every rank's owned whole-tile sums;
              operator_total = exact sum of every rank's 2^-64 J share.

The exchanges are small tensor all-gathers (crossing intervals are at most
the concurrency at each window edge) through ``Comm`` -- torch.distributed
(NCCL on GPU, gloo on CPU) -- or an in-process loopback that runs the ranks
one after the other (single-GPU parity tests).  The signature join of a
sharded pair partitions operators by signature hash: one fused peer-memory
scatter into persistent receive buffers (``Comm.exchange``) or one NCCL
all-to-all (``sharded_join``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import _native
from .energy import SignalError, _raise_interval_error

TILE = 1024
HALO = _native.DW_DIRECT_MAX + 4
US_PER_S = 1_000_000


# ------------------------------------------------------------------ plan


@dataclass(frozen=True)
class Window:
    rank: int
    world: int
    s0: int          # owned samples [s0, s1)
    s1: int
    p0: int          # owned pieces [p0, p1)
    p1: int
    l0: int          # held samples [l0, l1)
    l1: int


def plan(n_samples: int, world: int, kind: str) -> list[Window]:
    """Tile-aligned windows of (nearly) equal sample count."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if n_samples < 2 * TILE * world:
        raise ValueError(f"{n_samples} samples are too few to shard over {world} ranks")
    nterms = n_samples if kind == "step" else n_samples - 1
    cuts = [0] + [int(round(g * n_samples / world / TILE)) * TILE for g in range(1, world)] + [n_samples]
    out = []
    for g in range(world):
        s0, s1 = cuts[g], cuts[g + 1]
        p1 = s1 if g < world - 1 else nterms
        out.append(Window(g, world, s0, s1, s0, p1, max(s0 - TILE, 0), min(s1 + HALO, n_samples)))
    return out


# ----------------------------------------------------------------- comm


class Comm:
    """The collectives the sharded path needs, over torch.distributed: tensor
    all-gathers (NCCL moves device tensors over NVLink; gloo, for CPU tests,
    stages them on the host) and the join's record exchange.  With ``p2p``
    (every rank on this node, CUDA tensors) the exchange is one kernel storing
    into the peers' persistent receive buffers (``exchange``)."""

    def __init__(self, group=None, p2p: Optional[bool] = None):
        import os
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if p2p is None:  # CUDA IPC reaches only the ranks of this node
            p2p = (torch.cuda.is_available() and os.environ.get("DWB200_P2P", "1") != "0"
                   and int(os.environ.get("LOCAL_WORLD_SIZE", self.world)) == self.world)
        self.p2p = bool(p2p)
        self._mbox = None
        self._epoch = 0

    # ---- tensor collectives
    def _staged(self, t: torch.Tensor) -> bool:
        return t.device.type == "cuda" and self.dist.get_backend(self.group) == "gloo"

    def all_gather(self, t: torch.Tensor) -> list[torch.Tensor]:
        """Every rank's ``t`` (same shape everywhere), in rank order."""
        x = t.contiguous()
        if self._staged(x):
            return [o.to(t.device) for o in self.all_gather(x.cpu())]
        out = [torch.empty_like(x) for _ in range(self.world)]
        self.dist.all_gather(out, x, group=self.group)
        return out

    def gather_var(self, t: torch.Tensor) -> list[torch.Tensor]:
        """Every rank's ``t`` whose first dimension may differ per rank: the
        lengths first, then one all_gather of the padded rows."""
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        ns = [int(x) for x in torch.cat(self.all_gather(n)).cpu().tolist()]
        m = max(max(ns), 1)
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        return [o[:k] for o, k in zip(self.all_gather(pad), ns)]

    def all_to_all(self, tensors: list[torch.Tensor]) -> list[torch.Tensor]:
        """tensors[r] goes to rank r; returns what every rank sent here.  NCCL
        moves device tensors directly (NVLink); gloo stages them on the host."""
        dev = tensors[0].device
        if self._staged(tensors[0]):
            return [t.to(dev) for t in self.all_to_all([t.cpu() for t in tensors])]
        sizes = torch.tensor([t.numel() for t in tensors], dtype=torch.int64)
        sizes_dev = sizes.to(tensors[0].device)
        recv_sizes = torch.empty_like(sizes_dev)
        self.dist.all_to_all_single(recv_sizes, sizes_dev, group=self.group)
        rs = recv_sizes.cpu().tolist()
        send = torch.cat(tensors)
        recv = torch.empty(sum(rs), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send, output_split_sizes=rs, input_split_sizes=sizes.tolist(),
                                    group=self.group)
        return list(torch.split(recv, rs))

    # ---- the fused record exchange (persistent mailbox over CUDA IPC)
    def _mailbox(self, rows: int, dev) -> "_Mailbox":
        """This rank's receive buffer (rows of up to 6 int64) plus its arrival
        flags, and every peer's, IPC-mapped once.  Re-created (a collective)
        only when some rank needs more rows than the current capacity."""
        if self._mbox is None or self._mbox.rows < rows:
            if self._mbox is not None:
                self._mbox.close()
            self._mbox = _Mailbox(self, max(rows, 1 << 16) if self._mbox is None else 2 * rows, dev)
        return self._mbox

    def exchange(self, o: "ShardOps", with_rank: bool) -> torch.Tensor:
        """The records of ``o`` bound for this rank from every rank (rows of
        idx, sig, start, end, joules bits[, rank]).  Per call: one sizing pass
        and ONE all_gather of the count vectors (a tensor collective), then
        one kernel (dw_exchange_scatter) stores every record straight into its
        receiver's persistent buffer over peer memory, each sender publishes
        the call's epoch into the receivers' arrival flags, and this rank's
        stream waits on the device for every sender's flag -- no IPC handle
        traffic, no host sync after the scatter, no barrier.  (The count
        all_gather of the next call also orders the buffer's reuse: no peer
        can scatter again before this rank's stream has reached it.)"""
        L, p = _native.lib(), _native.ptr
        dev = o.sig.device
        st = _native.stream_handle()
        world, me = self.world, self.rank
        width = 6 if with_rank else 5
        n = int(o.sig.numel())
        counts = torch.empty(world, dtype=torch.int64, device=dev)
        _native.check(L.dw_exchange_count(p(o.sig), n, world, p(counts), st), "dw_exchange_count")
        mat = torch.stack(self.all_gather(counts)).cpu()  # mat[src][dst]
        recv_n = int(mat[:, me].sum())
        mb = self._mailbox(int(mat.sum(dim=0).max()), dev)  # rows of the largest receiver
        base = mat[:me].sum(dim=0).tolist() if me else [0] * world
        cols = [o.idx, o.sig, o.start, o.end, o.joules.view(torch.int64)] + ([o.rank] if with_rank else [])
        cols = [c.contiguous() for c in cols]
        cursor = torch.empty(world, dtype=torch.int64, device=dev)
        col_ptrs = (ctypes.c_void_p * width)(*[p(c) for c in cols])
        recv_ptrs = (ctypes.c_void_p * world)(*mb.recv_ptrs)
        base_arr = (ctypes.c_int64 * world)(*[int(x) for x in base])
        # rows are written with this call's width: the receive view below uses it too
        _native.check(L.dw_exchange_scatter(col_ptrs, width, p(o.sig), n, world, recv_ptrs, base_arr, p(cursor),
                                            st), "dw_exchange_scatter")
        self._epoch += 1
        flag_ptrs = (ctypes.c_void_p * world)(*mb.flag_ptrs)
        _native.check(L.dw_exchange_signal(flag_ptrs, world, me, self._epoch, st), "dw_exchange_signal")
        _native.check(L.dw_exchange_wait(p(mb.flags), world, self._epoch, p(mb.timeout), st), "dw_exchange_wait")
        return mb.recv[: recv_n * width].view(-1, width)

    def close(self) -> None:
        if self._mbox is not None:
            self._mbox.close()
            self._mbox = None


class _Mailbox:
    """One rank's persistent receive buffer + arrival flags (one allocation,
    one IPC handle) and the peers' mapped pointers."""

    def __init__(self, comm: Comm, rows: int, dev):
        L, p = _native.lib(), _native.ptr
        world, me = comm.world, comm.rank
        self.rows = rows
        self.buf = torch.zeros(rows * 6 + world + 2, dtype=torch.int64, device=dev)
        self.recv = self.buf[: rows * 6]
        self.flags = self.buf[rows * 6: rows * 6 + world]
        self.timeout = torch.zeros(1, dtype=torch.int32, device=dev)
        torch.cuda.current_stream(dev).synchronize()  # zeroed before any peer can signal into it
        handle = (ctypes.c_char * 64)()
        off = ctypes.c_int64(0)
        _native.check(L.dw_ipc_handle(p(self.buf), handle, ctypes.byref(off)), "dw_ipc_handle")
        rec = torch.zeros(9, dtype=torch.int64)
        rec[:8] = torch.frombuffer(bytearray(bytes(handle)), dtype=torch.int64)
        rec[8] = int(off.value)
        shared = [t.cpu() for t in comm.all_gather(rec.to(dev))]
        self.opened, self.recv_ptrs, self.flag_ptrs = [], [], []
        for d in range(world):
            if d == me:
                bp = p(self.buf)
            else:
                ptr = ctypes.c_void_p()
                hb = (ctypes.c_char * 64).from_buffer_copy(shared[d][:8].numpy().tobytes())
                _native.check(L.dw_ipc_open(hb, ctypes.byref(ptr)), "dw_ipc_open")
                self.opened.append(ptr)
                bp = ptr.value + int(shared[d][8])
            self.recv_ptrs.append(bp)
            self.flag_ptrs.append(bp + 8 * rows * 6)

    def close(self) -> None:
        L = _native.lib()
        for ptr in self.opened:
            L.dw_ipc_close(ptr)
        self.opened = []


class LocalComm:
    """World of one (the single-rank bench path): every collective is the identity."""
    rank, world, p2p = 0, 1, False

    def all_gather(self, t):
        return [t]

    def gather_var(self, t):
        return [t]

    def all_to_all(self, tensors):
        return tensors


# ------------------------------------------------------------ int128 helpers


def _i128(lo: int, hi: int) -> int:
    return (hi << 64) + (lo & 0xFFFFFFFFFFFFFFFF)


def term_fx_to_joules(v: int) -> float:
    """fx_to_double(v, 40) / 1e6 (csrc/dw_common.cuh): Python's int/int true
    division is correctly rounded, like the device's fixed-point rounding."""
    return (v / (1 << 40)) / US_PER_S


def joule_fx_to_double(v: int) -> float:
    return v / (1 << 64)


# ---------------------------------------------------------- rank inputs


@dataclass
class RankInputs:
    """What rank g holds of one trace (numpy or CUDA tensors)."""
    window: Window
    kind: str                 # "step" | "linear"
    ts: torch.Tensor          # samples [l0, l1)
    watts: torch.Tensor
    span_hi: int              # STEP: next global sample time (global span end on the last rank)
    glob: dict                # n_samples, ts_first, ts_last, w_first, w_last, span_lo, span_end
    sets: list                # per set: dict(idx, start, end) of the owned intervals (global idx)


def rank_inputs(cols, kind: str, window: Window, sets=("op", "k")) -> RankInputs:
    """Carve rank g's inputs out of a full trace (the driver/test path; a
    deployment reads only its window from the sharded trace files)."""
    ts, w = cols.device("ts"), cols.device("watts")
    S = int(ts.numel())
    first, last = int(ts[0].item()), int(ts[-1].item())
    span_end = cols.signal_span()[1] if kind == "step" else last
    g = window
    lts, lw = ts[g.l0:g.l1], w[g.l0:g.l1]
    span_hi = int(ts[g.l1].item()) if g.l1 < S else span_end
    t_lo = int(ts[g.s0].item()) if g.rank > 0 else None
    t_hi = int(ts[g.s1].item()) if g.rank < g.world - 1 else None
    out = []
    for name in sets:
        st = cols.device(f"{name}_start" if name == "op" else "k_start")
        en = cols.device(f"{name}_end" if name == "op" else "k_end")
        own = torch.ones_like(st, dtype=torch.bool)
        if t_lo is not None:
            own &= st >= t_lo
        if t_hi is not None:
            own &= st < t_hi
        idx = torch.nonzero(own).flatten()
        out.append({"idx": idx, "start": st[idx].contiguous(), "end": en[idx].contiguous()})
    glob = {"n_samples": S, "ts_first": first, "ts_last": last, "w_first": float(w[0].item()),
            "w_last": float(w[-1].item()), "span_lo": first, "span_end": span_end}
    return RankInputs(g, kind, lts.contiguous(), lw.contiguous(), span_hi, glob, out)


def _safe_end(inp: RankInputs) -> int:
    """Owned intervals ending at or before this time are computed whole locally."""
    g = inp.window
    if g.rank == g.world - 1:
        return inp.glob["span_end"]
    return int(inp.ts[g.s1 + _native.DW_DIRECT_MAX - g.l0].item())


def crossing(inp: RankInputs) -> torch.Tensor:
    """Owned intervals that end beyond the halo (phase 1, rank-local): rows of
    (set, global index, start, end), set-major in the rank's interval order."""
    safe = _safe_end(inp)
    rows = []
    for j, s in enumerate(inp.sets):
        m = s["end"] > safe
        idx = s["idx"][m]
        rows.append(torch.stack([torch.full_like(idx, j), idx, s["start"][m], s["end"][m]], dim=1))
    dev = inp.ts.device
    return torch.cat(rows) if rows else torch.empty(0, 4, dtype=torch.int64, device=dev)


def validate(inp: RankInputs) -> torch.Tensor:
    """First invalid owned interval per set, -1 for none (the reference's error
    order is op-major; the caller picks across ranks)."""
    lo_ok, hi_ok = inp.glob["span_lo"], inp.glob["span_end"]
    bad = []
    for s in inp.sets:
        m = (s["end"] < s["start"]) | (s["start"] < lo_ok) | (s["end"] > hi_ok)
        k = torch.nonzero(m).flatten()
        bad.append(s["idx"][k[0]] if k.numel() else torch.full((), -1, dtype=torch.int64, device=m.device))
    return torch.stack(bad) if bad else torch.empty(0, dtype=torch.int64)


@dataclass
class RankResult:
    joules: list             # per set: device f64 of the owned intervals computed whole (in inp order)
    whole: list              # per set: bool mask (inp order) of the intervals computed whole
    parts: torch.Tensor      # [nb, 2] int64: exact int128 (lo, hi) share of every crossing interval (union order)
    tile_fx: torch.Tensor    # [2] int64: int128 share of the ledger total


def compute(inp: RankInputs, union: torch.Tensor) -> RankResult:
    """Phase 2 (rank-local, GPU): whole intervals + shares of the crossing ones."""
    dev = _native.device()
    L = _native.lib()
    safe = _safe_end(inp)
    g = inp.window
    kinds = {"step": _native.DW_SIGNAL_STEP, "linear": _native.DW_SIGNAL_LINEAR}
    sig = _native.Signal(_native.ptr(inp.ts), _native.ptr(inp.watts), int(inp.ts.numel()),
                         int(inp.span_hi), kinds[inp.kind], 0)
    keep, sets, whole, outs = [], [], [], []
    for s in inp.sets:
        m = s["end"] <= safe
        st, en = s["start"][m].contiguous(), s["end"][m].contiguous()
        out = torch.empty(st.numel(), dtype=torch.float64, device=dev)
        keep += [st, en]
        whole.append(m)
        outs.append(out)
        sets.append(_native.IntervalSet(_native.ptr(st), _native.ptr(en), st.numel(), _native.ptr(out),
                                        1 if bool((st.numel() < 2) or bool((st[1:] >= st[:-1]).all())) else 0, 0))
    arr = (_native.IntervalSet * max(len(sets), 1))(*sets)
    union = union.to(dev)
    blo, bhi = union[:, 2].contiguous(), union[:, 3].contiguous()
    nb = int(union.shape[0])
    part = torch.zeros(max(2 * nb, 2), dtype=torch.int64, device=dev)
    tile_fx = torch.zeros(2, dtype=torch.int64, device=dev)
    win = _native.Window(g.l0, inp.glob["n_samples"], g.p0, g.p1, inp.glob["ts_first"], inp.glob["ts_last"],
                         inp.glob["w_first"], inp.glob["w_last"])
    sizes = (ctypes.c_int64 * max(len(sets), 1))(*[s.n for s in sets])
    ws = _native.Workspace.get(L.dw_attribute_workspace_size(sig.n, sizes, len(sets)))
    stream = _native.stream_handle()
    _native.check(L.dw_attribute_window(ctypes.byref(sig), arr, len(sets), ctypes.byref(win), _native.ptr(blo),
                                        _native.ptr(bhi), nb, _native.ptr(part), _native.ptr(tile_fx),
                                        ws.data_ptr(), ws.numel(), stream), "dw_attribute_window")
    st = _native.Status()
    L.dw_status(ws.data_ptr(), stream, ctypes.byref(st))
    if st.order_index >= 0:
        from .trace_model import TraceError
        raise TraceError("power samples must be strictly increasing in timestamp")
    return RankResult(outs, whole, part[: 2 * nb].view(-1, 2), tile_fx)


def _fx_exact(x: torch.Tensor) -> torch.Tensor:
    """Exact 2^-64 J fixed-point sum of x as an int128 (lo, hi) int64 pair (device)."""
    L = _native.lib()
    out = torch.zeros(2, dtype=torch.int64, device=x.device)
    ws = _native.Workspace.get(L.dw_fx_sum_workspace_size(x.numel()))
    _native.check(L.dw_fx_sum_exact(_native.ptr(x), x.numel(), _native.ptr(out), ws.data_ptr(), ws.numel(),
                                    _native.stream_handle()), "dw_fx_sum_exact")
    return out


def sum_i128(parts: torch.Tensor) -> torch.Tensor:
    """Exact sum over dim 0 of int128 values held as (lo, hi) int64 pairs
    ([R, ..., 2] -> [..., 2]) with carries on the device: the low word's two
    32-bit halves are summed separately (no overflow for < 2^31 terms)."""
    lo, hi = parts[..., 0], parts[..., 1]
    l0 = (lo & 0xFFFFFFFF).sum(dim=0)
    l1 = ((lo >> 32) & 0xFFFFFFFF).sum(dim=0)
    h = hi.sum(dim=0)
    l1 = l1 + (l0 >> 32)
    l0 = l0 & 0xFFFFFFFF
    h = h + (l1 >> 32)
    l1 = l1 & 0xFFFFFFFF
    return torch.stack([(l1 << 32) | l0, h], dim=-1)


def _ints(pairs: torch.Tensor) -> list[int]:
    """int128 (lo, hi) pairs -> Python ints, for the one rounding to double."""
    return [_i128(int(x), int(y)) for x, y in pairs.reshape(-1, 2).cpu().tolist()]


@dataclass
class ShardLedger:
    """Rank g's share of a sharded ledger: joules of its owned intervals (global
    indices ``idx`` per set) plus the global totals (equal on every rank)."""
    idx: list
    joules: list
    total_joules: float
    op_total: float
    idle_joules: float


def finish(inp: RankInputs, res: RankResult, block: tuple, all_parts: list, all_tiles: list) -> tuple:
    """Phase 3 (rank-local): this rank's owned joules -- the whole ones, and its
    crossing intervals' exactly summed shares (every rank's [nb, 2] shares of
    the union, summed on the device) rounded once.  ``block`` = (first union
    row of this rank's crossing intervals, per-set counts): the union holds
    them set-major, in this rank's interval order."""
    dev = res.joules[0].device if res.joules else _native.device()
    first, per_set = block
    nown = sum(per_set)
    mine = _ints(sum_i128(torch.stack([p[first:first + nown].to(dev) for p in all_parts]))) if nown else []
    cross = torch.tensor([term_fx_to_joules(v) for v in mine], dtype=torch.float64, device=dev)
    out, e = [], 0
    for j, s in enumerate(inp.sets):
        jl = torch.empty(s["idx"].numel(), dtype=torch.float64, device=dev)
        m = res.whole[j]
        jl[m] = res.joules[j]
        jl[~m] = cross[e:e + per_set[j]]
        e += per_set[j]
        out.append(jl)
    total = term_fx_to_joules(_ints(sum_i128(torch.stack([t.to(dev) for t in all_tiles])))[0])
    return out, total


def _block(rows_per_rank: list, rank: int, cross_rows: torch.Tensor, nsets: int) -> tuple:
    first = sum(int(r.shape[0]) for r in rows_per_rank[:rank])
    per_set = [int((cross_rows[:, 0] == j).sum()) for j in range(nsets)] if cross_rows.numel() else [0] * nsets
    return first, per_set


def sharded_ledger(cols, kind: str, comm: Comm, window: Optional[Window] = None,
                   inputs: Optional[RankInputs] = None) -> ShardLedger:
    """This rank's part of build_ledger over a time-window-sharded trace.  The
    exchanges are tensor all-gathers (NCCL on device tensors): the validation
    indices, the crossing intervals, the crossing shares + tile-sum share, and
    the operator-total share.  ``inputs``: the rank's window, already carved
    (``rank_inputs``); ``cols`` then only serves error reporting."""
    if inputs is None:
        if window is None:
            window = plan(cols.n_power, comm.world, kind)[comm.rank]
        inputs = rank_inputs(cols, kind, window)
    inp = inputs
    bad = torch.stack(comm.all_gather(validate(inp))).cpu().tolist()
    _raise_first_bad(cols, bad)
    mine = crossing(inp)
    rows = comm.gather_var(mine)
    union = torch.cat(rows)
    res = compute(inp, union)
    parts = comm.all_gather(torch.cat([res.parts.reshape(-1), res.tile_fx]))
    nb = int(union.shape[0])
    joules, total = finish(inp, res, _block(rows, comm.rank, mine, len(inp.sets)),
                           [p[: 2 * nb].view(-1, 2) for p in parts], [p[2 * nb:] for p in parts])
    op_fx = comm.all_gather(_fx_exact(joules[0]))
    op_total = joule_fx_to_double(_ints(sum_i128(torch.stack(op_fx)))[0])
    return ShardLedger([s["idx"] for s in inp.sets], joules, total, op_total, max(total - op_total, 0.0))


def _raise_first_bad(cols, bad: list) -> None:
    ops = [b[0] for b in bad if b[0] >= 0]
    ks = [b[1] for b in bad if len(b) > 1 and b[1] >= 0]
    if not ops and not ks:
        return
    bad_op = min(ops) if ops else -1
    bad_k = min(ks) if ks else -1
    owner = None
    if bad_k >= 0 and cols.k_op is not None:
        k_op = cols.k_op
        owner = int(k_op[bad_k].item() if isinstance(k_op, torch.Tensor) else k_op[bad_k])
    span = cols.signal_span()
    if bad_op >= 0 and (owner is None or bad_op <= owner):
        lo, hi = int(cols.device("op_start")[bad_op].item()), int(cols.device("op_end")[bad_op].item())
    else:
        lo, hi = int(cols.device("k_start")[bad_k].item()), int(cols.device("k_end")[bad_k].item())
    _raise_interval_error(lo, hi, span)


# ----------------------------------------------------- in-process loopback


def sharded_ledger_loopback(cols, kind: str, world: int) -> list[ShardLedger]:
    """All ranks of ``sharded_ledger`` in one process, one after the other
    (the collectives become list operations) -- the single-GPU parity check of
    the multi-GPU decomposition."""
    wins = plan(cols.n_power, world, kind)
    inps = [rank_inputs(cols, kind, w) for w in wins]
    _raise_first_bad(cols, [validate(i).cpu().tolist() for i in inps])
    rows = [crossing(i) for i in inps]
    union = torch.cat(rows)
    res = [compute(i, union) for i in inps]
    all_parts, all_tiles = [r.parts for r in res], [r.tile_fx for r in res]
    fin = [finish(i, r, _block(rows, g, rows[g], len(i.sets)), all_parts, all_tiles)
           for g, (i, r) in enumerate(zip(inps, res))]
    op_total = joule_fx_to_double(_ints(sum_i128(torch.stack([_fx_exact(f[0][0]) for f in fin])))[0])
    return [ShardLedger([s["idx"] for s in i.sets], f[0], f[1], op_total, max(f[1] - op_total, 0.0))
            for i, f in zip(inps, fin)]


def gather_ledger(parts: list[ShardLedger], n_ops: int, n_kernels: int):
    """Reassemble full per-op / per-kernel columns from every rank's share."""
    dev = parts[0].joules[0].device
    op = torch.empty(n_ops, dtype=torch.float64, device=dev)
    k = torch.empty(n_kernels, dtype=torch.float64, device=dev)
    for p in parts:
        op[p.idx[0].to(dev)] = p.joules[0].to(dev)
        k[p.idx[1].to(dev)] = p.joules[1].to(dev)
    return op, k


# ------------------------------------------------------ sharded signature join


@dataclass
class ShardOps:
    """One side's operators owned by this rank (global indices, increasing)."""
    idx: torch.Tensor        # int64 global op index
    sig: torch.Tensor        # int64 (the u64 signature's bits)
    start: torch.Tensor
    end: torch.Tensor
    joules: torch.Tensor     # f64
    rank: Optional[torch.Tensor] = None   # A side: id rank (report tie-break); None = index


def shard_ops(cols, led: ShardLedger, side_a: bool) -> ShardOps:
    idx = led.idx[0]
    sig = cols.device("op_sig")
    sig = sig if sig.dtype == torch.int64 else sig.view(torch.int64)
    rank = None
    if side_a:
        rank = cols.device("op_rank")[idx] if cols.op_rank is not None else idx.clone()
    return ShardOps(idx, sig[idx].contiguous(), cols.device("op_start")[idx].contiguous(),
                    cols.device("op_end")[idx].contiguous(), led.joules[0].contiguous(), rank)


def _dest(sig: torch.Tensor, world: int) -> torch.Tensor:
    return ((sig ^ (sig >> 31)) & 0x7FFFFFFF) % world


def _pack(o: ShardOps, with_rank: bool) -> torch.Tensor:
    cols = [o.idx, o.sig, o.start, o.end, o.joules.view(torch.int64)]
    if with_rank:
        cols.append(o.rank)
    return torch.stack(cols, dim=1)


def _partition(o: ShardOps, world: int, with_rank: bool) -> list[torch.Tensor]:
    """Records bound for each rank, in increasing global index."""
    rec = _pack(o, with_rank)
    d = _dest(o.sig, world)
    order = torch.sort(d, stable=True).indices
    counts = torch.bincount(d, minlength=world).cpu().tolist()
    return [t.reshape(-1) for t in torch.split(rec[order], counts)]


def _unpack(parts: list[torch.Tensor], width: int) -> dict:
    rec = torch.cat([p.reshape(-1, width) for p in parts]) if parts else torch.empty(0, width, dtype=torch.int64)
    rec = rec[torch.sort(rec[:, 0]).indices]  # global op order
    out = {"idx": rec[:, 0].contiguous(), "sig": rec[:, 1].contiguous(), "start": rec[:, 2].contiguous(),
           "end": rec[:, 3].contiguous(), "joules": rec[:, 4].contiguous().view(torch.float64)}
    if width == 6:
        out["rank"] = rec[:, 5].contiguous()
    return out


def _local_join(a: dict, b: dict, threshold: float, k: int):
    """The one-GPU signature join over this rank's signatures."""
    from .columns import TraceColumns
    from .energy import EnergyLedger, JoulesView
    from .join import join_diff
    dev = a["sig"].device
    empty = torch.empty(0, dtype=torch.int64, device=dev)

    def cols(d, rank):
        return TraceColumns(ts=empty, watts=empty.double(), trace_end=0, op_start=d["start"], op_end=d["end"],
                            k_start=empty, k_end=empty, op_sig=d["sig"], op_rank=rank, ops_sorted=None,
                            kernels_sorted=True)

    def led(d):
        return EnergyLedger(method="samples", per_kernel=JoulesView(None, empty.double(), "k"),
                        per_operator=JoulesView(None, d["joules"], "op"), idle_joules=0.0, total_joules=0.0)

    ca, cb = cols(a, a["rank"]), cols(b, None)
    jd = join_diff(ca, cb, led(a), led(b), threshold, k, full_columns=False, epw=False)
    return jd, ca, cb


@dataclass
class ShardJoinPart:
    """Phase-2 product of one rank: its top-k candidates with global op
    indices, as device tensors (the gathered form)."""
    key_hi: torch.Tensor     # [k]
    tie: torch.Tensor        # [k] nodes_a tie rank (-1: B-only)
    rows_i: torch.Tensor     # [k, 7] ia, ib, latency_a, latency_b, verdict, side, informational
    rows_f: torch.Tensor     # [k, 4] energy_a, energy_b, ratio, wasted
    stats: torch.Tensor      # [4] P, n_waste, wasted (int128 2^-64 J: lo, hi)
    b_only: torch.Tensor     # global indices of this rank's B-only operators


def _local_part(jd, ca, cb, a: dict, b: dict) -> ShardJoinPart:
    f = jd.order
    ia_l, ib_l = jd.pair_of(f)
    has_a, has_b = ia_l >= 0, ib_l >= 0
    neg = torch.full_like(ia_l, -1)
    ia = torch.where(has_a, a["idx"][ia_l.clamp(min=0)], neg) if a["idx"].numel() else neg
    ib = torch.where(has_b, b["idx"][ib_l.clamp(min=0)], neg) if b["idx"].numel() else neg
    c = jd.columns
    zf = torch.zeros((), dtype=torch.float64, device=f.device)
    zi = torch.zeros((), dtype=torch.int64, device=f.device)
    ea = torch.where(has_a, a["joules"][ia_l.clamp(min=0)], zf) if a["idx"].numel() else zf.expand_as(f)
    eb = torch.where(has_b, b["joules"][ib_l.clamp(min=0)], zf) if b["idx"].numel() else zf.expand_as(f)
    la = torch.where(has_a, (a["end"] - a["start"])[ia_l.clamp(min=0)], zi) if a["idx"].numel() else zi.expand_as(f)
    lb = torch.where(has_b, (b["end"] - b["start"])[ib_l.clamp(min=0)], zi) if b["idx"].numel() else zi.expand_as(f)
    tie = torch.where(has_a, a["rank"][ia_l.clamp(min=0)], neg) if a["idx"].numel() else neg
    waste = c.verdict[: jd.P] == VERDICT_WASTE_I8
    wasted_fx = _fx_exact(c.wasted[: jd.P][waste].contiguous()) if jd.P else torch.zeros(2, dtype=torch.int64,
                                                                                          device=f.device)
    stats = torch.cat([torch.tensor([jd.P], dtype=torch.int64, device=f.device),
                       waste.sum().reshape(1).to(torch.int64), wasted_fx])
    b_only = b["idx"][jd.b_only.to(torch.int64)] if jd.n_b_only else torch.empty(0, dtype=torch.int64,
                                                                                 device=f.device)
    rows_i = torch.stack([ia, ib, la.expand_as(f), lb.expand_as(f), c.verdict[f].to(torch.int64),
                          c.side[f].to(torch.int64), c.informational[f].to(torch.int64)], dim=1)
    rows_f = torch.stack([ea.expand_as(f), eb.expand_as(f), c.ratio[f], c.wasted[f]], dim=1)
    return ShardJoinPart(c.key_hi[f], tie, rows_i, rows_f, stats, b_only)


VERDICT_WASTE_I8 = 2


def _global_lo(part: ShardJoinPart, n_a: int, b_only_all: torch.Tensor) -> torch.Tensor:
    """key_lo = ~((tie + 1) << 32 | f) with the GLOBAL finding number f: the A
    op index, or n_a + the position of the B op among all B-only ops
    (``b_only_all``: every rank's B-only global indices, sorted on the device)."""
    ia, ib = part.rows_i[:, 0], part.rows_i[:, 1]
    pos = torch.searchsorted(b_only_all, ib.contiguous()) if b_only_all.numel() else torch.zeros_like(ib)
    f = torch.where(ia >= 0, ia, n_a + pos)
    return ~(((part.tie + 1) << 32) | f)


@dataclass
class ShardJoinResult:
    P: int
    n_waste: int
    wasted_joules: float
    top: list                # rows in report order (global op indices):
    #                          (ia, ib, ea, eb, la, lb, ratio, wasted, verdict, side, informational)


def sharded_join(A: ShardOps, B: ShardOps, n_a: int, comm: Comm, threshold: float = 0.10,
                 k: int = 100) -> ShardJoinResult:
    """Signature join of a time-window-sharded pair: operators go to the rank
    of hash(signature) (the fused peer-memory exchange, or one NCCL
    all-to-all), where every occurrence of their signature meets in global op
    order -- so the local join pairs exactly as the one-GPU join.  The B-only
    numbering (every rank's B-only indices gathered and sorted on the device)
    and the k candidates of every rank (tensor all-gathers) merge into the
    global report order (dist.merge_order)."""
    if getattr(comm, "p2p", False) and A.sig.is_cuda:
        a = _unpack([comm.exchange(A, True)], 6)
        b = _unpack([comm.exchange(B, False)], 5)
    else:
        a = _unpack(comm.all_to_all(_partition(A, comm.world, True)), 6)
        b = _unpack(comm.all_to_all(_partition(B, comm.world, False)), 5)
    jd, ca, cb = _local_join(a, b, threshold, k)
    part = _local_part(jd, ca, cb, a, b)
    b_only_all = torch.sort(torch.cat(comm.gather_var(part.b_only))).values
    lo = _global_lo(part, n_a, b_only_all)
    gathered = list(zip(comm.gather_var(part.key_hi), comm.gather_var(lo), comm.gather_var(part.rows_i),
                        comm.gather_var(part.rows_f), comm.all_gather(part.stats)))
    return _merge(gathered, k)


def _merge(gathered: list, k: int) -> ShardJoinResult:
    """gathered[r] = (key_hi, key_lo, rows_i, rows_f, stats) of rank r (tensors)."""
    from .dist import merge_order
    dev = gathered[0][0].device
    hi = torch.cat([g[0] for g in gathered])
    lo = torch.cat([g[1].to(dev) for g in gathered])
    rank = torch.cat([torch.full((int(g[0].numel()),), r, dtype=torch.int64, device=dev)
                      for r, g in enumerate(gathered)])
    pos = torch.cat([torch.arange(int(g[0].numel()), dtype=torch.int64, device=dev) for g in gathered])
    order = merge_order(hi, lo, rank, pos, k, by_finding=True)
    ri = torch.cat([g[2].to(dev) for g in gathered])[order].cpu().tolist()
    rf = torch.cat([g[3].to(dev) for g in gathered])[order].cpu().tolist()
    top = [(i[0], i[1], f[0], f[1], i[2], i[3], f[2], f[3], i[4], i[5], i[6]) for i, f in zip(ri, rf)]
    stats = torch.stack([g[4].to(dev) for g in gathered])
    P, n_waste = (int(x) for x in stats[:, :2].sum(dim=0).cpu().tolist())
    wasted = joule_fx_to_double(_ints(sum_i128(stats[:, 2:4]))[0])
    return ShardJoinResult(P, n_waste, wasted, top)


def sharded_join_loopback(As: list, Bs: list, n_a: int, threshold: float = 0.10, k: int = 100) -> ShardJoinResult:
    """Every rank of ``sharded_join`` in one process (single-GPU parity check)."""
    world = len(As)
    sends_a = [_partition(x, world, True) for x in As]
    sends_b = [_partition(x, world, False) for x in Bs]
    parts = []
    for r in range(world):
        a = _unpack([sends_a[s][r] for s in range(world)], 6)
        b = _unpack([sends_b[s][r] for s in range(world)], 5)
        jd, ca, cb = _local_join(a, b, threshold, k)
        parts.append(_local_part(jd, ca, cb, a, b))
    b_only_all = torch.sort(torch.cat([p.b_only for p in parts])).values
    gathered = [(p.key_hi, _global_lo(p, n_a, b_only_all), p.rows_i, p.rows_f, p.stats) for p in parts]
    return _merge(gathered, k)
