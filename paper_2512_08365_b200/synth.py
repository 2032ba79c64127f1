"""Seeded synthetic trace pairs for the BASELINE configs,
generated directly in HBM with torch's Philox generator (no host round trip).

    C2  decode-like pair, 1M ops, 10 kHz samples                     (configs[1])
    C3  4 concurrent streams with overlapping kernels, 10M ops       (configs[2])
    C4  100M ops / 1e9 samples per side (the single-B200 headline)   (configs[3])
    C5  64 pairs x 6.25M ops / 6.25e7 samples (multi-GPU corpus)     (configs[4])

Side A: per op 1..kmax back-to-back kernels with log-uniform durations, a
uniform inter-op gap, kernel watts U(150, 700) over a 75 W idle floor and a
signature drawn from a 64-name Zipf vocabulary x 16 shape buckets x 2 dtypes x
256 call sites.  Side B = A with (i) 1% of signatures drawing (1+m) x the
watts, m ~ U(0.02, 0.5)  (misconfiguration-like), (ii) 0.1% extra operators
inserted (redundant) and (iii) 0.1% operators renamed (api-misuse).  The power
column is the step ground truth read every ``span/S`` us (delay 0), so S is
exact; C4 / C5 jitter each read by up to a quarter period (an irregular,
host-polled meter: 7-bit timestamp deltas instead of a 1-bit regular clock).  Everything is a pure function of (config, seed).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from .columns import TraceColumns

IDLE_W = 75.0


@dataclass(frozen=True)
class SynthConfig:
    name: str
    n_ops: int
    n_samples: int
    seed: int
    kmax: int = 2
    kdur: tuple = (20, 3000)      # kernel duration log-uniform bounds, us
    gap: int = 200                # inter-op gap U{0..gap}, us
    streams: int = 1
    watt_frac: float = 0.01       # fraction of signatures with inflated watts on B
    insert_frac: float = 0.001
    rename_frac: float = 0.001
    jitter: float = 0.0           # sample-clock jitter, fraction of the period (NVML-like irregular reads)


CONFIGS = {
    "C2": SynthConfig("C2", 1_000_000, 0, seed=2, kmax=3, kdur=(5, 500), gap=20),
    "C3": SynthConfig("C3", 10_000_000, 0, seed=3, kmax=3, kdur=(5, 2000), gap=20, streams=4),
    "C4": SynthConfig("C4", 100_000_000, 1_000_000_000, seed=4, kmax=2, kdur=(20, 3000), gap=200, jitter=0.25),
    "C5": SynthConfig("C5", 6_250_000, 62_500_000, seed=5000, kmax=2, kdur=(20, 3000), gap=200, jitter=0.25),
}


def scaled(cfg: SynthConfig, n_ops: int, n_samples: int | None = None) -> SynthConfig:
    """Same distribution at a smaller size (tests, CPU-baseline samples)."""
    from dataclasses import replace
    if n_samples is None and cfg.n_samples:
        n_samples = max(2, int(cfg.n_samples * n_ops / cfg.n_ops))
    return replace(cfg, n_ops=n_ops, n_samples=n_samples or 0)


def _splitmix64(x: torch.Tensor) -> torch.Tensor:
    """SplitMix64 finaliser on int64 tensors (wrapping arithmetic)."""
    x = x + (-7046029254386353131)  # 0x9E3779B97F4A7C15
    x = (x ^ ((x >> 30) & 0x3FFFFFFFF)) * (-4658895280553007687)  # 0xBF58476D1CE4E5B9
    x = (x ^ ((x >> 27) & 0x1FFFFFFFFF)) * (-7723592293110705685)  # 0x94D049BB133111EB
    return x ^ ((x >> 31) & 0x1FFFFFFFF)


def signature(name, shape, dtype, callsite) -> torch.Tensor:
    """64-bit operator signature of (op name, shape bucket, dtype, call site)
    (DESIGN.md "signature join")."""
    h = _splitmix64(name.to(torch.int64) + 0x100000)
    h = _splitmix64(h ^ (shape.to(torch.int64) << 20))
    h = _splitmix64(h ^ (dtype.to(torch.int64) << 40))
    return _splitmix64(h ^ (callsite.to(torch.int64) << 48))


class _Ops:
    """Per-op attributes before timeline layout."""

    def __init__(self, kc, kdur, kw, gap, sig):
        self.kc, self.kdur, self.kw, self.gap, self.sig = kc, kdur, kw, gap, sig


def _draw_ops(n: int, cfg: SynthConfig, g: torch.Generator, dev) -> _Ops:
    kc = torch.randint(1, cfg.kmax + 1, (n,), generator=g, device=dev)
    K = int(kc.sum().item())
    lo, hi = math.log(cfg.kdur[0]), math.log(cfg.kdur[1])
    kdur = torch.exp(torch.rand(K, generator=g, device=dev, dtype=torch.float64) * (hi - lo) + lo)
    kdur = kdur.round().clamp_(min=1).to(torch.int64)
    kw = torch.rand(K, generator=g, device=dev, dtype=torch.float64) * 550.0 + 150.0
    gap = torch.randint(0, cfg.gap + 1, (n,), generator=g, device=dev)
    u = torch.rand(n, generator=g, device=dev, dtype=torch.float64)
    name = torch.floor(64.0 * u * u * u).to(torch.int64)  # Zipf-like skew
    shape = torch.randint(0, 16, (n,), generator=g, device=dev)
    dtype = torch.randint(0, 2, (n,), generator=g, device=dev)
    callsite = torch.randint(0, 256, (n,), generator=g, device=dev)
    return _Ops(kc, kdur, kw, gap, signature(name, shape, dtype, callsite))


def _kernel_offsets(kc: torch.Tensor) -> torch.Tensor:
    return torch.cumsum(kc, 0) - kc  # first kernel index of each op


def _layout(ops: _Ops, t0: int, dev):
    """Timeline: kernels back to back inside an op, ops separated by gaps."""
    n = ops.kc.numel()
    kop = torch.repeat_interleave(torch.arange(n, device=dev), ops.kc)
    op_dur = torch.zeros(n, dtype=torch.int64, device=dev).index_add_(0, kop, ops.kdur)
    step = op_dur + ops.gap
    op_start = t0 + torch.cumsum(step, 0) - step
    op_end = op_start + op_dur
    kfirst = _kernel_offsets(ops.kc)
    kcum = torch.cumsum(ops.kdur, 0) - ops.kdur  # exclusive over all kernels
    k_start = op_start[kop] + (kcum - kcum[kfirst][kop])
    k_end = k_start + ops.kdur
    return op_start, op_end, k_start, k_end, kop.to(torch.int32)


def _truth_at(ts: torch.Tensor, k_start, k_end, kw, chunk=1 << 26) -> torch.Tensor:
    """Step ground truth: kernel watts while a kernel runs, idle otherwise."""
    out = torch.empty(ts.numel(), dtype=torch.float64, device=ts.device)
    for a in range(0, ts.numel(), chunk):
        t = ts[a:a + chunk]
        i = torch.searchsorted(k_start, t, right=True) - 1
        ic = i.clamp(min=0)
        on = (i >= 0) & (t < k_end[ic])
        out[a:a + chunk] = torch.where(on, kw[ic], torch.full_like(t, IDLE_W, dtype=torch.float64))
    return out


_POW10 = [10.0 ** k for k in range(23)]  # exact doubles


def round9(w: torch.Tensor) -> torch.Tensor:
    """Watts at the trace format's on-disk precision: 9 significant decimal
    digits (trace_model.py:63-65, the reference writes every power sample
    that way), as the double nearest each decimal (one IEEE division)."""
    pos = w > 0
    p = (8 - torch.floor(torch.log10(torch.where(pos, w, torch.ones_like(w))))).to(torch.int64).clamp(0, 22)
    pw = torch.tensor(_POW10, dtype=torch.float64, device=w.device)[p]
    m = torch.round(w * pw)
    m = torch.where(m >= 1e9, torch.round(w * pw / 10.0) * 10.0, m)  # log10 landed one decade low
    return torch.where(pos, torch.div(m, pw), w)


def _power(op_end_max: int, t0: int, n_samples: int, k_start, k_end, kw, dev, jitter: float = 0.0,
           seed: int = 0):
    span = max(op_end_max - t0, 1)
    if n_samples <= 0:
        n_samples = max(2, span // 100)  # 10 kHz
    # samples at t0 + floor(i * span / (S-1)): the last one lands on the trace
    # end, so a sampled (trapezoid) view covers every interval.  With jitter J
    # each interior read moves by up to +-J periods (J < 1/2 keeps the clock
    # strictly increasing): a power meter polled by a host thread.
    period = span / (n_samples - 1)
    x = torch.arange(n_samples, device=dev, dtype=torch.float64)
    if jitter > 0:
        assert jitter < 0.5
        gj = torch.Generator(device=dev)
        gj.manual_seed(seed)
        x += (2.0 * torch.rand(n_samples, device=dev, dtype=torch.float64, generator=gj) - 1.0) * jitter
    ts = t0 + torch.floor(x * period).to(torch.int64)
    ts[0] = t0
    ts[-1] = t0 + span
    if period < 1:
        raise ValueError("more samples than microseconds in the span")
    return ts, _truth_at(ts, k_start, k_end, round9(kw))


def _b_side(a: _Ops, cfg: SynthConfig, g: torch.Generator, dev) -> _Ops:
    n = a.kc.numel()
    # (i) inflated watts for 1% of signatures
    sig_bits = (a.sig & 0xFFFF).to(torch.float64) / 65536.0
    hot = sig_bits < cfg.watt_frac
    mult = 1.0 + (0.02 + 0.48 * ((a.sig >> 16) & 0xFFFF).to(torch.float64) / 65536.0)
    op_mult = torch.where(hot, mult, torch.ones_like(mult))
    kop = torch.repeat_interleave(torch.arange(n, device=dev), a.kc)
    kw = a.kw * op_mult[kop]
    # (iii) api misuse: 0.1% of the signatures are served by a different
    # operator on B -- every occurrence renamed (systematic, like a framework
    # dispatching another kernel for that op everywhere)
    ren = (((a.sig >> 32) & 0xFFFF).to(torch.float64) / 65536.0) < cfg.rename_frac
    sig = torch.where(ren, _splitmix64(a.sig ^ 0x5DEECE66D), a.sig)
    # (ii) inserted ops: one extra op after each selected position
    ins = torch.rand(n, generator=g, device=dev) < cfg.insert_frac
    n_ins = int(ins.sum().item())
    extra = _draw_ops(n_ins, cfg, g, dev)
    extra.sig = _splitmix64(extra.sig ^ 0x1B873593)
    # interleave: new index of op i = i + (#inserted before or at i-1)
    shift = torch.cumsum(ins.to(torch.int64), 0) - ins.to(torch.int64)
    pos_a = torch.arange(n, device=dev) + shift
    pos_x = torch.nonzero(ins).flatten() + shift[ins] + 1
    nb = n + n_ins
    kc = torch.empty(nb, dtype=torch.int64, device=dev)
    kc[pos_a] = a.kc
    kc[pos_x] = extra.kc
    gap = torch.empty_like(kc)
    gap[pos_a] = a.gap
    gap[pos_x] = extra.gap
    sigb = torch.empty(nb, dtype=torch.int64, device=dev)
    sigb[pos_a] = sig
    sigb[pos_x] = extra.sig
    # kernels follow their ops
    kfirst_b = _kernel_offsets(kc)
    Kb = int(kc.sum().item())
    kdur = torch.empty(Kb, dtype=torch.int64, device=dev)
    kwb = torch.empty(Kb, dtype=torch.float64, device=dev)

    def scatter(src_dur, src_w, src_kc, pos):
        kop_s = torch.repeat_interleave(torch.arange(src_kc.numel(), device=dev), src_kc)
        within = torch.arange(src_dur.numel(), device=dev) - _kernel_offsets(src_kc)[kop_s]
        dst = kfirst_b[pos][kop_s] + within
        kdur[dst] = src_dur
        kwb[dst] = src_w

    scatter(a.kdur, kw, a.kc, pos_a)
    scatter(extra.kdur, extra.kw, extra.kc, pos_x)
    return _Ops(kc, kdur, kwb, gap, sigb)


def _columns(ops: _Ops, cfg: SynthConfig, t0: int, n_samples: int, dev, prefix: str) -> TraceColumns:
    op_start, op_end, k_start, k_end, kop = _layout(ops, t0, dev)
    end = int(op_end[-1].item())
    ts, watts = _power(end, t0, n_samples, k_start, k_end, ops.kw, dev, cfg.jitter,
                       cfg.seed * 2 + (prefix == "b"))
    n = op_start.numel()
    return TraceColumns(ts=ts, watts=watts, trace_end=max(end, int(ts[-1].item())),
                        op_start=op_start, op_end=op_end, k_start=k_start, k_end=k_end,
                        k_op=kop, op_sig=ops.sig,
                        ops_sorted=True, kernels_sorted=True)


def make_pair(cfg: SynthConfig | str, device=None) -> tuple[TraceColumns, TraceColumns]:
    """(side A, side B) columns resident on ``device`` (default: current CUDA device)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed)
    t0 = 1_000
    if cfg.streams > 1:
        return _make_pair_streams(cfg, g, dev, t0)
    a = _draw_ops(cfg.n_ops, cfg, g, dev)
    b = _b_side(a, cfg, g, dev)
    ca = _columns(a, cfg, t0, cfg.n_samples, dev, "a")
    del a
    cb = _columns(b, cfg, t0, cfg.n_samples, dev, "b")
    return ca, cb


def _make_pair_streams(cfg: SynthConfig, g, dev, t0: int):
    sides = []
    per = cfg.n_ops // cfg.streams
    a_streams = [_draw_ops(per, cfg, g, dev) for _ in range(cfg.streams)]
    offs = [int(x) for x in torch.randint(0, 5000, (cfg.streams,), generator=g, device=dev).tolist()]
    for side in (0, 1):
        parts = []
        for s, a in enumerate(a_streams):
            ops = a if side == 0 else _b_side(a, cfg, g, dev)
            op_start, op_end, k_start, k_end, kop = _layout(ops, t0 + offs[s], dev)
            parts.append((op_start, op_end, k_start, k_end, kop, ops))
        # merge ops of all streams by start; kernels follow their op (flattened order)
        op_start = torch.cat([p[0] for p in parts])
        op_end = torch.cat([p[1] for p in parts])
        sig = torch.cat([p[5].sig for p in parts])
        kc = torch.cat([p[5].kc for p in parts])
        k_start_all = torch.cat([p[2] for p in parts])
        k_end_all = torch.cat([p[3] for p in parts])
        order = torch.argsort(op_start, stable=True)
        kfirst = _kernel_offsets(kc)
        kc_o = kc[order]
        kop_new = torch.repeat_interleave(torch.arange(order.numel(), device=dev), kc_o)
        within = torch.arange(kop_new.numel(), device=dev) - _kernel_offsets(kc_o)[kop_new]
        src = kfirst[order][kop_new] + within
        k_start = k_start_all[src]
        k_end = k_end_all[src]
        end = int(op_end.max().item())
        span = end - t0
        n_samples = max(2, span // 100)
        ts = t0 + torch.floor(torch.arange(n_samples, device=dev, dtype=torch.float64)
                              * (span / (n_samples - 1))).to(torch.int64)
        ts[-1] = t0 + span
        watts = torch.full((n_samples,), IDLE_W, dtype=torch.float64, device=dev)
        for p in parts:  # power adds up across concurrent streams
            watts += _truth_at(ts, p[2], p[3], p[5].kw) - IDLE_W
        sides.append(TraceColumns(ts=ts, watts=watts, trace_end=max(end, int(ts[-1].item())),
                                  op_start=op_start[order], op_end=op_end[order],
                                  k_start=k_start, k_end=k_end, k_op=kop_new.to(torch.int32),
                                  op_sig=sig[order],
                                  ops_sorted=True, kernels_sorted=None))
    return sides[0], sides[1]
