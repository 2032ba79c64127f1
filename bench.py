#!/usr/bin/env python
"""Benchmark of the Magneton/diffwatt hot path on B200 (one JSON line).

A step = attribution of both traces of a pair (per-operator and per-kernel
joules, trapezoid over the trace's power samples) + the signature-join
differential diff (per finding: energy delta, time delta, energy-per-work
ratio and ranking key) + the top-k ranked report on the host: the BASELINE
config 4 workload (100M operators / 1e9 power samples per trace, SURVEY.md
8(d) C4) on one B200, generated in HBM from a fixed seed.  After the timed
runs the same path runs on the CPU baseline's sample and is compared with the
oracle ("parity").

  value  operator intervals (ops + kernels, both traces) attributed per second,
         inputs resident in HBM (inputs >> 126 MB L2, so no flush is needed)
  e2e    the same metric through the public API (pipeline.analyze) from pinned
         host buffers: every step copies both traces host->HBM and reads the
         report back
  N > 1  one process per GPU (torchrun), each rank its own pair (weak scaling);
         the per-rank top-k candidates are merged over NCCL (all_gather).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "operator-intervals attributed/sec and power-samples/sec; trace-pair diff latency"
UNIT = "operator-intervals/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="C4")
    ap.add_argument("--method", default="samples", choices=("samples", "ground_truth"))
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--summation", default="exact", choices=("exact", "reference"),
                    help="how each interval's pieces are summed (energy.build_ledger): the exact "
                         "fixed-point sum (default, the scale path) or the reference's sequential order")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-ops", type=int, default=2_000_000)
    ap.add_argument("--pairs", type=int, default=64, help="C5 corpus size (trace pairs)")
    ap.add_argument("--overlap", default="compat", choices=("compat", "split"),
                    help="energy.build_ledger overlap mode (split: power shared among concurrent intervals)")
    ap.add_argument("--shard", default="pair", choices=("pair", "window"),
                    help="N>1: 'pair' = every rank its own trace pair (weak scaling, corpus); "
                         "'window' = ONE pair split by time window over the ranks (strong scaling)")
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"))
    return ap.parse_args()


# ------------------------------------------------------------------ helpers


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a moment to start polling: wait for its first
            # line so a short timed region still gets sampled
            t0 = time.time()
            while not self.lines and self.proc.poll() is None and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None and not self.lines:
            # a timed region shorter than the polling period: one reading
            # right at its end (clocks have not dropped yet)
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=10).stdout.strip()
                if out:
                    self.lines.append(out.splitlines()[-1].strip())
                    self.post = True
            except (OSError, subprocess.SubprocessError):
                pass
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(sm)}
        if getattr(self, "post", False):
            out["note"] = "region shorter than the 100 ms polling period: one reading at its end"
        return out


def measured_peak_gbs():
    try:
        with open(ROOT / "MEASURED_PEAKS.json") as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def profiled_traffic(config: str, method: str):
    """dram bytes per tile-kernel launch from the committed ncu --set full summary."""
    try:
        with open(ROOT / "profiles" / "traffic.json") as fh:
            d = json.load(fh)
        return d.get(f"{config}:{method}")
    except (OSError, ValueError):
        return None


def attr_bytes(cols) -> int:
    """Algorithmic bytes of one ledger: 16 B per power sample + 24 B per
    interval (start/end in, joules out) -- SURVEY.md 8(d)."""
    return 16 * cols.n_power + 24 * (cols.n_ops + cols.n_kernels)


def diff_bytes(ca, cb, P: int) -> int:
    return 32 * (ca.n_ops + cb.n_ops) + 32 * P


# ------------------------------------------------------------------ CPU arm


def cpu_sample(cfg_name: str, n_ops: int, seed_shift: int = 0):
    """A bounded sample of the same workload, generated on the host."""
    import numpy as np  # noqa: F401
    from paper_2512_08365_b200 import synth
    cfg = synth.scaled(synth.CONFIGS[cfg_name], n_ops)
    from dataclasses import replace
    cfg = replace(cfg, seed=cfg.seed + seed_shift)
    ca, cb = synth.make_pair(cfg, device="cpu")
    return ca, cb


def cpu_step(ca, cb, method: str, k: int, mode=None):
    """The reference hot path restated in C (oracle/, pthreads over all host
    cores): ledger of both traces, signature join, detect rule, report order.
    ``mode``: the oracle's summation (default the reference's sequential
    sums; oracle.MODE_EXACT restates summation="exact")."""
    import numpy as np
    import oracle
    if mode is None:
        mode = oracle.MODE_REFERENCE
    kind = "linear" if method == "samples" else "step"
    out = []
    for c in (ca, cb):
        ts, w = c.host("ts"), c.host("watts")
        span_hi = None if kind == "linear" else c.signal_span()[1]
        out.append(oracle.ledger(kind, ts, w, span_hi, c.host("op_start"), c.host("op_end"),
                                 c.host("k_start"), c.host("k_end"), mode))
    ja, jb = out[0][0], out[1][0]
    sig_a = c_sig(ca)
    sig_b = c_sig(cb)
    ma, mb = oracle.join(sig_a, sig_b)
    na = len(ma)
    b_only = np.nonzero(mb < 0)[0]
    off_a = np.concatenate([np.arange(na + 1), np.full(len(b_only), na)]).astype(np.int64)
    mem_a = np.arange(na, dtype=np.int32)
    has_b = (ma >= 0).astype(np.int64)
    off_b = np.concatenate([[0], np.cumsum(has_b), np.sum(has_b) + np.arange(1, len(b_only) + 1)])
    mem_b = np.concatenate([ma[ma >= 0], b_only]).astype(np.int32)
    d = oracle.detect(off_a, mem_a, off_b, mem_b, ja, jb, ca.host("op_start"), ca.host("op_end"),
                      cb.host("op_start"), cb.host("op_end"), None, 0.10)
    tie = np.concatenate([np.arange(na) + 1, np.zeros(len(b_only), dtype=np.int64)])
    order = oracle.rank(d["verdict"], d["wasted"], tie)
    waste = d["verdict"] == 2
    return {"ledgers": out, "match_a": ma, "b_only": b_only, "order": order[:k],
            "n_waste": int(waste.sum()), "wasted": oracle.fx_sum(d["wasted"][waste])}


def parity_record(args, dev) -> dict:
    """The GPU path (pipeline.analyze, this run's summation) against the CPU
    oracle on the exact sample cpu_baseline times: ledgers, pairing, top-k
    order, waste count and wasted joules bit for bit under the same summation
    definition, and the per-operator joules against the reference's own
    sequential sums within the north star's 1e-6 relative."""
    import numpy as np
    import oracle
    from paper_2512_08365_b200.pipeline import analyze
    ca, cb = cpu_sample(args.config, args.cpu_sample_ops)
    mode = oracle.MODE_EXACT if args.summation == "exact" else oracle.MODE_DEVICE
    ref = cpu_step(ca, cb, args.method, args.k, mode)
    res = analyze(ca, cb, args.method, 0.10, args.k, summation=args.summation)
    led_eq = True
    for led, (po, pk, total, idle) in zip((res.ledger_a, res.ledger_b), ref["ledgers"]):
        led_eq &= bool(np.array_equal(led.per_operator.array(), po) and np.array_equal(led.per_kernel.array(), pk)
                       and led.total_joules == total and led.idle_joules == idle)
    jd = res.join
    join_eq = bool(np.array_equal(jd.match_a.cpu().numpy(), ref["match_a"]) and
                   np.array_equal(jd.b_only.cpu().numpy(), ref["b_only"]))
    topk_eq = bool(np.array_equal(jd.order.cpu().numpy(), ref["order"]))
    # the reference's sequential sums (MODE_REFERENCE) per operator
    kind = "linear" if args.method == "samples" else "step"
    rel = 0.0
    for c, led in ((ca, res.ledger_a), (cb, res.ledger_b)):
        f = oracle.integrate_linear if kind == "linear" else None
        lo, hi = c.host("op_start"), c.host("op_end")
        want = (f(c.host("ts"), c.host("watts"), lo, hi, oracle.MODE_REFERENCE) if f else
                oracle.integrate_step(c.host("ts"), c.host("watts"), c.signal_span()[1], lo, hi,
                                      oracle.MODE_REFERENCE))
        got = led.per_operator.array()
        nz = want != 0
        rel = max(rel, float(np.max(np.abs(got[nz] - want[nz]) / np.abs(want[nz]))) if nz.any() else 0.0)
    out = {"sample": f"{args.config} distribution, {ca.n_ops}+{cb.n_ops} ops, {ca.n_power}+{cb.n_power} samples",
           "oracle_mode": {oracle.MODE_EXACT: "MODE_EXACT", oracle.MODE_DEVICE: "MODE_DEVICE"}[mode],
           "ledgers_bit_exact": led_eq, "pairing_bit_exact": join_eq, "topk_order_equal": topk_eq,
           "n_waste_equal": jd.n_waste == ref["n_waste"], "wasted_joules_equal": jd.wasted_joules == ref["wasted"],
           "max_rel_err_vs_reference_sums": rel, "tolerance": 1e-6}
    out["pass"] = bool(led_eq and join_eq and topk_eq and out["n_waste_equal"] and out["wasted_joules_equal"]
                       and rel <= 1e-6)
    return out


def c_sig(c):
    import numpy as np
    s = c.host("op_sig")
    return np.ascontiguousarray(s).view(np.uint64)


def host_cpu() -> dict:
    """The host's CPU model (lscpu "Model name", from /proc/cpuinfo) and
    logical core count, reported beside every CPU number."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.lower().startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_baseline(args, steps: int = 1) -> dict:
    import oracle
    ca, cb = cpu_sample(args.config, args.cpu_sample_ops)
    intervals = ca.n_ops + ca.n_kernels + cb.n_ops + cb.n_kernels
    cpu_step(ca, cb, args.method, args.k)  # warm (page-in, thread start)
    t0 = time.perf_counter()
    for _ in range(steps):
        cpu_step(ca, cb, args.method, args.k)
    dt = (time.perf_counter() - t0) / steps
    return {"value": intervals / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "port",
            **host_cpu(),
            "sample": (f"{args.config} distribution scaled to {ca.n_ops}+{cb.n_ops} ops, "
                       f"{ca.n_power}+{cb.n_power} samples (pair); oracle/dw_oracle.c "
                       f"reference-order sums, {oracle.num_threads()} threads"),
            "seconds_per_step": dt}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    import oracle
    ca, cb = cpu_sample(args.config, args.cpu_sample_ops)
    intervals = ca.n_ops + ca.n_kernels + cb.n_ops + cb.n_kernels
    for _ in range(args.warmup):
        cpu_step(ca, cb, args.method, args.k)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_step(ca, cb, args.method, args.k)
    dt = (time.perf_counter() - t0) / args.steps
    v = intervals / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config} (bounded CPU sample)", "method": args.method,
                   "ops_per_trace": ca.n_ops, "samples_per_trace": ca.n_power},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "port", **host_cpu(),
                         "sample": f"{ca.n_ops}+{cb.n_ops} ops, {ca.n_power}+{cb.n_power} samples"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm


def run_ours(args, rank: int, world: int, local: int):
    import torch
    import torch.distributed as dist

    from paper_2512_08365_b200 import _native, synth
    from paper_2512_08365_b200.columns import TraceColumns
    from paper_2512_08365_b200.dist import merge_topk
    from paper_2512_08365_b200.pipeline import analyze

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = _native.lib()
    from dataclasses import replace
    cfg = replace(synth.CONFIGS[args.config], seed=synth.CONFIGS[args.config].seed + 1000 * rank)
    ca, cb = synth.make_pair(cfg, dev)
    for c in (ca, cb):
        for n in TraceColumns.HOT:
            c.device(n)
    torch.cuda.synchronize()
    intervals = ca.n_ops + ca.n_kernels + cb.n_ops + cb.n_kernels
    samples = ca.n_power + cb.n_power

    def step():
        res = analyze(ca, cb, args.method, 0.10, args.k, summation=args.summation, overlap=args.overlap)
        if world > 1:  # corpus top-k: merge every rank's k candidates over NCCL
            jd = res.join
            f = jd.order
            tie = jd.pair_of(f)[0].clamp(min=-1)  # A-op index (== id rank here), -1 for B-only
            lo = ~(((tie + 1) << 32) | f)
            merge_topk(jd.columns.key_hi[f], lo, args.k)
        return res

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    L.dw_kernel_time_ms(1)
    L.dw_kernel_timed_count(1)
    L.dw_kernel_timing(1)
    _native.launch_count(reset=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            res = step()
        e1.record()
        torch.cuda.synchronize()
    L.dw_kernel_timing(0)
    launches = _native.launch_count(reset=True)
    n_timed = int(L.dw_kernel_timed_count(1))
    kern_ms = L.dw_kernel_time_ms(1) / max(n_timed, 1)  # per tile-kernel launch (every launch timed)
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # phase split of one step (rank-local): attribution vs diff latency
    from paper_2512_08365_b200.energy import build_ledger
    from paper_2512_08365_b200.join import join_diff
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    la = build_ledger(ca, method=args.method, summation=args.summation, overlap=args.overlap)
    lb = build_ledger(cb, method=args.method, summation=args.summation, overlap=args.overlap)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    from paper_2512_08365_b200.detect import FindingColumns
    jd = join_diff(ca, cb, la, lb, 0.10, args.k, full_columns=False, epw=False, columns=FindingColumns.DELTAS)
    jd.top_findings(ca, cb)
    t2 = time.perf_counter()
    P = res.join.P

    # ---- e2e through the public API from pinned host buffers
    e2e = None
    e2e_skip = None
    if not args.no_e2e:
        del res, la, lb, jd
        # the host holds what a deployment ships: packed columns
        # (columns.PackedColumns) in pinned memory.  Pack on the device first:
        # the exact host bytes decide whether this box's memory holds every
        # local rank's copy (all local ranks share it).
        import psutil
        from paper_2512_08365_b200.columns import PackedColumns, pack
        try:
            packed = [pack(c) for c in (ca, cb)]
            need = sum(pc.host_bytes for pc in packed)
        except ValueError as exc:  # e.g. overlapping streams (C3): kernel starts not sorted
            packed, pack_refusal = None, str(exc)
            need = sum(getattr(c, n).numel() * getattr(c, n).element_size() for c in (ca, cb)
                       for n in TraceColumns.HOT + ("k_op",) if getattr(c, n, None) is not None)
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        avail = psutil.virtual_memory().available
        if need * local_world > 0.75 * avail:
            e2e_skip = (f"host memory: {local_world} ranks x {need / 1e9:.1f} GB pinned > 75% of "
                        f"{avail / 1e9:.0f} GB available")
            del packed
    if not args.no_e2e and e2e_skip is None and packed is None:
        # the trace does not pack: pinned unpacked columns
        def pin(t):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h
        pinned = []
        for c in (ca, cb):
            hc = TraceColumns(ts=pin(c.device("ts")), watts=pin(c.device("watts")), trace_end=c.trace_end,
                              op_start=pin(c.device("op_start")), op_end=pin(c.device("op_end")),
                              k_start=pin(c.device("k_start")), k_end=pin(c.device("k_end")),
                              op_sig=pin(c.device("op_sig")), ops_sorted=c.ops_sorted,
                              kernels_sorted=c.kernels_sorted,
                              k_op=pin(c.device("k_op")) if c.k_op is not None else None)
            hc._dev["first_last"] = c._first_last_ts()
            hc.host_bytes = sum(getattr(hc, n).numel() * getattr(hc, n).element_size()
                                for n in TraceColumns.HOT + ("k_op",) if getattr(hc, n) is not None)
            pinned.append(hc)
        h2d = sum(hc.host_bytes for hc in pinned)
        host_format = f"unpacked columns (int64 / f64 / u64; {pack_refusal})"
        for c in (ca, cb):
            c._dev.clear()
        del ca, cb
        torch.cuda.empty_cache()
        copy_stream = torch.cuda.Stream()
    elif not args.no_e2e and e2e_skip is None:
        pinned = []
        for c, pc in zip((ca, cb), packed):

            def pin(t):  # straight into pinned memory: no pageable staging copy
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t)
                return h
            hc = PackedColumns(pc.ts_base, pin(pc.ts), pin(pc.watts), pc.op_start_base, pin(pc.op_start),
                               pin(pc.op_end), pc.k_start_base, pin(pc.k_start), pin(pc.k_end), c.trace_end,
                               op_sig=pin(pc.op_sig), watts_p0=pc.watts_p0, ts_bias=pc.ts_bias,
                               op_sig_dict=pin(pc.op_sig_dict) if pc.op_sig_dict is not None else None,
                               ts_bits=pc.ts_bits, ts_step=pc.ts_step, watts_bits=pc.watts_bits, n_power=pc.n_power,
                               ts_last=pc._ts_last if pc.ts_bits is not None else None,
                               iv_bits=pc.iv_bits, n_ops=pc.n_ops, n_kernels=pc.n_kernels,
                               sig_bits=pc.sig_bits,
                               watts_rep=pin(pc.watts_rep) if pc.watts_rep is not None else None)
            hc._dev["first_last"] = c._first_last_ts()
            pinned.append(hc)
        del packed, pc
        h2d = sum(pc.host_bytes for pc in pinned)
        pc0 = pinned[0]
        tsw = pc0.ts.element_size()
        tsf = (f"{pc0.ts_bits}-bit packed" if pc0.ts_bits is not None else
               ("biased i8" if tsw == 1 else f"u{8 * tsw}"))
        def ivf(a, b):
            if a in pc0.iv_bits:
                return f"{pc0.iv_bits[a][0]}/{pc0.iv_bits[b][0]}-bit packed"
            return f"u{8 * getattr(pc0, a).element_size()}/u{8 * getattr(pc0, b).element_size()}"
        tsk = "residuals from the clock's line" if pc0.ts_step is not None else "deltas"
        host_format = (f"packed columns: ts {tsk} {tsf}, interval deltas/durations "
                       f"{ivf('op_start', 'op_end')} (ops) {ivf('k_start', 'k_end')} (kernels), watts "
                       + (("run-coded 9-digit decimal codes (change bitmap + "
                           + (f"{pc0.watts_bits[0]}-bit" if pc0.watts_bits is not None else "u32")
                           + " code per change, "
                           f"{pc0.watts.numel() / pc0.n_power:.3f} codes/sample)" if pc0.watts_rep is not None
                           else "9-digit decimal codes u32") if pc0.watts_p0 is not None else "f64")
                       + ((f", sig dictionary + {pc0.sig_bits}-bit codes" if pc0.sig_bits is not None else
                           f", sig dictionary + u{8 * pc0.op_sig.element_size()} codes")
                          if pc0.op_sig_dict is not None else ", sig u64"))
        for c in (ca, cb):
            c._dev.clear()
        del ca, cb
        torch.cuda.empty_cache()
        copy_stream = torch.cuda.Stream()

    if not args.no_e2e and e2e_skip is None:
        def e2e_step():
            for pc in pinned:
                pc.drop_device()
            r = analyze(pinned[0], pinned[1], args.method, 0.10, args.k, copy_stream=copy_stream,
                        summation=args.summation, overlap=args.overlap)
            return r

        for _ in range(max(5, args.warmup)):  # the first steps run up to 50 % slower (allocator, pinned pages)
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.e2e_steps)]
        f0.record()
        for i in range(args.e2e_steps):
            e2e_step()  # the report is on the host; nothing of the step outlives it (as in the warm-up)
            marks[i].record()
        f1.record()
        torch.cuda.synchronize()
        e_ms = f0.elapsed_time(f1) / args.e2e_steps
        if os.environ.get("DWB200_E2E_DEBUG"):
            prev = [f0] + marks[:-1]
            print("e2e steps ms:", [round(a.elapsed_time(b), 1) for a, b in zip(prev, marks)], file=sys.stderr)
        te = torch.tensor([e_ms], device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        # d2h: top-k indices/keys/columns + ledger totals read back for the report
        d2h = args.k * (8 * 2 + 8 * 6 + 3) + 8 * 8
        e2e = {"value": world * intervals / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(te.item()),
               "host_format": host_format,
               "overlap": "trace B H2D + decode under trace A attribution"}

    if rank != 0:
        return
    peak, peak_kind = measured_peak_gbs()
    a_bytes = None
    if a_bytes is None:
        a_bytes = (16 * samples + 24 * intervals) / 2
    achieved = a_bytes / (kern_ms * 1e-3) / 1e9
    step_bytes = 16 * samples + 24 * intervals + 32 * (2 * cfg.n_ops) + 32 * P
    line = {
        "metric": METRIC, "value": world * intervals / (ms_max / 1e3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: trace pair, {cfg.n_ops} ops and "
                               f"{cfg.n_samples} power samples per trace",
                   "method": args.method, "summation": args.summation, "overlap": args.overlap,
                   "intervals_per_pair": intervals,
                   "samples_per_pair": samples, "findings": P, "top_k": args.k,
                   "l2": (f"inputs (~{(16 * samples + 24 * intervals) / 1e9:.1f} GB/pair read per step) >> "
                          f"126 MB L2; no flush needed"),
                   "parallelism": f"pair-per-rank x{world}"},
        "samples_per_s": world * samples / (ms_max / 1e3),
        "attribution_ms": (t1 - t0) * 1e3, "diff_latency_ms": (t2 - t1) * 1e3,
        "step_hbm_fraction": (step_bytes / (ms_max * 1e-3) / 1e9) / peak,
        "roofline": {"bound": "hbm", "kernel": "attribute_tiles_kernel", "achieved": achieved,
                     "peak": peak, "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "bytes_per_launch": a_bytes, "launch_ms": kern_ms,
                     "traffic": profiled_traffic(args.config, args.method)},
        "e2e": e2e if e2e is not None else ({"skipped": e2e_skip} if e2e_skip else None),
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if world == 1:
        try:
            line["cpu_baseline"] = cpu_baseline(args)
        except Exception as exc:  # noqa: BLE001 - the baseline must not hide the GPU line
            line["cpu_baseline"] = {"error": repr(exc)}
        try:
            line["parity"] = (parity_record(args, dev) if args.overlap == "compat" else
                              {"skipped": "split ledgers: pinned to the oracle's dwo_split by tests/test_gpu_split.py"})
        except Exception as exc:  # noqa: BLE001
            line["parity"] = {"error": repr(exc), "pass": False}
    print(json.dumps(line), flush=True)


def run_window(args, rank: int, world: int, local: int):
    """Trace pairs time-window-sharded over the ranks: each
    rank attributes its window of both traces, crossing intervals and totals
    combine exactly, and the signature join runs hash-partitioned after one
    exchange.  Strong scaling: the work per step is fixed.  C4: one pair;
    C5: the corpus's pairs (as many as one GPU holds resident), each sharded
    over every rank."""
    import torch
    import torch.distributed as dist
    from dataclasses import replace

    from paper_2512_08365_b200 import _native, shard, synth

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _native.lib()
    kind = "linear" if args.method == "samples" else "step"
    comm = shard.Comm() if world > 1 else shard.LocalComm()
    cfg = synth.CONFIGS[args.config]
    n_pairs = args.pairs if args.config == "C5" else 1
    pairs = []
    for i in range(n_pairs):
        if pairs:
            free, _ = torch.cuda.mem_get_info(dev)
            per = torch.cuda.memory_allocated(dev) / len(pairs)
            if free < 16e9 + 1.0e9 * (len(pairs) + 1) + 1.1 * per:
                break
        ca, cb = synth.make_pair(replace(cfg, seed=cfg.seed + i) if n_pairs > 1 else cfg, dev)
        ia = shard.rank_inputs(ca, kind, shard.plan(ca.n_power, world, kind)[rank])
        ib = shard.rank_inputs(cb, kind, shard.plan(cb.n_power, world, kind)[rank])
        for c in (ca, cb):
            for n in ("op_sig", "op_start", "op_end"):
                c.device(n)
        pairs.append((ca, cb, ia, ib))
    n_res = torch.tensor([len(pairs)], device=dev if args.dist_backend == "nccl" else "cpu")
    if world > 1:  # every rank shards the same pairs
        dist.all_reduce(n_res, op=dist.ReduceOp.MIN)
    pairs = pairs[: int(n_res.item())]
    torch.cuda.synchronize()
    intervals = sum(a.n_ops + a.n_kernels + b.n_ops + b.n_kernels for a, b, _, _ in pairs)
    samples = sum(a.n_power + b.n_power for a, b, _, _ in pairs)

    def step():
        out = []
        for ca, cb, ia, ib in pairs:
            la = shard.sharded_ledger(ca, kind, comm, inputs=ia)
            lb = shard.sharded_ledger(cb, kind, comm, inputs=ib)
            out.append(shard.sharded_join(shard.shard_ops(ca, la, True), shard.shard_ops(cb, lb, False), ca.n_ops,
                                          comm, 0.10, args.k))
        return out

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    _native.launch_count(reset=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            res = step()
        e1.record()
        torch.cuda.synchronize()
    launches = _native.launch_count(reset=True)
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device="cuda" if args.dist_backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    if rank != 0:
        return
    what = (f"ONE trace pair, {cfg.n_ops} ops and {pairs[0][0].n_power} power samples per trace" if n_pairs == 1
            else f"{len(pairs)} of the corpus's {n_pairs} trace pairs ({cfg.n_ops} ops and {cfg.n_samples} power "
                 f"samples per trace), each")
    line = {
        "metric": METRIC, "value": intervals / (ms_max / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {what} time-window sharded", "method": args.method,
                   "pairs": len(pairs), "intervals_per_step": intervals, "findings": sum(r.P for r in res),
                   "top_k": args.k, "parallelism": f"time-window x{world} ({args.dist_backend})"},
        "samples_per_s": samples / (ms_max / 1e3),
        "gpu_launches": launches, "clocks": clocks.summary(),
        "n_waste": sum(r.n_waste for r in res), "wasted_joules": sum(r.wasted_joules for r in res),
    }
    print(json.dumps(line), flush=True)


def run_corpus(args, rank: int, world: int, local: int):
    """C5: a corpus of trace pairs (64 pairs, seeds 5000 + i,
    6.25M ops / 6.25e7 samples per trace).  Rank r owns the contiguous block of
    pairs [r * n / N, (r + 1) * n / N) (no data-path collective); a step is
    pipeline.analyze_corpus over the rank's resident pairs -- both ledgers and
    the join of every pair, ONE segmented top-k for all of them, the rank's
    corpus top-k -- plus, for N > 1, the corpus-wide top-k merged over NCCL.
    A rank holds its pairs resident in HBM while they fit (the whole 64-pair
    corpus is ~175 GB, so one B200 holds part of it: config names how many)."""
    import torch
    import torch.distributed as dist
    from dataclasses import replace

    from paper_2512_08365_b200 import _native, synth
    from paper_2512_08365_b200.columns import TraceColumns
    from paper_2512_08365_b200.dist import merge_topk
    from paper_2512_08365_b200.pipeline import analyze_corpus

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = _native.lib()
    base = synth.CONFIGS["C5"]
    n_total = args.pairs
    lo_p, hi_p = rank * n_total // world, (rank + 1) * n_total // world
    # HBM left after the resident pairs: analyze's transient workspaces
    # (~16 GB) + what each pair keeps until the segmented top-k (~1 GB: 32 B
    # per finding slot, the match / B-only columns, both ledgers' joules)
    pairs, ids = [], []
    for i in range(lo_p, hi_p):
        free, _ = torch.cuda.mem_get_info(dev)
        per = (torch.cuda.memory_allocated(dev) / len(pairs)) if pairs else 3.5e9
        if pairs and free < 16e9 + 1.0e9 * (len(pairs) + 1) + 1.1 * per:
            break
        ca, cb = synth.make_pair(replace(base, seed=base.seed + i), dev)
        for c in (ca, cb):
            for n in TraceColumns.HOT:
                c.device(n)
        pairs.append((ca, cb))
        ids.append(i)
    torch.cuda.synchronize()
    print(f"rank {rank}: {len(pairs)} of pairs {lo_p}..{hi_p - 1} resident, "
          f"{torch.cuda.memory_allocated(dev) / 1e9:.1f} GB allocated", file=sys.stderr, flush=True)
    intervals = sum(a.n_ops + a.n_kernels + b.n_ops + b.n_kernels for a, b in pairs)
    samples = sum(a.n_power + b.n_power for a, b in pairs)

    def step():
        res = analyze_corpus(pairs, args.method, 0.10, args.k, summation=args.summation)
        if world > 1:  # corpus-wide top-k: every rank's k candidates merged over NCCL
            hi, lo = [], []
            for p, f in res.top:
                jd = res.pairs[p].join
                ft = torch.tensor([f], dtype=torch.int64, device=dev)
                tie = jd.pair_of(ft)[0]
                if jd.columns.tie_rank is not None:
                    tie = torch.where(tie >= 0, jd.columns.tie_rank[tie.clamp(min=0)], tie)
                hi.append(jd.columns.key_hi[ft])
                lo.append(~(((tie + 1) << 32) | ft))
            if hi:
                merge_topk(torch.cat(hi), torch.cat(lo), args.k)
            else:
                e = torch.empty(0, dtype=torch.int64, device=dev)
                merge_topk(e, e, args.k)
        return res

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    L.dw_kernel_time_ms(1)
    L.dw_kernel_timed_count(1)
    L.dw_kernel_timing(1)
    _native.launch_count(reset=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            res = step()
        e1.record()
        torch.cuda.synchronize()
    L.dw_kernel_timing(0)
    launches = _native.launch_count(reset=True)
    n_timed = int(L.dw_kernel_timed_count(1))
    kern_ms = L.dw_kernel_time_ms(1) / max(n_timed, 1)
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms, float(intervals), float(samples), float(len(pairs))], device=dev, dtype=torch.float64)
    if world > 1:
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
    else:
        parts = [t]
    ms_max = max(float(x[0]) for x in parts)
    tot_iv = sum(float(x[1]) for x in parts)
    tot_s = sum(float(x[2]) for x in parts)
    resident = [int(x[3]) for x in parts]
    if rank != 0:
        return
    peak, peak_kind = measured_peak_gbs()
    a_bytes = (16 * samples + 24 * intervals) / (2 * len(pairs))  # one tile-kernel launch: one trace
    achieved = a_bytes / (kern_ms * 1e-3) / 1e9
    P = sum(ps.join.P for ps in res.pairs)
    line = {
        "metric": METRIC, "value": tot_iv / (ms_max / 1e3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"C5: corpus of {n_total} trace pairs ({base.n_ops} ops and {base.n_samples} "
                               f"power samples per trace), pair-sharded",
                   "pairs_per_rank_resident": resident, "pairs_timed": sum(resident),
                   "method": args.method, "summation": args.summation, "top_k_per_pair": args.k,
                   "findings_rank0": P,
                   "l2": "inputs (~2.7 GB per pair) >> 126 MB L2; no flush needed",
                   "parallelism": f"pair blocks x{world}; corpus top-k merged over NCCL"},
        "samples_per_s": tot_s / (ms_max / 1e3),
        "roofline": {"bound": "hbm", "kernel": "attribute_exact_kernel", "achieved": achieved,
                     "peak": peak, "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "bytes_per_launch": a_bytes, "launch_ms": kern_ms, "traffic": None},
        "e2e": {"skipped": "corpus mode times device-resident pairs only (the C4 line carries e2e)"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "n_waste_rank0": sum(ps.n_waste for ps in res.pairs),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.dist_backend == "gloo":  # (test setups: several ranks may share one GPU)
            local = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    try:
        if args.shard == "window":
            run_window(args, rank, world, local)
            return
        if args.config == "C5":
            run_corpus(args, rank, world, local)
            return
        run_ours(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
