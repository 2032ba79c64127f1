"""Generate golden vectors from the reference package (test infrastructure).

Runs ONLY in the build container, where the read-only reference lives at
/root/reference/pkg/src.  It imports the reference ``diffwatt`` package and
records its outputs on seeded inputs into small fixtures under tests/golden/:

* ``integrate_step.npz``   - random step signals + intervals -> reference
                             ``energy.integrate`` joules (src/energy.py:90-104)
* ``integrate_linear.npz`` - random sample sets + intervals -> reference
                             ``energy._integrate_samples`` (src/energy.py:108-130)
* ``replay.npz``           - reference ``build_ledger(method="replay")``
                             (src/energy.py:196-256, 306-311) on the sampler
                             demo trace and presets, several sampler settings
* ``scenarios/*.npz``      - simulator presets + fuzz/null corpora: SoA columns
                             of both traces, reference ledgers
                             (src/energy.py:280-331), reference segment pairs
                             (src/subgraph_match.py:322-422), ``detect_waste``
                             findings (src/detect.py:72-130) and ``report``
                             ranking (src/detect.py:256-278).

Nothing on the GPU box reads /root/reference: the fixtures are committed and
this script is the recipe that made them.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import os
import sys
import time
import types
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def _import_reference():
    # cli/figures need matplotlib, which is absent; the hot-path modules do not.
    sys.path.insert(0, REF_SRC)
    import diffwatt.detect as detect
    import diffwatt.energy as energy
    import diffwatt.graph as graph
    import diffwatt.simulate as simulate
    import diffwatt.subgraph_match as sm
    import diffwatt.trace_model as tm

    return types.SimpleNamespace(
        detect=detect, energy=energy, graph=graph, simulate=simulate, sm=sm, tm=tm
    )


VERDICT_CODE = {"below_threshold": 0, "tradeoff": 1, "waste": 2}
SIDE_CODE = {"-": 0, "A": 1, "B": 2}


def trace_columns(ref, trace, prefix):
    """Reference Trace -> SoA columns (ops in trace order, kernels flattened in
    op.kernel_ids order, power in record order)."""
    truth = ref.energy.ground_truth_signal(trace)
    span_lo, span_hi = truth.span()
    ops = trace.operators
    k_ids, k_start, k_end, k_op = [], [], [], []
    for i, op in enumerate(ops):
        for kid in op.kernel_ids:
            k = trace.kernels[kid]
            k_ids.append(kid)
            k_start.append(k.start)
            k_end.append(k.end)
            k_op.append(i)
    return {
        f"{prefix}_ts": np.array([p.timestamp for p in trace.power], dtype=np.int64),
        f"{prefix}_watts": np.array([p.watts for p in trace.power], dtype=np.float64),
        f"{prefix}_span": np.array([span_lo, span_hi], dtype=np.int64),
        f"{prefix}_op_start": np.array([o.start for o in ops], dtype=np.int64),
        f"{prefix}_op_end": np.array([o.end for o in ops], dtype=np.int64),
        f"{prefix}_op_ids": np.array([o.op_id for o in ops]),
        f"{prefix}_op_names": np.array([o.op_name for o in ops]),
        f"{prefix}_k_start": np.array(k_start, dtype=np.int64),
        f"{prefix}_k_end": np.array(k_end, dtype=np.int64),
        f"{prefix}_k_op": np.array(k_op, dtype=np.int32),
        f"{prefix}_k_ids": np.array(k_ids if k_ids else [""])[: len(k_ids)],
    }


def ledger_columns(trace, ledger, prefix):
    ops = trace.operators
    kids = [kid for op in ops for kid in op.kernel_ids]
    return {
        f"{prefix}_per_op": np.array([ledger.per_operator[o.op_id] for o in ops]),
        f"{prefix}_per_k": np.array([ledger.per_kernel[k] for k in kids], dtype=np.float64),
        f"{prefix}_total_idle": np.array([ledger.total_joules, ledger.idle_joules]),
    }


def sampled_columns(ref, trace, prefix, period, delay, seed):
    view = ref.energy.sampled_view(trace, period, delay, seed)
    return {
        f"{prefix}_ts": np.array([s.timestamp for s in view.samples], dtype=np.int64),
        f"{prefix}_watts": np.array([s.watts for s in view.samples], dtype=np.float64),
    }


def scenario_record(ref, manifest, name, sampled=True):
    t0 = time.time()
    ta, tb, truth = ref.simulate.generate(manifest)
    rec = {}
    rec.update(trace_columns(ref, ta, "a"))
    rec.update(trace_columns(ref, tb, "b"))
    la = ref.energy.build_ledger(ta)
    lb = ref.energy.build_ledger(tb)
    rec.update(ledger_columns(ta, la, "gt_a"))
    rec.update(ledger_columns(tb, lb, "gt_b"))
    if sampled:
        # default sampler (25 Hz, 200 ms delay, seed 0) and a 1 kHz zero-delay view
        for tag, period, delay in (("s40", 40_000, 200_000), ("s1", 1_000, 0)):
            for side, tr in (("a", ta), ("b", tb)):
                led = ref.energy.build_ledger(tr, method="sampled", period_us=period,
                                              delay_us=delay, seed=0)
                rec.update(ledger_columns(tr, led, f"{tag}_{side}"))
                rec.update(sampled_columns(ref, tr, f"{tag}_{side}_view", period, delay, 0))

    # reference pairing -> CSR over op indices
    g_a, g_b = ref.graph.build_graph(ta), ref.graph.build_graph(tb)
    eq, _ = ref.sm.match_tensors(g_a, g_b)
    res = ref.sm.recursive_match(g_a, g_b, eq)
    idx_a = {o.op_id: i for i, o in enumerate(ta.operators)}
    idx_b = {o.op_id: i for i, o in enumerate(tb.operators)}
    off_a, mem_a, off_b, mem_b = [0], [], [0], []
    out_diff = []
    for p in res.pairs:
        mem_a += [idx_a[o] for o in p.nodes_a]
        mem_b += [idx_b[o] for o in p.nodes_b]
        off_a.append(len(mem_a))
        off_b.append(len(mem_b))
        out_diff.append(ref.detect._boundary_rel_diff(p, ta, tb))
    rec["pair_off_a"] = np.array(off_a, dtype=np.int64)
    rec["pair_mem_a"] = np.array(mem_a, dtype=np.int32)
    rec["pair_off_b"] = np.array(off_b, dtype=np.int64)
    rec["pair_mem_b"] = np.array(mem_b, dtype=np.int32)
    rec["pair_out_diff"] = np.array(out_diff, dtype=np.float64)

    for theta in (0.10, 0.05):
        tag = f"det{int(round(theta * 100)):02d}"
        fs = ref.detect.detect_waste(res.pairs, la, lb, theta, trace_a=ta, trace_b=tb)
        rec[f"{tag}_energy"] = np.array([[f.energy_a, f.energy_b] for f in fs]).reshape(-1, 2)
        rec[f"{tag}_ratio"] = np.array([f.energy_ratio for f in fs], dtype=np.float64)
        rec[f"{tag}_lat"] = np.array([[f.latency_a, f.latency_b] for f in fs],
                                     dtype=np.int64).reshape(-1, 2)
        rec[f"{tag}_verdict"] = np.array([VERDICT_CODE[f.verdict] for f in fs], dtype=np.int8)
        rec[f"{tag}_side"] = np.array([SIDE_CODE[f.wasteful_side] for f in fs], dtype=np.int8)
        rec[f"{tag}_wasted"] = np.array([f.wasted_joules for f in fs], dtype=np.float64)
        rec[f"{tag}_info"] = np.array([f.informational for f in fs], dtype=np.bool_)
        rec[f"{tag}_category"] = np.array([f.category for f in fs] or [""])[: len(fs)]
        doc = ref.detect.report(fs, la, lb, theta)
        pos = {id(f): i for i, f in enumerate(fs)}
        rec[f"{tag}_rank"] = np.array([pos[id(f)] for f in doc.findings], dtype=np.int64)
        rec[f"{tag}_report"] = np.array(
            [doc.total_a, doc.total_b, doc.wasted_joules, doc.end_to_end_waste_pct]
        )
    rec["truth_waste_fraction"] = np.array([truth.end_to_end_waste_fraction])
    print(f"  {name}: {len(ta.operators)}/{len(tb.operators)} ops, "
          f"{len(ta.power)}/{len(tb.power)} power, {len(res.pairs)} pairs "
          f"[{time.time() - t0:.1f}s]", flush=True)
    return rec


def integrate_step_vectors(ref, seed=20260808, n_signals=24):
    """Random step signals, including long ones (thousands of segments) and
    intervals on and between breakpoints, zero-length and whole-span ones."""
    rng = np.random.default_rng(seed)
    PS = ref.energy.PowerSignal
    out = {"sig_off": [0], "ts": [], "watts": [], "span": [], "iv_off": [0], "lo": [], "hi": [],
           "joules": []}
    for s in range(n_signals):
        nseg = int(rng.choice([1, 2, 5, 12, 40, 300, 2500]))
        widths = rng.integers(1, 4000, size=nseg)
        if s % 3 == 0:
            widths = rng.integers(1, 6, size=nseg)  # dense breakpoints
        start = int(rng.integers(0, 10_000))
        bps = start + np.concatenate([[0], np.cumsum(widths)])
        watts = rng.uniform(0.0, 700.0, size=nseg)
        if s % 5 == 0:
            watts = np.round(watts, 1)
        segs = tuple((int(bps[i]), int(bps[i + 1]), float(watts[i])) for i in range(nseg))
        sig = PS(segments=segs)
        lo_s, hi_s = sig.span()
        ivs = []
        for _ in range(int(rng.integers(20, 60))):
            a, b = sorted(int(x) for x in rng.integers(lo_s, hi_s + 1, size=2))
            ivs.append((a, b))
        ivs += [(lo_s, hi_s), (lo_s, lo_s), (hi_s, hi_s)]
        for i in range(min(nseg, 8)):  # intervals aligned to breakpoints
            ivs.append((int(bps[i]), int(bps[min(nseg, i + 1 + int(rng.integers(0, 3)))])))
        for lo, hi in ivs:
            out["lo"].append(lo)
            out["hi"].append(hi)
            out["joules"].append(ref.energy.integrate(sig, (lo, hi)))
        out["ts"] += [int(x) for x in bps[:-1]]
        out["watts"] += [float(w) for w in watts]
        out["span"] += [lo_s, hi_s]
        out["sig_off"].append(len(out["ts"]))
        out["iv_off"].append(len(out["lo"]))
    return {
        "sig_off": np.array(out["sig_off"], dtype=np.int64),
        "ts": np.array(out["ts"], dtype=np.int64),
        "watts": np.array(out["watts"], dtype=np.float64),
        "span": np.array(out["span"], dtype=np.int64).reshape(-1, 2),
        "iv_off": np.array(out["iv_off"], dtype=np.int64),
        "lo": np.array(out["lo"], dtype=np.int64),
        "hi": np.array(out["hi"], dtype=np.int64),
        "joules": np.array(out["joules"], dtype=np.float64),
    }


def integrate_linear_vectors(ref, seed=20260809, n_signals=24):
    rng = np.random.default_rng(seed)
    PS = ref.energy.PowerSignal
    PSm = ref.tm.PowerSample
    out = {"sig_off": [0], "ts": [], "watts": [], "iv_off": [0], "lo": [], "hi": [], "joules": []}
    for s in range(n_signals):
        n = int(rng.choice([1, 2, 3, 10, 50, 400, 1500]))
        gaps = rng.integers(1, 3000, size=max(n - 1, 0))
        if s % 3 == 0:
            gaps = rng.integers(1, 4, size=max(n - 1, 0))
        t0 = int(rng.integers(0, 10_000))
        ts = t0 + np.concatenate([[0], np.cumsum(gaps)]).astype(np.int64)
        watts = rng.uniform(50.0, 700.0, size=n)
        samples = tuple(PSm(timestamp=int(t), watts=float(w)) for t, w in zip(ts, watts))
        sig = PS(samples=samples, period_us=1000, delay_us=0)
        lo_s, hi_s = sig.span()
        ivs = []
        for _ in range(int(rng.integers(20, 50))):
            a, b = sorted(int(x) for x in rng.integers(lo_s, hi_s + 1, size=2))
            ivs.append((a, b))
        ivs += [(lo_s, hi_s), (lo_s, lo_s), (hi_s, hi_s)]
        for i in range(min(n - 1, 8)):
            ivs.append((int(ts[i]), int(ts[min(n - 1, i + 1 + int(rng.integers(0, 3)))])))
        for lo, hi in ivs:
            out["lo"].append(lo)
            out["hi"].append(hi)
            out["joules"].append(ref.energy.integrate(sig, (lo, hi)))
        out["ts"] += [int(x) for x in ts]
        out["watts"] += [float(w) for w in watts]
        out["sig_off"].append(len(out["ts"]))
        out["iv_off"].append(len(out["lo"]))
    return {k: np.array(v, dtype=np.float64 if k in ("watts", "joules") else np.int64)
            for k, v in out.items()}


def error_vectors(ref):
    """Reference error messages for the SignalError / ValueError conventions."""
    PS = ref.energy.PowerSignal
    sig = PS(segments=((10, 100, 50.0), (100, 150, 70.0)))
    msgs = {}
    for name, iv in (("outside_lo", (0, 100)), ("outside_hi", (20, 151)),
                     ("reversed", (60, 50))):
        try:
            ref.energy.integrate(sig, iv)
        except ref.energy.SignalError as exc:
            msgs[name] = str(exc)
    try:
        PS().span()
    except ref.energy.SignalError as exc:
        msgs["empty"] = str(exc)
    try:
        PS.from_breakpoints((), 10)
    except ref.energy.SignalError as exc:
        msgs["no_power"] = str(exc)
    return msgs


def cfg1_record(ref):
    """BASELINE config 1: chain length 6700, seed 11, misconfig on segment 3
    (SURVEY.md 8(d) C1).  Ground-truth ledgers in full (~5 min/side in the
    reference); the 1 kHz sampled view in full, with reference joules for the
    first 500 operator and 500 kernel intervals (the full sampled ledger is
    ~45 min/side)."""
    sim = ref.simulate
    m = sim.ScenarioManifest(
        workload="cfg1", seed=11, template="chain", length=6700,
        inefficiency=sim.Inefficiency("misconfiguration", 3, 0.3, "matmul.allow_tf32"))
    rec = scenario_record(ref, m, "cfg1", sampled=False)
    ta, tb, _ = sim.generate(m)
    for side, tr in (("a", ta), ("b", tb)):
        view = ref.energy.sampled_view(tr, 1_000, 0, 0)
        rec[f"s1_{side}_view_ts"] = np.array([s.timestamp for s in view.samples], dtype=np.int64)
        rec[f"s1_{side}_view_watts"] = np.array([s.watts for s in view.samples])
        ops = tr.operators[:500]
        kids = [k for op in tr.operators for k in op.kernel_ids][:500]
        rec[f"s1_{side}_per_op500"] = np.array(
            [ref.energy.integrate(view, (o.start, o.end)) for o in ops])
        rec[f"s1_{side}_per_k500"] = np.array(
            [ref.energy.integrate(view, (tr.kernels[k].start, tr.kernels[k].end)) for k in kids])
    return rec


def trace_vectors(ref):
    """JSONL trace files written by the reference, its canonical re-emission,
    and the reference's exceptions for malformed inputs (trace_model.py:341-586)."""
    tdir = OUT / "traces"
    tdir.mkdir(exist_ok=True)
    sim, tm = ref.simulate, ref.tm
    for name in ("tf32_misconfig", "join_redundant"):
        pa, pb = sim.write_scenario(sim.preset(name), str(tdir / name))
        for path in (pa, pb):
            tr = tm.load_trace(path)
            with open(path + ".canonical", "w") as fh:
                fh.write("\n".join(tm.trace_to_lines(tr)) + "\n")
    good = open(tdir / "tf32_misconfig" / "trace_a.jsonl").read().splitlines()
    header = good[0]
    op = next(l for l in good if '"type":"op"' in l)
    cases = {
        "empty": [],
        "no_header": [op],
        "bad_json": [header, "{not json"],
        "bad_version": ['{"type":"header","schema_version":2,"system":"x","workload":"w","seed":0}'],
        "dup_header": [header, header],
        "unknown_type": [header, '{"type":"bogus"}'],
        "missing_field": [header, '{"type":"power","timestamp":5}'],
        "non_int": [header, '{"type":"power","timestamp":5.5,"watts":1.0}'],
        "neg_watts": [header, '{"type":"power","timestamp":5,"watts":-1.0}'],
        "power_order": [header, '{"type":"power","timestamp":5,"watts":1.0}',
                        '{"type":"power","timestamp":5,"watts":2.0}'],
        "op_end_lt_start": [header, '{"type":"op","op_id":"o","op_name":"n","input_tensor_ids":[],'
                            '"output_tensor_ids":[],"kernel_ids":[],"start":10,"end":5}'],
        "dup_op": [header] + ['{"type":"op","op_id":"o","op_name":"n","input_tensor_ids":[],'
                              '"output_tensor_ids":[],"kernel_ids":[],"start":1,"end":5}'] * 2,
        "missing_kernel": [header, '{"type":"op","op_id":"o","op_name":"n","input_tensor_ids":[],'
                           '"output_tensor_ids":[],"kernel_ids":["k"],"start":1,"end":5}'],
        "kernel_outside": [header, '{"type":"op","op_id":"o","op_name":"n","input_tensor_ids":[],'
                           '"output_tensor_ids":[],"kernel_ids":["k"],"start":1,"end":5}',
                           '{"type":"kernel","kernel_id":"k","kernel_name":"kn","correlation_id":1,'
                           '"start":2,"end":9,"backtrace":["a"]}'],
        "orphan_kernel": [header, '{"type":"kernel","kernel_id":"k","kernel_name":"kn","correlation_id":1,'
                          '"start":2,"end":9,"backtrace":["a"]}'],
        "kernel_zero_len": [header, '{"type":"kernel","kernel_id":"k","kernel_name":"kn","correlation_id":1,'
                            '"start":2,"end":2,"backtrace":["a"]}'],
        "missing_tensor": [header, '{"type":"op","op_id":"o","op_name":"n","input_tensor_ids":["t"],'
                           '"output_tensor_ids":[],"kernel_ids":[],"start":1,"end":5}'],
        "cycle": [header,
                  '{"type":"tensor","tensor_id":"t1","run":0,"shape":[1],"values":[1.0]}',
                  '{"type":"tensor","tensor_id":"t2","run":0,"shape":[1],"values":[1.0]}',
                  '{"type":"op","op_id":"a","op_name":"n","input_tensor_ids":["t2"],'
                  '"output_tensor_ids":["t1"],"kernel_ids":[],"start":1,"end":5}',
                  '{"type":"op","op_id":"b","op_name":"n","input_tensor_ids":["t1"],'
                  '"output_tensor_ids":["t2"],"kernel_ids":[],"start":1,"end":5}'],
    }
    out = {}
    for name, lines in cases.items():
        try:
            tm.parse_trace_lines(lines)
            out[name] = {"lines": lines, "exc": None, "msg": None}
        except Exception as exc:  # noqa: BLE001 - record what the reference raises
            out[name] = {"lines": lines, "exc": type(exc).__name__, "msg": str(exc)}
    with open(tdir / "errors.json", "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def replay_vectors(ref):
    """Reference build_ledger(method="replay") (src/energy.py:196-256, 306-311)
    on the sampler demo trace and the presets, for several sampler settings:
    SoA columns + per-op / per-kernel joules + total / idle."""
    out = {}
    cases = [("demo", ref.simulate.sampler_demo_traces()[0])]
    for preset in ("tf32_misconfig", "join_redundant", "attention_block"):
        cases.append((preset, ref.simulate.generate(ref.simulate.preset(preset))[0]))
    for i, m in enumerate(ref.simulate.fuzz(20260808, 4)):
        cases.append((f"fuzz{i}", ref.simulate.generate(m)[1]))
    settings = [("d", dict()), ("s2r100", dict(seed=2, repeat=100)),
                ("nodelay", dict(delay_us=0, period_us=5000, repeat=50)),
                ("fast", dict(period_us=1000, delay_us=300, repeat=7, seed=5))]
    names = []
    for name, tr in cases:
        out.update(trace_columns(ref, tr, name))
        for tag, kw in settings:
            led = ref.energy.build_ledger(tr, method="replay", **kw)
            out.update(ledger_columns(tr, led, f"{name}_{tag}"))
            names.append(f"{name}:{tag}")
    out["cases"] = np.array([c[0] for c in cases])
    out["settings"] = np.array(json.dumps(settings))
    return out


def classify_vectors(ref):
    """Reference detect.classify (src/detect.py:137-172), which detect_waste
    applies to every waste finding (:127-128), on the presets and a fuzz
    corpus: the two traces as JSONL lines (the reference's own writer) and,
    per finding in detect_waste order, (nodes_a, nodes_b, verdict, side,
    category, forced_gap_joules of the wasteful side)."""
    import tempfile

    import diffwatt.diagnose as dg

    def gaps(f, ta, tb):  # forced_gap_joules of the wasteful side (diagnose.py:372-387)
        if f.verdict != "waste":
            return None
        tr, nodes = (ta, f.pair.nodes_a) if f.wasteful_side == "A" else (tb, f.pair.nodes_b)
        return dg.forced_gap_joules(tr, list(nodes))

    sim = ref.simulate
    cases = [(p, sim.preset(p)) for p in ("tf32_misconfig", "join_redundant", "fused_api_misuse",
                                           "layout_null", "attention_block")]
    cases += [(f"fuzz_{i:03d}", m) for i, m in enumerate(sim.fuzz(20260808, 120))]
    out = {}
    tmp = Path(tempfile.mkdtemp())
    for name, manifest in cases:
        pa, pb = sim.write_scenario(manifest, str(tmp / name))
        ta, tb = ref.tm.load_trace(pa), ref.tm.load_trace(pb)
        la, lb = ref.energy.build_ledger(ta), ref.energy.build_ledger(tb)
        g_a, g_b = ref.graph.build_graph(ta), ref.graph.build_graph(tb)
        eq, _ = ref.sm.match_tensors(g_a, g_b)
        res = ref.sm.recursive_match(g_a, g_b, eq)
        fs = ref.detect.detect_waste(res.pairs, la, lb, 0.10, trace_a=ta, trace_b=tb)
        out[name] = {
            "a": open(pa).read().splitlines(), "b": open(pb).read().splitlines(),
            "findings": [[list(f.pair.nodes_a), list(f.pair.nodes_b), f.verdict, f.wasteful_side,
                          f.category, gaps(f, ta, tb)] for f in fs],
        }
    return out


def tensor_vectors(ref):
    """Reference match_tensors (subgraph_match.py:109-204) on the classify
    corpus (traces in classify.json.gz) and reference invariant sets
    (tensor_equiv.py:162-180) of seeded random tensors."""
    import gzip

    import diffwatt.tensor_equiv as te

    with gzip.open(OUT / "classify.json.gz", "rt") as fh:
        corpus = json.load(fh)
    import tempfile
    tmp = Path(tempfile.mkdtemp())
    extra = {}
    sim = ref.simulate
    for name, m in (("big_chain", sim.ScenarioManifest(workload="big", seed=77, template="chain", length=120)),
                    ("big_transformer", sim.ScenarioManifest(workload="big", seed=78, template="transformer",
                                                             length=3))):
        pa, pb = sim.write_scenario(m, str(tmp / name))
        extra[name] = {"a": open(pa).read().splitlines(), "b": open(pb).read().splitlines()}
    match = {}
    for name, c in list(corpus.items()) + list(extra.items()):
        ta, tb = ref.tm.parse_trace_lines(c["a"]), ref.tm.parse_trace_lines(c["b"])
        ga, gb = ref.graph.build_graph(ta), ref.graph.build_graph(tb)
        pairs, st = ref.sm.match_tensors(ga, gb)
        match[name] = {"pairs": [[p.tensor_a, p.tensor_b, p.score] for p in pairs.pairs],
                       "candidate_pairs": st.candidate_pairs, "full_checks": st.full_checks}
    rng = np.random.default_rng(20261017)
    shapes = [(3, 4), (7, 2), (5, 5), (1, 6), (16, 16), (40, 3), (2, 3, 4), (4, 4, 5), (2, 2, 2, 2),
              (3, 1, 5), (2, 3, 2, 3, 2), (6, 7, 8), (64, 33), (2, 2, 2, 2, 2, 2)]
    tensors, spectra = [], []
    for i, shp in enumerate(shapes):
        x = rng.standard_normal(shp)
        if i % 3 == 1:  # rank-deficient: an outer product
            x = np.multiply.outer(rng.standard_normal(shp[0]), rng.standard_normal(shp[1:]))
        if i % 4 == 2:
            x = x * 1e-7
        tensors.append(x)
        inv = te.invariant_set(x)
        spectra.append([list(s.singulars) for s in inv.spectra])
    return match, extra, {"shapes": [list(s) for s in shapes], "values": [t.ravel().tolist() for t in tensors],
                          "spectra": spectra}


def main():
    ref = _import_reference()
    if "--tensors" in sys.argv:
        import gzip
        t0 = time.time()
        match, extra, spec = tensor_vectors(ref)
        with gzip.open(OUT / "tensors.json.gz", "wt") as fh:
            json.dump({"match": match, "traces": extra, "random": spec}, fh, sort_keys=True)
        print(f"tensors done [{time.time() - t0:.1f}s]")
        return
    if "--classify" in sys.argv:
        t0 = time.time()
        import gzip
        with gzip.open(OUT / "classify.json.gz", "wt") as fh:
            json.dump(classify_vectors(ref), fh, sort_keys=True)
        print(f"classify done [{time.time() - t0:.1f}s]")
        return
    if "--replay" in sys.argv:
        t0 = time.time()
        np.savez_compressed(OUT / "replay.npz", **replay_vectors(ref))
        print(f"replay done [{time.time() - t0:.1f}s]")
        return
    if "--traces" in sys.argv:
        trace_vectors(ref)
        return
    if "--cfg1" in sys.argv:
        t0 = time.time()
        (OUT / "scenarios").mkdir(parents=True, exist_ok=True)
        np.savez_compressed(OUT / "scenarios" / "cfg1.npz", **cfg1_record(ref))
        print(f"cfg1 done [{time.time() - t0:.1f}s]")
        return
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / "scenarios").mkdir(exist_ok=True)
    t0 = time.time()
    np.savez_compressed(OUT / "integrate_step.npz", **integrate_step_vectors(ref))
    np.savez_compressed(OUT / "integrate_linear.npz", **integrate_linear_vectors(ref))
    print(f"integrate vectors [{time.time() - t0:.1f}s]", flush=True)
    with open(OUT / "errors.json", "w") as fh:
        json.dump(error_vectors(ref), fh, indent=1, sort_keys=True)

    names = []
    sim = ref.simulate
    for preset in ("tf32_misconfig", "join_redundant", "fused_api_misuse", "layout_null",
                   "attention_block"):
        rec = scenario_record(ref, sim.preset(preset), preset)
        np.savez_compressed(OUT / "scenarios" / f"preset_{preset}.npz", **rec)
        names.append(f"preset_{preset}")
    for i, m in enumerate(sim.fuzz(20260808, 50)):
        rec = scenario_record(ref, m, f"fuzz{i}", sampled=(i % 5 == 0))
        np.savez_compressed(OUT / "scenarios" / f"fuzz_{i:02d}.npz", **rec)
        names.append(f"fuzz_{i:02d}")
    for i, m in enumerate(sim.null_corpus(20260808, 10)):
        rec = scenario_record(ref, m, f"null{i}", sampled=(i % 5 == 0))
        np.savez_compressed(OUT / "scenarios" / f"null_{i:02d}.npz", **rec)
        names.append(f"null_{i:02d}")
    with open(OUT / "scenarios" / "index.json", "w") as fh:
        json.dump({"scenarios": names, "numpy": np.__version__,
                   "generator": "tests/golden/make_golden.py"}, fh, indent=1)
    print(f"done [{time.time() - t0:.1f}s]")


if __name__ == "__main__":
    main()
