"""The reference pipeline's stages at config 1, each through
this package on one B200: load (Python loader -- the trace carries tensor
snapshots), ground-truth ledgers, match_tensors, detect_waste with the
reference's pairs (bench_data/cfg1, scripts/ref_pairs_cfg1.py), report."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import build_ledger, detect_waste, match_tensors, report  # noqa: E402
from paper_2512_08365_b200.detect import SubgraphPair  # noqa: E402
from paper_2512_08365_b200.trace_model import load_trace  # noqa: E402


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return out, best


(ta, tb), t_load = timed(lambda: (load_trace("bench_data/cfg1/trace_a.jsonl"),
                                  load_trace("bench_data/cfg1/trace_b.jsonl")), 1)
(la, lb), t_led = timed(lambda: (build_ledger(ta), build_ledger(tb)))
_, t_match = timed(lambda: match_tensors(ta, tb))
pairs = [SubgraphPair(tuple(a), tuple(b), tuple(map(tuple, bl)), tuple(map(tuple, br)), d, c)
         for a, b, bl, br, d, c in json.load(open("bench_data/cfg1/ref_pairs.json"))]
fs, t_det = timed(lambda: detect_waste(pairs, la, lb, 0.10, trace_a=ta, trace_b=tb))
rep, t_rep = timed(lambda: report(fs, la, lb, 0.10))
print(json.dumps({"workload": "config 1 (chain 6700, seed 11): 10,142 ops + 15,239 kernels per trace",
                  "load_both_s": t_load, "ground_truth_ledgers_both_s": t_led, "match_tensors_s": t_match,
                  "detect_waste_s": t_det, "report_s": t_rep, "total_a": la.total_joules,
                  "total_b": lb.total_joules, "wasted_joules": rep.wasted_joules,
                  "reference_s": {"ledgers_both": 631, "build_graph+match_tensors": 125, "recursive_match": 16,
                                  "detect_waste": 6.65, "report": 0.01, "source": "BASELINE.md 2 (one core)"}}))
