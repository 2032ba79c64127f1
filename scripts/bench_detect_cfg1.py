"""detect_waste (device per-pair arithmetic + batched classification) on the
config-1 scenario with the reference's own pairs (bench_data/cfg1, made by
scripts/ref_pairs_cfg1.py), against the reference's findings and time."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import build_ledger, detect_waste  # noqa: E402
from paper_2512_08365_b200.detect import SubgraphPair  # noqa: E402
from paper_2512_08365_b200.trace_model import load_trace  # noqa: E402

ta = load_trace("bench_data/cfg1/trace_a.jsonl")
tb = load_trace("bench_data/cfg1/trace_b.jsonl")
pairs = [SubgraphPair(tuple(a), tuple(b), tuple(map(tuple, bl)), tuple(map(tuple, br)), d, c)
         for a, b, bl, br, d, c in json.load(open("bench_data/cfg1/ref_pairs.json"))]
ref = json.load(open("bench_data/cfg1/ref_detect.json"))
la, lb = build_ledger(ta, "sampled"), build_ledger(tb, "sampled")
times = []
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fs = detect_waste(pairs, la, lb, 0.10, trace_a=ta, trace_b=tb)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t)
got = [[f.verdict, f.category, f.wasteful_side, f.wasted_joules] for f in fs]
same = got == ref["findings"]
print(json.dumps({"pairs": len(pairs), "detect_s": times, "reference_detect_s": ref["detect_s"],
                  "identical_findings": same,
                  "mismatches": sum(1 for x, y in zip(got, ref["findings"]) if x != y)}))
