"""match_tensors at config-1 scale on the device (csrc/tensor.cu), against the
reference's result recorded here (bench_data/cfg1/ref_match.json, made by
scripts/ref_match_time.py).  Prints one JSON line with phase times."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import _native  # noqa: E402
from paper_2512_08365_b200 import tensor_match as tm  # noqa: E402
from paper_2512_08365_b200.trace_model import load_trace  # noqa: E402

ta = load_trace("bench_data/cfg1/trace_a.jsonl")
tb = load_trace("bench_data/cfg1/trace_b.jsonl")
ref = json.load(open("bench_data/cfg1/ref_match.json"))
times = []
for it in range(4):
    torch.cuda.synchronize()
    _native.lib().dw_launch_count(1)
    t = time.perf_counter()
    pairs, st = tm.match_tensors(ta, tb)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t)
launches = int(_native.lib().dw_launch_count(0))
same = [(p.tensor_a, p.tensor_b) for p in pairs.pairs] == [(a, b) for a, b, _ in ref["pairs"]]
worst = max((abs(p.score - s) for p, (_, _, s) in zip(pairs.pairs, ref["pairs"])), default=0.0)
# phase split of one call
t0 = time.perf_counter()
A, B = tm._GraphView(ta), tm._GraphView(tb)
t1 = time.perf_counter()
runs = max(min(ta.run_count, tb.run_count), 1)
sa, va, oa = tm._pack(ta, A.ids, runs)
sb, vb, ob = tm._pack(tb, B.ids, runs)
t2 = time.perf_counter()
from paper_2512_08365_b200.tensor_equiv import invariant_sets  # noqa: E402
torch.cuda.synchronize()
t3 = time.perf_counter()
inv = invariant_sets([s for s in sa if len(s.shape) > 1])
torch.cuda.synchronize()
t4 = time.perf_counter()
print(json.dumps({"workload": "config-1 scenario (reference simulator, chain 6700 segments)",
                  "tensors": [len(A.ids), len(B.ids)], "runs": runs, "candidate_pairs": st.candidate_pairs,
                  "full_checks": st.full_checks, "pairs": len(pairs), "same_pairs_as_reference": same,
                  "max_score_diff": worst, "ref_stats_equal": [st.candidate_pairs == ref["candidate_pairs"],
                                                               st.full_checks == ref["full_checks"]],
                  "match_s": times, "reference_match_s": ref["match_s"], "launches_per_call": launches // 4,
                  "phase_s": {"graph_view": t1 - t0, "pack": t2 - t1, "spectra_side_a": t4 - t3,
                              "unfoldings_side_a": sum(len(i.spectra) for i in inv)}}))
