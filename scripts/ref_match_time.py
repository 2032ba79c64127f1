"""Time the reference's match_tensors on the config-1 scenario (here, CPU)."""
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import diffwatt.graph as graph  # noqa: E402
import diffwatt.subgraph_match as sm  # noqa: E402
import diffwatt.trace_model as tmod  # noqa: E402

ta, tb = tmod.load_trace("bench_data/cfg1/trace_a.jsonl"), tmod.load_trace("bench_data/cfg1/trace_b.jsonl")
t = time.perf_counter()
ga, gb = graph.build_graph(ta), graph.build_graph(tb)
t1 = time.perf_counter()
pairs, st = sm.match_tensors(ga, gb)
t2 = time.perf_counter()
print(f"tensors {len(ta.tensors)}/{len(tb.tensors)} runs {ta.run_count}; build_graph {t1 - t:.1f}s "
      f"match_tensors {t2 - t1:.1f}s pairs {len(pairs)} {st}")
import json  # noqa: E402
json.dump({"pairs": [[p.tensor_a, p.tensor_b, p.score] for p in pairs.pairs], "candidate_pairs": st.candidate_pairs,
           "full_checks": st.full_checks, "match_s": t2 - t1}, open("bench_data/cfg1/ref_match.json", "w"))
