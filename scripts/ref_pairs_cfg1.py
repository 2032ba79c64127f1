"""Record the reference's recursive_match pairs (with boundaries) and its
detect_waste time on the config-1 scenario (here, CPU) for
scripts/bench_detect_cfg1.py."""
import json
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import diffwatt.detect as detect  # noqa: E402
import diffwatt.energy as energy  # noqa: E402
import diffwatt.graph as graph  # noqa: E402
import diffwatt.subgraph_match as sm  # noqa: E402
import diffwatt.trace_model as tmod  # noqa: E402

ta, tb = tmod.load_trace("bench_data/cfg1/trace_a.jsonl"), tmod.load_trace("bench_data/cfg1/trace_b.jsonl")
ga, gb = graph.build_graph(ta), graph.build_graph(tb)
eq, _ = sm.match_tensors(ga, gb)
res = sm.recursive_match(ga, gb, eq)
json.dump([[list(p.nodes_a), list(p.nodes_b), [list(x) for x in p.boundary_left],
            [list(x) for x in p.boundary_right], p.depth, p.coarse] for p in res.pairs],
          open("bench_data/cfg1/ref_pairs.json", "w"))
# detect_waste needs ledgers; the ground-truth ledgers take ~10 min here, so
# time detect_waste on the sampled ledgers (same code path after the ledger)
la, lb = energy.build_ledger(ta, "sampled"), energy.build_ledger(tb, "sampled")
t = time.perf_counter()
fs = detect.detect_waste(res.pairs, la, lb, 0.10, trace_a=ta, trace_b=tb)
dt = time.perf_counter() - t
json.dump({"detect_s": dt, "findings": [[f.verdict, f.category, f.wasteful_side, f.wasted_joules] for f in fs]},
          open("bench_data/cfg1/ref_detect.json", "w"))
print(f"pairs {len(res.pairs)} detect_waste {dt:.2f}s")
