import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_2512_08365_b200 import tensor_match as tm  # noqa: E402
from paper_2512_08365_b200.trace_model import load_trace  # noqa: E402

ta = load_trace("bench_data/cfg1/trace_a.jsonl")
tb = load_trace("bench_data/cfg1/trace_b.jsonl")
tm.match_tensors(ta, tb)
pr = cProfile.Profile()
pr.enable()
tm.match_tensors(ta, tb)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
