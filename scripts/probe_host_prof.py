"""cProfile of one C4 analyze() step (after warm-up): the host-side Python
cost between the library's launches."""
import cProfile, pstats, sys
import torch
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth
from paper_2512_08365_b200.pipeline import analyze
from paper_2512_08365_b200.columns import TraceColumns
a, b = synth.make_pair(sys.argv[1] if len(sys.argv) > 1 else "C4")
for c in (a, b):
    for n in TraceColumns.HOT:
        c.device(n)
for _ in range(3):
    analyze(a, b)
torch.cuda.synchronize()
import time
N = 5
t0 = time.perf_counter()
for _ in range(N):
    analyze(a, b)
torch.cuda.synchronize()
print(f"wall per step {1e3 * (time.perf_counter() - t0) / N:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    analyze(a, b)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(45)
