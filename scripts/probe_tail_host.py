"""Wall time of the host tail of one C4 analyze() step: top_findings (the k
rows' device gather + the host rows + classification), measured after the
rank has finished (synchronised), several repeats."""
import sys
import time
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
    res = analyze(a, b)
torch.cuda.synchronize()
jd = res.join
for classify in (True, False):
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        jd.top_findings(a, b, classify=classify)
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"top_findings classify={classify}: median {sorted(ts)[5]:.3f} ms  min {min(ts):.3f}")
t = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    analyze(a, b)
    t.append(1e3 * (time.perf_counter() - t0))
print(f"analyze wall: median {sorted(t)[2]:.3f} ms")
