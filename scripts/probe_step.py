"""One C4 bench step, for ncu launch lists (no timing claims)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth
from paper_2512_08365_b200.columns import TraceColumns
from paper_2512_08365_b200.pipeline import analyze
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ca, cb = synth.make_pair(cfg)
for c in (ca, cb):
    for n in TraceColumns.HOT:
        c.device(n)
torch.cuda.synchronize()
for _ in range(steps):
    r = analyze(ca, cb, "samples", 0.10, 100)
torch.cuda.synchronize()
print("P", r.join.P, "waste", r.join.n_waste)
