"""cProfile of one C4 analyze() step (device-resident columns): host-side cost."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth  # noqa: E402
from paper_2512_08365_b200.columns import TraceColumns  # noqa: E402
from paper_2512_08365_b200.pipeline import analyze  # noqa: E402

a, b = synth.make_pair("C4")
for c in (a, b):
    for n in TraceColumns.HOT:
        c.device(n)
for _ in range(3):
    analyze(a, b, "samples", 0.10, 100)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
analyze(a, b, "samples", 0.10, 100)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
