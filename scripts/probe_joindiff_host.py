"""cProfile of join_diff's host side (a C4 pair, prepared once, findings +
rank repeated)."""
import cProfile
import pstats
import sys
import torch
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth
from paper_2512_08365_b200.columns import TraceColumns
from paper_2512_08365_b200.detect import FindingColumns
from paper_2512_08365_b200.energy import build_ledger
from paper_2512_08365_b200.join import join_diff, join_prepare

a, b = synth.make_pair(sys.argv[1] if len(sys.argv) > 1 else "C4")
for c in (a, b):
    for n in TraceColumns.HOT:
        c.device(n)
la, lb = build_ledger(a, method="samples", summation="exact"), build_ledger(b, method="samples", summation="exact")
prep = join_prepare(a, b)
kw = dict(full_columns=False, epw=False, prep=prep, columns=FindingColumns.DELTAS)
for _ in range(3):
    join_diff(a, b, la, lb, 0.1, 100, **kw)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    join_diff(a, b, la, lb, 0.1, 100, **kw)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
