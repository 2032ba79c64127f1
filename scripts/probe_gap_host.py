"""Host time between join_prepare's return and the findings launch in one C4
analyze() step: the ledgers' status reads, join_diff's set-up."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth, join as J, energy as E
from paper_2512_08365_b200 import pipeline as PL
from paper_2512_08365_b200.columns import TraceColumns

a, b = synth.make_pair(sys.argv[1] if len(sys.argv) > 1 else "C4")
for c in (a, b):
    for n in TraceColumns.HOT:
        c.device(n)
marks = []
orig_prep, orig_find = J.join_prepare, J._native.lib().dw_join_findings


def prep(*x, **kw):
    r = orig_prep(*x, **kw)
    marks.append(("prep_return", time.perf_counter()))
    return r


PL.join_prepare = prep
orig_begin = PL._begin_ledger


def begin(*x, **kw):
    f = orig_begin(*x, **kw)

    def fin():
        t0 = time.perf_counter()
        r = f()
        marks.append(("ledger_finish %.1f us" % (1e6 * (time.perf_counter() - t0)), time.perf_counter()))
        return r
    return fin


PL._begin_ledger = begin
orig_rank = J.rank_order


def rank(*x, **kw):
    marks.append(("rank_call (findings launched)", time.perf_counter()))
    return orig_rank(*x, **kw)


J.rank_order = rank
for _ in range(4):
    marks.clear()
    PL.analyze(a, b)
    torch.cuda.synchronize()
t0 = marks[0][1]
for name, t in marks:
    print(f"{1e6 * (t - t0):9.1f} us  {name}")
