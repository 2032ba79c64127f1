"""Where the C4 diff phase's time goes (wall clock with a synchronize after
each stage): pairing (join_prepare), findings (dw_join_findings + rank), the
top-k report (top_findings: gathers, two D2H copies, classification)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth, build_ledger
from paper_2512_08365_b200.detect import FindingColumns
from paper_2512_08365_b200.join import join_diff, join_prepare

a, b = synth.make_pair(sys.argv[1] if len(sys.argv) > 1 else "C4")
la, lb = build_ledger(a, method="samples", summation="exact"), build_ledger(b, method="samples", summation="exact")
torch.cuda.synchronize()
for it in range(4):
    t0 = time.perf_counter()
    prep = join_prepare(a, b)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    jd = join_diff(a, b, la, lb, 0.10, 100, full_columns=False, epw=False, prep=prep, columns=FindingColumns.DELTAS)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    top = jd.top_findings(a, b)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"prepare {1e3*(t1-t0):.2f} ms  findings+rank {1e3*(t2-t1):.2f} ms  top_findings {1e3*(t3-t2):.2f} ms  "
          f"total {1e3*(t3-t0):.2f}", flush=True)
