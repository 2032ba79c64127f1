"""Perf probe: the C4 join diff (+ top-k) on device-resident ledgers (CUDA events)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth, build_ledger, _native
from paper_2512_08365_b200.join import join_diff
from paper_2512_08365_b200.detect import FindingColumns
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
a, b = synth.make_pair(name)
la, lb = build_ledger(a, method="samples"), build_ledger(b, method="samples")
torch.cuda.synchronize()
for it in range(iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    cols = FindingColumns.KEYS if "keys" in sys.argv else (FindingColumns.DELTAS if "deltas" in sys.argv else None)
    jd = join_diff(a, b, la, lb, 0.10, 100, full_columns=False, epw=False, columns=cols)
    top = jd.top_findings(a, b)
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    if it == iters - 1 and hasattr(_native.lib(), "dw_trace_report"):
        _native.lib().dw_trace_report()
    print(f"join_diff+top: {e0.elapsed_time(e1):.3f} ms (wall {1e3*(t1-t0):.3f})  P={jd.P} waste={jd.n_waste} wasted={jd.wasted_joules:.6f}", flush=True)
