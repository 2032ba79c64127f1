"""Cost of classifying the top-k join findings at C4 (diagnose.classify_pairs)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth  # noqa: E402
from paper_2512_08365_b200.energy import build_ledger  # noqa: E402
from paper_2512_08365_b200.join import join_diff  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
ca, cb = synth.make_pair(cfg)
la, lb = build_ledger(ca, method="samples"), build_ledger(cb, method="samples")
jd = join_diff(ca, cb, la, lb, 0.10, 100, full_columns=False, epw=False)
for cls in (False, True, False, True, True):
    torch.cuda.synchronize()
    t = time.perf_counter()
    top = jd.top_findings(ca, cb, classify=cls)
    torch.cuda.synchronize()
    print(f"classify={cls}: {1e3 * (time.perf_counter() - t):.2f} ms")
from collections import Counter  # noqa: E402
print(Counter(f.category for f in top if f.verdict == "waste"))
w = ca.device("watts")
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    m = w.min().item()
    print(f"watts.min over {w.numel()}: {1e3 * (time.perf_counter() - t):.2f} ms")
