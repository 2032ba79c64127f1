"""build_ledger(method="replay") time at scale (C5: 6.25M ops per trace)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import build_ledger, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
a, _ = synth.make_pair(cfg)
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    led = build_ledger(a, method="replay")
    torch.cuda.synchronize()
    print(f"{cfg} replay ledger: {a.n_ops} ops, {1e3 * (time.perf_counter() - t):.1f} ms, total {led.total_joules:.3f} J")
