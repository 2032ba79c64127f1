"""build_ledger(method="sampled") at scale: where the time goes."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import build_ledger, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
a, _ = synth.make_pair(cfg)
for it in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    led = build_ledger(a, method="sampled")
    torch.cuda.synchronize()
    print(f"{cfg} sampled ledger: {a.n_ops} ops, span {a.signal_span()}, {1e3 * (time.perf_counter() - t):.1f} ms")
pr = cProfile.Profile()
pr.enable()
build_ledger(a, method="sampled")
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
