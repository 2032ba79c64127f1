"""Per-column device decode times of a packed C4 trace (CUDA events)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth  # noqa: E402
from paper_2512_08365_b200.columns import pack  # noqa: E402

a, _ = synth.make_pair(sys.argv[1] if len(sys.argv) > 1 else "C4")
p = pack(a)
del a
torch.cuda.empty_cache()
for it in range(3):
    p.drop_device()
    torch.cuda.synchronize()
    out = []
    for n in ("ts", "watts", "op_start", "k_start", "op_sig"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.device(n)
        e1.record()
        torch.cuda.synchronize()
        out.append(f"{n} {e0.elapsed_time(e1):.2f}")
    print(" | ".join(out), "ms")
