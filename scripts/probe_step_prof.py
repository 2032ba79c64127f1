"""torch.profiler view of one C4 analyze() step (after warm-up): where the
host time between the library's kernels goes."""
import sys
import torch
from torch.profiler import profile, ProfilerActivity
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth
from paper_2512_08365_b200.pipeline import analyze
from paper_2512_08365_b200.columns import TraceColumns

a, b = synth.make_pair(sys.argv[1] if len(sys.argv) > 1 else "C4")
for c in (a, b):
    for n in TraceColumns.HOT:
        c.device(n)
for _ in range(3):
    analyze(a, b)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=False) as prof:
    analyze(a, b)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=30))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
prof.export_chrome_trace("gpurun_out/step_trace.json")
import json
ev = json.load(open("gpurun_out/step_trace.json"))["traceEvents"]
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
print("GPU events", len(gpu), "span us", gpu[-1]["ts"] + gpu[-1]["dur"] - gpu[0]["ts"])
busy = sum(e["dur"] for e in gpu)
print("busy us", busy)
gaps = []
for p, q in zip(gpu, gpu[1:]):
    g = q["ts"] - (p["ts"] + p["dur"])
    if g > 15:
        gaps.append((g, p["name"][:60], q["name"][:60]))
for g in sorted(gaps, reverse=True)[:25]:
    print(f"gap {g[0]:8.1f} us  after {g[1]}  before {g[2]}")
print("sum of gaps > 15 us:", sum(g[0] for g in gaps))
