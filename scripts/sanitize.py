"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck /
initcheck): every kernel of the C4 step at a small size -- the exact and the
reference-order tile kernels (step and linear signals), the long-interval and
scan kernels, the signature join (bucketed partition, bucket ranking,
findings), the top-k ranking -- plus the overlap split (C3 distribution).
    compute-sanitizer --tool racecheck python scripts/sanitize.py"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth, build_ledger
from paper_2512_08365_b200.pipeline import analyze

cfg = synth.scaled(synth.CONFIGS["C4"], int(sys.argv[1]) if len(sys.argv) > 1 else 30_000)
a, b = synth.make_pair(cfg)
for summation in ("exact", "reference"):
    an = analyze(a, b, summation=summation, lean=(summation == "exact"))
    print(summation, "findings", an.join.P, "top", len(an.report.findings) if hasattr(an, "report") else "")
c3a, c3b = synth.make_pair(synth.scaled(synth.CONFIGS["C3"], 20_000))
for summation in ("exact", "reference"):  # step signal (breakpoints)
    led = build_ledger(c3a, method="ground_truth", summation=summation)
    print("step ledger", summation, led.total_joules if hasattr(led, "total_joules") else "")
led = build_ledger(c3a, method="ground_truth", overlap="split")
print("split ledger done")
torch.cuda.synchronize()
print("sanitize workload done")
