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
# packed columns: bit-packed deltas / durations (reduce-then-scan), run-coded
# and plain decimal watts, dictionary signatures; the host-resident analysis
from paper_2512_08365_b200.columns import pack, PackedColumns
from paper_2512_08365_b200.pipeline import analyze_corpus
for c in (a, b):
    p = pack(c)
    assert p.watts_rep is not None
    for n in ("ts", "watts", "op_start", "op_end", "k_start", "k_end", "op_sig"):
        assert torch.equal(p.device(n), c.device(n)), n
    q = pack(c, runs=False)
    assert torch.equal(q.device("watts"), c.device("watts"))
pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)  # noqa: E731
hosts = []
for c in (a, b):
    q = pack(c)
    hosts.append(PackedColumns(q.ts_base, pin(q.ts), pin(q.watts), q.op_start_base, pin(q.op_start), pin(q.op_end),
                               q.k_start_base, pin(q.k_start), pin(q.k_end), q.trace_end, op_sig=pin(q.op_sig),
                               watts_p0=q.watts_p0, ts_bias=q.ts_bias, op_sig_dict=pin(q.op_sig_dict),
                               ts_bits=q.ts_bits, ts_step=q.ts_step, watts_bits=q.watts_bits, n_power=q.n_power, ts_last=q._ts_last, iv_bits=q.iv_bits,
                               n_ops=q.n_ops, n_kernels=q.n_kernels, sig_bits=q.sig_bits, watts_rep=pin(q.watts_rep)))
an = analyze(hosts[0], hosts[1], copy_stream=torch.cuda.Stream())
print("host-resident analysis", an.join.P)
ca = analyze_corpus([(a, b), (c3a, c3b)], k=20)
print("corpus", len(ca.top))
torch.cuda.synchronize()
print("sanitize workload done")
