"""Perf probe: attribution at a BASELINE config (device-resident inputs)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth, build_ledger, _native
from paper_2512_08365_b200.energy import PowerSignal, _run_ledger

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
kind = sys.argv[2] if len(sys.argv) > 2 else "step"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
summation = sys.argv[4] if len(sys.argv) > 4 else "reference"
t = time.time()
a, b = synth.make_pair(name)
torch.cuda.synchronize()
print(f"gen {name}: {time.time()-t:.1f}s  N={a.n_ops} K={a.n_kernels} S={a.n_power} kernels_sorted={a.kernels_sorted}", flush=True)
for side in (a, b):
    for c in ("op_start", "op_end", "k_start", "k_end"):
        side.device(c)
sig = PowerSignal.from_columns(a.ts, a.watts, a.signal_span()[1], kind)
torch.cuda.synchronize()
bytes_alg = 16 * a.n_power + 24 * (a.n_ops + a.n_kernels)
for it in range(iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    per_op, per_k, st = _run_ledger(a, sig, False, summation)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"ledger {kind} {summation}: {ms:.3f} ms  {bytes_alg/ms/1e6:.1f} GB/s alg  long={st.long_intervals} code={st.code} total={st.totals[0]:.6e}", flush=True)
L = _native.lib()
if hasattr(L, "dw_phase_prof"):
    import ctypes
    buf = (ctypes.c_ulonglong * 16)()
    L.dw_phase_prof(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); _run_ledger(a, sig, False); e1.record(); torch.cuda.synchronize()
    L.dw_phase_prof(buf, 1)
    nt = (a.n_power + 1023) // 1024
    names = ["wait_full", "ts32+bar", "terms+tilesum", "phase1+bar", "scan+bar", "scatter+bar",
             "phase2+bar", "prod_wait_empty", "prod_issue"]
    print(f"phase cycles per tile (per group / producer), ledger {e0.elapsed_time(e1):.3f} ms:")
    for i, nm in enumerate(names):
        print(f"  {nm:16s} {buf[i] / nt:9.1f}")
    print(f"  sum consumer     {sum(buf[i] for i in range(7)) / nt:9.1f}")
print("mem GB", torch.cuda.max_memory_allocated()/1e9)
