"""Ingestion timing: canonical JSONL (tensor-free, C2-shaped) -> device columns
with ingest.load_columns (GPU) vs the reference-compatible Python loader."""
import sys, time, os
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth, load_trace
from paper_2512_08365_b200.columns import TraceColumns
from paper_2512_08365_b200.ingest import load_columns


def write_canonical(cols, path):
    ts, w = cols.host("ts"), cols.host("watts")
    os_, oe, ks, ke, ko = (cols.host(n) for n in ("op_start", "op_end", "k_start", "k_end", "k_op"))
    kfirst = np.searchsorted(ko, np.arange(len(os_)))
    klast = np.searchsorted(ko, np.arange(len(os_)), side="right")
    with open(path, "w") as fh:
        fh.write('{"type":"header","schema_version":1,"system":"A:c2","workload":"probe","seed":2}\n')
        for i in range(len(os_)):
            kid = ",".join(f'"k{j}"' for j in range(kfirst[i], klast[i]))
            fh.write(f'{{"type":"op","op_id":"op{i:08d}","op_name":"n{i % 64}","input_tensor_ids":[],'
                     f'"output_tensor_ids":[],"kernel_ids":[{kid}],"start":{os_[i]},"end":{oe[i]}}}\n')
        order = np.argsort(ks, kind="stable")
        for j in order:
            fh.write(f'{{"type":"kernel","kernel_id":"k{j}","kernel_name":"kern","correlation_id":{j},'
                     f'"start":{ks[j]},"end":{ke[j]},"backtrace":["main"]}}\n')
        for a, b in zip(ts, w):
            fh.write(f'{{"type":"power","timestamp":{a},"watts":{float(f"{b:.9g}")!r}}}\n')


n_ops = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = synth.scaled(synth.CONFIGS["C2"], n_ops)
a, _ = synth.make_pair(cfg, device="cpu")
path = "/tmp/probe_ingest.jsonl"
t = time.time(); write_canonical(a, path); print(f"wrote {os.path.getsize(path) / 1e9:.2f} GB in {time.time() - t:.1f}s", flush=True)
for it in range(3):
    torch.cuda.synchronize(); t = time.time()
    c = load_columns(path)
    torch.cuda.synchronize(); dt = time.time() - t
    print(f"load_columns ({c.loaded_by}): {dt:.3f} s  {c.n_ops} ops {c.n_kernels} kernels {c.n_power} samples", flush=True)
small = synth.scaled(synth.CONFIGS["C2"], 20_000)
sa, _ = synth.make_pair(small, device="cpu")
write_canonical(sa, "/tmp/probe_small.jsonl")
t = time.time(); tr = load_trace("/tmp/probe_small.jsonl"); cs = TraceColumns.from_trace(tr); dt = time.time() - t
print(f"python load_trace + columns on {sa.n_ops} ops: {dt:.3f} s -> x{n_ops / sa.n_ops:.0f} = {dt * n_ops / sa.n_ops:.1f} s (linear)")
