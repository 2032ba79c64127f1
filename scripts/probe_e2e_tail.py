"""Where the e2e step's time goes after the last host->device byte (torch
profiler timeline of one bench-style step from pinned packed columns)."""
import json, sys
import torch
from torch.profiler import profile, ProfilerActivity
sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth
from paper_2512_08365_b200.columns import PackedColumns, pack
from paper_2512_08365_b200.pipeline import analyze

ca, cb = synth.make_pair("C4")
pinned = []
for c in (ca, cb):
    pc = pack(c)
    pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)  # noqa: E731
    hc = PackedColumns(pc.ts_base, pin(pc.ts), pin(pc.watts), pc.op_start_base, pin(pc.op_start), pin(pc.op_end),
                       pc.k_start_base, pin(pc.k_start), pin(pc.k_end), c.trace_end, op_sig=pin(pc.op_sig),
                       watts_p0=pc.watts_p0, ts_bias=pc.ts_bias, op_sig_dict=pin(pc.op_sig_dict),
                       ts_bits=pc.ts_bits, ts_step=pc.ts_step, watts_bits=pc.watts_bits, n_power=pc.n_power,
                       ts_last=pc._ts_last if pc.ts_bits is not None else None,
                       iv_bits=pc.iv_bits, n_ops=pc.n_ops, n_kernels=pc.n_kernels, sig_bits=pc.sig_bits,
                       watts_rep=None if pc.watts_rep is None else pin(pc.watts_rep))
    hc._dev["first_last"] = c._first_last_ts()
    pinned.append(hc)
del ca, cb
torch.cuda.empty_cache()
cs = torch.cuda.Stream()


def step():
    for p in pinned:
        p.drop_device()
    return analyze(pinned[0], pinned[1], copy_stream=cs)


for _ in range(5):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
ev = json.load(open("gpurun_out/e2e_trace.json"))["traceEvents"]
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
end = max(e["ts"] + e["dur"] for e in gpu)
h2d = [e for e in gpu if "HtoD" in e["name"] and e["dur"] > 100]
last = max(e["ts"] + e["dur"] for e in h2d)
print(f"step span {1e-3 * (end - t0):.2f} ms; last large H2D ends at {1e-3 * (last - t0):.2f} ms; tail {1e-3 * (end - last):.2f} ms")
print(f"H2D busy {1e-3 * sum(e['dur'] for e in h2d):.2f} ms over {len(h2d)} copies")
tail = [e for e in gpu if e["ts"] + e["dur"] > last]
agg = {}
for e in tail:
    k = e["name"][:60]
    agg[k] = agg.get(k, 0) + e["dur"]
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {1e-3 * v:7.3f} ms  {k}")

for e in h2d:
    print(f"  H2D {1e-3 * (e['ts'] - t0):8.2f} ms  dur {1e-3 * e['dur']:7.2f} ms  "
          f"{e.get('args', {}).get('bytes', 0) / 1e6:9.1f} MB  "
          f"{e.get('args', {}).get('memory bandwidth (GB/s)', 0)} GB/s")
