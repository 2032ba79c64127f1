"""Where the e2e step's time goes at C4: raw H2D bandwidth of the packed
pinned columns (one and two streams), device decode, and the full step."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth  # noqa: E402
from paper_2512_08365_b200.columns import PackedColumns, pack  # noqa: E402
from paper_2512_08365_b200.pipeline import analyze  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
ca, cb = synth.make_pair(cfg)
pinned = []
for c in (ca, cb):
    pc = pack(c)

    def pin(t):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h
    hc = PackedColumns(pc.ts_base, pin(pc.ts), pin(pc.watts), pc.op_start_base, pin(pc.op_start), pin(pc.op_end),
                       pc.k_start_base, pin(pc.k_start), pin(pc.k_end), c.trace_end, op_sig=pin(pc.op_sig),
                       watts_p0=pc.watts_p0, ts_bias=pc.ts_bias, op_sig_dict=pc.op_sig_dict.cpu(),
                       ts_bits=pc.ts_bits, ts_step=pc.ts_step, watts_bits=pc.watts_bits, n_power=pc.n_power,
                       ts_last=pc._ts_last if pc.ts_bits is not None else None,
                               iv_bits=pc.iv_bits, n_ops=pc.n_ops, n_kernels=pc.n_kernels,
                               sig_bits=pc.sig_bits, watts_rep=None if pc.watts_rep is None else pin(pc.watts_rep))
    hc._dev["first_last"] = c._first_last_ts()
    pinned.append(hc)
for c in (ca, cb):
    c._dev.clear()
del ca, cb
torch.cuda.empty_cache()
names = ("ts", "watts", "op_start", "op_end", "k_start", "k_end", "op_sig")
tensors = [[getattr(p, n) for n in names] for p in pinned]
nbytes = sum(t.numel() * t.element_size() for ts in tensors for t in ts)
dst = [[torch.empty_like(t, device="cuda") for t in ts] for ts in tensors]


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for mode in ("one stream", "two streams", "one stream", "two streams"):
    s2 = torch.cuda.Stream()
    torch.cuda.synchronize()
    e0 = ev()
    for i, (src, d) in enumerate(zip(tensors, dst)):
        st = s2 if (mode == "two streams" and i == 1) else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            for a, b in zip(src, d):
                b.copy_(a, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
    e1 = ev()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"H2D {mode}: {nbytes / 1e9:.2f} GB in {ms:.1f} ms = {nbytes / ms / 1e6:.1f} GB/s")
del dst
torch.cuda.empty_cache()
# decode only (columns already resident as packed device tensors)
for p in pinned:
    p.drop_device()
dev_packed = []
for p in pinned:
    q = PackedColumns(p.ts_base, p.ts.cuda(), p.watts.cuda(), p.op_start_base, p.op_start.cuda(), p.op_end.cuda(),
                      p.k_start_base, p.k_start.cuda(), p.k_end.cuda(), p.trace_end, op_sig=p.op_sig.cuda(),
                      watts_p0=p.watts_p0, ts_bias=p.ts_bias, op_sig_dict=p.op_sig_dict,
                      ts_bits=p.ts_bits, ts_step=p.ts_step, watts_bits=p.watts_bits, n_power=p.n_power, ts_last=p._ts_last if p.ts_bits is not None else None,
                      iv_bits=p.iv_bits, n_ops=p.n_ops, n_kernels=p.n_kernels, sig_bits=p.sig_bits,
                      watts_rep=None if p.watts_rep is None else p.watts_rep.cuda())
    q._dev["first_last"] = p._dev["first_last"]
    dev_packed.append(q)
for it in range(3):
    for q in dev_packed:
        q.drop_device()
    torch.cuda.synchronize()
    e0 = ev()
    for q in dev_packed:
        for n in ("ts", "watts", "op_start", "k_start"):
            q.device(n)
    e1 = ev()
    torch.cuda.synchronize()
    print(f"decode both traces (device-resident packed input): {e0.elapsed_time(e1):.2f} ms")
    e0 = ev()
    r = analyze(dev_packed[0], dev_packed[1], "samples", 0.10, 100)
    e1 = ev()
    torch.cuda.synchronize()
    print(f"analyze on decoded columns: {e0.elapsed_time(e1):.2f} ms")
del dev_packed
torch.cuda.empty_cache()
cs = torch.cuda.Stream()
for it in range(3):
    for p in pinned:
        p.drop_device()
    torch.cuda.synchronize()
    e0 = ev()
    r = analyze(pinned[0], pinned[1], "samples", 0.10, 100, copy_stream=cs)
    e1 = ev()
    torch.cuda.synchronize()
    print(f"e2e step: {e0.elapsed_time(e1):.1f} ms")
# bench-style: back-to-back steps in one timed region
for p in pinned:
    p.drop_device()
torch.cuda.synchronize()
e0 = ev()
for it in range(3):
    for p in pinned:
        p.drop_device()
    r = analyze(pinned[0], pinned[1], "samples", 0.10, 100, copy_stream=cs)
e1 = ev()
torch.cuda.synchronize()
print(f"e2e back-to-back x3: {e0.elapsed_time(e1) / 3:.1f} ms/step")
t0 = time.perf_counter()
for it in range(3):
    for p in pinned:
        p.drop_device()
    r = analyze(pinned[0], pinned[1], "samples", 0.10, 100, copy_stream=cs)
    torch.cuda.synchronize()
print(f"e2e synced x3 (wall): {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms/step")
