"""Host-side phase times of the e2e step (bench-style pinned packed columns):
finds where the occasional slow step spends its time."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2512_08365_b200 import synth  # noqa: E402
from paper_2512_08365_b200 import pipeline as pl  # noqa: E402
from paper_2512_08365_b200.columns import PackedColumns, pack  # noqa: E402

ca, cb = synth.make_pair("C4")
pinned = []
for c in (ca, cb):
    pc = pack(c)

    def pin(t):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h
    hc = PackedColumns(pc.ts_base, pin(pc.ts), pin(pc.watts), pc.op_start_base, pin(pc.op_start), pin(pc.op_end),
                       pc.k_start_base, pin(pc.k_start), pin(pc.k_end), c.trace_end, op_sig=pin(pc.op_sig),
                       watts_p0=pc.watts_p0, ts_bias=pc.ts_bias, op_sig_dict=pin(pc.op_sig_dict),
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
cs = torch.cuda.Stream()
T = {}
orig = {n: getattr(pl, n) for n in ("build_ledger", "join_prepare", "join_diff")}


def wrap(n):
    def f(*a, **k):
        t = time.perf_counter()
        r = orig[n](*a, **k)
        T.setdefault(n, []).append(time.perf_counter() - t)
        return r
    return f


for n in orig:
    setattr(pl, n, wrap(n))
import gc  # noqa: E402
for it in range(10):
    T.clear()
    for p in pinned:
        p.drop_device()
    torch.cuda.synchronize()
    g0 = gc.get_count()
    t0 = time.perf_counter()
    r = pl.analyze(pinned[0], pinned[1], "samples", 0.10, 100, copy_stream=cs)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ph = " ".join(f"{n}={'/'.join(f'{1e3 * x:.1f}' for x in v)}" for n, v in T.items())
    print(f"step {it}: wall {1e3 * (t2 - t0):.1f} ms (host {1e3 * (t1 - t0):.1f}) {ph} gc={g0}", flush=True)
