"""Time-window sharding end to end through REAL collectives (not the
in-process loopback): two processes share cuda:0 (gloo for the plumbing;
CUDA IPC works between processes on one device exactly as between the GPUs
of a node).  Each rank runs shard.sharded_ledger on its window of both traces
(tensor all-gathers of the validation indices, crossing intervals, int128
shares and totals) and shard.sharded_join (records exchanged by the NCCL-path
all-to-all, or by the fused peer-memory scatter into the persistent mailbox
with device-side arrival flags), twice in a row (the mailbox is reused, the
epochs advance).  Every rank must reproduce the one-GPU ledger totals and its
own intervals' joules bit for bit, and the one-GPU join's top-k."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _worker(rank: int, world: int, port: int, out_path: str, p2p: bool):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2512_08365_b200 import build_ledger, shard, synth
    from paper_2512_08365_b200.join import join_diff
    a, b = synth.make_pair(synth.scaled(synth.CONFIGS["C4"], 60_000))
    la, lb = build_ledger(a, method="samples"), build_ledger(b, method="samples")
    jd = join_diff(a, b, la, lb, 0.10, 40, full_columns=False, epw=False)
    top = jd.top_findings(a, b)
    ia, ib = jd.pair_of(jd.order)
    comm = shard.Comm(p2p=p2p)
    msgs = []
    for rep in range(2):
        sa = shard.sharded_ledger(a, "linear", comm)
        sb = shard.sharded_ledger(b, "linear", comm)
        for s, full in ((sa, la), (sb, lb)):
            if s.total_joules != full.total_joules or s.op_total != full.operator_total():
                msgs.append(f"rep {rep}: totals")
            if not torch.equal(s.joules[0].cpu(), torch.from_numpy(full.per_operator.array())[s.idx[0].cpu()]):
                msgs.append(f"rep {rep}: op joules")
            if not torch.equal(s.joules[1].cpu(), torch.from_numpy(full.per_kernel.array())[s.idx[1].cpu()]):
                msgs.append(f"rep {rep}: kernel joules")
        res = shard.sharded_join(shard.shard_ops(a, sa, True), shard.shard_ops(b, sb, False), a.n_ops, comm,
                                 0.10, 40)
        if (res.P, res.n_waste, res.wasted_joules) != (jd.P, jd.n_waste, jd.wasted_joules):
            msgs.append(f"rep {rep}: join totals {res.P, res.n_waste, res.wasted_joules}")
        if [r[0] for r in res.top] != ia.cpu().tolist() or [r[1] for r in res.top] != ib.cpu().tolist():
            msgs.append(f"rep {rep}: top-k pairs")
        if [r[7] for r in res.top] != [f.wasted_joules for f in top]:
            msgs.append(f"rep {rep}: top-k wasted")
    comm.close()
    with open(f"{out_path}.{rank}", "w") as fh:
        fh.write("ok" if not msgs else "; ".join(msgs))
    dist.barrier()
    dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("p2p", [False, True])
def test_sharded_ledger_and_join_two_processes(tmp_path, p2p):
    import torch.multiprocessing as mp
    world = 2
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(world, _free_port(), out, p2p), nprocs=world, join=True)
    for r in range(world):
        assert open(f"{out}.{r}").read() == "ok", r
