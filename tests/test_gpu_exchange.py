"""The fused record exchange of the time-window join (csrc/exchange.cu,
shard.Comm.exchange): two ranks sharing cuda:0 (CUDA IPC works between
processes on one device exactly as between the GPUs of a node), gloo for the
plumbing.  Every rank must receive exactly the records the reference
partition (shard._partition, the NCCL path's input) sends it, and the sharded
join must give the same result with and without the fused exchange."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ops(rank: int, n: int, with_rank: bool):
    from paper_2512_08365_b200.shard import ShardOps
    g = torch.Generator().manual_seed(100 + rank)
    idx = rank + 2 * torch.arange(n, dtype=torch.int64)
    sig = torch.randint(-2**62, 2**62, (n,), generator=g, dtype=torch.int64)
    if n:
        sig[::7] = sig[0]  # repeated signatures
    start = torch.randint(0, 10**9, (n,), generator=g, dtype=torch.int64)
    end = start + torch.randint(0, 1000, (n,), generator=g, dtype=torch.int64)
    joules = torch.rand(n, generator=g, dtype=torch.float64)
    rk = torch.randint(0, 10**6, (n,), generator=g, dtype=torch.int64) if with_rank else None
    dev = torch.device("cuda", 0)
    return ShardOps(idx.to(dev), sig.to(dev), start.to(dev), end.to(dev), joules.to(dev),
                    rk.to(dev) if rk is not None else None)


def _worker(rank: int, world: int, port: int, n: int, out_path: str):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2512_08365_b200 import shard
    comm = shard.Comm(p2p=True)
    ok = True
    for with_rank in (True, False):
        got = comm.exchange(_ops(rank, n + 1000 * rank, with_rank), with_rank).cpu()
        want = torch.cat([shard._partition(_ops(s, n + 1000 * s, with_rank), world, with_rank)[rank]
                          .reshape(-1, 6 if with_rank else 5).cpu() for s in range(world)])
        order_g = torch.argsort(got[:, 0])
        order_w = torch.argsort(want[:, 0])
        ok &= got.shape == want.shape and torch.equal(got[order_g], want[order_w])
    # a call larger than the mailbox (65536 rows at first): every rank re-creates
    # its receive buffer, re-maps the peers', and the epochs keep counting
    big = 150_000
    got = comm.exchange(_ops(rank, big + 7 * rank, True), True).cpu()
    want = torch.cat([shard._partition(_ops(s, big + 7 * s, True), world, True)[rank].reshape(-1, 6).cpu()
                      for s in range(world)])
    ok &= got.shape == want.shape and torch.equal(got[torch.argsort(got[:, 0])], want[torch.argsort(want[:, 0])])
    # empty sender on one rank
    e = _ops(rank, 0 if rank == 1 else 500, False)
    got = comm.exchange(e, False)
    total = torch.tensor([got.shape[0]])
    dist.all_reduce(total)
    ok &= int(total.item()) == (0 if world == 1 else 500)
    comm.close()
    with open(f"{out_path}.{rank}", "w") as fh:
        fh.write("ok" if ok else "mismatch")
    dist.barrier()
    dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_fused_exchange_matches_partition(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(world, _free_port(), 20000, out), nprocs=world, join=True)
    for r in range(world):
        assert open(f"{out}.{r}").read() == "ok", r
