"""Host logic of time-window sharding (paper_2512_08365_b200/shard.py) on CPU:
the window plan, and the two exchanges over a world_size-2 gloo group -- the
signature all-to-all of the sharded join and the globally numbered top-k
merge.  (The per-rank GPU compute is checked bit-exact against one GPU in
tests/test_gpu_shard.py.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2512_08365_b200 import shard


@pytest.mark.parametrize("S,world,kind", [(10_000, 2, "step"), (1_000_003, 8, "linear"), (4096, 2, "linear"),
                                          (77_777, 5, "step")])
def test_plan_tiles_the_signal(S, world, kind):
    w = shard.plan(S, world, kind)
    nterms = S if kind == "step" else S - 1
    assert w[0].s0 == 0 and w[-1].s1 == S and w[0].p0 == 0 and w[-1].p1 == nterms
    for a, b in zip(w, w[1:]):
        assert a.s1 == b.s0 and a.p1 == b.p0 and b.s0 % shard.TILE == 0
    for x in w:
        assert x.l0 % shard.TILE == 0 and x.l0 <= x.s0 and x.l1 >= min(x.s1 + shard.HALO, S)
        assert x.s1 > x.s0


def test_plan_rejects_tiny_signals():
    with pytest.raises(ValueError):
        shard.plan(3000, 2, "step")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ops(rank, world, n, seed):
    """This rank's owned ops of a global sequence (contiguous slice)."""
    rng = np.random.default_rng(seed)
    sig = rng.integers(0, 37, size=n).astype(np.int64) * 0x2545F4914F6CDD1 + 12345
    lo, hi = rank * n // world, (rank + 1) * n // world
    idx = torch.arange(lo, hi, dtype=torch.int64)
    return shard.ShardOps(idx, torch.from_numpy(sig[lo:hi]), idx * 10, idx * 10 + 5,
                          torch.from_numpy(rng.uniform(size=n)[lo:hi]), idx.clone()), sig


def _a2a_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = shard.Comm()
    o, sig = _ops(rank, world, 1000, 5)
    got = shard._unpack(comm.all_to_all(shard._partition(o, world, True)), 6)
    q.put((rank, got["idx"].tolist(), got["sig"].tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_signature_all_to_all_gloo():
    world, port = 2, _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_a2a_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict((r, (i, s)) for r, i, s in (q.get(timeout=120) for _ in range(world)))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    _, sig = _ops(0, world, 1000, 5)
    seen = []
    for r in range(world):
        idx, s = res[r]
        assert idx == sorted(idx)                      # global op order kept
        d = shard._dest(torch.tensor(s, dtype=torch.int64), world)
        assert bool((d == r).all())                    # every signature on its rank
        assert s == sig[idx].tolist()
        seen += idx
    assert sorted(seen) == list(range(1000))           # nothing lost or duplicated


def test_global_merge_matches_one_ranking():
    """Candidates of two ranks with global finding numbers merge into exactly
    the one-pair report order (ties by nodes_a, then finding number)."""
    rng = np.random.default_rng(3)
    P = 400
    wasted = np.round(rng.exponential(1.0, size=P), 1)
    verdict = rng.choice([0, 1, 2], size=P, p=[0.5, 0.2, 0.3]).astype(np.int8)
    tie = np.where(rng.random(P) < 0.2, -1, rng.integers(0, 50, size=P))
    want = list(oracle.rank(verdict, wasted, tie + 1))[:60]  # oracle's tie: 0 sorts first (B-only)
    owner = rng.integers(0, 2, size=P)
    gathered = []
    for r in range(2):
        mine = np.nonzero(owner == r)[0]
        bits = wasted[mine].view(np.uint64) & np.uint64(0x7FFFFFFFFFFFFFFF)
        hi = (bits | ((verdict[mine] == 2).astype(np.uint64) << np.uint64(63))).view(np.int64)
        lo = (~(((tie[mine] + 1).astype(np.uint64) << np.uint64(32)) | mine.astype(np.uint64))).view(np.int64)
        rows_i = torch.zeros(len(mine), 7, dtype=torch.int64)
        rows_i[:, 0] = torch.from_numpy(mine)
        gathered.append((torch.from_numpy(hi), torch.from_numpy(lo), rows_i,
                         torch.zeros(len(mine), 4, dtype=torch.float64), torch.zeros(4, dtype=torch.int64)))
    res = shard._merge(gathered, 60)
    assert [r[0] for r in res.top] == want
