"""world_size-2 gloo test of the corpus top-k merge (the one multi-GPU
exchange) -- runs on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _keys(rank, P, seed):
    import numpy as np
    rng = np.random.default_rng(seed + rank)
    wasted = np.round(rng.exponential(1.0, size=P), 1)   # many exact ties
    verdict = rng.choice([0, 1, 2], size=P, p=[0.6, 0.2, 0.2]).astype(np.int8)
    tie = rng.integers(0, 4, size=P)
    return wasted, verdict, tie


def _encode(wasted, verdict, tie):
    import numpy as np
    P = len(wasted)
    bits = wasted.view(np.uint64) & np.uint64(0x7FFFFFFFFFFFFFFF)
    hi = bits | ((verdict == 2).astype(np.uint64) << np.uint64(63))
    lo = ~(((tie.astype(np.uint64) + np.uint64(1)) << np.uint64(32)) | np.arange(P, dtype=np.uint64))
    return hi.view(np.int64), lo.view(np.int64)


def _worker(rank, world, port, k, P, seed, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_08365_b200.dist import merge_topk
    wasted, verdict, tie = _keys(rank, P, seed)
    order = oracle.rank(verdict, wasted, tie)[:k]          # each rank's own top-k
    hi, lo = _encode(wasted, verdict, tie)
    r, pos = merge_topk(torch.from_numpy(hi[order]), torch.from_numpy(lo[order]), k)
    if rank == 0:
        out.put([(int(a), int(order_b)) for a, order_b in zip(r.tolist(), pos.tolist())])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [1, 17, 64, 300])
def test_merge_topk_matches_global_ranking(k):
    world, P, seed = 2, 300, 99
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, P, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # reference: one global ranking over both ranks' findings, rank-major numbering
    import numpy as np
    W, V, T, owner, local = [], [], [], [], []
    for r in range(world):
        w, v, t = _keys(r, P, seed)
        W.append(w); V.append(v); T.append(t)
        owner += [r] * P
        local += list(range(P))
    order = oracle.rank(np.concatenate(V), np.concatenate(W), np.concatenate(T))[:k]
    per_rank_order = {r: list(oracle.rank(V[r], W[r], T[r])) for r in range(world)}
    want = [(owner[i], per_rank_order[owner[i]].index(local[i])) for i in order]
    assert got == want
