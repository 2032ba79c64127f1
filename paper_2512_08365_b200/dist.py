"""Multi-process plumbing for corpus analyses (one process per GPU).

Ranks own whole trace pairs: attribution and the join need no
data-path collective.  The one exchange is the corpus-wide ranking -- each rank
ranks its own findings on the device (dw_rank), then the k best candidates of
every rank are gathered and merged.  Works over NCCL (CUDA tensors) and gloo
(CPU tensors, tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

_FLIP = -0x8000000000000000  # unsigned order of 64-bit keys -> signed order


def _signed(u: torch.Tensor) -> torch.Tensor:
    return u ^ _FLIP


def merge_topk(key_hi: torch.Tensor, key_lo: torch.Tensor, k: int, group=None):
    """Global top-k over every rank's candidates.

    key_hi / key_lo are this rank's k best keys (int64 tensors holding the
    unsigned 128-bit report key of csrc/diff.cu, best first).  Returns
    (rank, position) of the global k best, best first: position indexes the
    owning rank's candidate list.  Equal (key_hi, nodes_a) across ranks fall to
    the lower rank (pairs are numbered rank-major: the corpus's stable order).
    """
    world = dist.get_world_size(group)
    n = int(key_hi.numel())
    counts = [torch.zeros(1, dtype=torch.int64, device=key_hi.device) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([n], dtype=torch.int64, device=key_hi.device), group=group)
    m = max(int(c.item()) for c in counts)
    pad_hi = torch.zeros(m, dtype=torch.int64, device=key_hi.device)
    pad_lo = torch.zeros(m, dtype=torch.int64, device=key_hi.device)
    pad_hi[:n] = key_hi
    pad_lo[:n] = key_lo
    hs = [torch.empty_like(pad_hi) for _ in range(world)]
    ls = [torch.empty_like(pad_lo) for _ in range(world)]
    dist.all_gather(hs, pad_hi, group=group)
    dist.all_gather(ls, pad_lo, group=group)
    hi = torch.cat([h[: int(c.item())] for h, c in zip(hs, counts)])
    lo = torch.cat([l[: int(c.item())] for l, c in zip(ls, counts)])
    rank = torch.cat([torch.full((int(c.item()),), r, dtype=torch.int64, device=hi.device)
                      for r, c in enumerate(counts)])
    pos = torch.cat([torch.arange(int(c.item()), dtype=torch.int64, device=hi.device)
                     for c in counts])
    order = merge_order(hi, lo, rank, pos, k)
    return rank[order], pos[order]


def merge_order(hi: torch.Tensor, lo: torch.Tensor, rank: torch.Tensor, pos: torch.Tensor, k: int,
                by_finding: bool = False):
    """Report order of gathered candidates: descending hi, then ascending
    nodes_a tie (upper half of lo, stored complemented), then corpus order
    (rank, position) -- LSD with stable sorts.  Returns the first k indices.
    ``by_finding``: the candidates are findings of ONE pair numbered globally
    (sharded join), so the whole lo (tie, then finding index) orders ties."""
    tie_part = _signed(lo) if by_finding else (lo >> 32) & 0xFFFFFFFF
    order = torch.arange(hi.numel(), device=hi.device)
    for key, desc in ((pos, False), (rank, False), (tie_part, True), (_signed(hi), True)):
        kk = key[order]
        idx = torch.sort(kk, descending=desc, stable=True).indices
        order = order[idx]
    return order[:k]
