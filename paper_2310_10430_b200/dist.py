"""Multi-rank plumbing for the time-slab decomposition (host side only).

One process per GPU.  Rank r owns global steps (r*n_t/P, (r+1)*n_t/P] (the same
partition biot_setup applies); once per outer iteration the library sends the
last owned slice of x^k to rank r+1 and receives its ghost (x^k of step
first_step-1) from rank r-1 with NCCL send/recv inside biot_iterate
(BASELINE.json north star (d); replaces the MPI Send/Recv pipeline of the
paper's Algorithm 5).  torch.distributed is used only to
broadcast the ncclUniqueId and for barriers / max-over-ranks timing.
"""
from __future__ import annotations

import torch


def slab(n_t: int, world: int, rank: int):
    """(first_step, n_t_local) of `rank`; n_t must be divisible by world."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("need 0 <= rank < world")
    if n_t % world:
        raise ValueError("n_t must be divisible by the number of time slabs")
    n_tl = n_t // world
    return rank * n_tl + 1, n_tl


def broadcast_nccl_id(make_id, group=None, src: int = 0, device=None) -> bytes:
    """Rank `src` calls make_id() -> 128 bytes; every rank returns the same bytes.
    device: where the broadcast buffer lives (a CUDA device for the nccl backend,
    None = host for gloo)."""
    import torch.distributed as dist
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == src:
        raw = make_id()
        if len(raw) != 128:
            raise ValueError("ncclUniqueId must be 128 bytes")
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    dist.broadcast(buf, src, group=group)
    return bytes(buf.cpu().numpy().tobytes())
