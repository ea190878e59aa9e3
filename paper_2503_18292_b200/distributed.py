"""Multi-GPU plumbing: requests shard across ranks with no data-path
collective (engine instances share nothing, reference SPEC.md:535); one
all-gather after the timed region collects outputs for verification.

One process per GPU, torch.distributed with NCCL on GPUs (gloo in the CPU
tests).  Rendezvous on 127.0.0.1.
"""
from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist


def shard_requests(global_ids: Sequence[int], rank: int, world: int) -> List[int]:
    """Contiguous, near-equal shards in global order (rank r gets block r)."""
    n = len(global_ids)
    per, rem = divmod(n, world)
    lo = rank * per + min(rank, rem)
    hi = lo + per + (1 if rank < rem else 0)
    return list(global_ids[lo:hi])


def gather_rows(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather equal-shaped per-rank tensors into [world * rows, ...] in rank order."""
    world = dist.get_world_size(group)
    if local.device.type == "cuda" and dist.get_backend(group) == "nccl":
        out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return out
    host = local.detach().cpu().contiguous()
    out = torch.empty((world * host.shape[0],) + tuple(host.shape[1:]), dtype=host.dtype)
    dist.all_gather(list(out.chunk(world)), host, group=group)
    return out.to(local.device)


def _backend_device(device, group=None):
    return device if dist.get_backend(group) == "nccl" else "cpu"


def max_over_ranks(value: float, device, group=None) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=_backend_device(device, group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, device, group=None) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=_backend_device(device, group))
    dist.all_reduce(t, group=group)
    return float(t.item())
