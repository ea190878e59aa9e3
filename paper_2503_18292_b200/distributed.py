"""Multi-GPU plumbing: requests shard across ranks with no data-path
collective (engine instances share nothing, reference SPEC.md:535); one
all-gather after the timed region collects outputs for verification.

One process per GPU, torch.distributed with NCCL on GPUs (gloo in the CPU
tests).  Rendezvous on 127.0.0.1.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from typing import Dict, List, Optional, Sequence

import torch
import torch.distributed as dist


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_local_ranks(script: str, argv: Sequence[str], nprocs: int, env: Optional[Dict[str, str]] = None) -> int:
    """Run `script argv` as `nprocs` ranks of one node (one process per GPU)
    through torch.distributed.run with a 127.0.0.1 rendezvous — what
    `bench.py --gpus N` does when it is not already inside a launcher.  NCCL
    logs its INFO lines (rank / channel / transport setup) to stderr so rank
    0's stdout stays one JSON line.  Returns the launcher's exit code."""
    e = dict(os.environ if env is None else env)
    e.setdefault("NCCL_DEBUG", "INFO")
    e.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nprocs}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", script, *argv]
    return subprocess.run(cmd, env=e).returncode


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


def gather_padded(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather 1-D uint8 payloads of different lengths: pad to the longest
    (one MAX all-reduce for the length), gather [world, max_len]."""
    n = torch.tensor([local.numel()], dtype=torch.int64, device=_backend_device(local.device, group))
    dist.all_reduce(n, op=dist.ReduceOp.MAX, group=group)
    buf = torch.zeros(int(n.item()), dtype=torch.uint8, device=local.device)
    buf[: local.numel()] = local
    return gather_rows(buf.view(1, -1), group)


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
