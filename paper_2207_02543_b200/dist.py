"""Multi-GPU plumbing for instance sharding (torch.distributed).

BASELINE.json: independent instances are sharded across the GPUs of one box
with NO data-path communication; the only collectives are the timing
max-over-ranks and the bookkeeping gathers below (NCCL on the GPU box, gloo
in the CPU tests)."""
from __future__ import annotations

import numpy as np


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_counts(local: np.ndarray, device=None) -> np.ndarray:
    """Concatenate each rank's int64 vector (equal lengths) in rank order."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return np.asarray(local)
    t = torch.as_tensor(np.asarray(local, dtype=np.int64), device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return np.concatenate([o.cpu().numpy() for o in out])
