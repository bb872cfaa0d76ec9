"""Multi-GPU plumbing for the multi-view workload, torch.distributed only.

Target views are independent units (the autostereoscopic display takes "all
views from leftmost to rightmost"; l.386: each novel view is one F_novel = R_G({G}, Pi_novel)).
The Gaussian set is produced once per frame (rank 0: ta_unproject) and broadcast over
NVLink/NVSwitch (NCCL); every rank renders a contiguous block of the targets; feature images
can be gathered to the display rank.  No collective runs inside a view.

Everything here works with any backend (NCCL on GPUs, gloo on CPU for the tests).
"""
from __future__ import annotations

from typing import List, Sequence


def shard(n_items: int, rank: int, world: int) -> List[int]:
    """Contiguous block of item indices of `rank` (balanced: sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return list(range(rank * n_items // world, (rank + 1) * n_items // world))


def broadcast_gaussians(tensors: Sequence, n_dev, src: int = 0, group=None) -> int:
    """Broadcast a Gaussian set from `src`: first the device count n (int64 tensor [1]), then the
    first n rows of each array in `tensors` (pos_alpha, cov, feat).  Returns n."""
    import torch.distributed as dist
    dist.broadcast(n_dev, src, group=group)
    n = int(n_dev.item())
    for t in tensors:
        if n:
            dist.broadcast(t[:n], src, group=group)
    return n


def gather_views(local_views: Sequence, n_views: int, rank: int, world: int, dst: int = 0, group=None):
    """Gather every rank's rendered views (tensors of identical shape) to `dst` in global view
    order; returns the list of n_views tensors on dst, None elsewhere.  Uses point-to-point
    send/recv so per-rank counts may differ by one."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return list(local_views)
    if rank == dst:
        out = [None] * n_views
        for r in range(world):
            idx = shard(n_views, r, world)
            for k, j in enumerate(idx):
                if r == dst:
                    out[j] = local_views[k]
                else:
                    buf = torch.empty_like(local_views[0]) if local_views else None
                    if buf is None:
                        raise ValueError("dst rank needs at least one local view to size buffers")
                    dist.recv(buf, src=r, group=group)
                    out[j] = buf
        return out
    for t in local_views:
        dist.send(t.contiguous(), dst=dst, group=group)
    return None


def reduce_scalar(x: float, op: str, device=None, group=None) -> float:
    """max / sum of a host scalar over ranks (timing is the max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM, group=group)
    return float(t.item())
