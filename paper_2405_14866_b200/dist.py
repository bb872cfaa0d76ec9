"""Multi-GPU plumbing for the multi-view workload, torch.distributed only.

Target views are independent units (the autostereoscopic display takes "all
views from leftmost to rightmost"; l.386: each novel view is one F_novel = R_G({G}, Pi_novel)).
The Gaussian set is produced once per frame (rank 0: ta_unproject) and broadcast over
NVLink/NVSwitch (NCCL); every rank renders a contiguous block of the targets; feature images
can be gathered to the display rank.  No collective runs inside a view.

Everything here works with any backend (NCCL on GPUs, gloo on CPU for the tests).
"""
from __future__ import annotations

from typing import List, Optional, Sequence


def shard(n_items: int, rank: int, world: int) -> List[int]:
    """Contiguous block of item indices of `rank` (balanced: sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return list(range(rank * n_items // world, (rank + 1) * n_items // world))


def broadcast_gaussians(tensors: Sequence, n_dev, src: int = 0, group=None, rows: Optional[int] = None) -> Optional[int]:
    """Broadcast a Gaussian set from `src`: the device count n (int64 tensor [1]) and the leading rows of
    each array in `tensors` (pos_alpha, cov, feat).

    With `rows` (a host-side upper bound on n, e.g. the previous frame's count; rows >= n is the
    caller's contract) nothing is read back to the host: the first `rows` rows are broadcast and the
    receivers' ta_rasterize(n = -1) reads the true n from the broadcast n_dev, so the call is fully
    stream-ordered.  Without it, n is read back (one host synchronisation) and exactly n rows are sent.
    Returns n when it was read back, else None."""
    import torch.distributed as dist
    dist.broadcast(n_dev, src, group=group)
    n = rows
    if n is None:
        n = int(n_dev.item())
    for t in tensors:
        if n:
            dist.broadcast(t[:n], src, group=group)
    return None if rows is not None else n


def gather_views(local_views: Sequence, n_views: int, rank: int, world: int, dst: int = 0, group=None):
    """Gather every rank's rendered views (tensors of identical shape) to `dst` in global view
    order; returns the list of n_views tensors on dst, None elsewhere.  When every rank holds the same
    number of views (n_views % world == 0) this is one collective gather (ncclGather over NVLink /
    NVSwitch on GPUs: rank 0's ingress carries (world-1)/world of the bytes) per local view slot;
    otherwise point-to-point send/recv (per-rank counts differ by one)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return list(local_views)
    if n_views % world == 0:
        per = n_views // world
        out = [None] * n_views if rank == dst else None
        for k in range(per):
            t = local_views[k].contiguous()
            if rank == dst:
                bufs = [t if r == dst else torch.empty_like(t) for r in range(world)]
                dist.gather(t, gather_list=bufs, dst=dst, group=group)
                for r in range(world):
                    out[r * per + k] = bufs[r]
            else:
                dist.gather(t, dst=dst, group=group)
        return out
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


class _CAI:
    """__cuda_array_interface__ wrapper of a raw device allocation (so torch can view it)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class PeerFrame:
    """The display rank's frame buffer -- F [n_views, H, W, C] and A [n_views, H, W], fp32 -- mapped into
    every rank's address space with CUDA IPC, so each rank's compositor writes its views' tiles straight
    into the display rank's memory (over NVLink / NVSwitch between GPUs): the render + gather of SURVEY
    8(e)(ii) fused into the compositor's output stores, with no separate gather pass.  Pass
    `view_ptrs(j)` as the feat_out / alpha_out of ta_rasterize_views (integer addresses are accepted).
    Completion: every rank synchronises its stream, then a barrier; after it the display rank reads
    `F` / `A` (torch views of the allocation).  The IPC handles travel by broadcast_object_list, so any
    backend works (NCCL on GPUs, gloo in the tests)."""

    def __init__(self, n_views: int, H: int, W: int, C: int, rank: int, world: int, dst: int = 0, group=None):
        import torch
        import torch.distributed as dist
        from cuda.bindings import runtime as rt
        self._rt = rt
        self.n_views, self.H, self.W, self.C, self.rank, self.dst = n_views, H, W, C, rank, dst
        self.fbytes = H * W * C * 4
        self.abytes = H * W * 4
        self.F = self.A = None
        self._own = []
        self._opened = []
        obj, fail = [None], None
        if rank == dst:
            try:
                err, pf = rt.cudaMalloc(n_views * self.fbytes)
                assert err == rt.cudaError_t.cudaSuccess, err
                self._own.append(pf)
                err, pa = rt.cudaMalloc(n_views * self.abytes)
                assert err == rt.cudaError_t.cudaSuccess, err
                self._own.append(pa)
                self.pF, self.pA = int(pf), int(pa)
                self.F = torch.as_tensor(_CAI(self.pF, (n_views, H, W, C), "<f4"), device="cuda")
                self.A = torch.as_tensor(_CAI(self.pA, (n_views, H, W), "<f4"), device="cuda")
                handles = []
                for p in (pf, pa):
                    err, h = rt.cudaIpcGetMemHandle(p)
                    assert err == rt.cudaError_t.cudaSuccess, err
                    handles.append(bytes(h.reserved))
                obj = [handles]
            except Exception as e:               # still take part in the broadcast, then raise
                fail = e
        if world > 1:
            dist.broadcast_object_list(obj, src=dst, group=group)
        if fail is not None or obj[0] is None:
            self.close()
            raise RuntimeError(f"PeerFrame: the display rank could not export its frame buffer ({fail})")
        if rank != dst:
            ptrs = []
            for hb in obj[0]:
                h = rt.cudaIpcMemHandle_t()
                h.reserved = hb
                err, p = rt.cudaIpcOpenMemHandle(h, rt.cudaIpcMemLazyEnablePeerAccess)
                assert err == rt.cudaError_t.cudaSuccess, err
                ptrs.append(p)
            self._opened = ptrs
            self.pF, self.pA = int(ptrs[0]), int(ptrs[1])

    def view_ptrs(self, j: int):
        """(F, A) device addresses of view j in this rank's mapping of the frame."""
        return self.pF + j * self.fbytes, self.pA + j * self.abytes

    def close(self):
        rt = self._rt
        for p in self._opened:
            rt.cudaIpcCloseMemHandle(p)
        self._opened = []
        self.F = self.A = None
        for p in self._own:
            rt.cudaFree(p)
        self._own = []


def reduce_scalar(x: float, op: str, device=None, group=None) -> float:
    """max / sum of a host scalar over ranks (timing is the max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM, group=group)
    return float(t.item())
