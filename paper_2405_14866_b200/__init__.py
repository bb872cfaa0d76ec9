"""paper_2405_14866_b200 -- B200-native latent-Gaussian rasterizer of Tele-Aloha (arXiv 2405.14866).

The hot path (lift foreground pixels to latent Gaussians, EWA-project them
to the novel view, bin to 16x16 tiles, order by (tile, depth, id), composite front to back) runs
in libtaloha.so -- hand-written CUDA for sm_100a behind the C ABI of include/ta.h.  This
package is the thin Python binding (argument marshalling) plus the multi-GPU harness
(torch.distributed over NCCL: broadcast of the Gaussian set, target views sharded by rank).

    ctx = Context(0)
    g = unproject(ctx, views, C=32, feat_dtype="f16", params=default_params())
    F, A = rasterize(ctx, g, K, R, t, H, W, params)
"""
from __future__ import annotations

from ._lib import (TA_FLAG_ASYNC, TA_FLAG_DEBUG_COUNTS, Context, GaussianBuffers, TaError, default_params,
                   default_blend_params,
                   extrinsics, intrinsics, lib, source_view)

__all__ = ["Context", "GaussianBuffers", "TaError", "default_params", "unproject", "rasterize", "views_to_device",
           "lib", "TA_FLAG_ASYNC", "TA_FLAG_DEBUG_COUNTS"]


def views_to_device(views, device="cuda"):
    """Upload source views (objects with .cam, .baseline, .disparity, .mask, .scale, .quat,
    .opacity, .feat numpy arrays, e.g. synthgen.SourceView) to CUDA tensors.  Returns
    (structs, keepalive) -- keep `keepalive` referenced while the structs are in use."""
    import numpy as np
    import torch

    def up(a):
        return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(device)

    structs, keep = [], []
    for v in views:
        t = [up(v.disparity), up(v.mask), up(v.scale), up(v.quat), up(v.opacity), up(v.feat)]
        keep.append(t)
        cam = v.cam
        structs.append(source_view(cam.H, cam.W, t[0], t[1], (cam.fx, cam.fy, cam.cx, cam.cy),
                                   np.asarray(cam.R, np.float32).reshape(9), np.asarray(cam.t, np.float32),
                                   v.baseline, t[2], t[3], t[4], t[5]))
    return structs, keep


def unproject(ctx: Context, view_structs, C: int, feat_dtype: str, params, capacity=None, out=None,
              stream=None) -> GaussianBuffers:
    """a1: ta_unproject over the given source views -> Gaussian buffers (count in .n_dev)."""
    if out is None:
        cap = capacity if capacity is not None else sum(int(v.H) * int(v.W) for v in view_structs)
        out = GaussianBuffers(cap, C, feat_dtype)
    ctx.unproject(view_structs, params, out, stream)
    return out


def rasterize(ctx: Context, g: GaussianBuffers, K, R, t, H: int, W: int, params, n: int = -1, out=None,
              stream=None):
    """a2-a6: ta_rasterize into (F [H,W,C] fp32 HWC, A [H,W] fp32) CUDA tensors."""
    import torch
    if out is None:
        out = (torch.empty((H, W, g.C), dtype=torch.float32, device=g.pos_alpha.device),
               torch.empty((H, W), dtype=torch.float32, device=g.pos_alpha.device))
    F, A = out
    ctx.rasterize(g, n, intrinsics(K), extrinsics(R, t), H, W, params, F, A, stream)
    return F, A
