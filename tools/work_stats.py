#!/usr/bin/env python
"""Compositor work counters on one c4 target (GPU; dev tool, not part of the product path).

Prints ta_debug_view.work (TA_FLAG_DEBUG_COUNTS) and per-8x8-block statistics of the per-pixel
composited-pair counts, i.e. how much of each warp's walk is shared by its 64 pixels."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import synthgen as sg
    import paper_2405_14866_b200 as tb
    from tests import _parity as P

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    ctx = tb.Context(0)
    scene = sg.make_config(cfg)
    C_ = scene.C
    g = tb.GaussianBuffers(scene.n_pixels, C_, scene.feat_dtype, device=dev)
    views, keep = tb.views_to_device(scene.views, device=dev)
    ctx.unproject(views, tb.default_params(), g, stream)
    cam = sg.make_targets("c4")[0] if cfg == "c3" else scene.targets[0]
    K, R, t = sg.cam_arrays(cam)
    Ki, Ri = tb.intrinsics(K), tb.extrinsics(R, t)
    H, W = cam.H, cam.W
    F = torch.empty((H, W, C_), dtype=torch.float32, device=dev)
    A = torch.empty((H, W), dtype=torch.float32, device=dev)
    ctx.rasterize(g, -1, Ki, Ri, H, W, tb.default_params(flags=tb.TA_FLAG_DEBUG_COUNTS), F, A, stream)
    torch.cuda.synchronize()
    d = ctx.debug_last()
    wk = [int(x) for x in d.work]
    nc = P.d2h(d.n_contrib, H * W, np.int32).reshape(H, W).astype(np.int64)
    names = ["list_read", "staged", "evaluated", "any_q", "accumulated", "pairs", "warps", "fill_rounds"]
    out = dict(zip(names, wk))
    out["K"] = int(d.K)
    out["Kc"] = int(d.Kc)
    out["pairs_check"] = int(nc.sum())
    Hb, Wb = (H + 7) // 8 * 8, (W + 7) // 8 * 8
    pad = np.zeros((Hb, Wb), np.int64)
    pad[:H, :W] = nc
    blk = pad.reshape(Hb // 8, 8, Wb // 8, 8).transpose(0, 2, 1, 3).reshape(-1, 64)
    nz = blk.max(1) > 0
    b = blk[nz]
    out["blocks_nonempty"] = int(nz.sum())
    out["px_nonzero"] = int((nc > 0).sum())
    out["pairs_per_px_nonzero"] = float(nc[nc > 0].mean())
    out["block_mean_of_max"] = float(b.max(1).mean())
    out["block_mean_of_mean"] = float(b.mean(1).mean())
    out["lane_util_accum"] = wk[5] / max(1, 64 * wk[4])
    out["lane_util_eval"] = wk[5] / max(1, 64 * wk[2])
    Aa = A.cpu().numpy()
    out["A_gt_0.9999"] = float((Aa > 1 - 1.0001e-4).mean())
    out["A_zero"] = float((Aa == 0).mean())
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
