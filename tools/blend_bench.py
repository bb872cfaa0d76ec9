#!/usr/bin/env python
"""Timing of the paper's blending stage (SURVEY 8(f) NEXT #1 + #2): the four c3 rig views (1024^2)
fused (ta_zbuffer, radius 1) and blended (ta_blend) into a 2048^2 parallax target -- the
resolution the paper blends at.  CUDA events, median of 30 after 5 warm-ups; one JSON line."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import synthgen as sg
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c3")
    cam = sg.make_targets("c4", res=2048, n_targets=3)[1]
    ctx = tb.Context(0)
    st = torch.cuda.current_stream()
    structs, keep = tb.views_to_device(s.views)
    cols = [torch.from_numpy(sg.view_colors(v.cam)).cuda() for v in s.views]
    K, R, t = sg.cam_arrays(cam)
    Ki, Ri = tb.intrinsics(K), tb.extrinsics(R, t)
    zf = torch.empty((cam.H, cam.W), dtype=torch.float32, device="cuda")
    rgb = torch.empty((cam.H, cam.W, 3), dtype=torch.float32, device="cuda")
    ws = torch.empty((cam.H, cam.W), dtype=torch.float32, device="cuda")
    p, bp = tb.default_params(), tb.default_blend_params()

    def zb():
        ctx.zbuffer(structs, p, Ki, Ri, cam.H, cam.W, 1, 0.1, zf, None, st)

    def bl():
        ctx.blend(structs, cols, p, bp, Ki, Ri, cam.H, cam.W, zf, rgb, ws, st)

    out = {}
    for name, fn in (("zbuffer_4x1024_to_2048", zb), ("blend_4views_2048", bl)):
        for _ in range(5):
            fn()
        ts = []
        for _ in range(30):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        out[name] = statistics.median(ts)
    npix = cam.H * cam.W
    filled = float((zf > 0).float().mean())
    # algorithmic bytes of the blend: read z_fused, write rgb + wsum (the per-view gathers hit L2)
    out["blend_alg_bytes"] = npix * (4 + 12 + 4)
    out["blend_GB/s"] = out["blend_alg_bytes"] / (out["blend_4views_2048"] / 1e3) / 1e9
    out["fused_fraction"] = filled
    out["total_ms"] = out["zbuffer_4x1024_to_2048"] + out["blend_4views_2048"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
