#!/usr/bin/env python
"""Timing of the compositing backward pass on c3 (1.67M Gaussians, 1024^2,
C = 32): ta_rasterize then ta_rasterize_backward with random dL/dF, dL/dA; CUDA events, median of 10
after 3 warm-ups.  One JSON line (dev tool)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import synthgen as sg
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c3")
    st = torch.cuda.current_stream()
    ctx = tb.Context(0)
    views, keep = tb.views_to_device(s.views)
    g = tb.GaussianBuffers(s.n_pixels, 32, "f16")
    p = tb.default_params()
    ctx.unproject(views, p, g, st)
    cam = s.targets[0]
    K, R, t = sg.cam_arrays(cam)
    Ki, Ri = tb.intrinsics(K), tb.extrinsics(R, t)
    H, W, C = cam.H, cam.W, 32
    F = torch.empty((H, W, C), dtype=torch.float32, device="cuda")
    A = torch.empty((H, W), dtype=torch.float32, device="cuda")
    gF = torch.randn((H, W, C), dtype=torch.float32, device="cuda")
    gA = torch.randn((H, W), dtype=torch.float32, device="cuda")
    n = g.n
    dm = torch.empty((n, 2), device="cuda")
    dc = torch.empty((n, 3), device="cuda")
    da = torch.empty((n,), device="cuda")
    dfe = torch.empty((n, C), device="cuda")
    fw, bw = [], []
    for it in range(13):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        ctx.rasterize(g, -1, Ki, Ri, H, W, p, F, A, st)
        e1.record(st)
        ctx.rasterize_backward(g, -1, H, W, p, gF, gA, dm, dc, da, dfe, st)
        e2.record(st)
        e2.synchronize()
        if it >= 3:
            fw.append(e0.elapsed_time(e1))
            bw.append(e1.elapsed_time(e2))
    print(json.dumps({"workload": "c3 view: 1.67M Gaussians, 1024^2, C = 32", "forward_ms": statistics.median(fw),
                      "backward_ms": statistics.median(bw)}))


if __name__ == "__main__":
    main()
