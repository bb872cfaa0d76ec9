#!/usr/bin/env python
"""BASELINE.json configs[4] (stress): 4 x 2048^2 sources (~6.7M Gaussians, log-normal scales
mu = ln 0.008 m, opacity U[0.2, 0.99], C = 64 fp16) rendered to 8 parallax targets at 2048^2 on one
GPU (views over 4 streams / contexts, as bench.py).  CUDA events over K frames after W warm-ups;
one JSON line (dev tool; the bench contract's workload is c4)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(steps=3, warmup=2, nstr=4):
    import torch
    import synthgen as sg
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c5")
    st = torch.cuda.current_stream()
    ctxs = [tb.Context(0) for _ in range(nstr)]
    side = [torch.cuda.Stream() for _ in range(nstr)]
    views, keep = tb.views_to_device(s.views)
    g = tb.GaussianBuffers(s.n_pixels, 64, "f16")
    cams = []
    for c in s.targets:
        K, R, t = sg.cam_arrays(c)
        cams.append((tb.intrinsics(K), tb.extrinsics(R, t)))
    H = W = 2048
    outs = [(torch.empty((H, W, 64), dtype=torch.float32, device="cuda"),
             torch.empty((H, W), dtype=torch.float32, device="cuda")) for _ in range(nstr)]
    psync, pasync = tb.default_params(), tb.default_params(flags=tb.TA_FLAG_ASYNC)
    ctxs[0].unproject(views, psync, g, st)
    kc = k = 0
    for (Ki, Ri) in cams:
        ctxs[0].rasterize(g, -1, Ki, Ri, H, W, psync, outs[0][0], outs[0][1], st)
        d = ctxs[0].debug_last()
        kc, k = max(kc, d.Kc), max(k, d.K)
    for cx in ctxs:
        cx.reserve(s.n_pixels, int(kc * 1.05) + 4096, H, W)

    def frame():
        ctxs[0].unproject(views, psync, g, st)
        ev = torch.cuda.Event()
        ev.record(st)
        for sd in side:
            sd.wait_event(ev)
        for j, (Ki, Ri) in enumerate(cams):
            F, A = outs[j % nstr]
            ctxs[j % nstr].rasterize(g, -1, Ki, Ri, H, W, pasync, F, A, side[j % nstr])
        for sd in side:
            e2 = torch.cuda.Event()
            e2.record(sd)
            st.wait_event(e2)

    for _ in range(warmup):
        frame()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(steps):
        frame()
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    print(json.dumps({"workload": "c5: 4 x 2048^2 sources, C = 64 fp16, 8 targets 2048^2 per frame",
                      "n_gaussians": int(g.n), "tile_entries_per_view": int(k), "ms_per_frame": ms,
                      "ms_per_view": ms / len(cams), "views_per_s": len(cams) * 1e3 / ms}))


if __name__ == "__main__":
    main()
