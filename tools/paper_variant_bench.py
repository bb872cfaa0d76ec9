#!/usr/bin/env python
"""the paper-exact frame -- lift cam0 + cam2 + cam3 (1024^2, R = I, C = 32 fp16)
and rasterize the viewer's two eye targets (1024^2) -- timed per frame with CUDA events (median of
20 frames after 5 warm-ups; the two eyes on two streams / contexts).  One JSON line (dev tool)."""
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
    s = sg.make_config("paper")
    st = torch.cuda.current_stream()
    ctxs = [tb.Context(0), tb.Context(0)]
    side = [torch.cuda.Stream(), torch.cuda.Stream()]
    views, keep = tb.views_to_device(s.views)
    g = tb.GaussianBuffers(s.n_pixels, 32, "f16")
    outs = [(torch.empty((c.H, c.W, 32), dtype=torch.float32, device="cuda"),
             torch.empty((c.H, c.W), dtype=torch.float32, device="cuda")) for c in s.targets]
    cams = []
    for c in s.targets:
        K, R, t = sg.cam_arrays(c)
        cams.append((tb.intrinsics(K), tb.extrinsics(R, t), c.H, c.W))
    psync, pasync = tb.default_params(), tb.default_params(flags=tb.TA_FLAG_ASYNC)
    ctxs[0].unproject(views, psync, g, st)
    kc = 0
    for cx, (Ki, Ri, H, W), (F, A) in zip(ctxs, cams, outs):
        cx.rasterize(g, -1, Ki, Ri, H, W, psync, F, A, st)
        kc = max(kc, cx.debug_last().Kc)
    for cx in ctxs:
        cx.reserve(s.n_pixels, int(kc * 1.1) + 4096, 1024, 1024)

    def frame():
        ctxs[0].unproject(views, psync, g, st)
        ev = torch.cuda.Event()
        ev.record(st)
        for k, (cx, (Ki, Ri, H, W), (F, A)) in enumerate(zip(ctxs, cams, outs)):
            side[k].wait_event(ev)
            cx.rasterize(g, -1, Ki, Ri, H, W, pasync, F, A, side[k])
        for sd in side:
            e2 = torch.cuda.Event()
            e2.record(sd)
            st.wait_event(e2)

    for _ in range(5):
        frame()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        frame()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    print(json.dumps({"workload": "paper-exact frame: 3 x 1024^2 lifted (R = I) + 2 eye targets 1024^2, C = 32",
                      "n_gaussians": int(g.n), "ms_per_frame": ms, "frames_per_s": 1e3 / ms,
                      "ms_min": min(ts), "ms_p90": sorted(ts)[int(0.9 * len(ts))]}))


if __name__ == "__main__":
    main()
