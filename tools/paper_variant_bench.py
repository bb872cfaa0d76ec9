#!/usr/bin/env python
"""the paper-exact frame -- lift cam0 + cam2 + cam3 (1024^2, R = I, C = 32 fp16)
and rasterize the viewer's two eye targets (1024^2) -- timed per frame with CUDA events (median of
20 frames after 5 warm-ups).  Two paths: the two-call API (ta_unproject, then ta_rasterize per eye on
two streams / contexts) and the fused front end (ta_render_sources with both eyes in one call, one
stream).  256 MB L2 flush between frames.  One JSON line (dev tool)."""
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

    cf = tb.Context(0)
    fouts = [(torch.empty((c.H, c.W, 32), dtype=torch.float32, device="cuda"),
              torch.empty((c.H, c.W), dtype=torch.float32, device="cuda")) for c in s.targets]
    Ks, RTs = [c[0] for c in cams], [c[1] for c in cams]
    cf.render_sources(views, 32, "f16", psync, Ks, RTs, 1024, 1024, [o[0] for o in fouts], [o[1] for o in fouts], st)

    def frame_fused():
        cf.render_sources(views, 32, "f16", pasync, Ks, RTs, 1024, 1024, [o[0] for o in fouts], [o[1] for o in fouts], st)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def timed(fn):
        for _ in range(5):
            fn()
        ts = []
        for _ in range(20):
            flush.add_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        return {"median": ts[len(ts) // 2], "min": ts[0], "p90": ts[int(0.9 * len(ts))]}

    def frame_one_stream():
        ctxs[0].unproject(views, psync, g, st)
        for (Ki, Ri, H, W), (F, A) in zip(cams, outs):
            ctxs[0].rasterize(g, -1, Ki, Ri, H, W, pasync, F, A, st)

    two = timed(frame)
    two1 = timed(frame_one_stream)
    fus = timed(frame_fused)
    same = all(torch.equal(a.view(torch.int32), b.view(torch.int32)) for (a, _), (b, _) in zip(outs, fouts)) and \
        all(torch.equal(a.view(torch.int32), b.view(torch.int32)) for (_, a), (_, b) in zip(outs, fouts))
    print(json.dumps({"workload": "paper-exact frame: 3 x 1024^2 lifted (R = I) + 2 eye targets 1024^2, C = 32",
                      "n_gaussians": int(g.n), "two_call_ms": two, "two_call_one_stream_ms": two1, "fused_ms": fus,
                      "frames_per_s": {"two_call": 1e3 / two["median"], "fused": 1e3 / fus["median"]},
                      "outputs_bit_identical": bool(same)}))


if __name__ == "__main__":
    main()
