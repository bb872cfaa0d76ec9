#!/usr/bin/env python
"""Timing of ta_zbuffer on the paper's use: cam0 (1024^2, c3 rig) lifted and
splatted into cam2 and cam3 (radius 1).  CUDA events around the call on its stream, median of 50
after 10 warm-ups; prints one JSON line (dev tool, not the bench contract)."""
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
    ctx = tb.Context(0)
    stream = torch.cuda.current_stream()
    structs, keep = tb.views_to_device([s.views[0]])
    outs = {}
    for k in (2, 3):
        cam = s.views[k].cam
        K, R, t = sg.cam_arrays(cam)
        d = torch.empty((cam.H, cam.W), dtype=torch.float32, device="cuda")
        dd = torch.empty_like(d)
        args = (structs, tb.default_params(), tb.intrinsics(K), tb.extrinsics(R, t), cam.H, cam.W, 1,
                s.views[k].baseline, d, dd, stream)
        for _ in range(10):
            ctx.zbuffer(*args)
        ts = []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.zbuffer(*args)
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        valid = int((s.views[0].mask != 0).sum())
        HW_s, HW_t = 1024 * 1024, cam.H * cam.W
        # algorithmic bytes: read disparity + mask of every source pixel, one 8-B z-buffer word per
        # target pixel cleared, read and resolved, depth + disparity written
        alg = HW_s * 5 + HW_t * (8 + 8 + 8)
        ms = statistics.median(ts)
        outs[f"cam0->cam{k}"] = {"ms": ms, "alg_bytes": alg, "GB/s": alg / (ms / 1e3) / 1e9,
                                 "lifted_points": valid, "atomics_max": valid * 9}
    print(json.dumps(outs))


if __name__ == "__main__":
    main()
