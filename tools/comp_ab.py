"""A/B of the compositors on the c4 workload (dev tool): the tensor-memory compositor (TA_COMPOSITOR=2) vs
the default mma.sync one on the same Gaussian set and targets -- A bit-identical, max |dF|, and
per-stage CUDA-event times (one stream, serialized)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import synthgen as sg
import paper_2405_14866_b200 as tb


def ctx_with(comp):
    os.environ["TA_COMPOSITOR"] = str(comp)
    c = tb.Context(0)
    os.environ.pop("TA_COMPOSITOR")
    return c


def main():
    nv = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    fast = "--fast" in sys.argv
    s = sg.make_config("c3")
    targets = sg.make_targets("c4", n_targets=32)[::32 // nv][:nv]
    c0 = ctx_with(2)      # tensor-memory compositor
    c1 = ctx_with(0)      # mma.sync compositor (default)
    p = tb.default_params()
    views, keep = tb.views_to_device(s.views)
    g = tb.unproject(c0, views, 32, "f16", p)
    torch.cuda.synchronize()
    H = W = 1024
    res = {}
    for name, cx in (("tm", c0), ("mma", c1)):
        outs = []
        pp = tb.default_params(exact_exp=0 if (fast and name == "tm") else 1)
        for cam in targets:
            K, R, t = sg.cam_arrays(cam)
            outs.append(tb.rasterize(cx, g, K, R, t, H, W, pp))
        torch.cuda.synchronize()
        cx.profile(True)
        cx.profile_read(reset=True)
        for _ in range(reps):
            for cam, (F, A) in zip(targets, outs):
                K, R, t = sg.cam_arrays(cam)
                tb.rasterize(cx, g, K, R, t, H, W, pp, out=(F, A))
        prof = cx.profile_read(reset=True)
        cx.profile(False)
        res[name] = (outs, {k: v[0] / max(1, v[1]) for k, v in prof.items()})
    for k in ("tm", "mma"):
        print(k, {a: round(b, 4) for a, b in res[k][1].items()})
    cam = targets[0]
    K, R, t = sg.cam_arrays(cam)
    tb.rasterize(c0, g, K, R, t, H, W, tb.default_params(flags=tb.TA_FLAG_DEBUG_COUNTS))
    torch.cuda.synchronize()
    wk = list(c0.debug_last().work)
    print("tm counters: entries read %d staged %d chunks %d fill steps %d" % (wk[0], wk[1], wk[6], wk[7]))
    tot = wk[2] + wk[3]
    if tot:
        print("warp cycles: fill %.3f composite %.3f (wait-before-store %.3f, idle waits %.3f) [fractions]" % (
            wk[2] / tot, wk[3] / tot, wk[4] / tot, wk[5] / tot))
    for (Ft, At), (Fm, Am) in zip(res["tm"][0], res["mma"][0]):
        da = int((At.view(torch.int32) != Am.view(torch.int32)).sum())
        df = float((Ft - Fm).abs().max())
        print(f"A mismatches {da}  max|dF| {df:.3e}  A>0.5 frac {float((At > 0.5).float().mean()):.3f}")


if __name__ == "__main__":
    main()
