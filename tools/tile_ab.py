"""A/B of the compositing tile side on the c3 Gaussian set rendered into c4 targets (dev tool): 8 x 8
tiles (default under 32-px coarse bins) vs 16 x 16 (TA_TILE_PX=16) -- F and A bit-identical, per-stage
CUDA-event times (one stream, serialized), the compositor's work counters, tile entries K."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import synthgen as sg
import paper_2405_14866_b200 as tb


def ctx_with(env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    c = tb.Context(0)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    return c


def main():
    nv = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    s = sg.make_config("c3")
    targets = sg.make_targets("c4", n_targets=32)[::32 // nv][:nv]
    arms = {"t16": ctx_with({"TA_TILE_PX": "16"}), "t8": ctx_with({"TA_TILE_PX": "8"})}
    p = tb.default_params()
    views, keep = tb.views_to_device(s.views)
    g = tb.unproject(arms["t8"], views, 32, "f16", p)
    torch.cuda.synchronize()
    H = W = 1024
    res = {}
    for name, cx in arms.items():
        outs = []
        for cam in targets:
            K, R, t = sg.cam_arrays(cam)
            outs.append(tb.rasterize(cx, g, K, R, t, H, W, p))
        torch.cuda.synchronize()
        cx.profile(True)
        cx.profile_read(reset=True)
        for _ in range(reps):
            for cam, (F, A) in zip(targets, outs):
                K, R, t = sg.cam_arrays(cam)
                tb.rasterize(cx, g, K, R, t, H, W, p, out=(F, A))
        prof = cx.profile_read(reset=True)
        cx.profile(False)
        cam = targets[0]
        K, R, t = sg.cam_arrays(cam)
        tb.rasterize(cx, g, K, R, t, H, W, tb.default_params(flags=tb.TA_FLAG_DEBUG_COUNTS))
        torch.cuda.synchronize()
        d = cx.debug_last()
        res[name] = dict(outs=outs, stages={k: round(v[0] / max(1, v[1]), 4) for k, v in prof.items()},
                         work=dict(zip(("read", "staged", "evaluated", "any_q", "accumulated", "pairs", "warps",
                                        "fill_rounds"), [int(x) for x in d.work])),
                         K=int(d.K), Kc=int(d.Kc), tile_px=int(d.tile_px))
    sameA = all(torch.equal(Aa.view(torch.int32), Ab.view(torch.int32))
                for (_, Aa), (_, Ab) in zip(res["t8"]["outs"], res["t16"]["outs"]))
    dF = max(float((Fa - Fb).abs().max()) for (Fa, _), (Fb, _) in zip(res["t8"]["outs"], res["t16"]["outs"]))
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "outs"} for k, v in res.items()}, indent=1))
    print("A bit-identical between tile sides:", sameA, " max|dF|:", dF)


if __name__ == "__main__":
    main()
