#!/usr/bin/env python
"""north_star (a) front end: ta_render_sources (fused lift + project + cull, one pass over the source
maps) vs ta_unproject + k_project of ta_rasterize, stage times by CUDA events (profile API), for the c3
single target and the paper's two eyes; HBM roofline of the fused pass (dev tool, one JSON line)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(reps=10):
    import torch
    import synthgen as sg
    import paper_2405_14866_b200 as tb
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    out = {}
    for name in ("c3", "paper"):
        s = sg.make_config(name)
        cams = s.targets[:2] if name == "paper" else s.targets[:1]
        views, keep = tb.views_to_device(s.views)
        p = tb.default_params()
        H = W = 1024
        Ks, RTs = [], []
        for c in cams:
            K, R, t = sg.cam_arrays(c)
            Ks.append(tb.intrinsics(K))
            RTs.append(tb.extrinsics(R, t))
        Fs = [torch.empty((H, W, 32), device="cuda") for _ in cams]
        As = [torch.empty((H, W), device="cuda") for _ in cams]
        cf = tb.Context(0)
        cf.render_sources(views, 32, "f16", p, Ks, RTs, H, W, Fs, As)
        cf.profile(True)
        cf.profile_read(reset=True)
        for _ in range(reps):
            cf.render_sources(views, 32, "f16", p, Ks, RTs, H, W, Fs, As)
        pf = cf.profile_read(reset=True)
        cf.profile(False)
        c2 = tb.Context(0)
        g = tb.GaussianBuffers(s.n_pixels, 32, "f16")
        c2.unproject(views, p, g)
        c2.rasterize(g, -1, Ks[0], RTs[0], H, W, p, Fs[0], As[0])
        c2.profile(True)
        c2.profile_read(reset=True)
        for _ in range(reps):
            c2.unproject(views, p, g)
            for k, r in zip(Ks, RTs):
                c2.rasterize(g, -1, k, r, H, W, p, Fs[0], As[0])
        p2 = c2.profile_read(reset=True)
        c2.profile(False)
        torch.cuda.synchronize()
        n = g.n
        px = s.n_pixels
        fused_ms = pf["project"][0] / reps
        two_ms = p2["unproject"][0] / reps + p2["project"][0] / reps
        # fused: read disparity 4 + mask 1 + scale 12 + quat 16 (or 0) + opacity 4 + features 2C per source
        # pixel (features only for lifted ones), write 2C + T (32 + 8) per lifted Gaussian
        qb = 16 if s.views[0].quat is not None else 0
        b = px * (4 + 1 + 12 + qb + 4) + n * 64 + n * (64 + len(cams) * 40)
        out[name] = {"targets": len(cams), "gaussians": int(n), "fused_front_ms": fused_ms,
                     "two_call_front_ms": two_ms, "fused_alg_bytes": int(b),
                     "fused_hbm_frac": b / (fused_ms / 1e3) / 1e9 / float(peaks["hbm_gbs"])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
