"""Compositor stage time of the default compositor on the c3 Gaussian set rendered into 4 of the c4
targets (dev tool for A/B of build variants): CUDA-event stage times (one stream, serialized), plus a
digest of every F / A bit so variants can be checked for identical output."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import synthgen as sg
import paper_2405_14866_b200 as tb


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    nv = int(args[0]) if len(args) > 0 else 4
    reps = int(args[1]) if len(args) > 1 else 5
    s = sg.make_config("c3")
    f32 = "--f32" in sys.argv
    if f32:                                   # fp32-stored features: the SIMT compositor
        for v in s.views:
            v.feat = v.feat.astype("float32")
        s.feat_dtype = "f32"
    targets = sg.make_targets("c4", n_targets=32)[::32 // nv][:nv]
    cx = tb.Context(0)
    p = tb.default_params()
    views, keep = tb.views_to_device(s.views)
    g = tb.unproject(cx, views, 32, "f32" if f32 else "f16", p)
    torch.cuda.synchronize()
    H = W = 1024
    outs = []
    for cam in targets:
        K, R, t = sg.cam_arrays(cam)
        outs.append(tb.rasterize(cx, g, K, R, t, H, W, p))
    torch.cuda.synchronize()
    h = hashlib.sha256()
    for F, A in outs:
        h.update(F.cpu().numpy().tobytes())
        h.update(A.cpu().numpy().tobytes())
    cx.profile(True)
    cx.profile_read(reset=True)
    for _ in range(reps):
        for cam, (F, A) in zip(targets, outs):
            K, R, t = sg.cam_arrays(cam)
            tb.rasterize(cx, g, K, R, t, H, W, p, out=(F, A))
    prof = cx.profile_read(reset=True)
    print(json.dumps({"stages_ms": {k: round(v[0] / max(1, v[1]), 4) for k, v in prof.items()},
                      "digest": h.hexdigest()[:16], "tag": os.environ.get("TAG", "")}))


if __name__ == "__main__":
    main()
