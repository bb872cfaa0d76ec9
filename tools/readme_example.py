#!/usr/bin/env python
"""The README's Python example, runnable (GPU): lift the c3 rig and render one target (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import synthgen as sg  # noqa: E402
import paper_2405_14866_b200 as tb  # noqa: E402

ctx = tb.Context(0)
scene = sg.make_config("c3")                                  # seeded 4 x 1024^2 rig, C = 32 fp16
views, keep = tb.views_to_device(scene.views)
g = tb.GaussianBuffers(scene.n_pixels, scene.C, scene.feat_dtype)
ctx.unproject(views, tb.default_params(), g)                  # a1: pixels -> Gaussians
K, R, t = sg.cam_arrays(scene.targets[0])
F = torch.empty((1024, 1024, scene.C), device="cuda")
A = torch.empty((1024, 1024), device="cuda")
ctx.rasterize(g, -1, tb.intrinsics(K), tb.extrinsics(R, t), 1024, 1024, tb.default_params(), F, A)
torch.cuda.synchronize()
print(f"n = {g.n}, alpha > 0 on {(A > 0).float().mean().item():.3f} of the pixels, |F| max {F.abs().max().item():.3f}")
# steady state: size the scratch once, then render without host synchronisation (and many views per call)
ctx.reserve(g.capacity, int(ctx.debug_last().Kc * 1.3), 1024, 1024)
fast = tb.default_params(flags=tb.TA_FLAG_ASYNC)
cams = [sg.cam_arrays(c) for c in sg.make_targets("c4")]             # the 32 parallax targets
Fs = [torch.empty((1024, 1024, scene.C), device="cuda") for _ in cams]
As = [torch.empty((1024, 1024), device="cuda") for _ in cams]
ctx.rasterize_views(g, -1, [tb.intrinsics(k) for k, _, _ in cams], [tb.extrinsics(r, t) for _, r, t in cams],
                    1024, 1024, fast, Fs, As, lanes=4)
assert not ctx.check_overflow()
torch.cuda.synchronize()
print("readme example ok: A(target 0) max", float(A.max()), "views", len(Fs), "A(view 16) max", float(As[16].max()))

