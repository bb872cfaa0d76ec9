#!/usr/bin/env python
"""One c5 view (4 x 2048^2 sources, C = 64, 2048^2 target) through ta_unproject + ta_rasterize, for
profiling the stress configuration (ncu launch lists).  Dev tool."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import synthgen as sg  # noqa: E402
import paper_2405_14866_b200 as tb  # noqa: E402

s = sg.make_config("c5", n_targets=1)
st = torch.cuda.current_stream()
ctx = tb.Context(0)
views, keep = tb.views_to_device(s.views)
g = tb.GaussianBuffers(s.n_pixels, 64, "f16")
p = tb.default_params()
ctx.unproject(views, p, g, st)
cam = s.targets[0]
K, R, t = sg.cam_arrays(cam)
F = torch.empty((cam.H, cam.W, 64), dtype=torch.float32, device="cuda")
A = torch.empty((cam.H, cam.W), dtype=torch.float32, device="cuda")
for _ in range(2):
    ctx.rasterize(g, -1, tb.intrinsics(K), tb.extrinsics(R, t), cam.H, cam.W, p, F, A, st)
torch.cuda.synchronize()
