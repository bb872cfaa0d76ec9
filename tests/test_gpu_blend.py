"""GPU parity of SURVEY 8(f) NEXT #1, occlusion-aware input-view blending (include/ta.h ta_blend;
PAPER.md l.420-444, Eqs. 6-10; R24) against the CPU oracle: colours and weight sums
bit-exact (the kernel follows the oracle's fp32 sequence with explicit rounding intrinsics)."""
import numpy as np
import pytest

import synthgen as sg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    import paper_2405_14866_b200 as tb
    assert torch.cuda.is_available()
    tb.lib(build_if_stale=True)
    return tb.Context(0)


def gpu_blend(ctx, views, colors, cam, radius=1, **bkw):
    import torch
    import paper_2405_14866_b200 as tb
    structs, keep = tb.views_to_device(views)
    cols = [torch.from_numpy(np.ascontiguousarray(c, np.float32)).cuda() for c in colors]
    K, R, t = sg.cam_arrays(cam)
    Ki, Ri = tb.intrinsics(K), tb.extrinsics(R, t)
    zf = torch.empty((cam.H, cam.W), dtype=torch.float32, device="cuda")
    ctx.zbuffer(structs, tb.default_params(), Ki, Ri, cam.H, cam.W, radius, 0.1, zf, None)
    rgb = torch.full((cam.H, cam.W, 3), float("nan"), dtype=torch.float32, device="cuda")
    ws = torch.full((cam.H, cam.W), float("nan"), dtype=torch.float32, device="cuda")
    ctx.blend(structs, cols, tb.default_params(), tb.default_blend_params(**bkw), Ki, Ri, cam.H, cam.W, zf, rgb, ws)
    torch.cuda.synchronize()
    return zf.cpu().numpy(), rgb.cpu().numpy(), ws.cpu().numpy()


def check_bits(a, b):
    same = a.view(np.uint32) == b.view(np.uint32)
    assert same.all(), f"{(~same).sum()} of {same.size} values differ; first {np.argwhere(~same)[:4]}"


def oracle_blend(views, colors, cam, radius=1, **bkw):
    import oracle
    _, zf, _ = oracle.zbuffer(views, cam, 0.1, radius=radius)
    rgb, ws = oracle.blend(views, colors, cam, zf, **bkw)
    return zf, rgb, ws


@pytest.mark.parametrize("tidx", [0, 2])
def test_rig_parallax_targets(ctx, tidx):
    """The textured rig (4 views) blended into parallax targets, reduced resolution."""
    s = sg.make_config("c3", res=256)
    cam = sg.make_targets("c4", res=256, n_targets=3)[tidx]
    colors = [sg.view_colors(v.cam) for v in s.views]
    zf, rgb, ws = gpu_blend(ctx, s.views, colors, cam)
    zo, ro, wo = oracle_blend(s.views, colors, cam)
    check_bits(zf, zo)
    check_bits(ws, wo)
    check_bits(rgb, ro)
    assert (wo > 0).mean() > 0.3


def test_paper_resolution_2048_target(ctx):
    """The paper blends at 2048^2: the four 1024^2 rig views into a 2048^2 target,
    compared bit-exactly on a 512-row band (the oracle's time bound) and for the whole image on
    the hole / weight structure."""
    s = sg.make_config("c3")
    cam = sg.make_targets("c4", res=2048, n_targets=3)[1]
    colors = [sg.view_colors(v.cam) for v in s.views]
    zf, rgb, ws = gpu_blend(ctx, s.views, colors, cam, radius=1)
    band = sg.crop_camera(cam, 0, 768, 2048, 512)
    import oracle
    rb, wb = oracle.blend(s.views, colors, band, zf[768:1280])
    check_bits(ws[768:1280], wb)
    check_bits(rgb[768:1280], rb)


@pytest.mark.parametrize("seed", range(3))
def test_random_scenes_with_textures(ctx, seed):
    rng = np.random.default_rng(100 + seed)
    s = sg.make_random_scene(seed, H=23 + 9 * seed, W=41 - 4 * seed, n_src=24)
    colors = [rng.uniform(0, 1, size=(v.cam.H, v.cam.W, 3)).astype(np.float32) for v in s.views]
    cam = s.targets[0]
    kw = dict(delta=0.05, edge_tau=0.5)
    zf, rgb, ws = gpu_blend(ctx, s.views, colors, cam, **kw)
    zo, ro, wo = oracle_blend(s.views, colors, cam, **kw)
    check_bits(zf, zo)
    check_bits(ws, wo)
    check_bits(rgb, ro)


def test_identity_view_and_errors(ctx):
    """SPEC S:294 / S:310: the novel camera equal to the only input view returns that view's colours
    (x_i.uv = (u, v) up to the fp32 rounding of lift + project, so the bilinear taps are the pixel
    itself to ~1e-6); argument errors are rejected."""
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c2", res=64)
    v = s.views[0]
    col = sg.view_colors(v.cam)
    zf, rgb, ws = gpu_blend(ctx, [v], [col], v.cam, radius=0)
    ok = ws >= 1e-4
    assert ok.mean() > 0.25
    assert np.allclose(rgb[ok], col[ok], atol=1e-4, rtol=0)
    structs, keep = tb.views_to_device([v])
    K, R, t = sg.cam_arrays(v.cam)
    c = torch.from_numpy(col).cuda()
    out = torch.empty((64, 64, 3), dtype=torch.float32, device="cuda")
    z = torch.zeros((64, 64), dtype=torch.float32, device="cuda")
    for bad in (dict(delta=0.0), dict(edge_tau=-1.0), dict(w_min=-1.0)):
        with pytest.raises(tb.TaError):
            ctx.blend(structs, [c], tb.default_params(), tb.default_blend_params(**bad), tb.intrinsics(K),
                      tb.extrinsics(R, t), 64, 64, z, out)


def test_w_min_zero_background_is_zero_not_nan(ctx):
    """w_min = 0: pixels without any weight (background, z_fused = 0) are holes of colour 0 on the GPU
    too (no 0/0), bit-exact against the oracle."""
    s = sg.make_config("c3", res=96)
    cam = sg.make_targets("c4", res=96, n_targets=3)[1]
    colors = [sg.view_colors(v.cam) for v in s.views]
    zf, rgb, ws = gpu_blend(ctx, s.views, colors, cam, w_min=0.0)
    zo, ro, wo = oracle_blend(s.views, colors, cam, w_min=0.0)
    assert np.all(np.isfinite(rgb)) and (ws == 0).sum() > 100
    check_bits(ws, wo)
    check_bits(rgb, ro)


@pytest.mark.parametrize("tau_c", [0.15, 0.0])
def test_appearance_consistency_mask_bit_exact(ctx, tau_c):
    """The appearance-consistency mask (R24): the textured rig with view 2's colours
    shifted by +0.5 in green (an inconsistent view), blended into a parallax target -- colours and weight
    sums bit-exact against the oracle with the mask on (the shifted view is dropped wherever the others
    agree) and off."""
    s = sg.make_config("c3", res=192)
    cam = sg.make_targets("c4", res=192, n_targets=3)[1]
    colors = [sg.view_colors(v.cam) for v in s.views]
    colors[2] = colors[2] + np.float32([0.0, 0.5, 0.0])
    zf, rgb, ws = gpu_blend(ctx, s.views, colors, cam, tau_c=tau_c)
    zo, ro, wo = oracle_blend(s.views, colors, cam, tau_c=tau_c)
    check_bits(ws, wo)
    check_bits(rgb, ro)
    if tau_c > 0:
        zf0, rgb0, ws0 = gpu_blend(ctx, s.views, colors, cam, tau_c=0.0)
        assert (ws < ws0).mean() > 0.05          # the mask removed weight somewhere
