"""GPU parity of SURVEY 8(f) NEXT #2, the cascade Z-buffer (include/ta.h ta_zbuffer; PAPER.md
l.351-352, R23) against the CPU oracle: depth and disparity bit-exact
(the same fp32 lifting / projection sequence and the same integer min-z decision on both sides)."""
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


def gpu_zbuffer(ctx, views, cam, baseline, radius, with_disp=True, params=None):
    import torch
    import paper_2405_14866_b200 as tb
    structs, keep = tb.views_to_device(views)
    K, R, t = sg.cam_arrays(cam)
    depth = torch.full((cam.H, cam.W), float("nan"), dtype=torch.float32, device="cuda")
    disp = torch.full((cam.H, cam.W), float("nan"), dtype=torch.float32, device="cuda") if with_disp else None
    ctx.zbuffer(structs, params or tb.default_params(), tb.intrinsics(K), tb.extrinsics(R, t), cam.H, cam.W, radius,
                baseline, depth, disp)
    torch.cuda.synchronize()
    return depth.cpu().numpy(), (disp.cpu().numpy() if with_disp else None)


def check_bits(gpu, ref):
    assert gpu.shape == ref.shape
    same = gpu.view(np.uint32) == ref.view(np.uint32)
    assert same.all(), f"{(~same).sum()} of {same.size} pixels differ; first {np.argwhere(~same)[:5]}"


@pytest.mark.parametrize("radius", [0, 1, 2])
def test_cascade_cam0_to_lower_pair(ctx, radius):
    """The paper's use: cam0's depth into cam2 and cam3 (reduced rig, ragged sizes)."""
    import oracle
    s = sg.make_config("c3", res=256)
    for k in (2, 3):
        tgt = s.views[k]
        cam = sg.crop_camera(tgt.cam, 3, 5, 241, 250)
        d, disp = gpu_zbuffer(ctx, [s.views[0]], cam, tgt.baseline, radius)
        _, dref, dispref = oracle.zbuffer([s.views[0]], cam, tgt.baseline, radius=radius)
        assert (dref > 0).mean() > 0.1
        check_bits(d, dref)
        check_bits(disp, dispref)


def test_full_size_cascade(ctx):
    """BASELINE configs[2] resolution: 1024^2 cam0 -> cam2, radius 1 (SPEC default)."""
    import oracle
    s = sg.make_config("c3")
    tgt = s.views[2]
    d, disp = gpu_zbuffer(ctx, [s.views[0]], tgt.cam, tgt.baseline, 1)
    _, dref, dispref = oracle.zbuffer([s.views[0]], tgt.cam, tgt.baseline, radius=1)
    check_bits(d, dref)
    check_bits(disp, dispref)


def test_multi_view_fusion_into_novel_view(ctx):
    """All four views into the parallax target (the fused-depth use of Eq. 6's z_fused)."""
    import oracle
    s = sg.make_config("c3", res=128)
    cam = sg.make_targets("c4", res=128, n_targets=3)[1]
    d, _ = gpu_zbuffer(ctx, s.views, cam, 0.1, 1, with_disp=False)
    _, dref, _ = oracle.zbuffer(s.views, cam, 0.1, radius=1)
    check_bits(d, dref)


@pytest.mark.parametrize("seed", range(4))
def test_random_scenes(ctx, seed):
    """Random disparities / masks / rotated targets, ragged sizes."""
    import oracle
    s = sg.make_random_scene(seed, H=19 + 7 * seed, W=33 - 3 * seed, n_src=20 + 5 * seed)
    cam = s.targets[0]
    d, disp = gpu_zbuffer(ctx, s.views, cam, 0.1, seed % 3)
    _, dref, dispref = oracle.zbuffer(s.views, cam, 0.1, radius=seed % 3)
    check_bits(d, dref)
    check_bits(disp, dispref)


def test_edge_cases(ctx):
    """A point on the optical axis, an empty source (all invalid -> all zero), and the
    argument errors."""
    import torch
    import paper_2405_14866_b200 as tb
    disp = np.zeros((1, 1), np.float32)
    disp[0, 0] = np.float32(100.0 * 0.2 / 2.0)
    src = sg.Camera(fx=100.0, fy=100.0, cx=0.0, cy=0.0, R=np.eye(3), t=np.zeros(3), H=1, W=1)
    v = sg.SourceView(cam=src, baseline=0.2, disparity=disp, mask=None, scale=None, quat=None, opacity=None,
                      feat=np.zeros((1, 1, 8), np.float32))
    tgt = sg.Camera(fx=100.0, fy=100.0, cx=7.0, cy=5.0, R=np.eye(3), t=np.zeros(3), H=11, W=15)
    d, dd = gpu_zbuffer(ctx, [v], tgt, 0.2, 0)
    assert np.count_nonzero(d) == 1 and d[5, 7] == np.float32(2.0) and dd[5, 7] == np.float32(10.0)
    v0 = sg.SourceView(cam=src, baseline=0.2, disparity=np.full((1, 1), -1.0, np.float32), mask=None, scale=None,
                       quat=None, opacity=None, feat=np.zeros((1, 1, 8), np.float32))
    d0, dd0 = gpu_zbuffer(ctx, [v0], tgt, 0.2, 1)
    assert not d0.any() and not dd0.any()
    structs, keep = tb.views_to_device([v])
    K, R, t = sg.cam_arrays(tgt)
    out = torch.empty((11, 15), dtype=torch.float32, device="cuda")
    for radius, base in ((9, 0.2), (-1, 0.2), (1, 0.0)):
        with pytest.raises(tb.TaError):
            ctx.zbuffer(structs, tb.default_params(), tb.intrinsics(K), tb.extrinsics(R, t), 11, 15, radius, base,
                        out, out)
