"""GPU parity of SURVEY 8(f) NEXT #4, the compositing backward pass (include/ta.h
ta_rasterize_backward; R25) against the CPU oracle's gradients (same fp32 per-pixel terms;
the GPU sums pixels with fp32 shuffles + atomics in no fixed order, the oracle in double):
every gradient within 1e-4 relative to the largest of its kind (+ 1e-6 absolute)."""
import numpy as np
import pytest

import synthgen as sg
from tests import _parity as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    import paper_2405_14866_b200 as tb
    assert torch.cuda.is_available()
    tb.lib(build_if_stale=True)
    return tb.Context(0)


def run_case(ctx, scene, seed=0):
    import torch
    import oracle
    gp = P.gpu_params(scene, flags=0)
    op = P.oracle_params(scene)
    g = P.gpu_unproject(ctx, scene, gp)
    go = oracle.unproject(scene, op)
    P.check_unproject(P.gaussians_to_host(g), go)
    cam = scene.targets[0]
    H, W, C = cam.H, cam.W, scene.C
    P.gpu_rasterize(ctx, g, cam, gp, debug=False)
    rng = np.random.default_rng(seed)
    GF = rng.standard_normal((H, W, C)).astype(np.float32)
    GA = rng.standard_normal((H, W)).astype(np.float32)
    n = g.n
    dm = torch.empty((n, 2), dtype=torch.float32, device="cuda")
    dc = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    da = torch.empty((n,), dtype=torch.float32, device="cuda")
    dfe = torch.empty((n, C), dtype=torch.float32, device="cuda")
    ctx.rasterize_backward(g, -1, H, W, gp, torch.from_numpy(GF).cuda(), torch.from_numpy(GA).cuda(), dm, dc, da, dfe)
    torch.cuda.synchronize()
    K, R, t = sg.cam_arrays(cam)
    pr = oracle.project(go, K, R, t, H, W, op)
    ranges, lst = oracle.tile_lists(pr, go["ids"], H, W)
    ref = oracle.composite_backward(go, pr, ranges, lst, H, W, GF, GA, op)
    got = dict(mean2=dm.cpu().numpy(), conic=dc.cpu().numpy(), alpha=da.cpu().numpy(), feat=dfe.cpu().numpy())
    for k in ("mean2", "conic", "alpha", "feat"):
        scale = max(np.abs(ref[k]).max(), 1e-30)
        err = np.abs(got[k] - ref[k]).max()
        assert err <= 1e-4 * scale + 1e-6, (k, err, scale)
        assert np.count_nonzero(ref[k]) > 0
    return ref


@pytest.mark.parametrize("seed", range(9))
def test_random_scenes(ctx, seed):
    """fp32 features and C = 8 fp16 (plain kernel), fp16 features with C in {16, 32, 64} (tensor-core
    kernel)."""
    C = (8, 16, 32, 64, 16, 32, 64, 32, 8)[seed]
    dt = "f16" if seed % 2 or seed >= 4 else "f32"
    k = seed % 8
    s = sg.make_random_scene(20 + seed, H=21 + 9 * k, W=47 - 6 * k, C=C, n_src=14 + 2 * k, feat_dtype=dt)
    run_case(ctx, s, seed)


@pytest.mark.parametrize("seed", [0, 1, 2, 5])
def test_tile8_lists(monkeypatch, seed):
    """The backward over the forward's opt-in 8 x 8 tile lists (TA_TILE_PX=8): the plain kernel (64
    threads per tile) for fp32 features / C = 8 fp16, the tensor-core kernel (one warp per tile) for
    fp16 C >= 16 -- gradients against the oracle."""
    import paper_2405_14866_b200 as tb
    monkeypatch.setenv("TA_TILE_PX", "8")
    c8 = tb.Context(0)
    C = (8, 16, 32, 64, 16, 32, 64, 32, 8)[seed]
    dt = "f16" if seed % 2 or seed >= 4 else "f32"
    k = seed % 8
    s = sg.make_random_scene(20 + seed, H=21 + 9 * k, W=47 - 6 * k, C=C, n_src=14 + 2 * k, feat_dtype=dt)
    run_case(c8, s, seed)
    assert c8.debug_last().tile_px == 8


def test_rig_reduced(ctx):
    """configs[2] distributions at 128^2 sources, ragged 72 x 104 target, C = 32 fp16."""
    run_case(ctx, sg.make_config("c3", res=128, target_hw=(72, 104)))


def test_rig_larger_target(ctx):
    """configs[2] distributions at 256^2 sources into a ragged 200 x 232 target (C = 32 fp16): the
    tensor-core kernel over many 8x8 blocks with long lists and mode changes."""
    run_case(ctx, sg.make_config("c3", res=256, target_hw=(200, 232)), seed=5)


def test_requires_forward_first(ctx):
    import torch
    import paper_2405_14866_b200 as tb
    c2 = tb.Context(0)
    s = sg.make_config("tiny", res=16)
    gp = P.gpu_params(s, flags=0)
    g = P.gpu_unproject(c2, s, gp)
    z = torch.zeros((16, 16, 8), dtype=torch.float32, device="cuda")
    with pytest.raises(tb.TaError):
        c2.rasterize_backward(g, -1, 16, 16, gp, z, z[..., 0], z, z, z, z)
