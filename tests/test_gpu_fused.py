"""north_star (a): the fused unproject + project + cull front end (include/ta.h ta_render_sources) is
bit-exact against the two-call path (ta_unproject, then ta_rasterize per target): F and A at every
pixel, the records, depth order and tile lists -- for one target and for the paper's two eyes,
and against the oracle on c2."""
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


def fused(ctx, scene, cams, params):
    import torch
    import paper_2405_14866_b200 as tb
    views, keep = tb.views_to_device(scene.views)
    H, W = cams[0].H, cams[0].W
    outs = [(torch.empty((H, W, scene.C), device="cuda"), torch.empty((H, W), device="cuda")) for _ in cams]
    Ks, RTs = [], []
    for cam in cams:
        K, R, t = sg.cam_arrays(cam)
        Ks.append(tb.intrinsics(K))
        RTs.append(tb.extrinsics(R, t))
    ctx.render_sources(views, scene.C, scene.feat_dtype, params, Ks, RTs, H, W, [o[0] for o in outs],
                       [o[1] for o in outs])
    torch.cuda.synchronize()
    return [(F.cpu().numpy(), A.cpu().numpy()) for F, A in outs]


def two_call(ctx, scene, cams, params):
    g = P.gpu_unproject(ctx, scene, params)
    return [P.gpu_rasterize(ctx, g, cam, params) for cam in cams]


def same_bits(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint8), np.ascontiguousarray(b).view(np.uint8))


@pytest.mark.parametrize("case", ["c3r", "paper256", "random3", "tiny"])
def test_fused_equals_two_call(ctx, case):
    if case == "c3r":
        s = sg.make_config("c3", res=256, target_hw=(136, 200)); cams = s.targets
    elif case == "paper256":
        s = sg.make_config("paper", res=256); cams = s.targets          # both eyes in one call
    elif case == "random3":
        s = sg.make_random_scene(3, H=45, W=70, C=16, n_src=30, feat_dtype="f16"); cams = s.targets
    else:
        s = sg.make_config("tiny"); cams = s.targets
    gp = P.gpu_params(s)
    ref = two_call(ctx, s, cams, gp)
    got = fused(ctx, s, cams, gp)
    for (F, A), r in zip(got, ref):
        assert same_bits(F, r["F"]) and same_bits(A, r["A"])
    # target 0's debug view: records, order and tile lists identical to the two-call path
    dv = ctx.debug_last()
    recs = P.d2h(dv.records, 8 * dv.n, np.uint32).reshape(-1, 8)
    assert dv.n == ref[0]["n"] and dv.K == ref[0]["K"]
    assert np.array_equal(recs, ref[0]["records"])
    assert np.array_equal(P.d2h(dv.order, dv.n, np.uint32), ref[0]["order"])
    assert np.array_equal(P.d2h(dv.tile_list, dv.K, np.uint32), ref[0]["list"])


def test_fused_paper_variant_full_size_both_eyes(ctx):
    """The paper-exact frame at full size (3 x 1024^2 sources, R = I, both 1024^2 eyes in one call,
    C = 32 fp16) bit-identical to ta_unproject + 2 x ta_rasterize; also with TA_FLAG_ASYNC."""
    import paper_2405_14866_b200 as tb
    s = sg.make_config("paper")
    gp = P.gpu_params(s)
    ref = [P.gpu_rasterize(ctx, P.gpu_unproject(ctx, s, gp), cam, gp, debug=False) for cam in s.targets]
    got = fused(ctx, s, s.targets, gp)
    for (F, A), r in zip(got, ref):
        assert same_bits(F, r["F"]) and same_bits(A, r["A"])
    got2 = fused(ctx, s, s.targets, P.gpu_params(s, flags=tb.TA_FLAG_ASYNC))
    for (F, A), r in zip(got2, ref):
        assert same_bits(F, r["F"]) and same_bits(A, r["A"])


def test_fused_against_oracle_c2(ctx, oracle_lib=None):
    """c2 through the fused front end against the CPU oracle: A bit-exact, F within 1e-4 at every pixel."""
    import oracle as O
    O.build()
    s = sg.make_config("c2")
    gp = P.gpu_params(s)
    op = P.oracle_params(s)
    (F, A), = fused(ctx, s, s.targets, gp)
    go = O.unproject(s, op)
    cam = s.targets[0]
    K, R, t = sg.cam_arrays(cam)
    pr = O.project(go, K, R, t, cam.H, cam.W, op)
    ranges, lst = O.tile_lists(pr, go["ids"], cam.H, cam.W)
    Fo, Ao, nc, _ = O.composite(go, pr, ranges, lst, cam.H, cam.W, op)
    P.check_composite({"F": F, "A": A}, Fo, Ao)


def test_fused_invalid_arguments(ctx):
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("tiny", res=16)
    views, keep = tb.views_to_device(s.views)
    F = torch.empty((16, 16, 8), device="cuda")
    A = torch.empty((16, 16), device="cuda")
    K, R, t = sg.cam_arrays(s.targets[0])
    Ki, Ri = tb.intrinsics(K), tb.extrinsics(R, t)
    with pytest.raises(tb.TaError) as e:     # T = 5 > 4
        ctx.render_sources(views, 8, "f32", P.gpu_params(s), [Ki] * 5, [Ri] * 5, 16, 16, [F] * 5, [A] * 5)
    assert e.value.status == 1
    with pytest.raises(tb.TaError) as e:     # C not supported
        ctx.render_sources(views, 12, "f32", P.gpu_params(s), [Ki], [Ri], 16, 16, [F], [A])
    assert e.value.status == 2
