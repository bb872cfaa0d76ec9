"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): tile lists and sort order bit-exact; features within 1e-4 absolute;
alpha bit-exact (T/A decisions are taken in the same fp32 sequence on both sides).
"""
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


@pytest.fixture(scope="module")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


def full_parity(ctx, O, scene, tidx=0, tiles=None, async_=False, same_f_bits=True, **pkw):
    """Every stage of the CUDA path against the oracle on one scene and target.  The rasterize call
    runs the instantiation bench.py times (flags = 0; with async_, TA_FLAG_ASYNC on a context sized
    by ta_reserve as in bench.py), then again with TA_FLAG_DEBUG_COUNTS, which must give the same bits
    (tests/_parity.gpu_rasterize)."""
    import paper_2405_14866_b200 as tb
    gp = P.gpu_params(scene, **pkw)
    op = P.oracle_params(scene, **pkw)
    g = P.gpu_unproject(ctx, scene, gp)
    gh = P.gaussians_to_host(g)
    go = O.unproject(scene, op)
    P.check_unproject(gh, go)
    cam = scene.targets[tidx]
    rctx = ctx
    if async_:
        sizing = P.gpu_rasterize(ctx, g, cam, gp, counts=False)
        rctx = tb.Context(0)
        rctx.reserve(g.capacity, max(int(sizing["Kc"] * 1.05), 1) + 1024, cam.H, cam.W)
        gp = P.gpu_params(scene, flags=tb.TA_FLAG_ASYNC, **pkw)
    out = P.gpu_rasterize(rctx, g, cam, gp, same_f_bits=same_f_bits)
    if async_:
        assert not rctx.check_overflow()
    K, R, t = sg.cam_arrays(cam)
    pr = O.project(go, K, R, t, cam.H, cam.W, op)
    P.check_project(out, pr, go["alpha"])
    P.check_order(out, pr, go["ids"])
    P.check_lists_vs_oracle(out, O, pr, go["ids"], cam.H, cam.W)
    ranges, lst = O.tile_lists(pr, go["ids"], cam.H, cam.W)          # the oracle composites 16 x 16 tiles
    F, A, nc, _ = O.composite(go, pr, ranges, lst, cam.H, cam.W, op, tiles=tiles)
    err = P.check_composite(out, F, A, nc, tiles=tiles, tx=(cam.W + 15) // 16)
    return out, err


def sample_tiles(ranges, TX, n_longest, n_random, seed):
    """The n_longest longest tile lists, n_random seeded random non-empty tiles and the 4 corners."""
    lens = ranges[:, 1].astype(np.int64) - ranges[:, 0]
    nonempty = np.nonzero(lens)[0]
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([np.argsort(lens, kind="stable")[-n_longest:],
                                     rng.choice(nonempty, min(n_random, len(nonempty)), replace=False),
                                     [0, TX - 1, len(lens) - TX, len(lens) - 1]])).astype(np.int32)


def test_tiny_config(ctx, oracle_lib):
    """configs[0] (Tiny) end to end: a1 .. a6."""
    out, err = full_parity(ctx, oracle_lib, sg.make_config("tiny"))
    assert out["K"] == 5400 and out["n"] == 4096


@pytest.mark.parametrize("seed", range(12))
def test_random_scenes(ctx, oracle_lib, seed):
    """Random anisotropic scenes, ragged targets (not multiples of 16), C in {8,16,32,64}, f16/f32."""
    C = (8, 16, 32, 64)[seed % 4]
    dt = "f16" if seed % 2 else "f32"
    s = sg.make_random_scene(seed, H=17 + 13 * seed, W=90 - 5 * seed, C=C, n_src=12 + 3 * seed, feat_dtype=dt)
    full_parity(ctx, oracle_lib, s)


@pytest.mark.parametrize("case", ["c2", "c2_async", "rand3", "rand6", "rand9", "c3_ragged"])
def test_tile8_lists_and_composite(oracle_lib, monkeypatch, case):
    """The opt-in 8 x 8 compositing tiles (TA_TILE_PX=8; 32-px coarse bins, 4 x 4 tiles per bin in the
    entry bits): every 8 x 8 tile list bit-exact against the oracle's lists for 8-px tiles, every
    pixel of F / A against the oracle; timed instantiation and TA_FLAG_ASYNC."""
    import paper_2405_14866_b200 as tb
    monkeypatch.setenv("TA_TILE_PX", "8")
    c8 = tb.Context(0)
    if case.startswith("rand"):
        seed = int(case[4:])
        C = (8, 16, 32, 64)[seed % 4]
        s = sg.make_random_scene(seed, H=17 + 13 * seed, W=90 - 5 * seed, C=C, n_src=12 + 3 * seed,
                                 feat_dtype="f16" if seed % 2 else "f32")
        out, _ = full_parity(c8, oracle_lib, s)
    elif case == "c3_ragged":
        out, _ = full_parity(c8, oracle_lib, sg.make_config("c3", res=256, target_hw=(136, 200)))
    else:
        out, _ = full_parity(c8, oracle_lib, sg.make_config("c2"), async_=case.endswith("async"))
    assert out["tile_px"] == 8


@pytest.mark.parametrize("f", [1.0, 0.55])
def test_focal_scale_sensitivity_configs(ctx, oracle_lib, f):
    """The footprint-sensitivity inputs of bench.py --focal-scale (f = 1.0 W, 0.55 W, body
    scaled to keep its image) at c2 size: every stage and every pixel against the oracle."""
    try:
        sg.set_focal_scale(f)
        s = sg.make_config("c2")
    finally:
        sg.set_focal_scale(1.95)
    full_parity(ctx, oracle_lib, s)


def test_c2_full(ctx, oracle_lib):
    """configs[1]: 2 x 512^2 sources, 512^2 target -- every stage, every pixel."""
    full_parity(ctx, oracle_lib, sg.make_config("c2"))


def test_c2_full_async(ctx, oracle_lib):
    """configs[1] in bench.py's launch mode: TA_FLAG_ASYNC on a ta_reserve'd context (no host
    synchronisation inside ta_rasterize) -- every stage, every pixel against the oracle."""
    full_parity(ctx, oracle_lib, sg.make_config("c2"), async_=True)


def test_c3_reduced_ragged(ctx, oracle_lib):
    """configs[2] distributions at 256^2 sources, ragged 200 x 136 target."""
    full_parity(ctx, oracle_lib, sg.make_config("c3", res=256, target_hw=(136, 200)))


def _c3_sampled_tiles(s, cam, n_longest=16, n_random=48, seed=0):
    import oracle as O
    op = P.oracle_params(s)
    go = O.unproject(s, op)
    K, R, t = sg.cam_arrays(cam)
    pr = O.project(go, K, R, t, cam.H, cam.W, op)
    ranges, _ = O.tile_lists(pr, go["ids"], cam.H, cam.W)
    return sample_tiles(ranges, (cam.W + 15) // 16, n_longest, n_random, seed)


@pytest.mark.parametrize("async_", [False, True])
def test_c3_full_size_sampled_tiles(ctx, oracle_lib, async_):
    """configs[2] at full size (4 x 1024^2, ~1.67M Gaussians, 1024^2 target) in the launch
    configuration bench.py times (flags = 0, and TA_FLAG_ASYNC after ta_reserve): a1-a5 bit-exact in
    full; a6 on 68 sampled tiles incl. the 16 longest lists, every stage checked against the oracle."""
    s = sg.make_config("c3")
    tiles = _c3_sampled_tiles(s, s.targets[0])
    assert len(tiles) >= 64
    out, err = full_parity(ctx, oracle_lib, s, tiles=tiles, async_=async_)
    assert out["n"] == 1666464


def test_c3_frame_timed_equals_counters_instantiation(ctx):
    """A whole c3 frame (1024^2, C = 32 fp16) rendered by the timed compositor instantiation
    (flags = 0) and by the counters instantiation (TA_FLAG_DEBUG_COUNTS) is bit-identical in F and A
    at every pixel (the oracle comparisons run both; this pins it on the full frame)."""
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c3")
    g = P.gpu_unproject(ctx, s, P.gpu_params(s))
    K, R, t = sg.cam_arrays(s.targets[0])
    F0, A0 = tb.rasterize(ctx, g, K, R, t, 1024, 1024, P.gpu_params(s, flags=0))
    F2, A2 = tb.rasterize(ctx, g, K, R, t, 1024, 1024, P.gpu_params(s, flags=tb.TA_FLAG_DEBUG_COUNTS))
    torch.cuda.synchronize()
    assert torch.equal(F0.view(torch.int32), F2.view(torch.int32))
    assert torch.equal(A0.view(torch.int32), A2.view(torch.int32))
    assert float(A0.max()) > 0.9


def test_c4_bench_targets_full_size(ctx, oracle_lib):
    """configs[3] exactly as bench.py renders it: the full c3 Gaussian set (4 x 1024^2 sources) into 4
    of the 32 parallax targets (phi = -15, -5.3, +5.3, +15 deg) at 1024^2, TA_FLAG_ASYNC on reserved
    contexts over 4 CUDA streams with overlapping views.  Per target: records, order and every tile
    list bit-exact; F / A / composited counts on 40 sampled tiles (incl. the 12 longest lists)."""
    import torch
    import oracle as O
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c3")
    targets = sg.make_targets("c4")
    picks = [0, 10, 21, 31]
    gp = P.gpu_params(s)
    op = P.oracle_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    go = O.unproject(s, op)
    kc = 0
    for j in picks:
        P.gpu_rasterize(ctx, g, targets[j], gp, debug=False)
        kc = max(kc, ctx.debug_last().Kc)
    ctxs = [tb.Context(0) for _ in picks]
    streams = [torch.cuda.Stream() for _ in picks]
    pa = P.gpu_params(s, flags=tb.TA_FLAG_ASYNC)
    outs = []
    for cx, st, j in zip(ctxs, streams, picks):
        cx.reserve(g.capacity, int(kc * 1.05) + 4096, 1024, 1024)
    torch.cuda.synchronize()
    for cx, st, j in zip(ctxs, streams, picks):        # overlapping views, as in bench.py
        K, R, t = sg.cam_arrays(targets[j])
        F = torch.empty((1024, 1024, s.C), device="cuda")
        A = torch.empty((1024, 1024), device="cuda")
        cx.rasterize(g, -1, tb.intrinsics(K), tb.extrinsics(R, t), 1024, 1024, pa, F, A, st)
        outs.append((F, A))
    torch.cuda.synchronize()
    for cx, j, (F, A) in zip(ctxs, picks, outs):
        assert not cx.check_overflow()
        cam = targets[j]
        out = P.gpu_rasterize(cx, g, cam, pa)          # debug views of this target (same async call)
        assert np.array_equal(out["F"].view(np.uint32), F.cpu().numpy().view(np.uint32))
        assert np.array_equal(out["A"].view(np.uint32), A.cpu().numpy().view(np.uint32))
        K, R, t = sg.cam_arrays(cam)
        pr = O.project(go, K, R, t, cam.H, cam.W, op)
        P.check_project(out, pr, go["alpha"])
        P.check_order(out, pr, go["ids"])
        P.check_lists_vs_oracle(out, O, pr, go["ids"], cam.H, cam.W)
        ranges, lst = O.tile_lists(pr, go["ids"], cam.H, cam.W)
        tiles = sample_tiles(ranges, 64, 12, 24, j)
        Fo, Ao, nc, _ = O.composite(go, pr, ranges, lst, cam.H, cam.W, op, tiles=tiles)
        P.check_composite(out, Fo, Ao, nc, tiles=tiles, tx=64)


def test_wide_target_64px_coarse_bins(ctx, oracle_lib):
    """A target wider than 1024 px bins in 64 x 64-pixel coarse bins (4 x 4 tiles, the tile rectangle
    in the entry bits; include/ta.h ta_rasterize): every stage and every tile list bit-exact, ragged
    in both directions (88 x 1100)."""
    out, _ = full_parity(ctx, oracle_lib, sg.make_config("c3", res=256, target_hw=(88, 1100)))
    assert out["K"] > 0


def test_large_ragged_target(ctx, oracle_lib):
    """A sparse scene in a 2300 x 3100 target: 64-px coarse bins over 49 x 36 bins, most tiles empty,
    every stage and every pixel against the oracle (C = 16 fp16)."""
    s = sg.make_random_scene(7, H=2300, W=3100, C=16, n_src=40, feat_dtype="f16")
    out, _ = full_parity(ctx, oracle_lib, s)
    assert out["K"] > 0 and out["tiles_x"] == 194 and out["tiles_y"] == 144


def test_coarse_bins_fall_back_for_large_capacity(ctx, oracle_lib):
    """With more than 2^24 Gaussian slots (n = -1: the capacity bounds the indices) a > 1024 px target
    keeps 32 x 32-pixel bins (28 index bits): different coarse binning, identical output bits."""
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c3", res=128, target_hw=(72, 1040))
    gp = P.gpu_params(s)
    cam = s.targets[0]
    small = P.gpu_unproject(ctx, s, gp)
    ref = P.gpu_rasterize(ctx, small, cam, gp)
    big = tb.GaussianBuffers((1 << 24) + 1, s.C, s.feat_dtype)
    views, keep = tb.views_to_device(s.views)
    ctx.unproject(views, gp, big)
    torch.cuda.synchronize()
    out = P.gpu_rasterize(ctx, big, cam, gp)
    assert out["n"] == ref["n"] and out["Kc"] != ref["Kc"]
    for k in ("F", "A", "order", "ranges", "list"):
        assert np.array_equal(out[k].view(np.uint8), ref[k].view(np.uint8)), k
    del big


@pytest.mark.parametrize("eye", [0, 1])
def test_paper_variant_reduced(ctx, oracle_lib, eye):
    """SURVEY 8(f) NEXT #3, the paper-exact variant: cam0 + cam2 + cam3 lifted
    with R = I (diagonal Sigma_w), both eye targets -- every stage, every pixel at 256^2."""
    s = sg.make_config("paper", res=256)
    assert len(s.views) == 3 and all(v.quat is None for v in s.views)
    full_parity(ctx, oracle_lib, s, tidx=eye)


def test_paper_variant_full_size_sampled_tiles(ctx, oracle_lib):
    """The paper-exact variant at 1024^2 (3 x 1024^2 sources), right eye: a1-a5 bit-exact in full,
    a6 on the 6 longest tile lists + 10 seeded random non-empty tiles."""
    s = sg.make_config("paper")
    cam = s.targets[1]
    import oracle as O
    op = P.oracle_params(s)
    go = O.unproject(s, op)
    K, R, t = sg.cam_arrays(cam)
    pr = O.project(go, K, R, t, cam.H, cam.W, op)
    ranges, _ = O.tile_lists(pr, go["ids"], cam.H, cam.W)
    lens = ranges[:, 1].astype(np.int64) - ranges[:, 0]
    rng = np.random.default_rng(3)
    tiles = np.unique(np.concatenate([np.argsort(lens)[-6:],
                                      rng.choice(np.nonzero(lens)[0], 10, replace=False)])).astype(np.int32)
    full_parity(ctx, oracle_lib, s, tidx=1, tiles=tiles)


def test_c4_views_vs_single_view(ctx, oracle_lib):
    """configs[3]: one Gaussian set, several parallax targets on one context; each equals the oracle
    on sampled tiles (the 32-view batch at reduced source resolution)."""
    s = sg.make_config("c4", res=256, target_hw=(256, 256), n_targets=5)
    gp = P.gpu_params(s)
    op = P.oracle_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    go = oracle_lib.unproject(s, op)
    for cam in s.targets:
        out = P.gpu_rasterize(ctx, g, cam, gp)
        K, R, t = sg.cam_arrays(cam)
        pr = oracle_lib.project(go, K, R, t, cam.H, cam.W, op)
        P.check_lists_vs_oracle(out, oracle_lib, pr, go["ids"], cam.H, cam.W)
        ranges, lst = oracle_lib.tile_lists(pr, go["ids"], cam.H, cam.W)
        F, A, nc, _ = oracle_lib.composite(go, pr, ranges, lst, cam.H, cam.W, op)
        P.check_composite(out, F, A, nc)


def test_concurrent_contexts_on_streams_match_sequential(ctx):
    """The bench's launch configuration: views of one frame alternate over 4 (context, stream) pairs
    with TA_FLAG_ASYNC after ta_reserve, kernels of different views overlapping; every view's F and A
    are bit-identical to the same view rendered alone on one context (full c3 sources, 8 targets)."""
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c3")
    targets = sg.make_targets("c4", n_targets=8)
    gp = P.gpu_params(s, flags=0)
    g = P.gpu_unproject(ctx, s, gp)
    H, W, C = 1024, 1024, s.C
    ref = []
    for cam in targets:
        K, R, t = sg.cam_arrays(cam)
        F, A = tb.rasterize(ctx, g, K, R, t, H, W, gp, n=-1)
        torch.cuda.synchronize()
        ref.append((F.clone(), A.clone(), ctx.debug_last().Kc))
    kc = max(r[2] for r in ref)
    ctxs = [tb.Context(0) for _ in range(4)]
    streams = [torch.cuda.Stream() for _ in range(4)]
    pa = tb.default_params(default_scale=s.default_scale, default_opacity=s.default_opacity, flags=tb.TA_FLAG_ASYNC)
    for cx in ctxs:
        cx.reserve(g.capacity, int(kc * 1.05) + 4096, H, W)
    outs = [(torch.empty((H, W, C), device="cuda"), torch.empty((H, W), device="cuda")) for _ in targets]
    torch.cuda.synchronize()
    for k, cam in enumerate(targets):
        K, R, t = sg.cam_arrays(cam)
        ctxs[k % 4].rasterize(g, -1, tb.intrinsics(K), tb.extrinsics(R, t), H, W, pa, outs[k][0], outs[k][1],
                              streams[k % 4])
    torch.cuda.synchronize()
    assert not any(cx.check_overflow() for cx in ctxs)
    for (F, A), (Fr, Ar, _) in zip(outs, ref):
        assert torch.equal(A.view(torch.int32), Ar.view(torch.int32))
        assert torch.equal(F.view(torch.int32), Fr.view(torch.int32))


def test_c5_stress_sampled_tiles(ctx, oracle_lib):
    """configs[4] (4 x 2048^2, ~6.7M Gaussians, C = 64, 2048^2 target): a1 + a2 bit-exact in full,
    a4 depth order, a3/a5 on sampled tiles via per-tile enumeration, a6 on the sampled tiles."""
    s = sg.make_config("c5", n_targets=1)
    gp = P.gpu_params(s)
    op = P.oracle_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    gh = P.gaussians_to_host(g)
    go = oracle_lib.unproject(s, op)
    P.check_unproject(gh, go)
    del gh
    cam = s.targets[0]
    out = P.gpu_rasterize(ctx, g, cam, gp)
    K, R, t = sg.cam_arrays(cam)
    pr = oracle_lib.project(go, K, R, t, cam.H, cam.W, op)
    P.check_project(out, pr, go["alpha"])
    P.check_order(out, pr, go["ids"])
    # a3/a5 on sampled GPU tiles (side tile_px): the oracle's definition -- every visible Gaussian whose
    # box covers the tile, in (dkey, id) order -- written out for those tiles
    vis = np.nonzero(pr["visible"])[0]
    ts = out["tile_px"]
    TXg = (cam.W + ts - 1) // ts
    lens = out["ranges"][:, 1].astype(np.int64) - out["ranges"][:, 0]
    rng = np.random.default_rng(1)
    gtiles = np.unique(np.concatenate([np.argsort(lens)[-3:], rng.choice(np.nonzero(lens)[0], 6, replace=False)]))

    def covering(tx, ty, side):
        r = pr["rect"][vis] // side
        cov = vis[(r[:, 0] <= tx) & (tx <= r[:, 1]) & (r[:, 2] <= ty) & (ty <= r[:, 3])]
        return cov[np.lexsort((go["ids"][cov], pr["dkey"][cov]))]

    for tt in gtiles:
        ty, tx = divmod(int(tt), TXg)
        a, b = out["ranges"][tt]
        assert np.array_equal(out["list"][a:b].astype(np.int64), covering(tx, ty, ts))
    # a6 on the 16 x 16 tiles holding them (the oracle composites 16 x 16 tiles)
    TX = (cam.W + 15) // 16
    tiles = np.unique([(int(tt) // TXg * ts // 16) * TX + (int(tt) % TXg) * ts // 16 for tt in gtiles])
    sub_ranges = np.zeros((TX * ((cam.H + 15) // 16), 2), np.uint32)
    chunks, pos = [], 0
    for tt in tiles:
        ty, tx = divmod(int(tt), TX)
        cov = covering(tx, ty, 16)
        sub_ranges[tt] = (pos, pos + len(cov))
        chunks.append(cov)
        pos += len(cov)
    F, A, nc, _ = oracle_lib.composite(go, pr, sub_ranges, np.concatenate(chunks), cam.H, cam.W, op,
                                       tiles=tiles.astype(np.int32))
    P.check_composite(out, F, A, nc, tiles=tiles, tx=TX)


# ------------------------------------------------------------------ closed forms / properties on the GPU

def test_identity_camera_reproduces_source(ctx):
    """north_star closed form on the GPU: identity target, sigma = 0.05 px, alpha = 1 ->
    F = fl(f * 0.99f), A = fl(1 - fl(1 - 0.99f)) bit-exactly."""
    rng = np.random.default_rng(3)
    H, W, f, B = 45, 61, 60.0, 0.1
    cam = sg.Camera(fx=f, fy=f, cx=(W - 1) / 2, cy=(H - 1) / 2, R=np.eye(3), t=np.zeros(3), H=H, W=W)
    d = rng.uniform(5, 15, (H, W)).astype(np.float32)
    z = (np.float32(f) * np.float32(B)) / d
    sc = (0.05 * z / f).astype(np.float32)
    feat = rng.standard_normal((H, W, 16)).astype(np.float32)
    v = sg.SourceView(cam=cam, baseline=B, disparity=d, mask=None, scale=np.repeat(sc[..., None], 3, -1), quat=None,
                      opacity=np.ones((H, W), np.float32), feat=feat)
    s = sg.Scene("ident", [v], [cam], 16, "f32")
    gp = P.gpu_params(s, dilation=0.0)
    g = P.gpu_unproject(ctx, s, gp)
    out = P.gpu_rasterize(ctx, g, cam, gp)
    a = np.float32(0.99)
    assert np.array_equal(out["F"], feat * a)
    assert np.all(out["A"] == np.float32(1.0) - (np.float32(1.0) - a))


def test_permutation_invariance_and_determinism(ctx):
    """Permuting the Gaussian arrays (ids travel) gives identical bits; repeated runs are bit-identical."""
    import torch
    s = sg.make_config("c2", res=128, target_hw=(112, 144))
    gp = P.gpu_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    cam = s.targets[0]
    a = P.gpu_rasterize(ctx, g, cam, gp, debug=False)
    b = P.gpu_rasterize(ctx, g, cam, gp, debug=False)
    assert np.array_equal(a["F"], b["F"]) and np.array_equal(a["A"], b["A"])
    n = g.n
    perm = torch.randperm(n, generator=torch.Generator().manual_seed(0)).cuda()
    g.pos_alpha[:n] = g.pos_alpha[:n][perm].clone()
    g.cov[:n] = g.cov[:n][perm].clone()
    g.feat[:n] = g.feat[:n][perm].clone()
    c = P.gpu_rasterize(ctx, g, cam, gp, debug=False)
    assert np.array_equal(a["F"], c["F"]) and np.array_equal(a["A"], c["A"])


def test_empty_and_degenerate_inputs(ctx):
    """Empty cloud, all culled (target looking away), n = 0: F = 0, A = 0 everywhere."""
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("tiny", res=32)
    s.views[0].mask = np.zeros((32, 32), np.uint8)
    gp = P.gpu_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    assert g.n == 0
    out = P.gpu_rasterize(ctx, g, s.targets[0], gp)
    assert np.all(out["F"] == 0) and np.all(out["A"] == 0) and out["K"] == 0
    s = sg.make_config("tiny", res=32)
    g = P.gpu_unproject(ctx, s, gp)
    away = sg.Camera(fx=32.0, fy=32.0, cx=15.5, cy=15.5, R=sg.rot_y(180.0), t=np.zeros(3), H=40, W=24)
    out = P.gpu_rasterize(ctx, g, away, gp)
    assert np.all(out["F"] == 0) and np.all(out["A"] == 0)
    out = P.gpu_rasterize(ctx, g, s.targets[0], gp, n=0)
    assert np.all(out["F"] == 0) and np.all(out["A"] == 0)
    torch.cuda.synchronize()


def test_async_reserve_and_overflow(ctx):
    """TA_FLAG_ASYNC after ta_reserve gives the same bits as a synchronous call; too small a
    reservation is reported by ta_check_overflow (no silent truncation)."""
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c2", res=128, target_hw=(128, 128))
    gp = P.gpu_params(s, flags=0)
    g = P.gpu_unproject(ctx, s, gp)
    cam = s.targets[0]
    ref = P.gpu_rasterize(ctx, g, cam, gp, debug=False)
    dbg = ctx.debug_last()
    ctx2 = tb.Context(0)
    ctx2.reserve(g.capacity, dbg.Kc, cam.H, cam.W)
    ga = P.gpu_params(s, flags=tb.TA_FLAG_ASYNC)
    out = P.gpu_rasterize(ctx2, g, cam, ga, debug=False)
    assert not ctx2.check_overflow()
    assert np.array_equal(out["F"], ref["F"]) and np.array_equal(out["A"], ref["A"])
    ctx3 = tb.Context(0)
    ctx3.reserve(g.capacity, dbg.Kc // 2, cam.H, cam.W)
    P.gpu_rasterize(ctx3, g, cam, ga, debug=False)
    assert ctx3.check_overflow()


def test_invalid_arguments_are_rejected(ctx):
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("tiny", res=16)
    gp = P.gpu_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    F = torch.empty((16, 16, 8), device="cuda")
    A = torch.empty((16, 16), device="cuda")
    bad_R = np.eye(3, dtype=np.float32).reshape(9) * 2
    with pytest.raises(tb.TaError) as e:
        ctx.rasterize(g, -1, tb.intrinsics((16, 16, 7.5, 7.5)), tb.extrinsics(bad_R, np.zeros(3)), 16, 16, gp, F, A)
    assert e.value.status == 1
    with pytest.raises(tb.TaError) as e:
        ctx.rasterize(g, -1, tb.intrinsics((-1, 16, 7.5, 7.5)), tb.extrinsics(np.eye(3).reshape(9), np.zeros(3)),
                      16, 16, gp, F, A)
    assert e.value.status == 1
    small = tb.GaussianBuffers(10, 8, "f32")
    views, keep = tb.views_to_device(s.views)
    with pytest.raises(tb.TaError) as e:
        ctx.unproject(views, gp, small)
    assert e.value.status == 5
    odd = tb.GaussianBuffers(256, 12, "f32")
    with pytest.raises(tb.TaError) as e:
        ctx.unproject(views, gp, odd)
    assert e.value.status == 2


@pytest.mark.parametrize("cfg", ["c2", "c3r"])
def test_tensor_memory_compositor_parity(oracle_lib, cfg):
    """The opt-in tensor-memory compositor (TA_COMPOSITOR=2: tcgen05.mma with the C-channel accumulators
    in TMEM, one 16 x 16 tile per 4-warp CTA) against the oracle: every stage, every pixel (c2 and the
    ragged reduced c3); A and composited counts bit-exact, F within 1e-4."""
    import os
    import paper_2405_14866_b200 as tb
    os.environ["TA_COMPOSITOR"] = "2"
    try:
        c = tb.Context(0)
    finally:
        os.environ.pop("TA_COMPOSITOR")
    s = sg.make_config("c2") if cfg == "c2" else sg.make_config("c3", res=256, target_hw=(136, 200))
    full_parity(c, oracle_lib, s)


@pytest.mark.parametrize("comp", ["3", "4"])
@pytest.mark.parametrize("cfg", ["c2", "c3r"])
def test_warp_specialized_compositor_parity(oracle_lib, cfg, comp):
    """The opt-in warp-specialized compositors (TA_COMPOSITOR=3: one producer warp per consumer warp,
    4: one producer for two consumers; staging buffers handed over mbarriers, accumulators in tensor
    memory) against the oracle: every stage and every pixel, A and composited counts bit-exact, F within
    1e-4."""
    import os
    import paper_2405_14866_b200 as tb
    os.environ["TA_COMPOSITOR"] = comp
    try:
        c = tb.Context(0)
    finally:
        os.environ.pop("TA_COMPOSITOR")
    s = sg.make_config("c2") if cfg == "c2" else sg.make_config("c3", res=256, target_hw=(136, 200))
    # the producer culls against the consumer's active box as last published, so which entries are staged
    # (and with them the grouping of the fp32 MMA sums) depends on timing: F can differ between runs in
    # its last bits, the decisions (A, counts) cannot
    full_parity(c, oracle_lib, s, same_f_bits=False)


@pytest.mark.parametrize("cfg", ["c2", "c3r"])
def test_register_accumulator_compositor_parity(oracle_lib, cfg):
    """fp16 C = 32 composites with its accumulators in tensor memory by default; TA_COMPOSITOR=1 keeps
    them in registers (64 staged entries per warp instead of 32).  That variant against the oracle,
    every stage and every pixel (A and composited counts bit-exact, F within 1e-4)."""
    import os
    import paper_2405_14866_b200 as tb
    os.environ["TA_COMPOSITOR"] = "1"
    try:
        c = tb.Context(0)
    finally:
        os.environ.pop("TA_COMPOSITOR")
    s = sg.make_config("c2") if cfg == "c2" else sg.make_config("c3", res=256, target_hw=(136, 200))
    full_parity(c, oracle_lib, s)


def test_accumulator_placement_same_alpha_c4_target(ctx):
    """Tensor-memory (default) vs register accumulators on a full 1024^2 c4 target: A and the
    composited counts bit-identical (same per-pixel decisions), F within 2e-6 (the staging depth
    changes only how the fp32 MMA sums are grouped)."""
    import os
    import torch
    import paper_2405_14866_b200 as tb
    os.environ["TA_COMPOSITOR"] = "1"
    try:
        c1 = tb.Context(0)
    finally:
        os.environ.pop("TA_COMPOSITOR")
    s = sg.make_config("c3")
    gp = P.gpu_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    cam = sg.make_targets("c4", n_targets=32)[7]
    a = P.gpu_rasterize(ctx, g, cam, gp, debug=False)
    b = P.gpu_rasterize(c1, g, cam, gp, debug=False)
    assert np.array_equal(a["A"].view(np.uint32), b["A"].view(np.uint32))
    assert np.abs(a["F"] - b["F"]).max() <= 2e-6
    pc = P.gpu_params(s, flags=tb.TA_FLAG_DEBUG_COUNTS)
    K, R, t = sg.cam_arrays(cam)
    for cx in (ctx, c1):
        tb.rasterize(cx, g, K, R, t, cam.H, cam.W, pc)
    torch.cuda.synchronize()
    na = P.d2h(ctx.debug_last().n_contrib, cam.H * cam.W, np.int32)
    nb = P.d2h(c1.debug_last().n_contrib, cam.H * cam.W, np.int32)
    assert np.array_equal(na, nb) and na.sum() > 0


@pytest.mark.parametrize("cfg", ["c2", "c3r"])
def test_fp32_features_timed_instantiation(ctx, oracle_lib, cfg):
    """fp32-stored features take k_composite<C, float, false> (the SIMT compositor; the counters
    instantiation runs after it and must give the same bits): c2 at full size and the reduced ragged
    c3 with their fp16 feature maps widened to fp32 (exact), every stage and every pixel against the
    oracle."""
    s = sg.make_config("c2") if cfg == "c2" else sg.make_config("c3", res=256, target_hw=(136, 200))
    for v in s.views:
        v.feat = v.feat.astype(np.float32)
    s.feat_dtype = "f32"
    out, err = full_parity(ctx, oracle_lib, s)
    assert out["K"] > 0


@pytest.mark.parametrize("case", [
    dict(cull_sigma=2.0, alpha_max=0.9, alpha_min=0.0, t_eps=1e-2, dilation=0.0),
    dict(cull_sigma=4.0, alpha_max=0.999, alpha_min=0.02, t_eps=1e-5, dilation=1.0),
    dict(cull_sigma=3.0, alpha_max=0.5, alpha_min=1.0 / 255.0, t_eps=0.3, dilation=0.3),
])
@pytest.mark.parametrize("C,dt", [(32, "f16"), (8, "f16"), (16, "f32")])
def test_non_default_raster_params(ctx, oracle_lib, case, C, dt):
    """Every raster constant is a parameter (R7-R10): the box width and q cut (cull_sigma), the alpha'
    clamp, the low-alpha skip, the stop threshold and the low-pass dilation away from their defaults,
    through every compositor instantiation (fp16 mma.sync C = 32 / 8, fp32 SIMT) -- every stage and every
    pixel against the oracle on a ragged random scene and the reduced rig."""
    s = sg.make_random_scene(11 + C, H=53, W=77, C=C, n_src=28, feat_dtype=dt)
    full_parity(ctx, oracle_lib, s, **case)
    r = sg.make_config("c3", res=128, target_hw=(72, 88))
    if dt == "f32" or C != 32:
        for v in r.views:
            v.feat = v.feat[..., :C].astype(np.float32 if dt == "f32" else np.float16)
        r.C, r.feat_dtype = C, dt
    full_parity(ctx, oracle_lib, r, **case)


@pytest.mark.parametrize("hw", [(1, 1), (1, 37), (45, 1), (17, 16)])
def test_degenerate_target_shapes(ctx, oracle_lib, hw):
    """Single-pixel, single-row, single-column and one-tile-plus-one-row targets (ragged tiles, boxes
    clamped to the image on every side): every stage and pixel against the oracle."""
    s = sg.make_random_scene(5, H=hw[0], W=hw[1], C=16, n_src=24, feat_dtype="f16")
    full_parity(ctx, oracle_lib, s)


@pytest.mark.parametrize("lanes,async_", [(1, False), (3, False), (4, True)])
def test_rasterize_views_equals_single_calls(ctx, lanes, async_):
    """ta_rasterize_views (one Gaussian set into T targets, spread over the context's lanes inside the
    library) is bit-identical to T ta_rasterize calls, in sync mode and with TA_FLAG_ASYNC after
    ta_reserve (which sizes the child contexts too); 7 parallax targets of the reduced c4."""
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c4", res=256, target_hw=(200, 248), n_targets=7)
    gp = P.gpu_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    refs, kc = [], 0
    for cam in s.targets:
        r = P.gpu_rasterize(ctx, g, cam, gp, debug=False)
        kc = max(kc, ctx.debug_last().Kc)
        refs.append(r)
    cx = tb.Context(0)
    p = gp
    if async_:
        cx.reserve(g.capacity, int(kc * 1.1) + 1024, 200, 248)
        p = P.gpu_params(s, flags=tb.TA_FLAG_ASYNC)
    Ks, RTs = [], []
    for cam in s.targets:
        K, R, t = sg.cam_arrays(cam)
        Ks.append(tb.intrinsics(K))
        RTs.append(tb.extrinsics(R, t))
    Fs = [torch.empty((200, 248, s.C), device="cuda") for _ in s.targets]
    As = [torch.empty((200, 248), device="cuda") for _ in s.targets]
    cx.rasterize_views(g, -1, Ks, RTs, 200, 248, p, Fs, As, lanes=lanes)
    torch.cuda.synchronize()
    assert not cx.check_overflow()
    for F, A, r in zip(Fs, As, refs):
        assert np.array_equal(F.cpu().numpy().view(np.uint32), r["F"].view(np.uint32))
        assert np.array_equal(A.cpu().numpy().view(np.uint32), r["A"].view(np.uint32))


def test_rasterize_views_invalid_arguments(ctx):
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("tiny", res=16)
    gp = P.gpu_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    K, R, t = sg.cam_arrays(s.targets[0])
    F = torch.empty((16, 16, 8), device="cuda")
    A = torch.empty((16, 16), device="cuda")
    for lanes in (0, 5):
        with pytest.raises(tb.TaError) as e:
            ctx.rasterize_views(g, -1, [tb.intrinsics(K)], [tb.extrinsics(R, t)], 16, 16, gp, [F], [A], lanes=lanes)
        assert e.value.status == 1
    with pytest.raises(tb.TaError) as e:
        ctx.rasterize_views(g, -1, [], [], 16, 16, gp, [], [], lanes=2)
    assert e.value.status == 1
