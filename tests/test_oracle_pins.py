"""Pins for the CPU oracle (oracle/taoracle.c) against things other than itself:
closed forms, worked examples (tests/golden), invariants, brute force on tiny inputs,
an independent float64 model (oracle/definition64.py), scipy, Monte Carlo.

Each test names the part it pins (a1..a6) and the passage it follows
(P:<line> = /root/reference/PAPER.md, S:<line> = SPEC.md).
"""
import json
import math
import os

import numpy as np
import pytest

import synthgen as sg

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def one_pixel_scene(fx, cx, cy, H, W, px, py, d, B, scale=None, quat=None, alpha=1.0, feat=None,
                    C=4, tgt=None, dscale=0.01):
    """Source view where only pixel (px, py) is foreground."""
    disp = np.full((H, W), d, np.float32)
    mask = np.zeros((H, W), np.uint8)
    mask[py, px] = 1
    cam = sg.Camera(fx=fx, fy=fx, cx=cx, cy=cy, R=np.eye(3), t=np.zeros(3), H=H, W=W)
    f = np.zeros((H, W, C), np.float32)
    if feat is not None:
        f[py, px] = feat
    op = np.full((H, W), alpha, np.float32)
    sc = None if scale is None else np.broadcast_to(np.asarray(scale, np.float32), (H, W, 3)).copy()
    q = None if quat is None else np.broadcast_to(np.asarray(quat, np.float32), (H, W, 4)).copy()
    v = sg.SourceView(cam=cam, baseline=B, disparity=disp, mask=mask, scale=sc, quat=q, opacity=op, feat=f)
    return sg.Scene(name="one", views=[v], targets=[tgt or cam], C=C, feat_dtype="f32",
                    default_scale=dscale, default_opacity=1.0)


# ------------------------------------------------------------------------------ exp_det (R13)

def test_exp_det_within_2ulp_of_float64_exp(oracle_lib):
    x = np.linspace(-4.5, 0.0, 400001).astype(np.float32)
    y = oracle_lib.exp_det(x).astype(np.float64)
    ref = np.exp(x.astype(np.float64))
    ulp = np.spacing(ref.astype(np.float32)).astype(np.float64)
    assert np.max(np.abs(y - ref) / ulp) <= 2.0
    assert oracle_lib.exp_det(np.float32([0.0]))[0] == 1.0
    # exact powers of two at x = -k ln2 (rounded) -- the 2^k scaling step
    for k in range(1, 7):
        assert abs(oracle_lib.exp_det(np.float32([-k * math.log(2)]))[0] - 2.0 ** -k) <= 2 * 2.0 ** (-k - 23)


# ------------------------------------------------------------------------------ a1 unproject

def test_golden_spec_examples(oracle_lib):
    """tests/golden/spec_examples.json: S:54-55 (project), S:63 (unproject), S:72 (z = fB/d)."""
    gold = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))
    for ex in gold["project"]:
        pos = np.array([ex["point"]], np.float32)
        cov = np.array([[1e-6, 0, 0, 1e-6, 0, 1e-6]], np.float32)
        K = [ex["fx"], ex["fy"], ex["cx"], ex["cy"]]
        H = W = int(2 * ex["cx"] + 2)
        pr = oracle_lib.project(dict(pos=pos, cov6=cov, alpha=np.ones(1, np.float32)), K, np.eye(3),
                                np.zeros(3), H, W, oracle_lib.make_params())
        assert pr["visible"][0] == 1
        assert np.allclose(pr["mean2"][0], ex["pixel"], atol=1e-4)
        assert pr["dkey"][0:1].view(np.float32)[0] == np.float32(ex["z"])
    for ex in gold["disparity_to_depth"] + gold["unproject"]:
        if "depth" in ex:       # optical axis at depth 2 via a disparity that encodes it
            f, B = ex["fx"], 0.2
            d = f * B / ex["depth"]
            px, py = ex["pixel"]
            want = ex["world"]
        else:
            f, B, d = ex["f"], ex["B"], ex["d"]
            px = py = 4
            want = [0.0, 0.0, ex["z"]]
        c = float(px)
        s = one_pixel_scene(f, c, c, 2 * px + 1, 2 * px + 1, px, py, d, B)
        g = oracle_lib.unproject(s)
        assert g["n"] == 1
        np.testing.assert_allclose(g["pos"][0], want, atol=1e-6)


def test_unproject_invalid_pixels_are_skipped(oracle_lib):
    """d <= d_min, non-finite d, mask 0, NaN opacity: skipped, not errors."""
    s = sg.make_config("tiny", res=16)
    v = s.views[0]
    v.disparity[0, 0] = 0.0
    v.disparity[0, 1] = -3.0
    v.disparity[0, 2] = np.nan
    v.disparity[0, 3] = np.inf
    v.opacity[0, 4] = np.nan
    v.mask = np.ones((16, 16), np.uint8)
    v.mask[0, 5] = 0
    g = oracle_lib.unproject(s, oracle_lib.make_params(default_scale=0.005))
    assert g["n"] == 256 - 6
    assert list(g["ids"]) == list(range(g["n"]))
    # opacity clamp to [0, 1]
    v.opacity[1, 0] = 1.5
    v.opacity[1, 1] = -0.5
    g = oracle_lib.unproject(s, oracle_lib.make_params(default_scale=0.005))
    a = g["alpha"]
    assert a.max() <= 1.0 and a.min() >= 0.0


def test_unproject_positions_lie_on_the_synthetic_body(oracle_lib):
    """Rig scene: every lifted point lies on the ray-cast ellipsoids (S:79 analytic scene)."""
    s = sg.make_config("c3", res=128, target_hw=(64, 64))
    g = oracle_lib.unproject(s)
    res = np.full(g["n"], np.inf)
    for c, a in sg.ELLIPSOIDS:
        r = np.sqrt(np.sum(((g["pos"].astype(np.float64) - c) / a) ** 2, axis=1)) - 1.0
        res = np.minimum(res, np.abs(r) * a.min())          # ~ metres off the surface
    assert res.max() < 2e-6


def test_unproject_project_round_trip(oracle_lib):
    """project(unproject(p, z)) = (p, z) for random cameras, <= 1e-4 px."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        H, W = 40, 56
        f = rng.uniform(30, 3000)
        Rw, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        Rw *= np.sign(np.linalg.det(Rw))
        t = rng.uniform(-1, 1, 3)
        cam = sg.Camera(fx=f, fy=f * rng.uniform(0.8, 1.2), cx=rng.uniform(10, 40), cy=rng.uniform(10, 30),
                        R=Rw, t=t, H=H, W=W)
        d = rng.uniform(1, 50, (H, W)).astype(np.float32)
        v = sg.SourceView(cam=cam, baseline=0.1, disparity=d, mask=None, scale=None, quat=None,
                          opacity=None, feat=np.zeros((H, W, 1), np.float32))
        s = sg.Scene("rt", [v], [cam], 1, "f32", default_scale=1e-4)
        g = oracle_lib.unproject(s, oracle_lib.make_params(default_scale=1e-4))
        K, R, tt = sg.cam_arrays(cam)
        pr = oracle_lib.project(g, K, R, tt, H, W, oracle_lib.make_params(dilation=0.0))
        ys, xs = np.mgrid[0:H, 0:W]
        z = (np.float32(cam.fx) * np.float32(0.1)) / d
        ok = pr["visible"].astype(bool)
        assert ok.mean() > 0.95
        err = np.abs(pr["mean2"] - np.stack([xs.ravel(), ys.ravel()], 1))[ok]
        assert err.max() < 1e-4 * max(1.0, f / 100)
        zz = pr["dkey"].view(np.float32)[ok]
        np.testing.assert_allclose(zz, z.ravel()[ok], rtol=2e-6)


def test_quaternion_covariance_matches_scipy(oracle_lib):
    """Sigma_w = R_q diag(s^2) R_q^T with R_q from the normalised (w,x,y,z) map (R4), vs scipy."""
    from scipy.spatial.transform import Rotation
    s = sg.make_random_scene(11, with_quat=True)
    g = oracle_lib.unproject(s)
    v = s.views[0]
    keep = (v.mask != 0)
    q = v.quat[keep].astype(np.float64)
    sc = v.scale[keep].astype(np.float64)
    Rq = Rotation.from_quat(q[:, [1, 2, 3, 0]]).as_matrix()
    S = Rq @ (sc[:, :, None] ** 2 * np.swapaxes(Rq, 1, 2))
    up = S[:, [0, 0, 0, 1, 1, 2], [0, 1, 2, 1, 2, 2]]
    np.testing.assert_allclose(g["cov6"], up, atol=1e-6 * np.abs(up).max())


# ------------------------------------------------------------------------------ a2 projection

def test_pure_rotation_homography_tiny(oracle_lib):
    """Tiny (target = R_y(5 deg), t = 0): mu' = K R K^-1 [x, y, 1]^T, independent of depth."""
    s = sg.make_config("tiny")
    g = oracle_lib.unproject(s, oracle_lib.make_params(default_scale=0.005))
    tgt = s.targets[0]
    K, R, t = sg.cam_arrays(tgt)
    pr = oracle_lib.project(g, K, R, t, 64, 64, oracle_lib.make_params())
    Km = np.array([[64.0, 0, 31.5], [0, 64.0, 31.5], [0, 0, 1]])
    ys, xs = np.mgrid[0:64, 0:64]
    h = (Km @ tgt.R @ np.linalg.inv(Km) @ np.stack([xs.ravel(), ys.ravel(), np.ones(4096)]))
    mu = (h[:2] / h[2]).T
    ok = pr["visible"].astype(bool)
    assert ok.sum() == 3793        # the survey's independent numpy model
    assert np.abs(pr["mean2"][ok] - mu[ok]).max() < 1e-4


def test_identity_target_isotropic_closed_form(oracle_lib):
    """Identity target, isotropic s: mu = source pixel, Sigma' = (f s / z)^2 I + 0.3 I."""
    f, d, B, sc = 500.0, 25.0, 0.1, 0.004
    s = one_pixel_scene(f, 31.5, 31.5, 64, 64, 40, 20, d, B, scale=[sc] * 3)
    g = oracle_lib.unproject(s)
    K, R, t = sg.cam_arrays(s.targets[0])
    pr = oracle_lib.project(g, K, R, t, 64, 64, oracle_lib.make_params())
    z = f * B / d
    assert np.abs(pr["mean2"][0] - [40, 20]).max() < 1e-4
    var = (f * sc / z) ** 2 + 0.3      # off-axis adds a tiny shear term; bound it
    np.testing.assert_allclose(pr["cov2d"][0, [0, 2]], [var, var], rtol=0.01)
    # exactly on axis the Jacobian has no shear term
    s = one_pixel_scene(f, 31.0, 31.0, 64, 64, 31, 31, d, B, scale=[sc] * 3)
    g = oracle_lib.unproject(s)
    K, R, t = sg.cam_arrays(s.targets[0])
    pr = oracle_lib.project(g, K, R, t, 64, 64, oracle_lib.make_params())
    np.testing.assert_allclose(pr["cov2d"][0], [var, 0.0, var], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(pr["conic"][0], [1 / var, 0.0, 1 / var], rtol=1e-6, atol=1e-9)


def test_ewa_covariance_vs_monte_carlo(oracle_lib):
    """Sigma' - dilation ~ covariance of pinhole-projected samples of N(x, Sigma_w) (linearisation,
    P:386-388 EWA of [kerbl20233d]); independent of the Jacobian code."""
    s = sg.make_random_scene(5, with_quat=True)
    g = oracle_lib.unproject(s)
    tgt = s.targets[0]
    K, R, t = sg.cam_arrays(tgt)
    pr = oracle_lib.project(g, K, R, t, tgt.H, tgt.W, oracle_lib.make_params(dilation=0.0))
    rng = np.random.default_rng(0)
    Rm, tm = R.reshape(3, 3).astype(np.float64), t.astype(np.float64)
    for i in np.nonzero(pr["visible"])[0][:12]:
        c6 = g["cov6"][i].astype(np.float64)
        S = np.array([[c6[0], c6[1], c6[2]], [c6[1], c6[3], c6[4]], [c6[2], c6[4], c6[5]]])
        # shrink the Gaussian so the linearisation error is negligible, then rescale
        k = 1e-3
        X = rng.multivariate_normal(g["pos"][i].astype(np.float64), S * k * k, size=200000)
        Xc = X @ Rm.T + tm
        u = K[0] * Xc[:, 0] / Xc[:, 2] + K[2]
        v = K[1] * Xc[:, 1] / Xc[:, 2] + K[3]
        emp = np.cov(np.stack([u, v])) / (k * k)
        got = np.array([[pr["cov2d"][i, 0], pr["cov2d"][i, 1]], [pr["cov2d"][i, 1], pr["cov2d"][i, 2]]])
        assert np.abs(emp - got).max() < 0.02 * np.abs(got).max()


def test_projection_matches_float64_model_on_rig(oracle_lib):
    """a1+a2 vs oracle/definition64.py (scipy rotations, matrix EWA) on c2/c3/c5-shaped rigs."""
    import oracle.definition64 as D
    for name, res in (("c2", 96), ("c3", 96), ("c5", 64)):
        s = sg.make_config(name, res=res, target_hw=(72, 80))
        g = oracle_lib.unproject(s)
        g64 = D.unproject(s)
        np.testing.assert_allclose(g["pos"], g64["pos"], atol=1e-6)
        tgt = s.targets[0]
        K, R, t = sg.cam_arrays(tgt)
        pr = oracle_lib.project(g, K, R, t, tgt.H, tgt.W)
        p64 = D.project(g64, tgt)
        vis = pr["visible"].astype(bool)
        assert (vis == p64["visible"]).mean() > 0.999
        m = vis & p64["visible"]
        assert np.abs(pr["mean2"][m] - p64["mean"][m]).max() < 1e-4
        c64 = p64["cov2"][m][:, [0, 0, 1], [0, 1, 1]]
        assert (np.abs(pr["cov2d"][m] - c64) / np.abs(c64).max(axis=1, keepdims=True)).max() < 1e-4
        assert (np.abs(pr["rect"][m] - p64["rect"][m]) <= 1).all()
        assert (pr["rect"][m] == p64["rect"][m]).mean() > 0.995
        z = pr["dkey"].view(np.float32)[m]
        np.testing.assert_allclose(z, p64["depth"][m], rtol=1e-6)


# ------------------------------------------------------------------------------ a3-a5 tile lists

@pytest.mark.parametrize("tile", [16, 8])
def test_tile_lists_equal_enumeration_brute_force(oracle_lib, tile):
    """Per tile: every visible Gaussian whose tile rect covers it, sorted by (dkey, id) (R12, R18);
    16 x 16 tiles ([kerbl20233d]) and the 8 x 8 tiles of the CUDA path under 32-px bins."""
    for seed in range(6):
        s = sg.make_random_scene(seed, H=45 + seed, W=70 - seed)
        g = oracle_lib.unproject(s)
        tgt = s.targets[0]
        K, R, t = sg.cam_arrays(tgt)
        pr = oracle_lib.project(g, K, R, t, tgt.H, tgt.W)
        ranges, lst = oracle_lib.tile_lists(pr, g["ids"], tgt.H, tgt.W, tile=tile)
        TX, TY = (tgt.W + tile - 1) // tile, (tgt.H + tile - 1) // tile
        total = 0
        for ty in range(TY):
            for tx in range(TX):
                want = []
                for i in np.nonzero(pr["visible"])[0]:
                    x0, x1, y0, y1 = pr["rect"][i]
                    if x0 // tile <= tx <= x1 // tile and y0 // tile <= ty <= y1 // tile:
                        want.append((int(pr["dkey"][i]), int(g["ids"][i]), int(i)))
                want.sort()
                a, b = ranges[ty * TX + tx]
                assert [w[2] for w in want] == list(lst[a:b])
                total += len(want)
        assert total == len(lst)
        # keys strictly increasing within a tile (a total order: ids unique)
        for a, b in ranges:
            keys = [(int(pr["dkey"][i]), int(g["ids"][i])) for i in lst[a:b]]
            assert all(k1 < k2 for k1, k2 in zip(keys, keys[1:]))


def test_tiny_entry_count(oracle_lib):
    """Tiny: K = 5,400 (independent numpy model)."""
    s = sg.make_config("tiny")
    g = oracle_lib.unproject(s, oracle_lib.make_params(default_scale=0.005))
    r = oracle_lib.rasterize(g, s.targets[0])
    assert len(r["list"]) == 5400


# ------------------------------------------------------------------------------ a6 composite

def test_single_isotropic_gaussian_closed_form(oracle_lib):
    """(i) One isotropic Gaussian: F(p) = f * min(0.99, alpha exp(-r^2/(2 sigma^2))) inside the
    3-sigma disc, 0 outside; A = the same alpha' (S:230 forward model)."""
    f, d, B, sc, al = 400.0, 20.0, 0.1, 0.01, 0.8
    feat = np.array([1.0, -2.0, 0.5, 3.0], np.float32)
    s = one_pixel_scene(f, 31.0, 31.0, 64, 64, 31, 31, d, B, scale=[sc] * 3, alpha=al, feat=feat)
    g = oracle_lib.unproject(s)
    r = oracle_lib.rasterize(g, s.targets[0])
    z = f * B / d
    var = (f * sc / z) ** 2 + 0.3
    ys, xs = np.mgrid[0:64, 0:64]
    r2 = (xs - 31.0) ** 2 + (ys - 31.0) ** 2
    a = np.minimum(0.99, al * np.exp(-0.5 * r2 / var))
    inside = (r2 / var <= 9.0) & (a >= 1 / 255)
    assert inside.sum() > 50
    want = np.where(inside[..., None], a[..., None] * feat, 0.0)
    np.testing.assert_allclose(r["F"], want, atol=2e-6)
    np.testing.assert_allclose(r["A"], np.where(inside, a, 0.0), atol=2e-7)


def test_two_coaxial_gaussians(oracle_lib):
    """(ii) S:234: front alpha' = 0.99 at z=1, back at z=2 -> centre within 1.5% of front."""
    H = W = 33
    c = 16.0
    f = 100.0
    disp = np.full((H, W), 5.0, np.float32)
    mask = np.zeros((H, W), np.uint8)
    mask[16, 16] = 1
    cam = sg.Camera(fx=f, fy=f, cx=c, cy=c, R=np.eye(3), t=np.zeros(3), H=H, W=W)
    views = []
    for z, feat, al in ((1.0, [1.0, 2.0], 1.0), (2.0, [-5.0, 4.0], 0.5)):
        fm = np.zeros((H, W, 2), np.float32)
        fm[16, 16] = feat
        views.append(sg.SourceView(cam=cam, baseline=z * 5.0 / f, disparity=disp, mask=mask,
                                   scale=None, quat=None, opacity=np.full((H, W), al, np.float32),
                                   feat=fm))
    s = sg.Scene("coax", views[::-1], [cam], 2, "f32", default_scale=0.03, default_opacity=1.0)
    g = oracle_lib.unproject(s)
    assert g["n"] == 2 and g["pos"][0, 2] > g["pos"][1, 2]      # back Gaussian has the lower id
    r = oracle_lib.rasterize(g, cam)
    F = r["F"][16, 16]
    assert np.all(np.abs(F - [1.0, 2.0]) <= 0.015 * np.abs([1.0, 2.0]) + 0.05)
    # back alpha' = 0.5 at its centre; T after the front = 0.01 (R9 clamp)
    np.testing.assert_allclose(F, 0.99 * np.array([1.0, 2.0]) + 0.01 * 0.5 * np.array([-5.0, 4.0]),
                               rtol=1e-5)
    np.testing.assert_allclose(r["A"][16, 16], 1 - 0.01 * 0.5, rtol=1e-6)
    # an opaque back Gaussian would take T below 1e-4: it is not composited (R10)
    views[1].opacity[:] = 1.0
    r = oracle_lib.rasterize(oracle_lib.unproject(s), cam)
    np.testing.assert_allclose(r["F"][16, 16], 0.99 * np.array([1.0, 2.0]), rtol=1e-6)


def test_identity_camera_reproduces_source_features(oracle_lib):
    """(iii) north_star closed form: identity target, dilation 0, s = 0.05 z / f (sigma = 0.05 px),
    alpha = 1 -> F = fl(f_src * 0.99f), A = fl(1 - fl(1 - 0.99f)) exactly, every pixel."""
    rng = np.random.default_rng(3)
    H, W, f, B = 37, 53, 60.0, 0.1
    cam = sg.Camera(fx=f, fy=f, cx=(W - 1) / 2, cy=(H - 1) / 2, R=np.eye(3), t=np.zeros(3), H=H, W=W)
    d = rng.uniform(5, 15, (H, W)).astype(np.float32)
    z = (np.float32(f) * np.float32(B)) / d
    sc = (0.05 * z / f).astype(np.float32)
    feat = rng.standard_normal((H, W, 8)).astype(np.float32)
    v = sg.SourceView(cam=cam, baseline=B, disparity=d, mask=None, scale=np.repeat(sc[..., None], 3, -1),
                      quat=None, opacity=np.ones((H, W), np.float32), feat=feat)
    s = sg.Scene("ident", [v], [cam], 8, "f32")
    g = oracle_lib.unproject(s)
    r = oracle_lib.rasterize(g, cam, oracle_lib.make_params(dilation=0.0))
    a = np.float32(0.99)
    assert np.array_equal(r["F"], feat * a)
    assert np.all(r["A"] == np.float32(1.0) - (np.float32(1.0) - a))


def _random_scene_raster(oracle_lib, seed, **kw):
    s = sg.make_random_scene(seed, **kw)
    g = oracle_lib.unproject(s)
    tgt = s.targets[0]
    return s, g, tgt, oracle_lib.rasterize(g, tgt)


def test_tiled_equals_bruteforce_on_50_scenes(oracle_lib):
    """(vii) S:250: tiled == brute force (all Gaussians per pixel, global (dkey,id) order) on
    >= 50 seeded scenes <= 64x64, <= 1000 Gaussians: F, A bit-exact."""
    for seed in range(50):
        H, W = 20 + (seed * 7) % 45, 20 + (seed * 11) % 45
        s, g, tgt, r = _random_scene_raster(oracle_lib, seed, H=H, W=W, n_src=10 + seed % 22,
                                            feat_dtype="f16" if seed % 3 == 0 else "f32")
        assert g["n"] <= 1000
        Fb, Ab, _ = oracle_lib.composite_bruteforce(g, r["proj"], H, W)
        assert np.array_equal(r["F"], Fb), seed
        assert np.array_equal(r["A"], Ab), seed


def test_invariants_alpha_range_monotone_convexity(oracle_lib):
    """(iv) A in [0,1), monotone; (v) |F| <= max|f| per channel."""
    for seed in range(10):
        s, g, tgt, r = _random_scene_raster(oracle_lib, 100 + seed)
        A, F = r["A"], r["F"]
        assert A.min() >= 0.0 and A.max() < 1.0
        fmax = np.abs(g["feat"].astype(np.float32)).max(axis=0)
        assert np.all(np.abs(F) <= fmax * (1 + 1e-6))
        # appending a Gaussian behind everything cannot decrease A anywhere
        far = {k: v.copy() for k, v in g.items() if k != "n"}
        far["pos"] = np.concatenate([far["pos"], [[0.0, 0.0, 50.0]]]).astype(np.float32)
        far["cov6"] = np.concatenate([far["cov6"], [[400, 0, 0, 400, 0, 1]]]).astype(np.float32)
        far["alpha"] = np.concatenate([far["alpha"], [0.9]]).astype(np.float32)
        far["ids"] = np.concatenate([far["ids"], [len(far["ids"])]])
        far["feat"] = np.concatenate([far["feat"], far["feat"][:1]])
        r2 = oracle_lib.rasterize(far, tgt)
        assert np.all(r2["A"] >= A)
        assert np.any(r2["A"] > A)


def test_permutation_invariance_bit_exact(oracle_lib):
    """(vi) S:248: permuting the Gaussian array (ids travel) leaves F, A unchanged, bit for bit."""
    for seed in range(5):
        s, g, tgt, r = _random_scene_raster(oracle_lib, 200 + seed)
        perm = np.random.default_rng(seed).permutation(g["n"])
        gp = {k: (v[perm] if k != "n" else v) for k, v in g.items()}
        rp = oracle_lib.rasterize(gp, tgt)
        assert np.array_equal(r["F"], rp["F"]) and np.array_equal(r["A"], rp["A"])


def test_colour_reduction_channel_independence(oracle_lib):
    """(viii) S:251: with C=3 the latent path is classic colour splatting -- channels composite
    independently, so a C=3 run equals the first 3 channels of a C=8 run bit for bit."""
    s, g, tgt, r = _random_scene_raster(oracle_lib, 300)
    g3 = dict(g)
    g3["feat"] = np.ascontiguousarray(g["feat"][:, :3])
    r3 = oracle_lib.rasterize(g3, tgt)
    assert np.array_equal(r3["F"], r["F"][..., :3]) and np.array_equal(r3["A"], r["A"])


def test_empty_cloud(oracle_lib):
    """empty cloud -> F = 0, A = 0."""
    s = sg.make_config("tiny", res=16)
    s.views[0].mask = np.zeros((16, 16), np.uint8)
    g = oracle_lib.unproject(s)
    assert g["n"] == 0
    r = oracle_lib.rasterize(g, s.targets[0])
    assert np.all(r["F"] == 0) and np.all(r["A"] == 0) and len(r["list"]) == 0


@pytest.mark.parametrize("which", ["tiny", "random"])
def test_composite_matches_float64_model(oracle_lib, which):
    """fp32 oracle vs the float64 definition (oracle/definition64.py) on tie-free scenes:
    max |dF| <= 1e-4 on pixels with the same contributor count, <= 0.5% of pixels differ."""
    import oracle.definition64 as D
    scenes = [sg.make_config("tiny")] if which == "tiny" else [sg.make_random_scene(k, C=8) for k in range(8)]
    for s in scenes:
        p = oracle_lib.make_params(default_scale=s.default_scale, default_opacity=s.default_opacity)
        g = oracle_lib.unproject(s, p)
        tgt = s.targets[0]
        r = oracle_lib.rasterize(g, tgt, p)
        g64 = D.unproject(s)
        p64 = D.project(g64, tgt)
        F64, A64, N64 = D.composite(g64, p64, tgt.H, tgt.W)
        same = r["n_contrib"] == N64
        assert same.mean() >= 0.995
        assert np.abs(r["F"] - F64)[same].max() <= 1e-4
        assert np.abs(r["A"] - A64)[same].max() <= 1e-5


# ------------------------------------------------------------------ NEXT #2: cascade Z-buffer (R23)
# PAPER.md P:351-352 ("lifted to a 3D point cloud ... rasterized to the viewpoints of cam2 and cam3.
# Z-buffers are extracted and converted back to disparity maps"), SPEC.md S:86-94 (points_zbuffer).

def _single_point_view(H, W, fx, cx, cy, px, py, z, B=0.1, R=None, t=None):
    disp = np.zeros((H, W), np.float32)
    disp[py, px] = np.float32(fx * B / z)
    cam = sg.Camera(fx=fx, fy=fx, cx=cx, cy=cy, R=np.eye(3) if R is None else R,
                    t=np.zeros(3) if t is None else t, H=H, W=W)
    return sg.SourceView(cam=cam, baseline=B, disparity=disp, mask=None, scale=None, quat=None,
                         opacity=None, feat=np.zeros((H, W, 8), np.float32))


def test_zbuffer_point_on_axis(oracle_lib):
    """one point on the optical axis at z = 2 -> single valid pixel at the principal point
    with depth 2 (splat radius 0); its disparity is fx*B/2."""
    import oracle
    v = _single_point_view(1, 1, 100.0, 0.0, 0.0, 0, 0, 2.0, B=0.2)
    tgt = sg.Camera(fx=100.0, fy=100.0, cx=7.0, cy=5.0, R=np.eye(3), t=np.zeros(3), H=11, W=15)
    _, depth, disp = oracle.zbuffer([v], tgt, 0.2, radius=0)
    assert np.count_nonzero(depth) == 1
    assert depth[5, 7] == np.float32(2.0)
    assert disp[5, 7] == np.float32(100.0 * 0.2 / 2.0)
    _, depth1, _ = oracle.zbuffer([v], tgt, 0.2, radius=1)      # radius 1: the 3 x 3 neighbourhood
    assert np.count_nonzero(depth1) == 9 and np.all(depth1[4:7, 6:9] == np.float32(2.0))


def test_zbuffer_min_z_and_tie_break(oracle_lib):
    """two points projecting to the same pixel with z = 1 and z = 3 -> depth 1, whatever
    the order of the views; equal depths resolve to the lowest source index."""
    import oracle
    tgt = sg.Camera(fx=100.0, fy=100.0, cx=4.0, cy=4.0, R=np.eye(3), t=np.zeros(3), H=9, W=9)
    a = _single_point_view(1, 1, 100.0, 0.0, 0.0, 0, 0, 1.0)
    b = _single_point_view(1, 1, 100.0, 0.0, 0.0, 0, 0, 3.0)
    for vs in ([a, b], [b, a]):
        zk, depth, _ = oracle.zbuffer(vs, tgt, 0.1, radius=0)
        assert depth[4, 4] == np.float32(1.0)
    zk, _, _ = oracle.zbuffer([a, a], tgt, 0.1, radius=0)
    assert int(zk[4, 4]) & 0xffffffff == 0                     # tie: the first view's pixel wins


def test_zbuffer_cascade_matches_ground_truth_depth(oracle_lib):
    """S:94 (derived): cam0's depth of the synthetic upper body warped into cam2 matches cam2's
    analytic (ray-cast) depth: median |error| < 5 mm on pixels both see."""
    import oracle
    s = sg.make_config("c3", res=256)
    cam0, cam2 = s.views[0], s.views[2]
    _, depth, disp = oracle.zbuffer([cam0], cam2.cam, cam2.baseline, radius=1)
    gt = np.where(cam2.mask != 0, np.float32(cam2.cam.fx * cam2.baseline) / cam2.disparity, 0.0)
    both = (depth > 0) & (gt > 0)
    assert both.mean() > 0.15
    err = np.abs(depth[both] - gt[both])
    assert np.median(err) < 0.005, np.median(err)
    # the disparity map is fx * B / z of the same pixels
    assert np.allclose(disp[both], np.float32(cam2.cam.fx) * np.float32(cam2.baseline) / depth[both], rtol=1e-6)


def test_zbuffer_matches_float64_model(oracle_lib):
    """Whole-rig z-buffer vs the independent float64 model (oracle/definition64.py): identical
    occupancy and depths within 1e-5 relative except where fp32 and float64 round a pixel centre
    to different pixels (mu within ~1e-5 px of a half-integer), which must be rare."""
    import oracle
    import oracle.definition64 as d64
    s = sg.make_config("c2", res=128)
    tgt = s.targets[0]
    _, depth, _ = oracle.zbuffer(s.views, tgt, 0.1, radius=1)
    ref = d64.zbuffer(s.views, tgt, radius=1)
    occ = (depth > 0) != (ref > 0)
    assert occ.mean() < 1e-3
    both = (depth > 0) & (ref > 0)
    rel = np.abs(depth[both] - ref[both]) / ref[both]
    assert np.mean(rel < 1e-5) > 0.999, np.mean(rel < 1e-5)


# ------------------------------------------------------ NEXT #1: occlusion-aware blending (R24)
# PAPER.md P:420-444 (Eqs. 6-10), SPEC.md S:282-312 (fuse_depth_to_novel, backproject_sample,
# visibility_weight, blend_views).

def _plane_view(H, W, f, z, color, tilt_deg=0.0, B=0.1):
    """A camera at the origin looking at a plane through (0, 0, z): fronto-parallel, or rotated about
    the y axis by tilt_deg (depth per pixel by ray-plane intersection); constant colour."""
    cam = sg.Camera(fx=f, fy=f, cx=(W - 1) / 2, cy=(H - 1) / 2, R=np.eye(3), t=np.zeros(3), H=H, W=W)
    xs = (np.arange(W) - cam.cx) / f
    ys = (np.arange(H) - cam.cy) / f
    n = np.array([np.sin(np.radians(tilt_deg)), 0.0, -np.cos(np.radians(tilt_deg))])
    dirs = np.stack(np.broadcast_arrays(xs[None, :], ys[:, None], np.ones((H, W))), -1)
    zz = (n @ np.array([0.0, 0.0, z])) / (dirs @ n)          # camera-space z of the hit
    disp = (f * B / zz).astype(np.float32)
    col = np.broadcast_to(np.asarray(color, np.float32), (H, W, 3)).copy()
    v = sg.SourceView(cam=cam, baseline=B, disparity=disp, mask=None, scale=None, quat=None, opacity=None,
                      feat=np.zeros((H, W, 8), np.float32))
    return v, col


def test_blend_frontal_weight_half_at_two_metres(oracle_lib):
    """frontal surface (cos = 1), all masks pass, ||x_i^cam|| = 2 m -> w_i = 0.5; one
    nonzero weight -> the output is that view's colour."""
    import oracle
    v, col = _plane_view(9, 9, 50.0, 2.0, (0.2, 0.4, 0.6))
    _, zf, _ = oracle.zbuffer([v], v.cam, 0.1, radius=0)
    rgb, ws = oracle.blend([v], [col], v.cam, zf)
    assert ws[4, 4] == np.float32(0.5)
    assert np.array_equal(rgb[4, 4], np.float32([0.2, 0.4, 0.6]))


def test_blend_occlusion_gate(oracle_lib):
    """|x_i.z - z_i| = 2 delta -> w_i = 0 (the pixel becomes a hole); just inside delta it counts."""
    import oracle
    v, col = _plane_view(9, 9, 50.0, 1.0, (0.5, 0.5, 0.5))
    zf = np.full((9, 9), np.float32(1.0 + 0.02), np.float32)
    _, ws = oracle.blend([v], [col], v.cam, zf, delta=0.01)
    assert ws[4, 4] == 0.0
    zf = np.full((9, 9), np.float32(1.005), np.float32)
    _, ws = oracle.blend([v], [col], v.cam, zf, delta=0.01)
    assert ws[4, 4] > 0.0


def test_blend_cosine_and_grazing(oracle_lib):
    """Eq. 8's cosine: a plane tilted 60 deg about y, seen head-on along the optical axis, weighs
    cos(60 deg) / distance; tilted to 90 deg the surface is grazing (no valid depth ahead)."""
    import oracle
    v, col = _plane_view(41, 41, 200.0, 1.0, (0.3, 0.3, 0.3), tilt_deg=60.0)
    _, zf, _ = oracle.zbuffer([v], v.cam, 0.1, radius=0)
    _, ws = oracle.blend([v], [col], v.cam, zf, edge_tau=1.0)
    assert abs(ws[20, 20] * 1.0 - 0.5) < 2e-3            # distance 1 m on the axis, cos 60 = 0.5


def test_blend_two_views_equal_weights_average(oracle_lib):
    """two views with equal weights and colours a, b -> (a + b) / 2 (|a - b| = 0.122 within the
    appearance-consistency threshold tau_c = 0.15; with the mask off the same holds for any colours)."""
    import oracle
    va, ca = _plane_view(9, 9, 50.0, 1.5, (0.4, 0.3, 0.5))
    vb, cb = _plane_view(9, 9, 50.0, 1.5, (0.5, 0.35, 0.45))
    _, zf, _ = oracle.zbuffer([va], va.cam, 0.1, radius=0)
    rgb, ws = oracle.blend([va, vb], [ca, cb], va.cam, zf)
    assert np.allclose(rgb[2:7, 2:7], np.float32([0.45, 0.325, 0.475]), atol=1e-7)
    vc, cc = _plane_view(9, 9, 50.0, 1.5, (0.6, 0.2, 0.0))
    rgb, ws = oracle.blend([va, vc], [ca, cc], va.cam, zf, tau_c=0.0)
    assert np.allclose(rgb[2:7, 2:7], np.float32([0.5, 0.25, 0.25]), atol=1e-7)


def test_blend_appearance_consistency_drops_outlier(oracle_lib):
    """SPEC.md l.300 / l.331 (the appearance-consistency mask of P:430-433): three equally weighted views
    of a plane, two agreeing colours a, b and an outlier o (|o - a| = 0.8 > tau_c): the weighted median
    sample is a or b, o is dropped, I_blend = (a + b) / 2 exactly like two views; the outlier's weight
    leaves the denominator (wsum = 2 w instead of 3 w).  A tau_c above every distance (or 0 = off)
    restores the three-view mean; the medoid is a sample, so a pixel never loses all its samples."""
    import oracle
    va, ca = _plane_view(9, 9, 50.0, 1.5, (0.4, 0.3, 0.5))
    vb, cb = _plane_view(9, 9, 50.0, 1.5, (0.45, 0.3, 0.5))
    vo, co = _plane_view(9, 9, 50.0, 1.5, (0.4, 0.3, 1.3))
    _, zf, _ = oracle.zbuffer([va], va.cam, 0.1, radius=0)
    rgb, ws = oracle.blend([va, vb, vo], [ca, cb, co], va.cam, zf)
    _, ws1 = oracle.blend([va], [ca], va.cam, zf)
    assert np.allclose(rgb[2:7, 2:7], np.float32([0.425, 0.3, 0.5]), atol=1e-7)
    assert np.allclose(ws[2:7, 2:7], 2 * ws1[2:7, 2:7], rtol=1e-6)
    for tau in (0.0, 2.0):
        rgb3, ws3 = oracle.blend([va, vb, vo], [ca, cb, co], va.cam, zf, tau_c=tau)
        assert np.allclose(rgb3[2:7, 2:7], np.float32([(0.4 + 0.45 + 0.4) / 3, 0.3, (0.5 + 0.5 + 1.3) / 3]), atol=1e-6)
        assert np.allclose(ws3[2:7, 2:7], 3 * ws1[2:7, 2:7], rtol=1e-6)
    rgb2, ws2 = oracle.blend([vo, va], [co, ca], va.cam, zf)        # two disagreeing views: the medoid survives
    assert np.all(ws2[2:7, 2:7] > 0) and np.allclose(rgb2[2:7, 2:7], np.float32([0.4, 0.3, 1.3]), atol=1e-7)


def test_blend_zero_weight_is_hole_even_with_w_min_zero(oracle_lib):
    """S:308 / S:333: a pixel with no valid sample is a hole of colour 0 -- also when the hole
    threshold w_min is 0 (no 0/0): background pixels of the rig (z_fused = 0) and pixels no view sees
    stay exactly 0 and finite."""
    import oracle
    s = sg.make_config("c3", res=96)
    cam = sg.make_targets("c4", res=96, n_targets=3)[1]
    colors = [sg.view_colors(v.cam) for v in s.views]
    _, zf, _ = oracle.zbuffer(s.views, cam, 0.1, radius=1)
    rgb, ws = oracle.blend(s.views, colors, cam, zf, w_min=0.0)
    assert np.all(np.isfinite(rgb))
    assert (ws == 0).sum() > 100 and np.all(rgb[ws == 0] == 0.0)
    rgb1, _ = oracle.blend(s.views, colors, cam, zf)
    assert np.array_equal(rgb[ws >= 1e-4], rgb1[ws >= 1e-4])


def test_blend_textured_body_psnr_and_convexity(oracle_lib):
    """S:312 (derived): the occlusion-free Lambertian synthetic scene (the world-space texture on the
    upper body) blended from the 4 rig views into a parallax target matches the texture at the
    target's own ray-cast hits: PSNR >= 31 dB (33.1 dB measured when fixed); S:326 convexity: every
    blended colour lies within the texture's range; holes inside the body are rare."""
    import oracle
    s = sg.make_config("c3", res=256)
    cam = sg.make_targets("c4", res=256, n_targets=3)[1]
    colors = [sg.view_colors(v.cam) for v in s.views]
    _, zf, _ = oracle.zbuffer(s.views, cam, 0.1, radius=1)
    rgb, ws = oracle.blend(s.views, colors, cam, zf)
    Xw, fg = sg.raycast_points(cam)
    gt = sg.texture(Xw)
    ok = (ws >= 1e-4) & fg
    assert (fg & (ws < 1e-4)).mean() < 0.01
    psnr = 10 * np.log10(1.0 / np.mean((rgb[ok] - gt[ok]) ** 2))
    assert psnr >= 31.0, psnr
    assert rgb[ok].min() >= np.float32(0.15) - 1e-6 and rgb[ok].max() <= np.float32(0.85) + 1e-6


def test_blend_matches_float64_model(oracle_lib):
    """The fp32 blending oracle vs the independent float64 model (oracle/definition64.py) on the
    textured rig, same z_fused: colours within 1e-4 wherever both give a blended pixel; the pixels
    whose thresholds (Occ, edge mask, validity) fall differently in fp32 and float64 are rare."""
    import oracle
    import oracle.definition64 as d64
    s = sg.make_config("c3", res=192)
    cam = sg.make_targets("c4", res=192, n_targets=3)[0]
    colors = [sg.view_colors(v.cam) for v in s.views]
    _, zf, _ = oracle.zbuffer(s.views, cam, 0.1, radius=1)
    rgb, ws = oracle.blend(s.views, colors, cam, zf)
    rgb64, ws64 = d64.blend(s.views, colors, cam, zf)
    both = (ws >= 1e-4) & (ws64 >= 1e-4)
    assert ((ws >= 1e-4) != (ws64 >= 1e-4)).mean() < 1e-3
    close = np.all(np.abs(rgb - rgb64) < 1e-4, axis=-1) & np.isclose(ws, ws64, rtol=1e-4)
    assert close[both].mean() > 0.995, close[both].mean()


# ----------------------------------------------------- NEXT #4: compositing backward pass (R25)

def test_backward_matches_finite_differences(oracle_lib):
    """The oracle's analytic gradients of L = sum G_F . F + G_A A (R25) against central
    finite differences of the independent float64 forward (definition64.composite2d) on a small
    random scene, for the parameters with the largest gradients (perturbations that flip a per-pixel
    decision are skipped: the gradient is defined with the decisions held fixed)."""
    import oracle
    import oracle.definition64 as d64
    s = sg.make_random_scene(3, H=24, W=20, C=4, n_src=14)
    s.views[0].feat = s.views[0].feat.astype(np.float32)
    op = oracle.make_params(default_scale=s.default_scale, default_opacity=s.default_opacity)
    g = oracle.unproject(s, op)
    cam = s.targets[0]
    K, R, t = sg.cam_arrays(cam)
    pr = oracle.project(g, K, R, t, cam.H, cam.W, op)
    ranges, lst = oracle.tile_lists(pr, g["ids"], cam.H, cam.W)
    rng = np.random.default_rng(7)
    GF = rng.standard_normal((cam.H, cam.W, s.C)).astype(np.float32)
    GA = rng.standard_normal((cam.H, cam.W)).astype(np.float32)
    grads = oracle.composite_backward(g, pr, ranges, lst, cam.H, cam.W, GF, GA, op)
    vis = np.nonzero(pr["visible"])[0]
    order = vis[np.lexsort((g["ids"][vis], pr["dkey"][vis]))]
    mean = pr["mean2"].astype(np.float64)
    conic = pr["conic"].astype(np.float64)
    alpha = g["alpha"].astype(np.float64)
    feat = g["feat"].astype(np.float64)
    rect = pr["rect"]

    def loss(mean_, conic_, alpha_, feat_):
        F, A, used = d64.composite2d(mean_, conic_, alpha_, feat_, rect, order, cam.H, cam.W)
        return float(np.sum(F * GF) + np.sum(A * GA)), used

    _, used0 = loss(mean, conic, alpha, feat)
    checked = 0
    for name, arr in (("mean2", mean), ("conic", conic), ("alpha", alpha), ("feat", feat)):
        an = grads[name]
        flat = np.argsort(-np.abs(an).reshape(-1))[:6]
        for fi in flat:
            idx = np.unravel_index(fi, an.shape)
            eps = 1e-4 * max(1.0, abs(arr[idx]))
            vals = []
            flipped = False
            for sgn in (1, -1):
                pert = [mean.copy(), conic.copy(), alpha.copy(), feat.copy()]
                k = ("mean2", "conic", "alpha", "feat").index(name)
                pert[k][idx] += sgn * eps
                L, used = loss(*pert)
                flipped |= used != used0
                vals.append(L)
            if flipped:
                continue
            fd = (vals[0] - vals[1]) / (2 * eps)
            assert abs(fd - an[idx]) <= 2e-3 * max(1.0, abs(fd)), (name, idx, fd, an[idx])
            checked += 1
    assert checked >= 16, checked


# ------------------------------------------------------------------------------ R8: the box is a conservative 3-sigma bound

def _min_q_outside_box(rect, mean, conic, H, W):
    """Smallest q = d^T conic d over the image pixels OUTSIDE each Gaussian's pixel box, in float64.
    q is convex and the centre lies inside the box (R18 rounding), so on each half-plane beyond a box
    edge the minimum is on the pixel line next to that edge; along the line it is at one of the two
    integers around the continuous minimiser (clamped to the image).  Edges on the image border have
    no outside pixels.  Returns one value per Gaussian (inf if the box covers the whole image)."""
    x0, x1, y0, y1 = (rect[:, k].astype(np.float64) for k in range(4))
    mx, my = mean[:, 0], mean[:, 1]
    a, b, c = conic[:, 0, 0], conic[:, 0, 1], conic[:, 1, 1]
    best = np.full(len(rect), np.inf)

    def along(fixed, is_x, ok):
        # points (fixed, y) (is_x) or (x, fixed); minimiser of the other coordinate, clamped
        if is_x:
            dx = fixed - mx
            ys = my - b * dx / c
            for yy in (np.floor(ys), np.ceil(ys)):
                dy = np.clip(yy, 0, H - 1) - my
                q = a * dx * dx + 2 * b * dx * dy + c * dy * dy
                np.minimum(best, np.where(ok, q, np.inf), out=best)
        else:
            dy = fixed - my
            xs = mx - b * dy / a
            for xx in (np.floor(xs), np.ceil(xs)):
                dx = np.clip(xx, 0, W - 1) - mx
                q = a * dx * dx + 2 * b * dx * dy + c * dy * dy
                np.minimum(best, np.where(ok, q, np.inf), out=best)

    along(x0 - 1, True, x0 > 0)
    along(x1 + 1, True, x1 < W - 1)
    along(y0 - 1, False, y0 > 0)
    along(y1 + 1, False, y1 < H - 1)
    return best


def _r8_margin(oracle_lib, scene, cam):
    """fp32 oracle boxes (a2) vs the exact float64 ellipse of definition64: min q outside the boxes."""
    from oracle import definition64 as D
    go = oracle_lib.unproject(scene)
    K, R, t = sg.cam_arrays(cam)
    pr = oracle_lib.project(go, K, R, t, cam.H, cam.W)
    g64 = D.unproject(scene)
    p64 = D.project(g64, cam)
    vis = pr["visible"].astype(bool)
    assert vis.sum() > 0
    assert np.all(p64["visible"][vis]), "fp32-visible Gaussian culled in float64"
    conic = np.linalg.inv(p64["cov2"][vis])
    q = _min_q_outside_box(pr["rect"][vis].astype(np.int64), p64["mean"][vis], conic, cam.H, cam.W)
    return float(q.min()), int(vis.sum())


@pytest.mark.parametrize("cfg,res", [("c2", 512), ("c3", 512), ("c5", 512)])
def test_r8_box_conservative_rig(oracle_lib, cfg, res):
    """DESIGN.md R8 / R18: the fp32 pixel box (h = 3 sqrt(Sigma'_xx)(1 + 2^-10) + 2^-10) contains every
    pixel whose exact (float64) Mahalanobis q is <= 9, so including the box in the inclusion predicate
    never drops a 3-sigma pixel: on the c2-, c3- and c5-shaped rigs (anisotropic, random rotations)
    every pixel outside every visible Gaussian's box has float64 q > 9."""
    s = sg.make_config(cfg, res=res, n_targets=1) if cfg == "c5" else sg.make_config(cfg, res=res)
    qmin, nvis = _r8_margin(oracle_lib, s, s.targets[0])
    assert nvis > 10000
    assert qmin > 9.0, qmin


def test_r8_box_conservative_random_anisotropic(oracle_lib):
    """R8 on 24 random anisotropic scenes (random rotations, log-normal scales), 8 of them with one
    axis stretched x 8 (needle-like footprints at every orientation): no pixel outside an fp32 box
    has float64 q <= 9."""
    worst = np.inf
    for seed in range(24):
        s = sg.make_random_scene(seed, H=40 + seed, W=64 - seed, n_src=20)
        if seed % 3 == 0:
            s.views[0].scale[..., seed % 3] *= 8.0
        qmin, _ = _r8_margin(oracle_lib, s, s.targets[0])
        worst = min(worst, qmin)
    assert worst > 9.0, worst
