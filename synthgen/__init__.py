"""Seeded synthetic inputs for the latent-Gaussian rasterizer (shared by tests, oracle and bench).

This module holds NO arithmetic of the method (no unprojection, projection, EWA,
binning or compositing).  It only synthesises the *inputs* the method consumes:
source views (disparity / mask / encoder maps / cameras) and target cameras, with
the shapes and value distributions BASELINE.json `configs` names (see DESIGN.md
"Input recipe").  The paper's THuman data (§5.1) is absent; these
seeded maps stand in for the encoder outputs M_f, M_s, M_alpha of Eq. 4
 and for the cascade's disparity maps.

Scene geometry (rig, ellipsoid body, plane) is built by ray casting analytic
shapes in float64: that is scene synthesis, the inverse of what the method does.

Conventions (R1): OpenCV camera axes (x right, y down, z forward),
extrinsics are world->camera X_c = R X_w + t, integer pixel (x, y) is the pixel
centre, principal point at the centre c = (W-1)/2.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

__all__ = [
    "Camera", "SourceView", "Scene", "make_config", "CONFIG_NAMES", "look_at",
    "rot_y", "make_random_scene",
]

CONFIG_NAMES = ("tiny", "c2", "c3", "c4", "c5", "paper")


@dataclass
class Camera:
    """Pinhole camera: intrinsics (pixels) + world->camera pose, H x W pixels."""
    fx: float
    fy: float
    cx: float
    cy: float
    R: np.ndarray  # (3,3) float64, world->camera, row-major
    t: np.ndarray  # (3,)  float64
    H: int
    W: int


@dataclass
class SourceView:
    cam: Camera
    baseline: float                    # metres; z = fx * baseline / d (R2)
    disparity: np.ndarray              # (H,W) float32, pixels
    mask: Optional[np.ndarray]         # (H,W) uint8 or None (= all ones)
    scale: Optional[np.ndarray]        # (H,W,3) float32 metres or None (-> default_scale)
    quat: Optional[np.ndarray]         # (H,W,4) float32 raw (w,x,y,z) or None (-> identity)
    opacity: Optional[np.ndarray]      # (H,W) float32 or None (-> default_opacity)
    feat: np.ndarray                   # (H,W,C) float32 or float16


@dataclass
class Scene:
    name: str
    views: List[SourceView]
    targets: List[Camera]
    C: int
    feat_dtype: str                    # "f32" | "f16"
    default_scale: float = 0.0
    default_opacity: float = 1.0
    notes: dict = field(default_factory=dict)

    @property
    def n_pixels(self) -> int:
        return sum(v.cam.H * v.cam.W for v in self.views)


# ----------------------------------------------------------------------------- cameras

def rot_y(deg: float) -> np.ndarray:
    """Right-handed rotation about +y by `deg` degrees (R17)."""
    a = math.radians(deg)
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]], dtype=np.float64)


def look_at(centre, target) -> tuple:
    """World->camera (R, t) for a camera at `centre` looking at `target`.

    OpenCV axes with world y pointing down (the display frame of the rig): camera
    z = forward, x = down x forward (right), y = forward x right (down).
    """
    c = np.asarray(centre, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - c
    f /= np.linalg.norm(f)
    down = np.array([0.0, 1.0, 0.0])
    x = np.cross(down, f)
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    R = np.stack([x, y, f])
    t = -R @ c
    return R, t


def _pinhole(W: int, H: int, focal_scale: float, R, t) -> Camera:
    f = focal_scale * W
    return Camera(fx=f, fy=f, cx=(W - 1) / 2.0, cy=(H - 1) / 2.0, R=np.asarray(R, np.float64),
                  t=np.asarray(t, np.float64), H=H, W=W)


# ----------------------------------------------------------------------------- rig scene
# SURVEY.md §8(d) "Rig": world = display frame, cams left/right/above the display
# (upper narrow pair cam0/cam1, lower wide pair cam2/cam3).
RIG_LOOK = np.array([0.0, 0.05, 1.45])
RIG_CAMS = {
    "cam0": (np.array([-0.06, -0.25, 0.0]), 0.12),
    "cam1": (np.array([0.06, -0.25, 0.0]), 0.12),
    "cam2": (np.array([-0.33, 0.0, 0.0]), 0.66),
    "cam3": (np.array([0.33, 0.0, 0.0]), 0.66),
}
# upper-body proxy: torso + head ellipsoids at 1.2-1.6 m over a background plane at 3 m
ELLIPSOIDS = (
    (np.array([0.0, 0.30, 1.55]), np.array([0.25, 0.36, 0.16])),
    (np.array([0.0, -0.20, 1.32]), np.array([0.085, 0.115, 0.10])),
)
PLANE_Z = 3.0
FOCAL_SCALE = 1.95
_BASE_ELLIPSOIDS = ELLIPSOIDS


def set_focal_scale(f: float = 1.95) -> None:
    """SURVEY 8(d) sensitivity: focal length f = f_scale * W for every rig camera and target, with the
    body scaled by 1.95 / f_scale about the look-at point so its image (and the ~40 % foreground) stays
    put while the Gaussians (metric scales unchanged) cover 1.95 / f_scale times fewer pixels per axis.
    1.95 is the human-scale headline."""
    global FOCAL_SCALE, ELLIPSOIDS
    k = 1.95 / float(f)
    FOCAL_SCALE = float(f)
    ELLIPSOIDS = tuple((RIG_LOOK + k * (c - RIG_LOOK), k * a) for c, a in _BASE_ELLIPSOIDS)


def _raycast_depth(cam: Camera):
    """Camera-space depth z of the first hit (ellipsoids, else plane) and the fg mask."""
    H, W = cam.H, cam.W
    xs = (np.arange(W, dtype=np.float64) - cam.cx) / cam.fx
    ys = (np.arange(H, dtype=np.float64) - cam.cy) / cam.fy
    dc = np.stack(np.broadcast_arrays(xs[None, :], ys[:, None], np.ones((H, W))), axis=-1)
    dw = dc @ cam.R            # R^T d_c, row vectors
    origin = -cam.R.T @ cam.t
    best = np.full((H, W), np.inf)
    for centre, axes in ELLIPSOIDS:
        o = (origin - centre) / axes
        d = dw / axes
        a = np.einsum("hwk,hwk->hw", d, d)
        b = 2.0 * np.einsum("hwk,k->hw", d, o)
        c = float(o @ o) - 1.0
        disc = b * b - 4 * a * c
        ok = disc >= 0
        sq = np.sqrt(np.where(ok, disc, 0.0))
        t0 = (-b - sq) / (2 * a)
        t1 = (-b + sq) / (2 * a)
        tt = np.where(t0 > 1e-6, t0, t1)
        hit = ok & (tt > 1e-6)
        best = np.where(hit & (tt < best), tt, best)
    fg = np.isfinite(best)
    tplane = (PLANE_Z - origin[2]) / dw[..., 2]
    z = np.where(fg, best, tplane)   # d_c has unit z, so the ray parameter is camera z
    return z, fg


# Procedural surface colour (input-view blending): an RGB pattern fixed in world
# space, so every view sees the same colour at the same surface point (a Lambertian scene) and the
# novel view's ground truth is the pattern at its own ray-cast hit.
_TEX_DIRS = np.array([[1.0, 0.3, 0.2], [-0.2, 1.0, 0.4], [0.3, -0.5, 1.0]])
_TEX_PHASE = np.array([0.3, 1.7, 2.9])
TEX_WAVELENGTH = 0.06      # metres


def texture(Xw: np.ndarray) -> np.ndarray:
    """RGB in [0.15, 0.85] of world points (..., 3) -> (..., 3) float64."""
    arg = 2.0 * np.pi * (Xw @ _TEX_DIRS.T) / TEX_WAVELENGTH + _TEX_PHASE
    return 0.5 + 0.35 * np.sin(arg)


def raycast_points(cam: Camera):
    """World point of the first hit (ellipsoids, else the background plane) per pixel + fg mask."""
    z, fg = _raycast_depth(cam)
    H, W = cam.H, cam.W
    xs = (np.arange(W, dtype=np.float64) - cam.cx) / cam.fx
    ys = (np.arange(H, dtype=np.float64) - cam.cy) / cam.fy
    Xc = np.stack(np.broadcast_arrays(xs[None, :] * z, ys[:, None] * z, z), axis=-1)
    Xw = (Xc - cam.t) @ cam.R
    return Xw, fg


def view_colors(cam: Camera) -> np.ndarray:
    """The RGB image [H][W][3] float32 a camera sees of the textured synthetic scene."""
    Xw, _ = raycast_points(cam)
    return texture(Xw).astype(np.float32)


def _rig_view(name: str, res: int, rng, log_mu: float, alpha_lo: float, C: int) -> SourceView:
    centre, baseline = RIG_CAMS[name]
    R, t = look_at(centre, RIG_LOOK)
    cam = _pinhole(res, res, FOCAL_SCALE, R, t)
    z, fg = _raycast_depth(cam)
    disparity = (cam.fx * baseline / z).astype(np.float32)
    # draw order per view: scale -> quat -> opacity -> features
    scale = np.exp(rng.normal(log_mu, 0.3, size=(res, res, 3))).astype(np.float32)
    quat = rng.standard_normal((res, res, 4)).astype(np.float32)
    opacity = rng.uniform(alpha_lo, 0.99, size=(res, res)).astype(np.float32)
    feat = np.empty((res, res, C), dtype=np.float16)
    rows = max(1, (1 << 22) // max(1, res * C))
    for r0 in range(0, res, rows):
        r1 = min(res, r0 + rows)
        feat[r0:r1] = rng.standard_normal((r1 - r0, res, C)).astype(np.float16)
    return SourceView(cam=cam, baseline=baseline, disparity=disparity,
                      mask=fg.astype(np.uint8), scale=scale, quat=quat, opacity=opacity, feat=feat)


def _arc_centre():
    """c3 target: on the arc between the pairs."""
    up = (RIG_CAMS["cam0"][0] + RIG_CAMS["cam1"][0]) / 2
    lo = (RIG_CAMS["cam2"][0] + RIG_CAMS["cam3"][0]) / 2
    u, l = up - RIG_LOOK, lo - RIG_LOOK
    rbar = 0.5 * (np.linalg.norm(u) + np.linalg.norm(l))
    d = u / np.linalg.norm(u) + l / np.linalg.norm(l)
    return RIG_LOOK + rbar * d / np.linalg.norm(d)


def _parallax_targets(n: int, res_w: int, res_h: int, span_deg: float = 15.0) -> List[Camera]:
    """n targets: the c3 centre rotated about the vertical axis through S by
    phi_j = -span + 2 span j/(n-1) (autostereoscopic parallax)."""
    c0 = _arc_centre()
    out = []
    for j in range(n):
        phi = -span_deg + (2 * span_deg * j / (n - 1) if n > 1 else 0.0)
        c = RIG_LOOK + rot_y(phi) @ (c0 - RIG_LOOK)
        R, t = look_at(c, RIG_LOOK)
        out.append(_pinhole(res_w, res_h, FOCAL_SCALE, R, t))
    return out


def make_rig_scene(name: str, res: int, cams, C: int, log_mu: float, alpha_lo: float,
                   targets: List[Camera], seed: int = 0) -> Scene:
    rng = np.random.default_rng(seed)
    views = [_rig_view(cn, res, rng, log_mu, alpha_lo, C) for cn in cams]
    return Scene(name=name, views=views, targets=targets, C=C, feat_dtype="f16")


def make_config(name: str, seed: int = 0, res: Optional[int] = None,
                target_hw: Optional[tuple] = None, n_targets: Optional[int] = None) -> Scene:
    """BASELINE.json configs: tiny (configs[0]), c2..c5 (configs[1..4]).

    `res` / `target_hw` / `n_targets` override sizes for parity cases that keep a
    config's distributions at a size the CPU oracle finishes in seconds.
    """
    if name == "tiny":
        H = W = res or 64
        rng = np.random.default_rng(seed)
        disparity = rng.uniform(8.0, 16.0, size=(H, W)).astype(np.float32)
        opacity = rng.uniform(0.3, 0.99, size=(H, W)).astype(np.float32)
        feat = rng.standard_normal((H, W, 8)).astype(np.float32)
        src = _pinhole(W, H, 1.0, np.eye(3), np.zeros(3))
        src.fx = src.fy = 64.0 * W / 64.0
        th, tw = target_hw or (H, W)
        tgt = Camera(fx=src.fx, fy=src.fy, cx=(tw - 1) / 2.0, cy=(th - 1) / 2.0, R=rot_y(5.0),
                     t=np.zeros(3), H=th, W=tw)
        v = SourceView(cam=src, baseline=0.1, disparity=disparity, mask=None, scale=None, quat=None,
                       opacity=opacity, feat=feat)
        return Scene(name="tiny", views=[v], targets=[tgt], C=8, feat_dtype="f32",
                     default_scale=0.005, default_opacity=1.0)
    if name == "c2":
        r = res or 512
        th, tw = target_hw or (r, r)
        R, t = look_at([0.0, 0.0, 0.0], RIG_LOOK)
        tgt = _pinhole(tw, th, FOCAL_SCALE, R, t)
        return make_rig_scene("c2", r, ("cam2", "cam3"), 32, math.log(0.004), 0.5, [tgt], seed)
    if name in ("c3", "c4"):
        r = res or 1024
        th, tw = target_hw or (r, r)
        if name == "c3":
            R, t = look_at(_arc_centre(), RIG_LOOK)
            targets = [_pinhole(tw, th, FOCAL_SCALE, R, t)]
        else:
            targets = _parallax_targets(n_targets or 32, tw, th)
        return make_rig_scene(name, r, ("cam0", "cam1", "cam2", "cam3"), 32, math.log(0.004), 0.5,
                              targets, seed)
    if name == "c5":
        r = res or 2048
        th, tw = target_hw or (r, r)
        return make_rig_scene("c5", r, ("cam0", "cam1", "cam2", "cam3"), 64, math.log(0.008), 0.2,
                              _parallax_targets(n_targets or 8, tw, th), seed)
    if name == "paper":
        # SURVEY 8(f) NEXT #3, the paper-exact variant: the three lifted views cam0, cam2, cam3
        # (P:358), rotation = identity (no quaternion map, so Sigma_w is diagonal), and the
        # two eye targets of one viewer per frame (left / right eye 64 mm apart on the c3 arc,
        # looking at S).  Same depth / scale / opacity / feature distributions as c3.
        r = res or 1024
        th, tw = target_hw or (r, r)
        sc = make_rig_scene("paper", r, ("cam0", "cam2", "cam3"), 32, math.log(0.004), 0.5, eye_targets(tw, th), seed)
        for v in sc.views:
            v.quat = None
        return sc
    raise ValueError(f"unknown config {name!r}; expected one of {CONFIG_NAMES}")


IPD = 0.064   # metres between the two eye targets of the paper-exact variant


def eye_targets(W: int, H: int) -> List[Camera]:
    """Left and right eye cameras: the c3 target centre moved -/+ IPD/2 along the display's x axis,
    both looking at S."""
    c = _arc_centre()
    out = []
    for sgn in (-1.0, 1.0):
        R, t = look_at(c + np.array([sgn * IPD / 2.0, 0.0, 0.0]), RIG_LOOK)
        out.append(_pinhole(W, H, FOCAL_SCALE, R, t))
    return out


def make_random_scene(seed: int, H: int = 48, W: int = 48, C: int = 8, n_src: int = 24,
                      feat_dtype: str = "f32", with_quat: bool = True) -> Scene:
    """Small random scene for property tests: one n_src x n_src source view with random
    disparity / anisotropic scales / rotations / opacities, seen by a randomly rotated
    and shifted target camera of H x W pixels (ragged vs 16x16 tiles)."""
    rng = np.random.default_rng(seed)
    s = n_src
    disparity = rng.uniform(4.0, 12.0, size=(s, s)).astype(np.float32)
    mask = (rng.uniform(size=(s, s)) < 0.85).astype(np.uint8)
    scale = np.exp(rng.normal(math.log(0.02), 0.5, size=(s, s, 3))).astype(np.float32)
    quat = rng.standard_normal((s, s, 4)).astype(np.float32) if with_quat else None
    opacity = rng.uniform(0.05, 1.0, size=(s, s)).astype(np.float32)
    featd = rng.standard_normal((s, s, C))
    feat = featd.astype(np.float16 if feat_dtype == "f16" else np.float32)
    src = Camera(fx=40.0, fy=40.0, cx=(s - 1) / 2, cy=(s - 1) / 2, R=np.eye(3), t=np.zeros(3), H=s, W=s)
    ang = rng.uniform(-8, 8)
    tgt = Camera(fx=float(rng.uniform(40, 70)), fy=float(rng.uniform(40, 70)), cx=(W - 1) / 2 + rng.uniform(-3, 3),
                 cy=(H - 1) / 2 + rng.uniform(-3, 3), R=rot_y(ang), t=rng.uniform(-0.05, 0.05, size=3), H=H, W=W)
    v = SourceView(cam=src, baseline=0.1, disparity=disparity, mask=mask, scale=scale, quat=quat,
                   opacity=opacity, feat=feat)
    return Scene(name=f"random{seed}", views=[v], targets=[tgt], C=C, feat_dtype=feat_dtype,
                 default_scale=0.01, default_opacity=1.0)


def cam_arrays(cam: Camera):
    """The float32 values both implementations receive at the boundary:
    K = (fx, fy, cx, cy), R (9, row-major, world->camera), t (3)."""
    K = np.array([cam.fx, cam.fy, cam.cx, cam.cy], dtype=np.float32)
    R = np.ascontiguousarray(cam.R, dtype=np.float32).reshape(9)
    t = np.ascontiguousarray(cam.t, dtype=np.float32).reshape(3)
    return K, R, t


DEFAULT_PARAMS = dict(dilation=0.3, alpha_max=0.99, alpha_min=float(np.float32(1.0 / 255.0)),
                      t_eps=1e-4, cull_sigma=3.0, z_near=0.01, d_min=0.0)


def make_targets(name: str, res: Optional[int] = None, target_hw: Optional[tuple] = None,
                 n_targets: Optional[int] = None) -> List[Camera]:
    """Target cameras of a config without synthesising the source maps (for ranks that only render)."""
    if name == "c2":
        r = res or 512
        th, tw = target_hw or (r, r)
        R, t = look_at([0.0, 0.0, 0.0], RIG_LOOK)
        return [_pinhole(tw, th, FOCAL_SCALE, R, t)]
    if name == "c3":
        r = res or 1024
        th, tw = target_hw or (r, r)
        R, t = look_at(_arc_centre(), RIG_LOOK)
        return [_pinhole(tw, th, FOCAL_SCALE, R, t)]
    if name == "c4":
        r = res or 1024
        th, tw = target_hw or (r, r)
        return _parallax_targets(n_targets or 32, tw, th)
    if name == "c5":
        r = res or 2048
        th, tw = target_hw or (r, r)
        return _parallax_targets(n_targets or 8, tw, th)
    if name == "paper":
        r = res or 1024
        th, tw = target_hw or (r, r)
        return eye_targets(tw, th)
    return make_config(name, res=res, target_hw=target_hw, n_targets=n_targets).targets


def crop_camera(cam: Camera, x0: int, y0: int, w: int, h: int) -> Camera:
    """The w x h window at (x0, y0) of `cam` as a camera of its own (same rays)."""
    return Camera(fx=cam.fx, fy=cam.fy, cx=cam.cx - x0, cy=cam.cy - y0, R=cam.R, t=cam.t, H=h, W=w)
