"""CPU oracle for the latent-Gaussian rasterizer (ctypes wrapper around taoracle.c).

TEST INFRASTRUCTURE ONLY -- only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import this package.  The product path
(paper_2405_14866_b200) never imports it; the two share no code.

Functions follow PAPER.md:
  unproject   a1  P:358 (disparity -> depth), P:374 (Gaussian properties)
  project     a2  P:386-388 (EWA splatting of [kerbl20233d])
  tile_lists  a3-a5  P:387 (tile binning + depth order of [kerbl20233d])
  composite   a6  P:386 F_novel = R_G({G}, Pi_novel), front-to-back
and the DESIGN.md readings R1-R18.  Pins: tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "taoracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain IEEE fp32, no contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Intr(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float)]


class _Extr(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3)]


class _Params(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("dilation", "alpha_max", "alpha_min", "t_eps", "cull_sigma",
                                         "z_near", "d_min", "default_scale", "default_opacity")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        i64, i32 = C.c_int64, C.c_int
        _lib.tao_exp_det.restype = C.c_float
        _lib.tao_exp_det.argtypes = [C.c_float]
        _lib.tao_exp_det_array.argtypes = [i64, P, P]
        _lib.tao_unproject_view.restype = i64
        _lib.tao_unproject_view.argtypes = [i32, i32, P, P, P, P, C.c_float, P, P, P, P, i32, i32, P,
                                            i64, P, P, P, P, P]
        _lib.tao_project.argtypes = [i64, P, P, P, P, i32, i32, P, P, P, P, P, P, P]
        _lib.tao_count_entries.restype = i64
        _lib.tao_count_entries.argtypes = [i64, P, P]
        _lib.tao_tile_lists.restype = i64
        _lib.tao_tile_lists.argtypes = [i64, P, P, P, P, i32, i32, P, P]
        _lib.tao_count_entries_tiled.restype = i64
        _lib.tao_count_entries_tiled.argtypes = [i64, P, P, i32]
        _lib.tao_tile_lists_tiled.restype = i64
        _lib.tao_tile_lists_tiled.argtypes = [i64, P, P, P, P, i32, i32, i32, P, P]
        _lib.tao_composite_tiles.argtypes = [i32, i32, i32, i32, P, P, P, P, P, P, P, P, P, i64, P, P,
                                             P, P]
        _lib.tao_zbuffer_view.argtypes = [i32, i32, P, P, P, P, C.c_float, P, i64, P, P, i32, i32, i32, P]
        _lib.tao_zbuffer_resolve.argtypes = [i64, P, C.c_float, C.c_float, P, P]
        _lib.tao_blend.argtypes = [i32, P, P, P, P, P, i32, i32, P, P, P]
        _lib.tao_composite_backward.argtypes = [i32, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, P, P, P, P]
        _lib.tao_composite_bruteforce.argtypes = [i32, i32, i32, i32, i64, P, P, P, P, P, P, P, P, P,
                                                  i32, i32, P, P, P]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def make_params(**kw) -> _Params:
    d = dict(dilation=0.3, alpha_max=0.99, alpha_min=float(np.float32(1.0 / 255.0)), t_eps=1e-4,
             cull_sigma=3.0, z_near=0.01, d_min=0.0, default_scale=0.0, default_opacity=1.0)
    d.update(kw)
    return _Params(**{k: float(v) for k, v in d.items()})


def _intr(K):
    K = np.asarray(K, np.float32)
    return _Intr(*[float(v) for v in K])


def _extr(R, t):
    e = _Extr()
    for i, v in enumerate(np.asarray(R, np.float32).reshape(9)):
        e.R[i] = float(v)
    for i, v in enumerate(np.asarray(t, np.float32).reshape(3)):
        e.t[i] = float(v)
    return e


def exp_det(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty_like(x)
    lib().tao_exp_det_array(x.size, _p(x), _p(y))
    return y


def _cam(cam):
    K = np.array([cam.fx, cam.fy, cam.cx, cam.cy], np.float32)
    return K, np.asarray(cam.R, np.float32), np.asarray(cam.t, np.float32)


def unproject(scene, params=None):
    """a1 over all views of a synthgen.Scene -> dict of Gaussian arrays (array order = id order)."""
    p = params or make_params(default_scale=scene.default_scale, default_opacity=scene.default_opacity)
    fb = 2 if scene.feat_dtype == "f16" else 4
    dt = np.float16 if fb == 2 else np.float32
    total = scene.n_pixels
    pos = np.empty((total, 3), np.float32)
    alpha = np.empty(total, np.float32)
    cov6 = np.empty((total, 6), np.float32)
    ids = np.empty(total, np.int64)
    feat = np.empty((total, scene.C), dt)
    n = 0
    for v in scene.views:
        K, R, t = _cam(v.cam)
        arrs = [np.ascontiguousarray(a) if a is not None else None
                for a in (v.disparity, v.mask, v.scale, v.quat, v.opacity, v.feat)]
        disp, mask, scale, quat, opac, f = arrs
        assert f.dtype == dt
        k = lib().tao_unproject_view(v.cam.H, v.cam.W, _p(disp), _p(mask), C.byref(_intr(K)),
                                     C.byref(_extr(R, t)), float(np.float32(v.baseline)), _p(scale),
                                     _p(quat), _p(opac), _p(f), scene.C, fb, C.byref(p), n,
                                     _p(pos[n:]), _p(alpha[n:]), _p(cov6[n:]), _p(ids[n:]),
                                     _p(feat[n:]))
        n += k
    return dict(pos=pos[:n].copy(), alpha=alpha[:n].copy(), cov6=cov6[:n].copy(), ids=ids[:n].copy(),
                feat=feat[:n].copy(), n=n)


def project(g, K, R, t, H, W, params=None):
    """a2 -> dict(visible, mean2, conic, cov2d, rect, dkey)."""
    p = params or make_params()
    n = len(g["alpha"])
    out = dict(visible=np.zeros(n, np.int32), mean2=np.zeros((n, 2), np.float32),
               conic=np.zeros((n, 3), np.float32), cov2d=np.zeros((n, 3), np.float32),
               rect=np.zeros((n, 4), np.int32), dkey=np.zeros(n, np.uint32))
    pos = np.ascontiguousarray(g["pos"], np.float32)
    cov6 = np.ascontiguousarray(g["cov6"], np.float32)
    lib().tao_project(n, _p(pos), _p(cov6), C.byref(_intr(K)), C.byref(_extr(R, t)), H, W, C.byref(p),
                      _p(out["visible"]), _p(out["mean2"]), _p(out["conic"]), _p(out["cov2d"]),
                      _p(out["rect"]), _p(out["dkey"]))
    return out


def tile_lists(pr, ids, H, W, tile=16):
    """a3-a5 -> (ranges[T,2] uint32, list[K] int64 array indices) ordered by (tile, dkey, id), for
    square tiles of side `tile` (16 = [kerbl20233d]; 8 = the CUDA path's tiles under 32-px bins)."""
    n = len(pr["visible"])
    ids = np.ascontiguousarray(ids, np.int64)
    K = lib().tao_count_entries_tiled(n, _p(pr["visible"]), _p(pr["rect"]), int(tile))
    T = ((W + tile - 1) // tile) * ((H + tile - 1) // tile)
    ranges = np.zeros((T, 2), np.uint32)
    lst = np.zeros(max(K, 1), np.int64)
    lib().tao_tile_lists_tiled(n, _p(pr["visible"]), _p(pr["rect"]), _p(pr["dkey"]), _p(ids), H, W, int(tile),
                               _p(ranges), _p(lst))
    return ranges, lst[:K]


def composite(g, pr, ranges, lst, H, W, params=None, tiles=None):
    """a6 tiled -> (F[H,W,C] f32, A[H,W] f32, n_contrib[H,W], n_eval[H,W]).  `tiles` limits
    the work to a subset of tile indices (other pixels stay NaN)."""
    p = params or make_params()
    feat = np.ascontiguousarray(g["feat"])
    Cc = feat.shape[1]
    fb = feat.dtype.itemsize
    F = np.full((H, W, Cc), np.nan, np.float32)
    A = np.full((H, W), np.nan, np.float32)
    nc = np.full((H, W), -1, np.int32)
    ne = np.full((H, W), -1, np.int32)
    tl = None if tiles is None else np.ascontiguousarray(tiles, np.int32)
    lst = np.ascontiguousarray(lst, np.int64)
    lib().tao_composite_tiles(H, W, Cc, fb, _p(np.ascontiguousarray(g["alpha"], np.float32)),
                              _p(pr["mean2"]), _p(pr["conic"]), _p(pr["rect"]), _p(feat), _p(ranges),
                              _p(lst), C.byref(p), _p(tl), 0 if tl is None else len(tl), _p(F), _p(A),
                              _p(nc), _p(ne))
    return F, A, nc, ne


def composite_bruteforce(g, pr, H, W, params=None, rows=None):
    """a6 without tiles: all visible Gaussians in (dkey, id) order per pixel."""
    p = params or make_params()
    feat = np.ascontiguousarray(g["feat"])
    Cc = feat.shape[1]
    y0, y1 = rows or (0, H)
    F = np.full((H, W, Cc), np.nan, np.float32)
    A = np.full((H, W), np.nan, np.float32)
    nc = np.full((H, W), -1, np.int32)
    n = len(pr["visible"])
    lib().tao_composite_bruteforce(H, W, Cc, feat.dtype.itemsize, n, _p(pr["visible"]), _p(pr["dkey"]),
                                   _p(np.ascontiguousarray(g["ids"], np.int64)),
                                   _p(np.ascontiguousarray(g["alpha"], np.float32)), _p(pr["mean2"]),
                                   _p(pr["conic"]), _p(pr["rect"]), _p(feat), C.byref(p), y0, y1, _p(F),
                                   _p(A), _p(nc))
    return F, A, nc


def rasterize(g, cam, params=None, tiles=None):
    """Whole hot path for one target camera (a2-a6) on a lifted Gaussian set."""
    K, R, t = _cam(cam)
    pr = project(g, K, R, t, cam.H, cam.W, params)
    ranges, lst = tile_lists(pr, g["ids"], cam.H, cam.W)
    F, A, nc, ne = composite(g, pr, ranges, lst, cam.H, cam.W, params, tiles)
    return dict(proj=pr, ranges=ranges, list=lst, F=F, A=A, n_contrib=nc, n_eval=ne)


def zbuffer(views, cam, baseline_tgt, radius=1, params=None):
    """NEXT #2 (R23): lift the valid pixels of the
    source views (synthgen.SourceView list, source index = running pixel offset over the views),
    splat min-z (tie-break lowest source index) into `cam` with splat radius `radius`.
    Returns (zkey[H,W] uint64, depth[H,W] f32 (0 = empty), disparity[H,W] f32 = fx*B/z (0 = empty))."""
    p = params or make_params()
    zkey = np.full(cam.H * cam.W, np.iinfo(np.uint64).max, np.uint64)
    Kt, Rt, tt = _cam(cam)
    off = 0
    for v in views:
        K, R, t = _cam(v.cam)
        disp = np.ascontiguousarray(v.disparity, np.float32)
        mask = None if v.mask is None else np.ascontiguousarray(v.mask, np.uint8)
        lib().tao_zbuffer_view(v.cam.H, v.cam.W, _p(disp), _p(mask), C.byref(_intr(K)), C.byref(_extr(R, t)),
                               float(np.float32(v.baseline)), C.byref(p), off, C.byref(_intr(Kt)),
                               C.byref(_extr(Rt, tt)), cam.H, cam.W, int(radius), _p(zkey))
        off += v.cam.H * v.cam.W
    depth = np.empty(cam.H * cam.W, np.float32)
    disp = np.empty(cam.H * cam.W, np.float32)
    lib().tao_zbuffer_resolve(zkey.size, _p(zkey), float(np.float32(cam.fx)), float(np.float32(baseline_tgt)),
                              _p(depth), _p(disp))
    return zkey.reshape(cam.H, cam.W), depth.reshape(cam.H, cam.W), disp.reshape(cam.H, cam.W)


class _BView(C.Structure):
    _fields_ = [("H", C.c_int32), ("W", C.c_int32), ("disp", C.c_void_p), ("mask", C.c_void_p),
                ("K", C.c_float * 4), ("R", C.c_float * 9), ("t", C.c_float * 3), ("baseline", C.c_float),
                ("color", C.c_void_p)]


class _BParams(C.Structure):
    _fields_ = [("delta", C.c_float), ("edge_tau", C.c_float), ("w_min", C.c_float), ("tau_c", C.c_float)]


def blend(views, colors, cam, z_fused, delta=0.01, edge_tau=0.02, w_min=1e-4, tau_c=0.15, params=None):
    """NEXT #1 (Eqs. 6-10; R24): occlusion-aware blending of the input
    views' colours into `cam` over the fused depth z_fused[H, W] (0 = none, e.g. zbuffer(...)[1]).
    colors: list of [H_i, W_i, 3] float32; tau_c: appearance-consistency threshold (SPEC.md l.331, 0 = off).
    Returns (rgb[H, W, 3] f32, wsum[H, W] f32)."""
    p = params or make_params()
    keep = []
    arr = (_BView * len(views))()
    for k, (v, col) in enumerate(zip(views, colors)):
        K, R, t = _cam(v.cam)
        disp = np.ascontiguousarray(v.disparity, np.float32)
        mask = None if v.mask is None else np.ascontiguousarray(v.mask, np.uint8)
        col = np.ascontiguousarray(col, np.float32)
        keep += [disp, mask, col]
        b = arr[k]
        b.H, b.W = v.cam.H, v.cam.W
        b.disp, b.mask, b.color = disp.ctypes.data, (None if mask is None else mask.ctypes.data), col.ctypes.data
        for j in range(4):
            b.K[j] = float(K[j])
        for j in range(9):
            b.R[j] = float(R.reshape(-1)[j])
        for j in range(3):
            b.t[j] = float(t[j])
        b.baseline = float(np.float32(v.baseline))
    bp = _BParams(float(delta), float(edge_tau), float(w_min), float(tau_c))
    Kn, Rn, tn = _cam(cam)
    zf = np.ascontiguousarray(z_fused, np.float32)
    rgb = np.empty((cam.H, cam.W, 3), np.float32)
    ws = np.empty((cam.H, cam.W), np.float32)
    lib().tao_blend(len(views), arr, C.byref(p), C.byref(bp), C.byref(_intr(Kn)), C.byref(_extr(Rn, tn)), cam.H,
                    cam.W, _p(zf), _p(rgb), _p(ws))
    return rgb, ws


def composite_backward(g, pr, ranges, lst, H, W, GF, GA, params=None):
    """NEXT #4 (R25): gradients of L = sum G_F . F + G_A A of the tiled a6 forward with
    respect to each Gaussian's mean2 [n,2], conic (ca, cb2, cc) [n,3], alpha [n] and feature row
    [n,C] (array order; float64 sums of fp32 per-pixel terms)."""
    p = params or make_params()
    feat = np.ascontiguousarray(g["feat"])
    n, Cc = feat.shape
    out = dict(mean2=np.zeros((n, 2)), conic=np.zeros((n, 3)), alpha=np.zeros(n), feat=np.zeros((n, Cc)))
    lib().tao_composite_backward(H, W, Cc, feat.dtype.itemsize, _p(np.ascontiguousarray(g["alpha"], np.float32)),
                                 _p(pr["mean2"]), _p(pr["conic"]), _p(pr["rect"]), _p(feat), _p(ranges),
                                 _p(np.ascontiguousarray(lst, np.int64)), C.byref(p),
                                 _p(np.ascontiguousarray(GF, np.float32)), _p(np.ascontiguousarray(GA, np.float32)),
                                 _p(out["mean2"]), _p(out["conic"]), _p(out["alpha"]), _p(out["feat"]))
    return out
