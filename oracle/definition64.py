"""Float64 model of the rasterizer definition -- an independent PIN for taoracle.c.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Written separately from
taoracle.c with whole-array linear algebra instead of the normative scalar
sequence: matrices are built with numpy / scipy (quaternion -> matrix via
scipy.spatial.transform.Rotation), the EWA covariance as J W Sigma W^T J^T
(PAPER.md P:386-388 via [kerbl20233d]), compositing per pixel with cumulative
products.  Real arithmetic in float64; its decisions (q <= 9, stop at T < 1e-4)
can therefore differ from the fp32 oracle on pixels that straddle a threshold,
which the pins count and bound instead of requiring equality.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial.transform import Rotation

MARGIN_REL = 1.0 + 2.0 ** -10
MARGIN_ABS = 2.0 ** -10


def unproject(scene, d_min=0.0):
    """a1 in float64: returns pos (n,3), cov (n,3,3), alpha (n,), ids (n,), feat (n,C) float64."""
    P, S, A, F = [], [], [], []
    for v in scene.views:
        cam = v.cam
        H, W = cam.H, cam.W
        d = v.disparity.astype(np.float64)
        keep = np.isfinite(d) & (d > d_min)
        if v.mask is not None:
            keep &= v.mask != 0
        op = (v.opacity.astype(np.float64) if v.opacity is not None
              else np.full((H, W), scene.default_opacity))
        keep &= ~np.isnan(op)
        ys, xs = np.nonzero(keep)                       # row-major order
        fx, fy = np.float64(np.float32(cam.fx)), np.float64(np.float32(cam.fy))
        cx, cy = np.float64(np.float32(cam.cx)), np.float64(np.float32(cam.cy))
        B = np.float64(np.float32(v.baseline))
        R = cam.R.astype(np.float32).astype(np.float64)
        t = cam.t.astype(np.float32).astype(np.float64)
        z = fx * B / d[ys, xs]
        Xc = np.stack([(xs - cx) / fx * z, (ys - cy) / fy * z, z], axis=1)
        P.append((Xc - t) @ R)                          # R^T (X_c - t) as row vectors
        if v.scale is not None:
            s = v.scale[ys, xs].astype(np.float64)
        else:
            s = np.full((len(xs), 3), np.float64(np.float32(scene.default_scale)))
        if v.quat is not None:
            q = v.quat[ys, xs].astype(np.float64)       # (w, x, y, z)
            Rq = Rotation.from_quat(q[:, [1, 2, 3, 0]]).as_matrix()
        else:
            Rq = np.broadcast_to(np.eye(3), (len(xs), 3, 3))
        S.append(Rq @ (s[:, :, None] ** 2 * np.swapaxes(Rq, 1, 2)))
        A.append(np.clip(op[ys, xs], 0.0, 1.0))
        F.append(v.feat[ys, xs].astype(np.float64))
    pos = np.concatenate(P)
    return dict(pos=pos, cov=np.concatenate(S), alpha=np.concatenate(A), feat=np.concatenate(F),
                ids=np.arange(len(pos)))


def project(g, cam, dilation=0.3, cull_sigma=3.0, z_near=0.01):
    """a2 in float64 -> visible, mean (n,2), cov2 (n,2,2), rect (n,4), depth (n,)."""
    fx, fy = np.float64(np.float32(cam.fx)), np.float64(np.float32(cam.fy))
    cx, cy = np.float64(np.float32(cam.cx)), np.float64(np.float32(cam.cy))
    R = cam.R.astype(np.float32).astype(np.float64)
    t = cam.t.astype(np.float32).astype(np.float64)
    X = g["pos"] @ R.T + t
    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    ok = z > z_near
    zs = np.where(ok, z, 1.0)
    mean = np.stack([fx * x / zs + cx, fy * y / zs + cy], axis=1)
    n = len(z)
    J = np.zeros((n, 2, 3))
    J[:, 0, 0] = fx / zs
    J[:, 0, 2] = -fx * x / zs ** 2
    J[:, 1, 1] = fy / zs
    J[:, 1, 2] = -fy * y / zs ** 2
    T = J @ R
    cov2 = T @ g["cov"] @ np.swapaxes(T, 1, 2) + dilation * np.eye(2)
    det = np.linalg.det(cov2)
    ok &= det > 0
    h = cull_sigma * np.sqrt(np.stack([cov2[:, 0, 0], cov2[:, 1, 1]], axis=1)) * MARGIN_REL + MARGIN_ABS
    lo = np.ceil(mean - h)
    hi = np.floor(mean + h)
    lim = np.array([cam.W - 1, cam.H - 1], np.float64)
    ok &= np.all(lo <= lim, axis=1) & np.all(hi >= 0, axis=1)
    lo = np.clip(lo, 0, lim)
    hi = np.clip(hi, 0, lim)
    ok &= np.all(lo <= hi, axis=1)
    rect = np.stack([lo[:, 0], hi[:, 0], lo[:, 1], hi[:, 1]], axis=1).astype(np.int64)
    return dict(visible=ok, mean=mean, cov2=cov2, rect=rect, depth=z)


def composite(g, pr, H, W, alpha_max=0.99, alpha_min=1.0 / 255.0, t_eps=1e-4, cull_sigma=3.0):
    """a6 brute force in float64: every pixel over all visible Gaussians by (depth, id)."""
    vis = np.nonzero(pr["visible"])[0]
    # R12: the depth order key is the camera depth as an fp32 number, ties by id
    zkey = pr["depth"][vis].astype(np.float32)
    order = vis[np.lexsort((g["ids"][vis], zkey))]
    mean = pr["mean"][order]
    conic = np.linalg.inv(pr["cov2"][order])
    rect = pr["rect"][order]
    al = g["alpha"][order]
    feat = g["feat"][order]
    C = feat.shape[1]
    F = np.zeros((H, W, C))
    A = np.zeros((H, W))
    NC = np.zeros((H, W), np.int64)
    for py in range(H):
        rowmask = (rect[:, 2] <= py) & (py <= rect[:, 3])
        idx = np.nonzero(rowmask)[0]
        if len(idx) == 0:
            continue
        for px in range(W):
            sel = idx[(rect[idx, 0] <= px) & (px <= rect[idx, 1])]
            if len(sel) == 0:
                continue
            d = np.array([px, py], np.float64) - mean[sel]
            q = np.einsum("ni,nij,nj->n", d, conic[sel], d)
            a = np.minimum(alpha_max, al[sel] * np.exp(-0.5 * q))
            use = (q <= cull_sigma ** 2) & (a >= alpha_min)
            sel, a = sel[use], a[use]
            if len(sel) == 0:
                continue
            Tn = np.cumprod(1.0 - a)
            stop = np.nonzero(Tn < t_eps)[0]
            m = stop[0] if len(stop) else len(a)
            Tb = np.concatenate([[1.0], Tn[:m]])
            w = a[:m] * Tb[:m]
            F[py, px] = w @ feat[sel[:m]]
            A[py, px] = 1.0 - Tb[m]
            NC[py, px] = m
    return F, A, NC


def zbuffer(views, cam, radius=1, z_near=0.01, d_min=0.0):
    """NEXT #2 in float64 with array ops: lift every valid
    pixel, project with K [R | t], nearest pixel by np.rint, min z over the (2r+1)^2 splat.
    Returns depth[H, W] float64 (0 = no point)."""
    H, W = cam.H, cam.W
    best = np.full((H, W), np.inf)
    R2 = np.asarray(cam.R, np.float32).astype(np.float64)
    t2 = np.asarray(cam.t, np.float32).astype(np.float64)
    f2 = np.float64(np.float32(cam.fx)), np.float64(np.float32(cam.fy))
    c2 = np.float64(np.float32(cam.cx)), np.float64(np.float32(cam.cy))
    for v in views:
        sc = v.cam
        d = v.disparity.astype(np.float64)
        keep = np.isfinite(d) & (d > d_min)
        if v.mask is not None:
            keep &= v.mask != 0
        ys, xs = np.nonzero(keep)
        fx, fy = np.float64(np.float32(sc.fx)), np.float64(np.float32(sc.fy))
        cx, cy = np.float64(np.float32(sc.cx)), np.float64(np.float32(sc.cy))
        z = fx * np.float64(np.float32(v.baseline)) / d[ys, xs]
        Xc = np.stack([(xs - cx) / fx * z, (ys - cy) / fy * z, z], axis=1)
        R = np.asarray(sc.R, np.float32).astype(np.float64)
        t = np.asarray(sc.t, np.float32).astype(np.float64)
        Xw = (Xc - t) @ R
        X = Xw @ R2.T + t2
        ok = X[:, 2] > z_near
        X = X[ok]
        px = np.rint(f2[0] * X[:, 0] / X[:, 2] + c2[0]).astype(np.int64)
        py = np.rint(f2[1] * X[:, 1] / X[:, 2] + c2[1]).astype(np.int64)
        for dy in range(-radius, radius + 1):
            for dx in range(-radius, radius + 1):
                qx, qy = px + dx, py + dy
                inb = (qx >= 0) & (qx < W) & (qy >= 0) & (qy < H)
                np.minimum.at(best, (qy[inb], qx[inb]), X[inb, 2])
    return np.where(np.isfinite(best), best, 0.0)


def blend(views, colors, cam, z_fused, delta=0.01, edge_tau=0.02, w_min=1e-4, z_near=0.01, d_min=0.0, tau_c=0.15):
    """NEXT #1 (Eqs. 6-10) in float64 with array operations: lift every pixel of
    z_fused, project into each view, bilinear colour / depth, Occ, edge mask, finite-difference
    normal, cos / distance weights, the appearance-consistency mask (the weighted
    medoid of the weighted samples by a full distance matrix, keep samples within tau_c of it; 0 = off),
    normalised sum.  Returns (rgb[H, W, 3], wsum[H, W]) float64."""
    H, W = cam.H, cam.W
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    R, t = f32(cam.R), f32(cam.t)
    fx, fy, cx, cy = (np.float64(np.float32(v)) for v in (cam.fx, cam.fy, cam.cx, cam.cy))
    vv, uu = np.nonzero(z_fused > 0)
    z = z_fused[vv, uu].astype(np.float64)
    Xc = np.stack([(uu - cx) / fx * z, (vv - cy) / fy * z, z], 1)
    Xw = (Xc - t) @ R
    C0 = -t @ R
    ray = Xw - C0
    ray /= np.linalg.norm(ray, axis=1, keepdims=True)
    Wv, Cv = [], []
    for v, col in zip(views, colors):
        sc = v.cam
        Ri, ti = f32(sc.R), f32(sc.t)
        fxi, fyi, cxi, cyi = (np.float64(np.float32(a)) for a in (sc.fx, sc.fy, sc.cx, sc.cy))
        d = v.disparity.astype(np.float64)
        valid = np.isfinite(d) & (d > d_min)
        if v.mask is not None:
            valid &= v.mask != 0
        zmap = np.where(valid, fxi * np.float64(np.float32(v.baseline)) / np.where(valid, d, 1.0), np.nan)
        Hi, Wi = sc.H, sc.W
        X = Xw @ Ri.T + ti
        Z = X[:, 2]
        with np.errstate(divide="ignore", invalid="ignore"):
            us = fxi * X[:, 0] / Z + cxi
            vs = fyi * X[:, 1] / Z + cyi
        ok = (Z > z_near) & (us >= 0) & (us <= Wi - 1) & (vs >= 0) & (vs <= Hi - 1)
        x0 = np.clip(np.floor(np.where(ok, us, 0)).astype(int), 0, max(Wi - 2, 0))
        y0 = np.clip(np.floor(np.where(ok, vs, 0)).astype(int), 0, max(Hi - 2, 0))
        x1, y1 = np.minimum(x0 + 1, Wi - 1), np.minimum(y0 + 1, Hi - 1)
        ax, ay = us - x0, vs - y0
        taps = [zmap[y0, x0], zmap[y0, x1], zmap[y1, x0], zmap[y1, x1]]
        ok &= np.all(np.isfinite(np.stack(taps)), axis=0)
        zs = (taps[0] * (1 - ax) + taps[1] * ax) * (1 - ay) + (taps[2] * (1 - ax) + taps[3] * ax) * ay
        ok &= np.abs(Z - zs) < delta
        px = np.clip(np.rint(np.where(ok, us, 0)).astype(int), 0, Wi - 1)
        py = np.clip(np.rint(np.where(ok, vs, 0)).astype(int), 0, Hi - 1)
        inb = (px >= 1) & (px <= Wi - 2) & (py >= 1) & (py <= Hi - 2)
        ok &= inb
        pxs, pys = np.clip(px, 1, Wi - 2), np.clip(py, 1, Hi - 2)

        def P(x, y):
            zz = zmap[y, x]
            return np.stack([(x - cxi) / fxi * zz, (y - cyi) / fyi * zz, zz], 1)
        zl, zr, zu, zd = zmap[pys, pxs - 1], zmap[pys, pxs + 1], zmap[pys - 1, pxs], zmap[pys + 1, pxs]
        ok &= np.isfinite(zl) & np.isfinite(zr) & np.isfinite(zu) & np.isfinite(zd) & np.isfinite(zmap[pys, pxs])
        with np.errstate(invalid="ignore"):
            ok &= np.maximum(np.abs(zr - zl), np.abs(zd - zu)) * 0.5 <= edge_tau
        n = np.cross(P(pxs + 1, pys) - P(pxs - 1, pys), P(pxs, pys + 1) - P(pxs, pys - 1))
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        flip = np.einsum("ij,ij->i", n, P(pxs, pys)) > 0
        n[flip] *= -1
        nw = n @ Ri
        cs = -np.einsum("ij,ij->i", ray, nw)
        ok &= cs > 0
        w = np.where(ok, cs / np.linalg.norm(X, axis=1), 0.0)
        c = col.astype(np.float64)
        cb = ((c[y0, x0] * (1 - ax)[:, None] + c[y0, x1] * ax[:, None]) * (1 - ay)[:, None] +
              (c[y1, x0] * (1 - ax)[:, None] + c[y1, x1] * ax[:, None]) * ay[:, None])
        Wv.append(w)
        Cv.append(np.nan_to_num(cb))
    Wm = np.stack(Wv, 1)                      # [pixels, views]
    Cm = np.stack(Cv, 1)                      # [pixels, views, 3]
    if tau_c > 0:
        # weighted medoid: the sample minimising the weighted sum of colour distances (ties: lowest view)
        dist = np.linalg.norm(Cm[:, :, None, :] - Cm[:, None, :, :], axis=3)        # [p, i, j]
        cost = np.einsum("pij,pj->pi", dist, Wm)
        cost = np.where(Wm > 0, cost, np.inf)
        med = Cm[np.arange(len(z)), np.argmin(cost, axis=1)]
        keep = np.linalg.norm(Cm - med[:, None, :], axis=2) <= tau_c
        Wm = np.where(keep, Wm, 0.0)
    acc = np.einsum("pv,pvk->pk", Wm, Cm)
    ws = Wm.sum(1)
    rgb = np.zeros((H, W, 3))
    wsum = np.zeros((H, W))
    good = ws >= w_min
    rgb[vv[good], uu[good]] = acc[good] / ws[good, None]
    wsum[vv, uu] = ws
    return rgb, wsum


def composite2d(mean, conic, alpha, feat, rect, order, H, W, alpha_max=0.99, alpha_min=1.0 / 255.0, t_eps=1e-4,
                cull_sigma=3.0):
    """a6 in float64 from 2D splat parameters (mean [n,2], conic (ca, cb2, cc) [n,3] with
    q = ca dx^2 + cb2 dx dy + cc dy^2, alpha, feat, pixel box rect [n,4]) composited in `order`
    (array indices, front to back).  Returns (F[H,W,C], A[H,W], set) where set[(py, px)] is the tuple
    of composited indices (to detect decision flips).  Used by the backward-pass pins."""
    order = np.asarray(order)
    m, cn, al, f, rc = mean[order], conic[order], alpha[order], feat[order], rect[order]
    C = f.shape[1]
    F = np.zeros((H, W, C))
    A = np.zeros((H, W))
    used = {}
    for py in range(H):
        for px in range(W):
            sel = np.nonzero((rc[:, 0] <= px) & (px <= rc[:, 1]) & (rc[:, 2] <= py) & (py <= rc[:, 3]))[0]
            if len(sel) == 0:
                continue
            dx = px - m[sel, 0]
            dy = py - m[sel, 1]
            q = cn[sel, 0] * dx * dx + cn[sel, 1] * dx * dy + cn[sel, 2] * dy * dy
            a = np.minimum(alpha_max, al[sel] * np.exp(-0.5 * q))
            use = (q <= cull_sigma ** 2) & (a >= alpha_min)
            sel, a = sel[use], a[use]
            if len(sel) == 0:
                continue
            Tn = np.cumprod(1.0 - a)
            stop = np.nonzero(Tn < t_eps)[0]
            k = stop[0] if len(stop) else len(a)
            Tb = np.concatenate([[1.0], Tn[:k]])
            F[py, px] = (a[:k] * Tb[:k]) @ f[sel[:k]]
            A[py, px] = 1.0 - Tb[k]
            used[(py, px)] = tuple(order[sel[:k]])
    return F, A, used
