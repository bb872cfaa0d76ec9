"""Helpers for the GPU parity tests: run the CUDA path through the C ABI, run the oracle on the
same seeded inputs, and compare stage by stage (records, depth order, tile lists, F, A)."""
from __future__ import annotations

import ctypes
import glob
import os

import numpy as np

import synthgen as sg

_cudart = None


def cudart():
    global _cudart
    if _cudart is None:
        import torch  # noqa: F401  (initialises CUDA)
        import nvidia.cuda_runtime as ncr
        path = glob.glob(os.path.join(list(ncr.__path__)[0], "lib", "libcudart.so*"))[0]
        _cudart = ctypes.CDLL(path)
        _cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    return _cudart


def d2h(ptr, count, dtype):
    """Copy `count` elements of `dtype` from a raw device pointer to a numpy array."""
    out = np.empty(int(count), dtype=dtype)
    if count:
        rc = cudart().cudaMemcpy(out.ctypes.data, ptr, out.nbytes, 2)
        assert rc == 0, rc
    return out


def oracle_params(scene, **kw):
    import oracle
    return oracle.make_params(default_scale=scene.default_scale, default_opacity=scene.default_opacity, **kw)


def gpu_params(scene, flags=0, **kw):
    import paper_2405_14866_b200 as tb
    return tb.default_params(default_scale=scene.default_scale, default_opacity=scene.default_opacity, flags=flags,
                             **kw)


def gpu_unproject(ctx, scene, params):
    import torch
    import paper_2405_14866_b200 as tb
    views, keep = tb.views_to_device(scene.views)
    g = tb.unproject(ctx, views, scene.C, scene.feat_dtype, params)
    torch.cuda.synchronize()
    g._keep = keep
    return g


def gaussians_to_host(g):
    n = g.n
    return dict(n=n, pos_alpha=g.pos_alpha[:n].cpu().numpy(), cov=g.cov[:n].cpu().numpy(),
                feat=g.feat[:n].cpu().numpy())


def gpu_rasterize(ctx, g, cam, params, n=-1, debug=True, counts=True, same_f_bits=True):
    """Rasterize with `params` as given -- by default flags = 0, the compositor instantiation bench.py
    times -- and pull every stage's output back to the host.  With `counts`, the same call is
    repeated with TA_FLAG_DEBUG_COUNTS added (the counters instantiation): its F and A must be
    bit-identical to the timed call, and its per-pixel composited-pair counts are returned."""
    import ctypes
    import torch
    import paper_2405_14866_b200 as tb
    K, R, t = sg.cam_arrays(cam)
    F, A = tb.rasterize(ctx, g, K, R, t, cam.H, cam.W, params, n=n)
    torch.cuda.synchronize()
    out = dict(F=F.cpu().numpy(), A=A.cpu().numpy())
    if not debug:
        return out
    d = ctx.debug_last()
    T = d.tiles_x * d.tiles_y
    out.update(n=d.n, K=d.K, P=d.P, tiles_x=d.tiles_x, tiles_y=d.tiles_y, sort_passes=d.sort_passes,
               tile_px=d.tile_px)
    out["records"] = d2h(d.records, 8 * d.n, np.uint32).reshape(-1, 8)
    out["order"] = d2h(d.order, d.n, np.uint32)
    out["keys_sorted"] = d2h(d.depth_keys, d.n, np.uint32)
    offs = d2h(d.tile_offsets, T + 1, np.uint32)
    out["ranges"] = np.stack([offs[:T], offs[1:T + 1]], axis=1)
    out["Kc"] = d.Kc
    out["list"] = d2h(d.tile_list, d.K, np.uint32)
    if d.n_contrib:
        out["n_contrib"] = d2h(d.n_contrib, cam.H * cam.W, np.int32).reshape(cam.H, cam.W)
    elif counts:
        pc = tb.default_params()
        ctypes.memmove(ctypes.byref(pc), ctypes.byref(params), ctypes.sizeof(pc))
        pc.flags = params.flags | tb.TA_FLAG_DEBUG_COUNTS
        F2, A2 = tb.rasterize(ctx, g, K, R, t, cam.H, cam.W, pc, n=n)
        torch.cuda.synchronize()
        if same_f_bits:   # (the warp-specialized variants group their fp32 MMA sums by timing: A only)
            assert torch.equal(F2.view(torch.int32), F.view(torch.int32)), "counters instantiation changed F"
        assert torch.equal(A2.view(torch.int32), A.view(torch.int32)), "counters instantiation changed A"
        d2 = ctx.debug_last()
        out["n_contrib"] = d2h(d2.n_contrib, cam.H * cam.W, np.int32).reshape(cam.H, cam.W)
        out["work"] = list(d2.work)
    return out


def oracle_gaussians_from_gpu(gh):
    """The GPU's Gaussian set in the oracle's dict layout (for a2-a6 parity on identical inputs)."""
    cov = gh["cov"]
    return dict(pos=np.ascontiguousarray(gh["pos_alpha"][:, :3]), alpha=np.ascontiguousarray(gh["pos_alpha"][:, 3]),
                cov6=np.ascontiguousarray(cov[:, :6]), ids=cov[:, 6].view(np.uint32).astype(np.int64),
                feat=np.ascontiguousarray(gh["feat"]), n=gh["n"])


def check_unproject(gh, go):
    """a1 parity: bit-exact positions, opacity, covariance, ids, features."""
    assert gh["n"] == go["n"]
    assert np.array_equal(gh["pos_alpha"][:, :3].view(np.uint32), go["pos"].view(np.uint32))
    assert np.array_equal(gh["pos_alpha"][:, 3].view(np.uint32), go["alpha"].view(np.uint32))
    assert np.array_equal(gh["cov"][:, :6].view(np.uint32), go["cov6"].view(np.uint32))
    assert np.array_equal(gh["cov"][:, 6].view(np.uint32).astype(np.int64), go["ids"])
    assert np.array_equal(gh["feat"].view(np.uint8), go["feat"].view(np.uint8))


def check_project(out, pr, alpha):
    """a2 parity: bit-exact splat records (mean, conic, alpha, pixel box) and visibility."""
    rec = out["records"]
    vis = pr["visible"].astype(bool)
    rx, ry = rec[:, 6], rec[:, 7]
    gvis = (rx & 0xffff) <= (rx >> 16)
    assert np.array_equal(gvis, vis)
    r = pr["rect"][vis]
    assert np.array_equal(rx[vis], (r[:, 0] | (r[:, 1] << 16)).astype(np.uint32))
    assert np.array_equal(ry[vis], (r[:, 2] | (r[:, 3] << 16)).astype(np.uint32))
    assert np.array_equal(rec[vis, 0:2], pr["mean2"][vis].view(np.uint32))
    assert np.array_equal(rec[vis, 2:4], pr["conic"][vis, 0:2].view(np.uint32))
    assert np.array_equal(rec[vis, 4], pr["conic"][vis, 2].view(np.uint32))
    assert np.array_equal(rec[:, 5], np.asarray(alpha, np.float32).view(np.uint32))


def check_order(out, pr, ids):
    """a4 parity: visible Gaussians in the GPU's depth-rank order == oracle (dkey, id) order."""
    vis = pr["visible"].astype(bool)
    order = out["order"].astype(np.int64)
    got = order[vis[order]]
    idx = np.nonzero(vis)[0]
    want = idx[np.lexsort((ids[idx], pr["dkey"][idx]))]
    assert np.array_equal(got, want)


def check_lists_vs_oracle(out, O, pr, ids, H, W):
    """a3/a5 parity at the GPU's compositing tile size (ta_debug_view.tile_px: 8 under 32-px coarse
    bins, 16 otherwise): the oracle's (tile, dkey, id) lists for that tile side, bit-exact."""
    assert out["tile_px"] in (8, 16)
    check_lists(out, *O.tile_lists(pr, ids, H, W, tile=out["tile_px"]))


def check_lists(out, ranges, lst):
    """a3/a5 parity: tile ranges and per-tile lists bit-exact."""
    assert len(out["ranges"]) == len(ranges), "tile counts differ (tile side)"
    assert out["K"] == len(lst)
    g = out["ranges"].astype(np.int64)
    o = ranges.astype(np.int64)
    glen, olen = g[:, 1] - g[:, 0], o[:, 1] - o[:, 0]
    assert np.array_equal(glen, olen)
    ne = olen > 0                     # empty tiles: the oracle reports (0, 0), the GPU (start, start)
    assert np.array_equal(g[ne], o[ne])
    assert np.array_equal(out["list"].astype(np.int64), lst)


def check_composite(out, F, A, nc=None, tiles=None, tx=None, atol=1e-4):
    """a6 parity: A and composited-pair counts bit-exact, F within atol (fp32 accumulate)."""
    if tiles is not None:
        m = np.zeros(A.shape, bool)
        for t in tiles:
            y, x = divmod(int(t), tx)
            m[y * 16:(y + 1) * 16, x * 16:(x + 1) * 16] = True
    else:
        m = np.ones(A.shape, bool)
    assert np.array_equal(out["A"][m].view(np.uint32), A[m].view(np.uint32)), \
        f"A mismatch at {np.count_nonzero(out['A'][m] != A[m])} pixels"
    err = np.abs(out["F"][m] - F[m]).max() if m.any() else 0.0
    assert err <= atol, err
    if nc is not None and "n_contrib" in out:
        assert np.array_equal(out["n_contrib"][m], nc[m])
    return float(err)
