"""The opt-in fast-exp mode (ta_raster_params.exact_exp = 0, R13): the
compositor evaluates exp(-q/2) with the SFU (ex2.approx) instead of the fixed sequence exp_det.  Its
parity is reported separately (stop-index mismatches, A ulps, max |dF| against the exact oracle) next to
the compositor time of both modes; the default exact mode stays bit-exact (the other GPU tests)."""
import json
import os

import numpy as np
import pytest

import synthgen as sg
from tests import _parity as P

pytestmark = pytest.mark.gpu
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


@pytest.fixture(scope="module")
def ctx():
    import torch
    import paper_2405_14866_b200 as tb
    assert torch.cuda.is_available()
    tb.lib(build_if_stale=True)
    return tb.Context(0)


def _parity_numbers(out, F, A, nc, mask):
    diff_nc = out["n_contrib"][mask] != nc[mask]
    ga, oa = out["A"][mask], A[mask]
    ulps = np.abs(ga.view(np.int32).astype(np.int64) - oa.view(np.int32).astype(np.int64))
    return {"pixels": int(mask.sum()), "stop_index_mismatch_pixels": int(diff_nc.sum()),
            "stop_index_mismatch_frac": float(diff_nc.mean()), "A_max_ulp": int(ulps.max()),
            "A_median_ulp": float(np.median(ulps)), "A_max_abs": float(np.abs(ga - oa).max()),
            "F_max_abs": float(np.abs(out["F"][mask] - F[mask]).max())}


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_fast_exp_parity_reported(ctx, cfg):
    """c2 (every pixel) and c3 (72 sampled tiles incl. the 16 longest lists): the fast mode against the
    exact oracle.  Bounds: stop decisions differ on < 0.1 % of pixels, |dA| <= 1e-3, |dF| <= 5e-3 (a
    moved stop changes one Gaussian's weight alpha' T with T ~ t_eps); the numbers are written to
    gpurun_out/fast_exp_<cfg>.json."""
    import torch
    import oracle as O
    import paper_2405_14866_b200 as tb
    s = sg.make_config(cfg)
    cam = s.targets[0]
    gp = P.gpu_params(s, exact_exp=0)
    op = P.oracle_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    go = O.unproject(s, op)
    out = P.gpu_rasterize(ctx, g, cam, gp)
    K, R, t = sg.cam_arrays(cam)
    pr = O.project(go, K, R, t, cam.H, cam.W, op)
    P.check_lists_vs_oracle(out, O, pr, go["ids"], cam.H, cam.W)      # a2-a5 unaffected by the exp mode
    ranges, lst = O.tile_lists(pr, go["ids"], cam.H, cam.W)
    TX = (cam.W + 15) // 16
    tiles = None
    if cfg == "c3":
        lens = ranges[:, 1].astype(np.int64) - ranges[:, 0]
        rng = np.random.default_rng(5)
        tiles = np.unique(np.concatenate([np.argsort(lens)[-16:], rng.choice(np.nonzero(lens)[0], 56, replace=False)]))
    F, A, nc, _ = O.composite(go, pr, ranges, lst, cam.H, cam.W, op, tiles=tiles)
    mask = np.ones(A.shape, bool) if tiles is None else ~np.isnan(A)
    num = _parity_numbers(out, F, A, nc, mask)
    # compositor time of both modes (CUDA events around the stage, same call otherwise)
    times = {}
    for name, ee in (("exact", 1), ("fast", 0)):
        p = P.gpu_params(s, exact_exp=ee)
        Fg, Ag = tb.rasterize(ctx, g, K, R, t, cam.H, cam.W, p)
        ctx.profile(True)
        ctx.profile_read(reset=True)
        for _ in range(10):
            tb.rasterize(ctx, g, K, R, t, cam.H, cam.W, p, out=(Fg, Ag))
        prof = ctx.profile_read(reset=True)
        ctx.profile(False)
        times[name] = prof["composite"][0] / prof["composite"][1]
    num.update(config=cfg, composite_ms=times)
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"fast_exp_{cfg}.json"), "w") as f:
        json.dump(num, f, indent=1)
    print(json.dumps(num))
    assert num["stop_index_mismatch_frac"] < 1e-3, num
    assert num["A_max_abs"] <= 1e-3 and num["F_max_abs"] <= 5e-3, num


def test_exact_mode_is_default_and_bit_exact(ctx):
    """exact_exp = 1 is the default and reproduces the oracle's A bits; exact_exp outside {0, 1} is
    rejected."""
    import paper_2405_14866_b200 as tb
    assert tb.default_params().exact_exp == 1
    s = sg.make_config("c3", res=128, target_hw=(96, 112))
    gp = P.gpu_params(s)
    g = P.gpu_unproject(ctx, s, gp)
    bad = P.gpu_params(s, exact_exp=2)
    with pytest.raises(tb.TaError) as e:
        P.gpu_rasterize(ctx, g, s.targets[0], bad, debug=False)
    assert e.value.status == 1
