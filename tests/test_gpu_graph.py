"""CUDA-Graph capture of the asynchronous per-frame chain (the system is "optimized
using CUDA Graphs"): ta_unproject + TA_FLAG_ASYNC ta_rasterize of several targets (and the fused front
end) captured once on a stream and replayed; every replay is bit-identical to the eager calls.  The
depth sort's look-back tag is a device counter advanced by k_init, so replays of the same launches do
not read the previous replay's words as current."""
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


def test_graph_replay_bit_identical_to_eager(ctx):
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("c3", res=256)
    cams = sg.make_targets("c4", res=256, n_targets=4)
    psync = P.gpu_params(s)
    pasync = P.gpu_params(s, flags=tb.TA_FLAG_ASYNC)
    views, keep = tb.views_to_device(s.views)
    g = tb.unproject(ctx, views, s.C, s.feat_dtype, psync)
    kc = 0
    arrs = [(sg.cam_arrays(c), c) for c in cams]
    for (K, R, t), c in arrs:
        tb.rasterize(ctx, g, K, R, t, c.H, c.W, psync)
        kc = max(kc, ctx.debug_last().Kc)
    ctx.reserve(g.capacity, int(kc * 1.2) + 4096, 256, 256)
    torch.cuda.synchronize()

    def frame(outs, stream):
        ctx.unproject(views, psync, g, stream)
        for ((K, R, t), c), (F, A) in zip(arrs, outs):
            ctx.rasterize(g, -1, tb.intrinsics(K), tb.extrinsics(R, t), c.H, c.W, pasync, F, A, stream)

    eager = [(torch.empty((256, 256, s.C), device="cuda"), torch.empty((256, 256), device="cuda")) for _ in cams]
    frame(eager, torch.cuda.current_stream())
    torch.cuda.synchronize()
    graph_out = [(torch.zeros((256, 256, s.C), device="cuda"), torch.zeros((256, 256), device="cuda")) for _ in cams]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):                   # warm-up on the capture stream
        frame(graph_out, side)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        frame(graph_out, torch.cuda.current_stream())
    for rep in range(3):
        for F, A in graph_out:
            F.zero_()
            A.zero_()
        graph.replay()
        torch.cuda.synchronize()
        for (F, A), (Fe, Ae) in zip(graph_out, eager):
            assert torch.equal(F.view(torch.int32), Fe.view(torch.int32)), rep
            assert torch.equal(A.view(torch.int32), Ae.view(torch.int32)), rep
    assert not ctx.check_overflow()


def test_graph_replay_fused_front_end(ctx):
    """The fused front end (ta_render_sources, both eyes of the paper variant, TA_FLAG_ASYNC) captured and
    replayed: bit-identical to its eager call."""
    import torch
    import paper_2405_14866_b200 as tb
    s = sg.make_config("paper", res=256)
    psync = P.gpu_params(s)
    pasync = P.gpu_params(s, flags=tb.TA_FLAG_ASYNC)
    views, keep = tb.views_to_device(s.views)
    Ks, RTs = [], []
    for c in s.targets:
        K, R, t = sg.cam_arrays(c)
        Ks.append(tb.intrinsics(K))
        RTs.append(tb.extrinsics(R, t))
    cf = tb.Context(0)

    def run(outs, p, stream):
        cf.render_sources(views, s.C, s.feat_dtype, p, Ks, RTs, 256, 256, [o[0] for o in outs], [o[1] for o in outs],
                          stream)

    eager = [(torch.empty((256, 256, s.C), device="cuda"), torch.empty((256, 256), device="cuda")) for _ in s.targets]
    run(eager, psync, torch.cuda.current_stream())           # sizes every scratch buffer
    torch.cuda.synchronize()
    out = [(torch.zeros((256, 256, s.C), device="cuda"), torch.zeros((256, 256), device="cuda")) for _ in s.targets]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        run(out, pasync, side)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        run(out, pasync, torch.cuda.current_stream())
    for rep in range(2):
        for F, A in out:
            F.zero_()
            A.zero_()
        graph.replay()
        torch.cuda.synchronize()
        for (F, A), (Fe, Ae) in zip(out, eager):
            assert torch.equal(F.view(torch.int32), Fe.view(torch.int32)), rep
            assert torch.equal(A.view(torch.int32), Ae.view(torch.int32)), rep


def test_output_guard_regions_untouched(ctx):
    """Out-of-bounds write check (compute-sanitizer is closed on this pool): F / A / z-buffer / blend /
    backward outputs are views into larger buffers whose guard bands hold a sentinel; after Tiny, a
    ragged reduced c2 (fp32 and fp16 features, sync / async, fused front end, tensor-memory compositor)
    every guard word is intact."""
    import os
    import torch
    import paper_2405_14866_b200 as tb
    os.environ["TA_COMPOSITOR"] = "2"
    try:
        ctx_tm = tb.Context(0)
    finally:
        os.environ.pop("TA_COMPOSITOR")
    SENT = -12345.5
    guard = 4096

    def guarded(shape):
        n = int(np.prod(shape))
        buf = torch.full((n + 2 * guard + 4,), SENT, device="cuda")
        off = guard + (-(guard) % 4)
        return buf, buf[off:off + n].view(*shape)

    def intact(buf, view):
        b = buf.cpu().numpy()
        off = view.storage_offset()
        n = view.numel()
        return np.all(b[:off] == SENT) and np.all(b[off + n:] == SENT)

    for name, kw, dt in (("tiny", {}, None), ("c2", {"res": 128, "target_hw": (97, 113)}, None),
                         ("rand", {}, "f32")):
        s = sg.make_random_scene(4, H=41, W=57, C=16, n_src=25, feat_dtype="f32") if name == "rand" else \
            sg.make_config(name, **kw)
        cam = s.targets[0]
        gp = P.gpu_params(s)
        g = P.gpu_unproject(ctx, s, gp)
        K, R, t = sg.cam_arrays(cam)
        bF, F = guarded((cam.H, cam.W, s.C))
        bA, A = guarded((cam.H, cam.W))
        for cx in (ctx, ctx_tm):
            cx.rasterize(g, -1, tb.intrinsics(K), tb.extrinsics(R, t), cam.H, cam.W, gp, F, A)
        views, keep = tb.views_to_device(s.views)
        ctx.render_sources(views, s.C, s.feat_dtype, gp, [tb.intrinsics(K)], [tb.extrinsics(R, t)], cam.H, cam.W,
                           [F], [A])
        ctx.rasterize(g, -1, tb.intrinsics(K), tb.extrinsics(R, t), cam.H, cam.W, gp, F, A)
        n = g.n
        bGF, GF = guarded((cam.H, cam.W, s.C))
        GF.normal_()
        GA = torch.randn((cam.H, cam.W), device="cuda")
        bdm, dm = guarded((n, 2))
        bdc, dc = guarded((n, 3))
        bda, da = guarded((n,))
        bdf, df = guarded((n, s.C))
        ctx.rasterize_backward(g, -1, cam.H, cam.W, gp, GF, GA, dm, dc, da, df)
        bz, zf = guarded((cam.H, cam.W))
        ctx.zbuffer(views, tb.default_params(), tb.intrinsics(K), tb.extrinsics(R, t), cam.H, cam.W, 1, 0.1, zf, None)
        torch.cuda.synchronize()
        for b, v in ((bF, F), (bA, A), (bdm, dm), (bdc, dc), (bda, da), (bdf, df), (bz, zf)):
            assert intact(b, v), name
