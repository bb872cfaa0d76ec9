"""Small end-to-end case for compute-sanitizer (memcheck / racecheck / synccheck; one tool per run):
Tiny and a reduced c2 through ta_unproject + ta_rasterize (fp32 SIMT and fp16 mma.sync compositors,
sync and TA_FLAG_ASYNC), the fused front end, the tensor-memory compositor, z-buffer and blending,
and the backward pass.  Exits 0 when every call succeeded (dev tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import synthgen as sg
    import paper_2405_14866_b200 as tb
    from tests import _parity as P
    ctx = tb.Context(0)
    os.environ["TA_COMPOSITOR"] = "2"
    ctx_tm = tb.Context(0)
    os.environ.pop("TA_COMPOSITOR")
    for name, kw in (("tiny", {}), ("c2", {"res": 128, "target_hw": (96, 112)})):
        s = sg.make_config(name, **kw)
        gp = P.gpu_params(s)
        g = P.gpu_unproject(ctx, s, gp)
        cam = s.targets[0]
        for cx in (ctx, ctx_tm):
            P.gpu_rasterize(cx, g, cam, gp)
        K, R, t = sg.cam_arrays(cam)
        ctx.reserve(g.capacity, ctx.debug_last().Kc + 1024, cam.H, cam.W)
        tb.rasterize(ctx, g, K, R, t, cam.H, cam.W, P.gpu_params(s, flags=tb.TA_FLAG_ASYNC))
        views, keep = tb.views_to_device(s.views)
        F = torch.empty((cam.H, cam.W, s.C), device="cuda")
        A = torch.empty((cam.H, cam.W), device="cuda")
        ctx.render_sources(views, s.C, s.feat_dtype, gp, [tb.intrinsics(K)], [tb.extrinsics(R, t)], cam.H, cam.W, [F], [A])
        # backward of the last forward on ctx
        tb.rasterize(ctx, g, K, R, t, cam.H, cam.W, gp)
        n = g.n
        GF = torch.randn((cam.H, cam.W, s.C), device="cuda")
        GA = torch.randn((cam.H, cam.W), device="cuda")
        dm, dc = torch.empty((n, 2), device="cuda"), torch.empty((n, 3), device="cuda")
        da, df = torch.empty((n,), device="cuda"), torch.empty((n, s.C), device="cuda")
        ctx.rasterize_backward(g, -1, cam.H, cam.W, gp, GF, GA, dm, dc, da, df)
        zf = torch.empty((cam.H, cam.W), device="cuda")
        ctx.zbuffer(views, tb.default_params(), tb.intrinsics(K), tb.extrinsics(R, t), cam.H, cam.W, 1, 0.1, zf, None)
        if name == "c2":
            cols = [torch.rand((v.cam.H, v.cam.W, 3), device="cuda") for v in s.views]
            rgb = torch.empty((cam.H, cam.W, 3), device="cuda")
            ctx.blend(views, cols, tb.default_params(), tb.default_blend_params(), tb.intrinsics(K),
                      tb.extrinsics(R, t), cam.H, cam.W, zf, rgb, None)
        torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
