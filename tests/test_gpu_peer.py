"""Fused render + gather: every rank's compositor writes its views straight into the
display rank's frame buffer through a CUDA IPC mapping (paper_2405_14866_b200.dist.PeerFrame) -- on a
multi-GPU box those are peer stores over NVLink / NVSwitch.  This run has one GPU, so the two ranks
share it (no kernel waits on another rank: each rank only writes, the display rank reads after a host
barrier); the host logic, the handle exchange (gloo) and the addressing are exactly the multi-GPU ones.
The frame must equal single-process ta_rasterize calls bit for bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_views, results):
    import torch
    import torch.distributed as dist
    import synthgen as sg
    import paper_2405_14866_b200 as tb
    from paper_2405_14866_b200 import dist as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        s = sg.make_config("c4", res=192, target_hw=(160, 176), n_targets=n_views)
        ctx = tb.Context(0)
        p = tb.default_params(default_scale=s.default_scale, default_opacity=s.default_opacity)
        views, keep = tb.views_to_device(s.views)
        g = tb.unproject(ctx, views, s.C, s.feat_dtype, p)
        frame = tdist.PeerFrame(n_views, 160, 176, s.C, rank, world)
        mine = tdist.shard(n_views, rank, world)
        Ks, RTs, fp, ap = [], [], [], []
        for j in mine:
            K, R, t = sg.cam_arrays(s.targets[j])
            Ks.append(tb.intrinsics(K))
            RTs.append(tb.extrinsics(R, t))
            f, a = frame.view_ptrs(j)
            fp.append(f)
            ap.append(a)
        ctx.rasterize_views(g, -1, Ks, RTs, 160, 176, p, fp, ap, lanes=2)
        torch.cuda.synchronize()
        dist.barrier()                                  # every rank's stores have landed
        ok = True
        if rank == 0:
            for j in range(n_views):
                K, R, t = sg.cam_arrays(s.targets[j])
                F, A = tb.rasterize(ctx, g, K, R, t, 160, 176, p)
                torch.cuda.synchronize()
                ok = ok and torch.equal(F.view(torch.int32), frame.F[j].view(torch.int32)) and \
                    torch.equal(A.view(torch.int32), frame.A[j].view(torch.int32))
            ok = ok and float(frame.A.max()) > 0.5
        dist.barrier()                                  # mappings closed before the owner frees
        if rank != 0:
            frame.close()
        dist.barrier()
        if rank == 0:
            frame.close()
        results[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_views", [4, 5])
def test_render_into_display_rank_frame(n_views):
    import torch.multiprocessing as mp
    import torch
    assert torch.cuda.is_available()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), n_views, results), nprocs=2, join=True)
    assert results[0] and results[1]
