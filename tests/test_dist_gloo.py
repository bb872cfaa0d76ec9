"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: view sharding, Gaussian-set
broadcast, gather of rendered views to the display rank, max-over-ranks timing."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_14866_b200 import dist as tdist


def test_shard_covers_every_view_once():
    for n in (1, 7, 8, 32):
        for world in (1, 2, 3, 4, 8):
            got = [i for r in range(world) for i in tdist.shard(n, r, world)]
            assert got == list(range(n))
            sizes = [len(tdist.shard(n, r, world)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cap, C = 100, 8
        g = torch.Generator().manual_seed(0)
        pos = torch.randn(cap, 4, generator=g)
        cov = torch.randn(cap, 8, generator=g)
        feat = torch.randn(cap, C, generator=g).to(torch.float16)
        if rank == 0:
            n_dev = torch.tensor([37], dtype=torch.int64)
            mine = (pos.clone(), cov.clone(), feat.clone())
        else:
            n_dev = torch.zeros(1, dtype=torch.int64)
            mine = (torch.zeros_like(pos), torch.zeros_like(cov), torch.zeros_like(feat))
        n = tdist.broadcast_gaussians(mine, n_dev)
        ok_bcast = n == 37 and all(torch.equal(a[:n], b[:n]) for a, b in zip(mine, (pos, cov, feat)))
        ok_tail = rank == 0 or all(torch.count_nonzero(a[n:]) == 0 for a in mine)
        # every rank "renders" its shard of 5 views; the display rank gathers them in view order
        n_views = 5
        local = [torch.full((3, 4), float(j)) for j in tdist.shard(n_views, rank, world)]
        out = tdist.gather_views(local, n_views, rank, world)
        ok_gather = True
        if rank == 0:
            ok_gather = len(out) == n_views and all(torch.equal(v, torch.full((3, 4), float(j)))
                                                     for j, v in enumerate(out))
        ms = tdist.reduce_scalar(10.0 + rank, "max")
        tot = tdist.reduce_scalar(1.0, "sum")
        results[rank] = (ok_bcast, ok_tail, ok_gather, ms, tot)
    finally:
        dist.destroy_process_group()


def test_two_rank_broadcast_gather_and_timing():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    for r in range(world):
        ok_bcast, ok_tail, ok_gather, ms, tot = results[r]
        assert ok_bcast and ok_tail and ok_gather
        assert ms == 11.0 and tot == 2.0
