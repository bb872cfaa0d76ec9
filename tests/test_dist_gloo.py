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
        # host-bound broadcast (no read-back of n): rows = an upper bound, n travels in n_dev
        mine2 = (pos.clone(), cov.clone(), feat.clone()) if rank == 0 else tuple(torch.zeros_like(a) for a in mine)
        n_dev2 = torch.tensor([37], dtype=torch.int64) if rank == 0 else torch.zeros(1, dtype=torch.int64)
        r2 = tdist.broadcast_gaussians(mine2, n_dev2, rows=40)
        ok_bcast = ok_bcast and r2 is None and int(n_dev2[0]) == 37 and all(
            torch.equal(a[:40], b[:40]) for a, b in zip(mine2, (pos, cov, feat)))
        # every rank "renders" its shard of the views; the display rank gathers them in view order
        # (5 views: per-rank counts differ -> send/recv; 4 views: equal shards -> collective gather)
        ok_gather = True
        for n_views in (5, 4):
            local = [torch.full((3, 4), float(j)) for j in tdist.shard(n_views, rank, world)]
            out = tdist.gather_views(local, n_views, rank, world)
            if rank == 0:
                ok_gather = ok_gather and len(out) == n_views and all(
                    torch.equal(v, torch.full((3, 4), float(j))) for j, v in enumerate(out))
            else:
                ok_gather = ok_gather and out is None
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


def _run_bench_dry(gpus, views):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(gpus), "--dry-run-dist",
                        "--views", str(views)], capture_output=True, text=True, env=env, timeout=240, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("views", [6, 5])
def test_bench_relaunches_itself_with_n_ranks(views):
    """`python bench.py --gpus 2` without a torchrun environment relaunches itself as 2 ranks
    (torch.distributed.run, 127.0.0.1); in the CPU dry run (gloo) rank 0 prints one line with
    n_gpus = 2, and every view gathered from the ranks equals the single-process rendering of that
    view index (equal shards: collective gather; 5 views: send/recv)."""
    d = _run_bench_dry(2, views)
    assert d["n_gpus"] == 2 and d["views"] == views
    assert d["views_equal"] and d["gaussians_equal"] and d["n_broadcast"] == 7


def test_bench_relaunch_command():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert b.relaunch_command(1, [], {}) is None
    assert b.relaunch_command(4, ["--gpus", "4"], {"WORLD_SIZE": "4"}) is None
    cmd = b.relaunch_command(4, ["--gpus", "4", "--steps", "3"], {})
    assert "torch.distributed.run" in cmd and "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]
