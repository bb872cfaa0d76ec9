#!/usr/bin/env python
"""bench.py -- target views/s of the latent-Gaussian rasterizer on B200 (BASELINE.json metric).

Step (one pass of the whole hot path) = one frame of the c4 workload
(BASELINE.json configs[3]): ta_unproject of the 4 x 1024^2 source views (1.67M Gaussians, C = 32,
fp16-stored features) on rank 0, NCCL broadcast of the Gaussian set when N > 1, then
ta_rasterize of this rank's share of the 32 parallax targets (1024^2, HWC fp32 + alpha).
`value` = 32 views x steps / max-over-ranks device time (strong scaling: 32 views per frame
regardless of N).  Inputs are resident in HBM before the timed region and larger than L2
(423 MB of source maps, 187 MB Gaussian set, 16.9M tile entries per view).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun each rank drives one GPU; rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "target views/sec and ms/view, 1024² 32-ch features, 1/2/4/8 B200; HBM roofline %"
HBM_FALLBACK_GBS = 6650.0
SM_CLOCK_MAX_MHZ = 1965.0
FP32_LANES_PER_SM = 128          # B200: 4 SMSPs x 32 FP32 lanes (B200_PROFILING.md / guide unit counts)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": HBM_FALLBACK_GBS, "sm_max_mhz": SM_CLOCK_MAX_MHZ}, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.proc = None
        self.dev = device_index

    def start(self):
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.dev).uuid)
            sel = ["--id=" + (uuid if uuid.startswith("GPU-") else "GPU-" + uuid)]
        except Exception:
            sel = ["-i", str(self.dev)]
        try:
            self.proc = subprocess.Popen(["nvidia-smi", *sel, "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle (CPU) leg
def oracle_crop_view(scene_g, cam, crop=256):
    """One bounded sample of the per-view work on the CPU oracle: the central crop x crop window of a
    1024^2 target (1/16 of its pixels) -- project all Gaussians, build the window's tile lists,
    composite every window pixel.  Returns seconds."""
    import oracle
    import synthgen as sg
    x0 = (cam.W - crop) // 2
    y0 = (cam.H - crop) // 2
    cc = sg.crop_camera(cam, x0, y0, crop, crop)
    t0 = time.perf_counter()
    oracle.rasterize(scene_g, cc)
    return time.perf_counter() - t0


def cpu_baseline_value(g, cam, steps=1, crop=256):
    ts = [oracle_crop_view(g, cam, crop) for _ in range(steps)]
    frac = (crop * crop) / float(cam.W * cam.H)
    t = statistics.mean(ts)
    return 1.0 / (t / frac), t, frac


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import synthgen as sg
    import oracle
    s = sg.make_config("c3")
    g = oracle.unproject(s)
    cam = sg.make_targets("c4")[0]
    for _ in range(args.warmup):
        oracle_crop_view(g, cam)
    ts = [oracle_crop_view(g, cam) for _ in range(args.steps)]
    frac = 256 * 256 / float(cam.W * cam.H)
    t = statistics.mean(ts)
    value = frac / t
    sample = ("oracle/taoracle.c single-threaded: per step the central 256x256 window (1/16 of the pixels) of a "
              "c4 1024^2 target -- EWA projection of all 1.67M Gaussians, (tile, depth, id) lists of the window, "
              "compositing of its 65,536 pixels; value = (1/16) / step seconds; unprojection (per frame, "
              "<1% of the oracle's per-view time) excluded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "ms_per_view": t * 1e3 / frac,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": workload_config(None, None),
            "cpu_baseline": {"value": value, "unit": "views/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(n, K):
    return {"workload": "c4: BASELINE.json configs[3] -- c3 Gaussian set (4 x 1024^2 sources, C=32 fp16-stored) "
                        "rendered to 32 parallax targets 1024^2 per frame",
            "views_per_step": 32, "target": "1024x1024", "C": 32, "feat_storage": "f16", "sources": "4x1024x1024",
            "n_gaussians": n, "entries_per_view": K,
            "l2": "no flush: inputs larger than L2 (423 MB source maps, 187 MB Gaussian set, "
                  "~68 MB tile lists + 138 MB output per view)",
            "parallelism": "target views sharded over ranks; Gaussian set NCCL-broadcast from rank 0"}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synthgen as sg
    import paper_2405_14866_b200 as tb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    n_views = args.views
    targets = sg.make_targets("c4", n_targets=n_views)
    from paper_2405_14866_b200 import dist as tdist
    mine = tdist.shard(n_views, rank, world)
    ctx = tb.Context(local)
    # views alternate over `streams` (context, CUDA stream) pairs so one view's projection / sort /
    # binning overlaps the previous view's compositing tail (one context per stream: its own scratch)
    nstr = max(1, args.streams)
    ctxs = [ctx] + [tb.Context(local) for _ in range(nstr - 1)]
    side = [torch.cuda.Stream() for _ in range(nstr)]
    C_, H, W = 32, 1024, 1024
    cap = 4 * 1024 * 1024
    g = tb.GaussianBuffers(cap, C_, "f16", device=dev)
    params_sync = tb.default_params()
    params = tb.default_params(flags=tb.TA_FLAG_ASYNC)

    scene = None
    views = keep = None
    if rank == 0:
        scene = sg.make_config("c3")
        views, keep = tb.views_to_device(scene.views, device=dev)
    cams = []
    for j in mine:
        K, R, t = sg.cam_arrays(targets[j])
        cams.append((tb.intrinsics(K), tb.extrinsics(R, t)))
    outs = [(torch.empty((H, W, C_), dtype=torch.float32, device=dev),
             torch.empty((H, W), dtype=torch.float32, device=dev)) for _ in mine]

    def broadcast(gb=None):
        gb = gb if gb is not None else g
        if world > 1:
            tdist.broadcast_gaussians((gb.pos_alpha, gb.cov, gb.feat), gb.n_dev, src=0)

    def step(p):
        if rank == 0:
            ctx.unproject(views, params_sync, g, stream)
        broadcast()
        if nstr == 1:
            for (Ki, Ri), (F, A) in zip(cams, outs):
                ctx.rasterize(g, -1, Ki, Ri, H, W, p, F, A, stream)
            return
        ready = torch.cuda.Event()
        ready.record(stream)
        for sd in side:
            sd.wait_event(ready)
        for k, ((Ki, Ri), (F, A)) in enumerate(zip(cams, outs)):
            ctxs[k % nstr].rasterize(g, -1, Ki, Ri, H, W, p, F, A, side[k % nstr])
        for sd in side:
            done = torch.cuda.Event()
            done.record(sd)
            stream.wait_event(done)

    # Steady-state frame pipeline: two Gaussian sets; while the views of frame f render
    # from one set, the next frame is lifted (rank 0) and NCCL-broadcast into the other set on a
    # separate stream, so the broadcast overlaps rendering.  Every step still lifts + broadcasts one
    # frame and renders one frame.
    gsets = [g, tb.GaussianBuffers(cap, C_, "f16", device=dev)]
    prep = torch.cuda.Stream()
    ctx_prep = tb.Context(local)
    pipe = {"k": 0, "ready": None, "free": [None, None]}

    def prepare(buf_i):
        gb = gsets[buf_i]
        with torch.cuda.stream(prep):
            if pipe["free"][buf_i] is not None:
                prep.wait_event(pipe["free"][buf_i])   # the renders that read this set are done
            if rank == 0:
                ctx_prep.unproject(views, params_sync, gb, prep)
            broadcast(gb)
            ev = torch.cuda.Event()
            ev.record(prep)
        return ev

    def step_pipelined(p):
        cur = pipe["k"] % 2
        if pipe["ready"] is None:
            pipe["ready"] = prepare(cur)
        for sd in side:
            sd.wait_event(pipe["ready"])
        gb = gsets[cur]
        for k, ((Ki, Ri), (F, A)) in enumerate(zip(cams, outs)):
            ctxs[k % nstr].rasterize(gb, -1, Ki, Ri, H, W, p, F, A, side[k % nstr])
        free = torch.cuda.Event()
        for sd in side:
            done = torch.cuda.Event()
            done.record(sd)
            stream.wait_event(done)
        free.record(stream)
        pipe["free"][cur] = free
        pipe["k"] += 1
        pipe["ready"] = prepare(pipe["k"] % 2)          # next frame's set, overlapping these renders

    # sizing pass (synchronous): learn K per view, reserve for async steps
    step(params_sync)
    torch.cuda.synchronize()
    kmax = kcmax = 0
    for (Ki, Ri), (F, A) in zip(cams, outs):
        ctx.rasterize(g, -1, Ki, Ri, H, W, params_sync, F, A, stream)
        d = ctx.debug_last()
        kmax, kcmax = max(kmax, d.K), max(kcmax, d.Kc)
    n_g = g.n
    for cx in ctxs:
        cx.reserve(cap, int(kcmax * 1.05) + 4096, H, W)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        return tdist.reduce_scalar(x, "max", device=dev)

    def sum_over_ranks(x):
        return tdist.reduce_scalar(x, "sum", device=dev)

    timed_step = step_pipelined if nstr > 1 else step
    for _ in range(args.warmup):
        timed_step(params)
    torch.cuda.synchronize()
    barrier()
    assert not any(cx.check_overflow() for cx in ctxs), "reserved tile-entry capacity overflowed"

    # ---------------- timed region (device time, CUDA events on the launching stream)
    if not args.no_stage_events and nstr == 1:
        ctx.profile(True)
        ctx.profile_read(reset=True)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = sum(cx.launches for cx in ctxs) + ctx_prep.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    marks = []                                        # step boundaries on the main stream (per-step spread)
    for _ in range(args.steps):
        timed_step(params)
        marks.append(torch.cuda.Event(enable_timing=True))
        marks[-1].record(stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_local = ev0.elapsed_time(ev1)
    step_ms = sorted([ev0.elapsed_time(marks[0])] + [a.elapsed_time(b) for a, b in zip(marks, marks[1:])])
    clk = clocks.stop()
    launches = int(sum_over_ranks(sum(cx.launches for cx in ctxs) + ctx_prep.launches - launches0))
    ms = max_over_ranks(ms_local)
    prof = None
    stage_timing = "stage events of context 0 inside the timed region (single stream)"
    if not args.no_stage_events:
        if nstr == 1:
            prof = ctx.profile_read(reset=True)
        else:
            # With several streams the kernels of different views overlap, so a stage's event pair
            # brackets other views' work too.  Per-kernel launch durations are therefore taken from
            # a serialized replay of the same K steps on one stream (CUDA events on that stream).
            ctx.profile(True)
            ctx.profile_read(reset=True)
            torch.cuda.synchronize()
            for _ in range(args.steps):
                if rank == 0:
                    ctx.unproject(views, params_sync, g, stream)
                broadcast()
                for (Ki, Ri), (F, A) in zip(cams, outs):
                    ctx.rasterize(g, -1, Ki, Ri, H, W, params, F, A, stream)
            torch.cuda.synchronize()
            prof = ctx.profile_read(reset=True)
            stage_timing = ("stage events over a single-stream replay of the K timed steps (the timed multi-stream "
                            "step overlaps kernels of different views, so per-kernel durations are not defined there)")
    ctx.profile(False)
    overflow = any(cx.check_overflow() for cx in ctxs)
    value = n_views * args.steps / (ms / 1e3)

    line = {"metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "ms_per_view": ms / (args.steps * n_views),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded synthgen rig: ellipsoid upper body, log-normal scales, random rotations)",
            "config": dict(workload_config(n_g, kmax), streams=nstr), "gpu_launches": launches, "clocks": clk,
            "overflow": overflow,
            "step_ms_rank0": {"median": step_ms[len(step_ms) // 2], "min": step_ms[0],
                              "p90": step_ms[min(len(step_ms) - 1, int(0.9 * len(step_ms)))],
                              "note": "device time between consecutive step boundaries on rank 0's main stream "
                                      "(frames are pipelined, so a step boundary is where its renders end)"}}

    # ---------------- roofline of the dominant kernel (rank 0's live stage events)
    if prof is not None and rank == 0:
        stages = {k: (v[0] / v[1] if v[1] else 0.0) for k, v in prof.items()}
        line["stages_ms_per_call"] = {k: round(v, 4) for k, v in stages.items()}
        line["stages_timing"] = stage_timing
        share = {k: v[0] for k, v in prof.items()}
        tot = sum(share.values())
        line["stages_share"] = {k: round(v / tot, 4) for k, v in share.items()} if tot else {}
        line["roofline"] = roofline(ctx, g, cams[0], outs[0], H, W, C_, stages, n_g, stream,
                                    ms_per_view=ms / (args.steps * n_views))

    # ---------------- end to end through the C ABI with host buffers
    if not args.no_e2e:
        line["e2e"] = e2e(args, ctx, g, views, keep, scene, cams, outs, H, W, C_, rank, world, stream,
                          broadcast, max_over_ranks, sum_over_ranks, params, params_sync)

    # ---------------- CPU oracle baseline (rank 0, N = 1 only)
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        import oracle
        go = oracle.unproject(scene)
        v, t, frac = cpu_baseline_value(go, targets[0])
        line["cpu_baseline"] = {"value": v, "unit": "views/s", "cores": 1, "kind": "oracle",
                                "sample": f"oracle/taoracle.c single-threaded on the central 256x256 window "
                                          f"({frac:.4f} of the pixels) of c4 target 0: projection of all Gaussians + "
                                          f"window tile lists + compositing, {t:.2f} s; value = fraction / seconds"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def roofline(ctx, g, cam0, out0, H, W, C_, stages, n_g, stream, ms_per_view=None):
    """Algorithmic bytes / flops per launch over the live
    per-launch time of each stage; the dominant stage is reported."""
    import numpy as np
    import torch
    import paper_2405_14866_b200 as tb
    from tests import _parity as P   # d2h helper only (no oracle use)
    Ki, Ri = cam0
    F, A = out0
    pc = tb.default_params(flags=tb.TA_FLAG_DEBUG_COUNTS)
    ctx.rasterize(g, -1, Ki, Ri, H, W, pc, F, A, stream)
    torch.cuda.synchronize()
    d = ctx.debug_last()
    rec = P.d2h(d.records, 8 * d.n, np.uint32).reshape(-1, 8)
    nvis = int(np.count_nonzero((rec[:, 6] & 0xffff) <= (rec[:, 6] >> 16)))
    pairs = int(P.d2h(d.n_contrib, H * W, np.int32).astype(np.int64).sum())
    K = int(d.K)
    Kc = int(d.Kc)
    NB = ((W + 31) // 32) * ((H + 31) // 32)
    peaks, src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", HBM_FALLBACK_GBS))
    mhz = float(peaks.get("sm_max_mhz", SM_CLOCK_MAX_MHZ))
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    fp32_tflops = sms * FP32_LANES_PER_SM * 2 * mhz * 1e6 / 1e12
    fb = 2 * C_
    bytes_alg = {
        "project": n_g * (48 + 32 + 8),
        "sort": 16 * n_g * max(1, d.sort_passes),
        "bin_count": 12 * nvis + 4 * NB * d.P,
        "bin_scan": 8 * NB * d.P,
        "bin_place": 12 * nvis + 4 * Kc + 4 * NB * d.P,
        "composite": 4 * Kc + nvis * (32 + fb) + 4 * H * W * (C_ + 1),
    }
    flops_comp = pairs * (2 * C_ + 12)
    dom = max((k for k in bytes_alg), key=lambda k: stages.get(k, 0.0))
    t = stages[dom] / 1e3
    if dom == "composite":
        hb = bytes_alg[dom] / t / 1e9
        fl = flops_comp / t / 1e12
        if fl / fp32_tflops >= hb / hbm:
            r = {"bound": "alu", "achieved": fl, "peak": fp32_tflops, "unit": "TFLOP/s", "frac": fl / fp32_tflops,
                 "peak_source": f"derived: {sms} SMs x {FP32_LANES_PER_SM} FP32 lanes x 2 x {mhz:.0f} MHz",
                 "hbm_frac": hb / hbm}
        else:
            r = {"bound": "hbm", "achieved": hb, "peak": hbm, "unit": "GB/s", "frac": hb / hbm,
                 "peak_source": src, "alu_frac": fl / fp32_tflops}
    else:
        hb = bytes_alg[dom] / t / 1e9
        r = {"bound": "hbm", "achieved": hb, "peak": hbm, "unit": "GB/s", "frac": hb / hbm, "peak_source": src}
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        kname = {"project": "k_project", "bin_count": "k_bin_count", "bin_place": "k_bin_place",
                 "composite": "k_composite_tc", "sort": "k_sort_pass"}.get(dom)
        if kname in tj:
            traffic = tj[kname]["dram_bytes"]
            r["traffic_source"] = "profiles/traffic.json <- " + tj[kname]["source"] + " (ncu --set full, one launch)"
    except Exception:
        pass
    r.update({"kernel": dom, "traffic": traffic, "ms_per_launch": stages[dom],
              "algorithmic_bytes_per_launch": bytes_alg[dom], "composited_pairs_per_view": pairs,
              "visible_gaussians": nvis, "entries_per_view": K, "coarse_entries_per_view": Kc})
    # whole-view roofline: all per-view algorithmic bytes vs the summed per-view stage time
    view_ms = ms_per_view if ms_per_view else sum(v for k, v in stages.items() if k != "unproject")
    b_view = n_g * 48 + nvis * fb + 16 * K + 4 * H * W * (C_ + 1)
    r["view"] = {"ms": view_ms, "alg_bytes": b_view, "hbm_frac": b_view / (view_ms / 1e3) / 1e9 / hbm,
                 "fp32_frac": flops_comp / (view_ms / 1e3) / 1e12 / fp32_tflops}
    return r


def e2e(args, ctx, g, views, keep, scene, cams, outs, H, W, C_, rank, world, stream, broadcast, max_over_ranks,
        sum_over_ranks, params, params_sync):
    """Same metric through the public API with HOST buffers: per step the source maps are copied
    H2D from pinned memory and every rendered view (F + A) is copied D2H into pinned memory."""
    import torch
    h2d = 0
    host_in = []
    if rank == 0:
        for dev_tensors in keep:
            for t in dev_tensors:
                if t is not None:
                    host_in.append((t.cpu().pin_memory(), t))
                    h2d += t.numel() * t.element_size()
    nbuf = 4
    host_out = [(torch.empty((H, W, C_), dtype=torch.float32).pin_memory(),
                 torch.empty((H, W), dtype=torch.float32).pin_memory()) for _ in range(nbuf)]
    d2h = len(cams) * (H * W * C_ * 4 + H * W * 4)
    copy = torch.cuda.Stream()        # D2H of the rendered views
    upload = torch.cuda.Stream()      # H2D of the next frame's source maps (PCIe is full duplex)
    rendered = [torch.cuda.Event() for _ in cams]
    copied = [torch.cuda.Event() for _ in cams]
    lifted = {"ev": None}

    def step():
        # inputs: H2D from pinned memory on the upload stream (once the previous frame's ta_unproject
        # has read the device copies), consumed by ta_unproject on the compute stream
        if host_in:
            if lifted["ev"] is not None:
                upload.wait_event(lifted["ev"])
            with torch.cuda.stream(upload):
                for h, d in host_in:
                    d.copy_(h, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(upload)
            stream.wait_event(ev)
        if rank == 0:
            ctx.unproject(views, params_sync, g, stream)
            lifted["ev"] = torch.cuda.Event()
            lifted["ev"].record(stream)
        broadcast()
        for k, ((Ki, Ri), (F, A)) in enumerate(zip(cams, outs)):
            stream.wait_event(copied[k])               # previous step's D2H of this buffer is done
            ctx.rasterize(g, -1, Ki, Ri, H, W, params, F, A, stream)
            rendered[k].record(stream)
            copy.wait_event(rendered[k])               # D2H of view k overlaps rendering of view k+1
            with torch.cuda.stream(copy):
                hf, ha = host_out[k % nbuf]
                hf.copy_(F, non_blocking=True)
                ha.copy_(A, non_blocking=True)
            copied[k].record(copy)

    steps = max(2, min(args.steps, 5))
    step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        step()
    done = torch.cuda.Event()
    done.record(copy)
    stream.wait_event(done)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    total_views = int(sum_over_ranks(len(cams)))
    return {"value": total_views * steps / (ms / 1e3),
            "unit": "views/s", "h2d_bytes_per_step": int(sum_over_ranks(h2d)),
            "d2h_bytes_per_step": int(sum_over_ranks(d2h)), "steps": steps,
            "note": "per step: source maps H2D from pinned host memory (upload stream) + ta_unproject + "
                    "ta_rasterize of every view + each view's F and A D2H into pinned host memory on a copy "
                    "stream overlapping the next view's rendering (H2D and D2H use the two PCIe directions)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--views", type=int, default=32)
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-stage-events", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
