#!/usr/bin/env python
"""Benchmark: forward 3DGS render with GEMM-compatible blending on B200.

Workload (BASELINE.json configs[4]): 6M Gaussians (SH degree 3) rendered at
1920x1080 from a 64-view camera orbit, views partitioned across the GPUs of
one node (one process per GPU), finished frames gathered to rank 0 over NCCL.
A step = the whole 64-view orbit (strong scaling: total work is fixed).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints one JSON line (rank 0). `--impl reference` times the CPU oracle (the
only reference this tier has) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec at 1080p per B200 and 8-GPU; tensor-pipe % and HBM GB/s"
UNIT = "frames/s"
INTERSECT = {"vanilla": (0, "vanilla 3-sigma rect"),
             "obox": (16, "GS_FLAG_OBOX: vanilla rect clipped to the opacity-aware alpha >= 1/255 box"),
             "tight": (8, "GS_FLAG_TIGHT: opacity-aware box + per-row ellipse column runs")}
VIEW_GROUP = int(os.environ.get("GS_BENCH_GROUP", "16"))   # views per preprocess launch (gs_set_view_group), binning chains concurrent
WORKLOAD = "C5: 6M Gaussians SH3, 1920x1080, 64-view orbit (BASELINE.json configs[4])"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        """Starts sampling every 100 ms and returns once the first sample is out (nvidia-smi
        takes a moment to start), so that the timed region that follows is covered."""
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.skip = 0
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        t0 = time.time()
        while time.time() - t0 < 10.0:
            with open(self.path) as f:
                n = sum(1 for _ in f)
            if n > 0:
                self.skip = n   # samples taken before the timed region are not counted
                return
            time.sleep(0.05)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in list(open(self.path))[self.skip:]:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: GS_BENCH_DEVICE pins every rank to one device (exercising the N > 1 host
    # path on a 1-GPU box with GS_BENCH_BACKEND=gloo); unset in real runs
    if os.environ.get("GS_BENCH_DEVICE") is not None:
        local = int(os.environ["GS_BENCH_DEVICE"])
    return ws, rank, local


def run_reference(args):
    """The oracle (oracle/, plain CPU) on a bounded sample of the same workload:
    each step renders one full 1920x1080 view of the C5 scene (preprocess,
    binning, f64 blending) on all host cores. Rank 0 only."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import oracle
    from paper_2604_02120_b200 import synth
    scene, cams, bg = synth.make_config("C5", views=args.views)
    threads = os.cpu_count() or 1
    times = []
    for k in range(args.warmup + args.steps):
        cam = cams[(k * 16) % len(cams)]
        t0 = time.perf_counter()
        oracle.render(scene, cam, bg, threads=threads, mask=False, obox=args.intersect == "obox")
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
    mean = sum(times) / len(times)
    value = 1.0 / mean
    sample = f"one full 1920x1080 view of the C5 scene per step (views 0,16,32,48 cycled), {threads} threads"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "views": args.views, "sample": "1 view per step",
                       "intersection": INTERSECT[args.intersect][1] if args.intersect != "tight" else INTERSECT["vanilla"][1]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(scene, cams, bg, obox, min_s=10.0, max_views=4):
    """Oracle timed on the host cores on a bounded sample of the same workload: views
    0, 1, ... of the orbit until at least min_s seconds (at most max_views views)."""
    import oracle
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    nv = 0
    while nv < min(max_views, len(cams)):
        oracle.render(scene, cams[nv], bg, threads=threads, mask=False, obox=obox)
        nv += 1
        if time.perf_counter() - t0 >= min_s:
            break
    dt = time.perf_counter() - t0
    return {"value": nv / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{nv} of the orbit's 1920x1080 views (views 0-{nv - 1}) of the C5 scene, "
                      f"{dt:.1f} s with {threads} threads"}


def _gpu_local_cpus(dev):
    """The CPU cores attached to GPU `dev`'s PCIe root (sysfs local_cpulist), or None."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(dev)
        bdf = f"{getattr(pr, 'pci_domain_id', 0):04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        cpus = set()
        for part in open(f"/sys/bus/pci/devices/{bdf}/local_cpulist").read().strip().split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2604_02120_b200 import (GS_BLEND_DIRECT, GS_BLEND_MMA, GS_BLEND_TC, GS_BLEND_TC_COLOR, GS_FLAG_STATS,
                                       GS_FLAG_TIGHT, GS_FLAG_TILE_LISTS, GS_FLAG_TIMING,
                                       Context, camera, opts, scene_to_device, scene_to_host, synth)
    from paper_2604_02120_b200.orbit import gather_frames_pipelined, gather_plan, partition_views, share_frames
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    # NUMA: this rank's host threads (and hence the pinned host buffers of the e2e path, placed
    # by first touch) on the cores of its GPU's PCIe root; the CPU oracle baseline gets every
    # core back
    all_cpus = os.sched_getaffinity(0)
    local_cpus = _gpu_local_cpus(local)
    if local_cpus:
        try:
            os.sched_setaffinity(0, local_cpus)
        except OSError:
            local_cpus = None
    backend = None
    if ws > 1:
        backend = os.environ.get("GS_BENCH_BACKEND", "nccl")   # gloo: test hook only (see _dist)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        if dist.get_world_size() != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but the process group has {dist.get_world_size()} ranks")
    scene, cams, bg = synth.make_config("C5", views=args.views)
    W, H = cams[0].W, cams[0].H
    mine = partition_views(args.views, ws, rank)
    per = len(mine)
    my_cams = [camera(cams[v]) for v in mine]
    blend = GS_BLEND_DIRECT if args.blend == "direct" else GS_BLEND_TC
    base_flags = INTERSECT[args.intersect][0]
    ctx = Context(local, max_points=scene.n, max_keys=args.max_keys, max_w=W, max_h=H)
    # view group: the rank's whole block up to 16 views (one scene read per group), the NCCL
    # gather in chunks of a quarter block that start as soon as their views are blended
    # (gs_stream_wait_view), so only the last chunk's transfer trails the rendering
    group, chunk = gather_plan(per, VIEW_GROUP)
    ctx.gs_set_view_group(group, True)
    st = scene_to_device(scene)
    fused = ws > 1 and args.gather == "fused"
    if fused:   # every rank's blends write straight into rank 0's frame buffers (CUDA IPC / NVLink)
        own = ((torch.empty((args.views, 3, H, W), device="cuda"), torch.empty((args.views, H, W), device="cuda"))
               if rank == 0 else (None, None))
        all_rgb, all_T = share_frames(own[0], own[1], rank, dist)
        out_rgb, out_T = all_rgb[mine.start:mine.stop], all_T[mine.start:mine.stop]
    else:
        out_rgb = torch.empty((per, 3, H, W), device="cuda")
        out_T = torch.empty((per, H, W), device="cuda")
    # GS_FLAG_STATIC_SCENE (a step's preprocess may overlap the previous step's last blends)
    # measured slower here (1210 vs 1233 fps: the overlap slows the blends); off by default
    static = 32 if os.environ.get("GS_BENCH_STATIC", "0") == "1" else 0
    o_plain = opts(bg, sh_degree=scene.sh_degree, blend=blend, flags=base_flags | static)
    o_timed = opts(bg, sh_degree=scene.sh_degree, blend=blend, flags=GS_FLAG_TIMING | base_flags | static)
    stream = torch.cuda.current_stream()

    gather_out = None
    if ws > 1 and rank == 0 and not fused:   # receive buffers of the frame gather, allocated once (untimed)
        gather_out = (torch.empty((ws, per, 3, H, W), device="cuda"), torch.empty((ws, per, H, W), device="cuda"))

    def step(o):
        ctx.gs_render_views(st, my_cams, W, H, o, out_rgb, out_T, stream)
        if fused:
            return   # the frames are already in rank 0's buffers when the blends complete
        # NCCL frame gather to rank 0, chunk by chunk as the views finish
        gather_frames_pipelined(out_rgb, out_T, ws, rank, chunk,
                                wait_views=lambda s, v: ctx.gs_stream_wait_view(s, v), dist=dist, out=gather_out)

    for _ in range(args.warmup):
        step(o_plain)
    torch.cuda.synchronize()
    ctx.gs_last_stats()
    ctx.gs_stage_times()                       # reset
    launches0 = ctx.gs_last_stats().launches
    clocks = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(o_timed)
    ev1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    stage_ms, frames = ctx.gs_stage_times()
    launches = ctx.gs_last_stats().launches - launches0
    if ws > 1:
        t = torch.tensor([elapsed_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = args.views * args.steps / (elapsed_ms / 1e3)

    # --- per-frame work counts for the roofline (one counting pass, untimed) ---
    o_stats = opts(bg, sh_degree=scene.sh_degree, blend=GS_BLEND_TC, flags=GS_FLAG_STATS | base_flags)
    n_eval = n_kept = n_keys = n_vis = 0
    sample_views = my_cams[:: max(1, per // 8)]
    for c in sample_views:
        ctx.gs_render(st, c, W, H, o_stats, out_rgb[0], out_T[0], stream)
        s = ctx.gs_last_stats()
        n_eval += s.pairs_evaluated
        n_kept += s.pairs_kept
        n_keys += s.n_keys
        n_vis += s.n_visible
    nv = len(sample_views)
    n_eval, n_kept, n_keys, n_vis = n_eval / nv, n_kept / nv, n_keys / nv, n_vis / nv
    # live stage times of the timed region: the group's binning chains overlap one
    # another there, so their per-chain time is not a per-frame cost; the blend (the
    # dominant kernel, the roofline below) and the preprocess run alone on the stream
    live_ms = [m / max(frames, 1) for m in stage_ms]
    # per-stage breakdown: one more orbit (untimed for `value`) with the chains serialised
    ctx.gs_set_view_group(group, False)
    ctx.gs_stage_times()
    ctx.gs_render_views(st, my_cams, W, H, o_timed, out_rgb, out_T, stream)
    torch.cuda.synchronize()
    ser_ms, ser_frames = ctx.gs_stage_times()
    ctx.gs_set_view_group(group, True)
    pre_ms, bin_ms, _ = (m / max(ser_frames, 1) for m in ser_ms)
    blend_ms = live_ms[2]

    peaks = _peaks()
    hbm = peaks.get("hbm_gbs") or 6650.0
    smax = peaks.get("sm_max_mhz") or 1965.0
    clk_mhz = clk.get("sm_mhz") or smax
    # issue roof of the blend: 148 SMs x 4 schedulers x 32 lanes per clock,
    # at the median SM clock measured during the timed region
    issue_peak = 148 * 128 * clk_mhz * 1e6 / 1e12        # T lane-slots/s
    N = scene.n
    M = scene.shs.shape[1]
    # algorithmic bytes: per view group the preprocess reads the 44 B of means,
    # scales, rotation and opacity of every Gaussian and the SH record (12 M B) of the ones
    # some view of the group projects (n_vis, the per-view count, is a lower bound of the
    # group's union); per view it writes the warp's slot count (4 B per 32 Gaussians) and
    # 60 B per visible Gaussian (index, depth, mean, conic+opacity, colour, rect, tiles)
    pre_bytes = (N * 44 + n_vis * 12 * M) / group + N / 8 + n_vis * 60
    # binning, the algorithmic traffic of the method's binning (per
    # visible Gaussian and per (Gaussian, tile) key K): compaction (read touched+depth, write
    # 8 B/vis), 3 depth passes (16 B/vis each + a histogram read) with the rect gather
    # (16 B/vis), duplication (8 B/key written), tile sort 2 passes (16 B/key each + histogram
    # read), ranges (4 B/key). The supertile scheme moves less (one pass over S ~ 0.31 K
    # supertile pairs; the per-tile split is the blend's filter), so this is the work the
    # canonical result needs, not the bytes the kernels move.
    bin_bytes = N * 8 + n_vis * 8 + 3 * 16 * n_vis + 4 * n_vis + 16 * n_vis + n_keys * 8 + \
        2 * 16 * n_keys + 4 * n_keys + 4 * n_keys
    # blend: SURVEY 8(d)'s issue roof -- 4 lane-slots per (Gaussian, pixel) pair the MMA
    # evaluates (the warp-level exit and the warp-uniform alpha-skip leave ~4 issue slots of
    # compositing per MMA pair; the Eq. 6 dot product itself runs on the tensor pipe)
    BLEND_SLOTS_PER_PAIR = 4.0
    blend_slots = BLEND_SLOTS_PER_PAIR * n_eval
    stages = {
        "preprocess": {"ms": pre_ms, "bound": "hbm", "achieved": pre_bytes / (pre_ms * 1e-3) / 1e9,
                       "peak": hbm, "unit": "GB/s", "view_group": group,
                       "timing": "per view; one launch covers a view group"},
        "binning": {"ms": bin_ms, "bound": "hbm", "achieved": bin_bytes / (bin_ms * 1e-3) / 1e9, "peak": hbm,
                    "unit": "GB/s", "kernels": "compaction, 3 depth passes, supertile-pair offsets, one 9-bit "
                    "supertile pass (expansion fused), supertile ranges", "timing": "chains serialised (extra orbit)"},
        "blend": {"ms": blend_ms, "bound": "alu", "achieved": blend_slots / (blend_ms * 1e-3) / 1e12,
                  "peak": issue_peak, "unit": "T lane-slots/s", "pairs_evaluated": n_eval, "pairs_kept": n_kept,
                  "slots_per_pair": BLEND_SLOTS_PER_PAIR,
                  "timing": "live, CUDA events around each launch in the timed region"},
    }
    for v in stages.values():
        v["frac"] = v["achieved"] / v["peak"]
    # the dominant single kernel is the blend (one launch per frame; binning is a chain
    # of ~28 short kernels, preprocess one). DRAM traffic / tensor-pipe % per launch come
    # from the committed ncu --set full capture (profiles/ncu_kernel_metrics.json).
    ncu = {}
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_kernel_metrics.json")))
    except Exception:
        pass
    bl = ncu.get("k_blend_tc", {})
    roof = {"kernel": "k_blend_tc", "bound": "alu", "achieved": stages["blend"]["achieved"],
            "peak": stages["blend"]["peak"], "unit": "T lane-slots/s", "frac": stages["blend"]["frac"],
            "traffic": bl.get("dram_bytes_per_launch"),
            "peak_note": ("issue roof: 148 SMs x 128 lanes x median SM clock of the timed region "
                          f"({clk_mhz:.0f} MHz); achieved = 4 lane-slots (SURVEY 8(d)) x the (Gaussian, pixel) "
                          "pairs the MMA evaluates per frame / live blend time"),
            "tensor_pipe_pct": bl.get("tensor_pipe_pct"), "issue_active_pct": bl.get("issue_active_pct"),
            "ncu_source": bl.get("source")}

    # --- N1: the CUDA-core direct blend (vanilla Alg. 1) and the warp-level mma.sync
    # blend (the paper's kernel shape) at batch sizes b = 32..256 (N2), on the same
    # orbit: blend ms per frame (live events) and orbit fps, A/B against tcgen05 ---
    ab = None
    if not args.no_ab and args.blend == "tc":
        def orbit_time(o):
            ctx.gs_render_views(st, my_cams, W, H, o, out_rgb, out_T, stream)   # warm
            torch.cuda.synchronize()
            ctx.gs_stage_times()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.gs_render_views(st, my_cams, W, H, o, out_rgb, out_T, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            dms, dfr = ctx.gs_stage_times()
            return dms[2] / max(dfr, 1), per / (e0.elapsed_time(e1) / 1e3)
        # every arm on the headline's lists (same intersection flag), the tcgen05 arm re-timed
        # in the same way beside them
        t_ms, t_fps = orbit_time(opts(bg, sh_degree=scene.sh_degree, blend=GS_BLEND_TC,
                                      flags=GS_FLAG_TIMING | base_flags))
        d_ms, d_fps = orbit_time(opts(bg, sh_degree=scene.sh_degree, blend=GS_BLEND_DIRECT,
                                      flags=GS_FLAG_TIMING | base_flags))
        # the tcgen05 blend on the per-tile lists the other arms read (kernel-to-kernel A/B;
        # the headline bins into supertile lists the tcgen05 blend filters itself)
        tl_ms, tl_fps = orbit_time(opts(bg, sh_degree=scene.sh_degree, blend=GS_BLEND_TC,
                                        flags=GS_FLAG_TIMING | GS_FLAG_TILE_LISTS | base_flags))
        ab = {"intersection": INTERSECT[args.intersect][1], "blend_tc_ms": t_ms, "fps_tc": t_fps,
              "lists": "tc: supertile lists filtered in the blend (headline); tc_tile_lists, direct, mma_sync: "
                       "per-tile lists (two-level binning), the same lists for the kernel A/B",
              "tc_tile_lists": {"blend_ms": tl_ms, "fps": tl_fps},
              "blend_direct_ms": d_ms, "fps_direct": d_fps, "speedup_tc_over_direct": d_ms / tl_ms, "mma_sync": {}}
        for b in (32, 64, 128, 256):
            m_ms, m_fps = orbit_time(opts(bg, sh_degree=scene.sh_degree, blend=GS_BLEND_MMA, batch=b,
                                          flags=GS_FLAG_TIMING | base_flags))
            ab["mma_sync"][f"b{b}"] = {"blend_ms": m_ms, "fps": m_fps, "speedup_tc_over_mma": m_ms / tl_ms}
        # N4: the colour sum as a second tcgen05 product (2 CTAs per SM), same lists
        c_ms, c_fps = orbit_time(opts(bg, sh_degree=scene.sh_degree, blend=GS_BLEND_TC_COLOR,
                                      flags=GS_FLAG_TIMING | base_flags))
        ab["tc_color"] = {"blend_ms": c_ms, "fps": c_fps, "speedup_tc_over_tc_color": c_ms / t_ms,
                          "note": "GS_BLEND_TC_COLOR (SURVEY N4): C += (alpha T) . colours^T on tcgen05, "
                                  "2 CTAs/SM; frames within the parity gate (tests)"}

    # --- N3: the other intersection modes (bit-identical frames, fewer pairs), one timed orbit each ---
    n3 = {}
    for mode in ([] if args.no_ab else [m for m in INTERSECT if m != args.intersect]):
        mflag = INTERSECT[mode][0]
        o_t = opts(bg, sh_degree=scene.sh_degree, blend=blend, flags=GS_FLAG_TIMING | mflag)
        ctx.gs_render_views(st, my_cams, W, H, o_t, out_rgb, out_T, stream)   # warm
        torch.cuda.synchronize()
        ctx.gs_stage_times()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.gs_render_views(st, my_cams, W, H, o_t, out_rgb, out_T, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        tms, tfr = ctx.gs_stage_times()
        ctx.gs_render(st, my_cams[0], W, H, opts(bg, sh_degree=scene.sh_degree, flags=GS_FLAG_STATS | mflag),
                      out_rgb[0], out_T[0], stream)
        ts = ctx.gs_last_stats()
        n3[mode] = {"fps": per / (e0.elapsed_time(e1) / 1e3),
                    "stage_ms_per_frame_live": dict(zip(("preprocess", "binning_chain_overlapped", "blend"),
                                                        (m / max(tfr, 1) for m in tms))),
                    "n_keys_view0": ts.n_keys, "pairs_evaluated_view0": ts.pairs_evaluated,
                    "note": INTERSECT[mode][1] + "; frames bit-identical to the vanilla-rect ones (tested)"}

    # --- SURVEY 8(e) option: tile-row split of ONE view. Per-band device time of band k
    # of n (what each of n GPUs would render; the band gather is not included) ---
    row_split = None
    if not args.no_ab and ws == 1:
        row_split = {}
        c0 = my_cams[0]
        for nb in (1, 2, 4, 8):
            worst = 0.0
            for k in range(nb):
                o_b = opts(bg, sh_degree=scene.sh_degree, blend=blend, flags=base_flags, band=k, n_bands=nb)
                for _ in range(2):
                    ctx.gs_render(st, c0, W, H, o_b, out_rgb[0], out_T[0], stream)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(5):
                    ctx.gs_render(st, c0, W, H, o_b, out_rgb[0], out_T[0], stream)
                e1.record(stream)
                torch.cuda.synchronize()
                worst = max(worst, e0.elapsed_time(e1) / 5)
            row_split[f"{nb}_bands"] = {"max_band_ms": worst, "speedup_vs_1": None}
        for v in row_split.values():
            v["speedup_vs_1"] = row_split["1_bands"]["max_band_ms"] / v["max_band_ms"]

    # --- N2: resolution sensitivity (1x / 2x / 3x of 1080p, same scene, orbit views) ---
    res_sweep = None
    if not args.no_sweep and ws == 1:
        res_sweep = {}
        o_r = opts(bg, sh_degree=scene.sh_degree, blend=blend, flags=base_flags)
        for sc in (1, 2, 3):
            Ws, Hs = W * sc, H * sc
            cams_s = [camera(c) for c in synth.orbit_cameras(args.views, Ws, Hs, math.radians(60.0))]
            cams_s = cams_s[:: max(1, args.views // args.sweep_views)][:args.sweep_views]
            ctx_s = ctx if sc == 1 else Context(local, max_points=scene.n, max_keys=args.max_keys * sc * sc,
                                                   max_w=Ws, max_h=Hs)
            rgb_s = torch.empty((len(cams_s), 3, Hs, Ws), device="cuda")
            T_s = torch.empty((len(cams_s), Hs, Ws), device="cuda")
            ctx_s.gs_render_views(st, cams_s, Ws, Hs, o_r, rgb_s, T_s, stream)   # warm
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(2):
                ctx_s.gs_render_views(st, cams_s, Ws, Hs, o_r, rgb_s, T_s, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / (2 * len(cams_s))
            ctx_s.gs_render(st, cams_s[0], Ws, Hs, opts(bg, sh_degree=scene.sh_degree, flags=GS_FLAG_STATS | base_flags),
                            rgb_s[0], T_s[0], stream)
            s0 = ctx_s.gs_last_stats()
            gx, gy = -(-Ws // 16), -(-Hs // 16)
            res_sweep[f"{sc}x"] = {"W": Ws, "H": Hs, "fps": 1e3 / ms, "ms_per_frame": ms, "views": len(cams_s),
                                   "n_keys_view0": s0.n_keys, "pairs_evaluated_view0": s0.pairs_evaluated,
                                   "binning": ("supertile" if -(-gx // 4) * -(-gy // 4) <= 512 else
                                               "two-level" if gx <= 512 and gy <= 512 else "one-level")}
            del rgb_s, T_s
            if ctx_s is not ctx:
                ctx_s.close()
        torch.cuda.empty_cache()

    # --- the other BASELINE.json config shapes (parity cases; reported for context):
    # single-view gs_render latency and an 8-view orbit of each, same intersection ---
    per_config = None
    if not args.no_configs and ws == 1:
        per_config = {}
        for name in ("C2", "C3", "C4a", "C4b"):
            sc_c, cams_c, bg_c = synth.make_config(name, views=8)
            Wc, Hc = cams_c[0].W, cams_c[0].H
            ctx_c = Context(local, max_points=sc_c.n, max_keys=args.max_keys, max_w=Wc, max_h=Hc)
            ctx_c.gs_set_view_group(8, True)
            st_c = scene_to_device(sc_c)
            cc = [camera(c) for c in cams_c]
            rgb_c = torch.empty((len(cc), 3, Hc, Wc), device="cuda")
            T_c = torch.empty((len(cc), Hc, Wc), device="cuda")
            o_c = opts(bg_c, sh_degree=sc_c.sh_degree, blend=blend, flags=base_flags)
            for _ in range(2):
                ctx_c.gs_render_views(st_c, cc, Wc, Hc, o_c, rgb_c, T_c, stream)
                ctx_c.gs_render(st_c, cc[0], Wc, Hc, o_c, rgb_c[0], T_c[0], stream)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            for _ in range(3):
                ctx_c.gs_render_views(st_c, cc, Wc, Hc, o_c, rgb_c, T_c, stream)
            e1.record(stream)
            for _ in range(5):
                ctx_c.gs_render(st_c, cc[0], Wc, Hc, o_c, rgb_c[0], T_c[0], stream)
            e2.record(stream)
            torch.cuda.synchronize()
            ctx_c.gs_render(st_c, cc[0], Wc, Hc, opts(bg_c, sh_degree=sc_c.sh_degree, flags=GS_FLAG_STATS | base_flags),
                            rgb_c[0], T_c[0], stream)
            s_c = ctx_c.gs_last_stats()
            per_config[name] = {"n_gaussians": sc_c.n, "W": Wc, "H": Hc,
                                "fps_orbit8": 3 * len(cc) / (e0.elapsed_time(e1) / 1e3),
                                "ms_single_view": e1.elapsed_time(e2) / 5, "n_visible_view0": s_c.n_visible,
                                "n_keys_view0": s_c.n_keys, "pairs_evaluated_view0": s_c.pairs_evaluated}
            ctx_c.close()
            del st_c, rgb_c, T_c
        torch.cuda.empty_cache()

    # --- end to end through the host-pointer C-ABI entry point ---------------
    # Every step copies the scene host -> device and all its frames device -> host. The
    # headline uses gs_render_views_host_async back to back (a serving loop: the next
    # step's upload overlaps this step's rendering; D2H overlaps rendering within a step),
    # timed from the first call to the completion of the last; the synchronous entry
    # point (each call returns after its frames are on the host) is reported beside it.
    e2e = None
    if not args.no_e2e:
        hs = scene_to_host(scene, pinned=True)
        h_rgb = torch.empty((per, 3, H, W), pin_memory=True)
        h_T = torch.empty((per, H, W), pin_memory=True)

        def run(async_, steps):
            # wall clock from an idle device to the completion of `steps` back-to-back calls (a
            # call completes on the caller's stream once its frames are on the host)
            torch.cuda.synchronize()
            if ws > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(steps):
                ctx.gs_render_views_host(hs, my_cams, W, H, o_plain, h_rgb, h_T, stream, async_=async_)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if ws > 1:
                t = torch.tensor([dt], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = float(t.item())
            return dt

        for _ in range(max(1, args.warmup)):   # warm-up (allocations, staging buffers)
            run(True, 1)
        # steady state of the serving loop: two runs of K1 and K2 back-to-back async calls; each
        # pays the pipeline fill once (the first call's upload has nothing to overlap), so the
        # difference of their times is K2 - K1 steady-state steps (each with its own scene H2D
        # and frame D2H)
        k1 = 4
        k2 = k1 + max(8, args.e2e_steps, args.steps)
        t1, t2 = run(True, k1), run(True, k2)
        v_async = args.views * (k2 - k1) / (t2 - t1)
        v_fill = args.views * k2 / t2
        v_sync = args.views * args.e2e_steps / run(False, args.e2e_steps)
        e2e_steps = k2 - k1
        in_bytes = sum(int(np.prod(a.shape)) * 4 for a in (scene.means, scene.scales, scene.rots,
                                                              scene.opacity, scene.shs))
        e2e = {"value": v_async, "unit": UNIT, "h2d_bytes_per_step": in_bytes,
               "d2h_bytes_per_step": per * 4 * W * H * 4, "steps": e2e_steps, "warmup": max(1, args.warmup),
               "fill_included_value": v_fill, "sync_value": v_sync,
               "note": "gs_render_views_host_async back to back, wall clock to the host having the frames: "
                       "steady state = (K2 - K1) steps / (T(K2) - T(K1)) for runs of K1 = 4 and K2 calls (the "
                       "pipeline fill cancels; fill_included_value = K2 steps / T(K2)); every step is a pinned "
                       "scene H2D + 64/N renders + frames D2H per rank; PCIe on this box moves ~85 GB/s with "
                       "both directions busy (profiles/r2_pcie_probe.txt), 3.54 GB per step (sync_value: "
                       "gs_render_views_host, each call returns with its frames on the host)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            os.sched_setaffinity(0, all_cpus)
        except OSError:
            pass
        cpu = cpu_baseline(scene, cams, bg, args.intersect == "obox")

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": WORKLOAD, "views": args.views, "n_gaussians": N, "W": W, "H": H,
                           "sh_degree": scene.sh_degree, "blend": args.blend,
                           "intersection": INTERSECT[args.intersect][1],
                           "frame_gather": ("none (1 GPU)" if ws == 1 else
                                            "fused: blends write into rank 0's frames via CUDA IPC / NVLink"
                                            if args.gather == "fused" else "NCCL gather per view group, overlapped"),
                           "parallelism": f"view-partition x{ws}" + (" + NCCL gather" if ws > 1 else ""),
                           "l2": "inputs larger than L2 (1.42 GB scene, 2.1 GB of frames per step)",
                           "host_cpus": (f"{len(local_cpus)} cores local to the GPU's PCIe root" if local_cpus
                                         else "unbound (no sysfs local_cpulist)")},
                "ms_per_frame": elapsed_ms / args.steps / per, "stage_ms_per_frame": {
                    k: v["ms"] for k, v in stages.items()},
                "stage_ms_per_frame_live": dict(zip(("preprocess", "binning_chain_overlapped", "blend"), live_ms)),
                "roofline": roof, "stages": stages, "clocks": clk,
                "comm": ({"backend": backend, "world_size": dist.get_world_size(),
                          "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if backend == "nccl" else None,
                          "view_group": group, "gather_chunk_views": chunk} if ws > 1 else None),
                "gpu_launches": int(launches), "e2e": e2e, "cpu_baseline": cpu, "ab_blend": ab, "intersection_modes": n3, "row_split_one_view": row_split, "other_configs": per_config,
                "resolution_sweep": res_sweep,
                "work_per_frame": {"n_visible": n_vis, "n_keys": n_keys, "pairs_evaluated": n_eval,
                                   "pairs_kept": n_kept}}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.cuda.synchronize()
        dist.barrier()   # (fused gather: rank 0's frame buffers stay mapped until every rank is done)
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--blend", default="tc", choices=["tc", "direct"])
    ap.add_argument("--max-keys", type=int, default=48 << 20)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ab", action="store_true")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "fused"],
                    help="N > 1: NCCL gather per view group (default) or blends writing into rank 0's frames "
                         "through CUDA IPC peer memory")
    ap.add_argument("--intersect", default="obox", choices=list(INTERSECT),
                    help="intersection mode of the headline (the others are timed alongside, N3)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the N2 resolution sweep")
    ap.add_argument("--no-configs", action="store_true", help="skip the C2-C4b config shapes")
    ap.add_argument("--sweep-views", type=int, default=8)
    args = ap.parse_args()
    ws_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and ws_env is None:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    if ws_env is not None and int(ws_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
