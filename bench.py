#!/usr/bin/env python
"""Benchmark of the MERF baked-scene render path on B200 (one JSON line on rank 0).

Workload (BASELINE.json metric "rays/sec and fps at 1920x1080 per B200"): the paper-scale
synthetic baked MERF scene (512^3 block-sparse grid, 3 x 2048^2 planes, C = 8, occupancy
32^3/128^3/256^3; config 2's scene) rendered from the config-4 orbit of 256 1920x1080 views.
A step = every rank renders its V views (RGBA8) with the fused render kernel and, for N > 1,
the finished frames are gathered to rank 0 over NCCL (the only collective; off the hot path).
Weak scaling: V views per rank per step; rank r of N takes views (s*V*N + i*N + r) mod 256.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl merf|reference]

`--impl reference` times the fp64 CPU oracle (the only "reference implementation" of this
tier: the paper publishes no code) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rays/sec and fps at 1920x1080 per B200 (1/2/4/8 GPUs); gather GB/s vs roofline"
W_IMG, H_IMG = 1920, 1080
N_ORBIT = 256
BYTES_APPEARANCE = 160      # 20 texels x 8 channels x 1 B
BYTES_DENSITY_ONLY = 20     # 20 texels x 1 B
BYTES_OUT = 4               # RGBA8 per ray
PAPER_CONTEXT = {"merf_fps_rtx3090_1080p_browser": 119, "merf_fps_m1_720p_browser": 28.3,
                 "source": "PAPER.md Table 2 (P:379, P:383); real scenes, other hardware"}


def views_for(rank: int, world: int, step: int, per_rank: int, n_orbit: int = N_ORBIT):
    """view indices rank `rank` renders at step `step` (weak scaling: per_rank fixed)."""
    return [(step * per_rank * world + i * world + rank) % n_orbit for i in range(per_rank)]


def gather_frames(frames, rank: int, world: int, group=None):
    """Reference semantics of the frame gather (gloo in the CPU tests): every rank's frame
    batch to rank 0.  On the GPU bench.py gathers through libmerf's merf_gather_frames (NCCL)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return [frames]
    out = [torch.empty_like(frames) for _ in range(world)] if rank == 0 else None
    dist.gather(frames, gather_list=out, dst=0, group=group)
    return out


def make_comm(M, rank: int, world: int, device: int):
    """libmerf's NCCL communicator; rank 0's unique id travels over the torch.distributed
    store (plumbing only)."""
    import torch.distributed as dist
    uid = [M.merf_comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    return M.Comm(uid[0], world, rank, device)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 6:
                self.rows.append(p)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _ncu_capture():
    """per-launch counters of the march kernel from the committed ncu --set full capture
    (profiles/render_traffic.json, written by tools/traffic_from_ncu.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "render_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _ncu_traffic():
    """dram bytes per launch of the render kernel from the committed ncu --set full capture."""
    return _ncu_capture().get("dram_bytes_per_launch")


def _capture_current():
    """does the committed capture describe the library built now?  (source digest stamp)"""
    try:
        from paper_2302_12249_b200.build import source_hash
        cap = _ncu_capture().get("source_sha16")
        return {"capture_source_sha16": cap, "build_source_sha16": source_hash(),
                "current": cap is not None and cap == source_hash()}
    except Exception as e:  # noqa: BLE001
        return {"current": False, "error": str(e)}


def march_instance(info) -> str:
    """the march template instance merf_render launches for this scene (merf_march.cu)"""
    paper = info["L"] == 512 and info["R"] == 2048 and list(info["level_res"])[-1] == 256
    return ("merf::march_kernel<448> (KF_ALLSRC|KF_SKIPTAB|KF_PAPER)" if paper
            else "merf::march_kernel<192> (KF_ALLSRC|KF_SKIPTAB)")


def issue_roofline(avg_launch_ms: float, sm_mhz: float, n_sm: int):
    """The limiter of the march kernel: instruction issue.  achieved = warp instructions per
    launch (ncu, same launch configuration) / (live launch time x SM clock x SMs), against 4
    (one issue per cycle per SM sub-partition)."""
    cap = _ncu_capture()
    inst = cap.get("warp_inst_per_launch")
    if not inst or not avg_launch_ms or not sm_mhz:
        return None
    ipc = inst / (avg_launch_ms * 1e-3 * sm_mhz * 1e6 * n_sm)
    return {"bound": "issue", "achieved": ipc, "peak": 4.0, "unit": "warp inst / cycle / SM",
            "frac": ipc / 4.0, "warp_inst_per_launch": inst, "capture": _capture_current(),
            "source": "instruction count: " + cap.get("source", "profiles/render_traffic.json")
                      + "; time: live CUDA events of this run; clock: nvidia-smi median during the run"}


def cpu_baseline(scene, cams, sample_stride: int = 1):
    """the fp64 oracle, as it stands, on all host cores: full 1080p orbit views (every
    `sample_stride`-th pixel), about 10 s of CPU work for 4 views."""
    import numpy as np
    from oracle import oracle as O
    osc = O.OracleScene(scene)
    pix = np.arange(0, W_IMG * H_IMG, sample_stride, dtype=np.int64)
    t0 = time.perf_counter()
    ev = 0
    for cam in cams:
        r = O.render(osc, cam, W_IMG, H_IMG, pixels=pix)
        ev += r["stats"]["evaluated"]
    dt = time.perf_counter() - t0
    n = len(pix) * len(cams)
    return {"value": n / dt, "unit": "rays/s", "cores": O.max_threads(), "kind": "oracle",
            "sample": f"{len(cams)} orbit views at 1920x1080 ({n} rays, every {sample_stride}th pixel), "
                      f"fp64, {dt:.1f} s wall, samples/ray {ev / n:.1f}",
            "seconds": dt}


def run_reference(args):
    """--impl reference: the CPU oracle on a bounded sample per step (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    from merf_inputs import make_scene, orbit_cameras
    from oracle import oracle as O
    sc = make_scene("c2")
    osc = O.OracleScene(sc)
    stride = 37     # ~56k rays per step: a step is ~1/37 of a view's pixels
    times, rays = [], 0
    for s in range(args.warmup + args.steps):
        v = views_for(0, 1, s, 1)[0]
        cam = orbit_cameras(N_ORBIT, indices=[v])[0]
        pix = np.arange(s % stride, W_IMG * H_IMG, stride, dtype=np.int64)
        t0 = time.perf_counter()
        O.render(osc, cam, W_IMG, H_IMG, pixels=pix)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            rays += len(pix)
    total = sum(times)
    value = rays / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "rays/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "orbit1080p_paper_scale_merf" + ("_dense_ablation" if args.dense else "")
                        + ("_mlp_ffma_ablation" if getattr(args, "mlp_ffma", False) else "")
                                   + ("_spherical_contraction" if args.spherical else "")
                                   + ("_persistent_fp32" if getattr(args, "sph_persistent", False) else ""), "scene": "c2 (512^3 sparse grid, 3x2048^2 planes)",
                       "sample": f"every {stride}th pixel of one 1920x1080 orbit view per step"},
            "cpu_baseline": {"value": value, "unit": "rays/s", "cores": O.max_threads(), "kind": "oracle",
                             "sample": f"every {stride}th pixel of one 1920x1080 orbit view per step"},
            "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "fps_equivalent": value / (W_IMG * H_IMG)}
    print(json.dumps(line), flush=True)
    return 0


def e2e_multi(M, scene, comm, batches, args, rank, world, dev, stream, gstream, frames, root_bufs, total_rays):
    """End to end at N > 1 through the public API, every step inside the timed region: each rank
    renders its views (merf_render, camera parameters host -> device), the frames are gathered to
    rank 0 (merf_gather_frames over NCCL), and rank 0 copies the gathered frames of all ranks to
    pinned host memory.  Max over ranks."""
    import torch
    import torch.distributed as dist
    V = args.views
    host = (torch.empty((world, V, H_IMG, W_IMG, 4), dtype=torch.uint8).pin_memory() if rank == 0 else None)
    cstream = torch.cuda.Stream()
    ready = [torch.cuda.Event() for _ in range(2)]      # gather of buffer b done
    copied = [torch.cuda.Event() for _ in range(2)]     # root's D2H of buffer b done

    def one(s, i):
        b = i & 1
        if i >= 2:
            stream.wait_event(copied[b] if rank == 0 else ready[b])
        M.merf_render(scene.handle, batches[s], W_IMG, H_IMG, frames[b], fmt=M.MERF_RGBA_U8, stream=stream)
        gstream.wait_stream(stream)
        comm.gather(frames[b], root_bufs[b], root=0, stream=gstream)
        ready[b].record(gstream)
        if rank == 0:
            cstream.wait_event(ready[b])
            with torch.cuda.stream(cstream):
                host.copy_(root_bufs[b], non_blocking=True)
            copied[b].record(cstream)

    for i, s in enumerate(range(min(2, args.warmup))):
        one(s, i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i, s in enumerate(range(args.warmup, args.warmup + args.steps)):
        one(s, i)
    stream.wait_stream(gstream)
    stream.wait_stream(cstream)
    e1.record(stream)
    comm.wait(stream=stream, timeout_ms=120000)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ems = float(t.item())
    return {"value": total_rays / (ems / 1e3), "unit": "rays/s",
            "h2d_bytes_per_step": world * V * 136, "d2h_bytes_per_step": world * V * W_IMG * H_IMG * 4,
            "nccl_bytes_per_step": (world - 1) * V * W_IMG * H_IMG * 4,
            "path": "per rank merf_render (device frames) -> merf_gather_frames to rank 0 (NCCL) -> rank 0 "
                    "copies all ranks' frames to pinned host memory; max over ranks"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="merf", choices=["merf", "reference"])
    ap.add_argument("--views", type=int, default=16, help="views per rank per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-gather", action="store_true",
                    help="run the N > 1 frame-gather and e2e path through a 1-rank NCCL communicator "
                         "(exercises it on one GPU; not a scaling measurement)")
    ap.add_argument("--spherical", action="store_true",
                    help="NEXT-2 comparison: the scene baked in the spherical contraction's space, "
                         "rendered with fixed contracted-arc-length steps and no AABB skipping")
    ap.add_argument("--sph-persistent", action="store_true",
                    help="with --spherical: the curve march in fp32 inside the persistent tile-scheduled "
                         "march kernel (like-for-like with the contract_pi path)")
    ap.add_argument("--dense", action="store_true",
                    help="ablation: dense lattice stepping gated by the finest level (no skipping)")
    ap.add_argument("--mlp-ffma", action="store_true",
                    help="ablation: the deferred MLP as FFMA chains instead of the tensor-core kernel")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    from merf_inputs import make_scene, orbit_cameras
    import paper_2302_12249_b200 as M

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert torch.cuda.is_available(), "bench.py needs a GPU (no CPU fallback)"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = f"cuda:{local}"

    sc = make_scene("c2", contraction="sph" if args.spherical else "pi")
    scene = M.Scene(sc, device=local)
    n_fin = sc.level_res[-1]
    occ_frac = float(np.unpackbits(sc.occ_finest.view(np.uint8)).sum()) / n_fin ** 3
    info = scene.info()
    V = args.views
    steps_total = args.warmup + args.steps
    batches = [orbit_cameras(N_ORBIT, indices=views_for(rank, world, s, V)) for s in range(steps_total)]

    extra_flags = ((M.MERF_DENSE if args.dense else 0) | (M.MERF_SPHERICAL if args.spherical else 0)
                   | (M.MERF_SPH_PERSISTENT if args.sph_persistent else 0)
                   | (M.MERF_MLP_FFMA if args.mlp_ffma else 0))
    stream = torch.cuda.Stream()
    gstream = torch.cuda.Stream()
    frames = [torch.empty((V, H_IMG, W_IMG, 4), dtype=torch.uint8, device=dev) for _ in range(2)]
    # the frame gather runs at N > 1 (and, to exercise the N > 1 code path on one GPU, with a
    # 1-rank communicator under --force-gather)
    gathering = world > 1 or args.force_gather
    comm = make_comm(M, rank, world, local) if gathering else None
    # the root's gather targets: [world][V][H][W][4], double buffered like the frames
    root_bufs = ([torch.empty((world, V, H_IMG, W_IMG, 4), dtype=torch.uint8, device=dev) for _ in range(2)]
                 if gathering and rank == 0 else [None, None])

    # ---- counters pass over exactly the launches timed below (untimed, same views)
    algo_bytes, n_eval, n_donly, n_skip, n_seg = [], 0, 0, 0, 0
    region_segs = [0] * 7
    with torch.cuda.stream(stream):
        for s in range(args.warmup, steps_total):
            st = M.merf_render(scene.handle, batches[s], W_IMG, H_IMG, frames[0], fmt=M.MERF_RGBA_U8,
                               flags=extra_flags, stream=stream, stats=True)
            app = st["evaluated"] - st["density_only"]
            algo_bytes.append(BYTES_APPEARANCE * app + BYTES_DENSITY_ONLY * st["density_only"])
            n_eval += st["evaluated"]
            n_donly += st["density_only"]
            n_skip += st["skips"]
            n_seg += st["segments"]
            region_segs = [a + b for a, b in zip(region_segs, st["region_segments"])]
    rays_per_step = V * W_IMG * H_IMG
    ws = M.merf_render_workspace_bytes(scene.handle, batches[args.warmup], W_IMG, H_IMG)
    vram = {"scene_device_bytes": info["device_bytes"], "baked_arrays_bytes": int(sc.nbytes()),
            "render_workspace_bytes": ws["bytes"], "workspace_bytes_per_ray": ws["bytes_per_ray"],
            "frame_buffers_bytes": 2 * V * H_IMG * W_IMG * 4,
            "note": "scene = every device layout built at upload (DESIGN 5); workspace = one merf_render "
                    "chunk (4 segment slots per ray for cameras inside the core, else 7; accumulators; "
                    "tile lists)"}

    gathered = [torch.cuda.Event() for _ in range(2)]   # buffer b's last gather finished

    def step(s):
        b = s & 1
        buf = frames[b]
        with torch.cuda.stream(stream):
            if gathering and s >= 2:
                stream.wait_event(gathered[b])       # reuse buffer b only after ITS gather (step s-2)
            ev0[s].record(stream)
            M.merf_render(scene.handle, batches[s], W_IMG, H_IMG, buf, fmt=M.MERF_RGBA_U8,
                          flags=(M.MERF_TIMED if s >= args.warmup else 0) | extra_flags, stream=stream)
            ev1[s].record(stream)
        if gathering:
            # the gather of step s (libmerf merf_gather_frames: grouped NCCL send/recv to rank
            # 0) overlaps the render of step s+1 (the other buffer)
            gstream.wait_stream(stream)
            comm.gather(buf, root_bufs[b], root=0, stream=gstream)
            gathered[b].record(gstream)

    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps_total)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps_total)]
    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t_start.record(stream)
    for s in range(args.warmup, steps_total):
        step(s)
    stream.wait_stream(gstream)
    t_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    if comm is not None:
        comm.wait(stream=gstream, timeout_ms=120000)  # NCCL async errors surface here
    ms = t_start.elapsed_time(t_end)
    call_ms = [ev0[s].elapsed_time(ev1[s]) for s in range(args.warmup, steps_total)]
    gather_check = None
    if gathering:
        # integrity of the last gather: rank 0's slot r holds rank r's last frames
        last = (steps_total - 1) & 1
        ck = torch.tensor([float(frames[last].sum(dtype=torch.int64).item())], dtype=torch.float64, device=dev)
        cks = [torch.zeros_like(ck) for _ in range(world)]
        if world > 1:
            dist.all_gather(cks, ck)
        else:
            cks = [ck]
        if rank == 0:
            got = [float(root_bufs[last][r].sum(dtype=torch.int64).item()) for r in range(world)]
            gather_check = all(abs(g - float(c.item())) == 0 for g, c in zip(got, cks))
    kt = M.merf_kernel_times_get(scene.handle, reset=True)
    rank_ms = [ms]
    if world > 1:
        t = torch.tensor([ms], device=dev)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)                      # per-rank times: imbalance
        rank_ms = [float(x.item()) for x in allt]
        ms = max(rank_ms)
    ms_per_step = ms / args.steps
    total_rays = rays_per_step * world * args.steps
    value = total_rays / (ms / 1e3)

    # ---- roofline of the dominant kernel: the persistent march kernel (CUDA events around
    # every launch, recorded by the library on the render stream with MERF_TIMED)
    peak, peak_src = _peaks()
    n_march = max(kt["march_launches"], 1)
    avg_launch_ms = kt["march_ms"] / n_march
    bytes_per_launch = sum(algo_bytes) / n_march
    achieved = bytes_per_launch / (avg_launch_ms / 1e3) / 1e9
    traffic = _ncu_traffic()
    dram_gbs = traffic / (avg_launch_ms / 1e3) / 1e9 if traffic else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "achieved_is": "algorithmic gather rate: the texel bytes the method reads (SURVEY 8(d) "
                               "model) / live launch time; served mostly by L1/L2, not HBM",
                "dram_gbs": dram_gbs, "dram_frac": dram_gbs / peak if dram_gbs else None,
                "dram_source": "ncu dram bytes per launch (profiles/render_traffic.json) / live launch time",
                "capture": _capture_current(),
                "kernel": march_instance(info) + " (persistent march: traversal + gather + composite)",
                "avg_launch_ms": avg_launch_ms, "launches": kt["march_launches"],
                "algorithmic_bytes_per_launch": bytes_per_launch,
                "bytes_model": "160 B per evaluated sample with alpha > 0, 20 B per density-only "
                               "sample (SURVEY 8(d)); launch = one chunk of 16 views",
                "l2_bytes_per_launch": _ncu_capture().get("l2_bytes_per_launch"),
                "note": "algorithmic gather bytes over the live launch time; texels are served from "
                        "L1 (86 % hit) and L2, DRAM traffic (`traffic`) is ~5 % of the algorithmic "
                        "bytes, so frac can exceed 1: the kernel is instruction-issue bound "
                        "(roofline_issue)",
                "pipeline_ms_per_step": {"setup": kt["setup_ms"] / args.steps,
                                         "march": kt["march_ms"] / args.steps,
                                         "shade": kt["shade_ms"] / args.steps,
                                         "merf_render_call": sum(call_ms) / len(call_ms)}}

    # ---- end to end through the C ABI with host buffers (pinned), copies in the timed region
    e2e = None
    if not args.no_e2e and gathering:
        e2e = e2e_multi(M, scene, comm, batches, args, rank, world, dev, stream, gstream, frames, root_bufs,
                        total_rays)
    elif not args.no_e2e:
        # a frame stream through the public API: each step's views are rendered and copied to
        # pinned host memory (merf_render_host_async: the copy of step s overlaps the render of
        # step s + 1); the timed region ends when the last step's frames are in host memory
        host = [torch.empty((V, H_IMG, W_IMG, 4), dtype=torch.uint8).pin_memory() for _ in range(2)]
        for s in range(min(2, args.warmup)):
            M.merf_render_host_async(scene.handle, batches[s], W_IMG, H_IMG, host[s & 1], fmt=M.MERF_RGBA_U8,
                                     stream=stream)
        M.merf_host_wait(scene.handle)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for s in range(args.warmup, steps_total):
            M.merf_render_host_async(scene.handle, batches[s], W_IMG, H_IMG, host[s & 1], fmt=M.MERF_RGBA_U8,
                                     stream=stream)
        M.merf_host_wait(scene.handle)
        ems = (time.perf_counter() - t0) * 1e3       # host clock: the frames are on the host
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": total_rays / (ems / 1e3), "unit": "rays/s",
               "h2d_bytes_per_step": V * 136, "d2h_bytes_per_step": V * W_IMG * H_IMG * 4,
               "path": "merf_render_host_async per step (C ABI: render into a scene-owned device buffer, "
                       "copy to pinned host memory on the scene's copy stream, overlapped with the next "
                       "step's render) + merf_host_wait; host wall clock from the first call to the last "
                       "frame in host memory"}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(sc, orbit_cameras(N_ORBIT, indices=[0, 64, 128, 192]), sample_stride=1)
        n_ray_timed = rays_per_step * args.steps
        line = {
            "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "orbit1080p_paper_scale_merf" + ("_dense_ablation" if args.dense else "")
                        + ("_mlp_ffma_ablation" if getattr(args, "mlp_ffma", False) else "")
                                   + ("_spherical_contraction" if args.spherical else "")
                                   + ("_persistent_fp32" if getattr(args, "sph_persistent", False) else ""),
                       "views_per_rank_per_step": V, "W": W_IMG, "H": H_IMG,
                       "scene": {k: info[k] for k in ("L", "R", "level_res", "n_blocks", "device_bytes")},
                       "vram": vram,
                       "block_fraction": info["n_blocks"] / (info["L"] // 8) ** 3 if info["L"] else None,
                       "finest_occupancy_fraction": occ_frac,
                       "l2": "no flush: inputs (scene %.0f MB) larger than the 126 MB L2; each step renders "
                             "different orbit views" % (info["device_bytes"] / 1e6),
                       "parallelism": f"views sharded over {world} rank(s), scene replicated, "
                                      "NCCL frame gather to rank 0",
                       "tile_order": ("raster" if V > 4 or os.environ.get("MERF_TILE_ORDER") == "raster" else
                                      "frame-sequence history: the previous step's tile durations (other views)"),
                       "dtype_detail": "u8 features; fp64 ray setup; int32 lattice; interpolation with 16-bit "
                                       "fixed-point weights (dp2a integer sums, exact partition); fp32 decode, "
                                       "composite and MLP accumulation; MLP operands split-fp16 mma.sync"},
            "fps": value / (W_IMG * H_IMG),
            "fps_per_gpu": value / (W_IMG * H_IMG) / world,
            "samples_per_sec": n_eval * world / (ms / 1e3),
            "mean_evaluated_samples_per_ray": n_eval / n_ray_timed,
            "density_only_fraction": n_donly / max(n_eval, 1),
            "mean_skips_per_ray": n_skip / n_ray_timed,
            "mean_segments_per_ray": n_seg / n_ray_timed,
            "segments_per_region": dict(zip(["core", "+x", "-x", "+y", "-y", "+z", "-z"], region_segs)),
            "rank_ms": rank_ms,
            "gather": ({"path": "libmerf merf_gather_frames (grouped ncclSend/ncclRecv to rank 0 on a side "
                                "stream, overlapped with the next step's render)",
                        "bytes_per_step": rays_per_step * 4 * (world - 1), "verified": gather_check}
                       if gathering else None),
            "rank_imbalance": max(rank_ms) / (sum(rank_ms) / len(rank_ms)),
            "gather_gbs": achieved,
            "roofline": roofline,
            "roofline_issue": issue_roofline(roofline["avg_launch_ms"], (clk or {}).get("sm_mhz") or 0,
                                             torch.cuda.get_device_properties(local).multi_processor_count),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": kt["setup_launches"] + kt["march_launches"] + kt["shade_launches"],
            "clocks": clk,
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    scene.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
