#!/usr/bin/env python
"""Throughput bench of the multi-camera RGB-D Gaussian-splat render path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg1]

A step is one frame of BASELINE config 1 (the metric's configuration): a 1M-Gaussian SH3
background + 4 x 20k object nodes with fresh random rigid poses, rendered by 5 cameras at
640x480 into RGB + depth + accumulated alpha. Under torchrun (N > 1) every rank renders its own
environment's frame (weak scaling, no data-path collective); the timed region is bracketed by a
barrier + synchronize on both sides and the elapsed device time is the max over ranks.

value  : camera-frames/s over all ranks, scene resident in HBM, outputs left in HBM
         (CUDA events on the renderer's stream).
e2e    : the same metric through the public API with host buffers: per step the node/camera
         tables go host->device and the 20 B/px RGB-D targets come back device->host into
         pinned memory (gsim_gpu_render), one host thread per renderer context.
roofline / cpu_baseline: see DESIGN.md §Measurement.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RGB-D camera-frames/sec (5 cams 640x480, 1M Gaussians)"
UNIT = "camera-frames/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return PEAKS_FALLBACK, "fallback"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---- algorithmic byte model ----------------------------------------

def stage_bytes(stats: dict, n_prims: int, sh_degree: int, pixels: int, n_cams: int) -> dict:
    """Minimum HBM bytes each stage of OUR pipeline must move for one step."""
    S, V, P, K = stats["slots"], stats["visible"], stats["pairs"], stats["consumed"]
    sh_bytes = 12 * (sh_degree + 1) ** 2
    M = stats["tiles"] // max(1, n_cams) * stats["chunks"]  # count-matrix entries
    return {
        # scene read once per batch (f64 geometry 88 B + fp32 SH) + 48 B record, 4 B key and
        # 4 B rect per visible slot, 4 B key per culled slot
        "preprocess": (88 + sh_bytes) * n_prims + 52 * V + 4 * S,
        # histogram reads S keys; pass 1 reads S keys, writes V (key, slot); passes 2-3 read
        # and write 8 B; pass 4 reads 8 B, writes the 4 B slot and gathers + writes the 4 B rect
        "depth_sort": 4 * S + 4 * S + 8 * V + 2 * 16 * V + 16 * V,
        # count: V sorted rects; column scan reads the count matrix twice and writes it once
        "binning": 4 * V + 12 * M,
        # scatter: V rects (recount) + V rects and slots (placement), column prefixes, P record
        # slots written
        "scatter": 12 * V + 4 * M + 4 * P,
        # K list entries + 48 B records (2 sectors: 64 B) + 20 B/px outputs
        "raster": 4 * K + 64 * K + 20 * pixels,
    }


PAPER_CAMERA_FRAMES_PER_S = 650.0 * 5  # BASELINE.md, stricter unit reading


def run_ours(args, rank, world, local):
    import torch
    from paper_2507_21981_b200 import Context, RenderTarget
    from paper_2507_21981_b200.scenes import CONFIGS

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = CONFIGS[args.config](seed=1000 + rank)  # each rank renders its own environment(s)
    # --contexts K: K renderer contexts (each its own stream and workspaces) take frames in
    # turn, so consecutive frames overlap on the GPU. The e2e leg drives each from its own host
    # thread, and a waiting thread spins: keep ranks x contexts within the host's cores.
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    n_ctx = max(1, min(args.contexts, max(2, cores // max(local_world, 1) - 1)))
    ctxs = [Context(local) for _ in range(n_ctx)]
    scenes = [c.upload(w.field) for c in ctxs]
    streams = [torch.cuda.ExternalStream(c.stream, device=torch.device("cuda", local)) for c in ctxs]
    outs = [torch.empty(sum(5 * c.width * c.height for c in w.cameras), dtype=torch.float32,
                        device=f"cuda:{local}") for _ in ctxs]
    ctx, scene, stream = ctxs[0], scenes[0], streams[0]
    n_cams = len(w.cameras)
    pixels = w.pixels()

    def step(i):
        k = i % len(ctxs)
        ptr = ctxs[k].render_device(scenes[k], w.frame_nodes(i, seed=rank), w.cameras, None,
                                    outs[k].data_ptr())
        if args.gather and dist:
            # BASELINE config 4: the frame (every rank's environment) goes to rank 0 over NCCL
            from paper_2507_21981_b200.shard import gather_frames
            torch.cuda.current_stream().wait_stream(streams[k])
            gather_frames(outs[k], world, outs[k].numel(), dst=0)
            streams[k].wait_stream(torch.cuda.current_stream())
        return ptr

    for i in range(args.warmup):
        step(i)
    ctx.synchronize()

    # ---- timed region: device-resident inputs and outputs -------------------------------
    # Frames are enqueued back to back: render_device is asynchronous (the pair-count check of
    # frame k is completed by the call for frame k+1), so the host builds the next frame's
    # plan while the GPU renders.
    for c in ctxs:
        c.synchronize()
    launches_before = sum(c.stats()["launches_total"] for c in ctxs)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    ev0.record(stream)
    for s in streams[1:]:
        s.wait_stream(stream)
    t_wall = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    for s in streams[1:]:
        stream.wait_stream(s)
    ev1.record(stream)
    ev1.synchronize()
    for c in ctxs:
        c.synchronize()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    clocks = sampler.stop()
    launches = sum(c.stats()["launches_total"] for c in ctxs) - launches_before

    # Stage times: the same frames again with per-stage CUDA events on the renderer's stream
    # (profiling mode reads them back after every frame, so this loop is not the timed one).
    ctx.set_profiling(True)
    stage_ms = {k: 0.0 for k in ("preprocess", "depth_sort", "binning", "scatter", "raster")}
    stats = None
    for i in range(args.steps):
        ctx.render_device(scene, w.frame_nodes(args.warmup + i, seed=rank), w.cameras, None,
                          outs[0].data_ptr())
        stats = ctx.stats()
        for k in stage_ms:
            stage_ms[k] += stats["ms_" + k]
    ctx.set_profiling(False)
    elapsed_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([elapsed_ms], device=f"cuda:{local}")
    if dist:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    value = world * args.steps * n_cams / (elapsed_ms / 1e3)

    # ---- e2e: public API, host buffers (pinned), H2D + D2H inside the timed region ------
    e2e = None
    if not args.no_e2e:
        # One host thread per context (the ctypes call releases the GIL): while one context
        # copies its frame to the host the other renders the next one, which is how a caller
        # of the synchronous API gets throughput.
        def host_targets():
            out = []
            for c in w.cameras:
                rgb = torch.empty((c.height, c.width, 3), dtype=torch.float32, pin_memory=True).numpy()
                dep = torch.empty((c.height, c.width), dtype=torch.float32, pin_memory=True).numpy()
                alp = torch.empty((c.height, c.width), dtype=torch.float32, pin_memory=True).numpy()
                out.append(RenderTarget(rgb, dep, alp))
            return out

        targets = [host_targets() for _ in ctxs]
        for k, c in enumerate(ctxs):
            for i in range(2):
                c.render(scenes[k], w.frame_nodes(i, seed=rank), w.cameras, None, targets[k])
        io = [[0, 0] for _ in ctxs]

        def worker(k):
            for i in range(k, args.steps, len(ctxs)):
                ctxs[k].render(scenes[k], w.frame_nodes(10_000 + i, seed=rank), w.cameras, None,
                               targets[k])
                st = ctxs[k].stats()
                io[k] = [st["h2d_bytes"], st["d2h_bytes"]]

        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        torch.cuda.synchronize()
        threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(ctxs))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        e1.record(stream)
        e1.synchronize()
        h2d, d2h = io[0]
        te = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{local}")
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * args.steps * n_cams / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(te.item()) / args.steps, "contexts": len(ctxs)}

        # Same loop through render_encoded: the compositing kernel writes
        # the reference CLI's outputs (sRGB RGB8, alpha8, 16-bit mm depth, PFM depth) and only
        # those bytes cross PCIe.
        from paper_2507_21981_b200 import EncodeOptions
        eo = EncodeOptions()
        blob_bytes = sum(eo.bytes_per_camera(c.width, c.height) for c in w.cameras)
        blobs = [torch.empty(blob_bytes, dtype=torch.uint8, pin_memory=True).numpy() for _ in ctxs]
        for k, c in enumerate(ctxs):
            c.render_encoded(scenes[k], w.frame_nodes(0, seed=rank), w.cameras, None, eo, out=blobs[k])
        io_enc = [[0, 0] for _ in ctxs]

        def worker_enc(k):
            for i in range(k, args.steps, len(ctxs)):
                ctxs[k].render_encoded(scenes[k], w.frame_nodes(20_000 + i, seed=rank), w.cameras,
                                       None, eo, out=blobs[k])
                st = ctxs[k].stats()
                io_enc[k] = [st["h2d_bytes"], st["d2h_bytes"]]

        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        torch.cuda.synchronize()
        threads = [threading.Thread(target=worker_enc, args=(k,)) for k in range(len(ctxs))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        e1.record(stream)
        e1.synchronize()
        te2 = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{local}")
        if dist:
            dist.all_reduce(te2, op=dist.ReduceOp.MAX)
        e2e["encoded"] = {"value": world * args.steps * n_cams / (float(te2.item()) / 1e3),
                          "unit": UNIT, "h2d_bytes_per_step": int(io_enc[0][0]),
                          "d2h_bytes_per_step": int(io_enc[0][1]),
                          "outputs": "rgb8 sRGB + alpha8 + depth16 mm + depth PFM (10 B/px)"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    pk, pk_kind = peaks()
    per_step_ms = {k: v / args.steps for k, v in stage_ms.items()}
    bytes_ = stage_bytes(stats, w.field.size(), w.field.sh_degree, pixels, n_cams)
    dominant = max(per_step_ms, key=per_step_ms.get)
    achieved = bytes_[dominant] / (per_step_ms[dominant] / 1e3) / 1e9 if per_step_ms[dominant] > 0 else 0.0
    total_ms = sum(per_step_ms.values())
    traffic = load_traffic(dominant)
    roofline = {
        "bound": "hbm", "kernel": dominant, "achieved": round(achieved, 1),
        "peak": pk["hbm_gbs"], "peak_kind": pk_kind, "unit": "GB/s",
        "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": traffic,
        "algorithmic_bytes": int(bytes_[dominant]),
        "share_of_step": round(per_step_ms[dominant] / total_ms, 3) if total_ms else None,
        "stages_ms": {k: round(v, 4) for k, v in per_step_ms.items()},
        "stages_gbs": {k: round(bytes_[k] / (per_step_ms[k] / 1e3) / 1e9, 1) if per_step_ms[k] > 0 else None
                       for k in per_step_ms},
        "pipeline_frac": round(sum(bytes_.values()) / (total_ms / 1e3) / 1e9 / pk["hbm_gbs"], 4)
        if total_ms else None,
    }
    # The rasterizer is FP32-issue-bound, not HBM-bound: its warp instructions
    # per frame (profiles/instructions.json, ncu) over the live stage time, against the issue
    # peak of 4 warp instructions per SM per cycle at the sampled SM clock.
    inst = load_profile_json("instructions.json", dominant)
    if inst and per_step_ms[dominant] > 0:
        sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
        n_sms = torch.cuda.get_device_properties(local).multi_processor_count
        peak_ipc = n_sms * 4 * sm_mhz * 1e6
        ach = inst / (per_step_ms[dominant] / 1e3)
        roofline["issue"] = {"kernel": dominant, "warp_instructions": int(inst),
                             "achieved": round(ach / 1e9, 1), "peak": round(peak_ipc / 1e9, 1),
                             "unit": "G warp-instr/s", "frac": round(ach / peak_ipc, 4)}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(elapsed_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak",
        # the paper's "650 FPS" for 5 cameras at 640x480 (RTX 6000 Ada), gated on the
        # stricter reading 650 five-camera frames/s = 3250 camera-frames/s
        "vs_baseline": round(value / PAPER_CAMERA_FRAMES_PER_S, 3) if args.config == "cfg1" else None,
        "vs_baseline_basis": "paper 650 five-camera frames/s = 3250 camera-frames/s (BASELINE.md)",
        "dtype": "f32 (f64 geometry)", "data": "synthetic",
        "config": {"workload": f"{args.config}: {w.description}", "gaussians": w.field.size(),
                   "sh_degree": w.field.sh_degree, "cameras_per_rank": n_cams,
                   "resolution": f"{w.cameras[0].width}x{w.cameras[0].height}",
                   "parallelism": (f"env-sharded x{world} (replicated background, "
                                   + ("frames gathered to rank 0 over NCCL each step)" if args.gather and world > 1
                                      else "no data-path collective)")),
                   "l2": "inputs larger than L2 (scene 300 MB, per-frame working set > 500 MB); no flush",
                   "seed": "1000+rank", "contexts_per_gpu": len(ctxs)},
        "five_camera_frames_per_s": round(value / n_cams, 2),
        "e2e": e2e,
        "gpu_launches": int(launches),
        "stats_last_step": {k: stats[k] for k in ("slots", "visible", "pairs", "consumed", "tiles",
                                                  "depth_passes", "chunks")},
        "roofline": roofline,
        "clocks": clocks,
        "wall_s_timed": round(wall, 4),
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def load_profile_json(name: str, stage: str):
    """Per-stage figure from a committed ncu summary under profiles/ (None if absent)."""
    p = ROOT / "profiles" / name
    if p.exists():
        try:
            return json.loads(p.read_text()).get(stage)
        except Exception:
            return None
    return None


def load_traffic(stage: str):
    """dram read+write bytes per frame of the stage's kernels from the committed ncu capture."""
    return load_profile_json("traffic.json", stage)


def cpu_baseline(w, budget_s: float) -> dict:
    """The reference CPU renderer (oracle/_ref, compiled from the reference's own sources) on
    a bounded sample of the same workload: whole 5-camera frames through gsim::render with
    set_thread_count(nproc) — the reference keeps min(cameras, threads) threads busy."""
    from oracle.oracle import REF_LIB, Oracle, Ref, cpu_count
    cores = cpu_count()
    if REF_LIB.exists():
        ref = Ref()
        ref.set_threads(cores)
        rf = ref.field(w.field)
        kind = "reference"
        render = lambda nodes: rf.render(nodes, w.cameras)  # noqa: E731
        # several cameras: one busy thread per camera (nested parallel_for runs inline,
        # parallel.cpp:41-43); a single camera parallelises its own loops over every thread
        busy = min(len(w.cameras), cores) if len(w.cameras) > 1 else cores
    else:  # port: our single-threaded C restatement
        orc = Oracle()
        kind = "port"
        render = lambda nodes: orc.render(w.field, nodes, w.cameras)  # noqa: E731
        busy = 1
    frames = 0
    t0 = time.perf_counter()
    while True:
        render(w.frame_nodes(frames))
        frames += 1
        if time.perf_counter() - t0 > budget_s or frames >= 8:
            break
    dt = time.perf_counter() - t0
    one = None
    if kind == "reference":
        # also the single-thread figure (one camera of one frame)
        ref.set_threads(1)
        t1 = time.perf_counter()
        rf.render(w.frame_nodes(frames), w.cameras[:1])
        d1 = time.perf_counter() - t1
        ref.set_threads(cores)
        one = {"value": round(1.0 / d1, 4), "unit": UNIT, "cores": 1,
               "sample": f"1 camera of {w.name} ({d1:.1f} s)"}
        rf.close()
    out = {"value": round(frames * len(w.cameras) / dt, 4), "unit": UNIT, "cores": busy,
           "kind": kind, "host_threads_configured": cores,
           "sample": f"{frames} frame(s) x {len(w.cameras)} cameras of {w.name} ({dt:.1f} s)"}
    if one:
        out["one_thread"] = one
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU renderer on this box's host cores."""
    if rank != 0:
        return
    from paper_2507_21981_b200.scenes import CONFIGS
    from oracle.oracle import REF_LIB, Oracle, Ref, cpu_count
    w = CONFIGS[args.config](seed=1000)
    cores = cpu_count()
    if REF_LIB.exists():
        ref = Ref()
        ref.set_threads(cores)
        rf = ref.field(w.field)
        kind = "reference"
        render = lambda nodes, cams: rf.render(nodes, cams)  # noqa: E731
    else:
        orc = Oracle()
        kind, busy = "port", 1
        render = lambda nodes, cams: orc.render(w.field, nodes, cams)  # noqa: E731
    # bound the run to a few minutes: whole frames if affordable, else one camera per step
    t0 = time.perf_counter()
    render(w.frame_nodes(0), w.cameras)
    per_frame = time.perf_counter() - t0
    cams = w.cameras
    if per_frame * (args.steps + args.warmup) > 150:
        cams = w.cameras[:1]
    if kind == "reference":
        busy = min(len(cams), cores) if len(cams) > 1 else cores
    for i in range(args.warmup):
        render(w.frame_nodes(i + 1), cams)
    t0 = time.perf_counter()
    for i in range(args.steps):
        render(w.frame_nodes(args.warmup + i + 1), cams)
    dt = time.perf_counter() - t0
    value = args.steps * len(cams) / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {w.description}", "gaussians": w.field.size(),
                   "cameras_per_step": len(cams)},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": busy, "kind": kind,
                         "host_threads_configured": cores,
                         "sample": f"{args.steps} steps x {len(cams)} camera(s) of {w.name}"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if kind == "reference":
        rf.close()
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["cfg0", "cfg1", "cfg2", "cfg3"], default="cfg1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--contexts", type=int, default=4,
                    help="renderer contexts taking frames in turn (frame-level overlap)")
    ap.add_argument("--gather", action="store_true",
                    help="N > 1: gather every step's frames to rank 0 (config 4) inside the timed step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
