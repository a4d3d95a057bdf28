#!/usr/bin/env python
"""Throughput bench of the multi-camera RGB-D Gaussian-splat render path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg1]

--gpus N > 1 without a torchrun environment re-launches itself under torch.distributed.run
(N ranks, 127.0.0.1); under torchrun, WORLD_SIZE must equal N.

cfg0-cfg3: a step is one frame of the BASELINE config (default cfg1, the metric's
configuration: a 1M-Gaussian SH3 background + 4 x 20k object nodes with fresh random rigid
poses, rendered by 5 cameras at 640x480 into RGB + depth + accumulated alpha). Under N > 1
every rank renders its own environment's frame (weak scaling, no data-path collective).
cfg4 (BASELINE config 4): a step is the whole 512-environment x 5-camera batch, split over the
ranks by environment; every rank renders its environments in chunks of <= 64 (config-2-sized
launches) straight into rank 0's gathered output over NVLink peer memory (--gather p2p, the
default: the compositing kernel's epilogue is the gather), or sends chunk j to rank 0 with grouped
NCCL point-to-point while chunk j+1 renders (--gather nccl); shard.ChunkGather. value is box-wide
camera-frames/s (strong scaling).
The timed region is bracketed by a barrier + synchronize on both sides and the elapsed device
time (CUDA events on the renderer's stream) is the max over ranks.

value  : camera-frames/s over all ranks, scene resident in HBM, outputs left in HBM.
e2e    : the same metric through the public API with host buffers: per step the node/camera
         tables go host->device and the 20 B/px RGB-D targets come back device->host into
         pinned memory (gsim_gpu_render), one host thread per renderer context.
roofline / cpu_baseline: see DESIGN.md §5.
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
PAPER_CAMERA_FRAMES_PER_S = 650.0 * 5  # BASELINE.md, stricter unit reading (one GPU)
FNV_SEED = 1469598103934665603


def peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def machine_descriptor() -> str:
    """bench.cpp:79-96: first /proc/cpuinfo model name + hardware threads."""
    model = "unknown-cpu"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{model} ({os.cpu_count() or 1} hw threads)"


class ClockSampler:
    """SM clock + throttle reasons sampled every ~1 ms through NVML during the timed region
    (nvidia-smi at 100 ms when NVML is unavailable)."""
    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.stop_ev = threading.Event()
        self.thread = None
        self.nvml = None

    SMI_QUERY = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")

    def _start_smi(self):
        try:
            fd, self.smi_path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.smi = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.SMI_QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.smi_path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.smi = None

    def _stop_smi(self) -> dict | None:
        if getattr(self, "smi", None) is None:
            return None
        time.sleep(0.25)
        self.smi.terminate()
        try:
            self.smi.wait(timeout=5)
        except Exception:
            self.smi.kill()
        rows = [[x.strip() for x in ln.split(",")] for ln in Path(self.smi_path).read_text().splitlines()]
        os.unlink(self.smi_path)
        rows = [r for r in rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        sm = [float(r[1]) for r in rows]
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)),
                "sm_max_mhz": max(float(r[2]) for r in rows), "reasons": reasons,
                "samples": len(rows), "source": "nvidia-smi, 100 ms"}

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = self.device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[self.device])
                except ValueError:
                    pass
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nvml = (pynvml, h)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
            self._start_smi()
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        pynvml, h = self.nvml
        while not self.stop_ev.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.001)

    def stop(self) -> dict | None:
        if self.nvml is None:
            return self._stop_smi()
        self.stop_ev.set()
        self.thread.join(timeout=2)
        pynvml, _ = self.nvml
        if not self.rows:
            return None
        sm = [r[0] for r in self.rows]
        reasons = sorted(name for name, attr in self.NAMES.items()
                         if any(r[1] & getattr(pynvml, attr, 0) for r in self.rows))
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)),
                "sm_max_mhz": float(self.max_mhz), "reasons": reasons, "samples": len(self.rows),
                "source": "nvml, ~1 ms"}


# ---- byte models ----------------------------------------------------------------

def survey_bytes(stats: dict, n_unique: int, n_obj: int, sh_degree: int, n_cams: int,
                 slots_per_cam: float, pixels: int) -> dict:
    """SURVEY.md §8(d) algorithmic bytes of one step (a reference-style pipeline that sorts the
    P pairs on 46-bit keys; fp32 records of 40 B): the model roofline.achieved uses."""
    V, P, K = stats["visible"], stats["pairs"], stats["consumed"]
    passes = math.ceil(46 / 8)
    return {
        "pose": 56 * n_obj,
        "preprocess": (44 + 12 * (sh_degree + 1) ** 2) * n_unique + 48 * V,
        "scan": 12 * n_cams * slots_per_cam,
        "duplicate": 16 * V + 12 * P,
        "sort": passes * 24 * P + 8 * P,
        "ranges": 8 * P,
        "raster": 44 * K + 20 * pixels,
    }


def stage_bytes(stats: dict, n_prims: int, sh_degree: int, pixels: int, n_cams: int) -> dict:
    """Minimum HBM bytes each stage of OUR pipeline moves for one step (its own layout)."""
    S, V, P, K = stats["slots"], stats["visible"], stats["pairs"], stats["consumed"]
    passes = stats["depth_passes"]
    sh_bytes = 12 * (sh_degree + 1) ** 2
    return {
        # scene read once per batch (f64 geometry 88 B + fp32 SH) + 48 B record, 4 B key and
        # 4 B rect per visible slot, 4 B key per culled slot
        "preprocess": (88 + sh_bytes) * n_prims + 52 * V + 4 * S,
        # histogram reads S keys; pass 1 reads S keys, writes V (key, slot); middle passes read
        # and write 8 B; the last pass reads 8 B, writes the 4 B slot and gathers + writes the rect
        "depth_sort": 4 * S + 4 * S + 8 * V + (passes - 2) * 16 * V + 16 * V,
        "binning": 4 * V,
        # recount V rects + V rects and slots for the placement, P record slots written
        "scatter": 12 * V + 4 * P,
        # 4 B list entry + 40 B record per consumed pair, 20 B per output pixel
        "raster": 44 * K + 20 * pixels,
    }


def load_profile_json(name: str, config: str, stage: str):
    """Per-stage figure from a committed ncu summary under profiles/, for THIS config only."""
    p = ROOT / "profiles" / name
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(config, {}).get(stage)
    except Exception:
        return None


# ---- our arm ------------------------------------------------------------------------------------

def run_ours(args, rank, world, local):
    import torch
    from paper_2507_21981_b200 import Context, RenderTarget
    from paper_2507_21981_b200.scenes import CONFIGS

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.config == "cfg4":
        return run_cfg4(args, rank, world, local, dist)
    w = CONFIGS[args.config](seed=1000 + rank)  # each rank renders its own environment(s)
    # --contexts K: K renderer contexts (each its own stream and workspaces) take frames in
    # turn, so consecutive frames overlap on the GPU. The e2e leg drives each from its own host
    # thread, and a waiting thread spins: keep ranks x contexts within the host's cores.
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    n_ctx = max(1, min(args.contexts, max(2, cores // max(local_world, 1) - 1)))
    if len(w.cameras) > 32:
        # config 2: one context's workspaces are ~36 GB and its launches fill the GPU; a second
        # context overlaps one batch's host copies with the next batch (measured: e2e 4,223 ->
        # 5,866, value 6,123 -> 6,225; a third adds nothing), when HBM holds both
        free = torch.cuda.mem_get_info(local)[0]
        n_ctx = min(n_ctx, 2 if free > 2 * (48 << 30) else 1)
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
        return ctxs[k].render_device(scenes[k], w.frame_nodes(i, seed=rank), w.cameras, None,
                                     outs[k].data_ptr())

    for i in range(args.warmup):
        step(i)
    for c in ctxs:
        c.synchronize()

    # ---- timed region: device-resident inputs and outputs -------------------------------
    # Frames are enqueued back to back: render_device is asynchronous (the pair-count check of
    # frame k is completed by the call for frame k+1), so the host builds the next frame's
    # plan while the GPU renders.
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
    n_prof = min(args.steps, 50)
    for i in range(n_prof):
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

    # first timed frame again (renders are deterministic): its image hash, bench.cpp:121-137
    first = ctx.render(scene, w.frame_nodes(args.warmup, seed=rank), w.cameras)
    h = FNV_SEED
    for tg in first:
        h = tg.hash(h)
    first_hash = f"{h:016x}"

    # ---- e2e: public API, host buffers (pinned), H2D + D2H inside the timed region ------
    e2e = None
    # The e2e legs run a steady-state window of at least 200 frames even when K is small: with
    # 5 threads x K/5 synchronous frames each, a 20-frame run is mostly pipeline fill and drain.
    # The window is reported (e2e.steps); the device-resident value above times exactly K.
    e2e_steps = max(args.steps, 200)
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

        # The synchronous API leaves a context idle while its calling thread waits for the copies
        # and builds the next call, so the e2e leg runs one more context (and thread) than the
        # device-resident leg (measured at config 1: 5 -> 6 contexts, e2e +1%, value -2%).
        n_e2e = args.e2e_contexts if args.e2e_contexts > 0 else (
            min(len(ctxs) + 1, max(2, cores // max(local_world, 1) - 1)) if len(w.cameras) <= 32 else len(ctxs))
        e_ctxs = list(ctxs)
        e_scenes = list(scenes)
        while len(e_ctxs) < n_e2e:
            e_ctxs.append(Context(local))
            e_scenes.append(e_ctxs[-1].upload(w.field))
        ctxs, scenes = e_ctxs[:n_e2e], e_scenes[:n_e2e]
        targets = [host_targets() for _ in ctxs]
        for k, c in enumerate(ctxs):
            for i in range(2):
                c.render(scenes[k], w.frame_nodes(i, seed=rank), w.cameras, None, targets[k])
        io = [[0, 0] for _ in ctxs]
        # every step's inputs (node poses, camera table) are prepared before the timed region as
        # the C tables the API takes; the render call itself still copies them host -> device
        from paper_2507_21981_b200.api import _cams_array, _nodes_array
        prebuilt = os.environ.get("BENCH_E2E_PYTHON_INPUTS") != "1"
        step_nodes = [_nodes_array(w.frame_nodes(10_000 + i, seed=rank)) if prebuilt else None
                      for i in range(e2e_steps)]
        cam_table = _cams_array(w.cameras) if prebuilt else w.cameras

        def worker(k):
            for i in range(k, e2e_steps, len(ctxs)):
                nodes_i = step_nodes[i] if prebuilt else w.frame_nodes(10_000 + i, seed=rank)
                ctxs[k].render(scenes[k], nodes_i, cam_table, None, targets[k])
            st = ctxs[k].stats()  # bytes copied by the context's last call (every call the same)
            io[k] = [st["h2d_bytes"], st["d2h_bytes"]]

        def timed_threads(fn):
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            torch.cuda.synchronize()
            threads = [threading.Thread(target=fn, args=(k,)) for k in range(len(ctxs))]
            for th in threads:
                th.start()
            for th in threads:
                th.join()
            e1.record(stream)
            e1.synchronize()
            te = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{local}")
            if dist:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            return float(te.item())

        te = timed_threads(worker)
        h2d, d2h = io[0]
        e2e = {"value": round(world * e2e_steps * n_cams / (te / 1e3), 2), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(te / e2e_steps, 4), "contexts": len(ctxs), "steps": e2e_steps,
               "api": "gsim_gpu_render (host float targets, pinned)"}

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

        enc_nodes = [_nodes_array(w.frame_nodes(20_000 + i, seed=rank)) if prebuilt else None
                     for i in range(e2e_steps)]

        def worker_enc(k):
            for i in range(k, e2e_steps, len(ctxs)):
                nodes_i = enc_nodes[i] if prebuilt else w.frame_nodes(20_000 + i, seed=rank)
                ctxs[k].render_encoded(scenes[k], nodes_i, cam_table, None, eo, out=blobs[k])
            st = ctxs[k].stats()
            io_enc[k] = [st["h2d_bytes"], st["d2h_bytes"]]

        te2 = timed_threads(worker_enc)
        e2e["encoded"] = {"value": round(world * e2e_steps * n_cams / (te2 / 1e3), 2),
                          "unit": UNIT, "h2d_bytes_per_step": int(io_enc[0][0]),
                          "d2h_bytes_per_step": int(io_enc[0][1]),
                          "outputs": "rgb8 sRGB + alpha8 + depth16 mm + depth PFM (10 B/px)"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    pk, pk_kind = peaks()
    per_step_ms = {k: v / n_prof for k, v in stage_ms.items()}
    bytes_ = stage_bytes(stats, w.field.size(), w.field.sh_degree, pixels, n_cams)
    dominant = max(per_step_ms, key=per_step_ms.get)
    total_ms = sum(per_step_ms.values())
    dom_ms = per_step_ms[dominant]
    achieved = bytes_[dominant] / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    n_obj = sum(n.range[1] - n.range[0] for k, n in enumerate(w.nodes) if k in set(w.object_nodes))
    sv = survey_bytes(stats, w.field.size(), n_obj, w.field.sh_degree, n_cams,
                      stats["slots"] / max(n_cams, 1), pixels)
    sv_total = sum(sv.values())
    ms_step = elapsed_ms / args.steps
    roofline = {
        "bound": "hbm", "kernel": "raster_kernel" if dominant == "raster" else dominant,
        "stage": dominant,
        "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "peak_kind": pk_kind, "unit": "GB/s",
        "frac": round(achieved / pk["hbm_gbs"], 4),
        "traffic": load_profile_json("traffic.json", args.config, dominant),
        "algorithmic_bytes": int(bytes_[dominant]),
        "bytes_model": ("SURVEY 8(d): 44 B per consumed pair (4 B index + 40 B record) x K + "
                        "20 B per pixel x X" if dominant == "raster" else "DESIGN.md §5 stage model"),
        "counts": {"K_consumed_pairs": stats["consumed"], "X_pixels": pixels},
        "stage_ms": round(dom_ms, 4),
        "share_of_step": round(dom_ms / total_ms, 3) if total_ms else None,
        "stages_ms": {k: round(v, 4) for k, v in per_step_ms.items()},
        "stages_gbs": {k: round(bytes_[k] / (per_step_ms[k] / 1e3) / 1e9, 1) if per_step_ms[k] > 0 else None
                       for k in per_step_ms},
        "sector_model": {  # 48 B records fetched as two 32 B sectors: what K4 really reads
            "bytes": int(68 * stats["consumed"] + 20 * pixels),
            "frac": round((68 * stats["consumed"] + 20 * pixels) / (dom_ms / 1e3) / 1e9 / pk["hbm_gbs"], 4)
            if dominant == "raster" and dom_ms > 0 else None},
        # the whole step against the SURVEY 8(d) pipeline model (a reference-style pipeline
        # that sorts the P pairs): its HBM floor over our measured step time
        "survey_pipeline": {"bytes": int(sv_total), "floor_ms": round(sv_total / pk["hbm_gbs"] / 1e6, 4),
                            "frac": round(sv_total / pk["hbm_gbs"] / 1e6 / ms_step, 4) if world == 1 else None,
                            "stages": {k: int(v) for k, v in sv.items()}},
    }
    # The rasterizer is FP32-issue-bound, not HBM-bound: its warp instructions
    # per frame (ncu, same config) over the live stage time, against the issue peak of 4 warp
    # instructions per SM per cycle at the sampled SM clock.
    inst = load_profile_json("instructions.json", args.config, dominant)
    if inst and dom_ms > 0:
        sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
        n_sms = torch.cuda.get_device_properties(local).multi_processor_count
        peak_ipc = n_sms * 4 * sm_mhz * 1e6
        ach = inst / (dom_ms / 1e3)
        roofline["issue"] = {"kernel": dominant, "warp_instructions": int(inst),
                             "achieved": round(ach / 1e9, 1), "peak": round(peak_ipc / 1e9, 1),
                             "unit": "G warp-instr/s", "frac": round(ach / peak_ipc, 4)}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "weak",
        # the paper's "650 FPS" for 5 cameras at 640x480 on ONE GPU (RTX 6000 Ada),
        # gated on the stricter reading 650 five-camera frames/s = 3250 camera-frames/s; per GPU
        "vs_baseline": round(value / world / PAPER_CAMERA_FRAMES_PER_S, 3) if args.config == "cfg1" else None,
        "vs_baseline_basis": ("device-resident value per GPU / paper 650 five-camera frames/s "
                              "= 3250 camera-frames/s (BASELINE.md)"),
        "dtype": "f32 (f64 geometry)", "data": "synthetic (seeded, BASELINE.json distributions)",
        "config": {"workload": f"{args.config}: {w.description}", "gaussians": w.field.size(),
                   "sh_degree": w.field.sh_degree, "cameras_per_rank": n_cams,
                   "resolution": f"{w.cameras[0].width}x{w.cameras[0].height}",
                   "parallelism": (f"env-sharded x{world} (replicated background, "
                                   "no data-path collective)"),
                   "l2": "inputs larger than L2 (scene 300 MB, per-frame working set > 500 MB); no flush",
                   "seed": "1000+rank", "contexts_per_gpu": n_ctx},
        "five_camera_frames_per_s": round(value / n_cams, 2),
        "e2e": e2e,
        "gpu_launches": int(launches),
        "first_frame_hash": first_hash,
        "machine": machine_descriptor(),
        "stats_last_step": {k: stats[k] for k in ("slots", "visible", "pairs", "consumed", "tiles",
                                                  "depth_passes", "groups")},
        "roofline": roofline,
        "clocks": clocks,
        "wall_s_timed": round(wall, 4),
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_cfg4(args, rank, world, local, dist):
    """BASELINE config 4: 512 envs x 5 cameras split by environment over the ranks, rendered in
    <= 64-env chunks, frames gathered to rank 0 (shard.ChunkGather) behind the next chunk."""
    import torch
    from paper_2507_21981_b200 import Context
    from paper_2507_21981_b200.scenes import config4_rank
    from paper_2507_21981_b200.shard import ChunkGather, env_range

    dev = torch.device("cuda", local)
    n_envs = args.envs
    b, e = env_range(n_envs, rank, world)
    ctx = Context(local)
    t0 = time.perf_counter()
    r = config4_rank(ctx, b, e, seed=1000)
    setup_s = time.perf_counter() - t0
    cams_per_env = r.cams_per_env
    px_per_env = sum(c.width * c.height for c in r.cameras[:cams_per_env])
    fpe = 5 * px_per_env
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    gather = ChunkGather(n_envs, fpe, args.chunk_envs, dev, rank=rank, world=world, dst=0,
                         mode=args.gather)
    chunk_cams = [r.camera_table(cb, ce) for cb, ce in gather.my_chunks]

    def step(i, sums=None):
        nodes = r.frame_nodes(i)
        with torch.cuda.stream(stream):
            for j in range(len(gather.my_chunks)):
                tgt = gather.target(j)
                ctx.render_device(r.scene, nodes, chunk_cams[j], None, tgt.ptr)
                if sums is not None:  # exact per-env checksums of what this rank sends
                    cb, ce = gather.my_chunks[j]
                    local = tgt.local
                    if local is None:  # stored in rank 0's memory: re-render (deterministic)
                        local = torch.empty((ce - cb) * fpe, dtype=torch.float32, device=dev)
                        ctx.render_device(r.scene, nodes, chunk_cams[j], None, local.data_ptr())
                    sums[cb:ce] = local.view(ce - cb, fpe).view(torch.int32).sum(1, dtype=torch.int64)
                gather.send(j)
            gather.finish()

    for i in range(args.warmup):
        step(i)
    ctx.synchronize()
    torch.cuda.synchronize()
    launches_before = ctx.stats()["launches_total"]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    ev0.record(stream)
    t_wall = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    clocks = sampler.stop()
    launches = ctx.stats()["launches_total"] - launches_before
    t = torch.tensor([ev0.elapsed_time(ev1)], device=dev)
    if dist:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    cam_frames = n_envs * cams_per_env
    value = args.steps * cam_frames / (elapsed_ms / 1e3)
    # One more step with checksums: rank 0's gathered blocks must equal, bit for bit, what every
    # rank rendered (exact integer sums of the float bits per environment).
    sums = torch.zeros(n_envs, dtype=torch.int64, device=dev)
    step(args.warmup + args.steps, sums)
    torch.cuda.synchronize()
    if dist:
        dist.all_reduce(sums)  # env ranges are disjoint: the sum assembles every rank's part
    check = None
    if rank == 0:
        got = gather.out.view(n_envs, fpe).view(torch.int32).sum(1, dtype=torch.int64)
        check = {"envs": n_envs, "mismatched_envs": int((got != sums).sum().item())}
        if world == 1:
            # batch == separate renders: env 3's cameras alone reproduce its block of the batch
            e3 = min(3, n_envs - 1)
            one = torch.empty(fpe, dtype=torch.float32, device=dev)
            ctx.render_device(r.scene, r.frame_nodes(args.warmup + args.steps),
                              r.camera_table(e3, e3 + 1), None, one.data_ptr())
            ctx.synchronize()
            check["env_batch_equals_single"] = bool(torch.equal(one, gather.out[e3 * fpe:(e3 + 1) * fpe]))
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(elapsed_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 (f64 geometry)", "data": "synthetic (seeded, BASELINE.json distributions)",
            "config": {"workload": f"cfg4: {n_envs} envs x {cams_per_env} cams 640x480, shared 1M SH3 "
                                   "background replica per GPU + each env's 4x20k objects",
                       "envs_per_rank": e - b, "chunk_envs": args.chunk_envs,
                       "gaussians_per_rank": r.scene.size,
                       "parallelism": "one rank: every environment rendered into the gathered output"
                       if world == 1 else f"env-sharded x{world}, frames gathered to rank 0 " + (
                           "(fused: the compositing kernels store into rank 0's HBM over NVLink "
                           "peer memory)" if args.gather == "p2p" else
                           "(grouped NCCL P2P, overlapped with the next chunk)"),
                       "gather_bytes_per_step": int(gather.bytes_to_dst * 4),
                       "l2": "inputs larger than L2; no flush", "seed": 1000},
            "gpu_launches": int(launches),
            "gather_check": check,
            "gather_mode": gather.mode if world > 1 else None,
            "gather_fallback": gather.fallback,
            "setup_s": round(setup_s, 1),
            "machine": machine_descriptor(),
            "clocks": clocks,
            "wall_s_timed": round(wall, 3),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


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
           "kind": kind, "host_threads_configured": cores, "machine": machine_descriptor(),
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
    cfg = args.config if args.config != "cfg4" else "cfg2"  # cfg4 = cfg2-shaped envs
    w = CONFIGS[cfg](seed=1000)
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
    render(w.frame_nodes(0), w.cameras[:5])
    per_frame = time.perf_counter() - t0
    cams = w.cameras[:5]
    if per_frame * (args.steps + args.warmup) > 150:
        cams = w.cameras[:1]
    if kind == "reference":
        busy = min(len(cams), cores) if len(cams) > 1 else cores
    for i in range(args.warmup):
        render(w.frame_nodes(i + 1), cams)
    first_hash = None
    hasher = Oracle()  # hash_target restated (oracle pinned to hash.hpp)
    t0 = time.perf_counter()
    for i in range(args.steps):
        targets = render(w.frame_nodes(args.warmup + i + 1), cams)
        if i == 0:  # bench.cpp:121-137 (hashing stays inside the timed loop, as there)
            h = FNV_SEED
            for tg in targets:
                h = hasher.hash_target(tg, h)
            first_hash = f"{h:016x}"
    dt = time.perf_counter() - t0
    value = args.steps * len(cams) / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {w.description}", "gaussians": w.field.size(),
                   "cameras_per_step": len(cams)},
        "first_frame_hash": first_hash,
        "machine": machine_descriptor(),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": busy, "kind": kind,
                         "host_threads_configured": cores, "machine": machine_descriptor(),
                         "sample": f"{args.steps} steps x {len(cams)} camera(s) of {w.name}"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if kind == "reference":
        rf.close()
    print(json.dumps(line), flush=True)


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"], default="cfg1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-contexts", type=int, default=0,
                    help="renderer contexts (host threads) of the e2e legs; 0: --contexts + 1")
    ap.add_argument("--contexts", type=int, default=5,
                    help="renderer contexts taking frames in turn (frame-level overlap)")
    ap.add_argument("--envs", type=int, default=512, help="cfg4: environments per step (box-wide)")
    ap.add_argument("--chunk-envs", type=int, default=64, help="cfg4: environments per launch")
    ap.add_argument("--gather", choices=["p2p", "nccl"], default="p2p",
                    help="cfg4, N > 1: frames stored into rank 0's HBM by the compositing kernels "
                         "over peer memory (p2p) or sent after each chunk with NCCL (nccl)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    if args.config == "cfg4" and args.steps == 400:
        args.steps = 3  # a cfg4 step is 2560 camera-frames
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
