"""LiDAR scan throughput: GaussianBvh::scan on the GPU vs the reference's
CPU tracer (oracle/_ref) on the BASELINE config-1 scene (1M SH3 background + 4 x 20k objects).

    python tools/bench_lidar.py [--scans 20] [--channels 32] [--step-deg 0.2]

The sensor sits at the scene centre (inside the Gaussian cloud, the worst case: every ray has
candidates all the way out). GPU: wall-clock of complete gsim_gpu_lidar_scan calls (H2D of the
ray table, all kernels, D2H of the returns). CPU: the reference GaussianBvh::build + scan on a
bounded sample of channels, scaled to the full ray count. Prints one JSON line.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2507_21981_b200 import Context  # noqa: E402
from paper_2507_21981_b200.api import LidarModel, RigidTransform  # noqa: E402
from paper_2507_21981_b200.scenes import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scans", type=int, default=20)
ap.add_argument("--channels", type=int, default=32)
ap.add_argument("--step-deg", type=float, default=0.2)
ap.add_argument("--cpu-channels", type=int, default=1)
ap.add_argument("--no-cpu", action="store_true")
ap.add_argument("--trace", type=int, default=0,
                help="also time N arbitrary rays through gsim_gpu_trace_rays (linear BVH)")
a = ap.parse_args()

w = CONFIGS["cfg1"](seed=1000)
nodes = w.frame_nodes(0)
lid = LidarModel(np.radians(np.linspace(-15.0, 15.0, a.channels)), np.radians(a.step_deg), 100.0,
                 RigidTransform((1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0)))
rays = a.channels * lid.azimuth_count()
ctx = Context(0)
scene = ctx.upload(w.field)
scan = ctx.lidar_scan(scene, nodes, lid)  # warm-up
t0 = time.perf_counter()
for _ in range(a.scans):
    scan = ctx.lidar_scan(scene, nodes, lid)
gpu_s = (time.perf_counter() - t0) / a.scans
line = {"metric": "LiDAR scans/s (1M-Gaussian cfg1 scene, sensor at the centre)",
        "gpu_scans_per_s": round(1.0 / gpu_s, 2), "gpu_ms_per_scan": round(gpu_s * 1e3, 3),
        "rays": rays, "returns": int(len(scan["ring"])), "channels": a.channels,
        "azimuth_step_deg": a.step_deg, "gaussians": w.field.size()}
if not a.no_cpu:
    from oracle.oracle import Ref
    ref = Ref()
    import os
    ref.set_threads(os.cpu_count() or 1)
    sub = LidarModel(lid.channels[: a.cpu_channels], lid.azimuth_step, lid.max_range, lid.pose)
    t0 = time.perf_counter()
    ref.lidar_scan(w.field, nodes, sub)  # GaussianBvh::build + scan
    cpu_s = time.perf_counter() - t0
    per_ray = cpu_s / (a.cpu_channels * lid.azimuth_count())
    line["cpu_reference"] = {"threads": os.cpu_count(), "sample_rays": a.cpu_channels * lid.azimuth_count(),
                             "sample_s": round(cpu_s, 2), "scans_per_s_extrapolated": round(1.0 / (per_ray * rays), 4),
                             "note": "includes one BVH build per sample (the reference rebuilds per scan)"}
if a.trace:
    # arbitrary rays (trace.cpp:113-123 per ray): origins in and around the cloud, random
    # directions, t_max 100 m; each call builds the BVH over the 1.08M posed boxes
    rng = np.random.default_rng(9)
    org = rng.uniform(-3.0, 3.0, (a.trace, 3))
    dirs = rng.normal(size=(a.trace, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    tmax = np.full(a.trace, 100.0)
    ctx.trace_rays(scene, nodes, org, dirs, tmax, 0.5)  # warm-up
    # median of 20 complete calls (wall clock: H2D of the rays, BVH build, traversal, trace, D2H)
    times = []
    for _ in range(20):
        t0 = time.perf_counter()
        hit, _, _ = ctx.trace_rays(scene, nodes, org, dirs, tmax, 0.5)
        times.append(time.perf_counter() - t0)
    gpu_t = float(np.median(times))
    line["trace_rays"] = {"rays": a.trace, "gpu_ms_per_call": round(gpu_t * 1e3, 2),
                          "gpu_rays_per_s": round(a.trace / gpu_t, 1),
                          "candidates_per_ray": round(ctx.stats()["pairs"] / a.trace, 1),
                          "hits": int(hit.sum()), "note": "BVH build + traversal + trace per call"}
    if not a.no_cpu:
        from oracle.oracle import Ref
        ref = Ref()
        import os
        ref.set_threads(os.cpu_count() or 1)
        k = min(a.trace, 2000)
        t0 = time.perf_counter()
        ref.trace_rays(w.field, nodes, org[:k], dirs[:k], tmax[:k], 0.5)  # BVH build + trace
        cpu_t = time.perf_counter() - t0
        line["trace_rays"]["cpu_reference"] = {"threads": os.cpu_count(), "sample_rays": k,
                                               "sample_s": round(cpu_t, 2),
                                               "rays_per_s": round(k / cpu_t, 1),
                                               "note": "GaussianBvh::build + trace (SAH BVH)"}
print(json.dumps(line))
