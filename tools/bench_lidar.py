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
print(json.dumps(line))
