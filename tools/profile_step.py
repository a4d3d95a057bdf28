"""Render a few BASELINE config-1 frames (for ncu launch lists and full captures).
Usage: python tools/profile_step.py [--frames N] [--warmup W] [--config cfg1]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2507_21981_b200 import Context  # noqa: E402
from paper_2507_21981_b200.scenes import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=2)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--config", default="cfg1")
a = ap.parse_args()
w = CONFIGS[a.config](seed=1000)
ctx = Context(0)
scene = ctx.upload(w.field)
for i in range(a.warmup + a.frames):
    ctx.render_device(scene, w.frame_nodes(i), w.cameras)
ctx.synchronize()
print("frames ok", ctx.stats())
