"""Where the synchronous drop-in's time goes: host CPU per render() call vs its wall time.
Usage: python tools/e2e_probe.py [--frames N]"""
import argparse
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_21981_b200 import Context, RenderTarget  # noqa: E402
from paper_2507_21981_b200.scenes import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=200)
a = ap.parse_args()
w = CONFIGS["cfg1"](seed=1000)
ctx = Context(0)
scene = ctx.upload(w.field)
tg = [RenderTarget(torch.empty((c.height, c.width, 3), pin_memory=True).numpy(),
                   torch.empty((c.height, c.width), pin_memory=True).numpy(),
                   torch.empty((c.height, c.width), pin_memory=True).numpy()) for c in w.cameras]
nodes = [w.frame_nodes(i) for i in range(a.frames)]
for i in range(5):
    ctx.render(scene, nodes[i], w.cameras, None, tg)
t0, c0 = time.perf_counter(), time.thread_time()
for i in range(a.frames):
    ctx.render(scene, nodes[i], w.cameras, None, tg)
t1, c1 = time.perf_counter(), time.thread_time()
print(f"render(): wall {1e3 * (t1 - t0) / a.frames:.3f} ms/frame, host CPU {1e3 * (c1 - c0) / a.frames:.3f} ms/frame")
t0, c0 = time.perf_counter(), time.thread_time()
for i in range(a.frames):
    ctx.render_device(scene, nodes[i], w.cameras)
ctx.synchronize()
t1, c1 = time.perf_counter(), time.thread_time()
print(f"render_device(): wall {1e3 * (t1 - t0) / a.frames:.3f} ms/frame, host CPU {1e3 * (c1 - c0) / a.frames:.3f} ms/frame")
t0 = time.perf_counter()
for i in range(a.frames):
    w.frame_nodes(i)
print(f"frame_nodes(): {1e3 * (time.perf_counter() - t0) / a.frames:.3f} ms")
