"""Where the e2e leg loses against the device rate: 4 host threads x synchronous frames,
(a) render_device + synchronize (no host copies) vs (b) render into pinned host targets."""
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2507_21981_b200 import Context, RenderTarget  # noqa: E402
from paper_2507_21981_b200.api import _cams_array, _nodes_array  # noqa: E402
from paper_2507_21981_b200.scenes import CONFIGS  # noqa: E402

w = CONFIGS["cfg1"](seed=1000)
n_ctx, steps = 4, 400
ctxs = [Context(0) for _ in range(n_ctx)]
scenes = [c.upload(w.field) for c in ctxs]
nodes = [_nodes_array(w.frame_nodes(i)) for i in range(steps)]
cams = _cams_array(w.cameras)
outs = [torch.empty(sum(5 * c.width * c.height for c in w.cameras), device="cuda:0") for _ in ctxs]
targets = []
for _ in ctxs:
    t = []
    for c in w.cameras:
        t.append(RenderTarget(torch.empty((c.height, c.width, 3), pin_memory=True).numpy(),
                              torch.empty((c.height, c.width), pin_memory=True).numpy(),
                              torch.empty((c.height, c.width), pin_memory=True).numpy()))
    targets.append(t)


def run(fn):
    for k in range(n_ctx):
        fn(k, 0)
    torch.cuda.synchronize()
    th = [threading.Thread(target=lambda k=k: [fn(k, i) for i in range(k, steps, n_ctx)]) for k in range(n_ctx)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    return steps * len(w.cameras) / (time.perf_counter() - t0)


def dev(k, i):
    ctxs[k].render_device(scenes[k], nodes[i], cams, None, outs[k].data_ptr())
    ctxs[k].synchronize()


def host(k, i):
    ctxs[k].render(scenes[k], nodes[i], cams, None, targets[k])


def dev_async(k, i):
    ctxs[k].render_device(scenes[k], nodes[i], cams, None, outs[k].data_ptr())


print("device, synchronous per frame:", round(run(dev)), "camera-frames/s")
print("host targets (render):", round(run(host)), "camera-frames/s")
print("device, asynchronous:", round(run(dev_async)), "camera-frames/s")
