"""Stress the synchronous render() handoff: N contexts on N host threads render config-1 frames
into pageable host targets (per-camera copies ordered after each camera's raster launch) and
every frame is compared with the first. A hang dumps every thread's stack after 100 s.

    python tools/stress_contexts.py [contexts=5] [frames=40]
"""
import faulthandler, sys, threading, time
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, '.')
import numpy as np
from paper_2507_21981_b200 import Context
from paper_2507_21981_b200.scenes import config1
w = config1(seed=5)
nctx = int(sys.argv[1]) if len(sys.argv) > 1 else 5
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ctxs = [Context(0) for _ in range(nctx)]
scenes = [c.upload(w.field) for c in ctxs]
want = ctxs[0].render(scenes[0], w.frame_nodes(1), w.cameras)
bad = [0]
def run(k):
    for i in range(frames):
        got = ctxs[k].render(scenes[k], w.frame_nodes(1), w.cameras)
        bad[0] += sum(not np.array_equal(g.rgb, t.rgb) for g, t in zip(got, want))
th = [threading.Thread(target=run, args=(k,)) for k in range(nctx)]
t0 = time.time()
[t.start() for t in th]; [t.join() for t in th]
print("ok", bad[0], round(time.time() - t0, 1))
