"""One gsim_gpu_trace_rays call on the config-1 scene (for ncu launch lists of the BVH path)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_21981_b200 import Context  # noqa: E402
from paper_2507_21981_b200.scenes import CONFIGS  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
w = CONFIGS["cfg1"](seed=1000)
ctx = Context(0)
scene = ctx.upload(w.field)
rng = np.random.default_rng(9)
org = rng.uniform(-3.0, 3.0, (n, 3))
d = rng.normal(size=(n, 3))
d /= np.linalg.norm(d, axis=1, keepdims=True)
for _ in range(2):
    hit, _, _ = ctx.trace_rays(scene, w.frame_nodes(0), org, d, np.full(n, 100.0), 0.5)
print("hits", int(hit.sum()), "candidates", ctx.stats()["pairs"])
