"""Streaming scene upload (gsim_gpu_scene_create / _write) and scatter blocks that take units of
several cameras (GSIM_GPU_SCATTER_CTAS): both must leave renders bit-identical."""
from __future__ import annotations

import os
import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest

from paper_2507_21981_b200 import ValidationError
from paper_2507_21981_b200.api import GaussianField
from tests.helpers import ref_camera

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _slice(f: GaussianField, a: int, b: int) -> GaussianField:
    return GaussianField(f.means[a:b], f.scales[a:b], f.rotations[a:b], f.opacities[a:b], f.sh[a:b],
                         f.sh_degree)


def test_streamed_scene_equals_upload(ctx, oracle):
    field = oracle.random_field(404, 5000, 3.0, 0.01, 0.2, 3)
    field.means[:, 2] += 3.0
    cams = [ref_camera(160, 120, 110.0)]
    want = ctx.render(ctx.upload(field), [], cams)[0]
    s = ctx.create_scene(5000, 3)
    for a, b in ((3000, 5000), (0, 1200), (1200, 3000)):  # any order
        s.write(a, _slice(field, a, b))
    got = ctx.render(s, [], cams)[0]
    assert np.array_equal(got.rgb, want.rgb) and np.array_equal(got.depth, want.depth)
    dm, _ = s.download()
    assert np.array_equal(dm, field.means)
    with pytest.raises(ValidationError, match="exceeds"):
        s.write(4500, _slice(field, 0, 600))
    with pytest.raises(ValidationError, match="sh_degree"):
        s.write(0, GaussianField(field.means[:10], field.scales[:10], field.rotations[:10],
                                 field.opacities[:10], field.sh[:10], 1))


SCRIPT = textwrap.dedent("""
    import sys, numpy as np
    sys.path.insert(0, {root!r})
    from oracle.oracle import Oracle
    from paper_2507_21981_b200 import Context
    from paper_2507_21981_b200.api import RigidTransform, quat_from_axis_angle
    from tests.helpers import ref_camera
    orc = Oracle()
    f = orc.random_field(9191, 60000, 3.0, 0.005, 0.05, 1)
    f.means[:, 2] += 3.0
    f.touch()
    small = ref_camera(64, 48, 40.0)       # 5 x 4 tile-grid cells: its units come first
    big = ref_camera(640, 480, 500.0)      # 41 x 31 cells: later units of the same blocks
    big.pose = RigidTransform(quat_from_axis_angle((0, 1, 0), 0.05), (0.1, 0.0, 0.0))
    ctx = Context(0)
    s = ctx.upload(f)
    ctx.render(s, [], [small, big])
    bad = 0
    for k, cam in enumerate((small, big)):
        offsets, values = ctx.tile_lists(k)
        splats = orc.project(f, [], cam)
        tb, vals = orc.rasterize_lists(splats, cam)
        bad += int(not np.array_equal(offsets[: len(tb)], tb))
        bad += int(not np.array_equal(values, splats["prim_index"][vals]))
    print("chunks", ctx.stats()["chunks"], "mismatches", bad)
    sys.exit(1 if bad else 0)
""")


def test_scatter_blocks_over_mixed_cameras():
    """with GSIM_GPU_SCATTER_CTAS=1 one scatter block places units of a small and then
    a large camera; the lane bitmaps must be clean over the large camera's whole grid."""
    env = dict(os.environ, GSIM_GPU_SCATTER_CTAS="1", GSIM_GPU_WARP_RECORDS="128")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT))], env=env,
                       capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
