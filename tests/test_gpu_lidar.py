"""GPU LiDAR (trace.cpp) against the pinned oracle (tests/test_lidar_pin.py
pins the oracle bit-exactly to the reference's GaussianBvh::scan / trace / trace_linear).

Bars: the same returns (ring and azimuth bit-exact, same order: channel-major, azimuth ascending,
misses omitted) and points within 1e-12 m: every hit decision and the (t, index) compositing
order are the reference's double arithmetic (-fmad=false, host-computed ray directions); only
exp differs (CUDA's vs glibc's, <= 1 ulp per response). trace_rays: hit flags equal, depth and
accumulated alpha within 1e-12.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_21981_b200 import ValidationError
from paper_2507_21981_b200.api import (GaussianField, LidarModel, NodeKind, RigidTransform,
                                       SceneNode, quat_from_axis_angle)
from tests.test_lidar_pin import LIDARS, golden_lidar, golden_nodes, two_nodes

pytestmark = pytest.mark.gpu

TOL = 1e-12


def assert_scan_close(g, r):
    assert np.array_equal(g["ring"], r["ring"])
    assert np.array_equal(g["azimuth"], r["azimuth"])
    if len(r["ring"]):
        assert np.abs(g["points"] - r["points"]).max() <= TOL


@pytest.mark.parametrize("k", range(len(LIDARS)))
def test_scan_matches_oracle(ctx, oracle, k):
    f = oracle.random_field(91 + k, 2500, 2.0, 0.02, 0.15, k % 2)
    nodes = two_nodes(2500)
    assert_scan_close(ctx.lidar_scan(ctx.upload(f), nodes, LIDARS[k]), oracle.lidar_scan(f, nodes, LIDARS[k]))


def test_scan_golden_config(ctx, oracle):
    g, lid = golden_lidar()
    f = oracle.random_field(g["seed"], g["count"], g["box"], g["slo"], g["shi"], g["deg"])
    nodes = golden_nodes(g["count"])
    got = ctx.lidar_scan(ctx.upload(f), nodes, lid)
    assert len(got["ring"]) == g["returns"]
    assert_scan_close(got, oracle.lidar_scan(f, nodes, lid))


def test_scan_edge_geometry(ctx, oracle):
    """Wrap-around at azimuth 0, a box around the sensor, near-pole channels, max-range cut."""
    rng = np.random.default_rng(4)
    n = 1200
    f = oracle.random_field(33, n, 2.5, 0.02, 0.3, 0)
    f.means[:40] = np.array([2.0, 0.0, 0.0]) + rng.normal(0, 0.05, (40, 3))  # straddles azimuth 0
    f.scales[40] = [1.5, 1.5, 1.5]                                           # box holds the sensor
    f.means[40] = [0.0, 0.0, 0.0]
    f.opacities[40] = 0.3
    f.touch()
    for lid in [LidarModel(np.radians([-2.0, 0.0, 2.0, 88.5, -91.0, 120.0]), np.radians(1.5), 3.0),
                LidarModel(np.radians(np.linspace(-10, 10, 6)), np.radians(0.75), 1.2,
                           RigidTransform(quat_from_axis_angle((0.3, 1, 0.2), 1.1), (0.05, 0.0, -0.1)))]:
        assert_scan_close(ctx.lidar_scan(ctx.upload(f), [], lid), oracle.lidar_scan(f, [], lid))


def test_scan_env_filter(ctx, oracle):
    f = oracle.random_field(12, 1800, 2.0, 0.02, 0.15, 0)
    nodes = two_nodes(1800)
    nodes[1].env = 3
    for env in (3, 5):
        lid = LidarModel(np.radians(np.linspace(-15, 15, 8)), np.radians(2.0), 8.0, env=env)
        assert_scan_close(ctx.lidar_scan(ctx.upload(f), nodes, lid), oracle.lidar_scan(f, nodes, lid))


def test_trace_rays_match_oracle(ctx, oracle):
    f = oracle.random_field(7, 1500, 2.0, 0.02, 0.2, 0)
    nodes = two_nodes(1500)
    rng = np.random.default_rng(3)
    org = rng.uniform(-3, 3, (600, 3))
    d = rng.normal(size=(600, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:10] = [[1.0, 0.0, 0.0]] * 10
    tmax = rng.uniform(0.5, 9.0, 600)
    g = ctx.trace_rays(ctx.upload(f), nodes, org, d, tmax, 0.4)
    r = oracle.trace_rays(f, nodes, org, d, tmax, 0.4)
    assert np.array_equal(g[0], r[0])
    assert np.abs(g[1] - r[1]).max() <= TOL and np.abs(g[2] - r[2]).max() <= TOL


def test_lidar_validation(ctx, oracle):
    f = oracle.random_field(3, 100, 1.0, 0.02, 0.1, 0)
    scene = ctx.upload(f)
    good = dict(channels=np.radians([0.0, 5.0]), azimuth_step=np.radians(2.0), max_range=5.0)
    for kw in [dict(good, channels=np.zeros(0)), dict(good, azimuth_step=np.radians(7.0)),
               dict(good, max_range=0.0), dict(good, alpha_threshold=1.5)]:
        with pytest.raises(ValidationError):
            ctx.lidar_scan(scene, [], LidarModel(**kw))
    with pytest.raises(ValidationError):
        ctx.lidar_scan(scene, [SceneNode("x", NodeKind.interactive, RigidTransform(), (50, 101))],
                       LidarModel(**good))
    empty = GaussianField(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0),
                          np.zeros((0, 48)), 0)
    assert len(ctx.lidar_scan(ctx.upload(empty), [], LidarModel(**good))["ring"]) == 0


def test_scan_dense_windows(ctx, oracle):
    """Hundreds of survivors per ray: the histogram windows over the candidate cache."""
    f = oracle.random_field(44, 20000, 0.6, 0.01, 0.05, 0)
    f.opacities[:] = 0.05  # slow saturation: many windows per ray
    f.touch()
    lid = LidarModel(np.radians(np.linspace(-20, 20, 6)), np.radians(4.0), 5.0)
    got = ctx.lidar_scan(ctx.upload(f), [], lid)
    assert_scan_close(got, oracle.lidar_scan(f, [], lid))
    assert len(got["ring"]) > 0


def test_trace_rays_bvh_larger_scene(ctx, oracle):
    """Arbitrary rays through the linear BVH (bvh.cu) on 60k primitives with posed nodes: rays
    from inside and outside the cloud, axis-aligned directions (zero components: infinite slab
    reciprocals), a ray along a box face, short and long t_max. Same results as the reference's
    tracer (trace_linear semantics: the candidate set is every box the ray hits)."""
    f = oracle.random_field(77, 60000, 2.5, 0.005, 0.12, 1)
    nodes = two_nodes(60000)
    rng = np.random.default_rng(11)
    n = 2500
    org = rng.uniform(-3.5, 3.5, (n, 3))
    d = rng.normal(size=(n, 3))
    d[:40] = 0.0
    d[np.arange(40), np.arange(40) % 3] = np.where(np.arange(40) % 2 == 0, 1.0, -1.0)
    d[40:60, 2] = 0.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tmax = rng.uniform(0.2, 12.0, n)
    tmax[:100] = 100.0
    g = ctx.trace_rays(ctx.upload(f), nodes, org, d, tmax, 0.3)
    cand = ctx.stats()["pairs"]
    r = oracle.trace_rays(f, nodes, org, d, tmax, 0.3)
    assert np.array_equal(g[0], r[0])
    assert np.abs(g[1] - r[1]).max() <= TOL and np.abs(g[2] - r[2]).max() <= TOL
    assert cand > 10 * n  # the BVH produced candidate lists (not the every-primitive path)


BRUTE_SCRIPT = """
import sys, numpy as np
sys.path.insert(0, {root!r})
from oracle.oracle import Oracle
from paper_2507_21981_b200 import Context
orc = Oracle()
f = orc.random_field(78, 20000, 2.0, 0.01, 0.15, 0)
rng = np.random.default_rng(5)
org = rng.uniform(-3, 3, (1500, 3)); d = rng.normal(size=(1500, 3))
d /= np.linalg.norm(d, axis=1, keepdims=True); t = rng.uniform(0.5, 9.0, 1500)
ctx = Context(0)
hit, dep, acc = ctx.trace_rays(ctx.upload(f), [], org, d, t, 0.4)
np.save(sys.argv[1], np.concatenate([hit.astype(np.float64), dep, acc]))
"""


def test_trace_rays_bvh_list_overflow_path(tmp_path):
    """Single-pass BVH lists start at 4 slots per ray (GSIM_GPU_BVH_CAPACITY): the first call
    overflows and takes the exact count + scan + fill path, the second runs with the grown
    capacity; both give the default's bits."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    script = BRUTE_SCRIPT.replace("hit, dep, acc = ctx.trace_rays(ctx.upload(f), [], org, d, t, 0.4)",
                                  "s = ctx.upload(f)\n"
                                  "ctx.trace_rays(s, [], org, d, t, 0.4)\n"
                                  "hit, dep, acc = ctx.trace_rays(s, [], org, d, t, 0.4)")
    outs = []
    for cap in ("4", ""):
        p = tmp_path / f"c{cap or 'def'}.npy"
        env = dict(os.environ)
        if cap:
            env["GSIM_GPU_BVH_CAPACITY"] = cap
        r = subprocess.run([sys.executable, "-c", script.format(root=root), str(p)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(p))
    assert np.array_equal(outs[0], outs[1])


def test_trace_rays_bvh_equals_every_primitive(tmp_path):
    """The BVH candidate lists and the every-primitive path (GSIM_GPU_TRACE_BRUTE=1) composite
    the same survivors in the same (t, index) order: bit-identical results."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    outs = []
    for brute in ("0", "1"):
        p = tmp_path / f"r{brute}.npy"
        env = dict(os.environ, GSIM_GPU_TRACE_BRUTE=brute)
        r = subprocess.run([sys.executable, "-c", BRUTE_SCRIPT.format(root=root), str(p)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(p))
    assert np.array_equal(outs[0], outs[1])
