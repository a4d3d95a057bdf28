"""SURVEY.md 8f row 4 (LiDAR, trace.cpp): pin the oracle's restatement. CPU only.

  1. against the reference itself (oracle/_ref, compiled from /root/reference): GaussianBvh::scan
     point clouds, GaussianBvh::trace (BVH) and trace_linear per ray, and the validation errors,
     all bit for bit;
  2. against the committed golden fixture made from the reference (tests/golden/golden.json
     "lidar", tests/golden/make_golden.py).
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import OracleStatus
from paper_2507_21981_b200.api import (GaussianField, LidarModel, NodeKind, RigidTransform,
                                       SceneNode, quat_from_axis_angle, quat_normalized)

GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def two_nodes(n, angle=0.3, t=(0.2, 0.1, 0.0)):
    return [SceneNode("bg", NodeKind.background, RigidTransform(), (0, 2 * n // 3)),
            SceneNode("obj", NodeKind.interactive, RigidTransform(quat_from_axis_angle((0, 0, 1), angle), t),
                      (2 * n // 3, n))]


def same_scan(a, b) -> bool:
    return all(np.array_equal(a[k], b[k]) for k in ("points", "ring", "azimuth"))


LIDARS = [
    # sensor inside the cloud, tilted
    LidarModel(np.radians(np.linspace(-15, 15, 16)), np.radians(2.0), 10.0,
               RigidTransform(quat_from_axis_angle((1, 0, 0), 0.1), (0.1, -0.2, 0.05))),
    # outside, unsorted channels incl. one near the pole, short range
    LidarModel(np.radians([10, -5, 0, 3, 89.99, -30]), np.radians(1.0), 4.0,
               RigidTransform(quat_from_axis_angle((0, 0, 1), 2.0), (-3.0, 0.5, 0.2))),
    # many rays, high threshold
    LidarModel(np.radians(np.linspace(-25, 5, 12)), np.radians(0.5), 6.0,
               RigidTransform((1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.3)), alpha_threshold=0.9),
]


@pytest.mark.parametrize("k", range(len(LIDARS)))
def test_scan_matches_reference(oracle, ref, k):
    f = oracle.random_field(91 + k, 2500, 2.0, 0.02, 0.15, k % 2)
    nodes = two_nodes(2500)
    a = oracle.lidar_scan(f, nodes, LIDARS[k])
    b = ref.lidar_scan(f, nodes, LIDARS[k])
    assert same_scan(a, b)
    assert 0 < len(a["ring"])


def test_trace_matches_reference_bvh_and_linear(oracle, ref):
    f = oracle.random_field(7, 1500, 2.0, 0.02, 0.2, 0)
    nodes = two_nodes(1500)
    rng = np.random.default_rng(3)
    org = rng.uniform(-3, 3, (400, 3))
    d = rng.normal(size=(400, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:10] = [[1.0, 0.0, 0.0]] * 10  # axis-parallel rays: the slab test's inf * 0 path
    tmax = rng.uniform(0.5, 9.0, 400)
    a = oracle.trace_rays(f, nodes, org, d, tmax, 0.4)
    b = ref.trace_rays(f, nodes, org, d, tmax, 0.4)
    c = ref.trace_rays(f, nodes, org, d, tmax, 0.4, linear=True)
    for x, y, z in zip(a, b, c):
        assert np.array_equal(x, y) and np.array_equal(y, z)
    assert 0 < a[0].mean() < 1


def status_of(fn):
    try:
        fn()
        return 0
    except OracleStatus as e:
        return e.status


def test_validation_matches_reference(oracle, ref):
    f = oracle.random_field(3, 100, 1.0, 0.02, 0.1, 0)
    good = dict(channels=np.radians([0.0, 5.0]), azimuth_step=np.radians(2.0), max_range=5.0)
    bad = [dict(good, channels=np.zeros(0)), dict(good, channels=[0.0, float("nan")]),
           dict(good, azimuth_step=0.0), dict(good, azimuth_step=np.radians(7.0)),
           dict(good, max_range=0.0), dict(good, max_range=-1.0)]
    for kw in bad:
        lid = LidarModel(**kw)
        assert status_of(lambda: oracle.lidar_scan(f, [], lid)) == 2
        assert status_of(lambda: ref.lidar_scan(f, [], lid)) == 2
    for thr in (0.0, 1.5, -0.1):
        lid = LidarModel(**good, alpha_threshold=thr)
        assert status_of(lambda: oracle.lidar_scan(f, [], lid)) == 2
        assert status_of(lambda: ref.lidar_scan(f, [], lid)) == 2
    over = [SceneNode("x", NodeKind.interactive, RigidTransform(), (50, 101))]
    assert status_of(lambda: oracle.lidar_scan(f, over, LidarModel(**good))) == 2
    assert status_of(lambda: ref.lidar_scan(f, over, LidarModel(**good))) == 2
    empty = GaussianField(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0),
                          np.zeros((0, 48)), 0)
    assert same_scan(oracle.lidar_scan(empty, [], LidarModel(**good)),
                     ref.lidar_scan(empty, [], LidarModel(**good)))


def golden_lidar():
    g = GOLDEN["lidar"]
    return g, LidarModel(np.radians(g["channels_deg"]), np.radians(g["azimuth_step_deg"]), g["max_range"],
                         RigidTransform(quat_normalized(tuple(g["pose_q"])), tuple(g["pose_t"])))


def golden_nodes(n):  # tests/golden/make_golden.py make_nodes("two", n)
    q = quat_normalized((0.9, 0.1, 0.3, 0.2))
    return [SceneNode("bg", NodeKind.background, RigidTransform(), (0, n // 2)),
            SceneNode("obj", NodeKind.interactive, RigidTransform(q, (0.1, -0.2, 0.3)), (n // 2, n))]


def test_oracle_reproduces_lidar_golden(oracle):
    g, lid = golden_lidar()
    f = oracle.random_field(g["seed"], g["count"], g["box"], g["slo"], g["shi"], g["deg"])
    scan = oracle.lidar_scan(f, golden_nodes(g["count"]), lid)
    assert len(scan["ring"]) == g["returns"]
    assert sha(scan["points"]) == g["points_sha"]
    assert sha(scan["ring"]) == g["ring_sha"] and sha(scan["azimuth"]) == g["azimuth_sha"]
