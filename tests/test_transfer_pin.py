"""SURVEY.md 8f row 3 (GS -> TSDF, transfer.cpp): pin the oracle's restatement and the library's
host-side pieces. CPU only.

  1. the oracle against the reference itself (oracle/_ref, compiled from /root/reference):
     render_depth_ring (cameras and masked depth), tsdf_fuse, gaussians_to_mesh's fused volume,
     and the validation errors, all bit for bit;
  2. the oracle against the committed golden fixture made from the reference
     (tests/golden/golden.json "transfer", tests/golden/make_golden.py);
  3. the library's host-only entry points (ring cameras, TsdfVolume::create validation) against
     the oracle through the C ABI (no GPU needed).
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import OracleStatus
from paper_2507_21981_b200 import abi
from paper_2507_21981_b200.api import CameraModel, GaussianField, ValidationError

GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def camera_table(cams) -> np.ndarray:  # tests/golden/make_golden.py
    return np.array([[c.fx, c.fy, c.cx, c.cy, c.width, c.height, *c.pose.rotation,
                      *c.pose.translation, c.near_plane, c.far_plane] for c in cams])


def same_cameras(a, b) -> bool:
    return np.array_equal(camera_table(a), camera_table(b))


# ---- 1. oracle == reference ----------------------------------------------------------------------

@pytest.mark.parametrize("seed,count,deg,n_views,radius,res", [
    (5, 300, 0, 8, 5.0, 32), (6, 800, 3, 9, 3.0, 40), (7, 150, 1, 12, 9.5, 24)])
def test_depth_ring_matches_reference(oracle, ref, seed, count, deg, n_views, radius, res):
    f = oracle.random_field(seed, count, 1.5, 0.02, 0.12, deg)
    ca, da = oracle.render_depth_ring(f, n_views, radius, res)
    cb, db = ref.render_depth_ring(f, n_views, radius, res)
    assert same_cameras(ca, cb)
    assert np.array_equal(da, db)
    assert 0.0 < (da > 0).mean() < 1.0  # both valid and masked pixels occur


def look_at_cam(oracle, eye, target, f, w, h, near=0.05, far=100.0):
    c = oracle.look_at(eye, target, f, f, w, h)
    c.near_plane, c.far_plane = near, far
    return c


def test_tsdf_fuse_matches_reference(oracle, ref):
    rng = np.random.default_rng(11)
    vo = oracle.tsdf_create((-1.0, -1.2, -0.9), 0.07, (30, 33, 27), 0.21)
    vr = ref.tsdf_create((-1.0, -1.2, -0.9), 0.07, (30, 33, 27), 0.21)
    assert np.array_equal(vo.tsdf, vr.tsdf) and np.array_equal(vo.weights, vr.weights)
    for k in range(7):
        eye = rng.uniform(-4, 4, 3)
        if k == 3:
            eye = np.array([0.2, 0.1, 0.0])  # inside the volume: voxels behind the camera
        cam = look_at_cam(oracle, eye, (0.0, 0.0, 0.0), float(rng.uniform(20, 60)), 64, 48)
        depth = rng.uniform(0.5, 6.0, (48, 64)).astype(np.float32)
        depth[rng.random((48, 64)) < 0.2] = 0.0        # invalid pixels
        depth[rng.random((48, 64)) < 0.02] = -1.0      # negative = invalid too
        oracle.tsdf_fuse(vo, cam, depth)
        ref.tsdf_fuse(vr, cam, depth)
    assert np.array_equal(vo.tsdf, vr.tsdf)
    assert np.array_equal(vo.weights, vr.weights)
    assert (vo.weights > 1).any() and (vo.tsdf < 0).any() and (vo.tsdf == 1).any()


@pytest.mark.parametrize("seed,deg,voxel", [(21, 0, 0.12), (22, 3, 0.09)])
def test_gaussians_to_tsdf_matches_reference(oracle, ref, seed, deg, voxel):
    f = oracle.random_field(seed, 500, 1.5, 0.02, 0.1, deg)
    a = oracle.gaussians_to_tsdf(f, voxel)
    b = ref.gaussians_to_tsdf(f, voxel)
    assert a.dims == b.dims and a.origin == b.origin and a.truncation == b.truncation
    assert np.array_equal(a.tsdf, b.tsdf) and np.array_equal(a.weights, b.weights)
    assert (a.weights > 0).mean() > 0.5


def status_of(fn):
    try:
        fn()
        return 0
    except OracleStatus as e:
        return e.status


def test_validation_matches_reference(oracle, ref):
    f = oracle.random_field(3, 50, 1.0, 0.02, 0.1, 0)
    empty = GaussianField(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0),
                          np.zeros((0, 48)), 0)
    one = GaussianField(np.zeros((1, 3)), np.zeros((1, 3)), np.array([[1.0, 0, 0, 0]]),
                        np.array([0.5]), np.zeros((1, 48)), 0)  # zero scale: degenerate box
    cases = [
        lambda o: o.render_depth_ring(f, 7, 5.0, 32),
        lambda o: o.render_depth_ring(f, 8, 0.0, 32),
        lambda o: o.render_depth_ring(f, 8, -1.0, 32),
        lambda o: o.render_depth_ring(f, 8, float("nan"), 32),
        lambda o: o.render_depth_ring(f, 8, 5.0, 8),   # resolution below 16: project throws
        lambda o: o.render_depth_ring(empty, 8, 5.0, 32),
        lambda o: o.render_depth_ring(one, 8, 5.0, 32),
        lambda o: o.tsdf_create((0, 0, 0), 0.0, (4, 4, 4), 0.1),
        lambda o: o.tsdf_create((0, 0, 0), 0.1, (4, 1, 4), 0.3),
        lambda o: o.tsdf_create((0, 0, 0), 0.1, (4, 4, 4), 0.19),
        lambda o: o.gaussians_to_tsdf(f, 0.0),
        lambda o: o.gaussians_to_tsdf(empty, 0.1),
        lambda o: o.gaussians_to_tsdf(one, 0.1),
    ]
    for k, case in enumerate(cases):
        so, sr = status_of(lambda: case(oracle)), status_of(lambda: case(ref))
        assert so == sr == abi_validation(), (k, so, sr)
    vol = oracle.tsdf_create((0, 0, 0), 0.1, (4, 4, 4), 0.3)
    volr = ref.tsdf_create((0, 0, 0), 0.1, (4, 4, 4), 0.3)
    bad = CameraModel(fx=-1.0, fy=10.0, cx=8, cy=8, width=16, height=16).to_c()
    for o, v in ((oracle, vol), (ref, volr)):
        assert status_of(lambda: o.tsdf_fuse(v, bad, np.ones((16, 16), np.float32))) == abi_validation()
        good = CameraModel(fx=10.0, fy=10.0, cx=8, cy=8, width=16, height=16).to_c()
        assert status_of(lambda: o.tsdf_fuse(v, good, np.ones((17, 16), np.float32))) == abi_validation()


def abi_validation() -> int:
    return 2  # GSIM_ERR_VALIDATION


# ---- 2. oracle == golden (made from the reference) ---------------------------------------------

def test_oracle_reproduces_transfer_golden(oracle):
    t = GOLDEN["transfer"]
    f = oracle.random_field(t["seed"], t["count"], t["box"], t["slo"], t["shi"], t["deg"])
    cams, depth = oracle.render_depth_ring(f, t["n_views"], t["radius"], t["resolution"])
    assert sha(camera_table(cams)) == t["ring_cams_sha"]
    assert sha(depth) == t["ring_depth_sha"]
    vol = oracle.gaussians_to_tsdf(f, t["voxel_size"])
    assert list(vol.dims) == t["dims"] and list(vol.origin) == t["origin"]
    assert vol.truncation == t["truncation"]
    assert sha(vol.tsdf) == t["tsdf_sha"] and sha(vol.weights) == t["weights_sha"]


# ---- 3. library host entry points == oracle (C ABI, no GPU) ------------------------------------

def test_library_ring_cameras_match_oracle(oracle):
    from paper_2507_21981_b200.api import depth_ring_cameras
    rng = np.random.default_rng(5)
    for _ in range(60):
        lo = rng.uniform(-3, 1, 3)
        hi = lo + rng.uniform(1e-3, 5, 3)
        nv, rad, res = int(rng.integers(8, 40)), float(rng.uniform(0.1, 30)), int(rng.integers(16, 512))
        assert same_cameras(depth_ring_cameras(lo, hi, nv, rad, res),
                            oracle.depth_ring_cameras(lo, hi, nv, rad, res))
    for args in [((0, 0, 0), (1, 1, 1), 7, 3.0, 32), ((0, 0, 0), (1, 1, 1), 8, 0.0, 32),
                 ((1, 1, 1), (1, 1, 1), 8, 3.0, 32)]:
        with pytest.raises(ValidationError):
            depth_ring_cameras(*args)
        with pytest.raises(OracleStatus):
            oracle.depth_ring_cameras(*args)


def test_library_tsdf_create_validation():
    from paper_2507_21981_b200.api import tsdf_create
    v = tsdf_create((0.5, -1, 2), 0.05, (10, 11, 12), 0.1)
    assert v.dims == (10, 11, 12) and v.voxel_size == 0.05 and v.truncation == 0.1
    assert v.origin == (0.5, -1.0, 2.0)
    for args in [((0, 0, 0), 0.0, (4, 4, 4), 0.1), ((0, 0, 0), -0.1, (4, 4, 4), 0.1),
                 ((0, 0, 0), 0.1, (1, 4, 4), 0.3), ((0, 0, 0), 0.1, (4, 4, 4), 0.1999)]:
        with pytest.raises(ValidationError):
            tsdf_create(*args)


def test_tsdf_volume_struct_layout():
    import ctypes as C
    assert C.sizeof(abi.gsim_tsdf_volume) == 3 * 8 + 8 + 3 * 4 + 4 + 8 + 8 + 8
