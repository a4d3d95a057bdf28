"""GPU scene feed: pose playback and the splat PLY loader, against the
pinned oracle (tests/test_encode_pin.py pins gso_pose_sample / gso_slerp / gso_load_splat_ply
bit-exactly to the reference's PoseStream, slerp and load_splat_ply).

Bars: translations, endpoints and the nlerp branch bit-exact (double, -fmad=false); the slerp
branch within 1e-15 absolute per quaternion component (CUDA acos/sin vs glibc, <= 2 ulp).
render_at: the images of a frame whose node poses are sampled on the GPU equal (north-star
image tolerance) those of the same frame rendered from the oracle's sampled poses.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_21981_b200 import IoError, ValidationError
from paper_2507_21981_b200.api import NodeKind, RigidTransform, SceneNode
from tests.helpers import parity_stats, ref_camera
from tests.test_encode_pin import ply_bytes, ply_error_cases, random_track

pytestmark = pytest.mark.gpu

QUAT_TOL = 1e-15


def test_tracks_sample_matches_oracle(ctx, oracle):
    rng = np.random.default_rng(21)
    tracks = []
    for k in range(25):
        n = int(rng.integers(0, 30)) if k else 0  # track 0 is empty
        if n == 0:
            tracks.append((np.zeros(0), np.zeros((0, 3)), np.zeros((0, 4))))
        else:
            tracks.append(random_track(rng, n, t0=rng.uniform(-2, 2), dup=k % 4 == 0))
    dev = ctx.upload_tracks(tracks)
    init = RigidTransform((0.8, -0.2, 0.1, 0.4), (0.5, -1.0, 2.0))
    worst = 0.0
    for k, (t, p, q) in enumerate(tracks):
        lo, hi = (t[0], t[-1]) if len(t) else (0.0, 1.0)
        ts = np.concatenate([rng.uniform(lo - 1, hi + 1, 300), t, [lo - 1e-9, hi]])
        got = dev.sample(k, ts, init)
        rc, want = oracle.pose_sample(t, p, q, init, ts)
        assert rc == 0
        assert np.array_equal(got[:, 4:], want[:, 4:]), k  # translations bit-exact
        d = np.abs(got[:, :4] - want[:, :4]).max(initial=0.0)
        worst = max(worst, d)
        assert d <= QUAT_TOL, (k, d)
        # outside the track's span: initial / last record, bit-exact
        outside = (ts < lo) | (ts >= hi)
        assert np.array_equal(got[outside], want[outside]), k
    assert worst <= QUAT_TOL


def test_tracks_validation(ctx):
    q1 = np.tile([1.0, 0, 0, 0], (3, 1))
    with pytest.raises(ValidationError):
        ctx.upload_tracks([(np.array([0.0, 1.0, 0.5]), np.zeros((3, 3)), q1)])  # decreasing
    with pytest.raises(ValidationError):
        ctx.upload_tracks([(np.array([0.0, np.nan, 2.0]), np.zeros((3, 3)), q1)])
    bad = q1.copy(); bad[1, 0] = np.inf
    with pytest.raises(ValidationError):
        ctx.upload_tracks([(np.array([0.0, 1.0, 2.0]), np.zeros((3, 3)), bad)])
    dev = ctx.upload_tracks([(np.array([0.0, 1.0, 2.0]), np.zeros((3, 3)), q1)])
    with pytest.raises(ValidationError):
        dev.sample(1, [0.5], RigidTransform())  # no such track


def scene_with_objects(oracle, n_bg=6000, n_obj=4, per_obj=800, seed=51):
    field = oracle.random_field(seed, n_bg + n_obj * per_obj, 3.0, 0.01, 0.2, 2)
    field.means[n_bg:] *= 0.15
    field.means[:, 2] += 3.5
    field.touch()
    nodes = [SceneNode("bg", NodeKind.background, RigidTransform(), (0, n_bg))]
    for k in range(n_obj):
        b = n_bg + k * per_obj
        nodes.append(SceneNode(f"obj{k}", NodeKind.interactive,
                               RigidTransform((1.0, 0, 0, 0), (0.3 * k - 0.45, 0.0, 0.0)),
                               (b, b + per_obj)))
    return field, nodes


def test_render_at_equals_render_of_sampled_poses(ctx, oracle):
    rng = np.random.default_rng(22)
    field, nodes = scene_with_objects(oracle)
    scene = ctx.upload(field)
    tracks = [random_track(rng, 12, t0=0.0) for _ in range(3)]
    for t, p, q in tracks:
        p *= 0.2
    dev = ctx.upload_tracks(tracks)
    node_track = [-1, 0, 1, -1, 2]  # object 2 keeps its pose
    cams = [ref_camera(128, 96, 90.0), ref_camera(64, 64, 50.0)]
    for time in (-1.0, 0.7, 1.9, 50.0):
        posed = []
        for k, n in enumerate(nodes):
            if node_track[k] >= 0:
                t, p, q = tracks[node_track[k]]
                rc, pose = oracle.pose_sample(t, p, q, n.pose, [time])
                assert rc == 0
                n = SceneNode(n.id, n.kind, RigidTransform(tuple(pose[0, :4]), tuple(pose[0, 4:])),
                              n.range)
            posed.append(n)
        got = ctx.render_at(scene, dev, time, nodes, node_track, cams)
        want = ctx.render(scene, posed, cams)
        ref = oracle.render(field, posed, cams)
        for g, w, r in zip(got, want, ref):
            st = parity_stats(g, w)
            assert st["rgb_ok"] >= 0.999 and st["depth_ok"] >= 0.999, (time, st)
            st = parity_stats(g, r)
            assert st["rgb_ok"] >= 0.999 and st["depth_ok"] >= 0.999, (time, st)
    # device destination (asynchronous) gives the same frame
    import torch
    n = sum(5 * c.width * c.height for c in cams)
    out = torch.zeros(n, dtype=torch.float32, device="cuda:0")
    ctx.render_at(scene, dev, 0.7, nodes, node_track, cams, device_out=out.data_ptr())
    ctx.synchronize()
    host = ctx.render_at(scene, dev, 0.7, nodes, node_track, cams)
    flat = out.cpu().numpy()
    assert np.array_equal(flat[: 3 * 128 * 96].reshape(96, 128, 3), host[0].rgb)


def test_render_at_validation(ctx, oracle):
    field, nodes = scene_with_objects(oracle, n_bg=500, per_obj=100)
    scene = ctx.upload(field)
    dev = ctx.upload_tracks([(np.array([0.0, 1.0]), np.zeros((2, 3)), np.tile([1.0, 0, 0, 0], (2, 1)))])
    cams = [ref_camera(32, 32)]
    with pytest.raises(ValidationError):  # scene.cpp:180-184
        ctx.render_at(scene, dev, 0.5, nodes, [0, -1, -1, -1, -1], cams)
    with pytest.raises(ValidationError):
        ctx.render_at(scene, dev, 0.5, nodes, [-1, 3, -1, -1, -1], cams)
    with pytest.raises(ValidationError):
        ctx.render_at(scene, dev, float("nan"), nodes, [-1, 0, -1, -1, -1], cams)


# ---- splat PLY -------------------------------------------------------------------------------

def test_load_ply_matches_oracle(ctx, oracle, tmp_path):
    """Means, rotations and SH bit-exact; scales within 1 ulp (CUDA exp), opacity = 1/(1+exp(-x))
    within 2 ulp."""
    for degree in range(4):
        for n in (0, 1, 3000):
            p = tmp_path / f"f{degree}_{n}.ply"
            p.write_bytes(ply_bytes(n, degree, seed=degree * 7 + n))
            rc, want = oracle.load_splat_ply(p)
            assert rc == 0
            scene = ctx.load_ply(p)
            assert scene.size == n and scene.sh_degree == degree
            got = scene.download_field()
            for k in ("means", "rotations", "sh"):
                assert np.array_equal(getattr(got, k), getattr(want, k)), (degree, n, k)
            for k in ("opacities", "scales"):
                g, w = getattr(got, k), getattr(want, k)
                ulps = 2 if k == "opacities" else 1
                assert np.all(np.abs(g - w) <= ulps * np.spacing(np.abs(w))), (degree, n, k)


def test_load_ply_errors(ctx, oracle, tmp_path):
    for name, data in ply_error_cases().items():
        p = tmp_path / f"{name}.ply"
        p.write_bytes(data)
        rc, _ = oracle.load_splat_ply(p)
        if rc == 0:
            assert ctx.load_ply(p).size == 20, name
        else:
            with pytest.raises(ValidationError):
                ctx.load_ply(p)
    with pytest.raises(IoError):
        ctx.load_ply(tmp_path / "missing.ply")


def test_render_of_ply_scene(ctx, oracle, tmp_path):
    """A PLY written by the oracle's field generator, loaded on the GPU and rendered, against
    the oracle's own load + render of the same file."""
    rng = np.random.default_rng(88)
    p = tmp_path / "scene.ply"
    n = 20000
    rows = np.frombuffer(ply_bytes(n, 3, seed=88).split(b"end_header\n", 1)[1], np.float32)
    rows = rows.reshape(n, -1).copy()
    rows[:, 0:2] = rng.uniform(-1.5, 1.5, (n, 2))
    rows[:, 2] = rng.uniform(2.0, 5.0, n)
    rows[:, 6:9] *= 0.5
    rows[:, 9:54] *= 0.2
    rows[:, -7:-4] = rng.uniform(-5.0, -2.5, (n, 3))
    p.write_bytes(ply_bytes(n, 3, rows=rows))
    rc, loaded = oracle.load_splat_ply(p)
    assert rc == 0
    scene = ctx.load_ply(p)
    cams = [ref_camera(160, 120, 120.0), ref_camera(64, 64, 60.0)]
    got = ctx.render(scene, [], cams)
    want = oracle.render(loaded, [], cams)
    assert got[0].accum_alpha.max() > 0.5
    for g, w in zip(got, want):
        st = parity_stats(g, w)
        assert st["rgb_ok"] >= 0.999 and st["depth_ok"] >= 0.999, st
