"""Pin the CPU oracle (oracle/gsim_oracle.c) before trusting it as the GPU checker.

Three anchors, all CPU-only:
  1. the reference itself (oracle/_ref, compiled from /root/reference sources): bit-exact;
  2. the committed golden fixtures (tests/golden/golden.json, made from the reference);
  3. the reference's own known-answer tests (test_raster.cpp, test_core_types.cpp and the
     C++ standard's mt19937_64 check value), re-expressed here because doctest is absent.
"""
from __future__ import annotations

import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

from paper_2507_21981_b200.api import (NodeKind, RasterOptions, RigidTransform, SceneNode,
                                       quat_from_axis_angle, quat_normalized)
from tests.helpers import flat_splat, max_diff, single_prim_field, ref_camera

GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def golden_nodes(kind, n):
    if kind == "none":
        return []
    q = quat_normalized((0.9, 0.1, 0.3, 0.2))
    return [SceneNode("bg", NodeKind.background, RigidTransform(), (0, n // 2)),
            SceneNode("obj", NodeKind.interactive, RigidTransform(q, (0.1, -0.2, 0.3)), (n // 2, n))]


# ---- anchor 3a: std::mt19937_64 / random_field ---------------------------------------------

def test_mt19937_64_standard_check_value(oracle):
    # [rand.predef]: the 10000th consecutive invocation of a default-constructed mt19937_64
    # (seed 5489) produces 9981545732273789042.
    assert int(oracle.mt19937_64(5489, 10000)[-1]) == 9981545732273789042


def test_random_field_matches_reference(oracle, ref):
    for seed, count, deg in [(1000, 100, 3), (9000, 700, 2), (77, 500, 0), (4242, 300, 1)]:
        a = oracle.random_field(seed, count, 3.0, 0.01, 0.25, deg)
        b = ref.random_field(seed, count, 3.0, 0.01, 0.25, deg)
        for k in ("means", "scales", "rotations", "opacities", "sh"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (seed, k)


# ---- anchor 2: golden fixtures ------------------------------------------------------------

@pytest.mark.parametrize("case", GOLDEN["cases"], ids=[c["name"] for c in GOLDEN["cases"]])
def test_oracle_reproduces_golden(oracle, case):
    field = oracle.random_field(case["seed"], case["count"], case["box"], case["slo"], case["shi"], case["deg"])
    field.means[:, 2] += case["dz"]
    assert sha(np.concatenate([field.means.ravel(), field.scales.ravel(), field.rotations.ravel(),
                               field.opacities, field.sh.ravel()])) == case["field_sha"]
    f, w, h = case["cam"]
    cam = ref_camera(w, h, f)
    splats = oracle.project(field, golden_nodes(case["nodes"], case["count"]), cam)
    assert len(splats) == case["n_splats"]
    assert sha(splats) == case["splats_sha"]
    assert str(oracle.hash_target(oracle.rasterize(splats, cam))) == case["tiled_hash"]
    assert str(oracle.hash_target(oracle.reference_rasterize(splats, cam))) == case["brute_hash"]
    norm = oracle.rasterize(splats, cam, RasterOptions(normalize_depth=True, transmittance_cutoff=1e-3))
    assert str(oracle.hash_target(norm)) == case["norm_hash"]
    tb, vals = oracle.rasterize_lists(splats, cam)
    assert len(vals) == case["n_pairs"]
    assert sha(np.concatenate([tb, vals])) == case["pairs_sha"]


def test_oracle_render_golden(oracle):
    g = GOLDEN["render"]
    field = oracle.random_field(g["seed"], g["count"], 3.0, 0.01, 0.2, 3)
    field.means[:, 2] += 3.0
    cams = [ref_camera(96, 80, 90.0), ref_camera(96, 80, 90.0)]
    cams[1].pose = RigidTransform(quat_normalized((0.99, 0.05, -0.05, 0.02)), (0.2, 0.0, 0.1))
    targets = oracle.render(field, golden_nodes("two", g["count"]), cams)
    assert [str(oracle.hash_target(t)) for t in targets] == g["hashes"]


def test_oracle_transform_golden(oracle):
    g = GOLDEN["transform"]
    f = oracle.random_field(g["seed"], g["count"], 2.0, 0.01, 0.3, 1)
    m, q = f.means.copy(), f.rotations.copy()
    rt = RigidTransform(quat_normalized((0.3, 0.5, -0.2, 0.7)), (0.5, -1.25, 2.0))
    assert oracle.transform_primitives(m, q, g["begin"], g["end"], rt) == 0
    assert sha(m) == g["means_sha"] and sha(q) == g["rot_sha"]


def test_oracle_look_at_golden(oracle):
    cam = oracle.look_at((5.0, 0.0, 0.0), (0.0, 0.0, 0.0), 554.2562584220407, 554.2562584220407, 640, 480)
    assert list(cam.pose.rotation) == GOLDEN["look_at"]["rotation"]
    assert list(cam.pose.translation) == GOLDEN["look_at"]["translation"]


# ---- anchor 1: the reference itself, bit-exact ----------------------------------------------

def test_oracle_bit_exact_vs_reference(oracle, ref):
    rng = np.random.Generator(np.random.PCG64(2024))
    for scene in range(20):  # acceptance.cpp:47-82 family
        count = int(50 + rng.integers(0, 1951))
        deg = int(rng.integers(0, 4))
        field = ref.random_field(9100 + scene, count, 3.0, 0.01, 0.05 + (scene % 5) * 0.06, deg)
        field.means[:, 2] += 3.2
        cam = ref_camera()
        nodes = golden_nodes("two" if scene % 3 == 0 else "none", count)
        sa, sb = oracle.project(field, nodes, cam), ref.project(field, nodes, cam)
        assert sa.tobytes() == sb.tobytes()
        for fn in ("rasterize", "reference_rasterize"):
            ta, tb = getattr(oracle, fn)(sa, cam), getattr(ref, fn)(sb, cam)
            assert np.array_equal(ta.rgb, tb.rgb) and np.array_equal(ta.depth, tb.depth)
            assert np.array_equal(ta.accum_alpha, tb.accum_alpha)


def test_oracle_render_vs_reference_baseline_camera(oracle, ref):
    """A BASELINE config-0 style camera (640x480, fov 60) on a 20k-splat field."""
    field = ref.random_field(555, 20000, 4.0, 0.005, 0.03, 0)
    f = 320.0 / math.tan(math.radians(30.0))
    cam = oracle.look_at((5.0, 0.0, 0.0), (0.0, 0.0, 0.0), f, f, 640, 480)
    ta = oracle.render(field, [], [cam])[0]
    tb = ref.render(field, [], [cam])[0]
    assert oracle.hash_target(ta) == oracle.hash_target(tb)


def test_oracle_transform_vs_reference(oracle, ref):
    for seed in range(5):
        f = oracle.random_field(100 + seed, 40, 2.0, 0.01, 0.3, 1)
        rt = RigidTransform(quat_normalized((0.2 + seed, -0.4, 0.1, 0.9)), (seed, -1.0, 0.5))
        m1, q1, m2, q2 = f.means.copy(), f.rotations.copy(), f.means.copy(), f.rotations.copy()
        oracle.transform_primitives(m1, q1, 3, 37, rt)
        ref.transform_primitives(m2, q2, 3, 37, rt)
        assert np.array_equal(m1, m2) and np.array_equal(q1, q2)


# ---- anchor 3b: the reference's known-answer tests on the oracle ---------------------------

def test_on_axis_footprint(oracle):  # test_raster.cpp:58-78
    field = single_prim_field((0, 0, 2), (0.1, 0.1, 0.1), 0.7)
    cam = ref_camera()
    s = oracle.project(field, [], cam)
    assert len(s) == 1
    assert s[0]["pixel_center"][0] == pytest.approx(cam.cx)
    assert s[0]["cov_xx"] == pytest.approx(25.3, rel=1e-9)
    assert s[0]["cov_yy"] == pytest.approx(25.3, rel=1e-9)
    assert abs(s[0]["cov_xy"]) < 1e-9
    assert s[0]["view_depth"] == pytest.approx(2.0)
    assert s[0]["alpha_peak"] == pytest.approx(0.7)


def test_behind_camera_culled(oracle):  # test_raster.cpp:80-87
    assert len(oracle.project(single_prim_field((0, 0, -1), (1, 1, 1), 0.5), [], ref_camera())) == 0


def test_shade_sh_known_answers(oracle):  # test_raster.cpp:98-117
    sh = [0.0] * 48
    assert oracle.shade_sh(sh, 0, (0, 0, 1))[0] == pytest.approx(0.5)
    sh[0] = 0.8
    rgb = oracle.shade_sh(sh, 0, (1, 0, 0))
    assert rgb[0] == pytest.approx(0.5 + 0.28209479177387814 * 0.8) and rgb[1] == pytest.approx(0.5)
    sh = [0.0] * 48
    for c in range(3):
        sh[c * 16 + 2] = 0.31
    up, down = oracle.shade_sh(sh, 1, (0, 0, 1)), oracle.shade_sh(sh, 1, (0, 0, -1))
    assert abs((up[0] - down[0]) - 2.0 * 0.4886025119 * 0.31) < 1e-9


def test_two_splat_recurrence(oracle):  # test_raster.cpp:119-133
    cam = ref_camera(32, 32, 50.0)
    c1, c2 = (1.0, 0.0, 0.2), (0.0, 1.0, 0.6)
    splats = np.concatenate([flat_splat(16, 16, 1.0, 0.5, c1), flat_splat(16, 16, 2.0, 0.5, c2)])
    t = oracle.rasterize(splats, cam)
    assert t.accum_alpha[9, 7] == pytest.approx(0.75)
    assert t.depth[9, 7] == pytest.approx(1.0)
    for ch in range(3):
        assert t.rgb[9, 7, ch] == pytest.approx(0.5 * c1[ch] + 0.25 * c2[ch])


def test_empty_renders_zeros(oracle):  # test_raster.cpp:135-140
    t = oracle.rasterize(np.zeros(0, dtype=flat_splat(0, 0, 1, 1, (0, 0, 0)).dtype), ref_camera(32, 32))
    assert not t.rgb.any() and not t.depth.any() and not t.accum_alpha.any()


def test_tiled_equals_brute_force(oracle):  # test_raster.cpp:142-157
    cam = ref_camera()
    for rnd in range(0, 25, 3):
        field = oracle.random_field(1000 + rnd, 100 + rnd * 17, 3.0, 0.01, 0.25, 3)
        field.means[:, 2] += 3.0
        s = oracle.project(field, [], cam)
        rgb, depth = max_diff(oracle.rasterize(s, cam), oracle.reference_rasterize(s, cam))
        assert rgb <= 1e-4 and depth <= 1e-3


@pytest.mark.parametrize("opacity", [0.3, 0.7, 0.995])
def test_single_splat_peak_alpha(oracle, opacity):  # test_raster.cpp:159-177
    field = single_prim_field((0, 0, 2), (0.05, 0.05, 0.05), opacity)
    cam = ref_camera(129, 129)
    cam.cx = cam.cy = 64.5
    t = oracle.rasterize(oracle.project(field, [], cam), cam)
    assert t.accum_alpha[64, 64] == pytest.approx(min(opacity, 0.99), rel=1e-5)


def test_monotone_alpha_without_cutoff(oracle):  # test_raster.cpp:213-229
    cam = ref_camera(64, 64)
    opt = RasterOptions(transmittance_cutoff=0.0)
    for rnd in range(5):
        field = oracle.random_field(3000 + rnd, 60, 2.0, 0.02, 0.3, 0)
        field.means[:, 2] += 2.5
        s = oracle.project(field, [], cam)
        if len(s) < 2:
            continue
        a = oracle.rasterize(s, cam, opt).accum_alpha
        b = oracle.rasterize(s[:-1], cam, opt).accum_alpha
        assert np.all(a >= b - 1e-6)


def test_rigid_equivariance(oracle):  # test_raster.cpp:231-253
    field = oracle.random_field(79, 200, 2.0, 0.02, 0.3, 2)
    nodes = [SceneNode("bg", NodeKind.background, RigidTransform(), (0, field.size()))]
    cam = ref_camera()
    cam.pose = RigidTransform(quat_from_axis_angle((0, 1, 0), 0.2), (0.1, -0.2, 4.0))
    before = oracle.rasterize(oracle.project(field, nodes, cam), cam)
    motion = RigidTransform(quat_from_axis_angle((1, 2, 3), 0.8), (5.0, -2.0, 1.0))
    moved = [SceneNode("bg", NodeKind.interactive, motion, (0, field.size()))]
    cam2 = ref_camera()
    cam2.pose = cam.pose * motion.inverse()
    after = oracle.rasterize(oracle.project(field, moved, cam2), cam2)
    rgb, depth = max_diff(before, after)
    assert rgb <= 1e-4 and depth <= 1e-3


def test_transform_identity_and_range(oracle):  # test_core_types.cpp:25-30, 99-113
    f = oracle.random_field(11, 50, 2.0, 0.01, 0.3, 2)
    m, q = f.means.copy(), f.rotations.copy()
    assert oracle.transform_primitives(m, q, 0, 50, RigidTransform()) == 0
    assert np.array_equal(m, f.means) and np.array_equal(q, f.rotations)
    assert oracle.transform_primitives(m, q, 5, 51, RigidTransform()) == 2  # validation error
    m2 = f.means.copy()
    oracle.transform_primitives(m2, f.rotations.copy(), 0, 5, RigidTransform((1, 0, 0, 0), (1, 0, 0)))
    assert np.array_equal(m2[5:], f.means[5:])
    assert np.allclose(m2[:5, 0], f.means[:5, 0] + 1)
