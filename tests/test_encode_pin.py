"""§8f rows 1-2 pins on CPU: the oracle's restatement of the reference's output writers
(image_io.cpp) and pose playback (pose_stream.cpp / math.hpp slerp) against the reference
itself, compiled from its sources into oracle/_ref (image_io.cpp against oracle/png_capture,
which records the row bytes handed to libpng). Also checks the product library's sRGB
threshold table, which needs no GPU."""
import ctypes as C

import numpy as np
import pytest

from paper_2507_21981_b200 import abi
from paper_2507_21981_b200.api import RigidTransform

ALL = abi.GSIM_ENCODE_RGB8 | abi.GSIM_ENCODE_ALPHA8 | abi.GSIM_ENCODE_DEPTH16 | abi.GSIM_ENCODE_DEPTH_PFM


def adversarial_values(rng, n):
    """Values around every quantisation step, the sRGB knee, the clamps and the specials."""
    specials = np.array([0.0, -0.0, 1.0, -1.0, 2.0, 0.5 / 255, 1.5 / 255, 254.5 / 255, 0.0031308,
                         0.04045, np.nan, np.inf, -np.inf, 1e-30, -1e-30, 0.999999, 1.0000001],
                        dtype=np.float32)
    steps = (np.arange(256, dtype=np.float64) + 0.5) / 255.0
    around = np.concatenate([np.nextafter(steps.astype(np.float32), np.float32(-1)),
                             steps.astype(np.float32),
                             np.nextafter(steps.astype(np.float32), np.float32(2))])
    rand = rng.uniform(-0.1, 1.1, n).astype(np.float32)
    return np.concatenate([specials, around, rand]).astype(np.float32)


def test_linear_to_srgb_matches_reference(oracle, ref):
    rng = np.random.default_rng(1)
    for v in list(rng.uniform(-0.5, 1.5, 2000)) + [0.0, 0.0031308, 0.00313081, 1.0, float("nan")]:
        a, b = oracle.linear_to_srgb(v), ref.linear_to_srgb(v)
        assert (a == b) or (np.isnan(a) and np.isnan(b)), v


@pytest.mark.parametrize("srgb", [True, False])
def test_rgb8_bytes_match_reference_writer(oracle, ref, srgb):
    rng = np.random.default_rng(2 + srgb)
    vals = adversarial_values(rng, 3000)
    vals = np.concatenate([vals, np.zeros((-len(vals)) % 3, np.float32)])
    w, h = 1, len(vals) // 3
    got = oracle.encode(abi.GSIM_ENCODE_RGB8, srgb, 1000.0, w, h, rgb=vals)
    want = ref.png_rgb8(vals, w, h, srgb)
    assert np.array_equal(got, want)


def test_gray8_and_gray16_bytes_match_reference_writers(oracle, ref):
    rng = np.random.default_rng(4)
    vals = adversarial_values(rng, 3000)
    w, h = len(vals), 1
    assert np.array_equal(oracle.encode(abi.GSIM_ENCODE_ALPHA8, 0, 1.0, w, h, alpha=vals),
                          ref.png_gray8(vals, w, h))
    depth = np.concatenate([vals * 70.0, np.array([65.5355, 65.5345, -0.0004, 1e15, 1e20, -1e20],
                                                  dtype=np.float32),
                            rng.uniform(0, 120, 500).astype(np.float32)]).astype(np.float32)
    for scale in (1000.0, 1.0, 256.0, 1e-3, -1000.0):
        got = oracle.encode(abi.GSIM_ENCODE_DEPTH16, 0, scale, len(depth), 1, depth=depth)
        want = ref.png_gray16(depth, len(depth), 1, scale)
        assert np.array_equal(got, want), scale


def test_pfm_body_matches_reference_writer(oracle, ref, tmp_path):
    rng = np.random.default_rng(5)
    w, h = 37, 23
    depth = rng.uniform(0, 50, w * h).astype(np.float32)
    depth[::17] = np.nan
    got = oracle.encode(abi.GSIM_ENCODE_DEPTH_PFM, 0, 1.0, w, h, depth=depth)
    want = ref.encode(abi.GSIM_ENCODE_DEPTH_PFM, 0, 1.0, w, h, depth=depth, tmpdir=tmp_path)
    assert np.array_equal(got, want)


def test_full_blob_layout_matches_reference_writers(oracle, ref, tmp_path):
    rng = np.random.default_rng(6)
    w, h = 19, 17
    rgb = rng.uniform(-0.05, 1.05, (h, w, 3)).astype(np.float32)
    depth = rng.uniform(0, 30, (h, w)).astype(np.float32)
    alpha = rng.uniform(0, 1, (h, w)).astype(np.float32)
    for flags in (ALL, abi.GSIM_ENCODE_RGB8 | abi.GSIM_ENCODE_DEPTH_PFM,
                  abi.GSIM_ENCODE_ALPHA8 | abi.GSIM_ENCODE_DEPTH16):
        for srgb in (0, 1):
            got = oracle.encode(flags, srgb, 1000.0, w, h, rgb, depth, alpha)
            want = ref.encode(flags, srgb, 1000.0, w, h, rgb, depth, alpha, tmpdir=tmp_path)
            assert np.array_equal(got, want), (flags, srgb)


def test_library_srgb_thresholds_step_exactly_where_the_reference_does(ref):
    """thresholds[k] is the first float whose reference code is >= k (the GPU's lookup table)."""
    lib = abi.load_library()
    thr = (C.c_float * 256)()
    lib.gsim_gpu_srgb_thresholds(thr)
    t = np.array(thr[:], dtype=np.float32)
    assert t[0] == -np.inf and np.all(np.diff(t[1:]) > 0)
    at = ref.png_rgb8(np.repeat(t[1:], 3), 1, 255, True)[::3]
    below = ref.png_rgb8(np.repeat(np.nextafter(t[1:], np.float32(-1)), 3), 1, 255, True)[::3]
    k = np.arange(1, 256)
    assert np.all(at >= k)
    assert np.all(below < k)


def test_encoded_bytes():
    lib = abi.load_library()
    assert lib.gsim_gpu_encoded_bytes(ALL, 640, 480) == 10 * 640 * 480
    assert lib.gsim_gpu_encoded_bytes(abi.GSIM_ENCODE_RGB8, 17, 3) == 3 * 17 * 3
    assert lib.gsim_gpu_encoded_bytes(64, 16, 16) == 0
    assert lib.gsim_gpu_encoded_bytes(ALL, 0, 16) == 0


# ---- pose playback ------------------------------------------------------------------------

def random_track(rng, n, t0=0.0, dup=False):
    dt = rng.uniform(0.01, 0.5, n)
    if dup and n > 3:
        dt[2] = 0.0  # repeated timestamp (legal: times may not decrease)
    t = t0 + np.cumsum(dt)
    p = rng.uniform(-3, 3, (n, 3))
    q = rng.normal(size=(n, 4)) * rng.uniform(0.5, 2.0, (n, 1))  # unnormalised on purpose
    if n > 1:
        q[1] = -q[0] * 1.7      # antipodal neighbour: shortest-arc sign flip
    if n > 5:
        q[5] = q[4] * (1 + 1e-14)  # nearly parallel: nlerp branch
    return t, p, q


def test_slerp_matches_reference(oracle, ref):
    rng = np.random.default_rng(7)
    for _ in range(300):
        a = rng.normal(size=4); a /= np.linalg.norm(a)
        b = rng.normal(size=4); b /= np.linalg.norm(b)
        if rng.uniform() < 0.2:
            b = a + rng.normal(size=4) * 1e-9
        t = rng.uniform(-0.2, 1.2)
        assert np.array_equal(oracle.slerp(a, b, t), ref.slerp(a, b, t))


def test_pose_sample_matches_reference(oracle, ref):
    rng = np.random.default_rng(8)
    init = RigidTransform((0.9, 0.1, -0.3, 0.2), (1.0, 2.0, 3.0))
    for trial in range(40):
        n = int(rng.integers(1, 40))
        t, p, q = random_track(rng, n, dup=trial % 3 == 0)
        ts = np.concatenate([rng.uniform(t[0] - 1, t[-1] + 1, 200), t, [t[0] - 1e-12, t[-1]]])
        rc_o, o = oracle.pose_sample(t, p, q, init, ts)
        rc_r, r = ref.pose_sample(t, p, q, init, ts)
        assert rc_o == rc_r == 0
        assert np.array_equal(o, r), trial


def test_pose_sample_validation_matches_reference(oracle, ref):
    init = RigidTransform()
    t = np.array([0.0, 1.0, 0.5])  # decreasing
    p = np.zeros((3, 3)); q = np.tile([1.0, 0, 0, 0], (3, 1))
    assert oracle.pose_sample(t, p, q, init, [0.2])[0] == ref.pose_sample(t, p, q, init, [0.2])[0] == 2
    t = np.array([0.0, np.inf])
    assert oracle.pose_sample(t, p[:2], q[:2], init, [0.2])[0] == 2
    assert ref.pose_sample(t, p[:2], q[:2], init, [0.2])[0] == 2
    q2 = q[:2].copy(); q2[1, 2] = np.nan
    assert oracle.pose_sample(np.array([0.0, 1.0]), p[:2], q2, init, [0.2])[0] == 2
    assert ref.pose_sample(np.array([0.0, 1.0]), p[:2], q2, init, [0.2])[0] == 2
    # empty track -> initial pose everywhere
    rc, o = oracle.pose_sample(np.zeros(0), np.zeros((0, 3)), np.zeros((0, 4)), init, [0.0, 5.0])
    assert rc == 0 and np.array_equal(o[0], [1, 0, 0, 0, 0, 0, 0])


# ---- splat PLY (splat_ply.cpp:40-162) ------------------------------------------------------

PLY_FIELDS = ("means", "scales", "rotations", "opacities", "sh")


def ply_bytes(n, degree, rows=None, header_edit=None, payload_floats=None, seed=0):
    """A splat PLY in the reference's layout (header + float rows), editable for error cases."""
    K = (degree + 1) ** 2
    props = ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
    props += [f"f_rest_{i}" for i in range(3 * (K - 1))]
    props += ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    lines = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    lines += [f"property float {p}" for p in props] + ["end_header"]
    if header_edit:
        lines = header_edit(lines)
    if rows is None:
        rng = np.random.default_rng(seed)
        rows = rng.normal(size=(n, len(props))).astype(np.float32)
        rows[:, -4:] = rng.normal(size=(n, 4))  # unnormalised rotations
        rows[: n // 3, -4:] /= np.linalg.norm(rows[: n // 3, -4:], axis=1, keepdims=True)
        rows[:, -7:-4] = rng.uniform(-6, -1, (n, 3))  # log scales
    data = np.asarray(rows, dtype=np.float32).tobytes()
    if payload_floats is not None:
        data = data[: 4 * payload_floats]
    return ("\n".join(lines) + "\n").encode() + data


def test_ply_loader_matches_reference(oracle, ref, tmp_path):
    for degree in range(4):
        for n in (0, 1, 257):
            p = tmp_path / f"f{degree}_{n}.ply"
            p.write_bytes(ply_bytes(n, degree, seed=degree * 10 + n))
            rc_o, fo = oracle.load_splat_ply(p)
            rc_r, fr = ref.load_splat_ply(p)
            assert rc_o == rc_r == 0, (degree, n)
            assert fo.sh_degree == fr.sh_degree == degree
            for k in PLY_FIELDS:
                assert np.array_equal(getattr(fo, k), getattr(fr, k)), (degree, n, k)
    # the reference's own writer -> both loaders (save->load is exact, splat_ply.hpp:22-24)
    field = oracle.random_field(77, 300, 2.0, 0.01, 0.3, 3)
    p = tmp_path / "saved.ply"
    assert ref.save_splat_ply(p, field) == 0
    rc_o, fo = oracle.load_splat_ply(p)
    rc_r, fr = ref.load_splat_ply(p)
    assert rc_o == rc_r == 0
    for k in PLY_FIELDS:
        assert np.array_equal(getattr(fo, k), getattr(fr, k)), k


def ply_error_cases(n=20, degree=1):
    K = (degree + 1) ** 2
    stride = 17 + 3 * (K - 1)
    rng = np.random.default_rng(3)
    good = np.frombuffer(ply_bytes(n, degree, seed=3).split(b"end_header\n", 1)[1], np.float32).reshape(n, stride)

    def rows_with(i, col, v):
        r = good.copy()
        r[i, col] = v
        return r

    def edit(fn):
        return lambda lines: fn(list(lines))

    return {
        "magic": ply_bytes(n, degree, header_edit=edit(lambda l: ["plyx"] + l[1:])),
        "ascii": ply_bytes(n, degree, header_edit=edit(lambda l: [l[0], "format ascii 1.0"] + l[2:])),
        "no_end": ply_bytes(0, degree, header_edit=edit(lambda l: l[:-1])),
        "no_format": ply_bytes(n, degree, header_edit=edit(lambda l: [l[0]] + l[2:])),
        "face": ply_bytes(n, degree, header_edit=edit(lambda l: l[:2] + ["element face 3"] + l[3:])),
        "double": ply_bytes(n, degree, header_edit=edit(lambda l: l[:3] + ["property double x"] + l[4:])),
        "order": ply_bytes(n, degree, header_edit=edit(lambda l: l[:3] + [l[4], l[3]] + l[5:])),
        "extra": ply_bytes(n, degree, header_edit=edit(lambda l: l[:-1] + ["property float extra", l[-1]])),
        "rest5": ply_bytes(n, degree, header_edit=edit(lambda l: [x for x in l if x != "property float f_rest_8"])),
        "token": ply_bytes(n, degree, header_edit=edit(lambda l: l[:2] + ["bogus"] + l[2:])),
        "truncated": ply_bytes(n, degree, payload_floats=n * stride - 1),
        "nonfinite": ply_bytes(n, degree, rows=rows_with(7, 4, np.nan)),
        "saturated": ply_bytes(n, degree, rows=rows_with(5, stride - 8, 60.0)),
        "scale_inf": ply_bytes(n, degree, rows=rows_with(9, stride - 6, 800.0)),
        "zero_rot": ply_bytes(n, degree, rows=np.concatenate([good[:4], np.hstack([good[4:5, :-4], np.zeros((1, 4), np.float32)]), good[5:]])),
        "comment_crlf": ply_bytes(n, degree, header_edit=edit(lambda l: [l[0], "comment hi\r"] + [x + "\r" for x in l[1:]])),
    }


def test_ply_loader_errors_match_reference(oracle, ref, tmp_path):
    for name, data in ply_error_cases().items():
        p = tmp_path / f"{name}.ply"
        p.write_bytes(data)
        rc_o, _ = oracle.load_splat_ply(p)
        rc_r, _ = ref.load_splat_ply(p)
        assert rc_o == rc_r, (name, rc_o, rc_r)
        assert rc_r == (0 if name == "comment_crlf" else 2), (name, rc_r)
    rc_o, _ = oracle.load_splat_ply(tmp_path / "missing.ply")
    rc_r, _ = ref.load_splat_ply(tmp_path / "missing.ply")
    assert rc_o == rc_r == 1
