"""GPU parity of the output encoders against the pinned oracle
(tests/test_encode_pin.py pins the oracle to the reference's image_io.cpp writers).

Bar: bit-exact bytes. The encoders are byte work: quantize8 / lround in double, the sRGB code
via the host-built threshold table, big-endian u16 depth, PFM rows bottom-up.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_21981_b200 import EncodeOptions, RenderTarget, ValidationError
from paper_2507_21981_b200.api import RasterOptions
from tests.helpers import ref_camera
from tests.test_encode_pin import ALL, adversarial_values

pytestmark = pytest.mark.gpu

FLAG_SETS = [ALL, EncodeOptions.RGB8, EncodeOptions.ALPHA8 | EncodeOptions.DEPTH16,
             EncodeOptions.RGB8 | EncodeOptions.DEPTH_PFM, EncodeOptions.DEPTH_PFM]


def oracle_blob(oracle, targets, opts):
    parts = []
    for t in targets:
        h, w = t.depth.shape
        parts.append(oracle.encode(opts.flags, opts.srgb, opts.depth_scale, w, h, t.rgb, t.depth,
                                   t.accum_alpha))
    return np.concatenate(parts) if parts else np.zeros(0, np.uint8)


def adversarial_target(rng, w, h):
    n = w * h
    v = adversarial_values(rng, 4 * n)
    rgb = rng.choice(v, 3 * n).reshape(h, w, 3).astype(np.float32)
    alpha = rng.choice(v, n).reshape(h, w).astype(np.float32)
    depth = np.concatenate([v * 70.0, rng.uniform(0, 100, n).astype(np.float32),
                            np.array([65.5355, 65.5345, 1e20, -1e20, np.nan], np.float32)])
    depth = rng.choice(depth, n).reshape(h, w).astype(np.float32)
    return RenderTarget(rgb, depth, alpha)


@pytest.mark.parametrize("w,h", [(64, 48), (17, 19), (1, 1)])
def test_encode_target_bit_exact(ctx, oracle, w, h):
    rng = np.random.default_rng(w * 1000 + h)
    t = adversarial_target(rng, w, h)
    for flags in FLAG_SETS:
        for srgb in (True, False):
            for scale in (1000.0, 1.0, -3.0):
                o = EncodeOptions(flags, srgb, scale)
                got = ctx.encode_target(t, o)
                want = oracle_blob(oracle, [t], o)
                assert np.array_equal(got, want), (flags, srgb, scale)


def test_encode_validation(ctx):
    t = RenderTarget.empty(16, 16)
    with pytest.raises(ValidationError):
        ctx.encode_target(t, EncodeOptions(0))
    with pytest.raises(ValidationError):
        ctx.encode_target(t, EncodeOptions(ALL | 64))
    with pytest.raises(ValidationError):
        ctx.encode_target(t, EncodeOptions(EncodeOptions.DEPTH16, depth_scale=float("nan")))


def scene_and_cameras(oracle, n_prims=6000, seed=31):
    field = oracle.random_field(seed, n_prims, 3.0, 0.01, 0.25, 3)
    field.means[:, 2] += 3.0
    cams = [ref_camera(160, 128, 110.0), ref_camera(33, 17, 25.0), ref_camera(64, 48, 60.0)]
    return field, cams


@pytest.mark.parametrize("normalize", [False, True])
def test_render_encoded_equals_render_then_encode(ctx, oracle, normalize):
    """The fused raster epilogue writes exactly the bytes the reference writers would produce
    from the float targets of the same render."""
    field, cams = scene_and_cameras(oracle)
    scene = ctx.upload(field)
    ropt = RasterOptions(normalize_depth=normalize)
    targets = ctx.render(scene, [], cams, ropt)
    assert any(t.accum_alpha.max() > 0.5 for t in targets)
    for flags in FLAG_SETS:
        o = EncodeOptions(flags, True, 1000.0)
        want = oracle_blob(oracle, targets, o)
        assert np.array_equal(ctx.render_encoded(scene, [], cams, ropt, o), want), flags
    # only the encoded bytes crossed to the host
    assert ctx.stats()["d2h_bytes"] == len(want)


def test_encode_of_device_output_and_device_destination(ctx, oracle):
    import torch
    field, cams = scene_and_cameras(oracle, seed=32)
    scene = ctx.upload(field)
    targets = ctx.render(scene, [], cams)
    o = EncodeOptions()
    want = oracle_blob(oracle, targets, o)
    n = sum(5 * c.width * c.height for c in cams)
    dev = torch.zeros(n, dtype=torch.float32, device="cuda:0")
    ctx.render_device(scene, [], cams, None, dev.data_ptr())
    ctx.synchronize()
    assert np.array_equal(ctx.encode(dev.data_ptr(), cams, o), want)
    out = torch.zeros(len(want), dtype=torch.uint8, device="cuda:0")
    ctx.encode(dev.data_ptr(), cams, o, device_out=out.data_ptr())
    ctx.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)
    out.zero_()
    ctx.render_encoded(scene, [], cams, None, o, device_out=out.data_ptr())
    ctx.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)
    views = o.split(want, cams)
    assert views[1]["rgb8"].shape == (17, 33, 3) and views[1]["depth16"].dtype == np.uint16
    assert np.array_equal(views[0]["depth_pfm"][::-1], targets[0].depth)


def test_render_encoded_camera_groups(oracle, monkeypatch):
    """40 cameras of mixed sizes, run as 3 camera groups (GSIM_GPU_GROUP_SLOTS budget): the
    encoded blocks still follow the batch's camera order."""
    from paper_2507_21981_b200 import Context
    field = oracle.random_field(41, 3000, 3.0, 0.01, 0.3, 1)
    field.means[:, 2] += 3.0
    cams = [ref_camera(32 + (k % 3) * 16, 32, 30.0 + k) for k in range(40)]
    monkeypatch.setenv("GSIM_GPU_GROUP_SLOTS", str(16 * 3000))
    ctx = Context(0)
    scene = ctx.upload(field)
    o = EncodeOptions(ALL, True, 1000.0)
    got = ctx.render_encoded(scene, [], cams, None, o)
    assert ctx.stats()["groups"] == 3
    want = oracle_blob(oracle, ctx.render(scene, [], cams), o)
    assert np.array_equal(got, want)


def test_render_encoded_overflow_rerun(ctx, oracle, monkeypatch):
    """Pair-buffer overflow found by the deferred check re-runs scatter + fused raster into the
    same encoded destination."""
    import torch
    from paper_2507_21981_b200 import Context
    field = oracle.random_field(99, 4000, 3.0, 0.01, 0.3, 2)
    field.means[:, 2] += 3.0
    cams = [ref_camera(160, 128, 110.0), ref_camera(96, 64, 70.0)]
    o = EncodeOptions()
    want = oracle_blob(oracle, ctx.render(ctx.upload(field), [], cams), o)
    monkeypatch.setenv("GSIM_GPU_INITIAL_PAIR_CAPACITY", "1000")
    small = Context(0)
    s = small.upload(field)
    assert np.array_equal(small.render_encoded(s, [], cams, None, o), want)  # synchronous
    out = torch.zeros(len(want), dtype=torch.uint8, device="cuda:0")
    monkeypatch.setenv("GSIM_GPU_INITIAL_PAIR_CAPACITY", "1000")
    small2 = Context(0)
    s2 = small2.upload(field)
    small2.render_encoded(s2, [], cams, None, o, device_out=out.data_ptr())
    small2.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)
