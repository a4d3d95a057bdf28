"""GPU GS -> TSDF (transfer.cpp) against the pinned oracle
(tests/test_transfer_pin.py pins the oracle bit-exactly to the reference).

Bars:
  * field bounds and the ring cameras: bit-exact (double, -fmad=false / host libm);
  * tsdf_fuse on the same depth maps: bit-exact grids (double per-view arithmetic in the
    reference's order; views fused in order by one thread per voxel);
  * render_depth_ring: the depth images within the north-star depth tolerance on pixels both
    sides call valid, and the validity mask (accumulated alpha >= 0.5) equal on >= 99.9% of
    pixels (the raster runs in fp32, so a pixel whose alpha sits at 0.5 may flip);
  * gaussians_to_tsdf (ring + fuse end to end): geometry bit-exact; >= 99% of voxels with the
    same weight and |tsdf diff| <= 1e-3 (the residue comes only from the fp32 depth maps).
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_21981_b200 import ValidationError
from paper_2507_21981_b200.api import GaussianField, TsdfVolume
from tests.test_transfer_pin import camera_table, same_cameras

pytestmark = pytest.mark.gpu


def fields(oracle):
    yield oracle.random_field(5, 300, 1.5, 0.02, 0.12, 0)
    yield oracle.random_field(6, 3000, 2.0, 0.01, 0.2, 3)
    f = oracle.random_field(8, 2000, 1.0, 0.005, 0.05, 1)
    f.means[:, 0] *= 3.0  # elongated box
    f.touch()
    yield f


def test_scene_bounds_bit_exact(ctx, oracle):
    for f in fields(oracle):
        lo, hi = ctx.scene_bounds(ctx.upload(f))
        olo, ohi = oracle.field_bounds(f)
        assert lo == olo and hi == ohi


def test_depth_ring_matches_oracle(ctx, oracle):
    for f, (nv, rad, res) in zip(fields(oracle), [(8, 5.0, 48), (10, 6.5, 64), (9, 7.0, 40)]):
        scene = ctx.upload(f)
        cams, depth = ctx.render_depth_ring(scene, nv, rad, res)
        ocams, odepth = oracle.render_depth_ring(f, nv, rad, res)
        assert same_cameras(cams, ocams)
        valid, ovalid = depth > 0, odepth > 0
        assert np.mean(valid == ovalid) >= 0.999
        both = valid & ovalid
        assert both.mean() > 0.05
        rel = np.abs(depth[both].astype(np.float64) - odepth[both]) / np.abs(odepth[both])
        assert np.mean(rel <= 1e-3) >= 0.999, float(rel.max())


def test_depth_ring_device_output(ctx, oracle):
    import torch
    f = oracle.random_field(9, 500, 1.5, 0.02, 0.1, 2)
    scene = ctx.upload(f)
    _, host = ctx.render_depth_ring(scene, 8, 5.0, 32)
    dev = torch.full((24, 32, 32), -7.0, dtype=torch.float32, device="cuda:0")
    ctx.render_depth_ring(scene, 8, 5.0, 32, device_out=dev.data_ptr())
    assert np.array_equal(dev.cpu().numpy(), host)


def test_tsdf_fuse_bit_exact_on_oracle_depth(ctx, oracle):
    f = oracle.random_field(13, 800, 1.5, 0.02, 0.1, 1)
    cams, depth = oracle.render_depth_ring(f, 8, 5.0, 48)
    ovol = oracle.tsdf_create((-1.7, -1.8, -1.6), 0.06, (57, 60, 55), 0.18)
    for k in range(len(cams)):
        oracle.tsdf_fuse(ovol, cams[k], depth[k])
    # device grids, all views in one call (host depth)
    vol = TsdfVolume(ovol.origin, ovol.voxel_size, ovol.dims, ovol.truncation).device_grids()
    ctx.tsdf_fuse(vol, list(cams), depth)
    got = vol.to_numpy()
    assert np.array_equal(got.tsdf, ovol.tsdf) and np.array_equal(got.weights, ovol.weights)
    # the same in two calls with device depth: identical to one batched call
    import torch
    vol2 = TsdfVolume(ovol.origin, ovol.voxel_size, ovol.dims, ovol.truncation).device_grids()
    d = torch.from_numpy(depth).cuda()
    ctx.tsdf_fuse(vol2, list(cams[:10]), d.data_ptr())
    ctx.tsdf_fuse(vol2, list(cams[10:]), d[10:].contiguous().data_ptr())
    got2 = vol2.to_numpy()
    assert np.array_equal(got2.tsdf, ovol.tsdf) and np.array_equal(got2.weights, ovol.weights)


def test_tsdf_fuse_adversarial_bit_exact(ctx, oracle):
    rng = np.random.default_rng(17)
    ovol = oracle.tsdf_create((-1.0, -1.2, -0.9), 0.07, (30, 33, 27), 0.21)
    vol = TsdfVolume(ovol.origin, ovol.voxel_size, ovol.dims, ovol.truncation).device_grids()
    cams, depths = [], []
    for k in range(9):
        eye = rng.uniform(-4, 4, 3) if k != 4 else np.array([0.2, 0.1, 0.0])  # inside: z <= 0
        c = oracle.look_at(eye, (0.0, 0.0, 0.0), float(rng.uniform(20, 60)), float(rng.uniform(20, 60)),
                           64, 48)
        d = rng.uniform(0.5, 6.0, (48, 64)).astype(np.float32)
        d[rng.random((48, 64)) < 0.2] = 0.0
        d[rng.random((48, 64)) < 0.02] = -1.0
        cams.append(c)
        depths.append(d)
        oracle.tsdf_fuse(ovol, c, d)
    ctx.tsdf_fuse(vol, cams, np.stack(depths))
    got = vol.to_numpy()
    assert np.array_equal(got.tsdf, ovol.tsdf) and np.array_equal(got.weights, ovol.weights)


@pytest.mark.parametrize("seed,deg,voxel", [(21, 0, 0.12), (22, 3, 0.05)])
def test_gaussians_to_tsdf_matches_oracle(ctx, oracle, seed, deg, voxel):
    f = oracle.random_field(seed, 1500, 1.5, 0.02, 0.1, deg)
    vol = ctx.gaussians_to_tsdf(ctx.upload(f), voxel).to_numpy()
    ovol = oracle.gaussians_to_tsdf(f, voxel)
    assert vol.dims == ovol.dims and vol.origin == ovol.origin and vol.truncation == ovol.truncation
    same_w = vol.weights == ovol.weights
    close = np.abs(vol.tsdf - ovol.tsdf) <= 1e-3
    assert np.mean(same_w & close) >= 0.99, (float(np.mean(same_w)), float(np.mean(close)))
    assert (vol.weights > 0).mean() > 0.5


def test_transfer_validation(ctx, oracle):
    empty = GaussianField(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0),
                          np.zeros((0, 48)), 0)
    f = oracle.random_field(3, 50, 1.0, 0.02, 0.1, 0)
    scene = ctx.upload(f)
    with pytest.raises(ValidationError):
        ctx.render_depth_ring(ctx.upload(empty), 8, 5.0, 32)
    for nv, rad, res in [(7, 5.0, 32), (8, 0.0, 32), (8, float("nan"), 32), (8, 5.0, 8)]:
        with pytest.raises(ValidationError):
            ctx.render_depth_ring(scene, nv, rad, res)
    with pytest.raises(ValidationError):
        ctx.gaussians_to_tsdf(scene, 0.0)
    with pytest.raises(ValidationError):
        ctx.gaussians_to_tsdf(ctx.upload(empty), 0.1)
    lo, hi = ctx.scene_bounds(ctx.upload(empty))
    assert lo == (np.inf,) * 3 and hi == (-np.inf,) * 3
    vol = TsdfVolume((0, 0, 0), 0.1, (4, 4, 4), 0.3)  # no grids
    with pytest.raises(ValidationError):
        ctx.tsdf_reset(vol)
    vol.device_grids()
    ctx.tsdf_reset(vol)
    bad = oracle.look_at((3, 0, 0), (0, 0, 0), 20.0, 20.0, 8, 8)  # resolution below 16
    with pytest.raises(ValidationError):
        ctx.tsdf_fuse(vol, [bad], np.ones((1, 8, 8), np.float32))
    assert camera_table([bad]).shape == (1, 15)
