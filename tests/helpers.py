"""Shared test helpers (scene builders mirroring the reference tests, comparison metrics)."""
from __future__ import annotations

import numpy as np

from paper_2507_21981_b200.abi import SPLAT_DTYPE
from paper_2507_21981_b200.api import CameraModel, GaussianField, RigidTransform


def ref_camera(w=128, h=128, f=100.0) -> CameraModel:
    """test_raster.cpp:18-28."""
    return CameraModel(fx=f, fy=f, cx=w * 0.5, cy=h * 0.5, width=w, height=h, near=0.05, far=100.0)


def flat_splat(u, v, depth, alpha, rgb):
    """test_raster.cpp:30-41: zero inverse covariance, alpha constant over the footprint."""
    s = np.zeros(1, dtype=SPLAT_DTYPE)
    s["pixel_center"] = (u, v)
    s["cov_xx"] = s["cov_yy"] = 1e12
    s["view_depth"] = depth
    s["alpha_peak"] = alpha
    s["rgb"] = rgb
    s["radius"] = 1e6
    return s


def single_prim_field(mean, scale, opacity, rotation=(1.0, 0.0, 0.0, 0.0), sh_degree=0):
    sh = np.zeros((1, 48))
    return GaussianField(np.array([mean], float), np.array([scale], float), np.array([rotation], float),
                         np.array([opacity], float), sh, sh_degree)


def max_diff(a, b):
    """(max |rgb diff|, max |depth diff|), test_raster.cpp:43-54."""
    return (float(np.max(np.abs(a.rgb.astype(np.float64) - b.rgb))),
            float(np.max(np.abs(a.depth.astype(np.float64) - b.depth))))


def parity_stats(gpu, ref, rgb_tol=2e-3, depth_rel=1e-3):
    """Fraction of pixels within the north-star tolerances (RGB max-abs per pixel, depth
    relative with a 1e-4 m absolute floor for near-empty pixels)."""
    drgb = np.max(np.abs(gpu.rgb.astype(np.float64) - ref.rgb), axis=-1)
    dd = np.abs(gpu.depth.astype(np.float64) - ref.depth)
    rel = dd / np.maximum(np.abs(ref.depth.astype(np.float64)), 1e-1)
    ok_rgb = float(np.mean(drgb <= rgb_tol))
    ok_depth = float(np.mean((rel <= depth_rel) | (dd <= 1e-4)))
    da = np.abs(gpu.accum_alpha.astype(np.float64) - ref.accum_alpha)
    return dict(rgb_ok=ok_rgb, depth_ok=ok_depth, rgb_max=float(drgb.max()),
                depth_rel_max=float(rel.max()), alpha_max=float(da.max()),
                rgb_p999=float(np.quantile(drgb, 0.999)))


def shifted(field: GaussianField, dz: float) -> GaussianField:
    field.means[:, 2] += dz
    field.touch()
    return field


IDENTITY = RigidTransform()
