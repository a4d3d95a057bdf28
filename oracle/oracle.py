"""ctypes front-end of the CPU checker. TEST INFRASTRUCTURE ONLY.

    Oracle  -> oracle/liboracle.so        our plain-C restatement (gsim_oracle.c)
    Ref     -> oracle/_ref/libgsim_ref.so the unmodified reference, compiled from its sources

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may use
this module, and only as the checker or the timed CPU baseline — never as a product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2507_21981_b200 import abi
from paper_2507_21981_b200.api import (CameraModel, GaussianField, RasterOptions, RenderTarget,
                                       SceneNode, TsdfVolume)

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libgsim_ref.so"

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p


def build_oracle(with_ref: bool = True) -> None:
    """make -C oracle (liboracle.so always; _ref only where /root/reference exists)."""
    target = "all" if with_ref else str(ORACLE_LIB)
    subprocess.run(["make", "-s", "-C", str(HERE), "-f", str(HERE / "Makefile"), target], check=True)


def _cams(cameras):
    arr = (abi.gsim_camera * max(len(cameras), 1))()
    for k, c in enumerate(cameras):
        arr[k] = c.to_c() if isinstance(c, CameraModel) else c
    return arr


def _nodes(nodes):
    arr = (abi.gsim_node * max(len(nodes), 1))()
    for k, n in enumerate(nodes):
        arr[k] = n.to_c() if isinstance(n, SceneNode) else n
    return arr


class OracleStatus(ValueError):
    """Non-zero status (1 io, 2 validation) from the oracle or the reference shim."""

    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: status {status}")
        self.status = status


def _ok(status: int, what: str) -> None:
    if status != 0:
        raise OracleStatus(status, what)


def _vec3(v):
    return (C.c_double * 3)(*[float(x) for x in v])


def _target(width, height):
    return RenderTarget.empty(width, height)


class Oracle:
    """Our C restatement of the reference path (liboracle.so)."""

    def __init__(self, path: Path | None = None):
        p = Path(path) if path else ORACLE_LIB
        if not p.exists():
            build_oracle(with_ref=False)
        self.lib = C.CDLL(str(p))
        L = self.lib
        L.gso_project.argtypes = [C.POINTER(abi.gsim_field_view), C.POINTER(abi.gsim_node), C.c_uint64,
                                  C.POINTER(abi.gsim_camera), _vp, C.c_uint64, _u64p]
        L.gso_rasterize.argtypes = [_vp, C.c_uint64, C.POINTER(abi.gsim_camera),
                                    C.POINTER(abi.gsim_raster_options), _fp, _fp, _fp]
        L.gso_reference_rasterize.argtypes = L.gso_rasterize.argtypes
        L.gso_rasterize_lists.argtypes = [_vp, C.c_uint64, C.POINTER(abi.gsim_camera), _u32p, _u32p,
                                          C.c_uint64, _u64p]
        L.gso_render.argtypes = [C.POINTER(abi.gsim_field_view), C.POINTER(abi.gsim_node), C.c_uint64,
                                 C.POINTER(abi.gsim_camera), C.c_uint64,
                                 C.POINTER(abi.gsim_raster_options), C.POINTER(abi.gsim_target)]
        L.gso_transform_primitives.argtypes = [_dp, _dp, C.c_uint64, C.c_uint64, C.c_uint64,
                                               C.POINTER(abi.gsim_rigid)]
        L.gso_random_field.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                       C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.gso_hash_target.argtypes = [_fp, _fp, _fp, C.c_int, C.c_int, C.c_uint64]
        L.gso_hash_target.restype = C.c_uint64
        L.gso_look_at.argtypes = [_dp, _dp, C.c_double, C.c_double, C.c_int, C.c_int, _dp,
                                  C.POINTER(abi.gsim_camera)]
        L.gso_shade_sh.argtypes = [_dp, C.c_int, _dp, _dp]
        L.gso_mt_seed.argtypes = [_vp, C.c_uint64]
        L.gso_mt_next.argtypes = [_vp]
        L.gso_mt_next.restype = C.c_uint64
        L.gso_linear_to_srgb.argtypes = [C.c_double]
        L.gso_linear_to_srgb.restype = C.c_double
        L.gso_encoded_bytes.argtypes = [C.c_uint32, C.c_int, C.c_int]
        L.gso_encoded_bytes.restype = C.c_uint64
        L.gso_encode.argtypes = [C.c_uint32, C.c_int, C.c_double, C.c_int, C.c_int, _fp, _fp, _fp,
                                 C.POINTER(C.c_uint8)]
        L.gso_load_splat_ply.argtypes = [C.c_char_p, C.c_uint64, _u64p, C.POINTER(C.c_int), _dp, _dp,
                                         _dp, _dp, _dp]
        L.gso_slerp.argtypes = [_dp, _dp, C.c_double, _dp]
        vol = C.POINTER(abi.gsim_tsdf_volume)
        L.gso_field_bounds.argtypes = [C.POINTER(abi.gsim_field_view), _dp, _dp]
        L.gso_depth_ring_cameras.argtypes = [_dp, _dp, C.c_int, C.c_double, C.c_int,
                                             C.POINTER(abi.gsim_camera)]
        L.gso_render_depth_ring.argtypes = [C.POINTER(abi.gsim_field_view), C.c_int, C.c_double,
                                            C.c_int, C.POINTER(abi.gsim_camera), _fp]
        L.gso_tsdf_create.argtypes = [_dp, C.c_double, C.POINTER(C.c_int32), C.c_double, vol]
        L.gso_tsdf_fuse.argtypes = [vol, C.POINTER(abi.gsim_camera), _fp, C.c_int, C.c_int]
        L.gso_gaussians_to_tsdf.argtypes = [C.POINTER(abi.gsim_field_view), C.c_double, vol]
        L.gso_trace_rays.argtypes = [C.POINTER(abi.gsim_field_view), C.POINTER(abi.gsim_node),
                                     C.c_uint64, _dp, _dp, _dp, C.c_uint64, C.c_double,
                                     C.POINTER(C.c_uint8), _dp, _dp]
        L.gso_lidar_scan.argtypes = [C.POINTER(abi.gsim_field_view), C.POINTER(abi.gsim_node),
                                     C.c_uint64, C.POINTER(abi.gsim_lidar), _dp, _u32p, _dp,
                                     C.c_uint64, _u64p]
        L.gso_pose_sample.argtypes = [_dp, _dp, _dp, C.c_uint64, C.POINTER(abi.gsim_rigid), _dp,
                                      C.c_uint64, C.POINTER(abi.gsim_rigid)]

    # -- fixtures ----------------------------------------------------------------------------
    def random_field(self, seed, count, box_extent, scale_lo, scale_hi, sh_degree) -> GaussianField:
        """oracle::random_field (tests/support/test_oracles.cpp:144-168), bit-exact."""
        m = np.zeros((count, 3)); s = np.zeros((count, 3)); q = np.zeros((count, 4))
        o = np.zeros(count); sh = np.zeros((count, 48))
        self.lib.gso_random_field(seed, count, box_extent, scale_lo, scale_hi, sh_degree,
                                  m.ctypes.data_as(_dp), s.ctypes.data_as(_dp), q.ctypes.data_as(_dp),
                                  o.ctypes.data_as(_dp), sh.ctypes.data_as(_dp))
        return GaussianField(m, s, q, o, sh, sh_degree)

    def mt19937_64(self, seed: int, n: int) -> np.ndarray:
        state = C.create_string_buffer(312 * 8 + 16)
        self.lib.gso_mt_seed(state, seed)
        return np.array([self.lib.gso_mt_next(state) for _ in range(n)], dtype=np.uint64)

    def look_at(self, eye, target, fx, fy, width, height, up=(0.0, 0.0, 1.0)) -> abi.gsim_camera:
        cam = abi.gsim_camera()
        e = (C.c_double * 3)(*eye); t = (C.c_double * 3)(*target); u = (C.c_double * 3)(*up)
        self.lib.gso_look_at(e, t, fx, fy, width, height, u, C.byref(cam))
        return cam

    def shade_sh(self, sh48, degree, view_dir):
        sh = (C.c_double * 48)(*sh48); d = (C.c_double * 3)(*view_dir); out = (C.c_double * 3)()
        self.lib.gso_shade_sh(sh, degree, d, out)
        return tuple(out)

    # -- GS -> TSDF (transfer.cpp) -------------------------------------------------------------
    def field_bounds(self, field: GaussianField):
        lo = (C.c_double * 3)(); hi = (C.c_double * 3)()
        v = field.view()
        self.lib.gso_field_bounds(C.byref(v), lo, hi)
        return tuple(lo), tuple(hi)

    def depth_ring_cameras(self, lo, hi, n_views: int, radius: float, resolution: int):
        cams = (abi.gsim_camera * (3 * max(n_views, 1)))()
        _ok(self.lib.gso_depth_ring_cameras(_vec3(lo), _vec3(hi), n_views, radius, resolution, cams),
            "depth_ring_cameras")
        return cams

    def render_depth_ring(self, field: GaussianField, n_views: int, radius: float, resolution: int):
        """-> (3 * n_views cameras, depth float32 (3 * n_views, resolution, resolution))."""
        n = 3 * max(n_views, 1)
        cams = (abi.gsim_camera * n)()
        depth = np.zeros((n, resolution, resolution), dtype=np.float32)
        v = field.view()
        _ok(self.lib.gso_render_depth_ring(C.byref(v), n_views, radius, resolution, cams,
                                           depth.ctypes.data_as(_fp)), "render_depth_ring")
        return cams, depth

    def tsdf_create(self, origin, voxel_size, dims, truncation) -> TsdfVolume:
        vol = TsdfVolume(origin, voxel_size, dims, truncation)
        if min(vol.dims) >= 2:
            vol.allocate()
        c = vol.to_c()
        _ok(self.lib.gso_tsdf_create(_vec3(origin), voxel_size, (C.c_int32 * 3)(*vol.dims),
                                     truncation, C.byref(c)), "tsdf_create")
        return vol

    def tsdf_fuse(self, vol: TsdfVolume, camera, depth: np.ndarray) -> None:
        depth = np.ascontiguousarray(depth, dtype=np.float32)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        c = vol.to_c()
        _ok(self.lib.gso_tsdf_fuse(C.byref(c), C.byref(cam), depth.ctypes.data_as(_fp),
                                   depth.shape[1], depth.shape[0]), "tsdf_fuse")

    def gaussians_to_tsdf(self, field: GaussianField, voxel_size: float) -> TsdfVolume:
        v = field.view()
        c = abi.gsim_tsdf_volume()
        _ok(self.lib.gso_gaussians_to_tsdf(C.byref(v), voxel_size, C.byref(c)), "gaussians_to_tsdf")
        vol = TsdfVolume.from_c(c).allocate()
        c = vol.to_c()
        _ok(self.lib.gso_gaussians_to_tsdf(C.byref(v), voxel_size, C.byref(c)), "gaussians_to_tsdf")
        return vol

    # -- LiDAR (trace.cpp) ---------------------------------------------------------------------
    def trace_rays(self, field: GaussianField, nodes, origins, directions, t_max, alpha_threshold=0.5):
        """trace_linear per ray -> (hit u8, depth, accum_alpha)."""
        o, d, t = _rays(origins, directions, t_max)
        n = len(t)
        hit = np.zeros(n, np.uint8); depth = np.zeros(n); acc = np.zeros(n)
        v = field.view()
        na = _nodes(nodes)
        _ok(self.lib.gso_trace_rays(C.byref(v), na, len(nodes), o.ctypes.data_as(_dp),
                                    d.ctypes.data_as(_dp), t.ctypes.data_as(_dp), n, alpha_threshold,
                                    hit.ctypes.data_as(C.POINTER(C.c_uint8)), depth.ctypes.data_as(_dp),
                                    acc.ctypes.data_as(_dp)), "trace_rays")
        return hit, depth, acc

    def lidar_scan(self, field: GaussianField, nodes, lidar) -> dict:
        """GaussianBvh::scan -> {"points" (n, 3), "ring" (n,), "azimuth" (n,)}."""
        v = field.view()
        na = _nodes(nodes)
        return _two_call_scan(lambda l, p, r, a, cap, cnt: self.lib.gso_lidar_scan(
            C.byref(v), na, len(nodes), l, p, r, a, cap, cnt), lidar, "lidar_scan")

    # -- the path ----------------------------------------------------------------------------
    def project(self, field: GaussianField, nodes, camera) -> np.ndarray:
        v = field.view()
        na = _nodes(nodes)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        out = np.zeros(max(field.size(), 1), dtype=abi.SPLAT_DTYPE)
        count = C.c_uint64(0)
        st = self.lib.gso_project(C.byref(v), na, len(nodes), C.byref(cam), out.ctypes.data_as(_vp),
                                  field.size(), C.byref(count))
        if st != abi.GSIM_OK:
            raise ValueError("oracle project: validation error")
        return out[: count.value].copy()

    def rasterize(self, splats, camera, options: RasterOptions | None = None) -> RenderTarget:
        splats = np.ascontiguousarray(splats, dtype=abi.SPLAT_DTYPE)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        opt = (options or RasterOptions()).to_c()
        t = _target(cam.width, cam.height)
        self.lib.gso_rasterize(splats.ctypes.data_as(_vp), len(splats), C.byref(cam), C.byref(opt),
                               t.rgb.ctypes.data_as(_fp), t.depth.ctypes.data_as(_fp),
                               t.accum_alpha.ctypes.data_as(_fp))
        return t

    def reference_rasterize(self, splats, camera, options: RasterOptions | None = None) -> RenderTarget:
        splats = np.ascontiguousarray(splats, dtype=abi.SPLAT_DTYPE)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        opt = (options or RasterOptions()).to_c()
        t = _target(cam.width, cam.height)
        self.lib.gso_reference_rasterize(splats.ctypes.data_as(_vp), len(splats), C.byref(cam),
                                         C.byref(opt), t.rgb.ctypes.data_as(_fp),
                                         t.depth.ctypes.data_as(_fp), t.accum_alpha.ctypes.data_as(_fp))
        return t

    def rasterize_lists(self, splats, camera):
        """(tile_begin[tiles+1], splat index per sorted pair) of raster.cpp:174-202."""
        splats = np.ascontiguousarray(splats, dtype=abi.SPLAT_DTYPE)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
        count = C.c_uint64(0)
        self.lib.gso_rasterize_lists(splats.ctypes.data_as(_vp), len(splats), C.byref(cam), None,
                                     None, 0, C.byref(count))
        tb = np.zeros(tiles + 1, np.uint32)
        vals = np.zeros(max(count.value, 1), np.uint32)
        self.lib.gso_rasterize_lists(splats.ctypes.data_as(_vp), len(splats), C.byref(cam),
                                     tb.ctypes.data_as(_u32p), vals.ctypes.data_as(_u32p),
                                     count.value, C.byref(count))
        return tb, vals[: count.value]

    def render(self, field: GaussianField, nodes, cameras, options: RasterOptions | None = None):
        v = field.view()
        na = _nodes(nodes)
        ca = _cams(cameras)
        opt = (options or RasterOptions()).to_c()
        targets = [_target(ca[k].width, ca[k].height) for k in range(len(cameras))]
        ta = (abi.gsim_target * max(len(cameras), 1))()
        for k, t in enumerate(targets):
            ta[k] = t.to_c()
        st = self.lib.gso_render(C.byref(v), na, len(nodes), ca, len(cameras), C.byref(opt), ta)
        if st != abi.GSIM_OK:
            raise ValueError("oracle render: validation error")
        return targets

    def transform_primitives(self, means, rotations, begin, end, rigid) -> int:
        r = rigid.to_c() if hasattr(rigid, "to_c") else rigid
        return self.lib.gso_transform_primitives(means.ctypes.data_as(_dp), rotations.ctypes.data_as(_dp),
                                                 len(means), begin, end, C.byref(r))

    def hash_target(self, t: RenderTarget, seed: int = 1469598103934665603) -> int:
        h, w = t.depth.shape
        return int(self.lib.gso_hash_target(t.rgb.ctypes.data_as(_fp), t.depth.ctypes.data_as(_fp),
                                            t.accum_alpha.ctypes.data_as(_fp), w, h, seed))


    # -- output encoding / pose playback ------------------------------------------------------
    def linear_to_srgb(self, v: float) -> float:
        return self.lib.gso_linear_to_srgb(v)

    def encode(self, flags, srgb, depth_scale, width, height, rgb=None, depth=None, alpha=None):
        """GSIM_ENCODE_* blob of one target (image_io.cpp writers' bytes)."""
        n = int(self.lib.gso_encoded_bytes(flags, width, height))
        out = np.zeros(max(n, 1), dtype=np.uint8)
        planes = [_plane(rgb, width * height * 3), _plane(depth, width * height), _plane(alpha, width * height)]
        rc = self.lib.gso_encode(flags, int(srgb), float(depth_scale), width, height,
                                 *[p.ctypes.data_as(_fp) for p in planes],
                                 out.ctypes.data_as(C.POINTER(C.c_uint8)))
        if rc != 0:
            raise ValueError(f"gso_encode rc={rc}")
        return out[:n]

    def load_splat_ply(self, path):
        return _load_ply(self.lib.gso_load_splat_ply, path)

    def slerp(self, a, b, t):
        o = np.zeros(4)
        self.lib.gso_slerp(np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(_dp),
                           np.ascontiguousarray(b, dtype=np.float64).ctypes.data_as(_dp), float(t),
                           o.ctypes.data_as(_dp))
        return o

    def pose_sample(self, rec_t, rec_p, rec_q, initial, ts):
        """(rc, [n_t] gsim_rigid) of one node's track sampled at ts (PoseStream::sample)."""
        return _pose_sample(self.lib.gso_pose_sample, rec_t, rec_p, rec_q, initial, ts)


def _load_ply(fn, path):
    """(status, GaussianField | None) through a two-call C loader."""
    count = C.c_uint64(0)
    degree = C.c_int(0)
    z = np.zeros(1)
    rc = fn(str(path).encode(), 0, C.byref(count), C.byref(degree), *[z.ctypes.data_as(_dp)] * 5)
    if rc != 0:
        return rc, None
    n = count.value
    m = np.zeros((max(n, 1), 3)); s = np.zeros((max(n, 1), 3)); q = np.zeros((max(n, 1), 4))
    o = np.zeros(max(n, 1)); sh = np.zeros((max(n, 1), 48))
    rc = fn(str(path).encode(), n, C.byref(count), C.byref(degree),
            *[a.ctypes.data_as(_dp) for a in (m, s, q, o, sh)])
    if rc != 0:
        return rc, None
    return 0, GaussianField(m[:n], s[:n], q[:n], o[:n], sh[:n], degree.value)


def _plane(a, n):
    if a is None:
        return np.zeros(max(n, 1), dtype=np.float32)
    return np.ascontiguousarray(a, dtype=np.float32).reshape(-1)


def _pose_sample(fn, rec_t, rec_p, rec_q, initial, ts):
    rt = np.ascontiguousarray(rec_t, dtype=np.float64).reshape(-1)
    rp = np.ascontiguousarray(rec_p, dtype=np.float64).reshape(-1)
    rq = np.ascontiguousarray(rec_q, dtype=np.float64).reshape(-1)
    tt = np.ascontiguousarray(ts, dtype=np.float64).reshape(-1)
    out = (abi.gsim_rigid * max(len(tt), 1))()
    init = initial.to_c() if hasattr(initial, "to_c") else initial
    rc = fn(rt.ctypes.data_as(_dp), rp.ctypes.data_as(_dp), rq.ctypes.data_as(_dp), len(rt),
            C.byref(init), tt.ctypes.data_as(_dp), len(tt), out)
    poses = np.array([list(out[k].rotation) + list(out[k].translation) for k in range(len(tt))],
                     dtype=np.float64).reshape(-1, 7)
    return rc, poses


class Ref:
    """The unmodified reference (oracle/_ref/libgsim_ref.so). Raises if it was never built."""

    def __init__(self, path: Path | None = None):
        p = Path(path) if path else REF_LIB
        if not p.exists():
            if Path("/root/reference/proj").exists():
                build_oracle(with_ref=True)
            if not p.exists():
                raise FileNotFoundError(f"{p} not built (needs /root/reference at build time)")
        # The reference's iostream users (save_splat_ply, write_pfm) need libstdc++'s unique
        # locale-facet symbols resolved globally; a RTLD_LOCAL-only load crashes in ofstream.
        C.CDLL("libstdc++.so.6", mode=C.RTLD_GLOBAL)
        self.lib = C.CDLL(str(p))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_field_create.argtypes = [C.POINTER(abi.gsim_field_view)]
        L.ref_field_create.restype = _vp
        L.ref_field_destroy.argtypes = [_vp]
        L.ref_project.argtypes = [_vp, C.POINTER(abi.gsim_node), C.c_uint64, C.POINTER(abi.gsim_camera),
                                  _vp, C.c_uint64, _u64p]
        L.ref_rasterize.argtypes = [_vp, C.c_uint64, C.POINTER(abi.gsim_camera),
                                    C.POINTER(abi.gsim_raster_options), _fp, _fp, _fp]
        L.ref_reference_rasterize.argtypes = L.ref_rasterize.argtypes
        L.ref_render.argtypes = [_vp, C.POINTER(abi.gsim_node), C.c_uint64, C.POINTER(abi.gsim_camera),
                                 C.c_uint64, C.POINTER(abi.gsim_raster_options), C.POINTER(abi.gsim_target)]
        L.ref_transform_primitives.argtypes = [_dp, _dp, C.c_uint64, C.c_uint64, C.c_uint64,
                                               C.POINTER(abi.gsim_rigid)]
        L.ref_look_at.argtypes = [_dp, _dp, C.c_double, C.c_double, C.c_int, C.c_int, _dp,
                                  C.POINTER(abi.gsim_camera)]
        L.ref_random_field.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                       C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_thread_count.restype = C.c_int
        L.ref_rigid_compose.argtypes = [C.POINTER(abi.gsim_rigid)] * 3
        u8p = C.POINTER(C.c_uint8)
        L.ref_linear_to_srgb.argtypes = [C.c_double]
        L.ref_linear_to_srgb.restype = C.c_double
        L.ref_png_rgb8.argtypes = [_fp, C.c_int, C.c_int, C.c_int, u8p, C.c_uint64, _u64p]
        L.ref_png_gray8.argtypes = [_fp, C.c_int, C.c_int, u8p, C.c_uint64, _u64p]
        L.ref_png_gray16.argtypes = [_fp, C.c_int, C.c_int, C.c_double, u8p, C.c_uint64, _u64p]
        L.ref_write_pfm.argtypes = [C.c_char_p, _fp, C.c_int, C.c_int]
        L.ref_load_splat_ply.argtypes = [C.c_char_p, C.c_uint64, _u64p, C.POINTER(C.c_int), _dp, _dp,
                                         _dp, _dp, _dp]
        L.ref_save_splat_ply.argtypes = [C.c_char_p, C.POINTER(abi.gsim_field_view)]
        L.ref_slerp.argtypes = [_dp, _dp, C.c_double, _dp]
        L.ref_pose_sample.argtypes = [_dp, _dp, _dp, C.c_uint64, C.POINTER(abi.gsim_rigid), _dp,
                                      C.c_uint64, C.POINTER(abi.gsim_rigid)]
        vol = C.POINTER(abi.gsim_tsdf_volume)
        L.ref_render_depth_ring.argtypes = [_vp, C.c_int, C.c_double, C.c_int,
                                            C.POINTER(abi.gsim_camera), _fp]
        L.ref_tsdf_create.argtypes = [_dp, C.c_double, C.POINTER(C.c_int32), C.c_double, vol]
        L.ref_tsdf_fuse.argtypes = [vol, C.POINTER(abi.gsim_camera), _fp, C.c_int, C.c_int]
        L.ref_gaussians_to_tsdf.argtypes = [_vp, C.c_double, vol]
        L.ref_trace_rays.argtypes = [_vp, C.POINTER(abi.gsim_node), C.c_uint64, _dp, _dp, _dp,
                                     C.c_uint64, C.c_double, C.c_int, C.POINTER(C.c_uint8), _dp, _dp]
        L.ref_lidar_scan.argtypes = [_vp, C.POINTER(abi.gsim_node), C.c_uint64,
                                     C.POINTER(abi.gsim_lidar), _dp, _u32p, _dp, C.c_uint64, _u64p]

    # -- GS -> TSDF (transfer.cpp) -------------------------------------------------------------
    def _with_field(self, field: GaussianField, fn):
        v = field.view()
        h = self.lib.ref_field_create(C.byref(v))
        try:
            return fn(h)
        finally:
            self.lib.ref_field_destroy(h)

    def render_depth_ring(self, field: GaussianField, n_views: int, radius: float, resolution: int):
        n = 3 * max(n_views, 1)
        cams = (abi.gsim_camera * n)()
        depth = np.zeros((n, resolution, resolution), dtype=np.float32)
        _ok(self._with_field(field, lambda h: self.lib.ref_render_depth_ring(
            h, n_views, radius, resolution, cams, depth.ctypes.data_as(_fp))), "ref render_depth_ring")
        return cams, depth

    def tsdf_create(self, origin, voxel_size, dims, truncation) -> TsdfVolume:
        vol = TsdfVolume(origin, voxel_size, dims, truncation)
        if min(vol.dims) >= 2:
            vol.allocate()
        c = vol.to_c()
        _ok(self.lib.ref_tsdf_create(_vec3(origin), voxel_size, (C.c_int32 * 3)(*vol.dims),
                                     truncation, C.byref(c)), "ref tsdf_create")
        return vol

    def tsdf_fuse(self, vol: TsdfVolume, camera, depth: np.ndarray) -> None:
        depth = np.ascontiguousarray(depth, dtype=np.float32)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        c = vol.to_c()
        _ok(self.lib.ref_tsdf_fuse(C.byref(c), C.byref(cam), depth.ctypes.data_as(_fp),
                                   depth.shape[1], depth.shape[0]), "ref tsdf_fuse")

    def gaussians_to_tsdf(self, field: GaussianField, voxel_size: float) -> TsdfVolume:
        def run(h):
            c = abi.gsim_tsdf_volume()
            _ok(self.lib.ref_gaussians_to_tsdf(h, voxel_size, C.byref(c)), "ref gaussians_to_tsdf")
            vol = TsdfVolume.from_c(c).allocate()
            c = vol.to_c()
            _ok(self.lib.ref_gaussians_to_tsdf(h, voxel_size, C.byref(c)), "ref gaussians_to_tsdf")
            return vol
        return self._with_field(field, run)

    # -- LiDAR (trace.cpp) ---------------------------------------------------------------------
    def trace_rays(self, field: GaussianField, nodes, origins, directions, t_max, alpha_threshold=0.5,
                   linear=False):
        o, d, t = _rays(origins, directions, t_max)
        n = len(t)
        hit = np.zeros(n, np.uint8); depth = np.zeros(n); acc = np.zeros(n)
        na = _nodes(nodes)
        _ok(self._with_field(field, lambda h: self.lib.ref_trace_rays(
            h, na, len(nodes), o.ctypes.data_as(_dp), d.ctypes.data_as(_dp), t.ctypes.data_as(_dp), n,
            alpha_threshold, int(linear), hit.ctypes.data_as(C.POINTER(C.c_uint8)),
            depth.ctypes.data_as(_dp), acc.ctypes.data_as(_dp))), "ref trace_rays")
        return hit, depth, acc

    def lidar_scan(self, field: GaussianField, nodes, lidar) -> dict:
        na = _nodes(nodes)
        return self._with_field(field, lambda h: _two_call_scan(
            lambda l, p, r, a, cap, cnt: self.lib.ref_lidar_scan(h, na, len(nodes), l, p, r, a, cap, cnt),
            lidar, "ref lidar_scan"))

    def set_threads(self, n: int) -> None:
        self.lib.ref_set_threads(n)

    def thread_count(self) -> int:
        return self.lib.ref_thread_count()

    def random_field(self, seed, count, box_extent, scale_lo, scale_hi, sh_degree) -> GaussianField:
        m = np.zeros((count, 3)); s = np.zeros((count, 3)); q = np.zeros((count, 4))
        o = np.zeros(count); sh = np.zeros((count, 48))
        self.lib.ref_random_field(seed, count, box_extent, scale_lo, scale_hi, sh_degree,
                                  m.ctypes.data_as(_dp), s.ctypes.data_as(_dp), q.ctypes.data_as(_dp),
                                  o.ctypes.data_as(_dp), sh.ctypes.data_as(_dp))
        return GaussianField(m, s, q, o, sh, sh_degree)

    def field(self, field: GaussianField):
        v = field.view()
        return RefField(self, self.lib.ref_field_create(C.byref(v)), field.size())

    def project(self, field: GaussianField, nodes, camera) -> np.ndarray:
        with_field = self.field(field)
        try:
            return with_field.project(nodes, camera)
        finally:
            with_field.close()

    def rasterize(self, splats, camera, options=None) -> RenderTarget:
        return self._raster(self.lib.ref_rasterize, splats, camera, options)

    def reference_rasterize(self, splats, camera, options=None) -> RenderTarget:
        return self._raster(self.lib.ref_reference_rasterize, splats, camera, options)

    def _raster(self, fn, splats, camera, options):
        splats = np.ascontiguousarray(splats, dtype=abi.SPLAT_DTYPE)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        opt = (options or RasterOptions()).to_c()
        t = _target(cam.width, cam.height)
        st = fn(splats.ctypes.data_as(_vp), len(splats), C.byref(cam), C.byref(opt),
                t.rgb.ctypes.data_as(_fp), t.depth.ctypes.data_as(_fp), t.accum_alpha.ctypes.data_as(_fp))
        if st != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return t

    def render(self, field: GaussianField, nodes, cameras, options=None):
        with_field = self.field(field)
        try:
            return with_field.render(nodes, cameras, options)
        finally:
            with_field.close()

    def transform_primitives(self, means, rotations, begin, end, rigid) -> int:
        r = rigid.to_c() if hasattr(rigid, "to_c") else rigid
        return self.lib.ref_transform_primitives(means.ctypes.data_as(_dp), rotations.ctypes.data_as(_dp),
                                                 len(means), begin, end, C.byref(r))

    def look_at(self, eye, target, fx, fy, width, height, up=(0.0, 0.0, 1.0)) -> abi.gsim_camera:
        cam = abi.gsim_camera()
        e = (C.c_double * 3)(*eye); t = (C.c_double * 3)(*target); u = (C.c_double * 3)(*up)
        self.lib.ref_look_at(e, t, fx, fy, width, height, u, C.byref(cam))
        return cam


    # -- image_io.cpp writers (row bytes captured at the libpng boundary) / pose playback -----
    def linear_to_srgb(self, v: float) -> float:
        return self.lib.ref_linear_to_srgb(v)

    def _capture(self, fn, *args, n):
        out = np.zeros(max(n, 1), dtype=np.uint8)
        size = C.c_uint64(0)
        rc = fn(*args, out.ctypes.data_as(C.POINTER(C.c_uint8)), len(out), C.byref(size))
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return out[: size.value]

    def png_rgb8(self, rgb, width, height, srgb):
        a = _plane(rgb, width * height * 3)
        return self._capture(self.lib.ref_png_rgb8, a.ctypes.data_as(_fp), width, height, int(srgb),
                             n=3 * width * height)

    def png_gray8(self, v, width, height):
        a = _plane(v, width * height)
        return self._capture(self.lib.ref_png_gray8, a.ctypes.data_as(_fp), width, height,
                             n=width * height)

    def png_gray16(self, v, width, height, scale):
        a = _plane(v, width * height)
        return self._capture(self.lib.ref_png_gray16, a.ctypes.data_as(_fp), width, height,
                             float(scale), n=2 * width * height)

    def write_pfm(self, path, v, width, height) -> bytes:
        a = _plane(v, width * height)
        rc = self.lib.ref_write_pfm(str(path).encode(), a.ctypes.data_as(_fp), width, height)
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return Path(path).read_bytes()

    def encode(self, flags, srgb, depth_scale, width, height, rgb=None, depth=None, alpha=None,
               tmpdir=None):
        """The GSIM_ENCODE_* blob assembled from the reference writers' own bytes."""
        import tempfile
        parts = []
        if flags & abi.GSIM_ENCODE_RGB8:
            parts.append(self.png_rgb8(rgb, width, height, srgb))
        if flags & abi.GSIM_ENCODE_ALPHA8:
            parts.append(self.png_gray8(alpha, width, height))
        if flags & abi.GSIM_ENCODE_DEPTH16:
            parts.append(self.png_gray16(depth, width, height, depth_scale))
        if flags & abi.GSIM_ENCODE_DEPTH_PFM:
            with tempfile.TemporaryDirectory(dir=tmpdir) as d:
                raw = self.write_pfm(Path(d) / "d.pfm", depth, width, height)
            header = f"Pf\n{width} {height}\n-1.0\n".encode()
            assert raw.startswith(header)
            parts.append(np.frombuffer(raw[len(header):], dtype=np.uint8))
        return np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint8)

    def load_splat_ply(self, path):
        return _load_ply(self.lib.ref_load_splat_ply, path)

    def save_splat_ply(self, path, field: GaussianField) -> int:
        v = field.view()
        return self.lib.ref_save_splat_ply(str(path).encode(), C.byref(v))

    def slerp(self, a, b, t):
        o = np.zeros(4)
        self.lib.ref_slerp(np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(_dp),
                           np.ascontiguousarray(b, dtype=np.float64).ctypes.data_as(_dp), float(t),
                           o.ctypes.data_as(_dp))
        return o

    def pose_sample(self, rec_t, rec_p, rec_q, initial, ts):
        return _pose_sample(self.lib.ref_pose_sample, rec_t, rec_p, rec_q, initial, ts)


class RefField:
    """A reference GaussianField built once (outside timed regions)."""

    def __init__(self, ref: Ref, handle, size: int):
        self.ref = ref
        self.handle = handle
        self.size = size

    def project(self, nodes, camera) -> np.ndarray:
        na = _nodes(nodes)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        out = np.zeros(max(self.size, 1), dtype=abi.SPLAT_DTYPE)
        count = C.c_uint64(0)
        st = self.ref.lib.ref_project(self.handle, na, len(nodes), C.byref(cam), out.ctypes.data_as(_vp),
                                      self.size, C.byref(count))
        if st != 0:
            raise ValueError(self.ref.lib.ref_last_error().decode())
        return out[: count.value].copy()

    def render(self, nodes, cameras, options=None, targets=None):
        na = _nodes(nodes)
        ca = _cams(cameras)
        opt = (options or RasterOptions()).to_c()
        if targets is None:
            targets = [_target(ca[k].width, ca[k].height) for k in range(len(cameras))]
        ta = (abi.gsim_target * max(len(cameras), 1))()
        for k, t in enumerate(targets):
            ta[k] = t.to_c()
        st = self.ref.lib.ref_render(self.handle, na, len(nodes), ca, len(cameras), C.byref(opt), ta)
        if st != 0:
            raise ValueError(self.ref.lib.ref_last_error().decode())
        return targets

    def close(self) -> None:
        if self.handle:
            self.ref.lib.ref_field_destroy(self.handle)
            self.handle = None


def ref_available() -> bool:
    return REF_LIB.exists() or Path("/root/reference/proj").exists()


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _rays(origins, directions, t_max):
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(directions, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(np.broadcast_to(np.asarray(t_max, np.float64), (len(o),)))
    return o, d, t


def _two_call_scan(fn, lidar, what: str) -> dict:
    """Size, then fill, a scan's point cloud through a (lidar, points, ring, azimuth, capacity,
    count) entry point."""
    lc = lidar.to_c() if hasattr(lidar, "to_c") else lidar
    cnt = C.c_uint64(0)
    z = np.zeros(1)
    _ok(fn(C.byref(lc), z.ctypes.data_as(_dp), np.zeros(1, np.uint32).ctypes.data_as(_u32p),
           z.ctypes.data_as(_dp), 0, C.byref(cnt)), what)
    n = cnt.value
    pts = np.zeros((max(n, 1), 3)); ring = np.zeros(max(n, 1), np.uint32); az = np.zeros(max(n, 1))
    _ok(fn(C.byref(lc), pts.ctypes.data_as(_dp), ring.ctypes.data_as(_u32p), az.ctypes.data_as(_dp),
           n, C.byref(cnt)), what)
    return {"points": pts[:n], "ring": ring[:n], "azimuth": az[:n]}
