"""Python host mirror of the reference render API, backed by the sm_100a C ABI.

Names, argument meaning and error behaviour follow the reference gsim library:
    GaussianField, SceneNode, NodeKind    gaussian.hpp:19-71
    RigidTransform                        math.hpp:217-239
    CameraModel (+ look_at)               camera.hpp:14-33, raster.cpp:25-42
    RasterOptions, ProjectedSplat         raster.hpp:20-36
    RenderTarget                          image.hpp:38-45
    project / rasterize / render          raster.hpp:54-67
    transform_primitives                  gaussian.hpp:76-77
    io_error / validation_error           errors.hpp:12-25
Every compute call goes through libgsim_gpu.so; there is no CPU path here.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field as dc_field
from typing import Sequence

import numpy as np

from . import abi


class IoError(RuntimeError):
    """io_error (errors.hpp:12-15): runtime / CUDA failure, CLI exit code 1."""


class ValidationError(ValueError):
    """validation_error (errors.hpp:18-21): bad input, CLI exit code 2."""


io_error = IoError
validation_error = ValidationError


def _check(status: int, ctx_ptr) -> None:
    if status == abi.GSIM_OK:
        return
    lib = abi.load_library()
    msg = lib.gsim_gpu_last_error(ctx_ptr)
    msg = msg.decode() if msg else ""
    if status == abi.GSIM_ERR_VALIDATION:
        raise ValidationError(msg)
    raise IoError(msg)


# ---- math.hpp (host-side helpers for building poses and cameras) -------------------------

def quat_mul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return (aw * bw - ax * bx - ay * by - az * bz,
            aw * bx + ax * bw + ay * bz - az * by,
            aw * by - ax * bz + ay * bw + az * bx,
            aw * bz + ax * by - ay * bx + az * bw)


def quat_rotate(q, v):
    w, x, y, z = q
    vx, vy, vz = v
    tx, ty, tz = 2.0 * (y * vz - z * vy), 2.0 * (z * vx - x * vz), 2.0 * (x * vy - y * vx)
    return (vx + tx * w + (y * tz - z * ty),
            vy + ty * w + (z * tx - x * tz),
            vz + tz * w + (x * ty - y * tx))


def quat_normalized(q):
    n = math.sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3])
    return tuple(c / n for c in q) if n > 0.0 else (1.0, 0.0, 0.0, 0.0)


def quat_from_axis_angle(axis, angle):
    n = math.sqrt(sum(a * a for a in axis))
    a = [c / n for c in axis] if n > 0 else [0.0, 0.0, 0.0]
    s = math.sin(0.5 * angle)
    return (math.cos(0.5 * angle), a[0] * s, a[1] * s, a[2] * s)


def quat_from_matrix(m):
    """Shepperd's method, math.hpp:158-187 (m row-major 3x3 nested)."""
    tr = m[0][0] + m[1][1] + m[2][2]
    if tr > 0.0:
        s = math.sqrt(tr + 1.0) * 2.0
        q = (0.25 * s, (m[2][1] - m[1][2]) / s, (m[0][2] - m[2][0]) / s, (m[1][0] - m[0][1]) / s)
    elif m[0][0] > m[1][1] and m[0][0] > m[2][2]:
        s = math.sqrt(1.0 + m[0][0] - m[1][1] - m[2][2]) * 2.0
        q = ((m[2][1] - m[1][2]) / s, 0.25 * s, (m[0][1] + m[1][0]) / s, (m[0][2] + m[2][0]) / s)
    elif m[1][1] > m[2][2]:
        s = math.sqrt(1.0 + m[1][1] - m[0][0] - m[2][2]) * 2.0
        q = ((m[0][2] - m[2][0]) / s, (m[0][1] + m[1][0]) / s, 0.25 * s, (m[1][2] + m[2][1]) / s)
    else:
        s = math.sqrt(1.0 + m[2][2] - m[0][0] - m[1][1]) * 2.0
        q = ((m[1][0] - m[0][1]) / s, (m[0][2] + m[2][0]) / s, (m[1][2] + m[2][1]) / s, 0.25 * s)
    return quat_normalized(q)


@dataclass
class RigidTransform:
    """SE(3) pose x -> R(q) x + t, q = (w, x, y, z) (math.hpp:217-239)."""
    rotation: tuple = (1.0, 0.0, 0.0, 0.0)
    translation: tuple = (0.0, 0.0, 0.0)

    @staticmethod
    def identity() -> "RigidTransform":
        return RigidTransform()

    def transform_point(self, p):
        r = quat_rotate(self.rotation, p)
        return (r[0] + self.translation[0], r[1] + self.translation[1], r[2] + self.translation[2])

    def __mul__(self, o: "RigidTransform") -> "RigidTransform":
        return RigidTransform(quat_normalized(quat_mul(self.rotation, o.rotation)),
                              self.transform_point(o.translation))

    def inverse(self) -> "RigidTransform":
        inv = (self.rotation[0], -self.rotation[1], -self.rotation[2], -self.rotation[3])
        t = quat_rotate(inv, self.translation)
        return RigidTransform(inv, (-t[0], -t[1], -t[2]))

    def to_c(self) -> abi.gsim_rigid:
        r = abi.gsim_rigid()
        for k in range(4):
            r.rotation[k] = float(self.rotation[k])
        for k in range(3):
            r.translation[k] = float(self.translation[k])
        return r


class NodeKind:
    background = abi.GSIM_NODE_BACKGROUND
    interactive = abi.GSIM_NODE_INTERACTIVE


@dataclass
class SceneNode:
    """Background or interactive entity driving a contiguous primitive range (gaussian.hpp:66-71).
    env = -1 (default) is the reference's semantics; env >= 0 limits the node to that env's
    cameras for batched multi-environment rendering."""
    id: str = ""
    kind: int = NodeKind.background
    pose: RigidTransform = dc_field(default_factory=RigidTransform)
    range: tuple = (0, 0)
    env: int = abi.GSIM_ENV_ALL

    def to_c(self) -> abi.gsim_node:
        n = abi.gsim_node()
        n.begin, n.end = int(self.range[0]), int(self.range[1])
        n.pose = self.pose.to_c()
        n.kind = int(self.kind)
        n.env = int(self.env)
        return n


@dataclass
class CameraModel:
    """Pinhole camera; pose maps world -> camera (x right, y down, z forward) (camera.hpp)."""
    id: str = ""
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0
    pose: RigidTransform = dc_field(default_factory=RigidTransform)
    near: float = 0.05
    far: float = 100.0
    env: int = 0

    def camera_center(self):
        return self.pose.inverse().translation

    @staticmethod
    def look_at(eye, target, fx, fy, width, height, up=(0.0, 0.0, 1.0)) -> "CameraModel":
        """CameraModel::look_at (raster.cpp:25-42)."""
        def sub(a, b): return (a[0] - b[0], a[1] - b[1], a[2] - b[2])
        def cross(a, b): return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])
        def normalized(a):
            n = math.sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2])
            return (a[0] / n, a[1] / n, a[2] / n) if n > 0 else (0.0, 0.0, 0.0)
        forward = normalized(sub(target, eye))
        right = normalized(cross(forward, up))
        if right[0] ** 2 + right[1] ** 2 + right[2] ** 2 < 1e-20:
            right = normalized(cross(forward, (0.0, 1.0, 0.0)))
        down = cross(forward, right)
        q = quat_from_matrix([list(right), list(down), list(forward)])
        t = quat_rotate(q, eye)
        return CameraModel(fx=fx, fy=fy, cx=width * 0.5, cy=height * 0.5, width=width,
                           height=height, pose=RigidTransform(q, (-t[0], -t[1], -t[2])))

    def to_c(self) -> abi.gsim_camera:
        c = abi.gsim_camera()
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.width, c.height = int(self.width), int(self.height)
        c.pose = self.pose.to_c()
        c.near_plane, c.far_plane = float(self.near), float(self.far)
        c.env = int(self.env)
        return c


@dataclass
class RasterOptions:
    """raster.hpp:31-36."""
    normalize_depth: bool = False
    transmittance_cutoff: float = 1e-4

    def to_c(self) -> abi.gsim_raster_options:
        o = abi.gsim_raster_options()
        o.normalize_depth = 1 if self.normalize_depth else 0
        o.transmittance_cutoff = float(self.transmittance_cutoff)
        return o


class EncodeOptions:
    """Which writer bytes to produce (include/gsim_gpu.h GSIM_ENCODE_*); defaults follow the
    reference CLI's render command (tools/gsim.cpp:57-66): sRGB 8-bit RGB, 8-bit alpha, PFM
    depth, and 16-bit millimetre depth."""

    RGB8 = abi.GSIM_ENCODE_RGB8
    ALPHA8 = abi.GSIM_ENCODE_ALPHA8
    DEPTH16 = abi.GSIM_ENCODE_DEPTH16
    DEPTH_PFM = abi.GSIM_ENCODE_DEPTH_PFM

    def __init__(self, flags: int = RGB8 | ALPHA8 | DEPTH16 | DEPTH_PFM, srgb: bool = True,
                 depth_scale: float = 1000.0):
        self.flags = int(flags)
        self.srgb = bool(srgb)
        self.depth_scale = float(depth_scale)

    def to_c(self) -> abi.gsim_encode_options:
        return abi.gsim_encode_options(self.flags, int(self.srgb), self.depth_scale)

    def bytes_per_camera(self, width: int, height: int) -> int:
        return int(abi.load_library().gsim_gpu_encoded_bytes(self.flags, width, height))

    def split(self, blob: np.ndarray, cameras) -> list[dict]:
        """Per-camera views of an encoded blob: rgb8 (H,W,3) u8, alpha8 (H,W) u8, depth16 (H,W)
        u16 (decoded from big-endian), depth_pfm (H,W) f32 rows bottom-up."""
        out, off = [], 0
        for c in cameras:
            w, h = c.width, c.height
            n = w * h
            d = {}
            if self.flags & self.RGB8:
                d["rgb8"] = blob[off:off + 3 * n].reshape(h, w, 3); off += 3 * n
            if self.flags & self.ALPHA8:
                d["alpha8"] = blob[off:off + n].reshape(h, w); off += n
            if self.flags & self.DEPTH16:
                d["depth16"] = blob[off:off + 2 * n].view(">u2").reshape(h, w).astype(np.uint16); off += 2 * n
            if self.flags & self.DEPTH_PFM:
                d["depth_pfm"] = blob[off:off + 4 * n].copy().view("<f4").reshape(h, w); off += 4 * n
            out.append(d)
        return out


@dataclass
class RenderTarget:
    """RGB + alpha-composited depth + accumulated alpha (image.hpp:38-45)."""
    rgb: np.ndarray
    depth: np.ndarray
    accum_alpha: np.ndarray

    @staticmethod
    def empty(width: int, height: int) -> "RenderTarget":
        return RenderTarget(np.zeros((height, width, 3), np.float32),
                            np.zeros((height, width), np.float32),
                            np.zeros((height, width), np.float32))

    def check(self, width: int, height: int, who: str = "target") -> None:
        """The library writes W*H*5 float32 values through these pointers: every plane must be
        a C-contiguous float32 array of the camera's shape (ValidationError otherwise)."""
        for name, arr, shape in (("rgb", self.rgb, (height, width, 3)),
                                 ("depth", self.depth, (height, width)),
                                 ("accum_alpha", self.accum_alpha, (height, width))):
            if not isinstance(arr, np.ndarray) or arr.dtype != np.float32:
                raise ValidationError(f"{who}.{name}: need a float32 numpy array")
            if not arr.flags["C_CONTIGUOUS"] or not arr.flags["WRITEABLE"]:
                raise ValidationError(f"{who}.{name}: need a writeable C-contiguous array")
            if arr.shape != shape:
                raise ValidationError(f"{who}.{name}: shape {arr.shape}, camera needs {shape}")

    def hash(self, seed: int = 1469598103934665603) -> int:
        """hash_target (hash.hpp:36-41), chained from `seed`."""
        h, w = self.depth.shape
        self.check(w, h)
        fp = C.POINTER(C.c_float)
        return int(abi.load_library().gsim_gpu_hash_target(
            w, h, self.rgb.ctypes.data_as(fp), self.depth.ctypes.data_as(fp),
            self.accum_alpha.ctypes.data_as(fp), C.c_uint64(seed)))

    def to_c(self) -> abi.gsim_target:
        t = abi.gsim_target()
        fp = C.POINTER(C.c_float)
        t.rgb = self.rgb.ctypes.data_as(fp)
        t.depth = self.depth.ctypes.data_as(fp)
        t.accum_alpha = self.accum_alpha.ctypes.data_as(fp)
        return t


def _targets_array(targets, cams_c, n: int):
    """C array of host targets, one per camera, each checked against its camera's size. A
    target already checked with the same three arrays and size reuses its C struct (callers
    that render into the same targets every frame pay the checks once)."""
    targets = list(targets)
    if len(targets) != n:
        raise ValidationError(f"render: {len(targets)} targets for {n} cameras")
    ta = (abi.gsim_target * max(n, 1))()
    for k, t in enumerate(targets):
        w, h = cams_c[k].width, cams_c[k].height
        key = (id(t.rgb), id(t.depth), id(t.accum_alpha), w, h)
        cached = getattr(t, "_c_cache", None)
        if cached is None or cached[0] != key:
            t.check(w, h, f"targets[{k}]")
            # the cache holds the arrays themselves, so their ids cannot be reused while cached
            cached = (key, t.to_c(), (t.rgb, t.depth, t.accum_alpha))
            t._c_cache = cached
        ta[k] = cached[1]
    return ta


class GaussianField:
    """Indexed Gaussian collection (gaussian.hpp:53-60) held as SoA float64 arrays:
    means (N,3), scales (N,3) linear, rotations (N,4) unit (w,x,y,z), opacities (N,)
    post-sigmoid, sh (N,48) channel-major sh[c*16+k]; sh_degree global."""

    def __init__(self, means, scales, rotations, opacities, sh, sh_degree: int):
        self.means = np.ascontiguousarray(means, dtype=np.float64).reshape(-1, 3)
        n = self.means.shape[0]
        self.scales = np.ascontiguousarray(scales, dtype=np.float64).reshape(n, 3)
        self.rotations = np.ascontiguousarray(rotations, dtype=np.float64).reshape(n, 4)
        self.opacities = np.ascontiguousarray(opacities, dtype=np.float64).reshape(n)
        sh = np.asarray(sh, dtype=np.float64)
        if sh.shape != (n, 48):
            full = np.zeros((n, 48))
            full[:, : sh.shape[1]] = sh.reshape(n, -1)
            sh = full
        self.sh = np.ascontiguousarray(sh)
        self.sh_degree = int(sh_degree)
        self.generation = 0  # bump after in-place edits so cached uploads are refreshed

    def size(self) -> int:
        return self.means.shape[0]

    def __len__(self) -> int:
        return self.size()

    def touch(self) -> None:
        self.generation += 1

    def view(self) -> abi.gsim_field_view:
        v = abi.gsim_field_view()
        dp = C.POINTER(C.c_double)
        v.count = self.size()
        v.sh_degree = self.sh_degree
        v.means, v.means_stride = self.means.ctypes.data_as(dp), 3
        v.scales, v.scales_stride = self.scales.ctypes.data_as(dp), 3
        v.rotations, v.rotations_stride = self.rotations.ctypes.data_as(dp), 4
        v.opacities, v.opacities_stride = self.opacities.ctypes.data_as(dp), 1
        v.sh, v.sh_stride = self.sh.ctypes.data_as(dp), 48
        return v


class TsdfVolume:
    """TsdfVolume (transfer.hpp:40-62): a voxel grid of truncated signed distances fused from
    depth maps. tsdf / weights are (dims[2], dims[1], dims[0]) float64 arrays, x fastest
    (index(), transfer.hpp:50-52); None until allocated."""

    def __init__(self, origin, voxel_size: float, dims, truncation: float, tsdf=None, weights=None):
        self.origin = tuple(float(v) for v in origin)
        self.voxel_size = float(voxel_size)
        self.dims = tuple(int(d) for d in dims)
        self.truncation = float(truncation)
        self.tsdf = tsdf
        self.weights = weights

    @property
    def voxel_count(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    @property
    def shape(self) -> tuple:
        return (self.dims[2], self.dims[1], self.dims[0])

    def allocate(self) -> "TsdfVolume":
        """Host grids in the TsdfVolume::create state (tsdf 1, weights 0)."""
        self.tsdf = np.ones(self.shape)
        self.weights = np.zeros(self.shape)
        return self

    def device_grids(self) -> "TsdfVolume":
        """Device grids (torch cuda float64 tensors) in the TsdfVolume::create state; the
        library's tsdf entry points take these."""
        import torch
        self.tsdf = torch.ones(self.shape, dtype=torch.float64, device="cuda")
        self.weights = torch.zeros(self.shape, dtype=torch.float64, device="cuda")
        return self

    def to_numpy(self) -> "TsdfVolume":
        """Copy of the volume with host grids."""
        conv = lambda a: a.detach().cpu().numpy() if hasattr(a, "detach") else a
        return TsdfVolume(self.origin, self.voxel_size, self.dims, self.truncation,
                          conv(self.tsdf), conv(self.weights))

    def to_c(self, tsdf_ptr: int | None = None, weights_ptr: int | None = None) -> abi.gsim_tsdf_volume:
        """C view; the grid pointers default to the volume's arrays (host numpy or device torch
        tensors), or NULL when unallocated."""
        v = abi.gsim_tsdf_volume()
        for k in range(3):
            v.origin[k] = self.origin[k]
            v.dims[k] = self.dims[k]
        v.voxel_size = self.voxel_size
        v.truncation = self.truncation
        dp = C.POINTER(C.c_double)

        def ptr(a):
            if a is None:
                return None
            if hasattr(a, "data_ptr"):  # torch tensor (device grids)
                assert a.is_contiguous() and a.element_size() == 8 and a.numel() == self.voxel_count
                return a.data_ptr()
            assert a.dtype == np.float64 and a.flags.c_contiguous and a.size == self.voxel_count
            return a.ctypes.data
        tsdf_ptr = ptr(self.tsdf) if tsdf_ptr is None else tsdf_ptr
        weights_ptr = ptr(self.weights) if weights_ptr is None else weights_ptr
        v.tsdf = C.cast(C.c_void_p(tsdf_ptr), dp) if tsdf_ptr else dp()
        v.weights = C.cast(C.c_void_p(weights_ptr), dp) if weights_ptr else dp()
        return v

    @staticmethod
    def from_c(v: abi.gsim_tsdf_volume) -> "TsdfVolume":
        return TsdfVolume(tuple(v.origin), v.voxel_size, tuple(v.dims), v.truncation)


class LidarModel:
    """LidarModel (trace.hpp:47-54): spinning scan, one ray per (channel elevation, azimuth step);
    pose maps sensor -> world."""

    def __init__(self, channels, azimuth_step: float, max_range: float,
                 pose: "RigidTransform | None" = None, alpha_threshold: float = 0.5, env: int = -1):
        self.channels = np.ascontiguousarray(channels, dtype=np.float64).reshape(-1)
        self.azimuth_step = float(azimuth_step)
        self.max_range = float(max_range)
        self.pose = pose or RigidTransform()
        self.alpha_threshold = float(alpha_threshold)
        self.env = int(env)

    def azimuth_count(self) -> int:  # lidar_azimuth_count, trace.cpp:162-164
        return int(round(2.0 * math.pi / self.azimuth_step))

    def to_c(self) -> abi.gsim_lidar:
        c = abi.gsim_lidar()
        c.channels = self.channels.ctypes.data_as(C.POINTER(C.c_double))
        c.n_channels = len(self.channels)
        c.azimuth_step = self.azimuth_step
        c.max_range = self.max_range
        c.pose = self.pose.to_c()
        c.alpha_threshold = self.alpha_threshold
        c.env = self.env
        c._keep = self.channels  # the C struct points into this array
        return c


def _nodes_array(nodes: Sequence[SceneNode]):
    if isinstance(nodes, C.Array) and nodes._type_ is abi.gsim_node:
        return nodes  # prebuilt table (scenes.nodes_table)
    arr = (abi.gsim_node * max(len(nodes), 1))()
    for k, n in enumerate(nodes):
        arr[k] = n.to_c() if isinstance(n, SceneNode) else n
    return arr


def _cams_array(cameras: Sequence[CameraModel]):
    if isinstance(cameras, C.Array) and cameras._type_ is abi.gsim_camera:
        return cameras
    arr = (abi.gsim_camera * max(len(cameras), 1))()
    for k, c in enumerate(cameras):
        arr[k] = c.to_c() if isinstance(c, CameraModel) else c
    return arr


class Scene:
    """A GaussianField resident in HBM on one context's device."""

    def __init__(self, ctx: "Context", handle: C.c_void_p, size: int):
        self.ctx = ctx
        self.handle = handle
        self.size = size

    def transform_primitives(self, begin: int, end: int, transform: RigidTransform) -> None:
        """transform_primitives (gaussian.cpp:65-79) on the device copy (K1)."""
        t = transform.to_c()
        _check(self.ctx.lib.gsim_gpu_transform_primitives(self.ctx.ptr, self.handle, begin, end,
                                                          C.byref(t)), self.ctx.ptr)

    def write(self, offset: int, field: GaussianField) -> None:
        """Fill primitives [offset, offset + field.size()) (gsim_gpu_scene_write)."""
        v = field.view()
        _check(self.ctx.lib.gsim_gpu_scene_write(self.ctx.ptr, self.handle, int(offset), C.byref(v)),
               self.ctx.ptr)

    def download(self):
        means = np.zeros((self.size, 3))
        rots = np.zeros((self.size, 4))
        dp = C.POINTER(C.c_double)
        _check(self.ctx.lib.gsim_gpu_scene_download(self.ctx.ptr, self.handle, means.ctypes.data_as(dp),
                                                    rots.ctypes.data_as(dp)), self.ctx.ptr)
        return means, rots

    @property
    def sh_degree(self) -> int:
        return int(self.ctx.lib.gsim_gpu_scene_sh_degree(self.handle))

    def download_field(self) -> "GaussianField":
        """Every plane of the device field, in the reference's per-primitive layout."""
        n = self.size
        arrs = [np.zeros((max(n, 1), w)) for w in (3, 3, 4, 1, 48)]
        dp = C.POINTER(C.c_double)
        _check(self.ctx.lib.gsim_gpu_scene_download_field(self.ctx.ptr, self.handle,
                                                          *[a.ctypes.data_as(dp) for a in arrs]),
               self.ctx.ptr)
        m, s, q, o, sh = (a[:n] for a in arrs)
        return GaussianField(m, s, q, o.reshape(-1), sh, self.sh_degree)

    def close(self) -> None:
        if self.handle:
            self.ctx.lib.gsim_gpu_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PoseTracks:
    """Device-resident pose tracks (PoseStream, pose_stream.hpp:22-49), one per driven node."""

    def __init__(self, ctx: "Context", handle: C.c_void_p, count: int):
        self.ctx, self.handle, self.count = ctx, handle, count

    def sample(self, track, time, initial) -> np.ndarray:
        """PoseStream::sample for queries (track[i], time[i], initial[i]); returns (n, 7) rows
        (qw, qx, qy, qz, tx, ty, tz)."""
        tr = np.ascontiguousarray(np.broadcast_to(track, np.shape(time)), dtype=np.uint32).reshape(-1)
        tt = np.ascontiguousarray(time, dtype=np.float64).reshape(-1)
        n = len(tt)
        inits = initial if isinstance(initial, (list, tuple)) else [initial] * n
        ia = (abi.gsim_rigid * max(n, 1))(*[r.to_c() for r in inits])
        out = (abi.gsim_rigid * max(n, 1))()
        _check(self.ctx.lib.gsim_gpu_tracks_sample(self.ctx.ptr, self.handle,
                                                   tr.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                   tt.ctypes.data_as(C.POINTER(C.c_double)), ia, n,
                                                   out), self.ctx.ptr)
        return np.array([list(out[k].rotation) + list(out[k].translation) for k in range(n)],
                        dtype=np.float64).reshape(-1, 7)

    def close(self) -> None:
        if self.handle:
            self.ctx.lib.gsim_gpu_tracks_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One device: a CUDA stream and grow-only HBM workspaces (gsim_gpu_context)."""

    def __init__(self, device: int = 0):
        self.lib = abi.load_library()
        p = C.c_void_p()
        st = self.lib.gsim_gpu_context_create(device, C.byref(p))
        if st != abi.GSIM_OK:
            msg = (self.lib.gsim_gpu_last_error(None) or b"").decode()
            raise (ValidationError if st == abi.GSIM_ERR_VALIDATION else IoError)(msg)
        self.ptr = p
        self.device = device
        self.lock = threading.Lock()

    def close(self) -> None:
        if self.ptr:
            self.lib.gsim_gpu_context_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self.lib.gsim_gpu_stream(self.ptr) or 0)

    def synchronize(self) -> None:
        _check(self.lib.gsim_gpu_synchronize(self.ptr), self.ptr)

    def set_profiling(self, enable: bool) -> None:
        _check(self.lib.gsim_gpu_set_profiling(self.ptr, 1 if enable else 0), self.ptr)

    def stats(self) -> dict:
        s = abi.gsim_render_stats()
        _check(self.lib.gsim_gpu_get_stats(self.ptr, C.byref(s)), self.ptr)
        return {name: getattr(s, name) for name, _ in s._fields_ if name != "reserved"}

    def upload(self, field: GaussianField) -> Scene:
        v = field.view()
        h = C.c_void_p()
        _check(self.lib.gsim_gpu_scene_upload(self.ptr, C.byref(v), C.byref(h)), self.ptr)
        return Scene(self, h, field.size())

    def create_scene(self, count: int, sh_degree: int) -> Scene:
        """A zeroed device field of `count` primitives, filled piecewise with Scene.write."""
        h = C.c_void_p()
        _check(self.lib.gsim_gpu_scene_create(self.ptr, int(count), int(sh_degree), C.byref(h)), self.ptr)
        return Scene(self, h, int(count))

    def load_ply(self, path) -> Scene:
        """load_splat_ply (splat_ply.cpp:40-162) straight into a device-resident field."""
        h = C.c_void_p()
        _check(self.lib.gsim_gpu_scene_load_ply(self.ptr, str(path).encode(), C.byref(h)), self.ptr)
        return Scene(self, h, int(self.lib.gsim_gpu_scene_size(h)))

    def project(self, scene: Scene, nodes: Sequence[SceneNode], camera: CameraModel) -> np.ndarray:
        na = _nodes_array(nodes)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        count = C.c_uint64(0)
        out = np.zeros(scene.size, dtype=abi.SPLAT_DTYPE)
        _check(self.lib.gsim_gpu_project(self.ptr, scene.handle, na, len(nodes), C.byref(cam),
                                         out.ctypes.data_as(C.c_void_p), scene.size, C.byref(count)),
               self.ptr)
        return out[: count.value].copy()

    def rasterize(self, splats: np.ndarray, camera: CameraModel,
                  options: RasterOptions | None = None) -> RenderTarget:
        splats = np.ascontiguousarray(splats, dtype=abi.SPLAT_DTYPE)
        cam = camera.to_c() if isinstance(camera, CameraModel) else camera
        opt = (options or RasterOptions()).to_c()
        t = RenderTarget.empty(cam.width, cam.height)
        tc = t.to_c()
        _check(self.lib.gsim_gpu_rasterize(self.ptr, splats.ctypes.data_as(C.c_void_p), len(splats),
                                           C.byref(cam), C.byref(opt), C.byref(tc)), self.ptr)
        return t

    def render(self, scene: Scene, nodes: Sequence[SceneNode], cameras: Sequence[CameraModel],
               options: RasterOptions | None = None,
               targets: Sequence[RenderTarget] | None = None) -> list[RenderTarget]:
        na = _nodes_array(nodes)
        ca = _cams_array(cameras)
        opt = (options or RasterOptions()).to_c()
        if targets is None:
            targets = [RenderTarget.empty(ca[k].width, ca[k].height) for k in range(len(cameras))]
        ta = _targets_array(targets, ca, len(cameras))
        _check(self.lib.gsim_gpu_render(self.ptr, scene.handle, na, len(nodes), ca, len(cameras),
                                        C.byref(opt), ta), self.ptr)
        return list(targets)

    def render_device(self, scene: Scene, nodes, cameras, options: RasterOptions | None = None,
                      device_out: int | None = None) -> int:
        """Asynchronous render into device memory; returns the output device pointer."""
        na = _nodes_array(nodes)
        ca = _cams_array(cameras)
        opt = (options or RasterOptions()).to_c()
        _check(self.lib.gsim_gpu_render_device(self.ptr, scene.handle, na, len(nodes), ca,
                                               len(cameras), C.byref(opt),
                                               C.c_void_p(device_out) if device_out else None),
               self.ptr)
        return device_out if device_out else int(self.lib.gsim_gpu_device_output(self.ptr))

    # -- pose playback (pose_stream.cpp / scene.cpp step_to) ----------------------------------
    def upload_tracks(self, tracks) -> PoseTracks:
        """tracks: list of (times[R], translations[R,3], rotations[R,4] as w,x,y,z) per node."""
        times = [np.asarray(t, dtype=np.float64).reshape(-1) for t, _, _ in tracks]
        begin = np.zeros(len(tracks) + 1, dtype=np.uint64)
        begin[1:] = np.cumsum([len(t) for t in times])
        cat = lambda xs, w: (np.ascontiguousarray(np.concatenate(xs), dtype=np.float64)
                             if xs and sum(len(x) for x in xs) else np.zeros(w))
        tt = cat(times, 1)
        pp = cat([np.asarray(p, dtype=np.float64).reshape(-1, 3) for _, p, _ in tracks], 3).reshape(-1)
        qq = cat([np.asarray(q, dtype=np.float64).reshape(-1, 4) for _, _, q in tracks], 4).reshape(-1)
        handle = C.c_void_p()
        dp = C.POINTER(C.c_double)
        _check(self.lib.gsim_gpu_tracks_upload(self.ptr, tt.ctypes.data_as(dp), pp.ctypes.data_as(dp),
                                               qq.ctypes.data_as(dp),
                                               begin.ctypes.data_as(C.POINTER(C.c_uint64)),
                                               len(tracks), C.byref(handle)), self.ptr)
        return PoseTracks(self, handle, len(tracks))

    def render_at(self, scene: Scene, tracks: PoseTracks, time: float, nodes, node_track,
                  cameras, options: RasterOptions | None = None, targets=None,
                  device_out: int | None = None):
        """Render with node poses sampled on the GPU at `time` (Scene::step_to + render_all).
        Host targets (synchronous) unless device_out is given."""
        na = _nodes_array(nodes)
        nt = np.ascontiguousarray(node_track, dtype=np.int64).reshape(-1)
        if len(nt) != len(nodes):
            raise ValidationError("render_at: node_track needs one entry per node")
        ca = _cams_array(cameras)
        opt = (options or RasterOptions()).to_c()
        if device_out:
            _check(self.lib.gsim_gpu_render_at(self.ptr, scene.handle, tracks.handle, float(time), na,
                                               nt.ctypes.data_as(C.POINTER(C.c_int64)), len(nodes),
                                               ca, len(cameras), C.byref(opt),
                                               C.c_void_p(device_out), None), self.ptr)
            return device_out
        if targets is None:
            targets = [RenderTarget.empty(ca[k].width, ca[k].height) for k in range(len(cameras))]
        ta = _targets_array(targets, ca, len(cameras))
        _check(self.lib.gsim_gpu_render_at(self.ptr, scene.handle, tracks.handle, float(time), na,
                                           nt.ctypes.data_as(C.POINTER(C.c_int64)), len(nodes), ca,
                                           len(cameras), C.byref(opt), None, ta), self.ptr)
        return targets

    # -- output encoding (image_io.cpp writers' bytes) -----------------------------------------
    def encode_target(self, target: "RenderTarget", options: EncodeOptions | None = None) -> np.ndarray:
        """Encode one host RenderTarget on the GPU (gsim_gpu_encode_host)."""
        o = options or EncodeOptions()
        h, w = target.depth.shape
        out = np.zeros(max(o.bytes_per_camera(w, h), 1), dtype=np.uint8)
        planes = [np.ascontiguousarray(a, dtype=np.float32) for a in (target.rgb, target.depth,
                                                                      target.accum_alpha)]
        fp = C.POINTER(C.c_float)
        oc = o.to_c()
        _check(self.lib.gsim_gpu_encode_host(self.ptr, w, h, *[a.ctypes.data_as(fp) for a in planes],
                                             C.byref(oc), out.ctypes.data_as(C.POINTER(C.c_uint8))),
               self.ptr)
        return out[: o.bytes_per_camera(w, h)]

    def encode(self, device_targets: int, cameras: Sequence[CameraModel],
               options: EncodeOptions | None = None, device_out: int | None = None):
        """Encode render_device output; returns a host blob, or device_out when given."""
        o = options or EncodeOptions()
        ca = _cams_array(cameras)
        oc = o.to_c()
        if device_out:
            _check(self.lib.gsim_gpu_encode(self.ptr, C.c_void_p(device_targets), ca, len(cameras),
                                            C.byref(oc), C.c_void_p(device_out), 1), self.ptr)
            return device_out
        n = sum(o.bytes_per_camera(c.width, c.height) for c in cameras)
        out = np.zeros(max(n, 1), dtype=np.uint8)
        _check(self.lib.gsim_gpu_encode(self.ptr, C.c_void_p(device_targets), ca, len(cameras),
                                        C.byref(oc), out.ctypes.data_as(C.c_void_p), 0), self.ptr)
        return out[:n]

    def render_encoded(self, scene: Scene, nodes, cameras, options: RasterOptions | None = None,
                       encode: EncodeOptions | None = None, out: np.ndarray | None = None,
                       device_out: int | None = None):
        """render + encode fused in the compositing kernel (gsim_gpu_render_encoded). Host blob
        (synchronous) unless device_out is given (asynchronous, like render_device)."""
        o = encode or EncodeOptions()
        na = _nodes_array(nodes)
        ca = _cams_array(cameras)
        opt = (options or RasterOptions()).to_c()
        oc = o.to_c()
        if device_out:
            _check(self.lib.gsim_gpu_render_encoded(self.ptr, scene.handle, na, len(nodes), ca,
                                                    len(cameras), C.byref(opt), C.byref(oc),
                                                    C.c_void_p(device_out), 1), self.ptr)
            return device_out
        n = sum(o.bytes_per_camera(c.width, c.height) for c in cameras)
        if out is None:
            out = np.zeros(max(n, 1), dtype=np.uint8)
        elif (not isinstance(out, np.ndarray) or out.dtype != np.uint8 or not out.flags["C_CONTIGUOUS"]
              or not out.flags["WRITEABLE"] or out.size < n):
            raise ValidationError(f"render_encoded: out must be a writeable contiguous uint8 array of "
                                  f">= {n} bytes")
        _check(self.lib.gsim_gpu_render_encoded(self.ptr, scene.handle, na, len(nodes), ca,
                                                len(cameras), C.byref(opt), C.byref(oc),
                                                out.ctypes.data_as(C.c_void_p), 0), self.ptr)
        return out[:n]

    # -- GS -> TSDF (transfer.cpp) -----------------------------------------
    def scene_bounds(self, scene: Scene):
        """field_bounds (transfer.cpp:27-34) of a device scene -> (lo, hi)."""
        lo = (C.c_double * 3)(); hi = (C.c_double * 3)()
        _check(self.lib.gsim_gpu_scene_bounds(self.ptr, scene.handle, lo, hi), self.ptr)
        return tuple(lo), tuple(hi)

    def render_depth_ring(self, scene: Scene, n_views: int, radius: float, resolution: int,
                          device_out: int | None = None):
        """render_depth_ring (transfer.cpp:81-124) -> (3 * n_views cameras, depth): a host float32
        (3 * n_views, resolution, resolution) array, or device_out filled asynchronously-safe
        (the call returns after the copy)."""
        n = 3 * max(int(n_views), 1)
        cams = (abi.gsim_camera * n)()
        if device_out:
            _check(self.lib.gsim_gpu_render_depth_ring(self.ptr, scene.handle, n_views, radius,
                                                       resolution, cams, C.c_void_p(device_out), 1),
                   self.ptr)
            return cams, device_out
        depth = np.zeros((n, resolution, resolution), dtype=np.float32)
        _check(self.lib.gsim_gpu_render_depth_ring(self.ptr, scene.handle, n_views, radius,
                                                   resolution, cams,
                                                   depth.ctypes.data_as(C.c_void_p), 0), self.ptr)
        return cams, depth

    def tsdf_reset(self, volume: "TsdfVolume") -> None:
        c = volume.to_c()
        _check(self.lib.gsim_gpu_tsdf_reset(self.ptr, C.byref(c)), self.ptr)

    def tsdf_fuse(self, volume: "TsdfVolume", cameras, depth) -> None:
        """tsdf_fuse (transfer.cpp:143-172) of the views in order; volume grids on the device
        (TsdfVolume.device_grids). depth: host float32 images (n, H, W) or a device pointer."""
        ca = _cams_array(cameras)
        c = volume.to_c()
        if isinstance(depth, int):
            _check(self.lib.gsim_gpu_tsdf_fuse(self.ptr, C.byref(c), ca, len(cameras),
                                               C.c_void_p(depth), 1), self.ptr)
            return
        d = np.ascontiguousarray(depth, dtype=np.float32)
        _check(self.lib.gsim_gpu_tsdf_fuse(self.ptr, C.byref(c), ca, len(cameras),
                                           d.ctypes.data_as(C.c_void_p), 0), self.ptr)

    def gaussians_to_tsdf(self, scene: Scene, voxel_size: float) -> "TsdfVolume":
        """gaussians_to_mesh up to the fused volume (transfer.cpp:174-198); device grids."""
        c = abi.gsim_tsdf_volume()
        _check(self.lib.gsim_gpu_gaussians_to_tsdf(self.ptr, scene.handle, voxel_size, C.byref(c)),
               self.ptr)
        vol = TsdfVolume.from_c(c).device_grids()
        c = vol.to_c()
        _check(self.lib.gsim_gpu_gaussians_to_tsdf(self.ptr, scene.handle, voxel_size, C.byref(c)),
               self.ptr)
        return vol

    # -- LiDAR (trace.cpp) --------------------------------------------------
    def lidar_scan(self, scene: Scene, nodes, lidar: "LidarModel") -> dict:
        """GaussianBvh::build(field, nodes).scan(lidar) -> {"points" (n, 3) sensor frame,
        "ring" (n,), "azimuth" (n,)} in channel-major, azimuth-ascending order, misses omitted."""
        na = _nodes_array(nodes)
        lc = lidar.to_c()
        cnt = C.c_uint64(0)
        dp, u32p = C.POINTER(C.c_double), C.POINTER(C.c_uint32)
        # a scan returns at most one point per ray: one call with that capacity
        cap = max(1, len(lidar.channels) * lidar.azimuth_count()) if lidar.azimuth_step > 0 else 1
        pts = np.zeros((cap, 3)); ring = np.zeros(cap, np.uint32); az = np.zeros(cap)
        _check(self.lib.gsim_gpu_lidar_scan(self.ptr, scene.handle, na, len(nodes), C.byref(lc),
                                            pts.ctypes.data_as(dp), ring.ctypes.data_as(u32p),
                                            az.ctypes.data_as(dp), cap, C.byref(cnt)), self.ptr)
        n = cnt.value
        return {"points": pts[:n], "ring": ring[:n], "azimuth": az[:n]}

    def trace_rays(self, scene: Scene, nodes, origins, directions, t_max, alpha_threshold: float = 0.5):
        """GaussianBvh::trace per ray -> (hit u8, depth, accum_alpha)."""
        o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(directions, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(np.broadcast_to(np.asarray(t_max, np.float64), (len(o),)))
        n = len(t)
        hit = np.zeros(max(n, 1), np.uint8); depth = np.zeros(max(n, 1)); acc = np.zeros(max(n, 1))
        dp = C.POINTER(C.c_double)
        na = _nodes_array(nodes)
        _check(self.lib.gsim_gpu_trace_rays(self.ptr, scene.handle, na, len(nodes), o.ctypes.data_as(dp),
                                            d.ctypes.data_as(dp), t.ctypes.data_as(dp), n,
                                            alpha_threshold, hit.ctypes.data_as(C.POINTER(C.c_uint8)),
                                            depth.ctypes.data_as(dp), acc.ctypes.data_as(dp)), self.ptr)
        return hit[:n], depth[:n], acc[:n]

    def tile_lists(self, camera: int):
        """Sorted per-tile lists of `camera` from the last render (tile offsets, indices)."""
        count = C.c_uint64(0)
        _check(self.lib.gsim_gpu_tile_lists(self.ptr, camera, None, None, 0, C.byref(count)), self.ptr)
        # tiles of that camera are needed to size the offsets array: ask with a big buffer
        offsets = np.zeros(256 * 256 + 1, dtype=np.uint32)
        values = np.zeros(max(count.value, 1), dtype=np.uint32)
        _check(self.lib.gsim_gpu_tile_lists(self.ptr, camera, offsets.ctypes.data_as(C.POINTER(C.c_uint32)),
                                            values.ctypes.data_as(C.POINTER(C.c_uint32)), count.value,
                                            C.byref(count)), self.ptr)
        return offsets, values[: count.value]


# ---- free functions with the reference's signatures ---------------------------------------

_default = {"ctx": None, "scene": None, "key": None}
_default_lock = threading.Lock()


def default_context() -> Context:
    with _default_lock:
        if _default["ctx"] is None:
            _default["ctx"] = Context(0)
        return _default["ctx"]


def _scene_for(field: GaussianField) -> Scene:
    ctx = default_context()
    key = (id(field), field.size(), field.generation, field.means.ctypes.data)
    with _default_lock:
        if _default["key"] != key:
            _default["scene"] = None
            _default["scene"] = ctx.upload(field)
            _default["key"] = key
        return _default["scene"]


def project(field: GaussianField, nodes: Sequence[SceneNode], camera: CameraModel) -> np.ndarray:
    """raster.hpp:54-56 — visible splats (ProjectedSplat records) in primitive order."""
    return default_context().project(_scene_for(field), nodes, camera)


def rasterize(splats: np.ndarray, camera: CameraModel, options: RasterOptions | None = None) -> RenderTarget:
    """raster.hpp:59-60."""
    return default_context().rasterize(splats, camera, options)


def render(field: GaussianField, nodes: Sequence[SceneNode], cameras: Sequence[CameraModel],
           options: RasterOptions | None = None) -> list[RenderTarget]:
    """raster.hpp:64-67 — one target per camera."""
    return default_context().render(_scene_for(field), nodes, cameras, options)


def transform_primitives(field: GaussianField, rng: tuple, transform: RigidTransform) -> None:
    """gaussian.hpp:76-77 — in place; runs K1 on the device copy and writes the result back."""
    begin, end = int(rng[0]), int(rng[1])
    if begin > end or end > field.size():
        raise ValidationError(f"transform_primitives: range [{begin},{end}) outside field of size {field.size()}")
    scene = _scene_for(field)
    scene.transform_primitives(begin, end, transform)
    means, rots = scene.download()
    field.means[:] = means
    field.rotations[:] = rots
    field.touch()
    with _default_lock:  # the device copy already holds the transformed field
        _default["key"] = (id(field), field.size(), field.generation, field.means.ctypes.data)


def depth_ring_cameras(lo, hi, n_views: int, radius: float, resolution: int):
    """The 3 * n_views cameras of render_depth_ring (transfer.cpp:84-112); host only."""
    lib = abi.load_library()
    cams = (abi.gsim_camera * (3 * max(int(n_views), 1)))()
    st = lib.gsim_gpu_depth_ring_cameras((C.c_double * 3)(*lo), (C.c_double * 3)(*hi), n_views,
                                         radius, resolution, cams)
    if st != 0:
        raise ValidationError("depth_ring_cameras: invalid ring (n_views < 8, radius, or box)")
    return cams


def tsdf_create(origin, voxel_size: float, dims, truncation: float) -> "TsdfVolume":
    """TsdfVolume::create (transfer.cpp:126-141) validation; geometry only (no grids)."""
    lib = abi.load_library()
    c = abi.gsim_tsdf_volume()
    st = lib.gsim_gpu_tsdf_create((C.c_double * 3)(*origin), voxel_size,
                                  (C.c_int32 * 3)(*[int(d) for d in dims]), truncation, C.byref(c))
    if st != 0:
        raise ValidationError("tsdf: invalid volume (voxel_size, dims >= 2, truncation >= 2 voxels)")
    return TsdfVolume.from_c(c)
