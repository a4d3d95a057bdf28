"""ctypes mirror of include/gsim_gpu.h and the loader of libgsim_gpu.so.

There is no fallback: if the CUDA library is missing or fails to load, every entry point
raises. Build it with ``python -m paper_2507_21981_b200.build`` (or __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libgsim_gpu.so"
# A/B measurement hook: another in-tree build of the same library (e.g. libgsim_gpu_b.so)
if os.environ.get("GSIM_GPU_LIB"):
    LIB_PATH = Path(__file__).resolve().parent / Path(os.environ["GSIM_GPU_LIB"]).name

GSIM_OK = 0
GSIM_ERR_IO = 1
GSIM_ERR_VALIDATION = 2
GSIM_NODE_BACKGROUND = 0
GSIM_NODE_INTERACTIVE = 1
GSIM_ENV_ALL = -1
GSIM_ENCODE_RGB8 = 1
GSIM_ENCODE_ALPHA8 = 2
GSIM_ENCODE_DEPTH16 = 4
GSIM_ENCODE_DEPTH_PFM = 8


class gsim_rigid(C.Structure):
    _fields_ = [("rotation", C.c_double * 4), ("translation", C.c_double * 3)]


class gsim_field_view(C.Structure):
    _fields_ = [
        ("count", C.c_uint64), ("sh_degree", C.c_int32), ("reserved", C.c_int32),
        ("means", C.POINTER(C.c_double)), ("means_stride", C.c_uint64),
        ("scales", C.POINTER(C.c_double)), ("scales_stride", C.c_uint64),
        ("rotations", C.POINTER(C.c_double)), ("rotations_stride", C.c_uint64),
        ("opacities", C.POINTER(C.c_double)), ("opacities_stride", C.c_uint64),
        ("sh", C.POINTER(C.c_double)), ("sh_stride", C.c_uint64),
    ]


class gsim_node(C.Structure):
    _fields_ = [("begin", C.c_uint64), ("end", C.c_uint64), ("pose", gsim_rigid),
                ("kind", C.c_int32), ("env", C.c_int32)]


class gsim_camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("pose", gsim_rigid),
                ("near_plane", C.c_double), ("far_plane", C.c_double),
                ("env", C.c_int32), ("reserved", C.c_int32)]


class gsim_raster_options(C.Structure):
    _fields_ = [("normalize_depth", C.c_int32), ("reserved", C.c_int32),
                ("transmittance_cutoff", C.c_double)]


class gsim_encode_options(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("srgb", C.c_int32), ("depth_scale", C.c_double)]


class gsim_projected_splat(C.Structure):
    _fields_ = [("pixel_center", C.c_double * 2), ("cov_xx", C.c_double), ("cov_xy", C.c_double),
                ("cov_yy", C.c_double), ("inv_xx", C.c_double), ("inv_xy", C.c_double),
                ("inv_yy", C.c_double), ("view_depth", C.c_double), ("alpha_peak", C.c_double),
                ("rgb", C.c_double * 3), ("radius", C.c_double), ("prim_index", C.c_uint32),
                ("reserved", C.c_uint32)]


class gsim_target(C.Structure):
    _fields_ = [("rgb", C.POINTER(C.c_float)), ("depth", C.POINTER(C.c_float)),
                ("accum_alpha", C.POINTER(C.c_float))]


class gsim_render_stats(C.Structure):
    _fields_ = [("slots", C.c_uint64), ("visible", C.c_uint64), ("pairs", C.c_uint64),
                ("tiles", C.c_uint64), ("launches", C.c_uint64), ("launches_total", C.c_uint64),
                ("consumed", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("depth_passes", C.c_uint32), ("chunks", C.c_uint32),
                ("ms_preprocess", C.c_float), ("ms_depth_sort", C.c_float),
                ("ms_binning", C.c_float), ("ms_scatter", C.c_float),
                ("ms_raster", C.c_float), ("ms_total", C.c_float),
                ("groups", C.c_uint32), ("last_group_cameras", C.c_uint32)]


class gsim_tsdf_volume(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("voxel_size", C.c_double), ("dims", C.c_int32 * 3),
                ("reserved", C.c_int32), ("truncation", C.c_double),
                ("tsdf", C.POINTER(C.c_double)), ("weights", C.POINTER(C.c_double))]


class gsim_lidar(C.Structure):
    _fields_ = [("channels", C.POINTER(C.c_double)), ("n_channels", C.c_uint64),
                ("azimuth_step", C.c_double), ("max_range", C.c_double), ("pose", gsim_rigid),
                ("alpha_threshold", C.c_double), ("env", C.c_int32), ("reserved", C.c_int32)]


# numpy view of gsim_projected_splat (ProjectedSplat, raster.hpp:20-29), 120 bytes
SPLAT_DTYPE = np.dtype([
    ("pixel_center", "<f8", (2,)), ("cov_xx", "<f8"), ("cov_xy", "<f8"), ("cov_yy", "<f8"),
    ("inv_xx", "<f8"), ("inv_xy", "<f8"), ("inv_yy", "<f8"), ("view_depth", "<f8"),
    ("alpha_peak", "<f8"), ("rgb", "<f8", (3,)), ("radius", "<f8"), ("prim_index", "<u4"),
    ("reserved", "<u4"),
])
assert SPLAT_DTYPE.itemsize == C.sizeof(gsim_projected_splat) == 120

# Every symbol include/gsim_gpu.h declares: (name, restype, argtypes)
_P = C.c_void_p
SIGNATURES = [
    ("gsim_gpu_version", C.c_char_p, []),
    ("gsim_gpu_context_create", C.c_int, [C.c_int, C.POINTER(_P)]),
    ("gsim_gpu_context_destroy", C.c_int, [_P]),
    ("gsim_gpu_last_error", C.c_char_p, [_P]),
    ("gsim_gpu_stream", _P, [_P]),
    ("gsim_gpu_synchronize", C.c_int, [_P]),
    ("gsim_gpu_set_profiling", C.c_int, [_P, C.c_int]),
    ("gsim_gpu_get_stats", C.c_int, [_P, C.POINTER(gsim_render_stats)]),
    ("gsim_gpu_scene_upload", C.c_int, [_P, C.POINTER(gsim_field_view), C.POINTER(_P)]),
    ("gsim_gpu_scene_destroy", C.c_int, [_P]),
    ("gsim_gpu_scene_create", C.c_int, [_P, C.c_uint64, C.c_int32, C.POINTER(_P)]),
    ("gsim_gpu_ipc_alloc", C.c_int, [C.c_int32, C.c_uint64, C.POINTER(_P), C.POINTER(C.c_uint8)]),
    ("gsim_gpu_ipc_free", C.c_int, [C.c_int32, _P]),
    ("gsim_gpu_ipc_open", C.c_int, [C.c_int32, C.POINTER(C.c_uint8), C.POINTER(_P)]),
    ("gsim_gpu_ipc_close", C.c_int, [C.c_int32, _P]),
    ("gsim_gpu_scene_write", C.c_int, [_P, _P, C.c_uint64, C.POINTER(gsim_field_view)]),
    ("gsim_gpu_scene_size", C.c_uint64, [_P]),
    ("gsim_gpu_transform_primitives", C.c_int, [_P, _P, C.c_uint64, C.c_uint64, C.POINTER(gsim_rigid)]),
    ("gsim_gpu_scene_download", C.c_int, [_P, _P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("gsim_gpu_scene_download_field", C.c_int, [_P, _P] + [C.POINTER(C.c_double)] * 5),
    ("gsim_gpu_scene_sh_degree", C.c_int32, [_P]),
    ("gsim_gpu_scene_load_ply", C.c_int, [_P, C.c_char_p, C.POINTER(_P)]),
    ("gsim_gpu_project", C.c_int, [_P, _P, C.POINTER(gsim_node), C.c_uint64, C.POINTER(gsim_camera),
                                   _P, C.c_uint64, C.POINTER(C.c_uint64)]),
    ("gsim_gpu_rasterize", C.c_int, [_P, _P, C.c_uint64, C.POINTER(gsim_camera),
                                     C.POINTER(gsim_raster_options), C.POINTER(gsim_target)]),
    ("gsim_gpu_render", C.c_int, [_P, _P, C.POINTER(gsim_node), C.c_uint64, C.POINTER(gsim_camera),
                                  C.c_uint64, C.POINTER(gsim_raster_options), C.POINTER(gsim_target)]),
    ("gsim_gpu_render_device", C.c_int, [_P, _P, C.POINTER(gsim_node), C.c_uint64,
                                         C.POINTER(gsim_camera), C.c_uint64,
                                         C.POINTER(gsim_raster_options), _P]),
    ("gsim_gpu_device_output", _P, [_P]),
    ("gsim_gpu_tile_lists", C.c_int, [_P, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                      C.c_uint64, C.POINTER(C.c_uint64)]),
    ("gsim_gpu_tracks_upload", C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_uint64,
                                         C.POINTER(_P)]),
    ("gsim_gpu_tracks_destroy", C.c_int, [_P]),
    ("gsim_gpu_tracks_count", C.c_uint64, [_P]),
    ("gsim_gpu_tracks_sample", C.c_int, [_P, _P, C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                                         C.POINTER(gsim_rigid), C.c_uint64, C.POINTER(gsim_rigid)]),
    ("gsim_gpu_render_at", C.c_int, [_P, _P, _P, C.c_double, C.POINTER(gsim_node),
                                     C.POINTER(C.c_int64), C.c_uint64, C.POINTER(gsim_camera),
                                     C.c_uint64, C.POINTER(gsim_raster_options), _P,
                                     C.POINTER(gsim_target)]),
    ("gsim_gpu_encoded_bytes", C.c_uint64, [C.c_uint32, C.c_int32, C.c_int32]),
    ("gsim_gpu_srgb_thresholds", None, [C.POINTER(C.c_float)]),
    ("gsim_gpu_hash_target", C.c_uint64, [C.c_int32, C.c_int32, C.POINTER(C.c_float),
                                          C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_uint64]),
    ("gsim_gpu_encode_host", C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_float),
                                       C.POINTER(C.c_float), C.POINTER(C.c_float),
                                       C.POINTER(gsim_encode_options), C.POINTER(C.c_uint8)]),
    ("gsim_gpu_encode", C.c_int, [_P, _P, C.POINTER(gsim_camera), C.c_uint64,
                                  C.POINTER(gsim_encode_options), _P, C.c_int32]),
    ("gsim_gpu_render_encoded", C.c_int, [_P, _P, C.POINTER(gsim_node), C.c_uint64,
                                          C.POINTER(gsim_camera), C.c_uint64,
                                          C.POINTER(gsim_raster_options),
                                          C.POINTER(gsim_encode_options), _P, C.c_int32]),
    ("gsim_gpu_scene_bounds", C.c_int, [_P, _P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("gsim_gpu_depth_ring_cameras", C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double),
                                              C.c_int32, C.c_double, C.c_int32,
                                              C.POINTER(gsim_camera)]),
    ("gsim_gpu_render_depth_ring", C.c_int, [_P, _P, C.c_int32, C.c_double, C.c_int32,
                                             C.POINTER(gsim_camera), _P, C.c_int32]),
    ("gsim_gpu_tsdf_create", C.c_int, [C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_int32),
                                       C.c_double, C.POINTER(gsim_tsdf_volume)]),
    ("gsim_gpu_tsdf_reset", C.c_int, [_P, C.POINTER(gsim_tsdf_volume)]),
    ("gsim_gpu_tsdf_fuse", C.c_int, [_P, C.POINTER(gsim_tsdf_volume), C.POINTER(gsim_camera),
                                     C.c_uint64, _P, C.c_int32]),
    ("gsim_gpu_gaussians_to_tsdf", C.c_int, [_P, _P, C.c_double, C.POINTER(gsim_tsdf_volume)]),
    ("gsim_gpu_tsdf_alloc", C.c_int, [_P, C.POINTER(gsim_tsdf_volume)]),
    ("gsim_gpu_tsdf_free", C.c_int, [C.POINTER(gsim_tsdf_volume)]),
    ("gsim_gpu_tsdf_download", C.c_int, [_P, C.POINTER(gsim_tsdf_volume), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]),
    ("gsim_gpu_lidar_scan", C.c_int, [_P, _P, C.POINTER(gsim_node), C.c_uint64, C.POINTER(gsim_lidar),
                                      C.POINTER(C.c_double), C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_double), C.c_uint64, C.POINTER(C.c_uint64)]),
    ("gsim_gpu_trace_rays", C.c_int, [_P, _P, C.POINTER(gsim_node), C.c_uint64, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_uint64,
                                      C.c_double, C.POINTER(C.c_uint8), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]),
    ("gsim_gpu_tsdf_upload", C.c_int, [_P, C.POINTER(gsim_tsdf_volume), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]),
]

_lib = None


def load_library(path: Path | None = None) -> C.CDLL:
    """Load libgsim_gpu.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build the CUDA extension first "
            "(python -m paper_2507_21981_b200.build); there is no CPU fallback")
    lib = C.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def header_symbols() -> list[str]:
    """Function names declared in include/gsim_gpu.h (parsed, for the ABI test)."""
    import re
    text = (Path(__file__).resolve().parent.parent / "include" / "gsim_gpu.h").read_text()
    return sorted(set(re.findall(r"\b(gsim_gpu_[a-z_]+)\s*\(", text)))
