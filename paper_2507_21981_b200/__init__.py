"""B200-native multi-camera RGB-D Gaussian-splat renderer (drop-in for gsim's render path).

Host API mirrors the reference (gsim::project / rasterize / render / transform_primitives);
all compute runs in libgsim_gpu.so (hand-written sm_100a CUDA behind the C ABI in
include/gsim_gpu.h). See DESIGN.md.
"""
from .api import (  # noqa: F401
    CameraModel,
    Context,
    EncodeOptions,
    GaussianField,
    IoError,
    LidarModel,
    NodeKind,
    PoseTracks,
    RasterOptions,
    RenderTarget,
    RigidTransform,
    Scene,
    SceneNode,
    TsdfVolume,
    ValidationError,
    default_context,
    depth_ring_cameras,
    io_error,
    project,
    quat_from_axis_angle,
    rasterize,
    render,
    transform_primitives,
    tsdf_create,
    validation_error,
)
from .abi import SPLAT_DTYPE, load_library  # noqa: F401

__all__ = [
    "CameraModel", "Context", "EncodeOptions", "GaussianField", "IoError", "LidarModel", "NodeKind", "PoseTracks", "RasterOptions",
    "RenderTarget", "RigidTransform", "Scene", "SceneNode", "TsdfVolume", "ValidationError",
    "SPLAT_DTYPE", "depth_ring_cameras", "tsdf_create",
    "default_context", "io_error", "load_library", "project", "quat_from_axis_angle",
    "rasterize", "render", "transform_primitives", "validation_error",
]
