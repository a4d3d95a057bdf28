"""Seeded synthetic workloads with the shapes of BASELINE.json's configs 0-4.

The paper's scenes and assets are not available; these generators stand in for them with
the distributions BASELINE.json states. Ambiguities are pinned once here and
documented in DESIGN.md:
  * FOV is horizontal: fx = fy = (W/2) / tan(30 deg); cx, cy = W/2, H/2 (look_at).
  * Object-node local means follow config 0 literally: U[-2, 2]^3 around the node origin.
  * Node poses: yaw ~ U[0, 2 pi) about +z, translation ~ U[-0.5, 0.5]^3, drawn per frame.
  * Camera jitter (config 2): eye += U[-5 cm, 5 cm]^3, then the look-at rotation is
    perturbed by a rotation with per-axis angles U[-3 deg, 3 deg].
  * Config 3 cameras: eyes (0, -6, 1.5) and (0, 6, 1.5) looking at (0, 0, 1.5).
The same arrays (float64, exactly representable) feed the GPU path and the CPU oracle.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .api import (CameraModel, GaussianField, NodeKind, RigidTransform, SceneNode,
                  quat_from_axis_angle, quat_mul, quat_normalized)

VGA = (640, 480)
FOV_DEG = 60.0


def focal_for(width: int, fov_deg: float = FOV_DEG) -> float:
    return (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)


def gaussians(rng: np.random.Generator, n: int, sh_degree: int, log_scale_mu=-4.5,
              log_scale_sigma=0.5, means: np.ndarray | None = None):
    """(means, scales, rotations, opacities, sh) per BASELINE config 0/1 distributions."""
    if means is None:
        means = rng.uniform(-2.0, 2.0, size=(n, 3))
    scales = np.exp(rng.normal(log_scale_mu, log_scale_sigma, size=(n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)  # uniform random unit quaternion
    opac = 1.0 / (1.0 + np.exp(-rng.normal(size=n)))
    opac = np.clip(opac, 1e-6, 1 - 1e-6)
    sh = np.zeros((n, 48))
    K = (sh_degree + 1) ** 2
    for c in range(3):
        sh[:, c * 16] = rng.normal(0.0, 0.3, size=n)              # DC
        if K > 1:
            sh[:, c * 16 + 1: c * 16 + K] = rng.normal(0.0, 0.2, size=(n, K - 1))
    return means, scales, q, opac, sh


def concat_fields(parts, sh_degree: int) -> GaussianField:
    m = np.concatenate([p[0] for p in parts])
    s = np.concatenate([p[1] for p in parts])
    q = np.concatenate([p[2] for p in parts])
    o = np.concatenate([p[3] for p in parts])
    sh = np.concatenate([p[4] for p in parts])
    return GaussianField(m, s, q, o, sh, sh_degree)


def random_node_pose(rng: np.random.Generator) -> RigidTransform:
    yaw = rng.uniform(0.0, 2.0 * math.pi)
    t = rng.uniform(-0.5, 0.5, size=3)
    return RigidTransform(quat_from_axis_angle((0.0, 0.0, 1.0), yaw), tuple(float(x) for x in t))


def ring_cameras(n: int, radius: float, height: float, width: int, height_px: int,
                 env: int = 0) -> list[CameraModel]:
    f = focal_for(width)
    cams = []
    for k in range(n):
        az = 2.0 * math.pi * k / n
        eye = (radius * math.cos(az), radius * math.sin(az), height)
        c = CameraModel.look_at(eye, (0.0, 0.0, 0.0), f, f, width, height_px)
        c.id = f"cam{k}"
        c.env = env
        cams.append(c)
    return cams


def jitter_camera(rng: np.random.Generator, cam: CameraModel) -> CameraModel:
    """Eye +-5 cm per axis, orientation +-3 deg per axis (uniform)."""
    center = cam.camera_center()
    eye = tuple(center[i] + rng.uniform(-0.05, 0.05) for i in range(3))
    ang = np.radians(rng.uniform(-3.0, 3.0, size=3))
    dq = (1.0, 0.0, 0.0, 0.0)
    for axis, a in zip(((1.0, 0, 0), (0, 1.0, 0), (0, 0, 1.0)), ang):
        dq = quat_mul(quat_from_axis_angle(axis, float(a)), dq)
    rot = quat_normalized(quat_mul(dq, cam.pose.rotation))  # perturb world->camera rotation
    from .api import quat_rotate
    t = quat_rotate(rot, eye)
    out = CameraModel(id=cam.id, fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width,
                      height=cam.height, pose=RigidTransform(rot, (-t[0], -t[1], -t[2])),
                      near=cam.near, far=cam.far, env=cam.env)
    return out


@dataclass
class Workload:
    name: str
    field: GaussianField
    nodes: list            # SceneNode list (poses are re-drawn per frame by frame_nodes)
    cameras: list
    object_nodes: list     # indices into nodes that move per frame
    description: str = ""

    def frame_nodes(self, frame: int, seed: int = 0) -> list:
        """Per-frame random rigid poses for the object nodes (config 1/2/4)."""
        rng = np.random.default_rng((seed, 7919, frame))
        out = []
        for k, n in enumerate(self.nodes):
            if k in self._movers:
                n = SceneNode(n.id, n.kind, random_node_pose(rng), n.range, n.env)
            out.append(n)
        return out

    @property
    def _movers(self):
        s = getattr(self, "_mover_set", None)
        if s is None:
            s = set(self.object_nodes)
            self._mover_set = s
        return s

    def pixels(self) -> int:
        return sum(c.width * c.height for c in self.cameras)


def config0(seed: int = 0, n: int = 100_000) -> Workload:
    """Single camera 640x480, 100k SH0 Gaussians, eye (5,0,0) looking at the origin."""
    rng = np.random.default_rng((seed, 0))
    field = concat_fields([gaussians(rng, n, 0)], 0)
    f = focal_for(640)
    cam = CameraModel.look_at((5.0, 0.0, 0.0), (0.0, 0.0, 0.0), f, f, 640, 480)
    cam.id = "cam0"
    nodes = [SceneNode("bg", NodeKind.background, RigidTransform(), (0, n))]
    return Workload("cfg0", field, nodes, [cam], [], "100k SH0, 1x640x480")


def _env_objects(rng, n_objects, per_object, sh_degree):
    return [gaussians(rng, per_object, sh_degree) for _ in range(n_objects)]


def config1(seed: int = 0, n_bg: int = 1_000_000, n_objects: int = 4, per_object: int = 20_000,
            n_cams: int = 5, size=VGA) -> Workload:
    """1M SH3 background + 4 x 20k object nodes, 5 ring cameras (r=4, z=1.5)."""
    rng = np.random.default_rng((seed, 1))
    parts = [gaussians(rng, n_bg, 3)] + _env_objects(rng, n_objects, per_object, 3)
    field = concat_fields(parts, 3)
    nodes = [SceneNode("bg", NodeKind.background, RigidTransform(), (0, n_bg))]
    movers = []
    b = n_bg
    for k in range(n_objects):
        nodes.append(SceneNode(f"obj{k}", NodeKind.interactive, RigidTransform(), (b, b + per_object)))
        movers.append(len(nodes) - 1)
        b += per_object
    cams = ring_cameras(n_cams, 4.0, 1.5, size[0], size[1])
    return Workload("cfg1", field, nodes, cams, movers, "1M SH3 + 4x20k objects, 5x640x480")


def config2(seed: int = 0, n_envs: int = 64, n_bg: int = 1_000_000, n_objects: int = 4,
            per_object: int = 20_000, cams_per_env: int = 5, size=VGA, env_offset: int = 0) -> Workload:
    """Shared 1M SH3 background; n_envs x (own 4 x 20k objects, 5 jittered cameras)."""
    rng = np.random.default_rng((seed, 2))
    parts = [gaussians(rng, n_bg, 3)]
    nodes = [SceneNode("bg", NodeKind.background, RigidTransform(), (0, n_bg))]
    movers = []
    cams = []
    b = n_bg
    base = ring_cameras(cams_per_env, 4.0, 1.5, size[0], size[1])
    for e in range(n_envs):
        erng = np.random.default_rng((seed, 2, env_offset + e))
        parts += _env_objects(erng, n_objects, per_object, 3)
        for k in range(n_objects):
            nodes.append(SceneNode(f"env{e}/obj{k}", NodeKind.interactive, RigidTransform(),
                                   (b, b + per_object), env=e))
            movers.append(len(nodes) - 1)
            b += per_object
        for c in base:
            jc = jitter_camera(erng, c)
            jc.env = e
            jc.id = f"env{e}/{c.id}"
            cams.append(jc)
    field = concat_fields(parts, 3)
    return Workload("cfg2", field, nodes, cams, movers,
                    f"shared 1M SH3 bg + {n_envs} envs x 4x20k objects, {n_envs * cams_per_env} cams")


def config3(seed: int = 0, n: int = 3_000_000) -> Workload:
    """3M SH3 room-like scene, log-scale N(-5, 0.7), 2 x 1280x720 cameras."""
    rng = np.random.default_rng((seed, 3))
    means = np.stack([rng.uniform(-5, 5, n), rng.uniform(-5, 5, n), rng.uniform(0, 3, n)], axis=1)
    field = concat_fields([gaussians(rng, n, 3, -5.0, 0.7, means=means)], 3)
    f = focal_for(1280)
    cams = []
    for k, y in enumerate((-6.0, 6.0)):
        c = CameraModel.look_at((0.0, y, 1.5), (0.0, 0.0, 1.5), f, f, 1280, 720)
        c.id = f"cam{k}"
        cams.append(c)
    nodes = [SceneNode("bg", NodeKind.background, RigidTransform(), (0, n))]
    return Workload("cfg3", field, nodes, cams, [], "3M SH3 room, 2x1280x720")


NODE_DTYPE = np.dtype([("begin", "<u8"), ("end", "<u8"), ("q", "<f8", (4,)), ("t", "<f8", (3,)),
                       ("kind", "<i4"), ("env", "<i4")])  # == abi.gsim_node (80 bytes)


@dataclass
class RankEnvs:
    """BASELINE config 4 on one rank: a device-resident scene holding a replica of the shared
    1M SH3 background followed by the rank's environments' 4 x 20k objects each (written
    piecewise, never materialised on the host as a whole), env-tagged nodes and cameras."""
    scene: object
    cameras: list
    cams_per_env: int
    env_begin: int
    env_end: int
    node_table: np.ndarray  # NODE_DTYPE rows: background, then 4 objects per env
    seed: int

    def frame_nodes(self, frame: int):
        """ctypes gsim_node table with fresh random rigid poses (yaw ~ U[0, 2pi) about +z,
        t ~ U[-0.5, 0.5]^3) for every object node (config 1/2/4 motion)."""
        import ctypes as C
        from . import abi
        rng = np.random.default_rng((self.seed, 7919, frame, self.env_begin))
        tab = self.node_table.copy()
        n = len(tab) - 1
        yaw = rng.uniform(0.0, 2.0 * math.pi, size=n)
        tab["q"][1:, 0] = np.cos(0.5 * yaw)
        tab["q"][1:, 3] = np.sin(0.5 * yaw)
        tab["t"][1:] = rng.uniform(-0.5, 0.5, size=(n, 3))
        arr = (abi.gsim_node * len(tab))()
        C.memmove(arr, tab.ctypes.data, tab.nbytes)
        return arr

    def camera_table(self, env_a: int, env_b: int):
        """ctypes gsim_camera table of envs [env_a, env_b) (global env indices)."""
        from . import abi
        cams = self.cameras[(env_a - self.env_begin) * self.cams_per_env:
                            (env_b - self.env_begin) * self.cams_per_env]
        arr = (abi.gsim_camera * len(cams))()
        for k, c in enumerate(cams):
            arr[k] = c.to_c()
        return arr


def config4_rank(ctx, env_begin: int, env_end: int, seed: int = 0, n_bg: int = 1_000_000,
                 n_objects: int = 4, per_object: int = 20_000, cams_per_env: int = 5,
                 size=VGA) -> RankEnvs:
    """Environments [env_begin, env_end) of config 4 on `ctx`'s device. The background and every
    env's objects/cameras come from the same seeded streams as config2 (env e of config 4 equals
    env e of config2(seed, n_envs > e)), so env renders can be checked against config 2."""
    rng = np.random.default_rng((seed, 2))
    n_env = env_end - env_begin
    total = n_bg + n_env * n_objects * per_object
    scene = ctx.create_scene(total, 3)
    scene.write(0, concat_fields([gaussians(rng, n_bg, 3)], 3))
    rows = [(0, n_bg, (1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0), NodeKind.background, -1)]
    cams = []
    base = ring_cameras(cams_per_env, 4.0, 1.5, size[0], size[1])
    b = n_bg
    for e in range(env_begin, env_end):
        erng = np.random.default_rng((seed, 2, e))
        objs = _env_objects(erng, n_objects, per_object, 3)
        scene.write(b, concat_fields(objs, 3))
        for k in range(n_objects):
            rows.append((b, b + per_object, (1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0), NodeKind.interactive, e))
            b += per_object
        for c in base:
            jc = jitter_camera(erng, c)
            jc.env = e
            jc.id = f"env{e}/{c.id}"
            cams.append(jc)
    table = np.array(rows, dtype=NODE_DTYPE)
    return RankEnvs(scene, cams, cams_per_env, env_begin, env_end, table, seed)


CONFIGS = {"cfg0": config0, "cfg1": config1, "cfg2": config2, "cfg3": config3}
