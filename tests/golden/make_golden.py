"""Generate tests/golden/golden.json from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
The reference has no golden files of its own: its tests synthesise scenes with
oracle::random_field (tests/support/test_oracles.cpp:144-168). These fixtures record what the
reference itself outputs on such scenes — FNV-1a hashes (hash.hpp:16-44) of project(),
rasterize(), reference_rasterize() and render() results, the sorted pair lists, and
transform_primitives() — so the C restatement can be pinned on a box without the reference.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Oracle, Ref  # noqa: E402
from paper_2507_21981_b200.api import (CameraModel, NodeKind, RasterOptions,  # noqa: E402
                                       RigidTransform, SceneNode, quat_normalized)

OUT = Path(__file__).resolve().parent / "golden.json"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def test_camera(w=128, h=128, f=100.0) -> CameraModel:  # test_raster.cpp:18-28
    return CameraModel(fx=f, fy=f, cx=w * 0.5, cy=h * 0.5, width=w, height=h)


def camera_table(cams) -> np.ndarray:
    """fx, fy, cx, cy, width, height, pose (q, t), near, far of C cameras, one row each."""
    return np.array([[c.fx, c.fy, c.cx, c.cy, c.width, c.height, *c.pose.rotation,
                      *c.pose.translation, c.near_plane, c.far_plane] for c in cams])


def cases():
    """Scene cases: acceptance.cpp:47-82 style, test_raster.cpp:142-157 style, nodes."""
    out = []
    rng = np.random.Generator(np.random.PCG64(2024))
    for scene in range(12):  # acceptance raster_oracle_equivalence family (subset)
        count = int(50 + rng.integers(0, 1951))
        deg = int(rng.integers(0, 4))
        out.append(dict(name=f"accept{scene}", seed=9000 + scene, count=count, box=3.0, slo=0.01,
                        shi=0.05 + (scene % 5) * 0.06, deg=deg, dz=3.2, cam=[100.0, 128, 128],
                        nodes="none"))
    for rnd in range(0, 25, 6):  # test_raster tiled == brute family
        out.append(dict(name=f"tiled{rnd}", seed=1000 + rnd, count=100 + rnd * 17, box=3.0, slo=0.01,
                        shi=0.25, deg=3, dz=3.0, cam=[100.0, 128, 128], nodes="none"))
    out.append(dict(name="nodes", seed=4242, count=3000, box=3.0, slo=0.01, shi=0.1, deg=2, dz=3.0,
                    cam=[120.0, 160, 96], nodes="two"))
    return out


def make_nodes(kind, n):
    if kind == "none":
        return []
    q = quat_normalized((0.9, 0.1, 0.3, 0.2))
    return [SceneNode("bg", NodeKind.background, RigidTransform(), (0, n // 2)),
            SceneNode("obj", NodeKind.interactive, RigidTransform(q, (0.1, -0.2, 0.3)), (n // 2, n))]


def main() -> None:
    ref = Ref()
    orc = Oracle()
    data = {"generator": "tests/golden/make_golden.py (reference compiled from /root/reference)",
            "cases": []}
    for c in cases():
        field = ref.random_field(c["seed"], c["count"], c["box"], c["slo"], c["shi"], c["deg"])
        field.means[:, 2] += c["dz"]
        f, w, h = c["cam"]
        cam = test_camera(w, h, f)
        nodes = make_nodes(c["nodes"], c["count"])
        splats = ref.project(field, nodes, cam)
        tiled = ref.rasterize(splats, cam)
        brute = ref.reference_rasterize(splats, cam)
        norm = ref.rasterize(splats, cam, RasterOptions(normalize_depth=True, transmittance_cutoff=1e-3))
        # the pair lists come from our restatement; their hash is checked against the reference
        # indirectly through the images, and directly against the GPU in tests/test_gpu_*.
        tb, vals = orc.rasterize_lists(splats, cam)
        entry = dict(c)
        entry.update(
            field_sha=sha(np.concatenate([field.means.ravel(), field.scales.ravel(), field.rotations.ravel(),
                                          field.opacities, field.sh.ravel()])),
            n_splats=int(len(splats)),
            splats_sha=sha(splats),
            tiled_hash=str(orc.hash_target(tiled)),
            brute_hash=str(orc.hash_target(brute)),
            norm_hash=str(orc.hash_target(norm)),
            n_pairs=int(len(vals)),
            pairs_sha=sha(np.concatenate([tb, vals])),
        )
        data["cases"].append(entry)
        print(entry["name"], entry["n_splats"], entry["n_pairs"])
    # render() through the reference on a two-camera batch
    field = ref.random_field(31337, 2000, 3.0, 0.01, 0.2, 3)
    field.means[:, 2] += 3.0
    cams = [test_camera(96, 80, 90.0), test_camera(96, 80, 90.0)]
    cams[1].pose = RigidTransform(quat_normalized((0.99, 0.05, -0.05, 0.02)), (0.2, 0.0, 0.1))
    targets = ref.render(field, make_nodes("two", 2000), cams)
    data["render"] = dict(seed=31337, count=2000, hashes=[str(orc.hash_target(t)) for t in targets])
    # transform_primitives (test_core_types.cpp family)
    f2 = ref.random_field(12, 50, 2.0, 0.01, 0.3, 1)
    m, q = f2.means.copy(), f2.rotations.copy()
    rt = RigidTransform(quat_normalized((0.3, 0.5, -0.2, 0.7)), (0.5, -1.25, 2.0))
    ref.transform_primitives(m, q, 5, 45, rt)
    data["transform"] = dict(seed=12, count=50, begin=5, end=45, means_sha=sha(m), rot_sha=sha(q))
    # look_at (raster.cpp:25-42) for the BASELINE config-0 camera
    cam = ref.look_at((5.0, 0.0, 0.0), (0.0, 0.0, 0.0), 554.2562584220407, 554.2562584220407, 640, 480)
    data["look_at"] = dict(rotation=list(cam.pose.rotation), translation=list(cam.pose.translation))
    # GS -> TSDF (transfer.cpp:81-198): render_depth_ring and gaussians_to_mesh's fused volume
    t = dict(seed=4040, count=600, box=1.5, slo=0.02, shi=0.1, deg=2, n_views=8, radius=6.0,
             resolution=48, voxel_size=0.1)
    f3 = ref.random_field(t["seed"], t["count"], t["box"], t["slo"], t["shi"], t["deg"])
    cams, depth = ref.render_depth_ring(f3, t["n_views"], t["radius"], t["resolution"])
    vol = ref.gaussians_to_tsdf(f3, t["voxel_size"])
    t.update(ring_cams_sha=sha(camera_table(cams)), ring_depth_sha=sha(depth),
             valid_fraction=float((depth > 0).mean()), dims=list(vol.dims),
             origin=list(vol.origin), truncation=vol.truncation, tsdf_sha=sha(vol.tsdf),
             weights_sha=sha(vol.weights), observed_fraction=float((vol.weights > 0).mean()))
    data["transfer"] = t
    # LiDAR (trace.cpp): GaussianBvh::build(field, nodes).scan(lidar)
    from paper_2507_21981_b200.api import LidarModel
    f4 = ref.random_field(5150, 1500, 2.0, 0.02, 0.15, 0)
    lid = LidarModel(np.radians(np.linspace(-15.0, 15.0, 8)), np.radians(3.0), 6.0,
                     RigidTransform(quat_normalized((0.99, 0.1, 0.0, 0.05)), (0.1, -0.2, 0.05)))
    scan = ref.lidar_scan(f4, make_nodes("two", 1500), lid)
    data["lidar"] = dict(seed=5150, count=1500, box=2.0, slo=0.02, shi=0.15, deg=0,
                         channels_deg=[float(x) for x in np.linspace(-15.0, 15.0, 8)],
                         azimuth_step_deg=3.0, max_range=6.0,
                         pose_q=[0.99, 0.1, 0.0, 0.05], pose_t=[0.1, -0.2, 0.05],
                         returns=int(len(scan["ring"])), points_sha=sha(scan["points"]),
                         ring_sha=sha(scan["ring"]), azimuth_sha=sha(scan["azimuth"]))
    OUT.write_text(json.dumps(data, indent=1) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
