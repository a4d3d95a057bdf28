"""Full-size GPU parity on the BASELINE.json configurations the bench runs.

The reference's own bar is per-scene oracle equivalence (acceptance.cpp:47-82) at the bench
shape (acceptance.cpp:245-291); these tests apply the north-star tolerances at full size:
  * config 1 (1.08M SH3 Gaussians with 4 posed object nodes, 5 x 640x480): every camera, images
    and per-tile index lists, against the oracle; one camera also against the unmodified
    reference (oracle/_ref gsim::render), which pins the C restatement at this scale
    (bit-identical images);
  * config 2 (shared 1M SH3 background + 64 envs x 4 x 20k objects, 320 jittered cameras): the
    whole batch in one render call; 8 sampled cameras across envs (first, last, the 31/32 and
    63/64 boundaries) against the oracle restricted to the camera's env, tile lists of the
    cameras whose lists the library still holds, and one env checked against the reference
    rendering the env's own field (background + its objects) to pin the env semantics;
  * config 3 (3M SH3 room, 2 x 1280x720): one full camera, images and tile lists.
The oracle cameras run in parallel host threads (ctypes releases the GIL).
Image tolerance: RGB max-abs <= 2e-3 and depth within 1e-3 relative (denominator floored at
0.1 m, or 1e-4 m absolute) on >= 99.9% of pixels (tests/helpers.py parity_stats).
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2507_21981_b200.api import GaussianField, RenderTarget, SceneNode
from tests.helpers import parity_stats

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _check(gpu, ref, what):
    st = parity_stats(gpu, ref)
    print(what, {k: (round(v, 6) if isinstance(v, float) else v) for k, v in st.items()})
    assert st["rgb_ok"] >= 0.999, (what, st)
    assert st["depth_ok"] >= 0.999, (what, st)
    return st


def _oracle_camera(oracle, field, nodes, cam):
    splats = oracle.project(field, nodes, cam)
    return splats, oracle.rasterize(splats, cam), oracle.rasterize_lists(splats, cam)


def _lists_equal(ctx, k, splats, lists, visible=None):
    """Tile lists of camera k of the last render equal the oracle's. The library reports record
    slots local to the camera; `visible` maps them to primitive indices when the camera does not
    see every primitive (env-tagged nodes of other envs)."""
    offsets, values = ctx.tile_lists(k)
    tb, vals = lists
    assert np.array_equal(offsets[: len(tb)], tb), k
    prims = values if visible is None else visible[values]
    assert np.array_equal(prims, splats["prim_index"][vals]), k
    return len(values)


def _visible_prims(nodes, cam, n):
    """Primitives a camera sees, in slot order: those of nodes with env -1 or the camera's env
    (plus any primitive no node covers), in primitive order."""
    seen = np.ones(n, bool)
    for nd in nodes:
        if nd.env >= 0 and nd.env != cam.env:
            seen[nd.range[0]: nd.range[1]] = False
    return np.nonzero(seen)[0].astype(np.int64)


def _device_targets(flat, cameras, picks):
    """RenderTargets of the picked cameras from a device output buffer (torch tensor)."""
    offs = np.zeros(len(cameras) + 1, np.int64)
    for k, c in enumerate(cameras):
        offs[k + 1] = offs[k] + 5 * c.width * c.height
    out = {}
    for k in picks:
        c = cameras[k]
        npx = c.width * c.height
        blk = flat[int(offs[k]): int(offs[k + 1])].cpu().numpy()
        out[k] = RenderTarget(blk[: 3 * npx].reshape(c.height, c.width, 3).copy(),
                              blk[3 * npx: 4 * npx].reshape(c.height, c.width).copy(),
                              blk[4 * npx:].reshape(c.height, c.width).copy())
    return out


def test_config1_all_cameras(ctx, oracle):
    from paper_2507_21981_b200.scenes import config1
    w = config1(seed=11)
    nodes = w.frame_nodes(3)
    s = ctx.upload(w.field)
    got = ctx.render(s, nodes, w.cameras)
    assert ctx.stats()["groups"] == 1
    with ThreadPoolExecutor(len(w.cameras)) as ex:
        ref = list(ex.map(lambda c: _oracle_camera(oracle, w.field, nodes, c), w.cameras))
    pairs = 0
    for k, (splats, img, lists) in enumerate(ref):
        _check(got[k], img, f"cfg1 camera {k}")
        pairs += _lists_equal(ctx, k, splats, lists)
    assert pairs == ctx.stats()["pairs"]


def test_config1_camera_against_reference(ctx, oracle, ref):
    """One config-1 camera through the unmodified reference's gsim::render (oracle/_ref): the C
    restatement is bit-identical to it at 1.08M Gaussians, and the GPU is within tolerance."""
    from paper_2507_21981_b200.scenes import config1
    w = config1(seed=12)
    nodes = w.frame_nodes(5)
    cam = w.cameras[1]
    rf = ref.field(w.field)
    try:
        r = rf.render(nodes, [cam])[0]
    finally:
        rf.close()
    o = oracle.render(w.field, nodes, [cam])[0]
    assert np.array_equal(o.rgb, r.rgb) and np.array_equal(o.depth, r.depth)
    assert np.array_equal(o.accum_alpha, r.accum_alpha)
    assert oracle.hash_target(o) == oracle.hash_target(r)
    g = ctx.render(ctx.upload(w.field), nodes, [cam])[0]
    _check(g, r, "cfg1 camera 1 vs reference")


CFG2_PICKS = (0, 31, 32, 63, 64, 161, 288, 319)


def _env_subfield(w, frame_nodes, env):
    """The reference-semantics scene of one env: background + the env's own objects (the frame's
    posed nodes re-indexed into the sub-field); the reference has no env tags."""
    bg = frame_nodes[0]
    objs = [n for n in frame_nodes[1:] if n.env == env]
    idx = [np.arange(bg.range[0], bg.range[1])] + [np.arange(n.range[0], n.range[1]) for n in objs]
    idx = np.concatenate(idx)
    f = w.field
    sub = GaussianField(f.means[idx], f.scales[idx], f.rotations[idx], f.opacities[idx], f.sh[idx],
                        f.sh_degree)
    nodes = [SceneNode(bg.id, bg.kind, bg.pose, bg.range)]
    b = bg.range[1] - bg.range[0]
    for n in objs:
        m = n.range[1] - n.range[0]
        nodes.append(SceneNode(n.id, n.kind, n.pose, (b, b + m)))
        b += m
    return sub, nodes


def test_config2_batch_sampled_cameras(ctx, oracle, ref):
    import torch
    from paper_2507_21981_b200.scenes import config2
    w = config2(seed=21)
    nodes = w.frame_nodes(2)
    s = ctx.upload(w.field)
    total = sum(5 * c.width * c.height for c in w.cameras)
    out = torch.empty(total, dtype=torch.float32, device="cuda:0")
    ctx.render_device(s, nodes, w.cameras, None, out.data_ptr())
    ctx.synchronize()
    st = ctx.stats()
    groups = st["groups"]
    got = _device_targets(out, w.cameras, CFG2_PICKS)
    cams = [w.cameras[k] for k in CFG2_PICKS]
    with ThreadPoolExecutor(len(cams)) as ex:
        res = list(ex.map(lambda c: _oracle_camera(oracle, w.field, nodes, c), cams))
    # tile lists: the library holds the lists of the last camera group it rendered
    first_held = len(w.cameras) - st["last_group_cameras"]
    checked = 0
    for k, (splats, img, lists) in zip(CFG2_PICKS, res):
        _check(got[k], img, f"cfg2 camera {k} (env {w.cameras[k].env})")
        if k >= first_held:
            _lists_equal(ctx, k - first_held, splats, lists,
                         _visible_prims(nodes, w.cameras[k], w.field.size()))
            checked += 1
    assert checked >= 2 if groups > 1 else checked == len(CFG2_PICKS)
    # env semantics pinned on the reference: env 12's camera = the reference rendering the
    # env's own field (background + its 4 objects)
    k = 64
    env = w.cameras[k].env
    sub, sub_nodes = _env_subfield(w, nodes, env)
    rf = ref.field(sub)
    try:
        r = rf.render(sub_nodes, [w.cameras[k]])[0]
    finally:
        rf.close()
    o = res[CFG2_PICKS.index(k)][1]
    assert np.array_equal(o.rgb, r.rgb) and np.array_equal(o.depth, r.depth)
    _check(got[k], r, f"cfg2 camera {k} vs reference env field")


def test_config3_full_camera(ctx, oracle):
    from paper_2507_21981_b200.scenes import config3
    w = config3(seed=31)
    s = ctx.upload(w.field)
    got = ctx.render(s, w.nodes, w.cameras)
    k = 1
    splats, img, lists = _oracle_camera(oracle, w.field, w.nodes, w.cameras[k])
    _check(got[k], img, "cfg3 camera 1 (1280x720, 3M)")
    n = _lists_equal(ctx, k, splats, lists)
    assert n > 5_000_000


def test_config1_options_full_size(ctx, oracle):
    """RasterOptions at full size (raster.hpp:31-36): normalize_depth and a 1e-3 transmittance
    cutoff on a config-1 camera, against the oracle; the tile lists do not depend on them."""
    from paper_2507_21981_b200.api import RasterOptions
    from paper_2507_21981_b200.scenes import config1
    w = config1(seed=13)
    nodes = w.frame_nodes(7)
    cam = w.cameras[3]
    opt = RasterOptions(normalize_depth=True, transmittance_cutoff=1e-3)
    g = ctx.render(ctx.upload(w.field), nodes, [cam], opt)[0]
    splats = oracle.project(w.field, nodes, cam)
    _check(g, oracle.rasterize(splats, cam, opt), "cfg1 camera 3, normalize_depth + cutoff 1e-3")
