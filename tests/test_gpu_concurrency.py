"""Concurrent renderer contexts (how bench.py and a multi-threaded caller drive the library).

Every context owns its stream, workspaces, onesweep status words and tickets; frames of different
contexts overlap on the GPU. The bar is bit-identity: a frame rendered while other contexts run
must equal the same frame rendered alone (raster.hpp:62-63 makes the reference's render a pure,
thread-count independent function, and so is ours).
"""
from __future__ import annotations

import threading

import numpy as np
import pytest

from paper_2507_21981_b200 import Context
from paper_2507_21981_b200.api import NodeKind, RigidTransform, SceneNode, quat_from_axis_angle
from tests.helpers import ref_camera

pytestmark = pytest.mark.gpu


def scene_and_frames(oracle, n_frames):
    field = oracle.random_field(4242, 20000, 3.0, 0.005, 0.08, 2)
    field.means[:, 2] += 3.0
    n = field.size()
    cams = []
    for k in range(3):
        c = ref_camera(160, 120, 140.0)
        c.pose = RigidTransform(quat_from_axis_angle((0, 1, 0), 0.07 * (k - 1)), (0.15 * (k - 1), 0.0, 0.0))
        cams.append(c)
    frames = []
    for i in range(n_frames):
        q = quat_from_axis_angle((0, 0, 1), 0.37 * i)
        frames.append([SceneNode("bg", NodeKind.background, RigidTransform(), (0, n - 3001)),
                       SceneNode("obj", NodeKind.interactive, RigidTransform(q, (0.05 * i, 0.0, 0.1)),
                                 (n - 3001, n))])
    return field, cams, frames


def same(a, b):
    return (np.array_equal(a.rgb, b.rgb) and np.array_equal(a.depth, b.depth)
            and np.array_equal(a.accum_alpha, b.accum_alpha))


def test_threaded_contexts_equal_sequential(oracle):
    field, cams, frames = scene_and_frames(oracle, 8)
    solo = Context(0)
    s0 = solo.upload(field)
    want = [solo.render(s0, nodes, cams) for nodes in frames]
    assert any(t.accum_alpha.max() > 0.5 for t in want[0])

    ctxs = [Context(0) for _ in range(4)]
    scenes = [c.upload(field) for c in ctxs]
    got = {}
    errors = []

    def worker(k):
        try:
            for rep in range(2):
                for i in range(k, len(frames), len(ctxs)):
                    got[(i, rep)] = ctxs[k].render(scenes[k], frames[i], cams)
        except Exception as e:  # noqa: BLE001 (reported below)
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(ctxs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for (i, rep), out in got.items():
        for c in range(len(cams)):
            assert same(out[c], want[i][c]), (i, rep, c)


def test_interleaved_device_frames_equal_sequential(oracle):
    import torch
    field, cams, frames = scene_and_frames(oracle, 6)
    ctxs = [Context(0) for _ in range(3)]
    scenes = [c.upload(field) for c in ctxs]
    floats = sum(5 * c.width * c.height for c in cams)
    outs = [torch.empty(floats, dtype=torch.float32, device="cuda:0") for _ in frames]
    # every context enqueues its frames without waiting; frames of different contexts overlap
    for i, nodes in enumerate(frames):
        ctxs[i % 3].render_device(scenes[i % 3], nodes, cams, None, outs[i].data_ptr())
    for c in ctxs:
        c.synchronize()
    solo = Context(0)
    s0 = solo.upload(field)
    for i, nodes in enumerate(frames):
        want = solo.render(s0, nodes, cams)
        flat = np.concatenate([np.concatenate([t.rgb.reshape(-1), t.depth.reshape(-1),
                                               t.accum_alpha.reshape(-1)]) for t in want])
        assert np.array_equal(outs[i].cpu().numpy(), flat), i


def test_overlapped_copies_equal_frame_copies(oracle, monkeypatch):
    """render() copies camera c while later cameras are composited (one raster launch per camera,
    the copy stream waits on its event); GSIM_GPU_OVERLAP_COPIES=0 copies after the frame. Same bytes, including
    multi-group batches (40 cameras -> several camera groups) and back-to-back frames."""
    field, cams, frames = scene_and_frames(oracle, 3)
    many = []
    for k in range(40):
        c = ref_camera(64, 48, 60.0)
        c.pose = RigidTransform(quat_from_axis_angle((0, 1, 0), 0.01 * k), (0.02 * k, 0.0, 0.0))
        many.append(c)
    # a small slot budget per camera group: the 40-camera batch runs as several groups
    monkeypatch.setenv("GSIM_GPU_GROUP_SLOTS", str(16 * field.size()))
    monkeypatch.setenv("GSIM_GPU_OVERLAP_COPIES", "0")
    plain = Context(0)
    monkeypatch.delenv("GSIM_GPU_OVERLAP_COPIES")
    fast = Context(0)
    sp, sf = plain.upload(field), fast.upload(field)
    from paper_2507_21981_b200 import EncodeOptions
    eo = EncodeOptions()
    for nodes in frames:
        for batch in (cams, many):
            want = plain.render(sp, nodes, batch)
            got = fast.render(sf, nodes, batch)
            assert all(same(a, b) for a, b in zip(got, want))
            # render_encoded's per-camera copies (the same counters) give the same bytes
            assert np.array_equal(fast.render_encoded(sf, nodes, batch, None, eo),
                                  plain.render_encoded(sp, nodes, batch, None, eo))
    assert fast.stats()["groups"] == 3


def test_pinned_and_pageable_targets_agree(oracle):
    """render() into page-locked targets (copies run asynchronously behind the compositing)
    and into ordinary numpy arrays (each copy blocks the caller) gives the same bytes."""
    import torch
    from paper_2507_21981_b200 import RenderTarget
    field, cams, frames = scene_and_frames(oracle, 2)
    ctx = Context(0)
    s = ctx.upload(field)
    pinned = [RenderTarget(torch.empty((c.height, c.width, 3), pin_memory=True).numpy(),
                           torch.empty((c.height, c.width), pin_memory=True).numpy(),
                           torch.empty((c.height, c.width), pin_memory=True).numpy()) for c in cams]
    for nodes in frames:
        want = ctx.render(s, nodes, cams)
        got = ctx.render(s, nodes, cams, None, pinned)
        assert all(same(a, b) for a, b in zip(got, want))


def test_overlapped_copies_never_stale(oracle):
    """The per-camera copies start on the event after the camera's raster launch. Stress that
    handoff (and, before it used events, a stream-wait-value handoff hung here about once in ten
    longer runs): 4 contexts on 4
    threads render 24 frames each into page-locked targets reused frame after frame, so a copy
    that overtook a tile's pixel stores would leave the previous frame's pixels in the target.
    Every frame must equal the same frame rendered alone."""
    import torch
    from paper_2507_21981_b200 import RenderTarget
    field, cams, frames = scene_and_frames(oracle, 12)
    solo = Context(0)
    s0 = solo.upload(field)
    want = [solo.render(s0, nodes, cams) for nodes in frames]

    def pinned():
        return [RenderTarget(torch.empty((c.height, c.width, 3), pin_memory=True).numpy(),
                             torch.empty((c.height, c.width), pin_memory=True).numpy(),
                             torch.empty((c.height, c.width), pin_memory=True).numpy()) for c in cams]
    ctxs = [Context(0) for _ in range(4)]
    scenes = [c.upload(field) for c in ctxs]
    bad, errors = [], []

    def worker(k):
        try:
            tg = pinned()
            for rep in range(24):
                i = (k + 5 * rep) % len(frames)
                out = ctxs[k].render(scenes[k], frames[i], cams, None, tg)
                if not all(same(a, b) for a, b in zip(out, want[i])):
                    bad.append((k, rep, i))
        except Exception as e:  # noqa: BLE001 (reported below)
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(ctxs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert not bad, bad


def test_threaded_encoded_renders_equal_single(oracle):
    """render_encoded from 3 contexts on 3 host threads (each camera's encoded block copied on
    the event after its raster launch, into pinned and into pageable blobs) gives the bytes of the
    same frames encoded by one context alone."""
    import torch
    from paper_2507_21981_b200 import EncodeOptions
    field, cams, frames = scene_and_frames(oracle, 6)
    eo = EncodeOptions()
    solo = Context(0)
    s0 = solo.upload(field)
    want = [solo.render_encoded(s0, nodes, cams, None, eo) for nodes in frames]
    ctxs = [Context(0) for _ in range(3)]
    scenes = [c.upload(field) for c in ctxs]
    nbytes = want[0].size
    bad, errors = [], []

    def worker(k):
        try:
            blob = (torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy() if k % 2 == 0
                    else np.empty(nbytes, dtype=np.uint8))
            for rep in range(8):
                i = (k + rep) % len(frames)
                got = ctxs[k].render_encoded(scenes[k], frames[i], cams, None, eo, out=blob)
                if not np.array_equal(got, want[i]):
                    bad.append((k, rep, i))
        except Exception as e:  # noqa: BLE001 (reported below)
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(3)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert not bad, bad
