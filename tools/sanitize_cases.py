"""compute-sanitizer workloads: small renders that exercise every race-prone
mechanism of the path, run under memcheck / racecheck / synccheck by tools/sanitize.sh.

    python tools/sanitize_cases.py smoke|copies|contexts|batch|determinism

smoke     __graft_entry__.smoke(): K2, key_hist, onesweep look-back, binning, scatter, raster
copies    3-camera render into host targets: one raster launch per camera, each camera's copies
          waiting on its event (host.cu launch_raster_stage / queue_camera_copies),
          then render_encoded (the same handoff for encoded blocks)
contexts  two contexts rendering concurrently from two host threads (shared device, separate
          streams and workspaces)
batch     a 12-camera env batch with a multi-unit scatter per camera (bitmap peers) and a
          1280x720 camera (u8 probe peers), plus a forced pair-buffer overflow re-run
"""
from __future__ import annotations

import os
import sys
import threading
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def scene(orc, seed=7, n=6000, deg=2):
    f = orc.random_field(seed, n, 3.0, 0.01, 0.2, deg)
    f.means[:, 2] += 3.0
    f.touch()
    return f


def cams(k, w=128, h=96):
    from paper_2507_21981_b200.api import CameraModel, RigidTransform, quat_from_axis_angle
    out = []
    for i in range(k):
        c = CameraModel(fx=90.0, fy=90.0, cx=w / 2, cy=h / 2, width=w, height=h)
        c.pose = RigidTransform(quat_from_axis_angle((0, 1, 0), 0.05 * (i - k / 2)), (0.1 * i, 0.0, 0.0))
        out.append(c)
    return out


def main(case: str) -> None:
    from oracle.oracle import Oracle
    from paper_2507_21981_b200 import Context, EncodeOptions
    orc = Oracle()
    from paper_2507_21981_b200 import abi
    print("library:", abi.LIB_PATH.name)
    if case == "smoke":
        import __graft_entry__ as g
        g.smoke()
        return
    if case == "copies":
        ctx = Context(0)
        f = scene(orc)
        s = ctx.upload(f)
        c3 = cams(3)
        a = ctx.render(s, [], c3)
        b = ctx.render(s, [], c3)
        assert all(np.array_equal(x.rgb, y.rgb) for x, y in zip(a, b))
        ctx.render_encoded(s, [], c3, None, EncodeOptions())
        print("copies ok")
        return
    if case == "contexts":
        f = scene(orc)
        ctxs = [Context(0), Context(0)]
        scenes = [c.upload(f) for c in ctxs]
        res = [None, None]

        def run(k):
            for _ in range(3):
                res[k] = ctxs[k].render(scenes[k], [], cams(2))
        th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert all(np.array_equal(x.rgb, y.rgb) for x, y in zip(res[0], res[1]))
        print("contexts ok")
        return
    if case == "batch":
        from paper_2507_21981_b200.api import NodeKind, RigidTransform, SceneNode, quat_from_axis_angle
        f = scene(orc, seed=9, n=30000, deg=1)
        nodes = [SceneNode("bg", NodeKind.background, RigidTransform(), (0, 20000))]
        for e in range(4):
            nodes.append(SceneNode(f"o{e}", NodeKind.interactive,
                                   RigidTransform(quat_from_axis_angle((0, 0, 1), 0.3 * e), (0.1 * e, 0, 0)),
                                   (20000 + 2500 * e, 22500 + 2500 * e), env=e))
        cs = cams(12)
        for i, c in enumerate(cs):
            c.env = i % 4
        big = cams(1, 1280, 720)[0]
        big.env = 0
        ctx = Context(0)
        s = ctx.upload(f)
        ctx.render(s, nodes, cs + [big])
        os.environ["GSIM_GPU_INITIAL_PAIR_CAPACITY"] = "5000"
        small = Context(0)
        ss = small.upload(f)
        small.render(ss, nodes, cs[:3])
        print("batch ok, pairs", small.stats()["pairs"])
        return
    if case == "determinism":
        # races would show as run-to-run differences: 3 contexts x 20 frames of a 1.08M-Gaussian
        # config-1 scene from 3 host threads, every output bit-identical to the first
        from paper_2507_21981_b200.scenes import config1
        w = config1(seed=5)
        nodes = w.frame_nodes(1)
        ctxs = [Context(0) for _ in range(3)]
        scenes = [c.upload(w.field) for c in ctxs]
        want = ctxs[0].render(scenes[0], nodes, w.cameras)
        bad = [0]

        def run(k):
            for _ in range(20):
                got = ctxs[k].render(scenes[k], nodes, w.cameras)
                bad[0] += sum(not (np.array_equal(g.rgb, t.rgb) and np.array_equal(g.depth, t.depth)
                                   and np.array_equal(g.accum_alpha, t.accum_alpha))
                              for g, t in zip(got, want))
        th = [threading.Thread(target=run, args=(k,)) for k in range(3)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        print("determinism: 60 frames x 5 cameras,", bad[0], "differ")
        assert bad[0] == 0
        return
    raise SystemExit(f"unknown case {case}")


if __name__ == "__main__":
    import faulthandler
    # a hang shows where every thread waits (debug_checks.sh kills the case at 900 s)
    faulthandler.dump_traceback_later(840, exit=True)
    main(sys.argv[1])
