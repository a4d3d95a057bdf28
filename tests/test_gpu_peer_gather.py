"""Config 4's fused gather (shard.ChunkGather mode "p2p", gsim_gpu_ipc_*): rank 1 renders its
environments straight into rank 0's output through a CUDA IPC mapping, and rank 0 finds them
equal, bit for bit, to its own renders of the same environments.

Both ranks share the one GPU of a gpurun box (same-device IPC); their kernels never wait on each
other (host barriers only), so this checks the plumbing and the data path, not NVLink timing."""
from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2507_21981_b200 import Context
    from paper_2507_21981_b200.scenes import config4_rank
    from paper_2507_21981_b200.shard import ChunkGather, env_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n_envs, small = 6, dict(n_bg=20_000, per_object=3_000, size=(160, 120))
    b, e = env_range(n_envs, rank, world)
    ctx = Context(0)
    r = config4_rank(ctx, b, e, seed=7, **small)
    cpe = r.cams_per_env
    fpe = 5 * sum(c.width * c.height for c in r.cameras[:cpe])
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    g = ChunkGather(n_envs, fpe, 2, dev, rank=rank, world=world, dst=0, mode="p2p")
    nodes = r.frame_nodes(3)
    with torch.cuda.stream(stream):
        for j, (cb, ce) in enumerate(g.my_chunks):
            buf = g.target(j)
            ctx.render_device(r.scene, nodes, r.camera_table(cb, ce), None, buf.data_ptr())
            g.send(j)
        g.finish()
    ok = True
    if rank == 0:
        # rank 0 renders every other rank's environments itself and compares
        for src in range(1, world):
            sb, se = env_range(n_envs, src, world)
            other = config4_rank(ctx, sb, se, seed=7, **small)
            want = torch.empty((se - sb) * fpe, dtype=torch.float32, device=dev)
            ctx.render_device(other.scene, _same_poses(other, 3),
                              other.camera_table(sb, se), None, want.data_ptr())
            ctx.synchronize()
            got = g.out[sb * fpe: se * fpe]
            ok = ok and bool(torch.equal(got, want)) and float(want.abs().sum()) > 0
    dist.barrier()
    if g.peer:
        g.peer.close()
    q.put((rank, ok))
    dist.destroy_process_group()


def _same_poses(r, frame):
    # frame_nodes seeds its poses by (seed, frame, env_begin): the table a rank used for its own
    # environments is reproduced by a RankEnvs built for the same environment range
    return r.frame_nodes(frame)


def _compute_mode() -> str:
    import subprocess
    try:
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=compute_mode", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=30).stdout.strip()
    except Exception:
        out = ""
    return out


def test_fused_peer_gather_two_ranks_one_gpu():
    if "Exclusive" in _compute_mode():
        pytest.skip("GPU in an exclusive compute mode: two processes cannot share it")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res
