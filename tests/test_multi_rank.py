"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 plumbing: environment sharding
covers every environment exactly once, the config-4 frame gather reassembles rank 0's full batch
in environment order, and the max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2507_21981_b200.shard import env_chunks, env_range


def test_env_range_partitions_exactly():
    for n in (1, 5, 64, 512, 513):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                b, e = env_range(n, r, world)
                assert 0 <= b <= e <= n
                seen.extend(range(b, e))
            assert seen == list(range(n))
            sizes = [env_range(n, r, world)[1] - env_range(n, r, world)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_env_chunks_cover_range():
    chunks = list(env_chunks(10, 200, 64))
    assert chunks[0] == (10, 74) and chunks[-1][1] == 200
    assert sum(e - b for b, e in chunks) == 190


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_envs, per_env, q):
    import torch.distributed as dist

    from paper_2507_21981_b200.shard import env_range, gather_frames, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = env_range(n_envs, rank, world)
    # rank-local "frames": value = env * 1000 + pixel index, env-major
    local = torch.cat([torch.arange(per_env, dtype=torch.float32) + env * 1000 for env in range(b, e)])
    full = gather_frames(local, n_envs, per_env, dst=0)
    t = max_over_ranks(float(rank + 1) * 1.5, torch.device("cpu"))
    if rank == 0:
        want = torch.cat([torch.arange(per_env, dtype=torch.float32) + env * 1000 for env in range(n_envs)])
        q.put((bool(torch.equal(full, want)), t))
    else:
        q.put((full is None, t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_envs", [7, 8])
def test_gather_frames_gloo_world2(n_envs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_envs, 12, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for ok, _ in results)
    assert all(t == 3.0 for _, t in results)  # max over ranks of (rank + 1) * 1.5


def _chunk_worker(rank, world, port, n_envs, per_env, chunk, steps, q):
    import torch.distributed as dist

    from paper_2507_21981_b200.shard import ChunkGather, env_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = ChunkGather(n_envs, per_env, chunk, torch.device("cpu"), dst=0)
    b, e = env_range(n_envs, rank, world)
    ok = True
    for step in range(steps):  # the bench's schedule: render chunk j, send j, next chunk
        for j, (cb, ce) in enumerate(g.my_chunks):
            buf = g.target(j).local
            buf.copy_(torch.cat([torch.arange(per_env, dtype=torch.float32) + env * 1000 + step * 1e6
                                 for env in range(cb, ce)]))
            g.send(j)
        g.finish()
        if rank == 0:
            want = torch.cat([torch.arange(per_env, dtype=torch.float32) + env * 1000 + step * 1e6
                              for env in range(n_envs)])
            ok = ok and bool(torch.equal(g.out, want))
    q.put((rank, ok, g.rounds, (b, e)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_envs,chunk", [(12, 2), (7, 2), (9, 4)])
def test_chunk_gather_schedule_gloo_world2(n_envs, chunk):
    """Config 4's schedule (shard.ChunkGather: chunks of <= chunk envs per rank, round j's grouped
    point-to-point batch, double-buffered sends reused across rounds and steps): rank 0 ends every
    step with every environment's frames in environment order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, 2, port, n_envs, 5, chunk, 3, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert results[0][1], results
    assert results[0][2] == -(-((n_envs + 1) // 2) // chunk)
