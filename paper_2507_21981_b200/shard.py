"""Multi-GPU plumbing: environment sharding and the frame gather of BASELINE config 4.

Every (environment, camera) render is independent given the replicated background, so the
render path shards by environment with no data-path collective. The only real
exchange is config 4's gather of finished frames to rank 0, done here with torch.distributed
point-to-point (NCCL over NVLink on the GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def env_range(n_envs: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced split of n_envs environments over world ranks: [begin, end)."""
    base, extra = divmod(n_envs, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def env_chunks(begin: int, end: int, chunk: int = 64):
    """Launch-sized chunks (config 2 size) of a rank's environments."""
    for b in range(begin, end, chunk):
        yield b, min(end, b + chunk)


def gather_frames(frames: torch.Tensor, n_envs: int, floats_per_env: int, dst: int = 0):
    """Gather every rank's frames (its env_range, env-major, floats_per_env floats each) to
    rank `dst`, which returns the full [n_envs * floats_per_env] tensor in environment order;
    other ranks return None. Grouped point-to-point sends, one per rank (NCCL has no gather)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    if rank != dst:
        dist.send(frames.contiguous(), dst=dst)
        return None
    out = torch.empty(n_envs * floats_per_env, dtype=frames.dtype, device=frames.device)
    reqs = []
    for r in range(world):
        b, e = env_range(n_envs, r, world)
        view = out[b * floats_per_env: e * floats_per_env]
        if r == dst:
            view.copy_(frames)
        elif e > b:
            reqs.append(dist.irecv(view, src=r))
    for q in reqs:
        q.wait()
    return out


class _CudaArray:
    """A raw device range seen through __cuda_array_interface__ (torch.as_tensor views it)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, n_floats: int, device) -> torch.Tensor:
    return torch.as_tensor(_CudaArray(ptr, n_floats), device=device)


class PeerBuffer:
    """Rank `dst`'s gathered output in peer memory (gsim_gpu_ipc_*): dst allocates and exports it,
    every other rank of the node opens it, so their renders can store straight into it."""

    def __init__(self, n_floats: int, device, rank: int, world: int, dst: int = 0):
        import ctypes as C
        from . import abi
        self.lib = abi.load_library()
        self.dev_index = device.index if isinstance(device, torch.device) else int(device)
        self.owner = rank == dst
        ptr = C.c_void_p()
        handle = (C.c_uint8 * 64)()
        ok = True
        if self.owner:
            ok = self.lib.gsim_gpu_ipc_alloc(self.dev_index, 4 * n_floats, C.byref(ptr), handle) == abi.GSIM_OK
        # the owner always takes part in the broadcast (None on failure), so no rank waits forever
        msg = [bytes(handle) if (self.owner and ok) else None]
        if world > 1:
            dist.broadcast_object_list(msg, src=dst)
        self.ptr, self.n = 0, n_floats
        if msg[0] is None:
            raise RuntimeError("gsim_gpu_ipc_alloc failed on the gathering rank")
        if not self.owner:
            h = (C.c_uint8 * 64).from_buffer_copy(msg[0])
            st = self.lib.gsim_gpu_ipc_open(self.dev_index, h, C.byref(ptr))
            if st != abi.GSIM_OK:
                raise RuntimeError("gsim_gpu_ipc_open failed (peer access between the ranks' GPUs?)")
        self.ptr = int(ptr.value)
        self.n = n_floats

    def view(self, first: int, count: int, device) -> torch.Tensor:
        return device_view(self.ptr + 4 * first, count, device)

    def close(self) -> None:
        if self.ptr:
            if self.owner:
                self.lib.gsim_gpu_ipc_free(self.dev_index, self.ptr)
            else:
                self.lib.gsim_gpu_ipc_close(self.dev_index, self.ptr)
            self.ptr = 0


class ChunkTarget:
    """A chunk's render destination: device pointer + local tensor view (None for peer memory)."""

    def __init__(self, ptr: int, local: torch.Tensor | None):
        self.ptr, self.local = int(ptr), local

    def data_ptr(self) -> int:
        return self.ptr


class ChunkGather:
    """BASELINE config 4's frame gather, overlapped with rendering.

    Every rank renders its env_range in chunks of <= chunk_envs environments (config-2-sized
    launches); round j moves every rank's chunk j to rank `dst` with one grouped point-to-point
    exchange (dist.batch_isend_irecv: NCCL over NVLink on the GPU box, gloo on CPU) while chunk
    j+1 renders. Issue send(j) on the stream that rendered chunk j (NCCL orders its transfer
    after that stream's work) and call target(j) on it before rendering: a send buffer is reused
    only after its previous transfer completed (double buffering). Rank `dst` renders straight
    into its slices of `out` ([n_envs * floats_per_env], environment order) and receives the
    others' chunks into theirs.
    """

    def __init__(self, n_envs: int, floats_per_env: int, chunk_envs: int, device, rank: int | None = None,
                 world: int | None = None, dst: int = 0, n_buffers: int = 2, dtype=torch.float32,
                 mode: str = "nccl"):
        initialized = dist.is_available() and dist.is_initialized()
        self.rank = rank if rank is not None else (dist.get_rank() if initialized else 0)
        self.world = world if world is not None else (dist.get_world_size() if initialized else 1)
        self.n_envs, self.fpe, self.dst = n_envs, floats_per_env, dst
        self.ranges = [env_range(n_envs, r, self.world) for r in range(self.world)]
        self.chunks = [list(env_chunks(b, e, chunk_envs)) for b, e in self.ranges]
        self.my_chunks = self.chunks[self.rank]
        self.rounds = max(len(c) for c in self.chunks)
        self.out = None
        self.bufs = []
        self.mode = mode if self.world > 1 else "local"
        self.device = device
        self.peer = None
        self.fallback = None
        if self.mode == "p2p":
            # fused gather: every rank's compositing kernel stores into dst's HBM over NVLink.
            # Every rank must be able to map dst's buffer, else all fall back to NCCL together.
            err = None
            try:
                self.peer = PeerBuffer(n_envs * floats_per_env, device, self.rank, self.world, dst)
            except RuntimeError as e:
                err = e
            ok = torch.tensor([0 if err else 1], dtype=torch.int32,
                              device=device if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 1:
                if self.rank == dst:
                    self.out = self.peer.view(0, n_envs * floats_per_env, device)
            else:
                if self.peer is not None:
                    self.peer.close()
                    self.peer = None
                self.mode = "nccl"
                self.fallback = f"p2p unavailable ({err or 'on another rank'}), NCCL used"
        if self.mode == "p2p":
            pass
        elif self.rank == dst:
            self.out = torch.empty(n_envs * floats_per_env, dtype=dtype, device=device)
        else:
            self.bufs = [torch.empty(chunk_envs * floats_per_env, dtype=dtype, device=device)
                         for _ in range(n_buffers)]
        self.pending = [[] for _ in range(max(n_buffers, 1))]
        self.recv_pending = []
        # floats rank dst receives per step
        self.bytes_to_dst = sum((e - b) * floats_per_env for r, (b, e) in enumerate(self.ranges) if r != dst)
        if self.world > 1:
            dist.barrier()  # the communicator exists before the first point-to-point batch

    def _view(self, b: int, e: int):
        return self.out[b * self.fpe: e * self.fpe]

    def target(self, j: int) -> "ChunkTarget":
        """Where this rank renders its chunk j (waits for the buffer's previous transfer): the
        device pointer to pass as the render's output, and a local tensor view of it, or None
        when the memory is another GPU's (p2p on ranks other than dst: no tensor is made over
        peer memory, which torch would attribute to the owner's device)."""
        b, e = self.my_chunks[j]
        if self.rank == self.dst:
            v = self._view(b, e)
            return ChunkTarget(v.data_ptr(), v)
        if self.mode == "p2p":
            return ChunkTarget(self.peer.ptr + 4 * b * self.fpe, None)
        slot = j % len(self.bufs)
        for w in self.pending[slot]:
            w.wait()
        self.pending[slot] = []
        v = self.bufs[slot][: (e - b) * self.fpe]
        return ChunkTarget(v.data_ptr(), v)

    def send(self, j: int) -> None:
        """Round j: this rank's chunk j to dst, and at dst every other rank's chunk j."""
        if self.world == 1 or self.mode == "p2p":
            return  # p2p: the render already stored the chunk in dst's memory
        ops = []
        if self.rank == self.dst:
            for r in range(self.world):
                if r != self.dst and j < len(self.chunks[r]):
                    b, e = self.chunks[r][j]
                    ops.append(dist.P2POp(dist.irecv, self._view(b, e), r))
        elif j < len(self.my_chunks):
            b, e = self.my_chunks[j]
            slot = j % len(self.bufs)
            ops.append(dist.P2POp(dist.isend, self.bufs[slot][: (e - b) * self.fpe], self.dst))
        if not ops:
            return
        works = dist.batch_isend_irecv(ops)
        if self.rank == self.dst:
            self.recv_pending.extend(works)
        else:
            self.pending[j % len(self.bufs)].extend(works)

    def finish(self) -> None:
        """Every transfer of the step is ordered before the current stream's next work (NCCL)
        or complete (gloo); on dst, `out` then holds every environment's frames. p2p: every
        rank's renders are complete (stream synchronised) before the barrier releases dst."""
        if self.mode == "p2p":
            torch.cuda.current_stream().synchronize()
            dist.barrier()
            return
        for works in self.pending:
            for w in works:
                w.wait()
        self.pending = [[] for _ in self.pending]
        for w in self.recv_pending:
            w.wait()
        self.recv_pending = []


def max_over_ranks(value: float, device) -> float:
    """Max of a per-rank scalar (device time) over all ranks."""
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
