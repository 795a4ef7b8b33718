"""Cells partitioned over ranks, one min-delay epoch at a time.

The reference runs its epoch loop (engine.cpp:913-942) with worker threads
sharing one process; here every rank (one process per GPU) owns a contiguous
gid range of cells with their incoming synapses (partition(): balanced by
compartments + synapse instances, mcg_build.cpp) and the ranks exchange each
epoch's spikes with one allgather of fixed-size blocks
  [count, (gid, step, t_bits) x block_cap]          (include/mcg.h)
before the next epoch expands them through each rank's local incoming edges.
Delivery order is fixed by the event keys (step, edge rank), so results do not
depend on the number of ranks.  Every rank can rebuild the reference's global
spike list (epoch by epoch, sorted by gid then step) from the gathered blocks.

The exchange is torch.distributed.all_gather_into_tensor: NCCL over NVLink
between GPUs, gloo on CPU tensors in the multi-process tests.
"""
import math
from typing import Callable, List, Optional, Tuple

import numpy as np

ENTRY = 3  # int64 per spike: gid, step, t (IEEE bits)


def block_len(block_cap: int) -> int:
    return 1 + ENTRY * int(block_cap)


def ceil_steps(t_ms: float, dt_ms: float) -> int:
    """engine.cpp:21-23"""
    return int(math.ceil(t_ms / dt_ms - 1e-9))


def partition(recipe, world: int) -> np.ndarray:
    """Shard bounds (world + 1 gids) the engine uses (mcg_partition)."""
    import ctypes as C
    from . import _abi as A
    from .engine import _check
    from .recipe import FlatRecipe, Recipe
    flat = recipe.flatten() if isinstance(recipe, Recipe) else recipe
    view = flat.view if isinstance(flat, FlatRecipe) else flat
    b = np.zeros(world + 1, np.uint32)
    _check(A.lib().mcg_partition(C.byref(view), int(world), b.ctypes.data_as(C.c_void_p)))
    return b


def pack_block(gid, step, t, block_cap: int) -> np.ndarray:
    """One rank's send block (host-side twin of the kernel's export)."""
    gid = np.asarray(gid, np.int64)
    n = len(gid)
    if n > block_cap:
        raise ValueError("spike block overflow")
    b = np.zeros(block_len(block_cap), np.int64)
    b[0] = n
    e = b[1:1 + ENTRY * n].reshape(n, ENTRY)
    e[:, 0] = gid
    e[:, 1] = np.asarray(step, np.int64)
    e[:, 2] = np.asarray(t, np.float64).view(np.int64)
    return b


def unpack_epoch(recv: np.ndarray, world: int, block_cap: int) -> Tuple[np.ndarray, np.ndarray]:
    """All ranks' spikes of one epoch in the reference's order: by gid, then
    detection step (Impl::exchange appends per cell in gid order, engine.cpp:877-888).
    Returns (t_ms, gid)."""
    bl = block_len(block_cap)
    gids, steps, ts = [], [], []
    for r in range(world):
        b = recv[r * bl:(r + 1) * bl]
        n = int(b[0])
        e = b[1:1 + ENTRY * n].reshape(n, ENTRY)
        gids.append(e[:, 0])
        steps.append(e[:, 1])
        ts.append(e[:, 2].view(np.float64))
    g = np.concatenate(gids) if gids else np.zeros(0, np.int64)
    s = np.concatenate(steps) if steps else np.zeros(0, np.int64)
    t = np.concatenate(ts) if ts else np.zeros(0, np.float64)
    o = np.lexsort((s, g))
    return t[o].copy(), g[o].astype(np.uint32)


class SpikeExchange:
    """Send/receive blocks + the allgather.

    The engine reads and writes the blocks on the device (`send`, `recv` are
    CUDA tensors for a GPU engine).  backend "nccl": allgather directly
    between the device buffers (NVLink).  backend "gloo": through host copies
    (multi-process CPU tests; several ranks sharing one GPU).  With
    device="cpu" the blocks themselves live on the host (no engine; tests of
    the exchange alone).  block_cap is agreed across ranks (all_reduce MAX)."""

    def __init__(self, local_cap: int, device: str = "cuda", group=None, backend: str = None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.backend = backend or dist.get_backend(group)
        staged = device != "cpu" and self.backend != "nccl"
        coll_dev = "cpu" if (device == "cpu" or staged) else device
        cap = torch.tensor([int(local_cap)], dtype=torch.int64, device=coll_dev)
        dist.all_reduce(cap, op=dist.ReduceOp.MAX, group=group)
        self.block_cap = int(cap.item())
        n = block_len(self.block_cap)
        self.send = torch.zeros(n, dtype=torch.int64, device=device)
        self.recv = torch.zeros(self.world * n, dtype=torch.int64, device=device)
        self._hs = torch.zeros(n, dtype=torch.int64) if staged else None
        self._hr = torch.zeros(self.world * n, dtype=torch.int64) if staged else None

    def allgather(self):
        if self._hs is None:
            self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        else:
            self._hs.copy_(self.send)
            self.dist.all_gather_into_tensor(self._hr, self._hs, group=self.group)
            self.recv.copy_(self._hr)


class ShardedEngine:
    """Engine shard of rank `rank` of `world` with the epoch loop + exchange.

    advance_to(t) runs epochs [step, step + L) (the last one clipped to t), each
    followed by the allgather, exactly as the reference partitions time.
    With record_spikes=True every rank accumulates the global spike list."""

    def __init__(self, recipe, options, rank: int, world: int, device: int = 0,
                 exchange: Optional[SpikeExchange] = None, record_spikes: bool = False,
                 backend: Optional[str] = None):
        from .engine import Engine
        self.engine = Engine(recipe, options, device=device, rank=rank, world=world)
        self.dt = float(options.dt_ms)
        self.world = world
        self.ex = exchange if exchange is not None else SpikeExchange(
            self.engine.shard_spike_cap(), device="cuda", backend=backend)
        self.engine.set_exchange_buffers(self.ex.send.data_ptr(), self.ex.recv.data_ptr(),
                                         self.ex.block_cap, world)
        self.record = record_spikes
        self._t: List[np.ndarray] = []
        self._g: List[np.ndarray] = []

    def advance_to(self, t_ms: float):
        target = ceil_steps(t_ms, self.dt)
        torch = self.ex.torch
        while self.engine.step() < target:
            torch.cuda.synchronize()  # the exchange ran on torch's stream
            self.engine.run_epoch(t_ms)
            self.ex.allgather()
            if self.record:
                t, g = unpack_epoch(self.ex.recv.cpu().numpy(), self.world, self.ex.block_cap)
                self._t.append(t)
                self._g.append(g)
        torch.cuda.synchronize()

    def spike_arrays(self) -> Tuple[np.ndarray, np.ndarray]:
        if not self._t:
            return np.zeros(0), np.zeros(0, np.uint32)
        return np.concatenate(self._t), np.concatenate(self._g)


def run_shards_in_process(recipe, options, world: int, t_ms: float,
                          device: int = 0) -> Tuple[np.ndarray, np.ndarray, list]:
    """All `world` shards in one process on one GPU, the allgather done by
    concatenating the send blocks (the single-GPU test of the sharded path).
    Returns the global spike list (t, gid) and the shard engines."""
    import torch
    from .engine import Engine
    engines = [Engine(recipe, options, device=device, rank=r, world=world) for r in range(world)]
    cap = max(e.shard_spike_cap() for e in engines)
    n = block_len(cap)
    sends = [torch.zeros(n, dtype=torch.int64, device="cuda") for _ in range(world)]
    recvs = [torch.zeros(world * n, dtype=torch.int64, device="cuda") for _ in range(world)]
    for e, s, r in zip(engines, sends, recvs):
        e.set_exchange_buffers(s.data_ptr(), r.data_ptr(), cap, world)
    target = ceil_steps(t_ms, float(options.dt_ms))
    ts, gs = [], []
    while engines[0].step() < target:
        torch.cuda.synchronize()
        for e in engines:
            e.run_epoch(t_ms)
        torch.cuda.synchronize()
        gathered = torch.cat(sends)
        for r in recvs:
            r.copy_(gathered)
        t, g = unpack_epoch(gathered.cpu().numpy(), world, cap)
        ts.append(t)
        gs.append(g)
    torch.cuda.synchronize()
    t = np.concatenate(ts) if ts else np.zeros(0)
    g = np.concatenate(gs) if gs else np.zeros(0, np.uint32)
    return t, g, engines
