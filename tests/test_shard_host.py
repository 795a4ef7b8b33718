"""Host side of the sharded epoch loop (CPU only): the partition the engine
uses, the exchange block format, and the allgather over world_size-2 gloo."""
import os
import socket

import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import shard


def small_mc_recipe():
    cfg = ref.default_consolidation(n_cells=50, n_exc=40, pattern=10, t_learn_ms=500.0, dt_ms=0.5,
                                    seed=11, multi_compartment=1)
    return ref.RefRecipe.consolidation(cfg)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7])
def test_partition_covers_every_cell_once(world):
    rr = small_mc_recipe()
    b = shard.partition(rr.view, world)
    n = rr.view.n_cells
    assert len(b) == world + 1 and b[0] == 0 and b[-1] == n
    assert np.all(np.diff(b.astype(np.int64)) >= 0)
    if world > 1:
        # balanced by cost: no shard holds more than ~2x its share of cells here
        assert np.max(np.diff(b.astype(np.int64))) <= 2 * (n // world) + 2


def test_block_roundtrip_restores_reference_order():
    cap = 5
    b0 = shard.pack_block([3, 1], [12, 10], [6.1, 5.05], cap)
    b1 = shard.pack_block([7, 2, 2], [11, 13, 10], [5.7, 6.6, 5.2], cap)
    t, g = shard.unpack_epoch(np.concatenate([b0, b1]), 2, cap)
    # Impl::exchange order: by gid, then detection step (engine.cpp:877-888)
    assert g.tolist() == [1, 2, 2, 3, 7]
    assert t.tolist() == [5.05, 5.2, 6.6, 6.1, 5.7]
    with pytest.raises(ValueError):
        shard.pack_block(range(6), range(6), np.zeros(6), cap)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = shard.SpikeExchange(local_cap=3 + rank, device="cpu")
        assert ex.block_cap == 3 + world - 1  # agreed maximum
        gid = [10 * rank + 5, 10 * rank + 1]
        blk = shard.pack_block(gid, [rank, rank + 1], [rank + 0.25, rank + 0.5], ex.block_cap)
        import torch
        ex.send.copy_(torch.from_numpy(blk))
        ex.allgather()
        t, g = shard.unpack_epoch(ex.recv.numpy(), world, ex.block_cap)
        out.put((rank, g.tolist(), t.tolist()))
    finally:
        dist.destroy_process_group()


def test_exchange_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    expect_g = [1, 5, 11, 15]
    expect_t = [0.5, 0.25, 1.5, 1.25]
    for _, g, t in res:
        assert g == expect_g and t == expect_t
