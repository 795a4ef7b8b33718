"""Sharded epoch loop on one GPU: `world` shards of one network in one
process (the allgather done by concatenation), merged spikes and per-cell
state bitwise equal to the single-engine run (and so to the reference)."""
import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import Engine, EngineOptions, shard

pytestmark = pytest.mark.gpu


def consolidation(mc):
    cfg = ref.default_consolidation(n_cells=50, n_exc=40, pattern=10, t_learn_ms=500.0, dt_ms=0.5,
                                    seed=11, multi_compartment=mc)
    return ref.RefRecipe.consolidation(cfg), cfg


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mc", [0, 1])
def test_shards_match_single_engine(gpu, world, mc):
    rr, cfg = consolidation(mc)
    opt = EngineOptions(cfg.dt_ms, cfg.seed)
    single = Engine(rr.view, opt)
    single.advance_to(1500.0)
    t1, g1 = single.spike_arrays()
    t2, g2, engines = shard.run_shards_in_process(rr.view, opt, world, 1500.0)
    assert len(t1) > 100
    np.testing.assert_array_equal(g1, g2)
    np.testing.assert_array_equal(t1.view(np.int64), t2.view(np.int64))
    b = shard.partition(rr.view, world)
    for r, e in enumerate(engines):
        assert e.gid_range() == (int(b[r]), int(b[r + 1]))
        for gid in range(int(b[r]), int(b[r + 1])):
            np.testing.assert_array_equal(single.cell(gid).v_mV, e.cell(gid).v_mV)
            if gid < cfg.n_exc:
                np.testing.assert_array_equal(single.cell(gid).groups[0].stc_h,
                                              e.cell(gid).groups[0].stc_h)


def test_busyring_shards_match_single_engine(gpu):
    cfg = ref.default_busyring(n_cells=16, ring_size=4, random_per_cell=50, tree_depth=1,
                               duration_ms=100.0, stdp_on_random=1)
    rr = ref.RefRecipe.busyring(cfg)
    opt = EngineOptions(cfg.dt_ms, cfg.seed)
    single = Engine(rr.view, opt)
    single.advance_to(100.0)
    t1, g1 = single.spike_arrays()
    t2, g2, _ = shard.run_shards_in_process(rr.view, opt, 2, 100.0)
    assert len(t1) > 0
    np.testing.assert_array_equal(g1, g2)
    np.testing.assert_array_equal(t1.view(np.int64), t2.view(np.int64))


def test_sharded_engine_refuses_plain_advance(gpu):
    rr, cfg = consolidation(0)
    e = Engine(rr.view, EngineOptions(cfg.dt_ms, cfg.seed), rank=0, world=2)
    with pytest.raises(Exception, match="sharded engine"):
        e.advance_to(10.0)
