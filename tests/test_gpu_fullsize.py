"""Full-size parity at the BASELINE.json configurations (reference engine with
all host cores as the oracle)."""
import os

import numpy as np
import pytest

import ref
from parity import assert_cells_equal, assert_spikes_equal, run_both
from test_gpu_builders import ref_cfg
from paper_2411_16445_b200 import network as N

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

STC = [(0, "stc_h", np.float64), (0, "stc_z", np.float64), (0, "stc_c", np.float64)]


def _run(view, dt, seed, sched):
    r = ref.RefEngine(view, dt, seed, os.cpu_count() or 1)
    from paper_2411_16445_b200 import Engine, EngineOptions
    g = Engine(view, EngineOptions(dt_ms=dt, seed=seed))
    for op in sched:
        for e in (r, g):
            if op[0] == "advance":
                e.advance_to(op[1])
            else:
                e.fast_forward_to(op[1], op[2])
    return r, g


def test_config3_mc_small_2s(gpu):
    """N=2000 MC (31 comps), seed 1: 2 s of background (5,082 spikes)."""
    c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
    rr = ref.RefRecipe.consolidation(ref_cfg(c), True)
    r, g = _run(rr.view, 0.5, 1, [("advance", 2000.0)])
    n = assert_spikes_equal(r, g)
    assert n == 5082
    assert_cells_equal(r, g, range(0, 2000, 7), fields=("v",))
    assert_cells_equal(r, g, range(0, 1600, 13), fields=(), group_fields=STC)


def test_config3_learning_phase(gpu):
    """N=2000 MC through the 100 Hz learning window (STC noise active)."""
    c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True,
                              t_learn_ms=1000.0)
    rr = ref.RefRecipe.consolidation(ref_cfg(c), True)
    r, g = _run(rr.view, 0.5, 1, [("advance", 3500.0)])
    assert_spikes_equal(r, g)
    assert_cells_equal(r, g, range(0, 1600, 5), fields=("v",), group_fields=STC)
    for gid in range(0, 1600, 50):
        for sp in range(2):
            np.testing.assert_array_equal(r.read("species", gid, sp),
                                          g.cell(gid)._comp("species", sp))


def test_busyring_default(gpu):
    """Default busyring (1024 cells, depth 2): SURVEY §8c golden 9,984 spikes."""
    rr = ref.RefRecipe.busyring(ref.default_busyring(ring_weight_uS=0.050515121785495443))
    r, g = _run(rr.view, 0.025, 0, [("advance", 200.0)])
    n = assert_spikes_equal(r, g)
    assert n == 9984


def test_config3_8h_protocol(gpu):
    """The flagship experiment at full size (N=2000 MC, seed 1): learning at
    10 s, detailed to 13 s, fast-forward across 8 h in coarse steps, recall
    (network.cpp:600-639). Spike trains through recall, every excitatory
    cell's STC state and probes of V are bitwise the reference's."""
    c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
    rr = ref.RefRecipe.consolidation(ref_cfg(c), True)
    t_recall = c.t_learn_ms + 8 * 3600e3
    t_ff0 = c.t_learn_ms + 3000.0
    t_ff1 = t_ff0 + np.floor((t_recall - 1000.0 - t_ff0) / c.coarse_dt_ms) * c.coarse_dt_ms
    sched = [("advance", t_ff0), ("ff", t_ff1, c.coarse_dt_ms), ("advance", t_recall + 500.0)]
    r, g = _run(rr.view, c.dt_ms, 1, sched)
    assert assert_spikes_equal(r, g) > 0
    assert_cells_equal(r, g, range(0, 1600), fields=(), group_fields=STC)
    assert_cells_equal(r, g, range(0, 2000, 11), fields=("v",))
