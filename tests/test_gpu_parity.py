"""Bitwise parity of the B200 engine against the reference engine (oracle/_ref)
on the reference's own recipe builders (network.cpp, bench.cpp).

Bar (BASELINE.json north_star): identical spike times and indices; state
(V, STC h/z/c, species, HH gates) identical too — we hold the engine to bitwise
equality everywhere, which is stricter than the 1e-9 relative fp64 bound."""
import numpy as np
import pytest

import ref
from parity import assert_cells_equal, assert_spikes_equal, run_both

pytestmark = pytest.mark.gpu

STC_FIELDS = [(0, "stc_h", np.float64), (0, "stc_z", np.float64), (0, "stc_c", np.float64),
              (0, "stc_sps_abs", np.float64)]


def small_net(**kw):  # test_engine.cpp:185-194
    base = dict(n_cells=50, n_exc=40, pattern=10, t_learn_ms=500.0, dt_ms=0.5, seed=11)
    base.update(kw)
    return ref.default_consolidation(**base)


def test_small_net_single_compartment(gpu):
    cfg = small_net()
    rr = ref.RefRecipe.consolidation(cfg)
    r, g = run_both(rr.view, 0.5, 11, [("advance", 1500.0)])
    n = assert_spikes_equal(r, g)
    assert n > 100
    assert_cells_equal(r, g, range(50), fields=("v",))
    assert_cells_equal(r, g, range(40), fields=(), group_fields=STC_FIELDS)


def test_small_net_multi_compartment(gpu):
    cfg = small_net(multi_compartment=1)
    rr = ref.RefRecipe.consolidation(cfg)
    r, g = run_both(rr.view, 0.5, 11, [("advance", 600.0), ("advance", 1500.0)])
    n = assert_spikes_equal(r, g)
    assert n > 100
    assert_cells_equal(r, g, range(50), fields=("v",))
    assert_cells_equal(r, g, range(40), fields=(), group_fields=STC_FIELDS)
    for gid in range(40):
        for sp in range(2):
            np.testing.assert_array_equal(r.read("species", gid, sp), g.cell(gid)._comp("species", sp))


def test_busyring_small_depth2(gpu):
    cfg = ref.default_busyring(n_cells=16, ring_size=4, random_per_cell=50, tree_depth=2,
                               duration_ms=100.0)
    rr = ref.RefRecipe.busyring(cfg)
    r, g = run_both(rr.view, cfg.dt_ms, cfg.seed, [("advance", 100.0)])
    n = assert_spikes_equal(r, g)
    assert n > 0
    assert_cells_equal(r, g, range(16), fields=("v", "hh_m", "hh_h", "hh_n"),
                       group_fields=[(0, "syn_kernel", np.float64)])


def test_busyring_small_stdp(gpu):
    cfg = ref.default_busyring(n_cells=16, ring_size=4, random_per_cell=50, tree_depth=1,
                               duration_ms=100.0, stdp_on_random=1)
    rr = ref.RefRecipe.busyring(cfg)
    r, g = run_both(rr.view, cfg.dt_ms, cfg.seed, [("advance", 100.0)])
    assert_spikes_equal(r, g)
    assert_cells_equal(r, g, range(16), fields=("v",),
                       group_fields=[(1, "stdp_w", np.float64), (1, "stdp_a_pre", np.float64),
                                     (1, "stdp_a_post", np.float64), (1, "syn_kernel", np.float64),
                                     (1, "stdp_last", np.int64)])


def test_fast_forward_8h_small(gpu):
    cfg = small_net(multi_compartment=1)
    rr = ref.RefRecipe.consolidation(cfg, eight_hour=True)
    t_ff0 = cfg.t_learn_ms + 3000.0
    t_recall = cfg.t_learn_ms + 8 * 3600e3
    t_ff1 = t_ff0 + np.floor((t_recall - 1000.0 - t_ff0) / cfg.coarse_dt_ms) * cfg.coarse_dt_ms
    sched = [("advance", t_ff0), ("ff", t_ff1, cfg.coarse_dt_ms), ("advance", t_recall + 500.0)]
    r, g = run_both(rr.view, 0.5, 11, sched)
    assert_spikes_equal(r, g)
    assert_cells_equal(r, g, range(50), fields=("v",))
    assert_cells_equal(r, g, range(40), fields=(), group_fields=STC_FIELDS)
