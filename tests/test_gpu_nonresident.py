"""The non-resident modes against the reference, bitwise, forced on a small
network (the hooks are read at engine construction):
  * k_batch with more cell batches than CTAs (each batch staged from global
    memory per epoch, STC state in global memory, kind blocks reused across
    batches, staged delivery per batch): MCG_NO_WARP + MCG_MAX_CELLS_PER_CTA;
  * k_warp with more cell groups than warps (each group staged per epoch by
    its warp, lazy calcium in global memory): MCG_WARP_GRID + MCG_WARP_WARPS."""
import os

import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import Engine, EngineOptions

pytestmark = pytest.mark.gpu


HOOKS = {"batch": {"MCG_NO_WARP": "1", "MCG_MAX_CELLS_PER_CTA": "2"},
         "warp": {"MCG_WARP_GRID": "3", "MCG_WARP_WARPS": "2"}}


@pytest.mark.parametrize("kernel", ["batch", "warp"])
@pytest.mark.parametrize("mc", [1, 0])
def test_nonresident_batches_bitwise(gpu, monkeypatch, mc, kernel):
    cfg = ref.default_consolidation(n_cells=320, n_exc=256, pattern=40, t_learn_ms=300.0, dt_ms=0.5,
                                    seed=7, multi_compartment=mc)
    rr = ref.RefRecipe.consolidation(cfg)
    r = ref.RefEngine(rr.view, 0.5, 7, 1)
    for k, v in HOOKS[kernel].items():
        monkeypatch.setenv(k, v)
    g = Engine(rr.view, EngineOptions(0.5, 7))
    for k in HOOKS[kernel]:
        monkeypatch.delenv(k)
    for t in (250.0, 700.0, 1000.0):
        r.advance_to(t)
        g.advance_to(t)
    rt, rg = r.spike_arrays()
    gt, gg = g.spike_arrays()
    assert len(rt) > 0
    assert np.array_equal(rt, gt) and np.array_equal(rg, gg)
    for gid in (0, 5, 39, 200, 300):
        np.testing.assert_array_equal(r.read("v", gid), g.cell(gid).v_mV)
        if gid < 256:
            np.testing.assert_array_equal(r.read("stc_h", gid, 0), g.cell(gid).groups[0].stc_h)
            np.testing.assert_array_equal(r.read("stc_c", gid, 0), g.cell(gid).groups[0].stc_c)
    assert g.make_checkpoint().data == r.make_checkpoint()
