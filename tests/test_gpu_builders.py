"""The product's network builders (paper_2411_16445_b200.network) reproduce
the reference builders' recipes exactly (network.cpp, bench.cpp), and the
config-1 driver reproduces run_stc_protocol's golden values."""
import numpy as np
import pytest

import ref
from recipe_compare import assert_recipes_equal
from paper_2411_16445_b200 import network as N

pytestmark = pytest.mark.gpu


def ref_cfg(c: N.ConsolidationConfig):
    r = ref.default_consolidation()
    for f, _ in ref.ref_consolidation_cfg._fields_:
        if f == "stc":
            continue
        v = getattr(c, f)
        setattr(r, f, int(v) if isinstance(v, bool) else v)
    return r


@pytest.mark.parametrize("mc,eight", [(False, False), (True, False), (True, True)])
def test_consolidation_builder_matches_reference(gpu, mc, eight):
    c = N.ConsolidationConfig(n_cells=300, n_exc=240, pattern=40, seed=5, multi_compartment=mc)
    mine = N.build_consolidation_network(c, eight).recipe.flatten()
    theirs = ref.RefRecipe.consolidation(ref_cfg(c), eight)
    assert_recipes_equal(mine.view, theirs.view)


def test_consolidation_builder_full_size(gpu):
    c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
    mine = N.build_consolidation_network(c, True).recipe.flatten()
    theirs = ref.RefRecipe.consolidation(ref_cfg(c), True)
    assert_recipes_equal(mine.view, theirs.view)


def test_busyring_builder_matches_reference(gpu):
    spec = N.default_busyring()
    spec.n_cells, spec.random_per_cell, spec.tree_depth = 16, 40, 2
    mine = N.build_busyring(spec).flatten()
    rc = ref.default_busyring(n_cells=16, random_per_cell=40, tree_depth=2)
    theirs = ref.RefRecipe.busyring(rc)
    assert_recipes_equal(mine.view, theirs.view)


def test_ring_weight_calibration_golden(gpu):
    # SURVEY §8c golden: default busyring ring weight 0.050515121785495443 uS
    w = N.calibrate_ring_weight(N.default_busyring())
    assert w == 0.050515121785495443


def test_stc_protocol_golden(gpu):
    # SURVEY §8c golden (STET trial 0, run_stc_protocol defaults)
    r = N.run_stc_protocol(N.StcSingleConfig(), N.StcProtocol.stet, 0)
    assert r.h_final == 4.5449467093946359
    assert r.z_final == 0.75323495592946443
    assert r.p_final == 0.24731552999708523


@pytest.mark.parametrize("proto", [1, 2, 3])
def test_stc_protocols_match_reference(gpu, proto):
    r = N.run_stc_protocol(N.StcSingleConfig(), proto, 1)
    h, z, p = ref.run_stc_protocol(proto, 1)
    assert (r.h_final, r.z_final, r.p_final) == (h, z, p)
