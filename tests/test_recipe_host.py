"""Host-side recipe handling: the Python recipe flattens to exactly the
recipe the reference builds (checked by running the reference engine on the
flattened recipe against the reference's own driver)."""
import numpy as np
import pytest

import ref
from recipe_compare import assert_recipes_equal
from paper_2411_16445_b200 import network as N
from paper_2411_16445_b200.recipe import (ConnectionSpec, EngineError, LifMembrane,
                                          PlacementSpec, Recipe, CellKindSpec, SynKind,
                                          SynSpec, ScriptedSource)


def test_stc_single_recipe_drives_reference_to_golden():
    """build_stc_single (network.cpp:318-349) -> flat -> reference engine ->
    the run_stc_protocol golden values (STET trial 0)."""
    cfg = N.StcSingleConfig()
    times = N.stc_protocol_times(N.StcProtocol.stet, cfg.t_onset_ms)
    r = N.build_stc_single(cfg, times)
    t_detailed = np.ceil((times[-1] + 2000.0) / 1000.0) * 1000.0
    r.kinds[0].membrane.bg_quiet_t0_ms = t_detailed - 500.0
    r.kinds[0].membrane.bg_quiet_t1_ms = cfg.t_eval_ms
    flat = r.flatten()
    e = ref.RefEngine(flat.view, cfg.dt_ms, cfg.seed, 1)
    e.advance_to(t_detailed)
    n_coarse = np.floor((cfg.t_eval_ms - t_detailed) / cfg.coarse_dt_ms)
    e.fast_forward_to(t_detailed + n_coarse * cfg.coarse_dt_ms, cfg.coarse_dt_ms)
    assert e.read("stc_h", 0, 0)[0] == 4.5449467093946359
    assert e.read("stc_z", 0, 0)[0] == 0.75323495592946443
    assert e.read("species", 0, 1)[0] == 0.24731552999708523


def test_flatten_roundtrip_through_reference():
    cfg = N.StcSingleConfig()
    r = N.build_stc_single(cfg, [10.0, 20.0])
    flat = r.flatten()
    back = ref.RefRecipe.from_flat(flat.view)
    assert_recipes_equal(flat.view, back.view)


def _error_recipes():
    """Recipes with build errors, each paired with the reference's message
    (Impl::build, engine.cpp:317-391: kinds first, then per connection dst,
    label, source/src and delay, in connection order)."""
    kind = CellKindSpec(membrane=LifMembrane(exact=True),
                        placements=[PlacementSpec("in", SynSpec(kind=SynKind.static_charge))])
    kind.segments = N.build_consolidation_cell(N.ConsolidationCellParams()).segments
    out = []
    r = Recipe(kinds=[kind], cell_kind=[0, 0], sources=[ScriptedSource([1.0])],
               connections=[ConnectionSpec(False, 0, 1, "nope", 0, 1.0, 5.0)])
    out.append((r, "connection label 'nope' not found"))
    out.append((Recipe(kinds=[kind], cell_kind=[0, 0], sources=[],
                       connections=[ConnectionSpec(False, 0, 7, "in", 0, 1.0, 5.0)]),
                "connection dst out of range"))
    # an earlier error wins: the kind check precedes every connection check
    out.append((Recipe(kinds=[kind], cell_kind=[0, 3], sources=[],
                       connections=[ConnectionSpec(False, 0, 1, "nope", 0, 1.0, 5.0)]),
                "cell kind out of range"))
    # connection order: a bad src on connection 0 before a bad label on connection 1
    out.append((Recipe(kinds=[kind], cell_kind=[0, 0], sources=[],
                       connections=[ConnectionSpec(False, 9, 1, "in", 0, 1.0, 5.0),
                                    ConnectionSpec(False, 0, 1, "gone", 0, 1.0, 5.0)]),
                "connection src out of range"))
    # a label resolving on no kind at an out-of-range destination: dst first
    out.append((Recipe(kinds=[kind], cell_kind=[0, 0], sources=[],
                       connections=[ConnectionSpec(False, 0, 1, "in", 0, 1.0, 5.0),
                                    ConnectionSpec(False, 0, 5, "gone", 0, 1.0, 5.0)]),
                "connection dst out of range"))
    return out


def test_build_errors_match_reference_messages():
    """flatten() passes unresolved labels and out-of-range indices through;
    the reference engine built from the flat recipe reports them in its own
    order, naming the label (tests/test_gpu_random.py checks the GPU engine
    raises the same)."""
    for r, msg in _error_recipes():
        flat = r.flatten()
        with pytest.raises(ref.RefError, match=msg):
            ref.RefEngine(flat.view, 0.5, 1, 1)


def test_grid_layout_matches_reference_discretize():
    """compartment numbering used by the builders == discretize (31 / 48 comps)."""
    for d, n in ((N.DendriteSize.small_dendrites, 31), (N.DendriteSize.large_dendrites, 48)):
        cell = N.build_consolidation_cell(N.ConsolidationCellParams(single_compartment=False,
                                                                    dendrites=d))
        g = N.grid_layout(cell.segments, 1.0)
        assert g.size == n
        r = Recipe(kinds=[CellKindSpec(segments=cell.segments)], cell_kind=[0])
        flat = r.flatten()
        k = flat.view.kinds[0]
        par = np.empty(64, np.int32)
        buf = [np.empty(64) for _ in range(4)]
        cnt = ref.lib().ref_discretize(k, 64, par.ctypes.data, *[b.ctypes.data for b in buf])
        assert cnt == n
    # small-dendrite parents
    cell = N.build_consolidation_cell(N.ConsolidationCellParams(single_compartment=False))
    g = N.grid_layout(cell.segments, 1.0)
    assert g.compartment_at(cell.apical_seg, 1.0) == 25
    assert g.compartment_at(cell.basal_seg, 1.0) == 30
    assert g.compartment_at(cell.soma_center_seg, 0.5) == 0


def test_single_neuron_plastic_recipe():
    """Config 2's recipe: per source one STC then one STDP connection,
    all onto cell 0 (a scalar dst broadcasts)."""
    from paper_2411_16445_b200 import network as N
    r = N.build_single_neuron_plastic(n_inputs=50, duration_ms=100.0, dt_ms=0.1)
    c = r.connections
    assert len(c) == 100
    assert list(c.src[:6]) == [0, 0, 1, 1, 2, 2]
    assert [c.labels[i] for i in c.label_idx[:4]] == ["rec", "stdp", "rec", "stdp"]
    assert set(c.dst.tolist()) == {0}
    assert r.flatten().view.n_connections == 100
