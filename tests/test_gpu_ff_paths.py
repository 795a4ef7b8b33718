"""fast_forward_to (engine.cpp:947-1034) on morphologies that select each of
the fast-forward kernels' paths (csrc/mcg_epoch.cuh): the register-resident
cells with the level-parallel lane solve (spider trees of <= 32 compartments),
the serial shared-memory solve (33-64 compartments, or a compartment with more
than MCG_FF_MAXCH children), the generic constant systems (three species) and
the general loop (two STC specs on one cell); with probes sampled at every
coarse step. Everything must equal the reference bitwise."""
import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import (CellKindSpec, ConnectionSpec, Engine, EngineOptions,
                                   LifMembrane, PlacementSpec, PoissonSource, PoissonWindow,
                                   ProbeSpec, ProbeWhat, Recipe, Segment, SelectionPolicy,
                                   SpeciesSpec, SynKind, SynSpec)

pytestmark = pytest.mark.gpu


def _segments(shape):
    soma = Segment(-1, 12.0, 5.0, 1, 1.0)
    if shape == "spider":       # 3 branches off the soma
        return [soma] + [Segment(0, 40.0, 0.8, 3, 1.0) for _ in range(3)]
    if shape == "star":         # 6 branches: the root has more than MCG_FF_MAXCH children
        return [soma] + [Segment(0, 20.0, 0.8, 3, 1.0) for _ in range(6)]
    if shape == "long":         # one long chain: 33-64 compartments
        return [soma, Segment(0, 100.0, 0.8, 3, 1.0), Segment(1, 80.0, 0.6, 3, 1.0)]
    raise ValueError(shape)


def _kind(shape, n_species=2, two_specs=False, target=5.0):
    k = CellKindSpec(segments=_segments(shape), target_compartment_um=target,
                     membrane=LifMembrane(exact=False, i_bg_nA=0.0, sigma_bg_nA_sqrt_ms=0.0))
    k.species = [SpeciesSpec("SPS", 1e-11, 0.0, 0.0), SpeciesSpec("PRP", 1e-12, 3600e3, 0.0)]
    if n_species == 3:
        k.species.append(SpeciesSpec("X", 5e-12, 1000e3, 0.0))
    k.prp.enabled = True
    k.placements = [PlacementSpec("stc", SynSpec(kind=SynKind.stc_charge, calcium_scale=2.0), 2, 0)]
    if two_specs:
        k.placements.append(PlacementSpec("stc2", SynSpec(kind=SynKind.stc_charge,
                                                          calcium_scale=1.5), 4, 0))
    return k


CASES = {
    "spider": dict(shape="spider"),
    "star": dict(shape="star"),
    "long": dict(shape="long", target=5.0),
    "three_species": dict(shape="spider", n_species=3),
    "two_specs": dict(shape="spider", two_specs=True),
}


def _recipe(case, n=6, seed=0):
    rng = np.random.default_rng(seed)
    kd = _kind(**CASES[case])
    src = [PoissonSource([PoissonWindow(0.0, 250.0, 150.0)]) for _ in range(4)]
    conns = []
    for dst in range(n):
        for s in range(4):
            for lab in [p.label for p in kd.placements]:
                conns.append(ConnectionSpec(True, s, dst, lab, SelectionPolicy.univalent,
                                            float(rng.uniform(2.0, 6.0)), 1.0))
        for pre in range(n):
            if pre != dst and rng.random() < 0.5:
                conns.append(ConnectionSpec(False, pre, dst, "stc", SelectionPolicy.univalent,
                                            float(rng.uniform(0.1, 0.5)), 2.0))
    probes = [ProbeSpec(0, ProbeWhat.syn_h, 0, 0, "stc", 0, 1),
              ProbeSpec(1, ProbeWhat.syn_z, 0, 0, "stc", 1, 1),
              ProbeSpec(2, ProbeWhat.species, 2, 0, "", 0, 1),
              ProbeSpec(3, ProbeWhat.species, 0, 1, "", 0, 2),
              ProbeSpec(4, ProbeWhat.voltage, 0, 0, "", 0, 1)]
    return Recipe(kinds=[kd], cell_kind=[0] * n, sources=src, connections=conns, probes=probes)


@pytest.mark.parametrize("case", sorted(CASES))
def test_fast_forward_paths(gpu, case):
    flat = _recipe(case).flatten()
    r = ref.RefEngine(flat.view, 0.5, 7, 1)
    g = Engine(flat, EngineOptions(0.5, 7))
    sched = [("a", 400.0), ("f", 400.0 + 800 * 50.0, 50.0), ("a", 400.0 + 800 * 50.0 + 60.0)]
    for op in sched:
        for e in (r, g):
            if op[0] == "a":
                e.advance_to(op[1])
            else:
                e.fast_forward_to(op[1], op[2])
    n_sp = CASES[case].get("n_species", 2)
    for gid in range(6):
        np.testing.assert_array_equal(r.read("v", gid), g.cell(gid).v_mV)
        for sp in range(n_sp):
            np.testing.assert_array_equal(r.read("species", gid, sp),
                                          g.cell(gid)._comp("species", sp))
        for gi in range(r.ngroups(gid)):
            if r.group_size(gid, gi) == 0:
                continue
            for f in ("stc_h", "stc_z", "stc_c", "stc_sps_abs"):
                np.testing.assert_array_equal(r.read(f, gid, gi),
                                              g.cell(gid).groups[gi]._read(f, np.float64))
    for p in range(5):
        rt, rv = r.trace_arrays(p)
        gt, gv = g.trace_arrays(p)
        np.testing.assert_array_equal(rt, gt)
        np.testing.assert_array_equal(rv, gv)
    assert g.make_checkpoint().data == r.make_checkpoint()
