"""k_point (csrc/mcg_point.cuh): independent exact-LIF point cells, the shape of
the single-synapse protocols (network.cpp:318-399, BASELINE config 1).

Seeded random recipes of point cells with STC and static-charge synapses,
species with PRP synthesis, background noise with a quiet window, every source
kind and every probe kind, and no cell-to-cell connections, through the
reference (oracle/_ref) and the B200 engine: the engine must pick k_point, and
spikes, every cell's state, traces and checkpoint bytes must be bitwise equal,
also across a checkpoint/restore continuation and a fast-forward."""
import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import (CellKindSpec, ConnectionSpec, Engine, EngineOptions,
                                   PlacementSpec, PoissonSource, PoissonWindow, ProbeSpec, ProbeWhat,
                                   Recipe, RegularSource, ScriptedSource, SelectionPolicy, SpeciesSpec,
                                   SynKind, SynSpec)
from paper_2411_16445_b200 import network as N

pytestmark = pytest.mark.gpu

K_POINT = 2  # mcg_stats.stepping_kernel
FIELDS = ("syn_weight", "stc_h", "stc_z", "stc_c", "stc_sps_abs")


def _recipe(seed):
    rng = np.random.default_rng(seed)
    kinds = []
    for _ in range(int(rng.integers(1, 3))):
        mem = N.point_lif(10.0, 10.0, -65.0, 10.0)
        mem.i_bg_nA = float(rng.uniform(0.3, 1.4))
        mem.sigma_bg_nA_sqrt_ms = float(rng.choice([0.0, 0.8, 1.58]))
        if rng.random() < 0.5:
            mem.bg_quiet_t0_ms, mem.bg_quiet_t1_ms = 120.0, 180.0
        k = CellKindSpec(segments=[N.tiny_cylinder()], membrane=mem)
        if rng.random() < 0.8:
            k.species = [SpeciesSpec("SPS", 1e-11, 0.0, 0.0), SpeciesSpec("PRP", 1e-12, 3600e3, 0.0)]
            k.prp.enabled = True
        stc = SynSpec(kind=SynKind.stc_charge, calcium_scale=float(rng.uniform(1.0, 4.0)))
        k.placements = [PlacementSpec("stc", stc, 0, int(rng.choice([0, 1, 3]))),
                        PlacementSpec("chg", SynSpec(kind=SynKind.static_charge), 0, 0)]
        kinds.append(k)
    n = int(rng.integers(1, 7))
    cell_kind = [int(x) for x in rng.integers(0, len(kinds), n)]
    srcs = [PoissonSource([PoissonWindow(0.0, 90.0, float(rng.uniform(80, 300))),
                           PoissonWindow(200.0, 260.0, float(rng.uniform(50, 200)))]),
            RegularSource(float(rng.uniform(0, 5)), float(rng.uniform(3, 9)), 30),
            ScriptedSource(sorted(float(x) for x in rng.uniform(0, 250, 40)))]
    conns = []
    for dst in range(n):
        kd = kinds[cell_kind[dst]]
        n_append = 0
        for _ in range(int(rng.integers(2, 7))):
            pl = kd.placements[int(rng.integers(0, 2))]
            if pl.syn.kind == SynKind.stc_charge and pl.count == 0:
                if n_append == 4:  # k_point holds up to 4 STC instances per cell
                    continue
                n_append += 1
            pol = SelectionPolicy(int(rng.integers(1, 3))) if pl.count > 1 else SelectionPolicy.univalent
            conns.append(ConnectionSpec(True, int(rng.integers(0, 3)), dst, pl.label, pol,
                                        float(rng.uniform(0.5, 3.0)), float(rng.choice([0.5, 1.0, 2.5]))))
    probes = []
    for _ in range(5):
        g = int(rng.integers(0, n))
        kd = kinds[cell_kind[g]]
        stc_has = kd.placements[0].count > 0
        what = ProbeWhat(int(rng.integers(0, 7)))
        if what == ProbeWhat.species and not kd.species:
            what = ProbeWhat.voltage
        if what >= ProbeWhat.syn_weight and not stc_has:
            what = ProbeWhat.voltage
        probes.append(ProbeSpec(g, what, 0, int(rng.integers(0, 2)) if kd.species else 0,
                                "stc" if what >= ProbeWhat.syn_weight else "", 0, int(rng.integers(1, 40))))
    return Recipe(kinds=kinds, cell_kind=cell_kind, sources=srcs, connections=conns, probes=probes)


def _compare(r, g, n, n_probes=0):
    rt, rg = r.spike_arrays()
    gt, gg = g.spike_arrays()
    np.testing.assert_array_equal(rg, gg)
    np.testing.assert_array_equal(rt.view(np.int64), gt.view(np.int64))
    for gid in range(n):
        cv = g.cell(gid)
        np.testing.assert_array_equal(r.read("v", gid), cv.v_mV, err_msg=f"gid {gid} v")
        for si, sp in enumerate(cv.species):
            np.testing.assert_array_equal(r.read("species", gid, si), sp, err_msg=f"gid {gid} species {si}")
        if r.group_size(gid, 0):
            for f in FIELDS:
                np.testing.assert_array_equal(r.read(f, gid, 0), cv.groups[0]._read(f, np.float64),
                                              err_msg=f"gid {gid} {f}")
    if n_probes:
        for p in range(n_probes):
            a, b = r.trace_arrays(p), g.trace_arrays(p)
            np.testing.assert_array_equal(a[0], b[0])
            np.testing.assert_array_equal(a[1].view(np.int64), b[1].view(np.int64), err_msg=f"probe {p}")


@pytest.mark.parametrize("seed", range(12))
def test_point_cells_bitwise(gpu, seed):
    rec = _recipe(seed)
    dt = [0.5, 0.2, 0.1, 0.25][seed % 4]
    flat = rec.flatten()
    r = ref.RefEngine(flat.view, dt, 7 + seed, 1)
    g = Engine(flat, EngineOptions(dt, 7 + seed))
    assert g.stats()["stepping_kernel"] == K_POINT
    for t in (33.0, 150.0, 300.0):
        r.advance_to(t)
        g.advance_to(t)
    _compare(r, g, len(rec.cell_kind), len(rec.probes))
    assert g.make_checkpoint().data == r.make_checkpoint()
    # continuation from each other's checkpoint, then a fast-forward
    ck = r.make_checkpoint()
    g2 = Engine(flat, EngineOptions(dt, 7 + seed))
    from paper_2411_16445_b200.engine import Checkpoint
    g2.restore(Checkpoint(ck))
    r.clear_spikes()  # the restored engine's spike list starts empty
    for e in (r, g2):
        e.advance_to(420.0)
    _compare(r, g2, len(rec.cell_kind))
    er = eg = None
    try:
        r.fast_forward_to(420.0 + 100 * 10.0, 10.0)
    except Exception as e:  # noqa: BLE001
        er = str(e)
    try:
        g2.fast_forward_to(420.0 + 100 * 10.0, 10.0)
    except Exception as e:  # noqa: BLE001
        eg = str(e)
    assert er == eg
    if er is None:
        _compare(r, g2, len(rec.cell_kind))


def test_stet_protocol_on_k_point(gpu):
    """config 1: STET trial 0 reaches SURVEY §8(c)'s golden h, z, p through k_point."""
    cfg = N.StcSingleConfig()
    res = N.run_stc_protocol(cfg, N.StcProtocol.stet, 0)
    assert res.h_final == 4.5449467093946359
    assert res.z_final == 0.75323495592946443
    assert res.p_final == 0.24731552999708523
