"""Randomized parity: seeded random recipes mixing every membrane (exact and
cable LIF, HH), every synapse kind (static charge / conductance / current,
STDP, homeostasis, STC), species with PRP synthesis, all three source kinds,
all selection policies and every probe kind, run through the reference
(oracle/_ref) and the B200 engine; spikes, state of every cell and group, and
traces must be bitwise equal (or both engines raise the same error)."""
import sys

import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import (CellKindSpec, ConnectionSpec, Engine, EngineOptions, HhMembrane,
                                   LifMembrane, PlacementSpec, PoissonSource, PoissonWindow,
                                   ProbeSpec, ProbeWhat, Recipe, RegularSource, ScriptedSource,
                                   Segment, SelectionPolicy, SpeciesSpec, SynKind, SynSpec)
from paper_2411_16445_b200 import network as N

pytestmark = pytest.mark.gpu

COND = (SynKind.static_cond, SynKind.stdp_cond)


def _segments(rng, n):
    segs = [Segment(-1, float(rng.uniform(8, 20)), float(rng.uniform(3, 8)), 1, 1.0)]
    for i in range(1, n):
        segs.append(Segment(int(rng.integers(0, i)), float(rng.uniform(10, 60)),
                            float(rng.uniform(0.4, 1.5)), 3, 1.0))
    return segs


def _kind(rng, which):
    if which == "exact":
        segs, mem = [N.tiny_cylinder()], N.point_lif(10.0, 10.0, -65.0, 10.0)
        mem.i_bg_nA, mem.sigma_bg_nA_sqrt_ms = float(rng.uniform(0.2, 1.1)), float(rng.uniform(0, 1.5))
        kinds = [SynKind.static_charge, SynKind.static_current, SynKind.homeo_current,
                 SynKind.stc_charge]
    elif which == "cable":
        segs = _segments(rng, int(rng.integers(1, 5)))
        mem = LifMembrane(exact=False, i_bg_nA=float(rng.uniform(0.0, 0.4)),
                          sigma_bg_nA_sqrt_ms=float(rng.uniform(0, 0.8)))
        kinds = list(SynKind)
    else:
        segs = _segments(rng, int(rng.integers(1, 4)))
        mem = HhMembrane()
        kinds = [SynKind.static_cond, SynKind.stdp_cond, SynKind.static_current,
                 SynKind.homeo_current, SynKind.stc_charge]
    k = CellKindSpec(segments=segs, target_compartment_um=float(rng.choice([2.0, 5.0, 20.0])),
                     membrane=mem)
    if which != "hh" and rng.random() < 0.7:
        k.species = [SpeciesSpec("SPS", 1e-11, 0.0, 0.0), SpeciesSpec("PRP", 1e-12, 3600e3, 0.0)]
        k.prp.enabled = True
    n_pl = int(rng.integers(1, 4))
    for p in range(n_pl):
        kd = SynKind(int(rng.choice([int(x) for x in kinds])))
        syn = SynSpec(kind=kd, tau_syn_ms=float(rng.uniform(1, 8)),
                      e_rev_mV=float(rng.choice([0.0, -80.0])),
                      calcium_scale=float(rng.uniform(0.5, 2.0)))
        syn.stdp.w0_uS = 0.01
        k.placements.append(PlacementSpec(f"p{p}", syn, 0, int(rng.choice([0, 0, 3]))))
    return k


def _recipe(seed, n=None):
    rng = np.random.default_rng(seed)
    which = ["exact", "cable", "hh"]
    kinds = [_kind(rng, w) for w in rng.choice(which, size=int(rng.integers(1, 4)))]
    n = int(rng.integers(6, 20)) if n is None else n
    cell_kind = [int(x) for x in rng.integers(0, len(kinds), n)]
    srcs = [PoissonSource([PoissonWindow(0.0, 150.0, float(rng.uniform(20, 200)))]),
            RegularSource(float(rng.uniform(0, 5)), float(rng.uniform(3, 9)), 20),
            ScriptedSource(sorted(float(x) for x in rng.uniform(0, 120, 10)))]
    conns = []
    for _ in range(int(rng.integers(3 * n, 8 * n))):
        dst = int(rng.integers(0, n))
        kd = kinds[cell_kind[dst]]
        pl = kd.placements[int(rng.integers(0, len(kd.placements)))]
        w = float(rng.uniform(0.5, 4.0)) if pl.syn.kind not in COND else float(rng.uniform(0.001, 0.02))
        if pl.syn.kind == SynKind.static_current:
            w = float(rng.uniform(0.05, 0.4))
        from_src = rng.random() < 0.4
        # univalent targets a one-instance group; pre-placed groups here have 3
        pol = SelectionPolicy(int(rng.integers(1, 3))) if pl.count > 1 else SelectionPolicy.univalent
        conns.append(ConnectionSpec(bool(from_src), int(rng.integers(0, 3 if from_src else n)), dst,
                                    pl.label, pol, w, float(rng.choice([0.5, 1.0, 2.5]))))
    probes = []
    for _ in range(4):
        g = int(rng.integers(0, n))
        kd = kinds[cell_kind[g]]
        pl = int(rng.integers(0, len(kd.placements)))
        what = ProbeWhat(int(rng.integers(0, 7)))
        if what == ProbeWhat.species and not kd.species:
            what = ProbeWhat.voltage
        # synapse probes read instance 0: only of pre-placed groups (never empty),
        # and only the fields that group's kind has
        sk = kd.placements[pl].syn.kind
        ok = kd.placements[pl].count > 0 and (
            what in (ProbeWhat.syn_weight, ProbeWhat.syn_kernel) or
            (what in (ProbeWhat.syn_h, ProbeWhat.syn_z, ProbeWhat.syn_c) and sk == SynKind.stc_charge))
        if what >= ProbeWhat.syn_weight and not ok:
            what = ProbeWhat.voltage
        probes.append(ProbeSpec(g, what, 0, int(rng.integers(0, 2)) if kd.species else 0,
                                kd.placements[pl].label if what >= ProbeWhat.syn_weight else "", 0,
                                int(rng.integers(1, 6))))
    return Recipe(kinds=kinds, cell_kind=cell_kind, sources=srcs, connections=conns, probes=probes)


FIELDS_GROUP = ("syn_weight", "syn_kernel", "stdp_a_pre", "stdp_a_post", "stdp_w", "homeo_w",
                "stc_h", "stc_z", "stc_c", "stc_sps_abs")


@pytest.mark.parametrize("seed", range(24))
def test_random_recipe_bitwise(gpu, seed):
    rec = _recipe(seed)
    dt = [0.5, 0.25, 0.1, 0.5][seed % 4]
    flat = rec.flatten()
    err_r = err_g = None
    try:
        r = ref.RefEngine(flat.view, dt, 100 + seed, 1)
    except Exception as e:  # noqa: BLE001
        err_r = str(e)
    try:
        g = Engine(flat, EngineOptions(dt, 100 + seed))
    except Exception as e:  # noqa: BLE001
        err_g = str(e)
    assert (err_r is None) == (err_g is None), (err_r, err_g)
    if err_r is not None:
        assert err_r == err_g
        return
    for t in (40.0, 97.0, 160.0):
        er = eg = None
        try:
            r.advance_to(t)
        except Exception as e:  # noqa: BLE001
            er = str(e)
        try:
            g.advance_to(t)
        except Exception as e:  # noqa: BLE001
            eg = str(e)
        assert er == eg
        if er is not None:
            return
    rt, rg = r.spike_arrays()
    gt, gg = g.spike_arrays()
    assert np.array_equal(rt, gt) and np.array_equal(rg, gg)
    for gid in range(len(rec.cell_kind)):
        cv = g.cell(gid)
        np.testing.assert_array_equal(r.read("v", gid), cv.v_mV, err_msg=f"gid {gid} v")
        for gi in range(r.ngroups(gid)):
            if r.group_size(gid, gi) == 0:
                continue
            for f in FIELDS_GROUP:
                try:
                    a = r.read(f, gid, gi)
                except Exception:  # noqa: BLE001  (field absent for this kind)
                    continue
                np.testing.assert_array_equal(a, cv.groups[gi]._read(f, np.float64),
                                              err_msg=f"gid {gid} group {gi} {f}")
    for p in range(len(rec.probes)):
        a, b = r.trace_arrays(p), g.trace_arrays(p)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), f"probe {p}"
    assert g.make_checkpoint().data == r.make_checkpoint()


def _wide_segments(rng, n):
    """Branchy trees: 6-40 segments, branches leaving their parent at 30 %, 50 %
    or 100 % of its length (nodes with several children inside a segment)."""
    n = int(rng.integers(6, 41))
    segs = [Segment(-1, float(rng.uniform(8, 20)), float(rng.uniform(3, 8)), 1, 1.0)]
    for i in range(1, n):
        segs.append(Segment(int(rng.integers(0, i)), float(rng.uniform(4, 30)),
                            float(rng.uniform(0.4, 1.5)), 3, float(rng.choice([0.3, 0.5, 1.0]))))
    return segs


@pytest.mark.parametrize("seed", range(8))
def test_random_trees_bitwise(gpu, monkeypatch, seed):
    """HH and conductance-driven cable cells on branchy random trees through the
    warp-parallel general solve (mcg_solve_tree_warp: one lane per chain,
    children gathered in descending index order) and, above 32 chains, the
    one-thread solve: spikes, state, probes and checkpoint bytes equal the
    reference's."""
    monkeypatch.setattr(sys.modules[__name__], "_segments", _wide_segments)
    test_random_recipe_bitwise(gpu, 1000 + seed)


@pytest.mark.parametrize("seed", range(6))
def test_random_recipe_sharded(gpu, seed):
    """The same random recipes cut into 2 or 3 shards (the allgather done in
    process): merged spikes and every cell's voltage equal the single engine's."""
    from paper_2411_16445_b200 import shard
    rec = _recipe(seed)
    dt = [0.5, 0.25, 0.1, 0.5][seed % 4]
    flat = rec.flatten()
    opt = EngineOptions(dt, 100 + seed)
    single = Engine(flat, opt)
    single.advance_to(120.0)
    t1, g1 = single.spike_arrays()
    world = 2 + seed % 2
    t2, g2, engines = shard.run_shards_in_process(flat.view, opt, world, 120.0)
    np.testing.assert_array_equal(g1, g2)
    np.testing.assert_array_equal(t1.view(np.int64), t2.view(np.int64))
    b = shard.partition(flat.view, world)
    for r, e in enumerate(engines):
        for gid in range(int(b[r]), int(b[r + 1])):
            np.testing.assert_array_equal(single.cell(gid).v_mV, e.cell(gid).v_mV)


@pytest.mark.parametrize("seed", range(6))
def test_random_recipe_fast_forward(gpu, seed):
    """fast_forward_to on the random recipes (engine.cpp:947-1034): both engines
    either fast-forward to identical state or reject the span with the same
    message (pending deliveries, spans that are not multiples of coarse dt)."""
    rec = _recipe(seed)
    dt = [0.5, 0.25, 0.1, 0.5][seed % 4]
    flat = rec.flatten()
    r = ref.RefEngine(flat.view, dt, 100 + seed, 1)
    g = Engine(flat, EngineOptions(dt, 100 + seed))
    for e in (r, g):
        e.advance_to(200.0)
    for t_ff, coarse in ((200.0 + 600 * 50.0, 50.0), (200.0 + 7.3, 5.0)):
        er = eg = None
        try:
            r.fast_forward_to(t_ff, coarse)
        except Exception as e:  # noqa: BLE001
            er = str(e)
        try:
            g.fast_forward_to(t_ff, coarse)
        except Exception as e:  # noqa: BLE001
            eg = str(e)
        assert er == eg
    for gid in range(len(rec.cell_kind)):
        np.testing.assert_array_equal(r.read("v", gid), g.cell(gid).v_mV)
        for gi in range(r.ngroups(gid)):
            if r.group_size(gid, gi) == 0:
                continue
            for f in ("stc_h", "stc_z", "stc_c"):
                try:
                    a = r.read(f, gid, gi)
                except Exception:  # noqa: BLE001
                    continue
                np.testing.assert_array_equal(a, g.cell(gid).groups[gi]._read(f, np.float64))
    assert g.make_checkpoint().data == r.make_checkpoint()


@pytest.mark.parametrize("seed", range(6))
def test_random_recipe_writes_and_restore(gpu, seed):
    """Mid-run writes of cell(gid).v_mV through the API, then a checkpoint of the
    B200 engine restored into a fresh one: both continuations equal the
    reference's."""
    rec = _recipe(seed)
    dt = [0.5, 0.25, 0.1, 0.5][seed % 4]
    flat = rec.flatten()
    r = ref.RefEngine(flat.view, dt, 100 + seed, 1)
    g = Engine(flat, EngineOptions(dt, 100 + seed))
    for e in (r, g):
        e.advance_to(60.0)
    rng = np.random.default_rng(seed)
    for gid in rng.integers(0, len(rec.cell_kind), 3):
        v = r.read("v", int(gid))
        if v.size == 0:
            continue
        v = v + rng.uniform(-3, 8, v.size)
        r.write_v(int(gid), v)
        g.cell(int(gid)).set_v(v)
    ck = g.make_checkpoint()
    assert ck.data == r.make_checkpoint()
    g2 = Engine(flat, EngineOptions(dt, 100 + seed))
    g2.restore(ck)
    for e in (r, g, g2):
        e.advance_to(150.0)
    rt, rg = r.spike_arrays()
    for e in (g, g2):
        t, i = e.spike_arrays()
        tail = rt > 60.0 if e is g2 else np.ones(len(rt), bool)
        assert np.array_equal(t, rt[tail]) and np.array_equal(i, rg[tail])
    for gid in range(len(rec.cell_kind)):
        np.testing.assert_array_equal(r.read("v", gid), g.cell(gid).v_mV)
        np.testing.assert_array_equal(r.read("v", gid), g2.cell(gid).v_mV)
    assert g2.make_checkpoint().data == r.make_checkpoint()


@pytest.mark.parametrize("seed", range(4))
def test_random_recipe_large_mixed(gpu, monkeypatch, seed):
    """Larger random networks (several mixed-kind cells per CTA); odd seeds in
    the non-resident batch mode (MCG_MAX_CELLS_PER_CTA)."""
    rec = _recipe(1000 + seed, n=260)
    dt = [0.5, 0.25][seed % 2]
    flat = rec.flatten()
    r = ref.RefEngine(flat.view, dt, 7 + seed, 1)
    if seed % 2:
        monkeypatch.setenv("MCG_MAX_CELLS_PER_CTA", "1")
    g = Engine(flat, EngineOptions(dt, 7 + seed))
    monkeypatch.delenv("MCG_MAX_CELLS_PER_CTA", raising=False)
    for t in (55.0, 130.0):
        r.advance_to(t)
        g.advance_to(t)
    rt, rg = r.spike_arrays()
    gt, gg = g.spike_arrays()
    assert len(rt) > 0
    assert np.array_equal(rt, gt) and np.array_equal(rg, gg)
    assert g.make_checkpoint().data == r.make_checkpoint()


def test_build_errors_match_reference(gpu):
    """Both engines raise the reference's message for each malformed recipe
    (error order of Impl::build, engine.cpp:317-391; the label by name)."""
    from test_recipe_host import _error_recipes
    from paper_2411_16445_b200.recipe import EngineError
    for r, msg in _error_recipes():
        flat = r.flatten()
        with pytest.raises(ref.RefError, match=msg):
            ref.RefEngine(flat.view, 0.5, 1, 1)
        with pytest.raises(EngineError, match=msg):
            Engine(flat, EngineOptions(0.5, 1))
