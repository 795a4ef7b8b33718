"""Probe traces and output files against the reference:
every probe kind's samples bitwise (engine.cpp:785-829) through detailed steps
and fast-forward, and spikes.csv / trace csv byte-identical to the reference's
writers (csvio.cpp:34-69) on each engine's own results."""
import math

import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import Engine, EngineOptions, ProbeSpec, ProbeWhat
from paper_2411_16445_b200 import network as N

pytestmark = pytest.mark.gpu


def _both(recipe, dt, seed, schedule):
    flat = recipe.flatten()
    r = ref.RefEngine(flat.view, dt, seed, 1)
    g = Engine(flat, EngineOptions(dt, seed))
    for op in schedule:
        if op[0] == "a":
            r.advance_to(op[1])
            g.advance_to(op[1])
        else:
            r.fast_forward_to(op[1], op[2])
            g.fast_forward_to(op[1], op[2])
    return r, g


def test_stc_single_traces_bitwise(gpu, tmp_path):
    cfg = N.StcSingleConfig()
    times = N.stc_protocol_times(0, cfg.t_onset_ms)  # STET
    rec = N.build_stc_single(cfg, times)
    t_det = math.ceil((times[-1] + 2000.0) / 1000.0) * 1000.0
    rec.kinds[0].membrane.bg_quiet_t0_ms = t_det - 500.0
    rec.kinds[0].membrane.bg_quiet_t1_ms = cfg.t_eval_ms
    n_coarse = 600
    r, g = _both(rec, cfg.dt_ms, cfg.seed + 3, [("a", t_det),
                                                ("f", t_det + n_coarse * cfg.coarse_dt_ms,
                                                 cfg.coarse_dt_ms)])
    for p in range(4):
        rt, rv = r.trace_arrays(p)
        gt, gv = g.trace_arrays(p)
        assert len(rt) > 0
        assert np.array_equal(rt, gt) and np.array_equal(rv, gv), f"probe {p}"
        a, b = tmp_path / f"g{p}.csv", tmp_path / f"r{p}.csv"
        g.write_trace_csv(p, str(a))
        ref.write_trace_csv(str(b), rt * 1e-3, rv)
        assert a.read_bytes() == b.read_bytes()


def test_network_voltage_species_probes_and_spikes_csv(gpu, tmp_path):
    c = N.ConsolidationConfig(n_cells=60, n_exc=48, pattern=12, t_learn_ms=100.0, seed=5,
                              multi_compartment=True)
    b = N.build_consolidation_network(c, False)
    rec = b.recipe
    rec.probes = [ProbeSpec(0, ProbeWhat.voltage, 0, 0, "", 0, 1),
                  ProbeSpec(3, ProbeWhat.voltage, 30, 0, "", 0, 3),
                  ProbeSpec(5, ProbeWhat.species, 30, 0, "", 0, 2),
                  ProbeSpec(5, ProbeWhat.species, 0, 1, "", 0, 7),
                  ProbeSpec(7, ProbeWhat.syn_h, 0, 0, "rec", 2, 5),
                  ProbeSpec(7, ProbeWhat.syn_c, 0, 0, "rec", 2, 5),
                  ProbeSpec(50, ProbeWhat.voltage, 0, 0, "", 0, 4)]
    r, g = _both(rec, 0.5, 5, [("a", 150.0), ("a", 400.0), ("a", 777.0)])
    for p in range(len(rec.probes)):
        rt, rv = r.trace_arrays(p)
        gt, gv = g.trace_arrays(p)
        assert len(rt) > 0
        assert np.array_equal(rt, gt) and np.array_equal(rv, gv), f"probe {p}"
    rt, rg = r.spike_arrays()
    assert len(rt) > 0
    a, b2 = tmp_path / "g.csv", tmp_path / "r.csv"
    g.write_spikes_csv(str(a))
    ref.write_spikes_csv(str(b2), rt * 1e-3, rg)
    assert a.read_bytes() == b2.read_bytes()
