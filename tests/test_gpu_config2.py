"""BASELINE config 2: one consolidation MC neuron (cable LIF,
31 or 48 compartments) with plastic synapses at the basal tip, an STC group
and an STDP conductance group, each Poisson input driving one synapse of each.
Not in the reference's drivers; built with the Recipe API and run through both
engines (the reference's own Engine via the oracle), bitwise."""
import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import Engine, EngineOptions
from paper_2411_16445_b200 import network as N

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_inputs,large,t_end", [(200, False, 1500.0), (1000, True, 600.0)])
def test_single_neuron_plastic_bitwise(gpu, n_inputs, large, t_end):
    rec = N.build_single_neuron_plastic(n_inputs=n_inputs, rate_hz=20.0, duration_ms=t_end,
                                        dt_ms=0.1, large_dendrites=large, w_stc=4.0,
                                        w_stdp_uS=0.02)
    flat = rec.flatten()
    r = ref.RefEngine(flat.view, 0.1, 5, 1)
    g = Engine(flat, EngineOptions(0.1, 5))
    for t in (t_end / 3, t_end):
        r.advance_to(t)
        g.advance_to(t)
    rt, rg = r.spike_arrays()
    gt, gg = g.spike_arrays()
    assert np.array_equal(rt, gt) and np.array_equal(rg, gg)
    c = g.cell(0)
    np.testing.assert_array_equal(r.read("v", 0), c.v_mV)
    for sp in range(2):
        np.testing.assert_array_equal(r.read("species", 0, sp), c._comp("species", sp))
    for f in ("stc_h", "stc_c", "stc_z"):
        np.testing.assert_array_equal(r.read(f, 0, 0), c.groups[0]._read(f, np.float64))
    for f in ("stdp_w", "stdp_a_pre", "stdp_a_post", "syn_kernel"):
        np.testing.assert_array_equal(r.read(f, 0, 1), c.groups[1]._read(f, np.float64))
    np.testing.assert_array_equal(r.read("stdp_last", 0, 1, dtype=np.int64),
                                  c.groups[1]._read("stdp_last", np.int64))
