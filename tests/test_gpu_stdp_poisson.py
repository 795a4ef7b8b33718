"""run_stdp_poisson (network.cpp:93-120), the reference's single neuron with a
plastic STDP conductance synapse and a static inhibitory one under Poisson
input: the device run's spikes and plastic-weight trace equal the reference
engine's (oracle/_ref) on the same recipe, bit for bit."""
import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import network as N

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 3])
def test_stdp_poisson_matches_reference(gpu, seed):
    cfg = N.StdpPoissonConfig(duration_ms=2000.0, seed=seed)
    res = N.run_stdp_poisson(cfg)
    flat = N.build_stdp_single_neuron(cfg).flatten()
    r = ref.RefEngine(flat.view, cfg.dt_ms, cfg.seed, 1)
    r.advance_to(cfg.duration_ms)
    rt, rg = r.spike_arrays()
    assert res.post_count == len(rt) > 0
    np.testing.assert_array_equal(res.spikes_t_s, rt * 1e-3)
    tt, w = r.trace_arrays(0)
    np.testing.assert_array_equal(res.weight, w)
    np.testing.assert_array_equal(res.weight_t_s, tt * 1e-3)
    assert res.pre_count > 0
