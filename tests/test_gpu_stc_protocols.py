"""The stc-protocols experiment (experiments.cpp:262-289) batched on the
device (network.run_stc_protocols: trials as cells of one engine with per-cell
RNG keys, mcg_set_cell_rng, on the point-cell kernel): every trial's final h,
z and PRP equal the reference's run_stc_protocol(cfg, p, t) (oracle/_ref) and
the single-trial device run, bit for bit, and the tag/synthesis flags and
traces equal the single-trial run's."""
import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import network as N

pytestmark = pytest.mark.gpu


def test_batched_protocols_match_reference(gpu):
    cfg = N.StcSingleConfig()
    protos = [N.StcProtocol.stet, N.StcProtocol.wtet, N.StcProtocol.slfs, N.StcProtocol.wlfs]
    trials = 3
    res = N.run_stc_protocols(cfg, protos, trials)
    for pi, p in enumerate(protos):
        for t in range(trials):
            g = res[pi][t]
            h, z, prp = ref.run_stc_protocol(p, t)
            assert (g.h_final, g.z_final, g.p_final) == (h, z, prp), (p, t)
    # the single-trial device run: flags and traces too
    one = N.run_stc_protocol(cfg, N.StcProtocol.slfs, 2)
    b = res[2][2]
    assert (b.max_abs_dh, b.tag_crossed, b.prp_crossed) == (one.max_abs_dh, one.tag_crossed, one.prp_crossed)
    for a, c in zip(b.traces, one.traces):
        np.testing.assert_array_equal(np.array(a), np.array(c))


def test_cell_rng_needs_point_kernel(gpu):
    """mcg_set_cell_rng is refused on the other stepping kernels."""
    c = N.ConsolidationConfig(n_cells=40, n_exc=32, pattern=8, seed=3, multi_compartment=True)
    e = N.Engine(N.build_consolidation_network(c, False).recipe, N.EngineOptions(0.5, 3))
    with pytest.raises(Exception, match="point-cell kernel"):
        e.set_cell_rng(np.arange(40), np.zeros(40))
