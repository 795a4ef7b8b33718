"""Protocol drivers on the B200 against the reference
(oracle/_ref), bitwise: every pairing trial's initial and final weight,
gb_dp_curve's points, and the STDP window."""
import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import protocols as PR
from paper_2411_16445_b200.recipe import StdpParams

pytestmark = pytest.mark.gpu


def test_gb_trials_bitwise(gpu):
    p = PR.GbParams()
    proto = PR.GbPairingProtocol(n_pairs=8, period_ms=250.0, settle_ms=500.0, dt_ms=0.5,
                                 trials=24, seed=3)
    deltas = [-100.0, -20.0, -5.0, 0.0, 5.0, 10.0, 30.0, 400.0]
    w0, wf = PR.gb_pairing_trials(p, deltas, proto)
    for di, d in enumerate(deltas):
        for t in range(proto.trials):
            rf, r0 = ref.gb_pairing_trial(p, d, proto, t, di)
            assert (w0[di, t], wf[di, t]) == (r0, rf), (d, t)


def test_gb_trials_noiseless_and_fine_dt(gpu):
    for p, dt in ((PR.GbParams(sigma_pl=0.0), 0.5), (PR.GbParams(), 0.05)):
        proto = PR.GbPairingProtocol(n_pairs=3, period_ms=300.0, settle_ms=200.0, dt_ms=dt,
                                     trials=8, seed=11)
        w0, wf = PR.gb_pairing_trials(p, [10.0, -10.0], proto)
        for di, d in enumerate((10.0, -10.0)):
            for t in range(proto.trials):
                assert (wf[di, t], w0[di, t]) == ref.gb_pairing_trial(p, d, proto, t, di)


def test_gb_dp_curve_bitwise(gpu):
    p = PR.GbParams()
    proto = PR.GbPairingProtocol(n_pairs=10, period_ms=200.0, settle_ms=400.0, dt_ms=0.5,
                                 trials=64, seed=999)
    deltas = [-50.0, -10.0, 0.0, 10.0, 50.0]
    got = PR.gb_dp_curve(p, deltas, proto)
    want = ref.gb_dp_curve(p, deltas, proto)
    for g, w in zip(got, want):
        assert (g.delta_t_ms, g.mean_initial, g.mean_final, g.mean_change, g.change_ci_half,
                g.ratio) == w


def test_stdp_window_bitwise(gpu):
    for p in (StdpParams(), StdpParams(tau_pre_ms=15.0, tau_post_ms=30.0, a_post_uS=-0.02)):
        deltas = np.concatenate([np.arange(-100.0, 101.0, 2.5), [1e-4, -1e-4, 500.0, -500.0]])
        got = PR.stdp_window(deltas, p)
        want = np.array([ref.stdp_window(d, p) for d in deltas])
        assert np.array_equal(got, want)
        assert PR.stdp_window(-10.0, p, n_pairs=7, period_ms=333.0) == \
            ref.stdp_window(-10.0, p, 7, 333.0)
