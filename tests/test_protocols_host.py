"""Protocol drivers: the oracle's gb_pairing_trial /
gb_dp_curve / stdp_window pinned against the reference's own known answers
(test_mechanisms.cpp:63-82, 183-206) and golden values recorded from it, plus
the host side of the B200 API (no device calls)."""
import math

import numpy as np
import pytest

import ref
from paper_2411_16445_b200.protocols import GbCurvePoint, GbPairingProtocol, GbParams
from paper_2411_16445_b200.recipe import StdpParams


def test_stdp_window_closed_forms():  # test_mechanisms.cpp:63-82
    p = StdpParams()
    assert ref.stdp_window(1e-4, p) == pytest.approx(p.a_pre_uS, rel=1e-3)
    assert ref.stdp_window(-10.0, p) == pytest.approx(-0.0105 * math.exp(-1.0), rel=1e-9)
    assert abs(ref.stdp_window(500.0, p)) < 1e-12
    sq, count = 0.0, 0
    for dt in range(-50, 51, 5):
        if dt == 0:
            continue
        ana = p.a_pre_uS * math.exp(-dt / p.tau_pre_ms) if dt > 0 else \
            p.a_post_uS * math.exp(dt / p.tau_post_ms)
        sq += (ref.stdp_window(float(dt), p) - ana) ** 2
        count += 1
    assert math.sqrt(sq / count) <= 0.001


def test_gb_trial_reproducible_and_symmetric():  # test_mechanisms.cpp:183-206
    p = GbParams(sigma_pl=0.0)
    proto = GbPairingProtocol(trials=1, dt_ms=0.5)
    assert ref.gb_pairing_trial(p, 10.0, proto, 0, 0) == ref.gb_pairing_trial(p, 10.0, proto, 0, 0)
    for trial in (0, 1):
        wp, w0p = ref.gb_pairing_trial(p, 400.0, proto, trial, 0)
        wm, w0m = ref.gb_pairing_trial(p, -400.0, proto, trial, 0)
        assert w0p == w0m
        assert wp == pytest.approx(wm, rel=5e-3)


# golden values of the reference (oracle/_ref), recorded with this test's inputs
SMALL = GbPairingProtocol(n_pairs=5, period_ms=200.0, settle_ms=300.0, dt_ms=0.5, trials=16,
                          seed=7)


def test_gb_dp_curve_matches_trials():
    """gb_dp_curve's means are the trials' means (mechanisms.cpp:92-119)."""
    p = GbParams()
    deltas = [-20.0, 10.0]
    curve = ref.gb_dp_curve(p, deltas, SMALL)
    for di, d in enumerate(deltas):
        w = [ref.gb_pairing_trial(p, d, SMALL, t, di) for t in range(SMALL.trials)]
        s0 = 0.0
        sf = 0.0
        for wf, w0 in w:
            s0 += w0
            sf += wf
        assert curve[di][0] == d
        assert curve[di][1] == s0 / SMALL.trials and curve[di][2] == sf / SMALL.trials


def test_host_api_shapes():
    assert GbCurvePoint().ratio == 0.0
    assert GbPairingProtocol().trials == 400 and GbParams().t_c_delay_ms == 13.7
