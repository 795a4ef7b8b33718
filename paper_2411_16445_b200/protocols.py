"""Standalone protocol drivers of the reference on the device.

Mirrors mechanisms.hpp:268-300 (proj/include/mcsim/mechanisms.hpp):

  gb_pairing_trial / gb_dp_curve   calcium-based bistable rule under pre/post
                                   pairing, Monte-Carlo over trials
                                   (mechanisms.cpp:40-119)
  stdp_window                      event-exact pair-STDP window
                                   (mechanisms.cpp:9-38)

Every trial (and every window point) is one device thread of the B200
library (include/mcg.h: mcg_gb_trials, mcg_gb_dp_curve, mcg_stdp_window); the
results are bitwise the reference's on the same parameters and seeds.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields
from typing import List, Sequence, Tuple, Union

import numpy as np

from . import _abi as A
from .engine import _check
from .recipe import StdpParams


@dataclass
class GbParams:  # mechanisms.hpp:80-92
    tau_w_ms: float = 150e3
    w_star: float = 0.5
    gamma_p: float = 321.808
    gamma_d: float = 200.0
    theta_p: float = 1.3
    theta_d: float = 1.0
    sigma_pl: float = 2.8248
    tau_c_ms: float = 20.0
    c_pre: float = 1.0
    c_post: float = 2.0
    t_c_delay_ms: float = 13.7


@dataclass
class GbPairingProtocol:  # mechanisms.hpp:276-283
    n_pairs: int = 60
    period_ms: float = 1000.0
    settle_ms: float = 5000.0
    dt_ms: float = 0.5
    trials: int = 400
    seed: int = 0


@dataclass
class GbCurvePoint:  # mechanisms.hpp:285-292
    delta_t_ms: float = 0.0
    mean_initial: float = 0.0
    mean_final: float = 0.0
    mean_change: float = 0.0
    change_ci_half: float = 0.0
    ratio: float = 0.0


def _gb_structs(p: GbParams, proto: GbPairingProtocol):
    cp = A.mcg_gb_params(*[float(getattr(p, f.name)) for f in fields(GbParams)])
    cq = A.mcg_gb_protocol(int(proto.n_pairs), int(proto.trials), float(proto.period_ms),
                           float(proto.settle_ms), float(proto.dt_ms), int(proto.seed))
    return cp, cq


def gb_pairing_trials(p: GbParams, delta_ts_ms: Sequence[float], proto: GbPairingProtocol,
                      device: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """(w0, w_final), each [len(delta_ts_ms), proto.trials]: gb_pairing_trial
    (mechanisms.cpp:40-90) for every trial t and delta index d (the trial key
    is (seed, t, d, 0/1))."""
    d = np.ascontiguousarray(delta_ts_ms, dtype=np.float64).reshape(-1)
    cp, cq = _gb_structs(p, proto)
    w0 = np.empty((d.size, max(int(proto.trials), 0)), dtype=np.float64)
    wf = np.empty_like(w0)
    _check(A.lib().mcg_gb_trials(device, C.byref(cp), d.ctypes.data, d.size, C.byref(cq),
                                 w0.ctypes.data, wf.ctypes.data))
    return w0, wf


def gb_pairing_trial(p: GbParams, delta_t_ms: float, proto: GbPairingProtocol, trial: int,
                     delta_index: int = 0, device: int = 0) -> Tuple[float, float]:
    """One trial: (final w, w0), the reference's return value and *w0_out."""
    q = GbPairingProtocol(**{**proto.__dict__, "trials": trial + 1})
    deltas = np.full(delta_index + 1, float(delta_t_ms))
    w0, wf = gb_pairing_trials(p, deltas, q, device)
    return float(wf[delta_index, trial]), float(w0[delta_index, trial])


def gb_dp_curve(p: GbParams, delta_ts_ms: Sequence[float], proto: GbPairingProtocol,
                device: int = 0) -> List[GbCurvePoint]:
    """Mean weight change over proto.trials trials for each delta_t
    (mechanisms.cpp:92-119)."""
    d = np.ascontiguousarray(delta_ts_ms, dtype=np.float64).reshape(-1)
    cp, cq = _gb_structs(p, proto)
    out = (A.mcg_gb_point * max(d.size, 1))()
    _check(A.lib().mcg_gb_dp_curve(device, C.byref(cp), d.ctypes.data, d.size, C.byref(cq), out))
    return [GbCurvePoint(*[getattr(out[i], f.name) for f in fields(GbCurvePoint)])
            for i in range(d.size)]


def stdp_window(delta_t_ms: Union[float, Sequence[float]], p: StdpParams = None,
                n_pairs: int = 60, period_ms: float = 1000.0,
                device: int = 0) -> Union[float, np.ndarray]:
    """Weight change per pair for two regular trains phase-shifted by delta_t
    (post relative to pre), mechanisms.cpp:9-38; scalar in, scalar out."""
    p = p or StdpParams()
    scalar = np.ndim(delta_t_ms) == 0
    d = np.ascontiguousarray(np.atleast_1d(delta_t_ms), dtype=np.float64)
    cp = A.mcg_stdp_params(p.tau_pre_ms, p.tau_post_ms, p.a_pre_uS, p.a_post_uS, p.w0_uS,
                           p.wmax_uS)
    out = np.empty(d.size, dtype=np.float64)
    _check(A.lib().mcg_stdp_window(device, C.byref(cp), d.ctypes.data, d.size, int(n_pairs),
                                   float(period_ms), out.ctypes.data))
    return float(out[0]) if scalar else out
