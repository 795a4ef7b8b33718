"""Shared helpers for the GPU parity tests: run the same flat recipe through
the reference engine (oracle/_ref) and the B200 engine and compare."""
import numpy as np

import ref  # oracle/ref.py (test infrastructure)
from paper_2411_16445_b200 import Engine, EngineOptions


def run_both(view, dt, seed, schedule):
    """schedule: list of ('advance', t) / ('ff', t, coarse)."""
    r = ref.RefEngine(view, dt, seed, 1)
    g = Engine(view, EngineOptions(dt_ms=dt, seed=seed))
    for op in schedule:
        if op[0] == "advance":
            r.advance_to(op[1])
            g.advance_to(op[1])
        else:
            r.fast_forward_to(op[1], op[2])
            g.fast_forward_to(op[1], op[2])
    return r, g


def assert_spikes_equal(r, g):
    rt, rg = r.spike_arrays()
    gt, gg = g.spike_arrays()
    assert len(rt) == len(gt), f"spike count ref {len(rt)} gpu {len(gt)}"
    if len(rt):
        bad = np.nonzero((rt != gt) | (rg != gg))[0]
        assert len(bad) == 0, (f"first mismatch at {bad[0]}: ref ({rt[bad[0]]!r},{rg[bad[0]]}) "
                               f"gpu ({gt[bad[0]]!r},{gg[bad[0]]})")
    return len(rt)


def assert_cells_equal(r, g, gids, fields=("v",), group_fields=()):
    for gid in gids:
        cv = g.cell(gid)
        for f in fields:
            a = r.read(f, gid)
            b = cv._comp(f) if f in ("v", "hh_m", "hh_h", "hh_n") else None
            np.testing.assert_array_equal(a, b, err_msg=f"gid {gid} field {f}")
        for gi, f, dt in group_fields:
            if gi >= r.ngroups(gid):
                continue
            a = r.read(f, gid, gi, dtype=dt)
            b = cv.groups[gi]._read(f, dt)
            np.testing.assert_array_equal(a, b, err_msg=f"gid {gid} group {gi} field {f}")
