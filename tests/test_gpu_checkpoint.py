"""Checkpoints of the B200 engine against the reference:
byte-identical MCSCKPT1 at the same point of the same run (pending inbox,
delayed-calcium queue, STDP / kernels / HH / STC state), bit-exact round trip
(test_engine.cpp:198-236), and restores across engines in both directions."""
import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import Checkpoint, Engine, EngineOptions

pytestmark = pytest.mark.gpu


def _consolidation():
    cfg = ref.default_consolidation(n_cells=50, n_exc=40, pattern=10, t_learn_ms=500.0, dt_ms=0.5,
                                    seed=11, multi_compartment=1)
    return ref.RefRecipe.consolidation(cfg), 0.5, 11


def _busyring(stdp):
    cfg = ref.default_busyring(n_cells=16, ring_size=4, random_per_cell=50, tree_depth=1,
                               stdp_on_random=1 if stdp else 0, duration_ms=40.0, dt_ms=0.025,
                               seed=3)
    cfg.ring_weight_uS = 0.05
    return ref.RefRecipe.busyring(cfg), 0.025, 3


def _cells_equal(a, b, n):
    for gid in range(n):
        np.testing.assert_array_equal(a.read("v", gid), b.cell(gid).v_mV)
        for gi in range(a.ngroups(gid)):
            if a.group_size(gid, gi) == 0:
                continue
            for f in ("stc_h", "stc_c", "syn_kernel", "stdp_w"):
                try:
                    x = a.read(f, gid, gi)
                except Exception:
                    continue
                np.testing.assert_array_equal(x, b.cell(gid).groups[gi]._read(f, np.float64))


@pytest.mark.parametrize("net", ["consolidation", "busyring", "busyring_stdp"])
def test_checkpoint_bytes_identical(gpu, net):
    rr, dt, seed = _consolidation() if net == "consolidation" else _busyring(net.endswith("stdp"))
    r = ref.RefEngine(rr.view, dt, seed, 1)
    g = Engine(rr.view, EngineOptions(dt, seed))
    for t in ((300.0, 600.0, 777.0) if net == "consolidation" else (7.5, 20.0, 31.3)):
        r.advance_to(t)
        g.advance_to(t)
        a = r.make_checkpoint()
        b = g.make_checkpoint().data
        if a != b:
            fa, ua = Checkpoint.deserialize(a)
            fb, ub = Checkpoint.deserialize(b)
            diff = [k for k in sorted(set(fa) | set(fb)) if k not in fa or k not in fb
                    or not np.array_equal(fa[k], fb[k])]
            diff += [k for k in sorted(set(ua) | set(ub)) if k not in ua or k not in ub
                     or not np.array_equal(ua[k], ub[k])]
            raise AssertionError(f"checkpoints differ at t={t}: {diff[:8]}")


def test_round_trip_and_cross_restore(gpu):
    rr, dt, seed = _consolidation()
    g1 = Engine(rr.view, EngineOptions(dt, seed))
    g1.advance_to(600.0)
    ck = g1.make_checkpoint()
    g1.advance_to(1200.0)
    r1 = ref.RefEngine(rr.view, dt, seed, 1)
    r1.advance_to(1200.0)
    # GPU -> GPU
    g2 = Engine(rr.view, EngineOptions(dt, seed))
    g2.restore(ck)
    assert g2.time_ms() == 600.0
    g2.advance_to(1200.0)
    # GPU -> reference, reference -> GPU
    r2 = ref.RefEngine(rr.view, dt, seed, 1)
    r2.restore(ck.data)
    r2.advance_to(1200.0)
    r3 = ref.RefEngine(rr.view, dt, seed, 1)
    r3.advance_to(600.0)
    g3 = Engine(rr.view, EngineOptions(dt, seed))
    g3.restore(r3.make_checkpoint())
    g3.advance_to(1200.0)
    t1, i1 = g1.spike_arrays()
    tail = t1 > 600.0
    for e in (g2, g3):
        t, i = e.spike_arrays()
        assert np.array_equal(t, t1[tail]) and np.array_equal(i, i1[tail])
    rt, ri = r1.spike_arrays()
    assert np.array_equal(rt, t1) and np.array_equal(ri, i1)
    rt2, ri2 = r2.spike_arrays()
    assert np.array_equal(rt2, t1[tail]) and np.array_equal(ri2, i1[tail])
    _cells_equal(r1, g2, 50)
    _cells_equal(r1, g3, 50)
    assert g2.make_checkpoint().data == r1.make_checkpoint()


def test_restore_rejects(gpu):
    rr, dt, seed = _consolidation()
    g = Engine(rr.view, EngineOptions(dt, seed))
    g.advance_to(100.0)
    data = g.make_checkpoint().data
    from paper_2411_16445_b200.recipe import EngineError
    with pytest.raises(EngineError, match="truncated|corrupted"):
        g.restore(data[:-7])
    other = Engine(rr.view, EngineOptions(0.25, seed))
    with pytest.raises(EngineError, match="dt mismatch"):
        other.restore(data)
