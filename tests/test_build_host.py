"""The recipe -> runtime build (Impl::build, engine.cpp:189-408) is independent
of the number of host threads it uses (mcg_build_digest, host only): the same
edge rank order, instances, CSR and queues, and the same first error — the one
the reference's sequential loop raises — for seeded random recipes and for a
network large enough for the default threaded path."""
import ctypes as C

import numpy as np
import pytest

from paper_2411_16445_b200 import _abi as A
from paper_2411_16445_b200 import network as N
from paper_2411_16445_b200.recipe import ConnectionTable, Recipe

import test_gpu_point as TP
import test_gpu_random as TR


def digest(view, threads, rank=0, world=1):
    opt = A.mcg_options(0.5, 1, 1, 0, rank, world)
    out = (C.c_uint64 * 4)()
    st = A.lib().mcg_build_digest(C.byref(view), C.byref(opt), int(threads), out)
    if st != 0:
        return ("error", st, A.lib().mcg_last_error().decode())
    return tuple(out)


@pytest.mark.parametrize("seed", range(16))
def test_random_recipes_thread_invariant(seed):
    for mod in (TR, TP):
        flat = mod._recipe(seed).flatten()
        for world, rank in ((1, 0), (3, 1)):
            ref = digest(flat.view, 1, rank, world)
            for t in (2, 5):
                assert digest(flat.view, t, rank, world) == ref, (mod.__name__, seed, world, t)


def _consolidation_like(n=20000, p=0.005, seed=3):
    """A consolidation network (the builder's kinds and sources) with random
    recurrent pairs instead of the device ER sampler: ~2 M connections."""
    rng = np.random.default_rng(seed)
    m = int(n * (n - 1) * p)
    src = np.sort(rng.integers(0, n, m).astype(np.uint32))
    dst = rng.integers(0, n, m).astype(np.uint32)
    real = N.er_pairs
    N.er_pairs = lambda *a, **k: (src, dst)
    try:
        c = N.ConsolidationConfig(n_cells=n, n_exc=n * 4 // 5, p_conn=p, seed=1, multi_compartment=True)
        return N.build_consolidation_network(c, True).recipe
    finally:
        N.er_pairs = real


def test_large_network_thread_invariant():
    flat = _consolidation_like().flatten()
    ref = digest(flat.view, 1)
    assert ref[1] > (1 << 20)  # above the default single-thread threshold
    assert digest(flat.view, 0) == ref  # default thread count
    assert digest(flat.view, 7) == ref
    assert digest(flat.view, 4, rank=1, world=2) == digest(flat.view, 1, rank=1, world=2)


def test_first_failing_connection_wins():
    """Two bad connections in different thread chunks: every thread count
    reports the earlier one (the reference's loop order)."""
    rec = _consolidation_like(n=6000, p=0.05)
    t = rec.connection_table()
    n = len(t)
    src, dst = t.src.copy(), t.dst.copy()
    k_early, k_late = n // 3, (9 * n) // 10
    dst[k_late] = 10 ** 7            # "connection dst out of range" (later)
    src[k_early] = 10 ** 7           # "connection src out of range" (earlier)
    bad = ConnectionTable(t.from_source, src, dst, t.labels, t.label_idx, t.policy, t.weight, t.delay_ms)
    flat = Recipe(kinds=rec.kinds, cell_kind=rec.cell_kind, sources=rec.sources, connections=bad).flatten()
    errs = {digest(flat.view, th) for th in (1, 2, 4, 8)}
    assert len(errs) == 1
    (e,) = errs
    assert e[0] == "error" and e[2] == "connection src out of range", e
