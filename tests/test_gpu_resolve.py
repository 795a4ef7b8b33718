"""Connection resolution on the device (mcg_resolve.cuh; Impl::build,
engine.cpp:357-391): the instances every connection lands on (append_instance,
select_target's cursors) and the edge records in rank order (EventOrder,
engine.cpp:25-31) equal the host build's bit for bit.  The host build is the
one pinned against the reference (tests/test_build_host.py,
tests/test_gpu_dropin.py); here each engine's own layout digest
(mcg_engine_layout_digest) is compared with mcg_build_digest of the same
recipe, and the engines that resolved on the device say so in their stats.
Every other -m gpu parity test runs through the device-resolved layout too
(it is the default for recipes without STDP placements)."""
import ctypes as C

import pytest

from paper_2411_16445_b200 import _abi as A
from paper_2411_16445_b200 import network as N
from paper_2411_16445_b200 import Engine, EngineOptions
from paper_2411_16445_b200.recipe import ConnectionTable, Recipe

import test_build_host as TB
import test_gpu_point as TP
import test_gpu_random as TR

pytestmark = pytest.mark.gpu


def _engine_digest(eng):
    out = (C.c_uint64 * 4)()
    assert A.lib().mcg_engine_layout_digest(eng._h, out) == 0, A.lib().mcg_last_error().decode()
    return tuple(out)


def _check(flat, dt=0.5, rank=0, world=1, expect_device=None):
    host = TB.digest(flat.view, 1, rank, world) if dt == 0.5 else None
    eng = Engine(flat, EngineOptions(dt, 1), rank=rank, world=world)
    st = eng.stats()
    if expect_device is not None:
        assert st["edges_on_device"] == int(expect_device)
    got = _engine_digest(eng)
    if host is not None:
        assert got == host
    return st["edges_on_device"], got


@pytest.mark.parametrize("seed", range(16))
def test_random_recipes_device_resolution(gpu, seed):
    """Seeded random recipes (every synapse kind, appended and pre-placed
    groups with every targeting policy, sources, ragged fan-in): the engine's
    layout equals the host build's; world 3 shards resolve their own edges."""
    n_dev = 0
    for mod in (TR, TP):
        flat = mod._recipe(seed).flatten()
        on_dev, _ = _check(flat)
        n_dev += on_dev
        _check(flat, rank=1, world=3)
    assert n_dev >= 1  # the point-cell recipes carry no STDP placement


def test_policies_and_appends_device(gpu):
    """Round-robin, round-robin-halt and univalent connections interleaved on
    the same pre-placed groups, appended groups filled out of destination
    order, sources and cells in one list."""
    rec = TR._recipe(3)
    t = rec.connection_table()
    import numpy as np
    rng = np.random.default_rng(11)
    n = len(t)
    perm = rng.permutation(n)  # connection order scrambled: cursors advance in the new order
    tt = ConnectionTable(t.from_source[perm], t.src[perm], t.dst[perm], t.labels,
                         t.label_idx[perm], t.policy[perm], t.weight[perm], t.delay_ms[perm])
    flat = Recipe(kinds=rec.kinds, cell_kind=rec.cell_kind, sources=rec.sources, connections=tt).flatten()
    _check(flat, expect_device=True)  # seed 3: no STDP placement


def test_large_network_device_resolution(gpu):
    """~2 M connections (the threaded host path's size class)."""
    flat = TB._consolidation_like().flatten()
    on_dev, d = _check(flat, expect_device=True)
    assert d[1] > (1 << 20)


def test_config5_layout_device_resolution(gpu):
    """Config 5 (100 k cells, p = 0.002, ~20 M connections): the engine's
    device-resolved layout equals the host build's."""
    c = N.ConsolidationConfig(n_cells=100000, n_exc=80000, p_conn=0.002, seed=1, multi_compartment=True,
                              dend_size=N.DendriteSize.large_dendrites)
    flat = N.build_consolidation_network(c, True).recipe.flatten()
    _check(flat, expect_device=True)


def test_host_resolution_switch(gpu, monkeypatch):
    """MCG_HOST_RESOLVE=1 keeps the host's pass 1 (same layout)."""
    flat = TR._recipe(5).flatten()
    monkeypatch.setenv("MCG_HOST_RESOLVE", "1")
    on_dev, d_host = _check(flat, expect_device=False)
    monkeypatch.delenv("MCG_HOST_RESOLVE")
    _, d_dev = _check(flat)
    assert d_host == d_dev
