"""Sharded runs across processes, checked bitwise against the reference.

  * two ranks (processes) sharing one GPU, ShardedEngine with the host-staged
    gloo allgather between epochs (tests/shard_worker.py): every rank's copy
    of the global spike list, and each rank's cells' V and STC h, equal the
    reference engine's (oracle/_ref) on the whole network;
  * the exchange inside the library (mcg_shard_init_nccl +
    mcg_shard_advance_to: stepping launch + ncclAllGather per epoch on the
    engine's stream, one host wait per 32 epochs) with a one-rank
    communicator (NCCL refuses two ranks on one device): spikes and state
    equal the reference, both with batched and with per-epoch host waits."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import ref
from paper_2411_16445_b200 import Engine, EngineOptions

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _reference(n_cells, t_end):
    cfg = ref.default_consolidation(n_cells=n_cells, n_exc=n_cells * 4 // 5, pattern=n_cells // 8,
                                    t_learn_ms=300.0, dt_ms=0.5, seed=5, multi_compartment=1)
    rr = ref.RefRecipe.consolidation(cfg)
    r = ref.RefEngine(rr.view, 0.5, 5, 4)
    for t in (200.0, t_end):
        r.advance_to(t)
    return rr, r, cfg


def test_two_processes_gloo_match_reference(gpu, tmp_path):
    n, t_end, world = 120, 900.0, 2
    port = _free_port()
    procs = []
    for rank in range(world):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen(
            [sys.executable, os.path.join(ROOT, "tests", "shard_worker.py"),
             str(tmp_path / f"r{rank}.npz"), str(n), str(t_end), "gloo"], env=env,
            stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    for p in procs:
        out, _ = p.communicate(timeout=600)
        assert p.returncode == 0, out[-3000:]
    rr, r, cfg = _reference(n, t_end)
    rt, rg = r.spike_arrays()
    assert len(rt) > 50
    for rank in range(world):
        d = np.load(tmp_path / f"r{rank}.npz")
        np.testing.assert_array_equal(d["g"], rg)
        np.testing.assert_array_equal(d["t"].view(np.int64), rt.view(np.int64))
        b, e = int(d["b"]), int(d["e"])
        np.testing.assert_array_equal(d["v"], np.concatenate([r.read("v", x) for x in range(b, e)]))
        h = [r.read("stc_h", x, 0) for x in range(b, min(e, cfg.n_exc))]
        if h:
            np.testing.assert_array_equal(d["h"], np.concatenate(h))


@pytest.mark.parametrize("sync", [False, True])
def test_nccl_exchange_in_library_matches_reference(gpu, monkeypatch, sync):
    n, t_end = 200, 1200.0
    rr, r, cfg = _reference(n, t_end)
    if sync:
        monkeypatch.setenv("MCG_SHARD_SYNC", "1")
    g = Engine(rr.view, EngineOptions(0.5, 5), rank=0, world=1)
    g.init_nccl(Engine.nccl_unique_id())
    for t in (200.0, t_end):
        g.shard_advance_to(t)
    rt, rg = r.spike_arrays()
    for tt, gg in (g.global_spike_arrays(), g.spike_arrays()):
        np.testing.assert_array_equal(gg, rg)
        np.testing.assert_array_equal(tt.view(np.int64), rt.view(np.int64))
    for x in range(0, n, 7):
        np.testing.assert_array_equal(g.cell(x).v_mV, r.read("v", x))
        if x < cfg.n_exc:
            np.testing.assert_array_equal(g.cell(x).groups[0].stc_h, r.read("stc_h", x, 0))
            np.testing.assert_array_equal(g.cell(x).groups[0].stc_c, r.read("stc_c", x, 0))
