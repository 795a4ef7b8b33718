"""Checkpoints, host side: the package's Checkpoint parser on
the reference's own MCSCKPT1 bytes, with the reference's corruption checks
(test_engine.cpp:238-253)."""
import pytest

import ref
from paper_2411_16445_b200 import Checkpoint
from paper_2411_16445_b200.recipe import EngineError


def _small_ref(t):
    cfg = ref.default_consolidation(n_cells=50, n_exc=40, pattern=10, t_learn_ms=500.0, dt_ms=0.5,
                                    seed=11)
    rr = ref.RefRecipe.consolidation(cfg)
    e = ref.RefEngine(rr.view, 0.5, 11, 1)
    e.advance_to(t)
    return rr, e


def test_reference_checkpoint_parses():
    rr, e = _small_ref(100.0)
    data = e.make_checkpoint()
    f64, u64 = Checkpoint.deserialize(data)
    assert u64["meta/step"][0] == 200
    assert f64["meta/dt_ms"][0] == 0.5
    assert "cell/0/v" in f64 and "cell/49/flags" in u64 and "cell/0/inbox_meta" in u64
    assert len(u64["cell/3/inbox_meta"]) == 4 * len(f64["cell/3/inbox_w"])


def test_corruption_detected():
    rr, e = _small_ref(100.0)
    data = e.make_checkpoint()
    with pytest.raises(EngineError, match="truncated|corrupted"):
        Checkpoint.deserialize(data[:-7])
    bad = bytearray(data)
    bad[3] = ord("X")
    with pytest.raises(EngineError, match="bad magic"):
        Checkpoint.deserialize(bytes(bad))


def test_save_load(tmp_path):
    rr, e = _small_ref(50.0)
    ck = Checkpoint(e.make_checkpoint())
    p = tmp_path / "ck.bin"
    ck.save(str(p))
    assert Checkpoint.load(str(p)).data == ck.data
    with pytest.raises(EngineError, match="cannot open"):
        Checkpoint.load(str(tmp_path / "missing.bin"))
