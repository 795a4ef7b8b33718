"""Output formats: spikes.csv / trace csv written by the
package are byte-identical to the reference's writers (csvio.cpp:34-69) on the
same data, including ties in time, awkward doubles and empty inputs."""
import numpy as np

import ref
from paper_2411_16445_b200 import csvio


def _same(tmp_path, name, ours, theirs):
    a, b = tmp_path / f"{name}_a.csv", tmp_path / f"{name}_b.csv"
    ours(str(a))
    theirs(str(b))
    assert a.read_bytes() == b.read_bytes()


def test_spikes_csv_bytes(tmp_path):
    rng = np.random.default_rng(5)
    t = np.round(rng.uniform(0, 2, 500), 3)  # many equal times
    t[::7] = 0.1 + 0.2  # 0.30000000000000004
    t[1] = 1e-300
    t[2] = 123456789.125
    g = rng.integers(0, 4000, 500).astype(np.uint32)
    _same(tmp_path, "sp", lambda p: csvio.write_spikes_csv(p, t, g),
          lambda p: ref.write_spikes_csv(p, t, g))
    _same(tmp_path, "empty", lambda p: csvio.write_spikes_csv(p, [], []),
          lambda p: ref.write_spikes_csv(p, [], []))
    t2, g2 = csvio.read_spikes_csv(str(tmp_path / "sp_a.csv"))
    order = np.lexsort((g, t))
    assert np.array_equal(t2, t[order]) and np.array_equal(g2, g[order])


def test_trace_csv_bytes(tmp_path):
    t = np.arange(0, 3, 0.001) * 1e-3
    v = -65.0 + np.sin(np.arange(t.size)) * 1e-7
    _same(tmp_path, "tr", lambda p: csvio.write_trace_csv(p, t, v),
          lambda p: ref.write_trace_csv(p, t, v))
    t2, v2 = csvio.read_trace_csv(str(tmp_path / "tr_a.csv"))
    assert np.array_equal(t2, t) and np.array_equal(v2, v)
