"""Fast-forward time of the config-3 8 h protocol (the coarse steps from 13 s
to the recall window), wall clock around fast_forward_to; MCG_LIB selects the
library. Prints a checksum of the STC state so A/B runs can be compared."""
import os, sys, time, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
b = N.build_consolidation_network(c, True)
e = Engine(b.recipe, EngineOptions(0.5, 1))
t_recall = c.t_learn_ms + 8 * 3600e3
t_ff0 = c.t_learn_ms + 3000.0
t_ff1 = t_ff0 + np.floor((t_recall - 1000.0 - t_ff0) / c.coarse_dt_ms) * c.coarse_dt_ms
e.advance_to(t_ff0)
t0 = time.perf_counter()
e.fast_forward_to(t_ff1, c.coarse_dt_ms)
dt = time.perf_counter() - t0
n = int((t_ff1 - t_ff0) / c.coarse_dt_ms)
hsh = hashlib.sha1()
for gid in range(0, 1600, 3):
    g = e.cell(gid).groups[0]
    hsh.update(g.stc_h.tobytes()); hsh.update(g.stc_z.tobytes())
    hsh.update(e.cell(gid)._comp("species", 0).tobytes()); hsh.update(e.cell(gid)._comp("species", 1).tobytes())
e.advance_to(t_recall + 500.0)
print(os.environ.get("MCG_LIB", "libmcg.so").split("/")[-1], f"ff {dt:.3f} s, {1e6 * dt / n:.2f} us/coarse step",
      "state", hsh.hexdigest()[:12], "spikes", len(e.spike_arrays()[0]), flush=True)
