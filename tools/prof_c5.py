"""Drive config 5 (100k cells x 48 comps, p = 0.002) for an ncu capture of one
non-resident k_batch launch:

  ncu --set full --import-source on -k regex:k_batch -s 2 -c 1 -o out python tools/prof_c5.py
"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions

c = N.ConsolidationConfig(n_cells=100000, n_exc=80000, p_conn=0.002, seed=1, multi_compartment=True,
                          dend_size=N.DendriteSize.large_dendrites)
t0 = time.perf_counter()
b = N.build_consolidation_network(c, True)
e = Engine(b.recipe, EngineOptions(0.5, 1))
print("setup_s", time.perf_counter() - t0, flush=True)
e.set_timing(True)
e.advance_to(float(os.environ.get("T0", "100")))
s0 = e.stats()
e.advance_to(float(os.environ.get("T1", "300")))
s1 = e.stats()
print("us_per_step", 1e3 * (s1["advance_ms"] - s0["advance_ms"]) / (s1["steps"] - s0["steps"]),
      "launches", s1["epoch_kernel_launches"] - s0["epoch_kernel_launches"], flush=True)
