"""Config 3 (or PROBE_N / PROBE_DEND=large) through k_warp for an ncu capture:
  ncu --set full --import-source on -k regex:k_warp -s 3 -c 1 -o out python tools/prof_warp.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
n = int(os.environ.get("PROBE_N", "2000"))
ne = n * 4 // 5
dend = N.DendriteSize.large_dendrites if os.environ.get("PROBE_DEND") == "large" else N.DendriteSize.small_dendrites
c = N.ConsolidationConfig(n_cells=n, n_exc=ne, p_conn=min(0.1, 0.1 * 1600 / ne), seed=1,
                          multi_compartment=True, dend_size=dend)
b = N.build_consolidation_network(c, True)
e = Engine(b.recipe, EngineOptions(0.5, 1))
e.advance_to(float(os.environ.get("T_END", "2000")))
print("spikes", len(e.spike_arrays()[0]))
