"""Drive the config-3 network for an ncu capture of one k_batch launch.

  ncu --set full --import-source on -k regex:k_batch -s 25 -c 1 -o out python tools/prof_batch.py
"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2411_16445_b200 import network as N, Engine, EngineOptions

c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
b = N.build_consolidation_network(c, True)
e = Engine(b.recipe, EngineOptions(0.5, 1))
e.advance_to(1000.0)
e.advance_to(1200.0)
print("steps", e.stats()["steps"], flush=True)
