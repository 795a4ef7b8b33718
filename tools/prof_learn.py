import sys
sys.path.insert(0, "/root/repo")
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
b = N.build_consolidation_network(c, True)
e = Engine(b.recipe, EngineOptions(0.5, 1))
e.advance_to(10400.0)
e.advance_to(10700.0)
print("steps", e.stats()["steps"], "launches", e.stats().get("kernel_launches"), flush=True)
