import os, sys, time
os.environ["MCG_PHASE_TIMING"] = "1"
sys.path.insert(0, '/root/repo')
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
b = N.build_consolidation_network(c, True)
e = Engine(b.recipe, EngineOptions(0.5, 1))
e.advance_to(1000.0)
t = time.time(); e.advance_to(3000.0); print("wall", time.time() - t, e.stats()["steps"], flush=True)
