import sys
sys.path.insert(0, '/root/repo')
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
b = N.build_consolidation_network(c, True)
e = Engine(b.recipe, EngineOptions(0.5, 1))
T = 0.0
while T < 2000:
    T += 25.0
    try:
        e.advance_to(T)
    except Exception as ex:
        print("FAILED at", T, ex); break
print("reached", T, len(e.spike_arrays()[0]) if T >= 2000 else -1, flush=True)
