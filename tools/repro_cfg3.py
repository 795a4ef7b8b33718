import sys
sys.path.insert(0, '/root/repo')
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
T = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
c = N.ConsolidationConfig(n_cells=n, n_exc=n * 4 // 5, pattern=min(150, n // 2), seed=1,
                          multi_compartment=True)
b = N.build_consolidation_network(c, True)
e = Engine(b.recipe, EngineOptions(0.5, 1))
e.advance_to(T)
print("ok", n, T, len(e.spike_arrays()[0]))
