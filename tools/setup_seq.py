import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MCG_PROFILE_BUILD"] = "1"
import bench
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
import torch
torch.cuda.set_device(0)
bench.flush_l2()
for name, n, dend in (("c3", 2000, 0), ("t4000", 4000, 0), ("c5", 100000, 1), ("c5b", 100000, 1)):
    ne = n * 4 // 5
    c = N.ConsolidationConfig(n_cells=n, n_exc=ne, p_conn=min(0.1, 0.1 * 1600 / ne), seed=1, multi_compartment=True,
                              dend_size=N.DendriteSize.large_dendrites if dend else N.DendriteSize.small_dendrites)
    e = b = None; gc.collect()
    t0 = time.perf_counter()
    b = N.build_consolidation_network(c, True)
    t1 = time.perf_counter()
    e = Engine(b.recipe, EngineOptions(0.5, 1))
    t2 = time.perf_counter()
    e.advance_to(100.0)
    print(name, f"build {t1-t0:.3f} engine {t2-t1:.3f}", flush=True)
