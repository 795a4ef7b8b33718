"""Config 5 setup broken down: the device ER sampler (mcg_er_connect), the rest
of build_consolidation_network, flatten, and Engine construction (build_model,
uploads, kernel setup; MCG_PROFILE_BUILD=1 prints the engine's own parts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
n = int(os.environ.get("PROBE_N", "100000"))
c = N.ConsolidationConfig(n_cells=n, n_exc=n * 4 // 5, p_conn=min(0.1, 0.1 * 1600 / (n * 4 // 5)), seed=1,
                          multi_compartment=True, dend_size=N.DendriteSize.large_dendrites)
Engine  # context: the first CUDA call pays the context creation
import ctypes as C
er = N.er_pairs
T = {}
def timed_er(*a, **k):
    t = time.perf_counter(); r = er(*a, **k); T["er_pairs"] = time.perf_counter() - t; return r
N.er_pairs = timed_er
N.uniform_stream((1, 0, 0, 0), 0, 4)  # warm the device (context, module load)
for rep in ("first in process", "second"):
    t0 = time.perf_counter()
    b = N.build_consolidation_network(c, True)
    t1 = time.perf_counter()
    f = b.recipe.flatten()
    t2 = time.perf_counter()
    e = Engine(f, EngineOptions(0.5, 1))
    t3 = time.perf_counter()
    print(f"{rep}: er_pairs {T['er_pairs']:.3f}  builder rest {t1 - t0 - T['er_pairs']:.3f}  flatten {t2 - t1:.3f}  "
          f"Engine() {t3 - t2:.3f}  total {t3 - t0:.3f} s", flush=True)
    del e, f, b
