"""µs per fine step of the config-3 network (or PROBE_N cells) over bio-time
windows, device-timed by the engine (advance_ms); MCG_LIB selects the library."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
n = int(os.environ.get("PROBE_N", "2000"))
c = N.ConsolidationConfig(n_cells=n, n_exc=n * 4 // 5, seed=1, multi_compartment=True)
b = N.build_consolidation_network(c, True)
e = Engine(b.recipe, EngineOptions(0.5, 1))
e.set_timing(True)
out = []
for t1 in (1000.0, 3000.0, 10000.0, 12000.0):
    s0 = e.stats()
    e.advance_to(t1)
    s1 = e.stats()
    out.append(f"{t1/1000:.0f}s:{1e3 * (s1['advance_ms'] - s0['advance_ms']) / (s1['steps'] - s0['steps']):.2f}")
print(os.environ.get("MCG_LIB", "libmcg.so").split("/")[-1], "us/step", " ".join(out), "spikes", len(e.spike_arrays()[0]), flush=True)
