"""Throughput of the consolidation network at other sizes (BASELINE configs:
the 4000-neuron target, config 5's 100k-cell network): build time, device
µs per fine step over 1 s of spontaneous activity, sim-s/wall-s and
compartment-updates/s.  SCALE_N cells (80 % excitatory), in-degree kept at
config 3's (p = 0.1 * 1600 / n_exc), SCALE_DEND=large for 48-compartment
cells (config 5)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
n = int(os.environ.get("SCALE_N", "4000"))
ne = n * 4 // 5
p = float(os.environ.get("SCALE_P", str(min(0.1, 0.1 * 1600 / ne))))
dend = N.DendriteSize.large_dendrites if os.environ.get("SCALE_DEND") == "large" else N.DendriteSize.small_dendrites
c = N.ConsolidationConfig(n_cells=n, n_exc=ne, p_conn=p, seed=1, multi_compartment=True, dend_size=dend)
t0 = time.time()
b = N.build_consolidation_network(c, True)
t1 = time.time()
e = Engine(b.recipe, EngineOptions(0.5, 1))
t2 = time.time()
e.set_timing(True)
e.advance_to(500.0)
s0 = e.stats()
e.advance_to(1500.0)
s1 = e.stats()
ms = s1["advance_ms"] - s0["advance_ms"]
steps = s1["steps"] - s0["steps"]
us = 1e3 * ms / steps
print(f"n={n} p={p:.4g} dend={'large' if dend == N.DendriteSize.large_dendrites else 'small'} "
      f"comps={s1['total_comps']} stc={s1['stc_synapses']} build_s={t1 - t0:.1f} engine_s={t2 - t1:.1f} "
      f"us_per_step={us:.2f} sim_s_per_wall_s={0.5e-3 / (us * 1e-6):.2f} "
      f"comp_updates_per_s={s1['total_comps'] / (us * 1e-6):.3g} spikes={len(e.spike_arrays()[0])}", flush=True)
