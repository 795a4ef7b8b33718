"""Wall time of the full 8 h consolidation protocol (network.cpp:600-639) on
config 3: the B200 engine vs the reference engine (oracle/_ref, all host
cores), per phase. Usage: python tools/protocol_8h_time.py"""
import os, sys, time
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import numpy as np
import ref
from test_gpu_builders import ref_cfg
from paper_2411_16445_b200 import network as N, Engine, EngineOptions

c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
t_recall = c.t_learn_ms + 8 * 3600e3
t_ff0 = c.t_learn_ms + 3000.0
t_ff1 = t_ff0 + np.floor((t_recall - 1000.0 - t_ff0) / c.coarse_dt_ms) * c.coarse_dt_ms
rr = ref.RefRecipe.consolidation(ref_cfg(c), True)
for name, mk in (("b200", lambda: Engine(rr.view, EngineOptions(dt_ms=c.dt_ms, seed=1))),
                 ("reference", lambda: ref.RefEngine(rr.view, c.dt_ms, 1, os.cpu_count() or 1))):
    e = mk()
    ts = [time.perf_counter()]
    e.advance_to(t_ff0); ts.append(time.perf_counter())
    e.fast_forward_to(t_ff1, c.coarse_dt_ms); ts.append(time.perf_counter())
    e.advance_to(t_recall + 500.0); ts.append(time.perf_counter())
    d = np.diff(ts)
    print(f"{name}: detailed 0-13 s {d[0]:.2f} s, fast-forward {d[1]:.2f} s, "
          f"recall {d[2]:.2f} s, total {ts[-1] - ts[0]:.2f} s", flush=True)
