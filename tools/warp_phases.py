"""k_warp per-phase breakdown (MCG_PHASE_TIMING=1: lane 0 of every warp
accumulates clock64 deltas per phase; the engine prints µs per fine step per
warp, mean | max warp, after each advance_to).  PROBE_CFG=config1 | config3
(default) | config5 | n4000; PROBE_T = comma-separated advance_to targets (ms)."""
import os, sys
os.environ["MCG_PHASE_TIMING"] = "1"
os.environ.setdefault("MCG_VERBOSE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
cfgn = os.environ.get("PROBE_CFG", "config3")
if cfgn == "config1":
    cfg = N.StcSingleConfig()
    times = N.stc_protocol_times(N.StcProtocol.stet, cfg.t_onset_ms)
    rec = N.build_stc_single(cfg, times)
    e = Engine(rec, EngineOptions(cfg.dt_ms, 1))
    dflt = "2000,20000,200000"
else:
    n, dend = {"config3": (2000, 0), "config5": (100000, 1), "n4000": (4000, 0)}[cfgn]
    ne = n * 4 // 5
    c = N.ConsolidationConfig(n_cells=n, n_exc=ne, p_conn=min(0.1, 0.1 * 1600 / ne), seed=1,
                              multi_compartment=True,
                              dend_size=N.DendriteSize.large_dendrites if dend else N.DendriteSize.small_dendrites)
    e = Engine(N.build_consolidation_network(c, True).recipe, EngineOptions(0.5, 1))
    dflt = "100,300" if cfgn == "config5" else "1000,3000,10000,12000"
e.set_timing(True)
for t1 in [float(x) for x in os.environ.get("PROBE_T", dflt).split(",")]:
    s0 = e.stats()
    e.advance_to(t1)
    s1 = e.stats()
    print(f"window -> {t1:g} ms: {1e3 * (s1['advance_ms'] - s0['advance_ms']) / max(1, s1['steps'] - s0['steps']):.3f} us/step",
          file=sys.stderr, flush=True)
