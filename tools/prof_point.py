"""Config 1 (STET, one point cell, one STC synapse) through k_point for an ncu
capture:  ncu --set full --import-source on -k regex:k_point -s 1 -c 1 -o out python tools/prof_point.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
cfg = N.StcSingleConfig()
times = N.stc_protocol_times(N.StcProtocol.stet, cfg.t_onset_ms)
e = Engine(N.build_stc_single(cfg, times), EngineOptions(cfg.dt_ms, 1))
e.set_timing(True)
e.advance_to(float(os.environ.get("T_END", "60000")))
s = e.stats()
print("us_per_step", 1e3 * s["advance_ms"] / s["steps"], "kernel", s["stepping_kernel"])
