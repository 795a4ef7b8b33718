"""Busyring (1024 HH cells, depth 2, dt 0.025 ms; BUSY_STDP=1: STDP on the
random synapses) through k_batch for an ncu capture:
  ncu --set full --import-source on -k regex:k_batch -s 2 -c 1 -o out python tools/prof_busyring.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
spec = N.default_busyring()
spec.stdp_on_random = os.environ.get("BUSY_STDP") == "1"
spec.ring_weight_uS = 0.050515121785495443  # calibrate_ring_weight(default spec), SURVEY §8(c) golden
e = Engine(N.build_busyring(spec), EngineOptions(spec.dt_ms, spec.seed))
e.advance_to(float(os.environ.get("T_END", "60")))
print("spikes", len(e.spike_arrays()[0]), "kernel", e.stats()["stepping_kernel"])
