"""Config 2 (one 48-compartment neuron, 1,000 STC + STDP inputs, dt 0.1 ms) through
k_batch for an ncu capture:
  ncu --set full --import-source on -k regex:k_batch -s 2 -c 1 -o out python tools/prof_config2.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
rec = N.build_single_neuron_plastic(n_inputs=1000, rate_hz=5.0, duration_ms=3000.0, dt_ms=0.1)
e = Engine(rec.flatten(), EngineOptions(0.1, 1))
e.advance_to(float(os.environ.get("T_END", "500")))
print("steps", e.stats()["steps"], "kernel", e.stats()["stepping_kernel"])
