import sys; sys.path.insert(0, ".")
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
rec = N.build_single_neuron_plastic(n_inputs=1000, rate_hz=5.0, duration_ms=3000.0, dt_ms=0.1)
e = Engine(rec.flatten(), EngineOptions(0.1, 1)); e.set_timing(True); e.advance_to(500.0); s0=e.stats(); e.advance_to(2500.0); s1=e.stats()
ms=s1["advance_ms"]-s0["advance_ms"]; print("config2 sim-s/wall-s", 2000.0/ms, "us/step", 1e3*ms/(s1["steps"]-s0["steps"]))
