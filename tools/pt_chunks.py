import os, sys
sys.path.insert(0, "/root/repo")
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
cfg = N.StcSingleConfig()
times = N.stc_protocol_times(N.StcProtocol.stet, cfg.t_onset_ms)
print("stim times", times[:3], times[-1], len(times))
e = Engine(N.build_stc_single(cfg, times), EngineOptions(cfg.dt_ms, 1))
e.set_timing(True)
t = 0.0
for k in range(48):
    s0 = e.stats(); t += 26214.4; e.advance_to(t); s1 = e.stats()
    print(f"{t/1000:7.1f}s  {1e3*(s1['advance_ms']-s0['advance_ms'])/(s1['steps']-s0['steps']):.3f} us/step  kern {1e3*(s1['epoch_kernel_ms']-s0['epoch_kernel_ms'])/(s1['steps']-s0['steps']):.3f}", flush=True)
