import sys; sys.path[:0]=['.']
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
cfg = N.StcSingleConfig()
times = N.stc_protocol_times(N.StcProtocol.stet, cfg.t_onset_ms)
rec = N.build_stc_single(cfg, times)
e = Engine(rec, EngineOptions(cfg.dt_ms, 1))
e.advance_to(2000.0)
