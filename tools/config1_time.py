"""Config 1 (run_stc_protocol, network.cpp:353-399): one STC synapse on a point
neuron, detailed through the stimulation then fast-forward to the evaluation
time. Wall time of the B200 engine vs the reference (oracle/_ref) per protocol."""
import os, sys, time
sys.path[:0] = [".", "oracle"]
import ref
from paper_2411_16445_b200 import network as N
cfg = N.StcSingleConfig()
N.run_stc_protocol(cfg, N.StcProtocol.stet, 0)  # warm-up (context, module load)
for p in ("stet", "wtet", "slfs", "wlfs"):
    pr = getattr(N.StcProtocol, p)
    t0 = time.perf_counter(); g = N.run_stc_protocol(cfg, pr, 0); t1 = time.perf_counter()
    h, z, _ = ref.run_stc_protocol(pr, 0); t2 = time.perf_counter()
    print(f"{p}: b200 {t1 - t0:.3f} s (z {g.z_final:.5f}), reference {t2 - t1:.3f} s (z {z:.5f})", flush=True)
