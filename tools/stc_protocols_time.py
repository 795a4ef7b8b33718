"""The stc-protocols experiment (experiments.cpp:262-289: 4 protocols x
TRIALS trials of run_stc_protocol, default 10) batched on one B200 vs the
reference (oracle/_ref), which runs the trials one after another on one core."""
import os, sys, time
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle")]
import ref
from paper_2411_16445_b200 import network as N
trials = int(os.environ.get("TRIALS", "10"))
cfg = N.StcSingleConfig()
protos = [N.StcProtocol.stet, N.StcProtocol.wtet, N.StcProtocol.slfs, N.StcProtocol.wlfs]
N.run_stc_protocols(cfg, [N.StcProtocol.wtet], 1)  # warm-up (context, modules)
t0 = time.perf_counter()
res = N.run_stc_protocols(cfg, protos, trials)
t1 = time.perf_counter()
same = True
for pi, p in enumerate(protos):
    for t in range(trials):
        h, z, prp = ref.run_stc_protocol(p, t)
        g = res[pi][t]
        same &= (g.h_final, g.z_final, g.p_final) == (h, z, prp)
t2 = time.perf_counter()
print(f"stc-protocols, 4 protocols x {trials} trials: b200 {t1 - t0:.2f} s, reference (one core, "
      f"sequential) {t2 - t1:.2f} s, every trial identical: {same}", flush=True)
