"""k_point debugging: seed-0 point recipe of tests/test_gpu_point.py stepped
one fine step at a time through both engines; first V mismatch per cell."""
import os, sys
sys.path[:0] = [".", "oracle", "tests"]
import numpy as np
import ref
from paper_2411_16445_b200 import Engine, EngineOptions
import test_gpu_point as T
seed = int(os.environ.get("SEED", "0"))
rec = T._recipe(seed)
dt = [0.5, 0.2, 0.1, 0.25][seed % 4]
flat = rec.flatten()
print("cells", len(rec.cell_kind), "kinds", rec.cell_kind, "dt", dt)
for k in rec.kinds:
    m = k.membrane
    print(" kind: i_bg", m.i_bg_nA, "sigma", m.sigma_bg_nA_sqrt_ms, "quiet", m.bg_quiet_t0_ms, m.bg_quiet_t1_ms,
          "species", len(k.species), "stc count", k.placements[0].count)
r = ref.RefEngine(flat.view, dt, 7 + seed, 1)
g = Engine(flat, EngineOptions(dt, 7 + seed))
print("kernel", g.stats()["stepping_kernel"])
bad = set()
step = int(os.environ.get("CHUNK", "1"))
sched = [float(x) for x in os.environ["SCHED"].split(",")] if "SCHED" in os.environ else [s * step * dt for s in range(1, 80)]
for t in sched:
    r.advance_to(t); g.advance_to(t)
    for gid in range(len(rec.cell_kind)):
        a, b = r.read("v", gid)[0], g.cell(gid).v_mV[0]
        if a != b and gid not in bad:
            bad.add(gid)
            print(f"t {t} gid {gid}: ref {a!r} gpu {b!r}")
    print("t", t, "spikes", len(r.spike_arrays()[0]), len(g.spike_arrays()[0]), g.stats()["epochs"], g.stats()["kernel_launches"])
print("spikes", len(r.spike_arrays()[0]), len(g.spike_arrays()[0]))
