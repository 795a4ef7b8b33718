"""Locate the first divergence of k_warp from k_batch: both engines on the same
recipe, advanced one epoch at a time; after each, spikes and every cell's V,
species and STC h/z/c/|h-h0| are compared."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
n = int(os.environ.get("PROBE_N", "2000"))
ne = n * 4 // 5
c = N.ConsolidationConfig(n_cells=n, n_exc=ne, seed=1, multi_compartment=True,
                          t_learn_ms=float(os.environ.get("T_LEARN", "10000")))
b = N.build_consolidation_network(c, True)
flat = b.recipe.flatten()
os.environ["MCG_VERBOSE"] = "1"
ew = Engine(flat, EngineOptions(0.5, 1))
os.environ["MCG_NO_WARP"] = "1"
eb = Engine(flat, EngineOptions(0.5, 1))
del os.environ["MCG_NO_WARP"]
T = float(os.environ.get("T_END", "600"))
t = 0.0
def state(e, g):
    cv = e.cell(g)
    out = {"v": cv.v_mV}
    for i, s in enumerate(cv.species):
        out[f"sp{i}"] = s
    if g < ne:
        gr = cv.groups[0]
        out.update(h=gr.stc_h, z=gr.stc_z, c=gr.stc_c, a=gr.sps_abs)
    return out
while t < T:
    t += 3.0
    ew.advance_to(t)
    eb.advance_to(t)
    tw, gw = ew.spike_arrays()
    tb, gb = eb.spike_arrays()
    bad = None
    if len(tw) != len(tb) or not (np.array_equal(tw, tb) and np.array_equal(gw, gb)):
        bad = f"spikes {len(tw)} vs {len(tb)}"
    nbad = 0
    for g in range(n):
        sw, sb = state(ew, g), state(eb, g)
        for k in sw:
            if not np.array_equal(sw[k], sb[k]):
                i = int(np.nonzero(sw[k] != sb[k])[0][0])
                print(f"t={t} cell {g} field {k}[{i}]: warp {sw[k][i]!r} batch {sb[k][i]!r} "
                      f"(n diff {int(np.sum(sw[k] != sb[k]))})", flush=True)
                bad = bad or "state"
        if bad == "state":
            nbad += 1
            if nbad >= 4:
                break
    if bad:
        print("first divergence at t =", t, bad, flush=True)
        if len(tw) != len(tb):
            m = min(len(tw), len(tb))
            d = np.nonzero((tw[:m] != tb[:m]) | (gw[:m] != gb[:m]))[0]
            if len(d):
                i = d[0]
                print("first differing spike", i, tw[i], gw[i], "vs", tb[i], gb[i])
        break
else:
    print("no divergence through t =", T)
