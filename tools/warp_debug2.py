"""Per-step V of one cell (probe) in k_warp vs k_batch; prints the first step
where they differ and the cell's spikes / the network's spikes around it."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_16445_b200 import network as N, Engine, EngineOptions, ProbeSpec
cell = int(os.environ.get("CELL", "7"))
c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=1, multi_compartment=True)
b = N.build_consolidation_network(c, True)
NCOMP = int(os.environ.get("NCOMP", "1"))
b.recipe.probes = [ProbeSpec(gid=cell, comp=k, every_steps=1) for k in range(NCOMP)]
flat = b.recipe.flatten()
ew = Engine(flat, EngineOptions(0.5, 1))
os.environ["MCG_NO_WARP"] = "1"
eb = Engine(flat, EngineOptions(0.5, 1))
for e in (ew, eb):
    e.advance_to(float(os.environ.get("T_END", "24")))
for k in range(NCOMP):
    tw_, vw_ = ew.trace_arrays(k)
    tb_, vb_ = eb.trace_arrays(k)
    dd = np.nonzero(vw_ != vb_)[0]
    if NCOMP > 1 and len(dd):
        print(f"comp {k}: first differing step {dd[0]} warp {vw_[dd[0]]!r} batch {vb_[dd[0]]!r}")
tw, vw = ew.trace_arrays(0)
tb, vb = eb.trace_arrays(0)
d = np.nonzero(vw != vb)[0]
print("first differing step", d[0] if len(d) else None, "t", tw[d[0]] if len(d) else None)
if len(d):
    i = d[0]
    for k in range(max(0, i - 3), min(len(vw), i + 3)):
        print(f"  t={tw[k]:.1f} warp {vw[k]!r} batch {vb[k]!r} diff {vw[k]-vb[k]!r}")
st, sg = eb.spike_arrays()
print("cell spikes (batch):", st[sg == cell][:10])
# edges into the cell: which sources spiked and when they arrive
src = flat.recipe.connections.src if hasattr(flat.recipe, "connections") else None
t = b.recipe.connection_table()
into = np.nonzero(t.dst == cell)[0]
pre = set(int(x) for x in t.src[into][t.from_source[into] == 0])
arr = [(float(tt), int(g)) for tt, g in zip(st, sg) if int(g) in pre and tt < 30]
print("presynaptic spikes before 30 ms:", arr[:40])
import ctypes
ctypes.CDLL(None).fflush(None)  # device printf goes through C stdio
