"""k_warp vs k_batch (MCG_NO_WARP=1) on the consolidation workloads: µs per fine
step over bio-time windows (engine CUDA events) and the spike trains of both
kernels compared.  PROBE_N cells (default 2000), PROBE_DEND=large, PROBE_T."""
import os, subprocess, sys
if "--child" in sys.argv:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    from paper_2411_16445_b200 import network as N, Engine, EngineOptions
    n = int(os.environ.get("PROBE_N", "2000"))
    ne = n * 4 // 5
    dend = N.DendriteSize.large_dendrites if os.environ.get("PROBE_DEND") == "large" else N.DendriteSize.small_dendrites
    c = N.ConsolidationConfig(n_cells=n, n_exc=ne, p_conn=min(0.1, 0.1 * 1600 / ne), seed=1,
                              multi_compartment=True, dend_size=dend)
    b = N.build_consolidation_network(c, True)
    e = Engine(b.recipe, EngineOptions(0.5, 1))
    e.set_timing(True)
    out = []
    for t1 in [float(x) for x in os.environ.get("PROBE_T", "1000,3000,10000,12000").split(",")]:
        s0 = e.stats()
        e.advance_to(t1)
        s1 = e.stats()
        out.append(f"{t1/1000:g}s:{1e3 * (s1['advance_ms'] - s0['advance_ms']) / (s1['steps'] - s0['steps']):.2f}")
    t, g = e.spike_arrays()
    np.save(sys.argv[-1], np.stack([t, g.astype(np.float64)]))
    hz = e.cell(0).groups[0].stc_h if c.n_exc > 0 else np.zeros(1)
    print("us/step", " ".join(out), "spikes", len(t), "h0", float(hz.sum()), flush=True)
    sys.exit(0)
import numpy as np
res = {}
for tag, env in (("k_warp", {}), ("k_batch", {"MCG_NO_WARP": "1"})):
    f = f"/tmp/ab_{tag}.npy"
    r = subprocess.run([sys.executable, __file__, "--child", f], env={**os.environ, **env, "MCG_VERBOSE": "1"},
                       capture_output=True, text=True)
    print(tag, r.stdout.strip(), r.stderr.strip()[-600:], flush=True)
    res[tag] = np.load(f) if os.path.exists(f) else None
a, b = res["k_warp"], res["k_batch"]
if a is not None and b is not None:
    same = a.shape == b.shape and np.array_equal(a, b)
    print("spike trains identical:", same, a.shape, b.shape)
