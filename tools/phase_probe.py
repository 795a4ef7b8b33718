"""Per-phase cycle breakdown of k_batch (MCG_PHASE_TIMING=1) over bio-time
windows of the config-3 workload; the engine prints cumulative totals (thread 0
of every CTA, summed over CTAs) after each advance_to, this prints the deltas
as µs per fine step per CTA."""
import os, re, sys, time, subprocess
if "--child" not in sys.argv:
    p = subprocess.run([sys.executable, __file__, "--child"] + sys.argv[1:], capture_output=True, text=True)
    print(p.stdout)
    wins = [l for l in p.stdout.splitlines() if l.startswith("window")]
    for tag in ("sum over CTAs", "CTA 0"):
        lines = [l for l in p.stderr.splitlines() if l.startswith(f"phase cycles ({tag})")]
        prev = None
        print(tag)
        for w, l in zip(wins, lines):
            v = [float(x.split(":")[1]) for x in l.split(":", 1)[1].split() if ":" in x]
            ctas = int(l.split("batches=")[1])
            d = v  # the engine resets its counters after every advance_to
            prev = v
            steps = int(w.split()[3])
            print(" ", w.split()[1], " ".join(f"{i}:{x / steps / ctas / 1965.0:.2f}" for i, x in enumerate(d) if x > 0))
    cta = [l for l in p.stderr.splitlines() if "per-CTA" in l or l.startswith("  CTA")]
    for w in range(len(cta) // 4):  # per window: summary + top 3 CTAs, cycles per step
        steps = int(wins[w].split()[3]) if w < len(wins) else 1
        print(wins[w].split()[1] if w < len(wins) else "", cta[4 * w])
        for l in cta[4 * w + 1:4 * w + 4]:
            head, rest = l.split(":", 1)
            vals = [x.split(":") for x in rest.split() if x.count(":") == 1]
            print("   ", head.strip(), " ".join(f"{i}:{float(x) / steps / 1965:.2f}" for i, x in vals if float(x) > 0))
    sys.exit(0)
os.environ["MCG_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16445_b200 import network as N, Engine, EngineOptions
n = int(os.environ.get("PROBE_N", "2000"))
ne = n * 4 // 5
dend = N.DendriteSize.large_dendrites if os.environ.get("PROBE_DEND") == "large" else N.DendriteSize.small_dendrites
c = N.ConsolidationConfig(n_cells=n, n_exc=ne, p_conn=min(0.1, 0.1 * 1600 / ne), seed=1,
                          multi_compartment=True, dend_size=dend)
if os.environ.get("PROBE_CFG") == "config1":
    cfg = N.StcSingleConfig()
    times = N.stc_protocol_times(N.StcProtocol.stet, cfg.t_onset_ms)
    rec = N.build_stc_single(cfg, times)
    e = Engine(rec.flatten() if hasattr(rec, "flatten") else rec, EngineOptions(cfg.dt_ms, 1))
elif os.environ.get("PROBE_CFG") == "config2":
    rec = N.build_single_neuron_plastic(n_inputs=1000, rate_hz=5.0, duration_ms=3000.0, dt_ms=0.1)
    e = Engine(rec.flatten(), EngineOptions(0.1, 1))
else:
    b = N.build_consolidation_network(c, True)
    e = Engine(b.recipe, EngineOptions(0.5, 1))
ctas = e.stats().get("batch_grid", 143)
for t1 in [float(x) for x in os.environ.get("PROBE_T", "1000,3000,10000,12000").split(",")]:
    s0 = e.stats()["steps"]
    a = time.time(); e.advance_to(t1); w = time.time() - a
    st = e.stats()["steps"] - s0
    print(f"window {t1:.0f} steps {st} {ctas} wall_us_per_step {1e6 * w / st:.2f}", flush=True)
