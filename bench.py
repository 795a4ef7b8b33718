#!/usr/bin/env python3
"""Benchmark: simulated-seconds per wall-second of the cable-cell integration
loop (Engine::advance_to) on BASELINE.json configs[2] / SURVEY §8(d) config 3:
the 2000-neuron multi-compartment (31 comps) recurrent network with synaptic
tagging and capture, seed 1, dt 0.5 ms, 8-hour protocol (learning at 10 s).

A step = 500 ms of biological time of that protocol (1000 fine steps), in
order from t = 0: W warm-up steps, then K timed steps (defaults cover the
spontaneous phase and the onset of the 100 Hz learning stimulus at 10 s).

  value   sim-s/wall-s, device-timed (CUDA events on the engine's stream),
          network state resident in HBM
  e2e     same metric through the public API with host buffers: engine
          construction from the host recipe (H2D), advance over the W+K steps,
          spikes and final STC weights back to the host (D2H), wall-clocked
  roofline  the persistent stepping kernel the engine picked (k_warp for the
          consolidation networks, else k_batch; one launch = up to 32
          min-delay epochs): algorithmic bytes per launch (SURVEY §8(d) B_step
          x fine steps per launch) / mean launch duration (CUDA events on the
          engine's stream around each launch)
  cpu_baseline  the reference engine (oracle/_ref, compiled from
          /root/reference) on the same recipe, all host threads, bounded sample

`--impl reference` times the reference's own CPU engine on the same workload
(rank 0 only) and prints the same JSON line with "impl": "reference".
"""
import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

STEP_MS = 500.0
DT_MS = 0.5
SEED = 1
N_CELLS, N_EXC = 2000, 1600
METRIC = "simulated s per wall s (consolidation network, fine steps)"
# both arms run the reference's build_consolidation_network recipe (seed 1); the
# GPU arm builds it with this repo's port (network.py), pinned equal to the
# reference builder's recipe at N = 300, 2000 and 4000 (tests/test_gpu_builders.py,
# tests/test_gpu_configs.py), the reference arm with the reference's own builder
DATA_NOTE = "synthetic: build_consolidation_network(config 3, seed 1) recipe"
UNIT = "sim-s/wall-s"


def data_note(n_gpus=1):
    if n_gpus <= 1:
        return DATA_NOTE
    nc, _, p = workload_size(n_gpus)
    return f"synthetic: build_consolidation_network(N={nc}, p={p:g}, seed 1) recipe"


def workload_size(n_gpus=1):
    """Weak-scaling family of the consolidation network: 2000 N cells over N
    GPUs with p = 0.1 / N, so every excitatory cell keeps config 3's in-degree
    (160 recurrent STC synapses).  N = 1 is config 3 itself; N = 2 is the
    north-star 4,000-neuron network; N = 50 would be config 5's cell count."""
    n = max(1, int(n_gpus))
    return N_CELLS * n, N_EXC * n, 0.1 / n


def workload_config(n_gpus=1):
    from paper_2411_16445_b200 import network as N
    nc, ne, p = workload_size(n_gpus)
    return N.ConsolidationConfig(n_cells=nc, n_exc=ne, p_conn=p, seed=SEED, multi_compartment=True,
                                 dt_ms=DT_MS)


L2_NOTE = ("GPU arm: a 256 MB buffer is written between timed steps (flushes the 126 MB L2); "
           "reference arm: host CPU, no device cache")


def config_block(n_gpus):
    """Identical in both arms (the driver compares them)."""
    if n_gpus <= 1:
        return {"workload": "config3: consolidation network N=2000 (1600 MC exc x 31 comps + 400 point inh), "
                            "p=0.1, STC synapses, seed 1, dt 0.5 ms, 8h protocol, step = 500 ms bio",
                "n_cells": N_CELLS, "compartments": 50000, "dt_ms": DT_MS, "step_bio_ms": STEP_MS,
                "parallelism": "single GPU", "l2": L2_NOTE}
    nc, ne, p = workload_size(n_gpus)
    return {"workload": f"config3 weak-scaled x{n_gpus}: consolidation network N={nc} ({ne} MC exc x 31 comps "
                        f"+ {nc - ne} point inh), p={p:g} (config 3's in-degree), STC synapses, seed 1, "
                        "dt 0.5 ms, 8h protocol, step = 500 ms bio",
            "n_cells": nc, "compartments": 31 * ne + (nc - ne), "dt_ms": DT_MS, "step_bio_ms": STEP_MS,
            "parallelism": f"cells sharded over {n_gpus} GPUs (contiguous gid ranges), spikes exchanged "
                           "once per min-delay epoch by an allgather",
            "l2": L2_NOTE}


def host_facts():
    """CPU model and glibc of the host the CPU figures were taken on."""
    model = "?"
    try:
        with open("/proc/cpuinfo") as f:
            model = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), "?")
    except OSError:
        pass
    try:
        libc = os.confstr("CS_GNU_LIBC_VERSION")
    except (ValueError, OSError):
        libc = "?"
    return {"cpu_model": model, "glibc": libc, "host_threads": os.cpu_count() or 1}


def ref_workload_recipe(n_gpus=1):
    """The workload's recipe from the REFERENCE's own builder
    (build_consolidation_network, network.cpp:426-598, in oracle/_ref): the
    reference arm never maps this repo's library."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref
    nc, ne, p = workload_size(n_gpus)
    cfg = ref.default_consolidation(n_cells=nc, n_exc=ne, p_conn=p, seed=SEED, multi_compartment=1,
                                    dt_ms=DT_MS)
    return ref.RefRecipe.consolidation(cfg, True)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


KERNELS = {0: "k_batch", 1: "k_warp", 2: "k_point"}


def stepping_kernel(st):
    return KERNELS.get(int(st.get("stepping_kernel", 0)), "k_batch")


def traffic_per_launch(steps_per_launch, kernel="k_batch"):
    """DRAM bytes (read + write) of one launch of the stepping kernel from the
    committed ncu capture (profiles/<kernel>_dram.json), scaled to the mean
    launch's fine steps so it is per launch like `achieved`."""
    p = os.path.join(ROOT, "profiles", f"{kernel}_dram.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["dram_bytes_per_launch"] * steps_per_launch / d["fine_steps_in_launch"]
    except Exception:
        return None


def algorithmic_bytes_per_step(st, events_per_step):
    """B_step = 16 sum C + 16 S sum C_s + 64 N_stc + 48 C_hh
    + 16 K_active + 36 sum C_unique + 32 E_step + 24 N_cells (K_active, C_unique = 0 here)."""
    return (16 * st["total_comps"] + 16 * st["species_comps"] + 64 * st["stc_synapses"]
            + 48 * st["hh_comps"] + 32 * events_per_step + 24 * N_CELLS)


def flush_l2():
    import torch
    buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    buf.fill_(1.0)
    torch.cuda.synchronize()
    del buf


def cpu_baseline(recipe_view, sample_ms, sample_ms_1w):
    """Reference engine (oracle/_ref) on the host cores, bounded samples: all
    host threads (the headline CPU figure) and one worker."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref
    cores = os.cpu_count() or 1
    e = ref.RefEngine(recipe_view, DT_MS, SEED, cores)
    t0 = time.perf_counter()
    e.advance_to(sample_ms)
    w = time.perf_counter() - t0
    del e
    e1 = ref.RefEngine(recipe_view, DT_MS, SEED, 1)
    t0 = time.perf_counter()
    e1.advance_to(sample_ms_1w)
    w1 = time.perf_counter() - t0
    del e1
    return {"value": (sample_ms * 1e-3) / w, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"config3 recipe, advance 0 -> {sample_ms:.0f} ms bio, workers={cores}",
            "one_worker": {"value": (sample_ms_1w * 1e-3) / w1, "unit": UNIT, "cores": 1,
                           "sample": f"advance 0 -> {sample_ms_1w:.0f} ms bio, workers=1"},
            **host_facts()}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    rr = ref_workload_recipe(args.gpus)
    import ref
    cores = os.cpu_count() or 1
    e = ref.RefEngine(rr.view, DT_MS, SEED, cores)
    t = 0.0
    for _ in range(args.warmup):
        t += STEP_MS
        e.advance_to(t)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        t += STEP_MS
        e.advance_to(t)
    wall = time.perf_counter() - t0
    val = args.steps * STEP_MS * 1e-3 / wall
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": data_note(args.gpus),
            "config": config_block(args.gpus),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": f"steps {args.warmup}..{args.warmup + args.steps} of 500 ms bio, "
                                       f"workers={cores}", **host_facts()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def other_configs():
    """Secondary measurements of the same run (not the headline): the
    north-star 4000-neuron network, config 5 (100k cells x 48 comps, in-degree
    of config 3) on one GPU with its HBM roofline, and the acceptance-3
    pairing curve (gb_dp_curve, 13 deltas x 4000 trials, dt 0.05 ms) on the
    device.  Device-timed (engine CUDA events) over a window after warm-up."""
    import time as _t
    from paper_2411_16445_b200 import Engine, EngineOptions
    from paper_2411_16445_b200 import network as N
    from paper_2411_16445_b200 import protocols as PR
    out = {}
    peak, _ = measured_peak_hbm()
    for name, n, dend, t_warm, t_end in (("target_4000", 4000, N.DendriteSize.small_dendrites, 500.0, 2500.0),
                                         ("config5_100k", 100000, N.DendriteSize.large_dendrites, 100.0, 600.0)):
        ne = n * 4 // 5
        c = N.ConsolidationConfig(n_cells=n, n_exc=ne, p_conn=min(0.1, 0.1 * 1600 / ne), seed=SEED,
                                  multi_compartment=True, dend_size=dend, dt_ms=DT_MS)
        e = b = None  # the previous configuration's engine and recipe released first
        gc.collect()
        t0 = _t.perf_counter()
        b = N.build_consolidation_network(c, True)
        e = Engine(b.recipe, EngineOptions(DT_MS, SEED))
        setup = _t.perf_counter() - t0
        e.set_timing(True)
        e.advance_to(t_warm)
        s0 = e.stats()
        e.advance_to(t_end)
        s1 = e.stats()
        sec = (s1["advance_ms"] - s0["advance_ms"]) * 1e-3
        steps = s1["steps"] - s0["steps"]
        ev = (s1["events_delivered"] - s0["events_delivered"]) / max(steps, 1)
        bstep = (16 * s1["total_comps"] + 16 * s1["species_comps"] + 64 * s1["stc_synapses"]
                 + 48 * s1["hh_comps"] + 32 * ev + 24 * n)
        ach = bstep * steps / sec / 1e9
        out[name] = {"n_cells": n, "compartments": s1["total_comps"], "stc_synapses": s1["stc_synapses"],
                     "p_conn": c.p_conn, "bio_ms": t_end - t_warm,
                     "sim_s_per_wall_s": (t_end - t_warm) * 1e-3 / sec,
                     "us_per_fine_step": 1e6 * sec / steps,
                     "compartment_updates_per_s": s1["total_comps"] * steps / sec,
                     "faster_than_real_time": (t_end - t_warm) * 1e-3 / sec > 1.0,
                     "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                                  "frac": ach / peak, "bytes_per_fine_step": bstep},
                     "setup_s": setup}
        e.close()
        del b
    # config 2: one MC neuron, 1000 Poisson inputs (5 Hz) onto STC + STDP synapses, dt 0.1 ms
    rec = N.build_single_neuron_plastic(n_inputs=1000, rate_hz=5.0, duration_ms=3000.0, dt_ms=0.1)
    e = Engine(rec.flatten(), EngineOptions(0.1, SEED))
    e.set_timing(True)
    e.advance_to(500.0)
    s0 = e.stats()
    e.advance_to(2500.0)
    s1 = e.stats()
    sec = (s1["advance_ms"] - s0["advance_ms"]) * 1e-3
    steps = s1["steps"] - s0["steps"]
    out["config2_single_neuron_1000"] = {"inputs": 1000, "dt_ms": 0.1, "bio_ms": 2000.0,
                                         "sim_s_per_wall_s": 2.0 / sec,
                                         "us_per_fine_step": 1e6 * sec / steps}
    e.close()
    # the whole 8 h experiment on config 3 (network.cpp:600-639): detailed to 13 s,
    # fast-forward across 8 h in 1 s coarse steps, recall; wall clock per phase
    c = N.ConsolidationConfig(n_cells=2000, n_exc=1600, seed=SEED, multi_compartment=True,
                              dt_ms=DT_MS)
    b = N.build_consolidation_network(c, True)
    e = Engine(b.recipe, EngineOptions(DT_MS, SEED))
    t_recall = c.t_learn_ms + 8 * 3600e3
    t_ff0 = c.t_learn_ms + 3000.0
    t_ff1 = t_ff0 + math.floor((t_recall - 1000.0 - t_ff0) / c.coarse_dt_ms) * c.coarse_dt_ms
    ts = [_t.perf_counter()]
    e.advance_to(t_ff0)
    ts.append(_t.perf_counter())
    e.fast_forward_to(t_ff1, c.coarse_dt_ms)
    ts.append(_t.perf_counter())
    e.advance_to(t_recall + 500.0)
    ts.append(_t.perf_counter())
    n_coarse = int(round((t_ff1 - t_ff0) / c.coarse_dt_ms))
    out["config3_8h_protocol"] = {"detailed_0_13s_s": ts[1] - ts[0], "fast_forward_s": ts[2] - ts[1],
                                  "recall_s": ts[3] - ts[2], "total_s": ts[3] - ts[0],
                                  "coarse_steps": n_coarse,
                                  "us_per_coarse_step": 1e6 * (ts[2] - ts[1]) / n_coarse,
                                  "spikes": int(len(e.spike_arrays()[0]))}
    e.close()
    del b
    out["busyring"] = busyring_configs()
    p = PR.GbParams()
    deltas = [-100.0, -50.0, -30.0, -20.0, -10.0, -5.0, 0.0, 5.0, 10.0, 20.0, 30.0, 50.0, 100.0]
    proto = PR.GbPairingProtocol(dt_ms=0.05, trials=4000, seed=999)
    import torch
    torch.cuda.synchronize()
    t0 = _t.perf_counter()
    curve = [PR.gb_dp_curve(p, [d], proto)[0] for d in deltas]  # acceptance.cpp:131
    wall = _t.perf_counter() - t0
    n_steps = int(math.ceil((100.0 + 100.0 + 60 * 1000.0 + 5000.0) / 0.05))
    out["gb_dp_curve_acceptance3"] = {"deltas": len(deltas), "trials": proto.trials, "dt_ms": proto.dt_ms,
                                      "wall_s": wall,
                                      "trial_steps_per_s": len(deltas) * proto.trials * n_steps / wall,
                                      "mean_change": [pt.mean_change for pt in curve]}
    out["config1_stc_protocols"] = stc_protocols_config()
    return out


def stc_protocols_config(trials=10):
    """Config 1 as the reference runs it: the stc-protocols experiment
    (experiments.cpp:262-289; 4 protocols x 10 trials of run_stc_protocol, the
    single STC synapse on a point neuron, each trial to 5 h with fast-forward).
    B200: trials as cells of one engine per protocol (network.run_stc_protocols);
    reference: oracle/_ref, the trials one after another on one core, as the
    experiment does.  Wall clock, both including engine construction."""
    import time as _t
    from paper_2411_16445_b200 import network as N
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref
    cfg = N.StcSingleConfig()
    protos = [N.StcProtocol.stet, N.StcProtocol.wtet, N.StcProtocol.slfs, N.StcProtocol.wlfs]
    N.run_stc_protocols(cfg, [N.StcProtocol.wtet], 1)  # module load, context
    t0 = _t.perf_counter()
    res = N.run_stc_protocols(cfg, protos, trials)
    t1 = _t.perf_counter()
    same = True
    for pi, p in enumerate(protos):
        for t in range(trials):
            h, z, prp = ref.run_stc_protocol(p, t)
            g = res[pi][t]
            same = same and (g.h_final, g.z_final, g.p_final) == (h, z, prp)
    t2 = _t.perf_counter()
    return {"protocols": 4, "trials": trials, "wall_s": t1 - t0,
            "reference": {"wall_s": t2 - t1, "kind": "reference (oracle/_ref)", "cores": 1},
            "speedup_vs_reference": (t2 - t1) / (t1 - t0), "every_trial_identical": same,
            "mean_z": [sum(r.z_final for r in row) / trials for row in res]}


BUSYRING_W = 0.050515121785495443  # SURVEY §8(c) golden: calibrated ring weight (bench.cpp:105-132)


def busyring_configs():
    """The HH + STDP workload (bench.cpp:134-194, run_bench_once): 1024 HH
    cells with depth-2 dendritic trees, rings of 4, 1000 zero-weight random
    synapses per cell, dt 0.025 ms, 200 ms; without and with STDP on the
    random synapses.  Both engines run the reference builder's recipe
    (oracle/_ref); setup and propagation are timed separately as run_bench
    does: device time (CUDA events) and wall for this library, wall for the
    reference with all host threads.  Spike counts of the two engines are
    reported side by side (the parity tests check the trains bitwise)."""
    import time as _t
    from paper_2411_16445_b200 import Engine, EngineOptions
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref
    cores = os.cpu_count() or 1
    out = {}
    for name, stdp in (("busyring_1024_d2", 0), ("busyring_1024_d2_stdp", 1)):
        rr = ref.RefRecipe.busyring(ref.default_busyring(ring_weight_uS=BUSYRING_W, stdp_on_random=stdp))
        view = rr.view
        t0 = _t.perf_counter()
        e = Engine(view, EngineOptions(0.025, 0), device=0)
        setup = _t.perf_counter() - t0
        e.set_timing(True)
        s0 = e.stats()
        t1 = _t.perf_counter()
        e.advance_to(200.0)
        prop_wall = _t.perf_counter() - t1
        s1 = e.stats()
        dev_s = (s1["advance_ms"] - s0["advance_ms"]) * 1e-3
        steps = s1["steps"] - s0["steps"]
        nsp = int(len(e.spike_arrays()[0]))
        comps = s1["total_comps"]
        e.close()
        t0 = _t.perf_counter()
        r = ref.RefEngine(view, 0.025, 0, cores)
        r_setup = _t.perf_counter() - t0
        t1 = _t.perf_counter()
        r.advance_to(200.0)
        r_prop = _t.perf_counter() - t1
        r_nsp = int(len(r.spike_arrays()[0]))
        del r
        out[name] = {"cells": 1024, "compartments": comps, "synapses": s1["total_synapses"],
                     "hh_comps": s1["hh_comps"], "bio_ms": 200.0, "dt_ms": 0.025, "steps": steps,
                     "prop_device_s": dev_s, "prop_wall_s": prop_wall, "setup_s": setup,
                     "us_per_fine_step": 1e6 * dev_s / max(steps, 1),
                     "compartment_updates_per_s": comps * steps / dev_s,
                     "spikes": nsp,
                     "reference": {"prop_wall_s": r_prop, "setup_s": r_setup, "workers": cores,
                                   "spikes": r_nsp, "kind": "reference (oracle/_ref)"},
                     "prop_speedup_vs_reference": r_prop / prop_wall}
        del rr
    return out


def run_gpu_arm(args):
    import numpy as np
    import torch
    from paper_2411_16445_b200 import Engine, EngineOptions
    from paper_2411_16445_b200 import network as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        return run_gpu_arm_sharded(args, world, rank)
    torch.cuda.set_device(0)
    cfg = workload_config()
    b = N.build_consolidation_network(cfg, True)
    flat = b.recipe.flatten()

    # ---- device-resident timing ----
    eng = Engine(flat, EngineOptions(DT_MS, SEED), device=0)
    eng.set_timing(True)
    t = 0.0
    for _ in range(args.warmup):
        t += STEP_MS
        eng.advance_to(t)
    flush_l2()
    s0 = eng.stats()
    clocks = ClockSampler(0)
    clocks.start()
    # device time of each step: the engine's own CUDA events around every
    # epoch kernel plus a host-synchronized bracket around the whole step
    wall_steps = []
    for _ in range(args.steps):
        flush_l2()
        torch.cuda.synchronize()
        a = time.perf_counter()
        t += STEP_MS
        eng.advance_to(t)   # returns after the step's last epoch completed
        wall_steps.append(time.perf_counter() - a)
    clk = clocks.stop()
    s1 = eng.stats()
    # device time: CUDA events recorded on the engine's stream around each
    # advance_to (mcg_stats.advance_ms); the wall bracket is reported beside it
    total = (s1["advance_ms"] - s0["advance_ms"]) * 1e-3
    wall_total = sum(wall_steps)
    value = args.steps * STEP_MS * 1e-3 / total
    n_launch = s1["epoch_kernel_launches"] - s0["epoch_kernel_launches"]
    kern_ms = s1["epoch_kernel_ms"] - s0["epoch_kernel_ms"]
    fine_steps = s1["steps"] - s0["steps"]
    ev_per_step = (s1["events_delivered"] - s0["events_delivered"]) / max(fine_steps, 1)
    bstep = algorithmic_bytes_per_step(s1, ev_per_step)
    steps_per_launch = fine_steps / max(n_launch, 1)
    per_launch_bytes = bstep * steps_per_launch
    mean_launch_s = kern_ms * 1e-3 / max(n_launch, 1)
    peak, peak_kind = measured_peak_hbm()
    achieved = per_launch_bytes / mean_launch_s / 1e9
    launches = s1["kernel_launches"] - s0["kernel_launches"]

    # ---- end to end through the public API, host buffers ----
    e2e_times = []
    e2e_parts = []
    h2d = d2h = 0
    for _ in range(3):  # best of three (one-shot host timings are noisy)
        torch.cuda.synchronize()
        a = time.perf_counter()
        eng2 = Engine(flat, EngineOptions(DT_MS, SEED), device=0)
        b1 = time.perf_counter()
        tt = 0.0
        for _ in range(args.warmup + args.steps):
            tt += STEP_MS
            eng2.advance_to(tt)
        b2 = time.perf_counter()
        st, sg = eng2.spike_arrays()
        hz = [eng2.cell(g).groups[0].stc_h for g in range(0, N_EXC, 1)]
        e2e_times.append(time.perf_counter() - a)
        e2e_parts.append({"construct_s": b1 - a, "advance_s": b2 - b1,
                          "read_back_s": e2e_times[-1] - (b2 - a)})
        d2h = st.nbytes + sg.nbytes + sum(h.nbytes for h in hz)
        v = flat.view
        h2d = (v.n_connections * (1 + 4 + 4 + 4 + 1 + 8 + 8)
               + s1["total_synapses"] * 8 * 12 + s1["total_comps"] * 8 * 5)
        eng2.close()
    e2e_val = (args.warmup + args.steps) * STEP_MS * 1e-3 / min(e2e_times)
    nsteps_e2e = args.warmup + args.steps

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(flat.view, args.cpu_sample_ms, args.cpu_sample_ms_1w)

    other = None if args.no_other else other_configs()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA_NOTE,
        "config": config_block(world),
        "compartment_updates_per_s": 50000 * fine_steps / total,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_per_launch(steps_per_launch, stepping_kernel(s1)),
                     "kernel": stepping_kernel(s1), "peak_kind": peak_kind,
                     "bytes_per_launch": per_launch_bytes, "mean_launch_ms": mean_launch_s * 1e3,
                     "steps_per_launch": steps_per_launch, "bytes_per_fine_step": bstep},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d / nsteps_e2e),
                "d2h_bytes_per_step": int(d2h / nsteps_e2e),
                "best_of": len(e2e_times),
                "parts": e2e_parts[int(np.argmin(e2e_times))]},
        "gpu_launches": int(launches),
        "clocks": clk,
        "stepping_kernel_share": kern_ms * 1e-3 / total,
        "wall_ms_per_step": 1e3 * wall_total / args.steps,
        "other_configs": other,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu_arm_sharded(args, world, rank):
    """N > 1: the weak-scaling family (workload_size: 2000 N cells, config 3's
    in-degree) partitioned over the ranks, one process per GPU.  The exchange
    runs inside libmcg (mcg_shard_init_nccl + mcg_shard_advance_to): per
    min-delay epoch one stepping launch and one ncclAllGather of the spike
    blocks on the engine's stream, the host waiting once per 32 epochs
    (engine.cpp:913-942 is the reference's epoch/exchange contract).  Timed
    with the engine's CUDA events around each advance (exchange included),
    max over ranks.  MCG_EXCHANGE=gloo runs the host-staged ShardedEngine
    instead (several ranks sharing one GPU; wall-clocked)."""
    import torch
    import torch.distributed as dist
    from paper_2411_16445_b200 import Engine, EngineOptions
    from paper_2411_16445_b200 import network as N
    from paper_2411_16445_b200 import shard

    local = int(os.environ.get("LOCAL_RANK", rank))
    backend = os.environ.get("MCG_EXCHANGE", "nccl")
    n_dev = torch.cuda.device_count()
    device = local % max(n_dev, 1)
    torch.cuda.set_device(device)
    dist.init_process_group(backend, rank=rank, world_size=world)
    coll_dev = "cuda" if backend == "nccl" else "cpu"
    b = N.build_consolidation_network(workload_config(world), True, device=device)
    flat = b.recipe.flatten()
    opt = EngineOptions(DT_MS, SEED)

    def make(rec=None):
        rec = flat if rec is None else rec
        if backend == "nccl":
            e = Engine(rec, opt, device=device, rank=rank, world=world)
            uid = torch.zeros(128, dtype=torch.uint8, device=coll_dev)
            if rank == 0:
                uid.copy_(torch.tensor(list(Engine.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, 0)
            e.init_nccl(bytes(uid.cpu().tolist()))
            return e, e.shard_advance_to, e.global_spike_arrays
        sh = shard.ShardedEngine(rec, opt, rank, world, device=device, backend=backend,
                                 record_spikes=True)
        return sh.engine, sh.advance_to, sh.spike_arrays

    eng, adv, spikes = make()
    eng.set_timing(True)
    t = 0.0
    for _ in range(args.warmup):
        t += STEP_MS
        adv(t)
    flush_l2()
    s0 = eng.stats()
    clocks = ClockSampler(device) if rank == 0 else None
    if clocks:
        clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        t += STEP_MS
        adv(t)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    dist.barrier()
    clk = clocks.stop() if clocks else None
    s1 = eng.stats()
    # device time: the engine's CUDA events around every advance call (the
    # in-library path); the gloo path stages through the host: wall clock
    dev_s = (s1["advance_ms"] - s0["advance_ms"]) * 1e-3 if backend == "nccl" else wall
    el = torch.tensor([dev_s], dtype=torch.float64, device=coll_dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    total = float(el.item())
    value = args.steps * STEP_MS * 1e-3 / total
    fine_steps = s1["steps"] - s0["steps"]
    n_launch = s1["epoch_kernel_launches"] - s0["epoch_kernel_launches"]
    kern_ms = s1["epoch_kernel_ms"] - s0["epoch_kernel_ms"]
    ev_per_step = (s1["events_delivered"] - s0["events_delivered"]) / max(fine_steps, 1)
    bstep = algorithmic_bytes_per_step(s1, ev_per_step)  # this rank's share
    steps_per_launch = fine_steps / max(n_launch, 1)
    mean_launch_s = kern_ms * 1e-3 / max(n_launch, 1)
    peak, peak_kind = measured_peak_hbm()
    achieved = bstep * steps_per_launch / max(mean_launch_s, 1e-12) / 1e9
    comps = torch.tensor([float(s1["total_comps"])], dtype=torch.float64, device=coll_dev)
    dist.all_reduce(comps)
    eng.close()
    # end to end through the public API: shard construction + W+K steps + spikes back
    torch.cuda.synchronize()
    dist.barrier()
    a = time.perf_counter()
    eng2, adv2, spikes2 = make()
    tt = 0.0
    for _ in range(args.warmup + args.steps):
        tt += STEP_MS
        adv2(tt)
    st_, sg_ = spikes2()
    e2e_wall = torch.tensor([time.perf_counter() - a], dtype=torch.float64, device=coll_dev)
    dist.all_reduce(e2e_wall, op=dist.ReduceOp.MAX)
    nsteps_e2e = args.warmup + args.steps
    e2e_val = nsteps_e2e * STEP_MS * 1e-3 / float(e2e_wall.item())
    v = flat.view
    h2d = v.n_connections * (1 + 4 + 4 + 4 + 1 + 8 + 8) + s1["total_synapses"] * 8 * 12 + s1["total_comps"] * 8 * 5
    d2h = st_.nbytes + sg_.nbytes
    eng2.close()
    # config 5 strong-scaled: the 100 k-cell network (48 comps, p = 0.002)
    # over the same ranks, 100 -> 300 ms after a 100 ms warm-up
    other = None
    if not args.no_other:
        c5 = N.ConsolidationConfig(n_cells=100000, n_exc=80000, p_conn=0.002, seed=SEED, multi_compartment=True,
                                   dend_size=N.DendriteSize.large_dendrites, dt_ms=DT_MS)
        t_s = time.perf_counter()
        f5 = N.build_consolidation_network(c5, True, device=device).recipe.flatten()
        e5, adv5, _ = make(f5)
        setup5 = time.perf_counter() - t_s
        e5.set_timing(True)
        adv5(100.0)
        a5 = e5.stats()
        torch.cuda.synchronize()
        dist.barrier()
        w5 = time.perf_counter()
        adv5(300.0)
        torch.cuda.synchronize()
        w5 = time.perf_counter() - w5
        b5 = e5.stats()
        d5 = (b5["advance_ms"] - a5["advance_ms"]) * 1e-3 if backend == "nccl" else w5
        t5 = torch.tensor([d5, setup5], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t5, op=dist.ReduceOp.MAX)
        steps5 = b5["steps"] - a5["steps"]
        other = {"config5_strong": {"n_cells": 100000, "n_gpus": world, "bio_ms": 200.0,
                                    "sim_s_per_wall_s": 0.2 / float(t5[0].item()),
                                    "us_per_fine_step": 1e6 * float(t5[0].item()) / max(steps5, 1),
                                    "setup_s": float(t5[1].item()), "scaling": "strong",
                                    "timing": "engine CUDA events, max over ranks" if backend == "nccl"
                                    else "wall clock (host-staged exchange), max over ranks"}}
        e5.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": data_note(world),
            "config": config_block(world),
            "compartment_updates_per_s": float(comps.item()) * fine_steps / total,
            "exchange": "ncclAllGather in libmcg" if backend == "nccl" else backend + " (host-staged)",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": stepping_kernel(s1) + " (rank 0)", "peak_kind": peak_kind,
                         "bytes_per_launch": bstep * steps_per_launch,
                         "mean_launch_ms": mean_launch_s * 1e3, "steps_per_launch": steps_per_launch},
            "cpu_baseline": None,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d / nsteps_e2e),
                    "d2h_bytes_per_step": int(d2h / nsteps_e2e)},
            "gpu_launches": int(s1["kernel_launches"] - s0["kernel_launches"]),
            "clocks": clk,
        }
        if other:
            line["other_configs"] = other
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-sample-ms", type=float, default=2000.0)
    ap.add_argument("--cpu-sample-ms-1w", type=float, default=1000.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other", action="store_true", help="skip the secondary configurations")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world:
        # one process per GPU: N > 1 runs under torchrun, which sets WORLD_SIZE
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} ranks (WORLD_SIZE={world}); launch with "
              f"python -m torch.distributed.run --nproc-per-node {args.gpus} --master-addr 127.0.0.1 "
              f"bench.py --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
