"""Network recipes of the reference's experiments, rebuilt for the B200 engine.

Mirrors (same parameters, same connection order, same random draws):
  build_consolidation_network / run_consolidation   network.cpp:426-639
  build_stc_single / stc_protocol_times / run_stc_protocol   network.cpp:289-399
  run_stc_protocols (the stc-protocols experiment, experiments.cpp:262-289,
                     trials batched as the cells of one engine)
  build_stdp_single_neuron / run_stdp_poisson       network.cpp:43-120
  build_busyring / calibrate_ring_weight / run_bench_once    bench.cpp:31-194
  build_single_neuron_plastic  (config 2 of BASELINE.json; not in the reference)
and the morphology builders they use (morphology.cpp:67-197).

The O(N^2) Erdos-Renyi sampler (network.cpp:34-39, 548-571) runs on the GPU
(mcg_er_connect) in the reference's loop order, and every other random draw
(busyring tree lengths and wiring) comes from the device RNG (mcg_device_math),
so the recipes are bit-identical to the reference builders' output.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A
from .engine import Engine, EngineOptions
from .recipe import par_take
from .recipe import (CellKindSpec, ConnectionSpec, ConnectionTable, EngineError, HhMembrane, LifMembrane,
                     MorphologyError, PlacementSpec, PoissonSource, PoissonWindow, ProbeSpec,
                     ProbeWhat, Recipe, Region, ScriptedSource, Segment, SelectionPolicy,
                     SpeciesSpec, StcParams, StdpParams, SynKind, SynSpec)

PI = math.pi
K_STREAM_CONNECTIVITY = 17   # network.cpp:14
K_STREAM_TREE = 23           # bench.cpp:14
K_STREAM_WIRING = 29         # bench.cpp:15


# ---- device RNG streams (mcg_device_math) -------------------------------------

def uniform_stream(key, n0: int, count: int, device: int = 0) -> np.ndarray:
    """uniform_for(key, n0 + i), i < count (rng.cpp:80-84), evaluated on the GPU."""
    out = np.empty(count, np.float64)
    if count:
        k = (C.c_uint64 * 4)(*[int(x) & (2**64 - 1) for x in key])
        st = A.lib().mcg_device_math(device, 4, None, count, k, n0,
                                     out.ctypes.data_as(C.c_void_p))
        if st != 0:
            raise RuntimeError(A.lib().mcg_last_error().decode())
    return out


def er_pairs(seed: int, n: int, p: float, device: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """All (i, j) with er_connected(seed, i, j, n, p), in i-major, j-minor order.

    One call into the sampler with buffers sized to the expected count plus a
    wide margin (mean n(n-1)p, +16 standard deviations); only if the sample
    is larger still does a second call run with the exact size."""
    L = A.lib()
    mean = float(n) * max(n - 1, 0) * min(max(p, 0.0), 1.0)
    cap = int(mean + 16.0 * math.sqrt(mean + 1.0) + 1024)
    for _ in range(2):
        src = np.empty(cap, np.uint32)
        dst = np.empty(cap, np.uint32)
        cnt = C.c_int64(cap)
        st = L.mcg_er_connect(device, seed, n, p, 0, n, src.ctypes.data_as(C.c_void_p),
                              dst.ctypes.data_as(C.c_void_p), C.byref(cnt))
        if st == 0:
            return src[:cnt.value], dst[:cnt.value]
        cnt = C.c_int64(0)  # buffer too small: the exact count, then once more
        st = L.mcg_er_connect(device, seed, n, p, 0, n, None, None, C.byref(cnt))
        if st != 0:
            raise RuntimeError(L.mcg_last_error().decode())
        cap = int(cnt.value)
    raise RuntimeError(L.mcg_last_error().decode())


# ---- morphology (morphology.cpp) --------------------------------------------------

@dataclass
class GridInfo:
    first: List[int]
    count: List[int]
    size: int

    def compartment_at(self, seg: int, pos: float) -> int:  # morphology.cpp:43-58
        first, count = self.first[seg], self.count[seg]
        pos = min(max(pos, 0.0), 1.0)
        kf = pos * count - 0.5
        k = int(math.ceil(kf - 0.5))
        k = min(max(k, 0), count - 1)
        return first + k


def grid_layout(segments: List[Segment], target_um: float) -> GridInfo:
    """Compartment numbering of discretize (morphology.cpp:67-143)."""
    n = len(segments)
    if n == 0:
        raise MorphologyError("discretize: empty segment list")
    root = [i for i, s in enumerate(segments) if s.parent is None]
    if len(root) != 1:
        raise MorphologyError("discretize: multiple roots" if root else "discretize: no root segment")
    order, placed = [root[0]], [False] * n
    placed[root[0]] = True
    h = 0
    while h < len(order):
        for s in range(n):
            if not placed[s] and segments[s].parent is not None and segments[s].parent == order[h]:
                order.append(s)
                placed[s] = True
        h += 1
    if len(order) != n:
        raise MorphologyError("discretize: cyclic parent references")
    first, count = [0] * n, [0] * n
    size = 0
    for idx in order:
        c = max(1, int(math.ceil(segments[idx].length_um / target_um - 1e-12)))
        first[idx], count[idx] = size, c
        size += c
    return GridInfo(first, count, size)


class CellSize:
    small_cells = 0
    large_cells = 1


class DendriteSize:
    small_dendrites = 0
    large_dendrites = 1


def consolidation_radius_um(c):
    return 6.0 if c == CellSize.small_cells else 12.0


def apical_length_um(d):
    return 12.5 if d == DendriteSize.small_dendrites else 25.0


def basal_length_um(d):
    return 5.0 if d == DendriteSize.small_dendrites else 10.0


def morpho_correction(d):
    return 1.035 if d == DendriteSize.small_dendrites else 1.020


@dataclass
class ConsolidationCellParams:  # morphology.hpp:84-93
    single_compartment: bool = True
    cell: int = CellSize.small_cells
    dendrites: int = DendriteSize.small_dendrites
    delta_l_um: float = 1.0
    soma_length_um: float = 12.0
    synthesis_compartment_um: float = 1.0


@dataclass
class ConsolidationCell:
    segments: List[Segment]
    soma_center_seg: int = 0
    apical_seg: int = 0
    basal_seg: int = 0


def tiny_cylinder() -> Segment:  # network.cpp:16-18
    return Segment(None, 2e-3, 1e-3, Region.soma, 1.0)


def build_consolidation_cell(p: ConsolidationCellParams) -> ConsolidationCell:
    """morphology.cpp:172-197"""
    if p.single_compartment:
        return ConsolidationCell([tiny_cylinder()])
    r = consolidation_radius_um(p.cell)
    half = 0.5 * (p.soma_length_um - p.synthesis_compartment_um)
    if half <= 0:
        raise MorphologyError("consolidation cell: soma shorter than synthesis compartment")
    segs = [Segment(None, p.synthesis_compartment_um, r, Region.soma, 1.0),
            Segment(0, half, r, Region.soma, 1.0),
            Segment(0, half, r, Region.soma, 0.0),
            Segment(1, apical_length_um(p.dendrites), r, Region.apical_dendrite, 1.0),
            Segment(2, basal_length_um(p.dendrites), r, Region.basal_dendrite, 1.0)]
    return ConsolidationCell(segs, 0, 3, 4)


# ---- consolidation network (network.hpp:152-220, network.cpp:426-639) -----------

@dataclass
class ConsolidationConfig:
    n_cells: int = 2000
    n_exc: int = 1600
    p_conn: float = 0.1
    pattern: int = 150
    seed: int = 0
    workers: int = 1
    dt_ms: float = 0.5
    multi_compartment: bool = False
    cell_size: int = CellSize.small_cells
    dend_size: int = DendriteSize.small_dendrites
    d_p: float = 1e-11
    d_sps: float = 1e-11
    stc: StcParams = field(default_factory=StcParams)
    in_vivo_factor: float = 0.6
    tau_mem_ms: float = 10.0
    r_mem_MOhm: float = 10.0
    v_rev_mV: float = -65.0
    v_reset_mV: float = -70.0
    v_thresh_mV: float = -55.0
    t_ref_ms: float = 2.0
    i_bg_nA: float = 0.15
    sigma_bg_nA_sqrt_ms: float = 1.5811388300841898
    w_rec_scale: float = 0.25
    w_ei_mV: float = 2.1
    w_ie_mV: float = -8.4
    w_ii_mV: float = -8.4
    delay_ms: float = 3.0
    n_stim_sources: int = 25
    t_learn_ms: float = 10000.0
    learn_duration_ms: float = 2000.0
    learn_rate_hz: float = 100.0
    recall_duration_ms: float = 200.0
    recall_rate_hz: float = 150.0
    w_stim_mV: float = 0.8
    coarse_dt_ms: float = 1000.0
    adjacency_file: Optional[str] = None
    checkpoint_out: Optional[str] = None


@dataclass
class ConsolidationBuild:
    recipe: Recipe
    as_: List[int]
    ans: List[int]
    ctrl: List[int]
    c_morpho: float = 1.0


def build_consolidation_network(cfg: ConsolidationConfig, eight_hour: bool,
                                device: int = 0) -> ConsolidationBuild:
    if cfg.pattern > cfg.n_exc:
        raise EngineError("pattern size exceeds the excitatory population")
    if cfg.adjacency_file:
        raise EngineError("adjacency files are not supported by this builder")
    stc = cfg.stc
    t_recall = cfg.t_learn_ms + 8 * 3600e3 if eight_hour else cfg.t_learn_ms + 10000.0
    c_morpho = 1.0
    basal_comp = apical_comp = soma_comp = 0
    if cfg.multi_compartment:
        mp = ConsolidationCellParams(single_compartment=False, cell=cfg.cell_size,
                                     dendrites=cfg.dend_size)
        cell = build_consolidation_cell(mp)
        segs, target = cell.segments, mp.delta_l_um
        g = grid_layout(cell.segments, mp.delta_l_um)
        soma_comp = g.compartment_at(cell.soma_center_seg, 0.5)
        apical_comp = g.compartment_at(cell.apical_seg, 1.0)
        basal_comp = g.compartment_at(cell.basal_seg, 1.0)
        c_morpho = morpho_correction(cfg.dend_size)
    else:
        segs, target = [tiny_cylinder()], 1.0
    lm = LifMembrane(tau_mem_ms=cfg.tau_mem_ms, r_mem_MOhm=cfg.r_mem_MOhm, v_rev_mV=cfg.v_rev_mV,
                     v_reset_mV=cfg.v_reset_mV, v_thresh_mV=cfg.v_thresh_mV,
                     t_ref_ms=cfg.t_ref_ms, i_bg_nA=cfg.i_bg_nA,
                     sigma_bg_nA_sqrt_ms=cfg.sigma_bg_nA_sqrt_ms, noise_comp=soma_comp,
                     detector_comp=soma_comp, exact=not cfg.multi_compartment)
    if eight_hour:
        lm.bg_quiet_t0_ms = cfg.t_learn_ms + 2500.0
        lm.bg_quiet_t1_ms = cfg.t_learn_ms + 3000.0
    exc = CellKindSpec(segments=segs, target_compartment_um=target, membrane=lm)
    exc.species = [SpeciesSpec("SPS", cfg.d_sps, 0.0, 0.0),
                   SpeciesSpec("PRP", cfg.d_p, stc.tau_p_ms, 0.0)]
    exc.prp.enabled = True
    exc.prp.comp = soma_comp
    exc.placements = [
        PlacementSpec("rec", SynSpec(kind=SynKind.stc_charge, stc=replace(stc),
                                     calcium_scale=cfg.in_vivo_factor), basal_comp, 0),
        PlacementSpec("ext", SynSpec(kind=SynKind.static_charge), apical_comp, 0),
        PlacementSpec("isyn", SynSpec(kind=SynKind.static_charge), soma_comp, 0)]
    im = replace(lm, noise_comp=0, detector_comp=0, exact=True)
    inh = CellKindSpec(segments=[tiny_cylinder()], membrane=im,
                       placements=[PlacementSpec("ein", SynSpec(kind=SynKind.static_charge), 0, 0),
                                   PlacementSpec("iin", SynSpec(kind=SynKind.static_charge), 0, 0)])
    n, n_exc = cfg.n_cells, cfg.n_exc
    cell_kind = np.ones(n, np.uint32)
    cell_kind[:n_exc] = 0

    src, dst = er_pairs(cfg.seed, n, cfg.p_conn, device)
    # label per pair (network.cpp:551-569): exc->exc "rec", exc->inh "ein",
    # inh->exc "isyn", inh->inh "iin" = 2 (src is inh) + (dst is inh)
    n_rec = len(src)
    pat = cfg.pattern
    n_stim = cfg.n_stim_sources * (pat + pat // 2)
    tot = n_rec + n_stim
    # the connection table's columns, filled in place (no concatenation copies)
    lab = np.empty(tot, np.int32)
    np.add(np.left_shift((src >= n_exc).view(np.uint8), 1, dtype=np.int32), (dst >= n_exc).view(np.uint8),
           out=lab[:n_rec], dtype=np.int32)
    wlut = np.array([cfg.w_rec_scale * c_morpho, cfg.w_ei_mV, cfg.w_ie_mV, cfg.w_ii_mV, cfg.w_stim_mV])
    c_src = np.empty(tot, np.uint32)
    c_dst = np.empty(tot, np.uint32)
    c_src[:n_rec] = src
    c_dst[:n_rec] = dst
    del src, dst
    from_source = np.zeros(tot, np.uint8)
    delay = np.full(tot, cfg.delay_ms, np.float64)

    sources: List = []
    off = n_rec

    def add_pool(t0, dur, rate, g1):  # network.cpp:576-592
        nonlocal off
        for _ in range(cfg.n_stim_sources):
            sources.append(PoissonSource([PoissonWindow(t0, t0 + dur, rate)]))
            sl = slice(off, off + g1)
            c_src[sl] = len(sources) - 1
            c_dst[sl] = np.arange(g1, dtype=np.uint32)
            lab[sl] = 4  # "ext"
            from_source[sl] = 1
            delay[sl] = cfg.dt_ms
            off += g1

    add_pool(cfg.t_learn_ms, cfg.learn_duration_ms, cfg.learn_rate_hz, pat)
    add_pool(t_recall, cfg.recall_duration_ms, cfg.recall_rate_hz, pat // 2)
    conns = ConnectionTable(from_source, c_src, c_dst, ["rec", "ein", "isyn", "iin", "ext"], lab,
                            int(SelectionPolicy.univalent), par_take(wlut, lab), delay)
    r = Recipe(kinds=[exc, inh], cell_kind=cell_kind, sources=sources, connections=conns)
    return ConsolidationBuild(r, list(range(pat // 2)), list(range(pat // 2, pat)),
                              list(range(pat, n_exc)), c_morpho)


@dataclass
class ConsolidationResult:
    spikes_t_s: np.ndarray
    spikes_gid: np.ndarray
    final_h: np.ndarray
    final_z: np.ndarray


def run_consolidation(cfg: ConsolidationConfig, eight_hour: bool, device: int = 0):
    """network.cpp:600-639 (without the recall-quotient analysis)."""
    b = build_consolidation_network(cfg, eight_hour, device)
    eng = Engine(b.recipe, EngineOptions(cfg.dt_ms, cfg.seed, cfg.workers), device=device)
    if not eight_hour:
        t_recall = cfg.t_learn_ms + 10000.0
        eng.advance_to(t_recall + 500.0)
    else:
        t_recall = cfg.t_learn_ms + 8 * 3600e3
        t_ff0 = cfg.t_learn_ms + 3000.0
        eng.advance_to(t_ff0)
        t_ff1 = t_ff0 + math.floor((t_recall - 1000.0 - t_ff0) / cfg.coarse_dt_ms) * cfg.coarse_dt_ms
        eng.fast_forward_to(t_ff1, cfg.coarse_dt_ms)
        eng.advance_to(t_recall + 500.0)
    t, g = eng.spike_arrays()
    hs, zs = [], []
    for gid in range(cfg.n_exc):
        grp = eng.cell(gid).groups[0]
        hs.append(grp.stc_h)
        zs.append(grp.stc_z)
    return ConsolidationResult(t * 1e-3, g, np.concatenate(hs) if hs else np.zeros(0),
                               np.concatenate(zs) if zs else np.zeros(0))


# ---- single synapse with tagging and capture (network.hpp:99-148) ---------------

class StcProtocol:
    stet, wtet, slfs, wlfs, none = range(5)


def stc_protocol_times(p: int, onset_ms: float) -> List[float]:  # network.cpp:289-314
    t: List[float] = []
    if p == StcProtocol.stet:
        for train in range(3):
            for k in range(100):
                t.append(onset_ms + train * 600e3 + k * 10.0)
    elif p == StcProtocol.wtet:
        t = [onset_ms + k * 10.0 for k in range(21)]
    elif p == StcProtocol.slfs:
        for b in range(900):
            for k in range(3):
                t.append(onset_ms + b * 1000.0 + k * 50.0)
    elif p == StcProtocol.wlfs:
        t = [onset_ms + k * 1000.0 for k in range(900)]
    return t


@dataclass
class StcSingleConfig:  # network.hpp:104-118
    stc: StcParams = field(default_factory=StcParams)
    dt_ms: float = 0.2
    seed: int = 0
    t_onset_ms: float = 10000.0
    t_eval_ms: float = 5 * 3600e3
    coarse_dt_ms: float = 10000.0
    trace_every_ms: float = 1000.0
    tau_mem_ms: float = 10.0
    r_mem_MOhm: float = 10.0
    v_gap_mV: float = 10.0
    i_bg_nA: float = 0.3
    sigma_bg_nA_sqrt_ms: float = 1.5811388300841898


def point_lif(tau_ms, r_MOhm, v_rev, v_gap) -> LifMembrane:  # network.cpp:20-30
    return LifMembrane(tau_mem_ms=tau_ms, r_mem_MOhm=r_MOhm, v_rev_mV=v_rev,
                       v_reset_mV=v_rev - 5.0, v_thresh_mV=v_rev + v_gap, exact=True)


def build_stc_single(cfg: StcSingleConfig, pre_times: List[float]) -> Recipe:
    """network.cpp:318-349 (config 1 of BASELINE.json)."""
    m = point_lif(cfg.tau_mem_ms, cfg.r_mem_MOhm, -65.0, cfg.v_gap_mV)
    m.i_bg_nA = cfg.i_bg_nA
    m.sigma_bg_nA_sqrt_ms = cfg.sigma_bg_nA_sqrt_ms
    kind = CellKindSpec(segments=[tiny_cylinder()], membrane=m,
                        species=[SpeciesSpec("SPS", 0.0, 0.0, 0.0),
                                 SpeciesSpec("PRP", 0.0, cfg.stc.tau_p_ms, 0.0)],
                        placements=[PlacementSpec("syn", SynSpec(kind=SynKind.stc_charge,
                                                                 stc=replace(cfg.stc)), 0, 1)])
    kind.prp.enabled = True
    kind.prp.comp = 0
    every = max(1, int(cfg.trace_every_ms / cfg.dt_ms))
    r = Recipe(kinds=[kind], cell_kind=[0], sources=[ScriptedSource(list(pre_times))])
    r.connections = ConnectionTable(1, [0], [0], ["syn"], 0, 0, 1.0, cfg.dt_ms)
    r.probes = [ProbeSpec(0, ProbeWhat.syn_h, 0, 0, "syn", 0, every),
                ProbeSpec(0, ProbeWhat.syn_z, 0, 0, "syn", 0, every),
                ProbeSpec(0, ProbeWhat.syn_c, 0, 0, "syn", 0, every),
                ProbeSpec(0, ProbeWhat.species, 0, 1, "", 0, every)]
    return r


@dataclass
class StcRunResult:
    h_final: float
    z_final: float
    p_final: float
    max_abs_dh: float
    tag_crossed: bool
    prp_crossed: bool
    traces: list


def run_stc_protocol(cfg: StcSingleConfig, proto: int, trial: int, device: int = 0):
    """network.cpp:353-399"""
    times = stc_protocol_times(proto, cfg.t_onset_ms)
    t_last = times[-1] if times else cfg.t_onset_ms
    r = build_stc_single(cfg, times)
    t_detailed = t_last + 2000.0
    t_detailed = math.ceil(t_detailed / 1000.0) * 1000.0
    m = r.kinds[0].membrane
    m.bg_quiet_t0_ms = t_detailed - 500.0
    m.bg_quiet_t1_ms = cfg.t_eval_ms
    eng = Engine(r, EngineOptions(cfg.dt_ms, cfg.seed + trial, 1), device=device)
    eng.advance_to(t_detailed)
    span = cfg.t_eval_ms - t_detailed
    n_coarse = math.floor(span / cfg.coarse_dt_ms)
    eng.fast_forward_to(t_detailed + n_coarse * cfg.coarse_dt_ms, cfg.coarse_dt_ms)
    tr = eng.traces()
    hs = [v for _, v in tr[0]]
    max_dh = max([abs(h - cfg.stc.h0_mV) for h in hs], default=0.0)
    g = eng.cell(0).groups[0]
    return StcRunResult(float(g.stc_h[0]), float(g.stc_z[0]), float(eng.cell(0).species[1][0]),
                        max_dh, max_dh > cfg.stc.theta_tag_mV, max_dh > cfg.stc.theta_pro_mV, tr)


def run_stc_protocols(cfg: StcSingleConfig, protocols: Sequence[int], trials: int, device: int = 0,
                      max_cells: int = 128) -> List[List["StcRunResult"]]:
    """The stc-protocols experiment (experiments.cpp:262-289) on the device:
    run_stc_protocol(cfg, p, t) for every protocol p and trial t < trials,
    results[i][t] for protocols[i], each bitwise the single-trial run.

    Trials are independent single-cell simulations that differ only in the
    seed (cfg.seed + t) and share the stimulus times, so one engine holds up to
    `max_cells` trials as cells of one recipe (same kind, one shared scripted
    source, four probes per cell) with per-cell RNG keys (seed + t, gid 0:
    mcg_set_cell_rng), and runs them on the point-cell kernel, one cell per
    CTA; the protocols' engines run concurrently on their own streams."""
    import threading
    jobs = []
    for pi, proto in enumerate(protocols):
        for t0 in range(0, trials, max_cells):
            jobs.append((pi, proto, list(range(t0, min(trials, t0 + max_cells)))))
    out: List[List[Optional[StcRunResult]]] = [[None] * trials for _ in protocols]
    errors: List[BaseException] = []

    def run(pi, proto, tids):
        try:
            times = stc_protocol_times(proto, cfg.t_onset_ms)
            t_last = times[-1] if times else cfg.t_onset_ms
            one = build_stc_single(cfg, times)
            t_detailed = math.ceil((t_last + 2000.0) / 1000.0) * 1000.0
            kind = one.kinds[0]
            kind.membrane.bg_quiet_t0_ms = t_detailed - 500.0
            kind.membrane.bg_quiet_t1_ms = cfg.t_eval_ms
            n = len(tids)
            probes = []
            for c in range(n):  # the single-trial probes, per cell
                probes += [replace(p, gid=c) for p in one.probes]
            r = Recipe(kinds=[kind], cell_kind=[0] * n, sources=list(one.sources),
                       connections=ConnectionTable(1, [0] * n, list(range(n)), ["syn"], 0, 0, 1.0, cfg.dt_ms),
                       probes=probes)
            eng = Engine(r, EngineOptions(cfg.dt_ms, cfg.seed, 1), device=device)
            eng.set_cell_rng([cfg.seed + t for t in tids], [0] * n)
            eng.advance_to(t_detailed)
            span = cfg.t_eval_ms - t_detailed
            n_coarse = math.floor(span / cfg.coarse_dt_ms)
            eng.fast_forward_to(t_detailed + n_coarse * cfg.coarse_dt_ms, cfg.coarse_dt_ms)
            tr = eng.traces()
            for c, t in enumerate(tids):
                hs = [v for _, v in tr[4 * c]]
                max_dh = max([abs(h - cfg.stc.h0_mV) for h in hs], default=0.0)
                g = eng.cell(c).groups[0]
                out[pi][t] = StcRunResult(float(g.stc_h[0]), float(g.stc_z[0]), float(eng.cell(c).species[1][0]),
                                          max_dh, max_dh > cfg.stc.theta_tag_mV, max_dh > cfg.stc.theta_pro_mV,
                                          tr[4 * c:4 * c + 4])
            eng.close()
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=run, args=j) for j in jobs]
    for x in th:
        x.start()
    for x in th:
        x.join()
    if errors:
        raise errors[0]
    return out


# ---- single neuron driven by plastic + static Poisson inputs (network.hpp:17-41) ----

@dataclass
class StdpPoissonConfig:  # network.hpp:19-30
    duration_ms: float = 10000.0
    dt_ms: float = 0.1
    seed: int = 0
    rate_exc_hz: float = 100.0
    rate_inh_hz: float = 30.0
    w_inh_uS: float = 1.0
    tau_syn_ms: float = 5.0
    e_exc_mV: float = 0.0
    e_inh_mV: float = -80.0
    stdp: StdpParams = field(default_factory=StdpParams)


def build_stdp_single_neuron(cfg: StdpPoissonConfig) -> Recipe:
    """network.cpp:43-91: one tiny-cylinder cable LIF neuron (1 uS leak), an
    STDP conductance synapse driven by an excitatory Poisson source and a
    static conductance synapse driven by an inhibitory one; the plastic
    weight is probed every 10 ms."""
    m = LifMembrane(tau_mem_ms=10.0, r_mem_MOhm=1.0, v_rev_mV=-65.0, v_reset_mV=-70.0, v_thresh_mV=-55.0)
    exc = SynSpec(kind=SynKind.stdp_cond, tau_syn_ms=cfg.tau_syn_ms, e_rev_mV=cfg.e_exc_mV, stdp=replace(cfg.stdp))
    inh = SynSpec(kind=SynKind.static_cond, tau_syn_ms=cfg.tau_syn_ms, e_rev_mV=cfg.e_inh_mV)
    kind = CellKindSpec(segments=[tiny_cylinder()], target_compartment_um=1.0, membrane=m,
                        placements=[PlacementSpec("exc", exc, 0, 0), PlacementSpec("inh", inh, 0, 0)])
    r = Recipe(kinds=[kind], cell_kind=[0],
               sources=[PoissonSource([PoissonWindow(0.0, cfg.duration_ms, cfg.rate_exc_hz)]),
                        PoissonSource([PoissonWindow(0.0, cfg.duration_ms, cfg.rate_inh_hz)])],
               connections=[ConnectionSpec(True, 0, 0, "exc", SelectionPolicy.univalent, cfg.stdp.w0_uS, cfg.dt_ms),
                            ConnectionSpec(True, 1, 0, "inh", SelectionPolicy.univalent, cfg.w_inh_uS, cfg.dt_ms)],
               probes=[ProbeSpec(0, ProbeWhat.syn_weight, 0, 0, "exc", 0, max(1, int(10.0 / cfg.dt_ms)))])
    return r


@dataclass
class StdpPoissonResult:  # network.hpp:34-39
    pre_count: int
    post_count: int
    weight_t_s: np.ndarray
    weight: np.ndarray
    spikes_t_s: np.ndarray
    spikes_gid: np.ndarray


def run_stdp_poisson(cfg: StdpPoissonConfig, device: int = 0) -> StdpPoissonResult:
    """network.cpp:93-120 on the device; pre_count re-draws the excitatory
    source's Bernoulli trials (uniform_for(key(seed, 2^32, 3, 0), s) < rate dt
    1e-3) for reporting, as the reference does."""
    eng = Engine(build_stdp_single_neuron(cfg), EngineOptions(cfg.dt_ms, cfg.seed, 1), device=device)
    eng.advance_to(cfg.duration_ms)
    tt, w = eng.trace_arrays(0)
    st, sg = eng.spike_arrays()
    steps = int(math.ceil(cfg.duration_ms / cfg.dt_ms))
    u = uniform_stream((cfg.seed, 0x100000000, 3, 0), 0, steps, device)
    pre = int(np.count_nonzero(u < cfg.rate_exc_hz * cfg.dt_ms * 1e-3))
    return StdpPoissonResult(pre, len(st), tt * 1e-3, w, st * 1e-3, sg)


# ---- busyring (bench.hpp / bench.cpp) ---------------------------------------------

@dataclass
class BusyringSpec:
    n_cells: int = 1024
    ring_size: int = 4
    random_per_cell: int = 1000
    delay_ms: float = 5.0
    ring_weight_uS: float = 0.0
    tau_syn_ms: float = 2.0
    tree_depth: int = 2
    stdp_on_random: bool = False
    stdp: StdpParams = field(default_factory=StdpParams)
    duration_ms: float = 200.0
    dt_ms: float = 0.025
    seed: int = 0
    workers: int = 1


def default_busyring() -> BusyringSpec:  # bench.cpp:31-40
    s = BusyringSpec()
    s.stdp = StdpParams(tau_pre_ms=10.0, tau_post_ms=10.0, a_pre_uS=0.01, a_post_uS=-0.01,
                        wmax_uS=10.0, w0_uS=0.0)
    return s


def busyring_cell_segments(depth: int, seed: int, gid: int, device: int = 0) -> List[Segment]:
    """bench.cpp:42-68"""
    segs = [Segment(None, 12.6, 6.3, Region.soma, 1.0)]
    if depth <= 0:
        return segs
    ndraw = sum(2 ** l for l in range(1, depth + 1))
    u = uniform_stream((seed, gid, K_STREAM_TREE, 0), 0, ndraw, device)
    draw = 0
    frontier = [0]
    for _level in range(1, depth + 1):
        nxt = []
        for parent in frontier:
            for _child in range(2):
                segs.append(Segment(parent, 10.0 + 10.0 * u[draw], 0.6, Region.generic, 1.0))
                draw += 1
                nxt.append(len(segs) - 1)
        frontier = nxt
    return segs


def busyring_kind(spec: BusyringSpec, gid: int, device: int = 0) -> CellKindSpec:  # bench.cpp:72-101
    kind = CellKindSpec(segments=busyring_cell_segments(spec.tree_depth, spec.seed, gid, device),
                        target_compartment_um=20.0 if spec.tree_depth <= 0 else 2.0,
                        membrane=HhMembrane())
    kind.placements = [
        PlacementSpec("ring", SynSpec(kind=SynKind.static_cond, tau_syn_ms=spec.tau_syn_ms,
                                      e_rev_mV=0.0), 0, 0),  # default StdpParams, as bench.cpp:80-86
        PlacementSpec("load", SynSpec(kind=SynKind.stdp_cond if spec.stdp_on_random
                                      else SynKind.static_cond, tau_syn_ms=spec.tau_syn_ms,
                                      e_rev_mV=0.0, stdp=replace(spec.stdp)), 0, 0)]
    return kind


def calibrate_ring_weight(spec: BusyringSpec, latency_ms: float = 0.3, device: int = 0) -> float:
    """bench.cpp:105-132: bisection on a one-cell engine run."""
    needed = 0.0
    for sample in range(3):
        kind = busyring_kind(spec, sample, device)
        lo, hi = 1e-5, 2.0
        for _ in range(30):
            w = 0.5 * (lo + hi)
            r = Recipe(kinds=[kind], cell_kind=[0], sources=[ScriptedSource([5.0])])
            r.connections = ConnectionTable(1, [0], [0], ["ring"], 0, 0, w, spec.dt_ms)
            eng = Engine(r, EngineOptions(spec.dt_ms, spec.seed, 1), device=device)
            eng.advance_to(5.0 + max(2.0, 4 * latency_ms))
            t, _ = eng.spike_arrays()
            ok = bool(np.any(t <= 5.0 + spec.dt_ms + latency_ms))
            eng.close()
            if ok:
                hi = w
            else:
                lo = w
        needed = max(needed, hi)
    return 1.5 * needed


def build_busyring(spec: BusyringSpec, device: int = 0) -> Recipe:
    """bench.cpp:134-178"""
    if spec.ring_size <= 0 or spec.n_cells % spec.ring_size != 0:
        raise EngineError("busyring: n_cells must be a multiple of the ring size")
    w_ring = spec.ring_weight_uS if spec.ring_weight_uS > 0 else calibrate_ring_weight(spec, device=device)
    n, k = spec.n_cells, spec.ring_size
    kinds = [busyring_kind(spec, g, device) for g in range(n)]
    g = np.arange(n, dtype=np.int64)
    base = g - g % k
    nxt = base + (g + 1 - base) % k
    ring = ConnectionTable(0, g, nxt, ["ring"], 0, 0, w_ring, spec.delay_ms)
    m = spec.random_per_cell
    u = uniform_stream((spec.seed, 0, K_STREAM_WIRING, 0), 0, n * m, device)
    rdst = np.minimum((u * float(n)).astype(np.uint64), n - 1).astype(np.uint32)
    rsrc = np.repeat(np.arange(n, dtype=np.uint32), m)
    load = ConnectionTable(0, rsrc, rdst, ["load"], 0, 0, 0.0, spec.delay_ms)
    bases = np.arange(0, n, k)
    stim = ConnectionTable(1, np.arange(len(bases)), bases, ["ring"], 0, 0, w_ring, spec.dt_ms)
    return Recipe(kinds=kinds, cell_kind=np.arange(n, dtype=np.uint32),
                  sources=[ScriptedSource([0.0]) for _ in bases],
                  connections=ConnectionTable.concat([ring, load, stim]))


# ---- config 2: one MC neuron with 1000 plastic synapses (BASELINE.json configs[1]) ---

def build_single_neuron_plastic(n_inputs: int = 1000, rate_hz: float = 5.0,
                                duration_ms: float = 10000.0, dt_ms: float = 0.1,
                                large_dendrites: bool = False, w_stc: float = 1.0,
                                w_stdp_uS: float = 0.01) -> Recipe:
    """consolidation MC cell (31/48 comps, cable LIF),
    an STC group and an STDP group at the basal tip, each input source driving
    one synapse of each group."""
    mp = ConsolidationCellParams(single_compartment=False,
                                 dendrites=DendriteSize.large_dendrites if large_dendrites
                                 else DendriteSize.small_dendrites)
    cell = build_consolidation_cell(mp)
    g = grid_layout(cell.segments, mp.delta_l_um)
    soma = g.compartment_at(cell.soma_center_seg, 0.5)
    basal = g.compartment_at(cell.basal_seg, 1.0)
    lm = LifMembrane(noise_comp=soma, detector_comp=soma, exact=False)
    stc = StcParams()
    kind = CellKindSpec(segments=cell.segments, target_compartment_um=1.0, membrane=lm,
                        species=[SpeciesSpec("SPS", 1e-11, 0.0, 0.0),
                                 SpeciesSpec("PRP", 1e-11, stc.tau_p_ms, 0.0)])
    kind.prp.enabled = True
    kind.prp.comp = soma
    kind.placements = [PlacementSpec("rec", SynSpec(kind=SynKind.stc_charge, stc=stc,
                                                    calcium_scale=0.6), basal, 0),
                       PlacementSpec("stdp", SynSpec(kind=SynKind.stdp_cond, e_rev_mV=0.0,
                                                     stdp=StdpParams(w0_uS=w_stdp_uS)), basal, 0)]
    srcs = [PoissonSource([PoissonWindow(0.0, duration_ms, rate_hz)]) for _ in range(n_inputs)]
    s = np.arange(n_inputs)
    a = ConnectionTable(1, s, 0, ["rec"], 0, 0, w_stc, dt_ms)
    b = ConnectionTable(1, s, 0, ["stdp"], 0, 0, w_stdp_uS, dt_ms)
    # per source: one rec then one stdp connection (connection order = seq)
    conn = ConnectionTable.concat([a, b])
    order = np.argsort(np.concatenate([2 * s, 2 * s + 1]), kind="stable")
    conn = ConnectionTable(conn.from_source[order], conn.src[order], conn.dst[order], conn.labels,
                           conn.label_idx[order], conn.policy[order], conn.weight[order],
                           conn.delay_ms[order])
    return Recipe(kinds=[kind], cell_kind=[0], sources=srcs, connections=conn)
