"""Declarative network description — Python mirror of the reference's
recipe.hpp (/root/reference/proj/include/mcsim/recipe.hpp:24-189),
mechanisms.hpp parameter structs (:20-194) and morphology.hpp Segment (:26-32).

Field names, order and defaults are the reference's, so a recipe written
against the reference reads the same here.  `Recipe.flatten()` produces the
plain-pointer `mcg_recipe` of include/mcg.h; labels (placement labels,
species names) are resolved here exactly as the reference resolves them
(first placement with the label: CellRT::find_group, engine.cpp:92-96; last
species with the name: build_kind, engine.cpp:253-254).

Connections may be given as a list of ConnectionSpec (the reference's form)
or as a ConnectionTable (the same columns as numpy arrays), which the network
builders use for the 10^5..10^7-connection configurations.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Union

import numpy as np

from . import _abi as A


class EngineError(RuntimeError):
    """mcsim::EngineError (engine.hpp:16-18)."""


class NumericError(RuntimeError):
    """mcsim::NumericError (tree_solver.hpp:11-13)."""


class TargetingError(RuntimeError):
    """mcsim::TargetingError (recipe.hpp:138-140)."""


class MorphologyError(RuntimeError):
    """mcsim::MorphologyError (morphology.hpp:55-57)."""


class Region(enum.IntEnum):  # morphology.hpp:12-19
    soma = 0
    apical_dendrite = 1
    basal_dendrite = 2
    spine_neck = 3
    spine_head = 4
    generic = 5


@dataclass
class Segment:  # morphology.hpp:26-32
    parent: Optional[int] = None
    length_um: float = 0.0
    radius_um: float = 0.0
    tag: Region = Region.generic
    parent_pos: float = 1.0


@dataclass
class LifMembrane:  # recipe.hpp:24-42
    tau_mem_ms: float = 10.0
    r_mem_MOhm: float = 10.0
    v_rev_mV: float = -65.0
    v_reset_mV: float = -70.0
    v_thresh_mV: float = -55.0
    t_ref_ms: float = 2.0
    r_axial_ohm_m: float = 1.0
    i_bg_nA: float = 0.0
    sigma_bg_nA_sqrt_ms: float = 0.0
    bg_quiet_t0_ms: float = 0.0
    bg_quiet_t1_ms: float = 0.0
    noise_comp: int = 0
    detector_comp: int = 0
    exact: bool = False


@dataclass
class HhMembrane:  # recipe.hpp:45-57
    c_m: float = 1e-2
    r_axial_ohm_m: float = 1.0
    g_leak: float = 3.0
    e_leak_mV: float = -54.387
    g_na: float = 1200.0
    e_na_mV: float = 50.0
    g_k: float = 360.0
    e_k_mV: float = -77.0
    v_init_mV: float = -65.0
    threshold_mV: float = -20.0
    detector_comp: int = 0


@dataclass
class NoMembrane:  # recipe.hpp:60
    pass


@dataclass
class SpeciesSpec:  # recipe.hpp:66-71
    name: str = ""
    diffusivity: float = 0.0
    decay_tau_ms: float = 0.0
    init: float = 0.0


class SynKind(enum.IntEnum):  # recipe.hpp:73-80
    static_charge = 0
    static_cond = 1
    static_current = 2
    stdp_cond = 3
    homeo_current = 4
    stc_charge = 5


@dataclass
class StdpParams:  # mechanisms.hpp:20-27
    tau_pre_ms: float = 20.0
    tau_post_ms: float = 10.0
    a_pre_uS: float = 0.01
    a_post_uS: float = -0.0105
    w0_uS: float = 1.0
    wmax_uS: float = 10.0


@dataclass
class HomeostasisParams:  # mechanisms.hpp:57-63
    dw_plus_nA: float = 0.35
    dw_minus_nA: float = -0.35
    w_init_nA: float = 0.0
    wmax_nA: float = 5.0
    w_varying_nA: float = 3.5


@dataclass
class StcParams:  # mechanisms.hpp:175-194
    h0_mV: float = 4.20075
    tau_h_ms: float = 688.4e3
    tau_c_ms: float = 48.8
    gamma_p: float = 1645.6
    gamma_d: float = 313.1
    theta_p: float = 3.0
    theta_d: float = 1.2
    sigma_pl_mV: float = 2.90436
    c_pre: float = 1.0
    c_post: float = 0.2758
    t_c_delay_ms: float = 18.8
    tau_z_ms: float = 3600e3
    f_int: float = 0.1
    theta_tag_mV: float = 0.840149
    tau_p_ms: float = 3600e3
    p_max: float = 10.0
    theta_pro_mV: float = 2.10037


@dataclass
class SynSpec:  # recipe.hpp:82-90
    kind: SynKind = SynKind.static_charge
    tau_syn_ms: float = 5.0
    e_rev_mV: float = 0.0
    stdp: StdpParams = field(default_factory=StdpParams)
    homeo: HomeostasisParams = field(default_factory=HomeostasisParams)
    stc: StcParams = field(default_factory=StcParams)
    calcium_scale: float = 1.0


@dataclass
class PlacementSpec:  # recipe.hpp:93-98
    label: str = ""
    syn: SynSpec = field(default_factory=SynSpec)
    comp: int = 0
    count: int = 0


@dataclass
class PrpUnitSpec:  # recipe.hpp:100-103
    enabled: bool = False
    comp: int = 0


@dataclass
class CellKindSpec:  # recipe.hpp:105-114
    segments: List[Segment] = field(default_factory=list)
    target_compartment_um: float = 1.0
    membrane: Union[LifMembrane, HhMembrane, NoMembrane] = field(default_factory=NoMembrane)
    species: List[SpeciesSpec] = field(default_factory=list)
    placements: List[PlacementSpec] = field(default_factory=list)
    prp: PrpUnitSpec = field(default_factory=PrpUnitSpec)
    sps_species: str = "SPS"
    prp_species: str = "PRP"

    def find_group(self, label: str) -> int:  # CellRT::find_group, engine.cpp:92-96
        for i, p in enumerate(self.placements):
            if p.label == label:
                return i
        return -1


@dataclass
class PoissonWindow:  # recipe.hpp:118-121
    t0_ms: float = 0.0
    t1_ms: float = 0.0
    rate_hz: float = 0.0


@dataclass
class PoissonSource:  # recipe.hpp:123-125
    windows: List[PoissonWindow] = field(default_factory=list)


@dataclass
class RegularSource:  # recipe.hpp:126-129
    t0_ms: float = 0.0
    period_ms: float = 0.0
    count: int = 0


@dataclass
class ScriptedSource:  # recipe.hpp:130-132
    times_ms: List[float] = field(default_factory=list)


class SelectionPolicy(enum.IntEnum):  # recipe.hpp:136
    univalent = 0
    round_robin = 1
    round_robin_halt = 2


@dataclass
class ConnectionSpec:  # recipe.hpp:151-159 (field order is ABI: brace-init in tests)
    from_source: bool = False
    src: int = 0
    dst: int = 0
    label: str = ""
    policy: SelectionPolicy = SelectionPolicy.univalent
    weight: float = 0.0
    delay_ms: float = 1.0


class ConnectionTable:
    """Column form of a connection list (same fields as ConnectionSpec).

    `label` is given as `labels` (distinct label strings) plus `label_idx`
    (int32 index per connection)."""

    def __init__(self, from_source, src, dst, labels: Sequence[str], label_idx, policy, weight,
                 delay_ms):
        n = len(src)
        self.from_source = np.ascontiguousarray(np.broadcast_to(from_source, n), dtype=np.uint8)
        self.src = np.ascontiguousarray(src, dtype=np.uint32)
        self.dst = np.ascontiguousarray(np.broadcast_to(dst, n), dtype=np.uint32)
        self.labels = list(labels)
        self.label_idx = np.ascontiguousarray(np.broadcast_to(label_idx, n), dtype=np.int32)
        self.policy = np.ascontiguousarray(np.broadcast_to(policy, n), dtype=np.uint8)
        self.weight = np.ascontiguousarray(np.broadcast_to(weight, n), dtype=np.float64)
        self.delay_ms = np.ascontiguousarray(np.broadcast_to(delay_ms, n), dtype=np.float64)

    def __len__(self):
        return len(self.src)

    @staticmethod
    def concat(tables: Sequence["ConnectionTable"]) -> "ConnectionTable":
        lut = {}
        idx = []
        for t in tables:
            remap = np.array([lut.setdefault(l, len(lut)) for l in t.labels], dtype=np.int32)
            idx.append(remap[t.label_idx] if len(t.labels) else t.label_idx)
        cat = lambda a: np.concatenate([getattr(t, a) for t in tables])
        return ConnectionTable(cat("from_source"), cat("src"), cat("dst"), list(lut),
                               np.concatenate(idx), cat("policy"), cat("weight"),
                               cat("delay_ms"))

    @staticmethod
    def from_specs(specs: Sequence[ConnectionSpec]) -> "ConnectionTable":
        labels: List[str] = []
        lut = {}
        li = np.empty(len(specs), np.int32)
        for i, c in enumerate(specs):
            j = lut.get(c.label)
            if j is None:
                j = lut[c.label] = len(labels)
                labels.append(c.label)
            li[i] = j
        return ConnectionTable(
            np.array([c.from_source for c in specs], np.uint8),
            np.array([c.src for c in specs], np.uint32), np.array([c.dst for c in specs], np.uint32),
            labels, li, np.array([int(c.policy) for c in specs], np.uint8),
            np.array([c.weight for c in specs], np.float64),
            np.array([c.delay_ms for c in specs], np.float64))

    def spec(self, i: int) -> ConnectionSpec:
        return ConnectionSpec(bool(self.from_source[i]), int(self.src[i]), int(self.dst[i]),
                              self.labels[self.label_idx[i]], SelectionPolicy(int(self.policy[i])),
                              float(self.weight[i]), float(self.delay_ms[i]))


class ProbeWhat(enum.IntEnum):  # recipe.hpp:163-171
    voltage = 0
    species = 1
    syn_weight = 2
    syn_h = 3
    syn_z = 4
    syn_c = 5
    syn_kernel = 6


@dataclass
class ProbeSpec:  # recipe.hpp:173-181
    gid: int = 0
    what: ProbeWhat = ProbeWhat.voltage
    comp: int = 0
    species: int = 0
    label: str = ""
    instance: int = 0
    every_steps: int = 1


SourceSpec = Union[PoissonSource, RegularSource, ScriptedSource]


@dataclass
class Recipe:  # recipe.hpp:183-189
    kinds: List[CellKindSpec] = field(default_factory=list)
    cell_kind: Union[List[int], np.ndarray] = field(default_factory=list)
    sources: List[SourceSpec] = field(default_factory=list)
    connections: Union[List[ConnectionSpec], ConnectionTable] = field(default_factory=list)
    probes: List[ProbeSpec] = field(default_factory=list)

    def connection_table(self) -> ConnectionTable:
        if isinstance(self.connections, ConnectionTable):
            return self.connections
        return ConnectionTable.from_specs(self.connections)

    def flatten(self) -> "FlatRecipe":
        return FlatRecipe(self)


def par_take(table, idx, out=None, dtype=None):
    """np.take(table, idx) split over host threads for long index arrays
    (numpy releases the GIL inside take)."""
    n = len(idx)
    if out is None:
        out = np.empty(n, dtype or table.dtype)
    if n < (1 << 20):
        np.take(table, idx, out=out)
        return out
    import concurrent.futures as cf
    import os
    k = max(1, min(16, os.cpu_count() or 1))
    bounds = [n * i // k for i in range(k + 1)]
    with cf.ThreadPoolExecutor(k) as ex:
        list(ex.map(lambda i: np.take(table, idx[bounds[i]:bounds[i + 1]], out=out[bounds[i]:bounds[i + 1]]),
                    range(k)))
    return out


def _arr(a, ctype):
    """(numpy array kept alive, ctypes pointer)"""
    return a.ctypes.data_as(C.POINTER(ctype))


class FlatRecipe:
    """`mcg_recipe` view of a Recipe; owns every buffer the view points at."""

    def __init__(self, r: Recipe):
        self._keep = []
        keep = self._keep.append
        nk = len(r.kinds)
        kinds = (A.mcg_kind * max(nk, 1))()
        for k, ks in enumerate(r.kinds):
            fk = kinds[k]
            segs = ks.segments
            par = np.array([-1 if s.parent is None else int(s.parent) for s in segs], np.int32)
            ln = np.array([s.length_um for s in segs], np.float64)
            rd = np.array([s.radius_um for s in segs], np.float64)
            tg = np.array([int(s.tag) for s in segs], np.uint8)
            pp = np.array([s.parent_pos for s in segs], np.float64)
            for a in (par, ln, rd, tg, pp):
                keep(a)
            fk.n_segments = len(segs)
            fk.seg_parent = _arr(par, C.c_int32)
            fk.seg_length_um = _arr(ln, C.c_double)
            fk.seg_radius_um = _arr(rd, C.c_double)
            fk.seg_tag = _arr(tg, C.c_uint8)
            fk.seg_parent_pos = _arr(pp, C.c_double)
            fk.target_compartment_um = ks.target_compartment_um
            m = ks.membrane
            if isinstance(m, LifMembrane):
                fk.membrane = 1
                for f, _ in A.mcg_lif._fields_:
                    v = getattr(m, f)
                    setattr(fk.lif, f, int(v) if f in ("noise_comp", "detector_comp", "exact") else v)
            elif isinstance(m, HhMembrane):
                fk.membrane = 2
                for f, _ in A.mcg_hh._fields_:
                    setattr(fk.hh, f, getattr(m, f))
            else:
                fk.membrane = 0
            sp = (A.mcg_species * max(len(ks.species), 1))()
            keep(sp)
            fk.sps_idx = fk.prp_idx = -1
            for i, s in enumerate(ks.species):
                sp[i].diffusivity = s.diffusivity
                sp[i].decay_tau_ms = s.decay_tau_ms
                sp[i].init = s.init
                if s.name == ks.sps_species:
                    fk.sps_idx = i
                if s.name == ks.prp_species:
                    fk.prp_idx = i
            fk.n_species = len(ks.species)
            fk.species = C.cast(sp, C.POINTER(A.mcg_species))
            pl = (A.mcg_placement * max(len(ks.placements), 1))()
            keep(pl)
            for i, p in enumerate(ks.placements):
                fp = pl[i]
                fp.comp = p.comp
                fp.count = p.count
                sy = p.syn
                fp.syn.kind = int(sy.kind)
                fp.syn.tau_syn_ms = sy.tau_syn_ms
                fp.syn.e_rev_mV = sy.e_rev_mV
                for f, _ in A.mcg_stdp_params._fields_:
                    setattr(fp.syn.stdp, f, getattr(sy.stdp, f))
                for f, _ in A.mcg_homeo_params._fields_:
                    setattr(fp.syn.homeo, f, getattr(sy.homeo, f))
                for f in A.STC_FIELDS:
                    setattr(fp.syn.stc, f, getattr(sy.stc, f))
                fp.syn.calcium_scale = sy.calcium_scale
            fk.n_placements = len(ks.placements)
            fk.placements = C.cast(pl, C.POINTER(A.mcg_placement))
            fk.prp_enabled = 1 if ks.prp.enabled else 0
            fk.prp_comp = ks.prp.comp
        keep(kinds)

        cell_kind = np.ascontiguousarray(r.cell_kind, dtype=np.uint32)
        keep(cell_kind)
        ns = len(r.sources)
        srcs = (A.mcg_source * max(ns, 1))()
        keep(srcs)
        for i, s in enumerate(r.sources):
            fs = srcs[i]
            if isinstance(s, PoissonSource):
                fs.type = 0
                vals = np.array([x for w in s.windows for x in (w.t0_ms, w.t1_ms, w.rate_hz)],
                                np.float64)
            elif isinstance(s, RegularSource):
                fs.type = 1
                vals = np.zeros(0, np.float64)
                fs.t0_ms, fs.period_ms, fs.count = s.t0_ms, s.period_ms, int(s.count)
            else:
                fs.type = 2
                vals = np.array(s.times_ms, np.float64)
            keep(vals)
            fs.n_values = len(vals)
            fs.values = _arr(vals, C.c_double)

        t = r.connection_table()
        n_cells = len(cell_kind)
        # label -> group per (dst kind); -1 where missing (the engine reports it)
        lut = np.full((max(nk, 1), max(len(t.labels), 1)), -1, np.int32)
        for k, ks in enumerate(r.kinds):
            for li, lab in enumerate(t.labels):
                lut[k, li] = ks.find_group(lab)
        # unresolved labels and out-of-range destinations or kinds pass through
        # as -1: the engine's build reports them in the reference's order
        # (engine.cpp:317-391), naming the label from the table below
        group = np.full(len(t), -1, np.int32)
        if len(t) and n_cells > 0 and int(t.dst.max()) < n_cells and int(cell_kind.max()) < nk \
                and int(t.label_idx.min()) >= 0 and int(t.label_idx.max()) < lut.shape[1]:
            # every destination and kind in range: one gather through the
            # flattened (kind, label) table
            flat_lut = lut.ravel()
            if lut.shape[1] == 1:
                idx = par_take(cell_kind.astype(np.int32), t.dst)
            else:
                idx = par_take(cell_kind.astype(np.int32) * np.int32(lut.shape[1]), t.dst)
                idx += t.label_idx
            par_take(flat_lut, idx, out=group)
        elif len(t):
            ok = t.dst < n_cells
            dk = np.full(len(t), -1, np.int64)
            dk[ok] = cell_kind[t.dst[ok]]
            ok &= (dk >= 0) & (dk < nk)
            group[ok] = lut[dk[ok], t.label_idx[ok]]
        label_idx = np.ascontiguousarray(t.label_idx, dtype=np.int32)
        label_txt = (C.c_char_p * max(len(t.labels), 1))(*[s.encode() for s in t.labels])
        for a in (t.from_source, t.src, t.dst, group, t.policy, t.weight, t.delay_ms, label_idx,
                  label_txt):
            keep(a)

        npb = len(r.probes)
        p_gid = np.array([p.gid for p in r.probes], np.uint32)
        p_what = np.array([int(p.what) for p in r.probes], np.uint8)
        p_comp = np.array([p.comp for p in r.probes], np.int32)
        p_sp = np.array([p.species for p in r.probes], np.int32)
        p_grp = np.full(npb, -1, np.int32)
        for i, p in enumerate(r.probes):
            if p.label:
                if p.gid >= n_cells:
                    raise EngineError("probe label not found")
                g = r.kinds[cell_kind[p.gid]].find_group(p.label)
                if g < 0:
                    raise EngineError("probe label not found")
                p_grp[i] = g
        p_inst = np.array([p.instance for p in r.probes], np.int32)
        p_every = np.array([p.every_steps for p in r.probes], np.int32)
        for a in (p_gid, p_what, p_comp, p_sp, p_grp, p_inst, p_every):
            keep(a)

        v = A.mcg_recipe()
        v.n_kinds = nk
        v.kinds = C.cast(kinds, C.POINTER(A.mcg_kind))
        v.n_cells = n_cells
        v.cell_kind = _arr(cell_kind, C.c_uint32)
        v.n_sources = ns
        v.sources = C.cast(srcs, C.POINTER(A.mcg_source))
        v.n_connections = len(t)
        v.conn_from_source = _arr(t.from_source, C.c_uint8)
        v.conn_src = _arr(t.src, C.c_uint32)
        v.conn_dst = _arr(t.dst, C.c_uint32)
        v.conn_group = _arr(group, C.c_int32)
        v.conn_policy = _arr(t.policy, C.c_uint8)
        v.conn_weight = _arr(t.weight, C.c_double)
        v.conn_delay_ms = _arr(t.delay_ms, C.c_double)
        v.n_probes = npb
        v.probe_gid = _arr(p_gid, C.c_uint32)
        v.probe_what = _arr(p_what, C.c_uint8)
        v.probe_comp = _arr(p_comp, C.c_int32)
        v.probe_species = _arr(p_sp, C.c_int32)
        v.probe_group = _arr(p_grp, C.c_int32)
        v.probe_instance = _arr(p_inst, C.c_int32)
        v.probe_every = _arr(p_every, C.c_int32)
        v.n_labels = len(t.labels)
        v.labels = C.cast(label_txt, C.POINTER(C.c_char_p))
        v.conn_label = _arr(label_idx, C.c_int32)
        self.view = v
        self.n_cells = n_cells
        self.recipe = r
