// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the parity checker, never shipped).
//
// A thin extern "C" layer over the UNMODIFIED reference (mcsim, compiled from
// /root/reference/proj/src/*.cpp by oracle/build_ref.sh into oracle/_ref/).
// It lets the Python tests drive the reference's own Engine with exactly the
// same flat recipe (include/mcg.h) that the B200 engine consumes, and exports
// the reference's recipe builders (network.cpp, bench.cpp) as flat recipes so
// both engines run the reference's own topology.  Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
#include <cstring>
#include <span>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "mcg.h"
#include "mcsim/bench.hpp"
#include "mcsim/engine.hpp"
#include "mcsim/mechanisms.hpp"
#include "mcsim/network.hpp"
#include "mcsim/rng.hpp"
#include "mcsim/tree_solver.hpp"

using namespace mcsim;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return MCG_OK;
  } catch (const NumericError& e) {
    g_err = e.what();
    return MCG_ERR_NUMERIC;
  } catch (const TargetingError& e) {
    g_err = e.what();
    return MCG_ERR_TARGETING;
  } catch (const MorphologyError& e) {
    g_err = e.what();
    return MCG_ERR_MORPHOLOGY;
  } catch (const EngineError& e) {
    g_err = e.what();
    return MCG_ERR_ENGINE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MCG_ERR_ARGUMENT;
  }
}

// placement labels of a flat recipe: a prefix no user label carries, so an
// unresolved label passed through by text never matches one
std::string glabel(int i) { return "\x1fg" + std::to_string(i); }
std::string slabel(int i) { return "s" + std::to_string(i); }

StcParams to_stc(const mcg_stc_params& p) {
  StcParams s;
  s.h0_mV = p.h0_mV; s.tau_h_ms = p.tau_h_ms; s.tau_c_ms = p.tau_c_ms;
  s.gamma_p = p.gamma_p; s.gamma_d = p.gamma_d; s.theta_p = p.theta_p;
  s.theta_d = p.theta_d; s.sigma_pl_mV = p.sigma_pl_mV; s.c_pre = p.c_pre;
  s.c_post = p.c_post; s.t_c_delay_ms = p.t_c_delay_ms; s.tau_z_ms = p.tau_z_ms;
  s.f_int = p.f_int; s.theta_tag_mV = p.theta_tag_mV; s.tau_p_ms = p.tau_p_ms;
  s.p_max = p.p_max; s.theta_pro_mV = p.theta_pro_mV;
  return s;
}
mcg_stc_params from_stc(const StcParams& s) {
  return {s.h0_mV, s.tau_h_ms, s.tau_c_ms, s.gamma_p, s.gamma_d, s.theta_p,
          s.theta_d, s.sigma_pl_mV, s.c_pre, s.c_post, s.t_c_delay_ms, s.tau_z_ms,
          s.f_int, s.theta_tag_mV, s.tau_p_ms, s.p_max, s.theta_pro_mV};
}

// flat (mcg.h) -> mcsim::Recipe, with synthetic unique labels
Recipe to_recipe(const mcg_recipe& f) {
  Recipe r;
  for (int k = 0; k < f.n_kinds; ++k) {
    const mcg_kind& fk = f.kinds[k];
    CellKindSpec ks;
    for (int s = 0; s < fk.n_segments; ++s) {
      Segment seg;
      if (fk.seg_parent[s] >= 0) seg.parent = static_cast<std::uint32_t>(fk.seg_parent[s]);
      seg.length_um = fk.seg_length_um[s];
      seg.radius_um = fk.seg_radius_um[s];
      seg.tag = static_cast<Region>(fk.seg_tag[s]);
      seg.parent_pos = fk.seg_parent_pos[s];
      ks.segments.push_back(seg);
    }
    ks.target_compartment_um = fk.target_compartment_um;
    if (fk.membrane == MCG_MEMBRANE_LIF) {
      const mcg_lif& l = fk.lif;
      LifMembrane m;
      m.tau_mem_ms = l.tau_mem_ms; m.r_mem_MOhm = l.r_mem_MOhm; m.v_rev_mV = l.v_rev_mV;
      m.v_reset_mV = l.v_reset_mV; m.v_thresh_mV = l.v_thresh_mV; m.t_ref_ms = l.t_ref_ms;
      m.r_axial_ohm_m = l.r_axial_ohm_m; m.i_bg_nA = l.i_bg_nA;
      m.sigma_bg_nA_sqrt_ms = l.sigma_bg_nA_sqrt_ms; m.bg_quiet_t0_ms = l.bg_quiet_t0_ms;
      m.bg_quiet_t1_ms = l.bg_quiet_t1_ms; m.noise_comp = l.noise_comp;
      m.detector_comp = l.detector_comp; m.exact = l.exact != 0;
      ks.membrane = m;
    } else if (fk.membrane == MCG_MEMBRANE_HH) {
      const mcg_hh& h = fk.hh;
      HhMembrane m;
      m.c_m = h.c_m; m.r_axial_ohm_m = h.r_axial_ohm_m; m.g_leak = h.g_leak;
      m.e_leak_mV = h.e_leak_mV; m.g_na = h.g_na; m.e_na_mV = h.e_na_mV; m.g_k = h.g_k;
      m.e_k_mV = h.e_k_mV; m.v_init_mV = h.v_init_mV; m.threshold_mV = h.threshold_mV;
      m.detector_comp = h.detector_comp;
      ks.membrane = m;
    } else {
      ks.membrane = NoMembrane{};
    }
    for (int s = 0; s < fk.n_species; ++s)
      ks.species.push_back(SpeciesSpec{slabel(s), fk.species[s].diffusivity,
                                       fk.species[s].decay_tau_ms, fk.species[s].init});
    ks.sps_species = fk.sps_idx >= 0 ? slabel(fk.sps_idx) : "__none__";
    ks.prp_species = fk.prp_idx >= 0 ? slabel(fk.prp_idx) : "__none__";
    for (int p = 0; p < fk.n_placements; ++p) {
      const mcg_placement& fp = fk.placements[p];
      PlacementSpec ps;
      ps.label = glabel(p);
      ps.comp = fp.comp;
      ps.count = fp.count;
      ps.syn.kind = static_cast<SynKind>(fp.syn.kind);
      ps.syn.tau_syn_ms = fp.syn.tau_syn_ms;
      ps.syn.e_rev_mV = fp.syn.e_rev_mV;
      const mcg_stdp_params& sp = fp.syn.stdp;
      ps.syn.stdp = StdpParams{sp.tau_pre_ms, sp.tau_post_ms, sp.a_pre_uS, sp.a_post_uS,
                               sp.w0_uS, sp.wmax_uS};
      const mcg_homeo_params& hp = fp.syn.homeo;
      ps.syn.homeo = HomeostasisParams{hp.dw_plus_nA, hp.dw_minus_nA, hp.w_init_nA,
                                       hp.wmax_nA, hp.w_varying_nA};
      ps.syn.stc = to_stc(fp.syn.stc);
      ps.syn.calcium_scale = fp.syn.calcium_scale;
      ks.placements.push_back(ps);
    }
    ks.prp.enabled = fk.prp_enabled != 0;
    ks.prp.comp = fk.prp_comp;
    r.kinds.push_back(std::move(ks));
  }
  r.cell_kind.assign(f.cell_kind, f.cell_kind + f.n_cells);
  for (int s = 0; s < f.n_sources; ++s) {
    const mcg_source& fs = f.sources[s];
    if (fs.type == MCG_SRC_POISSON) {
      PoissonSource ps;
      for (int i = 0; i + 2 < fs.n_values; i += 3)
        ps.windows.push_back(PoissonWindow{fs.values[i], fs.values[i + 1], fs.values[i + 2]});
      r.sources.push_back(ps);
    } else if (fs.type == MCG_SRC_REGULAR) {
      r.sources.push_back(RegularSource{fs.t0_ms, fs.period_ms, fs.count});
    } else {
      r.sources.push_back(ScriptedSource{std::vector<double>(fs.values, fs.values + fs.n_values)});
    }
  }
  r.connections.reserve(f.n_connections);
  for (int64_t i = 0; i < f.n_connections; ++i) {
    ConnectionSpec c;
    c.from_source = f.conn_from_source[i] != 0;
    c.src = f.conn_src[i];
    c.dst = f.conn_dst[i];
    c.label = f.conn_group[i] >= 0 ? glabel(f.conn_group[i])
              : (f.labels && f.conn_label && f.conn_label[i] >= 0 && f.conn_label[i] < f.n_labels)
                  ? std::string(f.labels[f.conn_label[i]]) : "__missing__";
    c.policy = static_cast<SelectionPolicy>(f.conn_policy[i]);
    c.weight = f.conn_weight[i];
    c.delay_ms = f.conn_delay_ms[i];
    r.connections.push_back(std::move(c));
  }
  for (int i = 0; i < f.n_probes; ++i) {
    ProbeSpec p;
    p.gid = f.probe_gid[i];
    p.what = static_cast<ProbeWhat>(f.probe_what[i]);
    p.comp = f.probe_comp[i];
    p.species = f.probe_species[i];
    p.label = f.probe_group[i] >= 0 ? glabel(f.probe_group[i]) : "";
    p.instance = f.probe_instance[i];
    p.every_steps = f.probe_every[i];
    r.probes.push_back(p);
  }
  return r;
}

}  // namespace

// ---- flat recipe export of the reference's own builders ------------------

struct ref_recipe {
  Recipe src;
  // owned storage behind the flat view
  std::vector<mcg_kind> kinds;
  std::vector<std::vector<int32_t>> seg_parent;
  std::vector<std::vector<double>> seg_len, seg_rad, seg_pos;
  std::vector<std::vector<uint8_t>> seg_tag;
  std::vector<std::vector<mcg_species>> species;
  std::vector<std::vector<mcg_placement>> placements;
  std::vector<std::vector<std::string>> labels;
  std::vector<mcg_source> sources;
  std::vector<std::vector<double>> source_vals;
  std::vector<uint8_t> c_from, c_policy;
  std::vector<uint32_t> c_src, c_dst;
  std::vector<int32_t> c_group;
  std::vector<double> c_w, c_d;
  std::vector<uint32_t> p_gid;
  std::vector<uint8_t> p_what;
  std::vector<int32_t> p_comp, p_species, p_group, p_instance, p_every;
  std::vector<uint32_t> cell_kind;
  mcg_recipe view{};
  // builder side info
  std::vector<uint32_t> as, ans, ctrl;
  double c_morpho = 1.0;
};

static void flatten(ref_recipe& h) {
  const Recipe& r = h.src;
  const std::size_t nk = r.kinds.size();
  h.kinds.resize(nk);
  h.seg_parent.resize(nk); h.seg_len.resize(nk); h.seg_rad.resize(nk);
  h.seg_pos.resize(nk); h.seg_tag.resize(nk); h.species.resize(nk);
  h.placements.resize(nk); h.labels.resize(nk);
  for (std::size_t k = 0; k < nk; ++k) {
    const CellKindSpec& ks = r.kinds[k];
    mcg_kind& fk = h.kinds[k];
    std::memset(&fk, 0, sizeof fk);
    for (const auto& s : ks.segments) {
      h.seg_parent[k].push_back(s.parent ? static_cast<int32_t>(*s.parent) : -1);
      h.seg_len[k].push_back(s.length_um);
      h.seg_rad[k].push_back(s.radius_um);
      h.seg_pos[k].push_back(s.parent_pos);
      h.seg_tag[k].push_back(static_cast<uint8_t>(s.tag));
    }
    fk.n_segments = static_cast<int32_t>(ks.segments.size());
    fk.seg_parent = h.seg_parent[k].data();
    fk.seg_length_um = h.seg_len[k].data();
    fk.seg_radius_um = h.seg_rad[k].data();
    fk.seg_parent_pos = h.seg_pos[k].data();
    fk.seg_tag = h.seg_tag[k].data();
    fk.target_compartment_um = ks.target_compartment_um;
    if (const auto* m = std::get_if<LifMembrane>(&ks.membrane)) {
      fk.membrane = MCG_MEMBRANE_LIF;
      fk.lif = {m->tau_mem_ms, m->r_mem_MOhm, m->v_rev_mV, m->v_reset_mV, m->v_thresh_mV,
                m->t_ref_ms, m->r_axial_ohm_m, m->i_bg_nA, m->sigma_bg_nA_sqrt_ms,
                m->bg_quiet_t0_ms, m->bg_quiet_t1_ms, m->noise_comp, m->detector_comp,
                m->exact ? 1 : 0};
    } else if (const auto* hm = std::get_if<HhMembrane>(&ks.membrane)) {
      fk.membrane = MCG_MEMBRANE_HH;
      fk.hh = {hm->c_m, hm->r_axial_ohm_m, hm->g_leak, hm->e_leak_mV, hm->g_na, hm->e_na_mV,
               hm->g_k, hm->e_k_mV, hm->v_init_mV, hm->threshold_mV, hm->detector_comp};
    } else {
      fk.membrane = MCG_MEMBRANE_NONE;
    }
    fk.sps_idx = fk.prp_idx = -1;
    for (std::size_t s = 0; s < ks.species.size(); ++s) {
      const auto& sp = ks.species[s];
      h.species[k].push_back({sp.diffusivity, sp.decay_tau_ms, sp.init});
      if (sp.name == ks.sps_species && fk.sps_idx < 0) fk.sps_idx = static_cast<int32_t>(s);
      if (sp.name == ks.prp_species && fk.prp_idx < 0) fk.prp_idx = static_cast<int32_t>(s);
    }
    // build_kind assigns the LAST matching species (engine.cpp:253-254)
    for (std::size_t s = 0; s < ks.species.size(); ++s) {
      if (ks.species[s].name == ks.sps_species) fk.sps_idx = static_cast<int32_t>(s);
      if (ks.species[s].name == ks.prp_species) fk.prp_idx = static_cast<int32_t>(s);
    }
    fk.n_species = static_cast<int32_t>(ks.species.size());
    fk.species = h.species[k].data();
    for (const auto& p : ks.placements) {
      mcg_placement fp;
      std::memset(&fp, 0, sizeof fp);
      fp.comp = p.comp;
      fp.count = p.count;
      fp.syn.kind = static_cast<int32_t>(p.syn.kind);
      fp.syn.tau_syn_ms = p.syn.tau_syn_ms;
      fp.syn.e_rev_mV = p.syn.e_rev_mV;
      fp.syn.stdp = {p.syn.stdp.tau_pre_ms, p.syn.stdp.tau_post_ms, p.syn.stdp.a_pre_uS,
                     p.syn.stdp.a_post_uS, p.syn.stdp.w0_uS, p.syn.stdp.wmax_uS};
      fp.syn.homeo = {p.syn.homeo.dw_plus_nA, p.syn.homeo.dw_minus_nA, p.syn.homeo.w_init_nA,
                      p.syn.homeo.wmax_nA, p.syn.homeo.w_varying_nA};
      fp.syn.stc = from_stc(p.syn.stc);
      fp.syn.calcium_scale = p.syn.calcium_scale;
      h.placements[k].push_back(fp);
      h.labels[k].push_back(p.label);
    }
    fk.n_placements = static_cast<int32_t>(ks.placements.size());
    fk.placements = h.placements[k].data();
    fk.prp_enabled = ks.prp.enabled ? 1 : 0;
    fk.prp_comp = ks.prp.comp;
  }
  h.source_vals.resize(r.sources.size());
  h.sources.resize(r.sources.size());
  for (std::size_t s = 0; s < r.sources.size(); ++s) {
    mcg_source& fs = h.sources[s];
    std::memset(&fs, 0, sizeof fs);
    if (const auto* ps = std::get_if<PoissonSource>(&r.sources[s])) {
      fs.type = MCG_SRC_POISSON;
      for (const auto& w : ps->windows) {
        h.source_vals[s].push_back(w.t0_ms);
        h.source_vals[s].push_back(w.t1_ms);
        h.source_vals[s].push_back(w.rate_hz);
      }
    } else if (const auto* rs = std::get_if<RegularSource>(&r.sources[s])) {
      fs.type = MCG_SRC_REGULAR;
      fs.t0_ms = rs->t0_ms;
      fs.period_ms = rs->period_ms;
      fs.count = rs->count;
    } else {
      fs.type = MCG_SRC_SCRIPTED;
      h.source_vals[s] = std::get<ScriptedSource>(r.sources[s]).times_ms;
    }
    fs.n_values = static_cast<int32_t>(h.source_vals[s].size());
    fs.values = h.source_vals[s].data();
  }
  const std::size_t nc = r.connections.size();
  h.c_from.resize(nc); h.c_policy.resize(nc); h.c_src.resize(nc); h.c_dst.resize(nc);
  h.c_group.resize(nc); h.c_w.resize(nc); h.c_d.resize(nc);
  for (std::size_t i = 0; i < nc; ++i) {
    const auto& c = r.connections[i];
    h.c_from[i] = c.from_source;
    h.c_policy[i] = static_cast<uint8_t>(c.policy);
    h.c_src[i] = c.src;
    h.c_dst[i] = c.dst;
    h.c_w[i] = c.weight;
    h.c_d[i] = c.delay_ms;
    int32_t g = -1;
    if (c.dst < r.cell_kind.size() && r.cell_kind[c.dst] < nk) {
      const auto& lab = h.labels[r.cell_kind[c.dst]];
      for (std::size_t j = 0; j < lab.size(); ++j)
        if (lab[j] == c.label) { g = static_cast<int32_t>(j); break; }
    }
    h.c_group[i] = g;
  }
  for (const auto& p : r.probes) {
    h.p_gid.push_back(p.gid);
    h.p_what.push_back(static_cast<uint8_t>(p.what));
    h.p_comp.push_back(p.comp);
    h.p_species.push_back(p.species);
    int32_t g = -1;
    if (!p.label.empty() && p.gid < r.cell_kind.size()) {
      const auto& lab = h.labels[r.cell_kind[p.gid]];
      for (std::size_t j = 0; j < lab.size(); ++j)
        if (lab[j] == p.label) { g = static_cast<int32_t>(j); break; }
    }
    h.p_group.push_back(g);
    h.p_instance.push_back(p.instance);
    h.p_every.push_back(p.every_steps);
  }
  h.cell_kind = r.cell_kind;
  mcg_recipe& v = h.view;
  v.n_kinds = static_cast<int32_t>(nk);
  v.kinds = h.kinds.data();
  v.n_cells = static_cast<int32_t>(h.cell_kind.size());
  v.cell_kind = h.cell_kind.data();
  v.n_sources = static_cast<int32_t>(h.sources.size());
  v.sources = h.sources.data();
  v.n_connections = static_cast<int64_t>(nc);
  v.conn_from_source = h.c_from.data();
  v.conn_src = h.c_src.data();
  v.conn_dst = h.c_dst.data();
  v.conn_group = h.c_group.data();
  v.conn_policy = h.c_policy.data();
  v.conn_weight = h.c_w.data();
  v.conn_delay_ms = h.c_d.data();
  v.n_probes = static_cast<int32_t>(h.p_gid.size());
  v.probe_gid = h.p_gid.data();
  v.probe_what = h.p_what.data();
  v.probe_comp = h.p_comp.data();
  v.probe_species = h.p_species.data();
  v.probe_group = h.p_group.data();
  v.probe_instance = h.p_instance.data();
  v.probe_every = h.p_every.data();
}

// ConsolidationConfig (network.hpp:152-196) minus the optional file paths
struct ref_consolidation_cfg {
  int32_t n_cells, n_exc;
  double p_conn;
  int32_t pattern;
  uint64_t seed;
  int32_t workers;
  double dt_ms;
  int32_t multi_compartment, cell_size, dend_size;
  double d_p, d_sps;
  mcg_stc_params stc;
  double in_vivo_factor;
  double tau_mem_ms, r_mem_MOhm, v_rev_mV, v_reset_mV, v_thresh_mV, t_ref_ms;
  double i_bg_nA, sigma_bg_nA_sqrt_ms, w_rec_scale, w_ei_mV, w_ie_mV, w_ii_mV, delay_ms;
  int32_t n_stim_sources;
  double t_learn_ms, learn_duration_ms, learn_rate_hz, recall_duration_ms, recall_rate_hz;
  double w_stim_mV, coarse_dt_ms;
};

static ConsolidationConfig to_cfg(const ref_consolidation_cfg& c) {
  ConsolidationConfig k;
  k.n_cells = c.n_cells; k.n_exc = c.n_exc; k.p_conn = c.p_conn; k.pattern = c.pattern;
  k.seed = c.seed; k.workers = c.workers; k.dt_ms = c.dt_ms;
  k.multi_compartment = c.multi_compartment != 0;
  k.cell_size = c.cell_size ? CellSize::large_cells : CellSize::small_cells;
  k.dend_size = c.dend_size ? DendriteSize::large_dendrites : DendriteSize::small_dendrites;
  k.d_p = c.d_p; k.d_sps = c.d_sps; k.stc = to_stc(c.stc); k.in_vivo_factor = c.in_vivo_factor;
  k.tau_mem_ms = c.tau_mem_ms; k.r_mem_MOhm = c.r_mem_MOhm; k.v_rev_mV = c.v_rev_mV;
  k.v_reset_mV = c.v_reset_mV; k.v_thresh_mV = c.v_thresh_mV; k.t_ref_ms = c.t_ref_ms;
  k.i_bg_nA = c.i_bg_nA; k.sigma_bg_nA_sqrt_ms = c.sigma_bg_nA_sqrt_ms;
  k.w_rec_scale = c.w_rec_scale; k.w_ei_mV = c.w_ei_mV; k.w_ie_mV = c.w_ie_mV;
  k.w_ii_mV = c.w_ii_mV; k.delay_ms = c.delay_ms; k.n_stim_sources = c.n_stim_sources;
  k.t_learn_ms = c.t_learn_ms; k.learn_duration_ms = c.learn_duration_ms;
  k.learn_rate_hz = c.learn_rate_hz; k.recall_duration_ms = c.recall_duration_ms;
  k.recall_rate_hz = c.recall_rate_hz; k.w_stim_mV = c.w_stim_mV;
  k.coarse_dt_ms = c.coarse_dt_ms;
  return k;
}

// BusyringSpec (bench.hpp:20-34)
struct ref_busyring_cfg {
  int32_t n_cells, ring_size, random_per_cell;
  double delay_ms, ring_weight_uS, tau_syn_ms;
  int32_t tree_depth, stdp_on_random;
  mcg_stdp_params stdp;
  double duration_ms, dt_ms;
  uint64_t seed;
  int32_t workers;
};

static BusyringSpec to_spec(const ref_busyring_cfg& c) {
  BusyringSpec s;
  s.n_cells = c.n_cells; s.ring_size = c.ring_size; s.random_per_cell = c.random_per_cell;
  s.delay_ms = c.delay_ms; s.ring_weight_uS = c.ring_weight_uS; s.tau_syn_ms = c.tau_syn_ms;
  s.tree_depth = c.tree_depth; s.stdp_on_random = c.stdp_on_random != 0;
  s.stdp = StdpParams{c.stdp.tau_pre_ms, c.stdp.tau_post_ms, c.stdp.a_pre_uS, c.stdp.a_post_uS,
                      c.stdp.w0_uS, c.stdp.wmax_uS};
  s.duration_ms = c.duration_ms; s.dt_ms = c.dt_ms; s.seed = c.seed; s.workers = c.workers;
  return s;
}

struct ref_engine {
  std::unique_ptr<Engine> eng;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// defaults of the reference's config structs, so Python mirrors start equal
void ref_default_consolidation(ref_consolidation_cfg* out) {
  ConsolidationConfig k;
  ref_consolidation_cfg& c = *out;
  c.n_cells = k.n_cells; c.n_exc = k.n_exc; c.p_conn = k.p_conn; c.pattern = k.pattern;
  c.seed = k.seed; c.workers = k.workers; c.dt_ms = k.dt_ms;
  c.multi_compartment = k.multi_compartment; c.cell_size = k.cell_size == CellSize::large_cells;
  c.dend_size = k.dend_size == DendriteSize::large_dendrites;
  c.d_p = k.d_p; c.d_sps = k.d_sps; c.stc = from_stc(k.stc); c.in_vivo_factor = k.in_vivo_factor;
  c.tau_mem_ms = k.tau_mem_ms; c.r_mem_MOhm = k.r_mem_MOhm; c.v_rev_mV = k.v_rev_mV;
  c.v_reset_mV = k.v_reset_mV; c.v_thresh_mV = k.v_thresh_mV; c.t_ref_ms = k.t_ref_ms;
  c.i_bg_nA = k.i_bg_nA; c.sigma_bg_nA_sqrt_ms = k.sigma_bg_nA_sqrt_ms;
  c.w_rec_scale = k.w_rec_scale; c.w_ei_mV = k.w_ei_mV; c.w_ie_mV = k.w_ie_mV;
  c.w_ii_mV = k.w_ii_mV; c.delay_ms = k.delay_ms; c.n_stim_sources = k.n_stim_sources;
  c.t_learn_ms = k.t_learn_ms; c.learn_duration_ms = k.learn_duration_ms;
  c.learn_rate_hz = k.learn_rate_hz; c.recall_duration_ms = k.recall_duration_ms;
  c.recall_rate_hz = k.recall_rate_hz; c.w_stim_mV = k.w_stim_mV;
  c.coarse_dt_ms = k.coarse_dt_ms;
}

void ref_default_busyring(ref_busyring_cfg* out) {
  BusyringSpec s = default_busyring();
  ref_busyring_cfg& c = *out;
  c.n_cells = s.n_cells; c.ring_size = s.ring_size; c.random_per_cell = s.random_per_cell;
  c.delay_ms = s.delay_ms; c.ring_weight_uS = s.ring_weight_uS; c.tau_syn_ms = s.tau_syn_ms;
  c.tree_depth = s.tree_depth; c.stdp_on_random = s.stdp_on_random;
  c.stdp = {s.stdp.tau_pre_ms, s.stdp.tau_post_ms, s.stdp.a_pre_uS, s.stdp.a_post_uS,
            s.stdp.w0_uS, s.stdp.wmax_uS};
  c.duration_ms = s.duration_ms; c.dt_ms = s.dt_ms; c.seed = s.seed; c.workers = s.workers;
}

void ref_default_stc_params(mcg_stc_params* out) { *out = from_stc(StcParams{}); }

int ref_build_consolidation(const ref_consolidation_cfg* cfg, int eight_hour, ref_recipe** out) {
  return guard([&] {
    auto h = std::make_unique<ref_recipe>();
    auto b = build_consolidation_network(to_cfg(*cfg), eight_hour != 0);
    h->src = std::move(b.recipe);
    h->as = b.as; h->ans = b.ans; h->ctrl = b.ctrl; h->c_morpho = b.c_morpho;
    flatten(*h);
    *out = h.release();
  });
}

int ref_build_busyring(const ref_busyring_cfg* cfg, ref_recipe** out) {
  return guard([&] {
    auto h = std::make_unique<ref_recipe>();
    h->src = build_busyring(to_spec(*cfg));
    flatten(*h);
    *out = h.release();
  });
}

double ref_calibrate_ring_weight(const ref_busyring_cfg* cfg) {
  double w = 0;
  guard([&] { w = calibrate_ring_weight(to_spec(*cfg)); });
  return w;
}

int ref_recipe_from_flat(const mcg_recipe* f, ref_recipe** out) {
  return guard([&] {
    auto h = std::make_unique<ref_recipe>();
    h->src = to_recipe(*f);
    flatten(*h);
    *out = h.release();
  });
}

const mcg_recipe* ref_recipe_view(const ref_recipe* h) { return &h->view; }
const char* ref_recipe_label(const ref_recipe* h, int kind, int placement) {
  return h->labels[kind][placement].c_str();
}
double ref_recipe_c_morpho(const ref_recipe* h) { return h->c_morpho; }
void ref_recipe_destroy(ref_recipe* h) { delete h; }

int ref_engine_create(const mcg_recipe* f, double dt_ms, uint64_t seed, int workers,
                      ref_engine** out) {
  return guard([&] {
    auto e = std::make_unique<ref_engine>();
    e->eng = std::make_unique<Engine>(to_recipe(*f), EngineOptions{dt_ms, seed, workers});
    *out = e.release();
  });
}
void ref_engine_destroy(ref_engine* e) { delete e; }
int ref_advance_to(ref_engine* e, double t) { return guard([&] { e->eng->advance_to(t); }); }
int ref_fast_forward_to(ref_engine* e, double t, double c) {
  return guard([&] { e->eng->fast_forward_to(t, c); });
}
int64_t ref_step(ref_engine* e) { return e->eng->step(); }
double ref_time_ms(ref_engine* e) { return e->eng->time_ms(); }
int64_t ref_num_spikes(ref_engine* e) { return static_cast<int64_t>(e->eng->spikes().size()); }
void ref_get_spikes(ref_engine* e, double* t, uint32_t* gid) {
  const auto& s = e->eng->spikes();
  for (std::size_t i = 0; i < s.size(); ++i) {
    t[i] = s[i].t_ms;
    gid[i] = s[i].gid;
  }
}
void ref_clear_spikes(ref_engine* e) { e->eng->clear_spikes(); }
int64_t ref_trace_len(ref_engine* e, int p) {
  return static_cast<int64_t>(e->eng->traces()[p].size());
}
void ref_get_trace(ref_engine* e, int p, double* t, double* v) {
  const auto& tr = e->eng->traces()[p];
  for (std::size_t i = 0; i < tr.size(); ++i) {
    t[i] = tr[i].first;
    v[i] = tr[i].second;
  }
}
int32_t ref_cell_ncomp(ref_engine* e, uint32_t gid) {
  return static_cast<int32_t>(e->eng->grid_of(gid).size());
}
int32_t ref_cell_ngroups(ref_engine* e, uint32_t gid) {
  return static_cast<int32_t>(e->eng->cell(gid).groups.size());
}
int64_t ref_group_size(ref_engine* e, uint32_t gid, int32_t g) {
  return e->eng->cell(gid).groups[g].size();
}
int32_t ref_cell_parent(ref_engine* e, uint32_t gid, int32_t comp) {
  return e->eng->grid_of(gid).parent[comp];
}

// same field numbering as mcg_read_state (include/mcg.h)
int ref_read_state(ref_engine* e, int field, uint32_t gid, int index, int64_t off, int64_t n,
                   void* out) {
  return guard([&] {
    const CellRT& c = e->eng->cell(gid);
    double* d = static_cast<double*>(out);
    int64_t* q = static_cast<int64_t*>(out);
    int32_t* ii = static_cast<int32_t*>(out);
    auto fd = [&](const std::vector<double>& v) {
      for (int64_t i = 0; i < n; ++i) d[i] = v.at(off + i);
    };
    switch (field) {
      case MCG_FIELD_V: fd(c.v_mV); return;
      case MCG_FIELD_SPECIES: fd(c.species.at(index)); return;
      case MCG_FIELD_HH_M: fd(c.hh_m); return;
      case MCG_FIELD_HH_H: fd(c.hh_h); return;
      case MCG_FIELD_HH_N: fd(c.hh_n); return;
      case MCG_FIELD_DETECTOR_PREV_V: d[0] = c.detector_prev_v; return;
      case MCG_FIELD_REFRACTORY_UNTIL: q[0] = c.refractory_until; return;
      case MCG_FIELD_DETECTOR_ARMED: q[0] = c.detector_armed ? 1 : 0; return;
      case MCG_FIELD_INTERNAL_SEQ: q[0] = c.internal_seq; return;
      default: break;
    }
    const SynGroupRT& g = c.groups.at(index);
    for (int64_t i = 0; i < n; ++i) {
      const std::size_t k = static_cast<std::size_t>(off + i);
      switch (field) {
        case MCG_FIELD_SYN_COMP: ii[i] = g.comp.at(k); break;
        case MCG_FIELD_SYN_WEIGHT: d[i] = g.weight.at(k); break;
        case MCG_FIELD_SYN_KERNEL: d[i] = g.kernel.at(k); break;
        case MCG_FIELD_STDP_A_PRE: d[i] = g.stdp.at(k).a_pre; break;
        case MCG_FIELD_STDP_A_POST: d[i] = g.stdp.at(k).a_post; break;
        case MCG_FIELD_STDP_W: d[i] = g.stdp.at(k).w; break;
        case MCG_FIELD_STDP_LAST: q[i] = g.stdp_last_step.at(k); break;
        case MCG_FIELD_HOMEO_W: d[i] = g.homeo.at(k).w; break;
        case MCG_FIELD_STC_H: d[i] = g.stc.at(k).h; break;
        case MCG_FIELD_STC_Z: d[i] = g.stc.at(k).z; break;
        case MCG_FIELD_STC_C: d[i] = g.stc.at(k).c; break;
        case MCG_FIELD_STC_SPS_ABS: d[i] = g.sps_abs.at(k); break;
        default: throw std::invalid_argument("unknown field");
      }
    }
  });
}

// ---- numerics primitives (pin the restatement and the device ports) -------

void ref_threefry(const uint64_t key[4], const uint64_t ctr[4], uint64_t out[4]) {
  RngKey k{{key[0], key[1], key[2], key[3]}};
  RngCounter c{{ctr[0], ctr[1], ctr[2], ctr[3]}};
  const auto x = threefry4x64(k, c);
  for (int i = 0; i < 4; ++i) out[i] = x[i];
}
double ref_uniform_for(const uint64_t key[4], uint64_t n) {
  return uniform_for(RngKey{{key[0], key[1], key[2], key[3]}}, n);
}
double ref_normal_for(const uint64_t key[4], uint64_t n) {
  return normal_for(RngKey{{key[0], key[1], key[2], key[3]}}, n);
}
int ref_er_connected(uint64_t seed, uint32_t src, uint32_t dst, uint32_t n, double p) {
  return er_connected(seed, src, dst, n, p) ? 1 : 0;
}

// solve_tree on an explicit parent array (tree_solver.cpp:46-74)
int ref_solve_tree(int n, const int32_t* parent, const double* cap, const double* g,
                   const double* coupling, const double* rhs, double* v) {
  return guard([&] {
    CompartmentGrid grid;
    grid.parent.assign(parent, parent + n);
    grid.length_um.assign(n, 1.0);
    solve_tree(grid, std::span<const double>(cap, n), std::span<const double>(g, n),
               std::span<const double>(coupling, n), std::span<const double>(rhs, n),
               std::span<double>(v, n));
  });
}

// discretize (morphology.cpp:67-143): returns the compartment count, fills
// up to `cap` entries of parent / length / area / xs / volume
int ref_discretize(const mcg_kind* k, int cap, int32_t* parent, double* length, double* area,
                   double* xs, double* volume) {
  int n = -1;
  guard([&] {
    std::vector<Segment> segs;
    for (int s = 0; s < k->n_segments; ++s) {
      Segment seg;
      if (k->seg_parent[s] >= 0) seg.parent = static_cast<std::uint32_t>(k->seg_parent[s]);
      seg.length_um = k->seg_length_um[s];
      seg.radius_um = k->seg_radius_um[s];
      seg.tag = static_cast<Region>(k->seg_tag[s]);
      seg.parent_pos = k->seg_parent_pos[s];
      segs.push_back(seg);
    }
    const auto g = discretize(segs, k->target_compartment_um);
    n = g.size();
    for (int i = 0; i < n && i < cap; ++i) {
      parent[i] = g.parent[i];
      length[i] = g.length_um[i];
      area[i] = g.lateral_area_um2[i];
      xs[i] = g.cross_section_um2[i];
      volume[i] = g.volume_um3[i];
    }
  });
  return n;
}

// run_stc_protocol (network.cpp:353-399) with default StcSingleConfig
int ref_run_stc_protocol(int proto, uint64_t trial, double* h_final, double* z_final,
                         double* p_final) {
  return guard([&] {
    StcSingleConfig cfg;
    const auto r = run_stc_protocol(cfg, static_cast<StcProtocol>(proto), trial);
    *h_final = r.h_final;
    *z_final = r.z_final;
    *p_final = r.p_final;
  });
}

// gb_pairing_trial / gb_dp_curve / stdp_window (mechanisms.cpp:9-119)
static GbParams gb_from(const mcg_gb_params* q) {
  GbParams p;
  p.tau_w_ms = q->tau_w_ms;
  p.w_star = q->w_star;
  p.gamma_p = q->gamma_p;
  p.gamma_d = q->gamma_d;
  p.theta_p = q->theta_p;
  p.theta_d = q->theta_d;
  p.sigma_pl = q->sigma_pl;
  p.tau_c_ms = q->tau_c_ms;
  p.c_pre = q->c_pre;
  p.c_post = q->c_post;
  p.t_c_delay_ms = q->t_c_delay_ms;
  return p;
}
static GbPairingProtocol proto_from(const mcg_gb_protocol* q) {
  GbPairingProtocol r;
  r.n_pairs = q->n_pairs;
  r.period_ms = q->period_ms;
  r.settle_ms = q->settle_ms;
  r.dt_ms = q->dt_ms;
  r.trials = q->trials;
  r.seed = q->seed;
  return r;
}
double ref_gb_pairing_trial(const mcg_gb_params* p, double delta_t_ms, const mcg_gb_protocol* proto,
                            uint64_t trial, uint64_t delta_index, double* w0) {
  return gb_pairing_trial(gb_from(p), delta_t_ms, proto_from(proto), trial, delta_index, w0);
}
int ref_gb_dp_curve(const mcg_gb_params* p, const double* deltas, int n, const mcg_gb_protocol* proto,
                    mcg_gb_point* out) {
  return guard([&] {
    const auto c = gb_dp_curve(gb_from(p), std::vector<double>(deltas, deltas + n), proto_from(proto));
    for (int i = 0; i < n; ++i) {
      out[i].delta_t_ms = c[i].delta_t_ms;
      out[i].mean_initial = c[i].mean_initial;
      out[i].mean_final = c[i].mean_final;
      out[i].mean_change = c[i].mean_change;
      out[i].change_ci_half = c[i].change_ci_half;
      out[i].ratio = c[i].ratio;
    }
  });
}
double ref_stdp_window(const mcg_stdp_params* q, double delta_t_ms, int n_pairs, double period_ms) {
  StdpParams p;
  p.tau_pre_ms = q->tau_pre_ms;
  p.tau_post_ms = q->tau_post_ms;
  p.a_pre_uS = q->a_pre_uS;
  p.a_post_uS = q->a_post_uS;
  p.w0_uS = q->w0_uS;
  p.wmax_uS = q->wmax_uS;
  return stdp_window(delta_t_ms, p, n_pairs, period_ms);
}

// Engine::make_checkpoint + serialize / deserialize + restore (engine.cpp:1036-1325)
int ref_make_checkpoint(ref_engine* e, uint8_t* buf, int64_t cap, int64_t* size) {
  return guard([&] {
    const auto b = e->eng->make_checkpoint().serialize();
    *size = static_cast<int64_t>(b.size());
    if (buf) {
      if (cap < *size) throw EngineError("checkpoint: buffer too small");
      std::memcpy(buf, b.data(), b.size());
    }
  });
}
int ref_restore(ref_engine* e, const uint8_t* buf, int64_t size) {
  return guard([&] {
    e->eng->restore(Checkpoint::deserialize(std::span<const uint8_t>(buf, static_cast<size_t>(size))));
  });
}

// direct writes of cell(gid).v_mV (the tests mutate the reference's CellRT)
int ref_write_v(ref_engine* e, uint32_t gid, const double* v, int64_t n) {
  return guard([&] {
    auto& c = e->eng->cell(gid);
    if (static_cast<int64_t>(c.v_mV.size()) != n) throw EngineError("write_v: size mismatch");
    for (int64_t i = 0; i < n; ++i) c.v_mV[i] = v[i];
  });
}

}  // extern "C"
