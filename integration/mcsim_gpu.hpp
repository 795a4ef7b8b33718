// mcsim_gpu.hpp — drop-in replacement of mcsim::Engine (engine.hpp:126-167)
// backed by the B200 engine's C ABI (include/mcg.h, libmcg.so).
//
// A maintainer of the reference adds this header to its include path, links
// libmcg.so, and swaps `mcsim::Engine` for `mcsim_gpu::Engine`:
//   * the constructor takes the same Recipe / EngineOptions aggregates;
//   * time_ms / dt_ms / step / advance_to / fast_forward_to / spikes /
//     clear_spikes / num_cells / traces keep their signatures and semantics;
//   * cell(gid) returns a CellRT mirror read from the device (v_mV, species,
//     HH gates, detector state, synapse groups with weights, kernels, STDP,
//     homeostasis and STC state); edits made through it are written back to
//     the device before the next advance (the mirror is lazily synced, as the
//     reference's observers expect: test_engine.cpp:106, 178-180, 213-226);
//   * failures rethrow the reference's exception types with its messages
//     (EngineError, NumericError, TargetingError, MorphologyError).
// make_checkpoint / restore exchange MCSCKPT1 bytes through the reference's
// own Checkpoint type; either engine restores the other's.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <variant>
#include <vector>

#include "mcg.h"
#include "mcsim/engine.hpp"
#include "mcsim/morphology.hpp"
#include "mcsim/recipe.hpp"
#include "mcsim/tree_solver.hpp"

namespace mcsim_gpu {

[[noreturn]] inline void rethrow(mcg_status st) {
  const std::string msg = mcg_last_error();
  switch (st) {
    case MCG_ERR_NUMERIC: throw mcsim::NumericError(msg);
    case MCG_ERR_TARGETING: throw mcsim::TargetingError(msg);
    case MCG_ERR_MORPHOLOGY: throw mcsim::MorphologyError(msg);
    default: throw mcsim::EngineError(msg);
  }
}
inline void check(mcg_status st) {
  if (st != MCG_OK) rethrow(st);
}

// mcsim::Recipe -> the ABI's flat recipe (labels resolved to placement
// indices; species names to indices with build_kind's last-match rule,
// engine.cpp:253-254).  Owns every array the view points into.
class FlatRecipe {
 public:
  explicit FlatRecipe(const mcsim::Recipe& r) {
    const std::size_t nk = r.kinds.size();
    kinds_.resize(nk);
    seg_parent_.resize(nk);
    seg_len_.resize(nk);
    seg_rad_.resize(nk);
    seg_pos_.resize(nk);
    seg_tag_.resize(nk);
    species_.resize(nk);
    placements_.resize(nk);
    labels_.resize(nk);
    for (std::size_t k = 0; k < nk; ++k) flatten_kind(r.kinds[k], k);
    source_vals_.resize(r.sources.size());
    sources_.resize(r.sources.size());
    for (std::size_t s = 0; s < r.sources.size(); ++s) flatten_source(r.sources[s], s);
    for (const auto& c : r.connections) {
      c_from_.push_back(c.from_source ? 1 : 0);
      c_src_.push_back(c.src);
      c_dst_.push_back(c.dst);
      c_group_.push_back(label_index(r, c.dst, c.label));
      if (c_group_.back() < 0) {  // unresolved: keep the text for the build's message
        c_label_.resize(c_group_.size(), -1);
        c_label_.back() = static_cast<int32_t>(miss_text_.size());
        miss_text_.push_back(c.label);
      }
      c_policy_.push_back(static_cast<uint8_t>(c.policy));
      c_w_.push_back(c.weight);
      c_d_.push_back(c.delay_ms);
    }
    for (const auto& p : r.probes) {
      p_gid_.push_back(p.gid);
      p_what_.push_back(static_cast<uint8_t>(p.what));
      p_comp_.push_back(p.comp);
      p_species_.push_back(p.species);
      p_group_.push_back(p.label.empty() ? -1 : label_index(r, p.gid, p.label));
      p_instance_.push_back(p.instance);
      p_every_.push_back(p.every_steps);
    }
    cell_kind_ = r.cell_kind;
    view_.n_kinds = static_cast<int32_t>(nk);
    view_.kinds = kinds_.data();
    view_.n_cells = static_cast<int32_t>(cell_kind_.size());
    view_.cell_kind = cell_kind_.data();
    view_.n_sources = static_cast<int32_t>(sources_.size());
    view_.sources = sources_.data();
    view_.n_connections = static_cast<int64_t>(c_src_.size());
    view_.conn_from_source = c_from_.data();
    view_.conn_src = c_src_.data();
    view_.conn_dst = c_dst_.data();
    view_.conn_group = c_group_.data();
    if (!miss_text_.empty()) {
      c_label_.resize(c_group_.size(), -1);
      for (const auto& t : miss_text_) miss_ptr_.push_back(t.c_str());
      view_.n_labels = static_cast<int32_t>(miss_ptr_.size());
      view_.labels = miss_ptr_.data();
      view_.conn_label = c_label_.data();
    }
    view_.conn_policy = c_policy_.data();
    view_.conn_weight = c_w_.data();
    view_.conn_delay_ms = c_d_.data();
    view_.n_probes = static_cast<int32_t>(p_gid_.size());
    view_.probe_gid = p_gid_.data();
    view_.probe_what = p_what_.data();
    view_.probe_comp = p_comp_.data();
    view_.probe_species = p_species_.data();
    view_.probe_group = p_group_.data();
    view_.probe_instance = p_instance_.data();
    view_.probe_every = p_every_.data();
  }
  const mcg_recipe* view() const { return &view_; }

 private:
  int32_t label_index(const mcsim::Recipe& r, uint32_t gid, const std::string& label) const {
    if (gid >= r.cell_kind.size() || r.cell_kind[gid] >= labels_.size()) return -1;
    const auto& lab = labels_[r.cell_kind[gid]];
    for (std::size_t j = 0; j < lab.size(); ++j)
      if (lab[j] == label) return static_cast<int32_t>(j);
    return -1;
  }

  void flatten_kind(const mcsim::CellKindSpec& ks, std::size_t k) {
    mcg_kind& fk = kinds_[k];
    std::memset(&fk, 0, sizeof fk);
    for (const auto& s : ks.segments) {
      seg_parent_[k].push_back(s.parent ? static_cast<int32_t>(*s.parent) : -1);
      seg_len_[k].push_back(s.length_um);
      seg_rad_[k].push_back(s.radius_um);
      seg_pos_[k].push_back(s.parent_pos);
      seg_tag_[k].push_back(static_cast<uint8_t>(s.tag));
    }
    fk.n_segments = static_cast<int32_t>(ks.segments.size());
    fk.seg_parent = seg_parent_[k].data();
    fk.seg_length_um = seg_len_[k].data();
    fk.seg_radius_um = seg_rad_[k].data();
    fk.seg_parent_pos = seg_pos_[k].data();
    fk.seg_tag = seg_tag_[k].data();
    fk.target_compartment_um = ks.target_compartment_um;
    if (const auto* m = std::get_if<mcsim::LifMembrane>(&ks.membrane)) {
      fk.membrane = MCG_MEMBRANE_LIF;
      fk.lif = {m->tau_mem_ms, m->r_mem_MOhm, m->v_rev_mV,  m->v_reset_mV,
                m->v_thresh_mV, m->t_ref_ms, m->r_axial_ohm_m, m->i_bg_nA,
                m->sigma_bg_nA_sqrt_ms, m->bg_quiet_t0_ms, m->bg_quiet_t1_ms,
                m->noise_comp, m->detector_comp, m->exact ? 1 : 0};
    } else if (const auto* h = std::get_if<mcsim::HhMembrane>(&ks.membrane)) {
      fk.membrane = MCG_MEMBRANE_HH;
      fk.hh = {h->c_m,  h->r_axial_ohm_m, h->g_leak,    h->e_leak_mV,    h->g_na, h->e_na_mV,
               h->g_k, h->e_k_mV,         h->v_init_mV, h->threshold_mV, h->detector_comp};
    } else {
      fk.membrane = MCG_MEMBRANE_NONE;
    }
    fk.sps_idx = fk.prp_idx = -1;
    for (std::size_t s = 0; s < ks.species.size(); ++s) {
      const auto& sp = ks.species[s];
      species_[k].push_back({sp.diffusivity, sp.decay_tau_ms, sp.init});
      if (sp.name == ks.sps_species) fk.sps_idx = static_cast<int32_t>(s);
      if (sp.name == ks.prp_species) fk.prp_idx = static_cast<int32_t>(s);
    }
    fk.n_species = static_cast<int32_t>(ks.species.size());
    fk.species = species_[k].data();
    for (const auto& p : ks.placements) {
      mcg_placement fp;
      std::memset(&fp, 0, sizeof fp);
      fp.comp = p.comp;
      fp.count = p.count;
      const mcsim::SynSpec& y = p.syn;
      fp.syn.kind = static_cast<int32_t>(y.kind);
      fp.syn.tau_syn_ms = y.tau_syn_ms;
      fp.syn.e_rev_mV = y.e_rev_mV;
      fp.syn.stdp = {y.stdp.tau_pre_ms, y.stdp.tau_post_ms, y.stdp.a_pre_uS,
                     y.stdp.a_post_uS,  y.stdp.w0_uS,       y.stdp.wmax_uS};
      fp.syn.homeo = {y.homeo.dw_plus_nA, y.homeo.dw_minus_nA, y.homeo.w_init_nA,
                      y.homeo.wmax_nA, y.homeo.w_varying_nA};
      const mcsim::StcParams& c = y.stc;
      fp.syn.stc = {c.h0_mV,    c.tau_h_ms,    c.tau_c_ms, c.gamma_p,      c.gamma_d, c.theta_p,
                    c.theta_d,  c.sigma_pl_mV, c.c_pre,    c.c_post,       c.t_c_delay_ms,
                    c.tau_z_ms, c.f_int,       c.theta_tag_mV, c.tau_p_ms, c.p_max,
                    c.theta_pro_mV};
      fp.syn.calcium_scale = y.calcium_scale;
      placements_[k].push_back(fp);
      labels_[k].push_back(p.label);
    }
    fk.n_placements = static_cast<int32_t>(ks.placements.size());
    fk.placements = placements_[k].data();
    fk.prp_enabled = ks.prp.enabled ? 1 : 0;
    fk.prp_comp = ks.prp.comp;
  }

  void flatten_source(const mcsim::SourceSpec& src, std::size_t s) {
    mcg_source& fs = sources_[s];
    std::memset(&fs, 0, sizeof fs);
    if (const auto* ps = std::get_if<mcsim::PoissonSource>(&src)) {
      fs.type = MCG_SRC_POISSON;
      for (const auto& w : ps->windows) {
        source_vals_[s].push_back(w.t0_ms);
        source_vals_[s].push_back(w.t1_ms);
        source_vals_[s].push_back(w.rate_hz);
      }
    } else if (const auto* rs = std::get_if<mcsim::RegularSource>(&src)) {
      fs.type = MCG_SRC_REGULAR;
      fs.t0_ms = rs->t0_ms;
      fs.period_ms = rs->period_ms;
      fs.count = rs->count;
    } else {
      fs.type = MCG_SRC_SCRIPTED;
      source_vals_[s] = std::get<mcsim::ScriptedSource>(src).times_ms;
    }
    fs.n_values = static_cast<int32_t>(source_vals_[s].size());
    fs.values = source_vals_[s].data();
  }

  std::vector<mcg_kind> kinds_;
  std::vector<std::vector<int32_t>> seg_parent_;
  std::vector<std::vector<double>> seg_len_, seg_rad_, seg_pos_;
  std::vector<std::vector<uint8_t>> seg_tag_;
  std::vector<std::vector<mcg_species>> species_;
  std::vector<std::vector<mcg_placement>> placements_;
  std::vector<std::vector<std::string>> labels_;
  std::vector<mcg_source> sources_;
  std::vector<std::vector<double>> source_vals_;
  std::vector<uint8_t> c_from_, c_policy_, p_what_;
  std::vector<uint32_t> c_src_, c_dst_, p_gid_, cell_kind_;
  std::vector<int32_t> c_group_, p_comp_, p_species_, p_group_, p_instance_, p_every_;
  std::vector<double> c_w_, c_d_;
  std::vector<int32_t> c_label_;        // per connection: index into miss_text_ (-1: resolved)
  std::vector<std::string> miss_text_;  // unresolved connection labels, for error messages
  std::vector<const char*> miss_ptr_;
  mcg_recipe view_{};
};

// one rank of a sharded engine (one process per GPU): this rank's index, the
// rank count, its device, and the NCCL id made by nccl_unique_id() on one rank
// and shared by the caller (MPI_Bcast, a file, torch.distributed, ...)
struct Shard {
  int rank = 0, world = 1, device = 0;
  std::array<std::uint8_t, 128> nccl_id{};
};

inline std::array<std::uint8_t, 128> nccl_unique_id() {
  std::array<std::uint8_t, 128> id{};
  check(mcg_nccl_unique_id(id.data()));
  return id;
}

class Engine {
 public:
  Engine(const mcsim::Recipe& recipe, const mcsim::EngineOptions& opt, int device = 0)
      : recipe_(recipe) {
    const FlatRecipe flat(recipe);
    const mcg_options o{opt.dt_ms, opt.seed, opt.workers, device, 0, 1};
    check(mcg_create(flat.view(), &o, &eng_));
    dt_ = mcg_dt_ms(eng_);
  }
  // a shard: this rank's cells (contiguous gid range, mcg_partition) with the
  // spike exchange inside the library (ncclAllGather once per min-delay
  // epoch, engine.cpp:913-942); spikes() is the global list, cell(gid) is
  // defined for this rank's gids.  make_checkpoint / restore / fast_forward_to
  // are refused, as mcg_* refuses them for a sharded engine.
  Engine(const mcsim::Recipe& recipe, const mcsim::EngineOptions& opt, const Shard& shard)
      : recipe_(recipe), sharded_(true) {
    const FlatRecipe flat(recipe);
    const mcg_options o{opt.dt_ms, opt.seed, opt.workers, shard.device, shard.rank, shard.world};
    check(mcg_create(flat.view(), &o, &eng_));
    dt_ = mcg_dt_ms(eng_);
    check(mcg_shard_init_nccl(eng_, shard.nccl_id.data()));
  }
  ~Engine() {
    if (eng_) mcg_destroy(eng_);
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  double time_ms() const { return mcg_time_ms(eng_); }
  double dt_ms() const { return dt_; }
  std::int64_t step() const { return mcg_step(eng_); }

  void advance_to(double t_ms) {
    flush_mirrors();
    check(sharded_ ? mcg_shard_advance_to(eng_, t_ms) : mcg_advance_to(eng_, t_ms));
    invalidate();
  }
  void fast_forward_to(double t_ms, double coarse_dt_ms) {
    flush_mirrors();
    check(mcg_fast_forward_to(eng_, t_ms, coarse_dt_ms));
    invalidate();
  }

  const std::vector<mcsim::SpikeRecord>& spikes() const {
    if (!spikes_ok_) {
      const int64_t n = sharded_ ? mcg_shard_num_global_spikes(eng_) : mcg_num_spikes(eng_);
      std::vector<double> t(static_cast<std::size_t>(n));
      std::vector<uint32_t> g(static_cast<std::size_t>(n));
      if (n > 0)
        check(sharded_ ? mcg_shard_get_global_spikes(eng_, 0, n, t.data(), g.data())
                       : mcg_get_spikes(eng_, 0, n, t.data(), g.data()));
      spikes_.resize(static_cast<std::size_t>(n));
      for (int64_t i = 0; i < n; ++i) spikes_[i] = {t[i], g[i]};
      spikes_ok_ = true;
    }
    return spikes_;
  }
  void clear_spikes() {
    check(mcg_clear_spikes(eng_));
    spikes_.clear();
    spikes_ok_ = true;
  }

  int num_cells() const { return mcg_num_cells(eng_); }

  // Engine::make_checkpoint / restore (engine.hpp:139-140): the bytes are
  // MCSCKPT1, so the reference's own Checkpoint type carries them and either
  // engine restores the other's checkpoints
  mcsim::Checkpoint make_checkpoint() {
    flush_mirrors();
    int64_t n = 0;
    check(mcg_checkpoint(eng_, nullptr, 0, &n));
    std::vector<std::uint8_t> b(static_cast<std::size_t>(n));
    check(mcg_checkpoint(eng_, b.data(), n, &n));
    return mcsim::Checkpoint::deserialize(b);
  }
  void restore(const mcsim::Checkpoint& c) {
    const std::vector<std::uint8_t> b = c.serialize();
    // mirrors taken before the restore describe the state being replaced:
    // drop them unwritten, or the next flush would overwrite the restored state
    cells_.clear();
    check(mcg_restore(eng_, b.data(), static_cast<int64_t>(b.size())));
    invalidate();
  }

  // lazily synced host mirror of one cell (written back before the next advance)
  mcsim::CellRT& cell(std::uint32_t gid) {
    auto it = cells_.find(gid);
    if (it == cells_.end()) it = cells_.emplace(gid, read_cell(gid)).first;
    return it->second;
  }

  const std::vector<std::vector<std::pair<double, double>>>& traces() const {
    if (!traces_ok_) {
      traces_.assign(recipe_.probes.size(), {});
      for (std::size_t p = 0; p < traces_.size(); ++p) {
        const int64_t n = mcg_trace_len(eng_, static_cast<int32_t>(p));
        std::vector<double> t(static_cast<std::size_t>(n)), v(static_cast<std::size_t>(n));
        if (n > 0) check(mcg_get_trace(eng_, static_cast<int32_t>(p), t.data(), v.data()));
        for (int64_t i = 0; i < n; ++i) traces_[p].emplace_back(t[i], v[i]);
      }
      traces_ok_ = true;
    }
    return traces_;
  }

  mcg_engine* handle() { return eng_; }
  bool sharded() const { return sharded_; }

 private:
  template <class T>
  std::vector<T> field(int32_t f, uint32_t gid, int32_t index, int64_t count) const {
    std::vector<T> out(static_cast<std::size_t>(count));
    if (count > 0) check(mcg_read_state(eng_, f, gid, index, 0, count, out.data()));
    return out;
  }
  template <class T>
  void put(int32_t f, uint32_t gid, int32_t index, const std::vector<T>& v) {
    if (!v.empty())
      check(mcg_write_state(eng_, f, gid, index, 0, static_cast<int64_t>(v.size()), v.data()));
  }

  mcsim::CellRT read_cell(uint32_t gid) const {
    mcsim::CellRT c;
    c.gid = gid;
    const int n = mcg_cell_ncomp(eng_, gid);
    const mcsim::CellKindSpec& ks = recipe_.kinds[recipe_.cell_kind[gid]];
    c.v_mV = field<double>(MCG_FIELD_V, gid, 0, n);
    for (std::size_t s = 0; s < ks.species.size(); ++s)
      c.species.push_back(field<double>(MCG_FIELD_SPECIES, gid, static_cast<int32_t>(s), n));
    if (std::holds_alternative<mcsim::HhMembrane>(ks.membrane)) {
      c.hh_m = field<double>(MCG_FIELD_HH_M, gid, 0, n);
      c.hh_h = field<double>(MCG_FIELD_HH_H, gid, 0, n);
      c.hh_n = field<double>(MCG_FIELD_HH_N, gid, 0, n);
    }
    c.detector_prev_v = field<double>(MCG_FIELD_DETECTOR_PREV_V, gid, 0, 1)[0];
    c.refractory_until = field<int64_t>(MCG_FIELD_REFRACTORY_UNTIL, gid, 0, 1)[0];
    c.detector_armed = field<int64_t>(MCG_FIELD_DETECTOR_ARMED, gid, 0, 1)[0] != 0;
    c.internal_seq = static_cast<uint32_t>(field<int64_t>(MCG_FIELD_INTERNAL_SEQ, gid, 0, 1)[0]);
    const int ng = mcg_cell_ngroups(eng_, gid);
    for (int g = 0; g < ng; ++g) {
      mcsim::SynGroupRT G;
      G.label = ks.placements[g].label;
      G.spec = ks.placements[g].syn;
      const int64_t sz = mcg_group_size(eng_, gid, g);
      const auto comp = field<int32_t>(MCG_FIELD_SYN_COMP, gid, g, sz);
      G.comp.assign(comp.begin(), comp.end());
      G.weight = field<double>(MCG_FIELD_SYN_WEIGHT, gid, g, sz);
      G.kernel = field<double>(MCG_FIELD_SYN_KERNEL, gid, g, sz);
      const auto a_pre = field<double>(MCG_FIELD_STDP_A_PRE, gid, g, sz);
      const auto a_post = field<double>(MCG_FIELD_STDP_A_POST, gid, g, sz);
      const auto w = field<double>(MCG_FIELD_STDP_W, gid, g, sz);
      G.stdp_last_step = field<int64_t>(MCG_FIELD_STDP_LAST, gid, g, sz);
      const auto hw = field<double>(MCG_FIELD_HOMEO_W, gid, g, sz);
      const auto h = field<double>(MCG_FIELD_STC_H, gid, g, sz);
      const auto z = field<double>(MCG_FIELD_STC_Z, gid, g, sz);
      const auto cc = field<double>(MCG_FIELD_STC_C, gid, g, sz);
      G.sps_abs = field<double>(MCG_FIELD_STC_SPS_ABS, gid, g, sz);
      for (int64_t i = 0; i < sz; ++i) {
        G.stdp.push_back({a_pre[i], a_post[i], w[i]});
        G.homeo.push_back({hw[i]});
        G.stc.push_back({h[i], z[i], cc[i]});
      }
      c.groups.push_back(std::move(G));
    }
    return c;
  }

  void write_cell(uint32_t gid, const mcsim::CellRT& c) {
    put(MCG_FIELD_V, gid, 0, c.v_mV);
    for (std::size_t s = 0; s < c.species.size(); ++s)
      put(MCG_FIELD_SPECIES, gid, static_cast<int32_t>(s), c.species[s]);
    put(MCG_FIELD_HH_M, gid, 0, c.hh_m);
    put(MCG_FIELD_HH_H, gid, 0, c.hh_h);
    put(MCG_FIELD_HH_N, gid, 0, c.hh_n);
    put(MCG_FIELD_DETECTOR_PREV_V, gid, 0, std::vector<double>{c.detector_prev_v});
    put(MCG_FIELD_REFRACTORY_UNTIL, gid, 0, std::vector<int64_t>{c.refractory_until});
    put(MCG_FIELD_DETECTOR_ARMED, gid, 0, std::vector<int64_t>{c.detector_armed ? 1 : 0});
    for (std::size_t g = 0; g < c.groups.size(); ++g) {
      const mcsim::SynGroupRT& G = c.groups[g];
      const int32_t gi = static_cast<int32_t>(g);
      std::vector<double> a_pre, a_post, w, hw, h, z, cc;
      for (const auto& s : G.stdp) {
        a_pre.push_back(s.a_pre);
        a_post.push_back(s.a_post);
        w.push_back(s.w);
      }
      for (const auto& s : G.homeo) hw.push_back(s.w);
      for (const auto& s : G.stc) {
        h.push_back(s.h);
        z.push_back(s.z);
        cc.push_back(s.c);
      }
      put(MCG_FIELD_SYN_WEIGHT, gid, gi, G.weight);
      put(MCG_FIELD_SYN_KERNEL, gid, gi, G.kernel);
      put(MCG_FIELD_STDP_A_PRE, gid, gi, a_pre);
      put(MCG_FIELD_STDP_A_POST, gid, gi, a_post);
      put(MCG_FIELD_STDP_W, gid, gi, w);
      put(MCG_FIELD_STDP_LAST, gid, gi, G.stdp_last_step);
      put(MCG_FIELD_HOMEO_W, gid, gi, hw);
      put(MCG_FIELD_STC_H, gid, gi, h);
      put(MCG_FIELD_STC_Z, gid, gi, z);
      put(MCG_FIELD_STC_C, gid, gi, cc);
      put(MCG_FIELD_STC_SPS_ABS, gid, gi, G.sps_abs);
    }
  }

  void flush_mirrors() {
    for (auto& [gid, c] : cells_) write_cell(gid, c);
    cells_.clear();
  }
  void invalidate() {
    spikes_ok_ = traces_ok_ = false;
  }

  mcsim::Recipe recipe_;
  mcg_engine* eng_ = nullptr;
  bool sharded_ = false;
  double dt_ = 0.0;
  std::map<uint32_t, mcsim::CellRT> cells_;
  mutable std::vector<mcsim::SpikeRecord> spikes_;
  mutable bool spikes_ok_ = false;
  mutable std::vector<std::vector<std::pair<double, double>>> traces_;
  mutable bool traces_ok_ = false;
};

}  // namespace mcsim_gpu
