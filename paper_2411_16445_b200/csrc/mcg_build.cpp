// mcg_build.cpp — recipe -> device layout (see mcg_build.h).
//
// Compiled as plain host C++ with -ffp-contract=off and no -march, exactly
// like the reference (proj/CMakeLists.txt:4-10), and calling glibc exp where
// the reference does, so build-time constants match bit for bit.
#include "mcg_build.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <map>
#include <numbers>
#include <exception>
#include <thread>

#include "mcg_rng.h"

namespace mcg {

namespace {

constexpr double kPi = std::numbers::pi;

[[noreturn]] void engine_error(const std::string& m) { throw Error(MCG_ERR_ENGINE, m); }
[[noreturn]] void morph_error(const std::string& m) { throw Error(MCG_ERR_MORPHOLOGY, m); }

// HH rate functions (engine.cpp:41-54), host glibc exp
double hh_alpha_m(double v) {
  const double x = v + 40.0;
  if (std::fabs(x) < 1e-7) return 1.0;
  return 0.1 * x / (1.0 - std::exp(-x / 10.0));
}
double hh_beta_m(double v) { return 4.0 * std::exp(-(v + 65.0) / 18.0); }
double hh_alpha_h(double v) { return 0.07 * std::exp(-(v + 65.0) / 20.0); }
double hh_beta_h(double v) { return 1.0 / (1.0 + std::exp(-(v + 35.0) / 10.0)); }
double hh_alpha_n(double v) {
  const double x = v + 55.0;
  if (std::fabs(x) < 1e-7) return 0.1;
  return 0.01 * x / (1.0 - std::exp(-x / 10.0));
}
double hh_beta_n(double v) { return 0.125 * std::exp(-(v + 65.0) / 80.0); }

// select_target (engine.cpp:58-74)
int select_target(int group_size, int policy, int& cursor) {
  if (group_size <= 0) throw Error(MCG_ERR_TARGETING, "select_target: empty group");
  switch (policy) {
    case MCG_POLICY_UNIVALENT:
      if (group_size != 1)
        throw Error(MCG_ERR_TARGETING, "select_target: univalent needs a single item");
      return 0;
    case MCG_POLICY_ROUND_ROBIN: {
      const int i = cursor % group_size;
      cursor = (i + 1) % group_size;
      return i;
    }
    case MCG_POLICY_ROUND_ROBIN_HALT:
      return cursor % group_size;
  }
  throw Error(MCG_ERR_TARGETING, "select_target: unknown policy");
}

struct KindRT {  // build_kind outputs not stored in McgKind
  std::vector<double> cap_nF, g_leak, g_leak_rhs, axial, g_na, g_k, cf;
  std::vector<std::vector<double>> sp_coupling;
  std::vector<int64_t> ca_delay;  // per placement
  double c_tot = 0;
};

// TreeSolver::axial_conductance_uS (tree_solver.cpp:19-30)
std::vector<double> axial_conductance(const Grid& g, double r_l) {
  std::vector<double> a(g.size(), 0.0);
  for (int i = 1; i < g.size(); ++i) {
    const int p = g.parent[i];
    const double r = r_l * (0.5 * g.length[i] / g.xs[i] + 0.5 * g.length[p] / g.xs[p]);
    a[i] = 1.0 / r;
  }
  return a;
}

// TreeSolver::diffusive_coupling (tree_solver.cpp:32-44)
std::vector<double> diffusive_coupling(const Grid& g, double diffusivity_si) {
  std::vector<double> b(g.size(), 0.0);
  if (diffusivity_si <= 0) return b;
  const double d = diffusivity_si * 1e9;  // units::diff_um2_per_ms
  for (int i = 1; i < g.size(); ++i) {
    const int p = g.parent[i];
    const double r = 0.5 * g.length[i] / (d * g.xs[i]) + 0.5 * g.length[p] / (d * g.xs[p]);
    b[i] = 1.0 / r;
  }
  return b;
}

}  // namespace

bool eliminate_constant(int n, const int32_t* parent, const double* cap, const double* gs,
                        const double* coupling, double* f, double* d) {
  for (int i = 0; i < n; ++i) {
    d[i] = cap[i] + gs[i];
    f[i] = 0.0;
  }
  for (int i = 1; i < n; ++i) {
    d[i] += coupling[i];
    d[parent[i]] += coupling[i];
  }
  for (int i = n - 1; i >= 1; --i) {
    if (d[i] <= 0.0) return false;
    f[i] = coupling[i] / d[i];
    d[parent[i]] -= f[i] * coupling[i];
  }
  return d[0] > 0.0;
}

int chain_schedule(int n, const int32_t* parent, std::vector<int32_t>& idx, int& a_first) {
  if (n < 2) return 0;
  std::vector<int32_t> child(n, -1), nchild(n, 0);
  std::vector<int32_t> tops;
  for (int i = 1; i < n; ++i) {
    const int p = parent[i];
    if (p < 0 || p >= i) return 0;
    ++nchild[p];
    child[p] = i;
    if (p == 0) tops.push_back(i);
  }
  for (int i = 1; i < n; ++i)
    if (nchild[i] > 1) return 0;
  if (tops.empty() || tops.size() > 2) return 0;
  // chains top -> leaf
  std::vector<std::vector<int32_t>> ch;
  for (int t : tops) {
    std::vector<int32_t> c;
    for (int i = t; i >= 0; i = child[i]) c.push_back(i);
    ch.push_back(c);
  }
  if (ch.size() == 1) ch.emplace_back();
  int ia = 0;
  if (ch[1].size() > ch[0].size()) ia = 1;
  const std::vector<int32_t>& A = ch[ia];
  const std::vector<int32_t>& B = ch[1 - ia];
  a_first = (B.empty() || A.front() > B.front()) ? 1 : 0;
  const int lp = static_cast<int>((A.size() + 3) / 4 * 4);
  idx.assign(2 * lp + 1, -1);
  // leaf side padded: position lp-1 is the top, lp-1-k the k-th node below it
  for (size_t k = 0; k < A.size(); ++k) idx[lp - 1 - k] = A[k];
  for (size_t k = 0; k < B.size(); ++k) idx[2 * lp - 1 - k] = B[k];
  idx[2 * lp] = 0;
  return lp;
}

// host threads for the connection passes of build_model (MCG_BUILD_THREADS,
// default: the hardware threads, at most 16; one below 1 M connections)
int build_threads(int64_t nconn) {
  if (const char* e = std::getenv("MCG_BUILD_THREADS")) return std::clamp(std::atoi(e), 1, 64);
  if (nconn < (int64_t(1) << 20)) return 1;
  return std::clamp(static_cast<int>(std::thread::hardware_concurrency()), 1, 16);
}

int tree_chains(int n, const int32_t* parent, std::vector<int32_t>& out) {
  out.clear();
  if (n < 2) return 0;
  std::vector<std::vector<int32_t>> kids(n);
  for (int i = 1; i < n; ++i) {
    if (parent[i] < 0 || parent[i] >= i) return 0;
    kids[parent[i]].push_back(i);  // ascending
  }
  struct Chain {
    std::vector<int32_t> nodes;
    int level;
    std::vector<int32_t> child;  // chain ids
  };
  std::vector<Chain> ch;
  std::vector<std::pair<int32_t, int32_t>> todo{{0, -1}};  // (top node, parent chain)
  for (size_t t = 0; t < todo.size(); ++t) {
    const int id = static_cast<int>(ch.size());
    if (id >= 32) return 0;
    Chain c;
    c.level = todo[t].second < 0 ? 0 : ch[todo[t].second].level + 1;
    int x = todo[t].first;
    c.nodes.push_back(x);
    while (kids[x].size() == 1) {
      x = kids[x][0];
      c.nodes.push_back(x);
    }
    if (todo[t].second >= 0) ch[todo[t].second].child.push_back(id);
    ch.push_back(std::move(c));
    for (int k : kids[x]) todo.emplace_back(k, id);
  }
  int maxlev = 0, maxch = 0;
  for (Chain& c : ch) {
    maxlev = std::max(maxlev, c.level);
    maxch = std::max(maxch, static_cast<int>(c.child.size()));
    // descending top index: the order solve_tree's loop applies them
    std::sort(c.child.begin(), c.child.end(),
              [&](int a, int b) { return ch[a].nodes[0] > ch[b].nodes[0]; });
  }
  const int nch = static_cast<int>(ch.size());
  out = {nch, maxlev, maxch};
  int off = 0;
  for (const Chain& c : ch) {
    out.push_back(off);
    out.push_back(static_cast<int32_t>(c.nodes.size()));
    out.push_back(c.level);
    out.push_back(static_cast<int32_t>(c.child.size()));
    for (int q = 0; q < maxch; ++q) out.push_back(q < static_cast<int>(c.child.size()) ? c.child[q] : -1);
    off += static_cast<int>(c.nodes.size());
  }
  for (const Chain& c : ch) out.insert(out.end(), c.nodes.begin(), c.nodes.end());
  return nch;
}

// v = n copies of x, filled by nthr threads (parallel first touch)
template <class T, class Al>
void par_fill(std::vector<T, Al>& v, int64_t n, T x, int nthr) {
  v.clear();
  v.resize(static_cast<size_t>(n));
  if (nthr <= 1 || n < (int64_t(1) << 16)) {
    std::fill(v.begin(), v.end(), x);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nthr; ++t)
    th.emplace_back([&, t] { std::fill(v.begin() + n * t / nthr, v.begin() + n * (t + 1) / nthr, x); });
  for (auto& q : th) q.join();
}

int64_t ceil_steps(double t_ms, double dt_ms) {
  return static_cast<int64_t>(std::ceil(t_ms / dt_ms - 1e-9));  // engine.cpp:21-23
}

// discretize (morphology.cpp:67-143)
Grid discretize(const mcg_kind& k) {
  const int n = k.n_segments;
  if (n == 0) morph_error("discretize: empty segment list");
  if (!(k.target_compartment_um > 0)) morph_error("discretize: target length must be positive");
  int root = -1;
  for (int s = 0; s < n; ++s) {
    if (!(k.seg_length_um[s] > 0) || !(k.seg_radius_um[s] > 0))
      morph_error("discretize: non-positive segment geometry");
    if (k.seg_parent_pos[s] < 0 || k.seg_parent_pos[s] > 1)
      morph_error("discretize: parent_pos outside [0,1]");
    if (k.seg_parent[s] < 0) {
      if (root >= 0) morph_error("discretize: multiple roots");
      root = s;
    } else if (k.seg_parent[s] >= n) {
      morph_error("discretize: parent index out of range");
    }
  }
  if (root < 0) morph_error("discretize: no root segment");
  std::vector<int> order{root};
  std::vector<char> placed(n, 0);
  placed[root] = 1;
  for (std::size_t head = 0; head < order.size(); ++head)
    for (int s = 0; s < n; ++s)
      if (!placed[s] && k.seg_parent[s] >= 0 && k.seg_parent[s] == order[head]) {
        order.push_back(s);
        placed[s] = 1;
      }
  if (static_cast<int>(order.size()) != n) morph_error("discretize: cyclic parent references");

  struct Range { int first = 0, count = 0; };
  std::vector<Range> ranges(n);
  Grid g;
  for (int idx : order) {
    const double len = k.seg_length_um[idx], rad = k.seg_radius_um[idx];
    const int count = std::max(1, static_cast<int>(std::ceil(len / k.target_compartment_um - 1e-12)));
    const double dl = len / count;
    const double area_xs = kPi * rad * rad;
    ranges[idx] = {g.size(), count};
    for (int kk = 0; kk < count; ++kk) {
      int parent_comp;
      if (kk > 0) {
        parent_comp = ranges[idx].first + kk - 1;
      } else if (k.seg_parent[idx] < 0) {
        parent_comp = -1;
      } else {
        const Range& pr = ranges[k.seg_parent[idx]];
        const double kf = k.seg_parent_pos[idx] * pr.count - 0.5;
        int q = static_cast<int>(std::ceil(kf - 0.5));
        q = std::clamp(q, 0, pr.count - 1);
        parent_comp = pr.first + q;
      }
      g.length.push_back(dl);
      g.area.push_back(2 * kPi * rad * dl);
      g.xs.push_back(area_xs);
      g.volume.push_back(area_xs * dl);
      g.parent.push_back(parent_comp);
      g.tag.push_back(k.seg_tag[idx]);
      g.segment_of.push_back(static_cast<uint32_t>(idx));
    }
  }
  for (double vv : g.volume) g.total_volume += vv;
  return g;
}

void partition(const mcg_recipe& r, int world, std::vector<uint32_t>& bounds) {
  const int n = r.n_cells;
  bounds.assign(world + 1, 0);
  bounds[world] = static_cast<uint32_t>(n);
  if (world <= 1 || n == 0) return;
  // cost per cell: compartments + synapse instances (placements + connections)
  std::vector<int64_t> kcost(r.n_kinds, 0);
  for (int k = 0; k < r.n_kinds; ++k) {
    int64_t comps = 0;
    try { comps = discretize(r.kinds[k]).size(); } catch (...) { comps = 1; }
    int64_t pre = 0;
    for (int p = 0; p < r.kinds[k].n_placements; ++p) pre += r.kinds[k].placements[p].count;
    kcost[k] = comps + pre;
  }
  std::vector<int64_t> cost(n);
  for (int c = 0; c < n; ++c)
    cost[c] = (r.cell_kind[c] < static_cast<uint32_t>(r.n_kinds)) ? kcost[r.cell_kind[c]] : 1;
  for (int64_t i = 0; i < r.n_connections; ++i)
    if (r.conn_dst[i] < static_cast<uint32_t>(n)) cost[r.conn_dst[i]] += 1;
  int64_t total = 0;
  for (int64_t c : cost) total += c;
  int64_t acc = 0;
  int w = 1;
  for (int c = 0; c < n && w < world; ++c) {
    acc += cost[c];
    while (w < world && acc * world >= total * w) bounds[w++] = static_cast<uint32_t>(c + 1);
  }
  while (w < world) bounds[w++] = static_cast<uint32_t>(n);
}

namespace {
// MCG_PROFILE_BUILD=1: host build stage times on stderr
struct StageTimer {
  bool on = std::getenv("MCG_PROFILE_BUILD") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "build %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};
}  // namespace

void build_model(const mcg_recipe& r, const mcg_options& opt, HostModel& m, int threads, bool defer_edges) {
  StageTimer tm;
  const double dt = opt.dt_ms;
  m.dt = dt;
  m.seed = opt.seed;
  m.rank = opt.rank;
  m.world = opt.world < 1 ? 1 : opt.world;
  m.n_cells_global = r.n_cells;
  std::vector<uint32_t> bounds;
  partition(r, m.world, bounds);
  m.gid_begin = bounds[m.rank];
  m.gid_end = bounds[m.rank + 1];
  m.max_shard_cells = 0;  // every rank's cell count is known from the partition
  for (int q = 0; q < m.world; ++q)
    m.max_shard_cells = std::max<int32_t>(m.max_shard_cells, static_cast<int32_t>(bounds[q + 1] - bounds[q]));

  // ---- kinds (build_kind, engine.cpp:189-278) ----
  const int nk = r.n_kinds;
  std::vector<KindRT> krt(nk);
  m.kinds.resize(nk);
  m.grids.resize(nk);
  m.k_sp_off.resize(nk + 1, 0);
  for (int ki = 0; ki < nk; ++ki) {
    const mcg_kind& spec = r.kinds[ki];
    McgKind& K = m.kinds[ki];
    K = McgKind{};
    KindRT& k = krt[ki];
    Grid& g = m.grids[ki];
    g = discretize(spec);
    const int n = g.size();
    K.n = n;
    k.cap_nF.assign(n, 0.0);
    k.g_leak.assign(n, 0.0);
    k.g_leak_rhs.assign(n, 0.0);
    k.g_na.assign(n, 0.0);
    k.g_k.assign(n, 0.0);
    k.axial.assign(n, 0.0);
    k.cf.assign(n, 0.0);
    if (spec.membrane == MCG_MEMBRANE_LIF) {
      const mcg_lif& L = spec.lif;
      K.dyn = L.exact ? MCG_DYN_LIF_EXACT : MCG_DYN_LIF;
      if (L.exact && n != 1) engine_error("exact LIF requires a single compartment");
      double area_tot = 0;
      for (int i = 0; i < n; ++i) area_tot += g.area[i];
      k.c_tot = L.tau_mem_ms / L.r_mem_MOhm;
      for (int i = 0; i < n; ++i) {
        const double share = g.area[i] / area_tot;
        k.cap_nF[i] = k.c_tot * share;
        k.g_leak[i] = share / L.r_mem_MOhm;
        k.g_leak_rhs[i] = k.g_leak[i] * L.v_rev_mV;
      }
      k.axial = axial_conductance(g, L.r_axial_ohm_m);
      K.ref_steps = ceil_steps(L.t_ref_ms, dt);
      K.detector_comp = L.detector_comp;
      K.noise_comp = L.noise_comp;
      K.threshold = L.v_thresh_mV;
      K.has_detector = 1;
      K.has_bg = (L.i_bg_nA != 0.0 || L.sigma_bg_nA_sqrt_ms != 0.0) ? 1 : 0;
      K.v_rev = L.v_rev_mV;
      K.r_mem = L.r_mem_MOhm;
      K.v_reset = L.v_reset_mV;
      K.i_bg = L.i_bg_nA;
      K.sig_bg = L.sigma_bg_nA_sqrt_ms / std::sqrt(dt);
      K.bg_t0 = L.bg_quiet_t0_ms;
      K.bg_t1 = L.bg_quiet_t1_ms;
      K.lif_exact_f = std::exp(-dt / L.tau_mem_ms);
    } else if (spec.membrane == MCG_MEMBRANE_HH) {
      const mcg_hh& H = spec.hh;
      K.dyn = MCG_DYN_HH;
      for (int i = 0; i < n; ++i) {
        const double a = g.area[i];
        k.cap_nF[i] = H.c_m * a * 1e-3;
        k.c_tot += k.cap_nF[i];
        k.g_leak[i] = H.g_leak * a * 1e-6;
        k.g_leak_rhs[i] = k.g_leak[i] * H.e_leak_mV;
        if (g.tag[i] == MCG_REGION_SOMA) {
          k.g_na[i] = H.g_na * a * 1e-6;
          k.g_k[i] = H.g_k * a * 1e-6;
        }
      }
      k.axial = axial_conductance(g, H.r_axial_ohm_m);
      K.detector_comp = H.detector_comp;
      K.threshold = H.threshold_mV;
      K.has_detector = 1;
      K.e_na = H.e_na_mV;
      K.e_k = H.e_k_mV;
    } else {
      K.dyn = MCG_DYN_NONE;
    }
    if (K.dyn != MCG_DYN_NONE)
      for (int i = 0; i < n; ++i) k.cf[i] = k.c_tot / k.cap_nF[i];

    K.n_species = spec.n_species;
    K.sps_idx = spec.sps_idx;
    K.prp_idx = spec.prp_idx;
    for (int s = 0; s < spec.n_species; ++s)
      k.sp_coupling.push_back(diffusive_coupling(g, spec.species[s].diffusivity));

    K.n_groups = spec.n_placements;
    K.spec0 = static_cast<int32_t>(m.specs.size());
    for (int p = 0; p < spec.n_placements; ++p) {
      const mcg_placement& pl = spec.placements[p];
      const mcg_syn_spec& sy = pl.syn;
      McgSpec S{};
      S.kind = sy.kind;
      S.comp = pl.comp;
      S.count = pl.count;
      S.f_decay = std::exp(-dt / sy.tau_syn_ms);
      S.e_rev = sy.e_rev_mV;
      S.tau_pre = sy.stdp.tau_pre_ms;
      S.tau_post = sy.stdp.tau_post_ms;
      S.a_pre = sy.stdp.a_pre_uS;
      S.a_post = sy.stdp.a_post_uS;
      S.wmax = sy.stdp.wmax_uS;
      S.dw_plus = sy.homeo.dw_plus_nA;
      S.dw_minus = sy.homeo.dw_minus_nA;
      S.h_wmax = sy.homeo.wmax_nA;
      const mcg_stc_params& P = sy.stc;
      S.h0 = P.h0_mV;
      S.tau_h = P.tau_h_ms;
      S.theta_p = P.theta_p;
      S.theta_d = P.theta_d;
      S.gamma_p = P.gamma_p;
      S.gamma_d = P.gamma_d;
      S.sigma = P.sigma_pl_mV;
      S.f_int = P.f_int;
      S.tau_z = P.tau_z_ms;
      S.r_tau_h = mcg_recip(S.tau_h);
      S.r_tau_z = mcg_recip(S.tau_z);
      S.theta_tag = P.theta_tag_mV;
      S.cf = std::exp(-dt / P.tau_c_ms);
      S.nz1 = P.sigma_pl_mV * std::sqrt(double(1) / P.tau_h_ms) * std::sqrt(dt);
      S.nz2 = P.sigma_pl_mV * std::sqrt(double(2) / P.tau_h_ms) * std::sqrt(dt);
      S.cpre_s = P.c_pre * sy.calcium_scale;
      S.cpost_s = P.c_post * sy.calcium_scale;
      int64_t d = 0;
      if (sy.kind == MCG_SYN_STC_CHARGE) {
        d = ceil_steps(P.t_c_delay_ms, dt);
        if (spec.prp_enabled) {  // make_prp_synthesis (mechanisms.hpp:258-262)
          K.prp_theta_star = P.theta_pro_mV / g.total_volume;
          K.prp_rate = g.total_volume * P.p_max / P.tau_p_ms;
        }
        ++K.n_stc_groups;
      }
      if (K.dyn == MCG_DYN_LIF_EXACT &&
          (sy.kind == MCG_SYN_STATIC_COND || sy.kind == MCG_SYN_STDP_COND))
        engine_error("exact LIF supports only current/charge synapses");
      S.ca_delay = d;
      k.ca_delay.push_back(d);
      m.specs.push_back(S);
    }
    if (spec.prp_enabled) {
      K.prp_enabled = 1;
      K.prp_comp = spec.prp_comp;
      if (spec.sps_idx < 0 || spec.prp_idx < 0)
        engine_error("synthesis unit needs SPS and PRP species");
    }

    // flattened per-kind arrays (+ per-step constants hoisted)
    K.arr = static_cast<int64_t>(m.k_parent.size());
    for (int i = 0; i < n; ++i) {
      m.k_parent.push_back(g.parent[i]);
      m.k_cap_dt.push_back(k.cap_nF[i] / dt);
      m.k_g_leak.push_back(k.g_leak[i]);
      m.k_g_leak_rhs.push_back(k.g_leak_rhs[i]);
      m.k_axial.push_back(k.axial[i]);
      m.k_g_na.push_back(k.g_na[i]);
      m.k_g_k.push_back(k.g_k[i]);
      m.k_cf.push_back(k.cf[i]);
      m.k_volume.push_back(g.volume[i]);
      m.k_rvol.push_back(mcg_recip(g.volume[i]));
    }
    // LIF-cable V system without active conductances: cap/dt, g_leak + 0.0
    // (engine.cpp:680-686 with has_gsyn == false)
    {
      std::vector<double> capv(n), gsv(n), fv(n, 0.0), dv(n, 0.0);
      for (int i = 0; i < n; ++i) {
        capv[i] = k.cap_nF[i] / dt;
        gsv[i] = k.g_leak[i] + 0.0;
      }
      K.v_const = (K.dyn == MCG_DYN_LIF &&
                   eliminate_constant(n, g.parent.data(), capv.data(), gsv.data(),
                                      k.axial.data(), fv.data(), dv.data()))
                      ? 1 : 0;
      for (int i = 0; i < n; ++i) {
        m.k_vf.push_back(fv[i]);
        m.k_vd.push_back(dv[i]);
        m.k_vr.push_back(mcg_recip(dv[i]));
      }
    }
    K.sp_arr = static_cast<int64_t>(m.k_sp_cap_dt.size());
    m.k_sp_off[ki] = static_cast<int64_t>(m.k_sp_decay_tau.size());
    K.sp_const = 1;
    for (int s = 0; s < spec.n_species; ++s) {
      const double tau = spec.species[s].decay_tau_ms;
      m.k_sp_decay_tau.push_back(tau);
      std::vector<double> cs(n), gss(n), fs(n, 0.0), ds(n, 0.0);
      for (int i = 0; i < n; ++i) {
        cs[i] = g.volume[i] / dt;
        gss[i] = tau > 0 ? g.volume[i] / tau : 0.0;
        m.k_sp_cap_dt.push_back(cs[i]);
        m.k_sp_gs.push_back(gss[i]);
        m.k_sp_coupling.push_back(k.sp_coupling[s][i]);
        m.k_sp_init.push_back(spec.species[s].init);
      }
      if (n > 1 && !eliminate_constant(n, g.parent.data(), cs.data(), gss.data(),
                                       k.sp_coupling[s].data(), fs.data(), ds.data()))
        K.sp_const = 0;
      for (int i = 0; i < n; ++i) {
        m.k_sp_f.push_back(fs[i]);
        m.k_sp_d.push_back(ds[i]);
        m.k_sp_r.push_back(mcg_recip(ds[i]));
      }
    }
    m.k_sp_off[ki + 1] = static_cast<int64_t>(m.k_sp_decay_tau.size());
    // chain schedule of the constant systems: every eliminated diagonal of
    // the systems that use it must have a usable reciprocal (mcg_recip != 0)
    {
      std::vector<int32_t> idx;
      int a_first = 1;
      int lp = (K.v_const || K.sp_const) ? chain_schedule(n, g.parent.data(), idx, a_first) : 0;
      for (int i = 0; lp > 0 && i < n; ++i) {
        if (K.v_const && m.k_vr[K.arr + i] == 0.0) lp = 0;
        for (int sp = 0; K.sp_const && sp < spec.n_species; ++sp)
          if (m.k_sp_r[K.sp_arr + int64_t(sp) * n + i] == 0.0) lp = 0;
      }
      K.ch_lp = lp;
      K.ch_afirst = a_first;
      K.ch_arr = static_cast<int64_t>(m.k_ch_idx.size());
      if (lp > 0) m.k_ch_idx.insert(m.k_ch_idx.end(), idx.begin(), idx.end());
    }
    // chains of the general V solve (HH, LIF cable with conductances)
    K.gch_n = 0;
    K.gch_pad = 0;
    K.gch_arr = 0;
    if (n >= 2 && (K.dyn == MCG_DYN_HH || K.dyn == MCG_DYN_LIF) && !std::getenv("MCG_NO_TREE_WARP")) {
      std::vector<int32_t> sched;
      const int nch = tree_chains(n, g.parent.data(), sched);
      if (nch > 0) {
        K.gch_n = nch;
        K.gch_arr = static_cast<int64_t>(m.k_ch_idx.size());
        m.k_ch_idx.insert(m.k_ch_idx.end(), sched.begin(), sched.end());
      }
    }
  }

  tm.mark("kinds");
  // ---- local cells (engine.cpp:317-348) ----
  const uint32_t g0 = m.gid_begin, g1 = m.gid_end;
  for (uint32_t gid = 0; gid < static_cast<uint32_t>(r.n_cells); ++gid)
    if (r.cell_kind[gid] >= static_cast<uint32_t>(nk)) engine_error("cell kind out of range");
  const int nl = static_cast<int>(g1 - g0);
  m.cell_kind.resize(nl);
  m.comp_off.resize(nl + 1);
  m.sp_off.resize(nl + 1);
  m.cg_off.resize(nl + 1);
  m.det_prev.resize(nl);
  m.armed.assign(nl, 1);
  m.refr_until.assign(nl, 0);
  m.internal_seq.assign(nl, 0);
  int64_t comps = 0, sps = 0, cgs = 0;
  for (int c = 0; c < nl; ++c) {
    const int kid = static_cast<int>(r.cell_kind[g0 + c]);
    m.cell_kind[c] = kid;
    const McgKind& K = m.kinds[kid];
    m.comp_off[c] = comps;
    m.sp_off[c] = sps;
    m.cg_off[c] = cgs;
    comps += K.n;
    sps += static_cast<int64_t>(K.n) * K.n_species;
    cgs += K.n_groups;
  }
  m.comp_off[nl] = comps;
  m.sp_off[nl] = sps;
  m.cg_off[nl] = cgs;
  m.v.assign(comps, 0.0);
  m.hh_m.assign(comps, 0.0);
  m.hh_h.assign(comps, 0.0);
  m.hh_n.assign(comps, 0.0);
  m.species.assign(sps, 0.0);
  for (int c = 0; c < nl; ++c) {
    const McgKind& K = m.kinds[m.cell_kind[c]];
    const mcg_kind& spec = r.kinds[m.cell_kind[c]];
    const int64_t o = m.comp_off[c];
    if (K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT) {
      for (int i = 0; i < K.n; ++i) m.v[o + i] = spec.lif.v_rev_mV;
      m.det_prev[c] = spec.lif.v_rev_mV;
    } else if (K.dyn == MCG_DYN_HH) {
      const double v = spec.hh.v_init_mV;
      const double mm = hh_alpha_m(v) / (hh_alpha_m(v) + hh_beta_m(v));
      const double hh = hh_alpha_h(v) / (hh_alpha_h(v) + hh_beta_h(v));
      const double nn = hh_alpha_n(v) / (hh_alpha_n(v) + hh_beta_n(v));
      for (int i = 0; i < K.n; ++i) {
        m.v[o + i] = v;
        m.hh_m[o + i] = mm;
        m.hh_h[o + i] = hh;
        m.hh_n[o + i] = nn;
      }
      m.det_prev[c] = v;
    } else {
      m.det_prev[c] = 0.0;
    }
    for (int s = 0; s < K.n_species; ++s)
      for (int i = 0; i < K.n; ++i)
        m.species[m.sp_off[c] + static_cast<int64_t>(s) * K.n + i] = spec.species[s].init;
  }

  tm.mark("cells");
  // ---- connections (Impl::build, engine.cpp:357-391) in two passes over the
  // connection list, both in the reference's order:
  //   pass 0  the reference's checks in its order (dst, label, targeting,
  //           source/src range, delay vs dt), min_delay_steps, and counts:
  //           appended instances per (cell, group), edges per rank bucket
  //           (src_key, sources last: EventOrder, engine.cpp:25-31), source
  //           edges per source;
  //   pass 1  instance selection (append or select_target's cursors) and each
  //           local edge written straight into its slot of the rank order
  //           (a stable counting sort by src_key: connections arrive in seq
  //           order), with the static-charge payload (comp, w * cf[comp]).
  const int64_t nconn = r.n_connections;
  const size_t nk1 = static_cast<size_t>(r.n_cells) + 1;  // rank buckets; the last: sources
  std::vector<int64_t> app(cgs, 0);            // appended instances per (cell, group)
  std::vector<int64_t> cg_conns(cgs, 0);       // local connections per (cell, group)
  std::vector<int64_t> bucket(nk1 + 1, 0);     // local edges per rank bucket
  std::vector<int64_t> src_cnt(std::max(r.n_sources, 0) + 1, 0);
  {
    // contiguous chunks of the connection list on host threads, each with its
    // own counts; an error is rethrown from the first failing connection, so
    // the message is the one the reference's sequential loop raises
    struct Part {
      std::vector<int64_t> app, cg_conns, bucket, src_cnt;
      int64_t min_delay = -1;
      int64_t err_ci = -1;
      std::exception_ptr err;
    };
    const int nthr0 = threads > 0 ? threads : build_threads(nconn);
    std::vector<Part> parts(nthr0);
    auto scan = [&](int t) {
      Part& P = parts[t];
      const bool own = t > 0;  // thread 0 counts into the totals directly
      if (own) {
        P.app.assign(cgs, 0);
        P.cg_conns.assign(cgs, 0);
        P.bucket.assign(nk1 + 1, 0);
        P.src_cnt.assign(src_cnt.size(), 0);
      }
      int64_t* ap = own ? P.app.data() : app.data();
      int64_t* cc = own ? P.cg_conns.data() : cg_conns.data();
      int64_t* bk = own ? P.bucket.data() : bucket.data();
      int64_t* sc = own ? P.src_cnt.data() : src_cnt.data();
      const int64_t c0 = nconn * t / nthr0, c1 = nconn * (t + 1) / nthr0;
      int scratch = 0;
      int64_t ci = c0;
      try {
        for (; ci < c1; ++ci) {
          const uint32_t dst = r.conn_dst[ci];
          if (dst >= static_cast<uint32_t>(r.n_cells)) engine_error("connection dst out of range");
          const int32_t gi = r.conn_group[ci];
          const mcg_kind& dspec = r.kinds[r.cell_kind[dst]];
          if (gi < 0 || gi >= dspec.n_placements) {
            const int32_t li = (r.labels && r.conn_label) ? r.conn_label[ci] : -1;
            engine_error("connection label '" +
                         ((li >= 0 && li < r.n_labels && r.labels[li]) ? std::string(r.labels[li])
                                                                        : "#" + std::to_string(gi)) +
                         "' not found");
          }
          const bool local = dst >= g0 && dst < g1;
          const mcg_placement& pl = dspec.placements[gi];
          if (local) {
            const int64_t cg = m.cg_off[dst - g0] + gi;
            if (pl.count == 0) ++ap[cg];
            else (void)select_target(pl.count, r.conn_policy[ci], scratch);  // its errors, in order
            ++cc[cg];
          }
          if (r.conn_from_source[ci]) {
            if (r.conn_src[ci] >= static_cast<uint32_t>(r.n_sources))
              engine_error("connection source out of range");
            if (local) {
              ++bk[nk1];
              ++sc[r.conn_src[ci] + 1];
            }
          } else {
            if (r.conn_src[ci] >= static_cast<uint32_t>(r.n_cells))
              engine_error("connection src out of range");
            if (r.conn_delay_ms[ci] < dt * (1.0 - 1e-12))
              engine_error("configuration: dt exceeds a connection delay");
            const int64_t d = ceil_steps(r.conn_delay_ms[ci], dt);
            if (P.min_delay < 0 || d < P.min_delay) P.min_delay = d;
            if (local) ++bk[r.conn_src[ci] + 1];
          }
        }
      } catch (...) {
        P.err_ci = ci;
        P.err = std::current_exception();
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nthr0; ++t) th.emplace_back(scan, t);
    scan(0);
    for (auto& x : th) x.join();
    for (int t = 0; t < nthr0; ++t)  // chunks are in order: the first error is the reference's
      if (parts[t].err) std::rethrow_exception(parts[t].err);
    for (int t = 0; t < nthr0; ++t) {
      const Part& P = parts[t];
      if (P.min_delay >= 0 && (m.min_delay_steps < 0 || P.min_delay < m.min_delay_steps))
        m.min_delay_steps = P.min_delay;
      if (t == 0) continue;
      for (int64_t q = 0; q < cgs; ++q) {
        app[q] += P.app[q];
        cg_conns[q] += P.cg_conns[q];
      }
      for (size_t q = 0; q < bucket.size(); ++q) bucket[q] += P.bucket[q];
      for (size_t q = 0; q < src_cnt.size(); ++q) src_cnt[q] += P.src_cnt[q];
    }
  }
  tm.mark("connections");
  // ---- instance layout: per (cell, group) the pre-placed instances, then the
  // appended ones in connection order
  m.cgs.resize(cgs);
  int64_t ninst = 0;
  for (int c = 0; c < nl; ++c) {
    const McgKind& K = m.kinds[m.cell_kind[c]];
    for (int gi = 0; gi < K.n_groups; ++gi) {
      const int64_t cg = m.cg_off[c] + gi;
      const McgSpec& S = m.specs[K.spec0 + gi];
      McgCellGroup& G = m.cgs[cg];
      G.inst = ninst;
      G.size = static_cast<int32_t>(S.count + app[cg]);
      G.active_n = 0;
      G.spec = K.spec0 + gi;
      G.fifo = -1;
      ninst += G.size;
    }
  }
  const int nthr = build_threads(nconn);
  // instance state: the arrays that start all zero (kernel, STDP traces,
  // z, calcium, |h - h0|, and STDP / homeostatic weights when no group has
  // that kind) stay empty here and are zero-filled on the device
  m.n_inst = ninst;
  bool any_stdp = false, any_homeo = false;
  for (const McgCellGroup& G : m.cgs) {
    any_stdp |= m.specs[G.spec].kind == MCG_SYN_STDP_COND && G.size > 0;
    any_homeo |= m.specs[G.spec].kind == MCG_SYN_HOMEO_CURRENT && G.size > 0;
  }
  m.i_kernel.clear();
  m.i_stdp_pre.clear();
  m.i_stdp_post.clear();
  m.i_stdp_last.clear();
  m.i_stc_z.clear();
  m.i_stc_c.clear();
  m.i_sps_abs.clear();
  par_fill(m.i_comp, ninst, int32_t(0), nthr);
  par_fill(m.i_weight, ninst, 0.0, nthr);
  par_fill(m.i_stc_h, ninst, 0.0, nthr);
  if (any_stdp) par_fill(m.i_stdp_w, ninst, 0.0, nthr);
  else m.i_stdp_w.clear();
  if (any_homeo) par_fill(m.i_homeo_w, ninst, 0.0, nthr);
  else m.i_homeo_w.clear();
  for (int c = 0; c < nl; ++c) {
    const McgKind& K = m.kinds[m.cell_kind[c]];
    for (int gi = 0; gi < K.n_groups; ++gi) {
      const McgCellGroup& G = m.cgs[m.cg_off[c] + gi];
      const McgSpec& S = m.specs[K.spec0 + gi];
      for (int i = 0; i < G.size; ++i) m.i_comp[G.inst + i] = S.comp;  // appended ones: pl.comp too
    }
  }
  // ---- rank order: bucket offsets (cell src keys ascending, sources last)
  for (size_t k = 0; k < nk1; ++k) bucket[k + 1] += bucket[k];
  int64_t ne = bucket[nk1];
  m.n_edges = ne;
  m.edges_deferred = defer_edges && !any_stdp && ne > 0;
  if (m.edges_deferred) {
    // per (cell, group): where its connections start in cg order, and what
    // the device needs to pick instances and form the static-charge payload
    m.cg_conn_off.assign(cgs + 1, 0);
    for (int64_t q = 0; q < cgs; ++q) m.cg_conn_off[q + 1] = m.cg_conn_off[q] + cg_conns[q];
    m.cg_static.assign(cgs, 0);
    m.cg_count.assign(cgs, 0);
    m.cg_comp.assign(cgs, -1);
    m.cg_cf.assign(cgs, 0.0);
    for (int c = 0; c < nl; ++c) {
      const McgKind& K = m.kinds[m.cell_kind[c]];
      for (int gi = 0; gi < K.n_groups; ++gi) {
        const int64_t cg = m.cg_off[c] + gi;
        const McgSpec& S = m.specs[m.cgs[cg].spec];
        m.cg_static[cg] = S.kind == MCG_SYN_STATIC_CHARGE;
        m.cg_count[cg] = S.count;
        m.cg_comp[cg] = S.comp;
        if (S.comp >= 0 && S.comp < K.n) m.cg_cf[cg] = m.k_cf[K.arr + S.comp];
      }
    }
  }
  // every edge slot is written by pass 1 (no fill), but the payload columns
  if (m.edges_deferred) ne = 0;  // the device writes them
  m.e_dst.resize(ne);
  m.e_group.resize(ne);
  m.e_inst.resize(ne);
  m.e_weight.resize(ne);
  m.e_delay.resize(ne);
  m.e_src.resize(ne);
  m.e_seq.resize(ne);
  par_fill(m.e_comp, ne, int32_t(-1), nthr);
  par_fill(m.e_wcf, ne, 0.0, nthr);
  m.out_begin.assign(r.n_cells, 0);
  m.out_end.assign(r.n_cells, 0);
  for (int g = 0; g < r.n_cells; ++g)
    if (bucket[g + 1] > bucket[g]) {
      m.out_begin[g] = bucket[g];
      m.out_end[g] = bucket[g + 1];
    }
  for (int q = 0; q < r.n_sources; ++q) src_cnt[q + 1] += src_cnt[q];
  m.src_edge_off.assign(src_cnt.begin(), src_cnt.begin() + (r.n_sources + 1));
  m.src_edges.resize(src_cnt[std::max(r.n_sources, 0)]);
  // ---- pass 1: instances, then edges; both scan the connections in order,
  // split over host threads by what they write (destination cells for the
  // instances, rank buckets for the edges) so that every thread sees its own
  // connections in the reference's order
  HVec<uint32_t> inst_of(static_cast<size_t>(m.edges_deferred ? 0 : nconn));  // every local one is written
  if (!m.edges_deferred) {
    auto instances = [&](int c_lo, int c_hi) {
      std::vector<int32_t> cursor;  // SelectionCursor per (dst, label), cells [c_lo, c_hi)
      const int64_t cg_lo = m.cg_off[c_lo], cg_hi = m.cg_off[c_hi];
      std::vector<int64_t> run(cg_hi - cg_lo, 0);  // appended so far per (cell, group)
      cursor.assign(cg_hi - cg_lo, 0);
      for (int64_t ci = 0; ci < nconn; ++ci) {
        const uint32_t dst = r.conn_dst[ci];
        if (dst < g0 + uint32_t(c_lo) || dst >= g0 + uint32_t(c_hi)) continue;
        const int64_t cg = m.cg_off[dst - g0] + r.conn_group[ci];
        const McgCellGroup& G = m.cgs[cg];
        const int32_t count = m.specs[G.spec].count;
        uint32_t instance;
        if (count == 0) {
          instance = static_cast<uint32_t>(run[cg - cg_lo]++);
          m.i_weight[G.inst + instance] = r.conn_weight[ci];
        } else {
          instance = static_cast<uint32_t>(select_target(count, r.conn_policy[ci], cursor[cg - cg_lo]));
        }
        inst_of[ci] = instance;
      }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nthr; ++t) {
      const int c_lo = static_cast<int>(int64_t(nl) * t / nthr), c_hi = static_cast<int>(int64_t(nl) * (t + 1) / nthr);
      if (t + 1 < nthr) th.emplace_back(instances, c_lo, c_hi);
      else instances(c_lo, c_hi);
    }
    for (auto& x : th) x.join();
  }
  if (!m.edges_deferred) {
    // bucket ranges balanced by edge count; the source bucket (last) with the
    // source CSR goes to the last thread
    auto edges = [&](size_t k_lo, size_t k_hi) {
      std::vector<int64_t> pos(bucket.begin() + k_lo, bucket.begin() + k_hi);
      std::vector<int64_t> spos;
      if (k_hi == nk1) spos.assign(src_cnt.begin(), src_cnt.begin() + std::max(r.n_sources, 0));
      int64_t maxd = 0;
      for (int64_t ci = 0; ci < nconn; ++ci) {
        const uint32_t dst = r.conn_dst[ci];
        if (dst < g0 || dst >= g1) continue;
        const bool from_src = r.conn_from_source[ci] != 0;
        const size_t key = from_src ? nk1 - 1 : static_cast<size_t>(r.conn_src[ci]);
        if (key < k_lo || key >= k_hi) continue;
        const int32_t gi = r.conn_group[ci];
        const int c = static_cast<int>(dst - g0);
        const McgCellGroup& G = m.cgs[m.cg_off[c] + gi];
        const McgSpec& S = m.specs[G.spec];
        const double w = r.conn_weight[ci];
        const uint32_t instance = inst_of[ci];
        const int64_t e = pos[key - k_lo]++;
        m.e_dst[e] = c;
        m.e_group[e] = gi;
        m.e_inst[e] = instance;
        m.e_weight[e] = w;
        m.e_delay[e] = ceil_steps(r.conn_delay_ms[ci], dt);
        m.e_src[e] = from_src ? 0xFFFFFFFFu : r.conn_src[ci];
        m.e_seq[e] = static_cast<uint32_t>(ci);
        maxd = std::max(maxd, m.e_delay[e]);
        if (from_src) m.src_edges[spos[r.conn_src[ci]]++] = e;
        // static-charge edges: the instance's compartment and w * cf[comp]
        // (the product apply_event forms, engine.cpp:455-459), so staged
        // delivery reads one edge record instead of chasing group -> comp
        if (S.kind == MCG_SYN_STATIC_CHARGE) {
          const McgKind& K = m.kinds[m.cell_kind[c]];
          const int comp = m.i_comp[G.inst + instance];
          m.e_comp[e] = comp;
          m.e_wcf[e] = w * m.k_cf[K.arr + comp];
        }
      }
      return maxd;
    };
    std::vector<size_t> cut(nthr + 1, nk1);
    cut[0] = 0;
    for (int t = 1; t < nthr; ++t) {  // first bucket whose start passes t / nthr of the edges
      const int64_t want = ne * t / nthr;
      cut[t] = static_cast<size_t>(std::upper_bound(bucket.begin(), bucket.begin() + nk1, want) - bucket.begin()) - 1;
      cut[t] = std::max(cut[t], cut[t - 1]);
      cut[t] = std::min(cut[t], nk1 - 1);
    }
    std::vector<int64_t> maxd(nthr, 0);
    std::vector<std::thread> th;
    for (int t = 0; t < nthr; ++t) {
      if (t + 1 < nthr) th.emplace_back([&, t] { maxd[t] = edges(cut[t], cut[t + 1]); });
      else maxd[t] = edges(cut[t], cut[t + 1]);
    }
    for (auto& x : th) x.join();
    for (int64_t d : maxd) m.max_delay_steps = std::max(m.max_delay_steps, d);
  }
  tm.mark("edges + instances");
  // ---- per-group state and delayed-calcium queues
  for (int c = 0; c < nl; ++c) {
    const McgKind& K = m.kinds[m.cell_kind[c]];
    for (int gi = 0; gi < K.n_groups; ++gi) {
      const int64_t cg = m.cg_off[c] + gi;
      const McgSpec& S = m.specs[K.spec0 + gi];
      McgCellGroup& G = m.cgs[cg];
      for (int i = 0; i < G.size; ++i) {
        const int64_t j = G.inst + i;
        if (S.kind == MCG_SYN_STDP_COND) m.i_stdp_w[j] = m.i_weight[j];  // any_stdp: allocated
        if (S.kind == MCG_SYN_HOMEO_CURRENT) m.i_homeo_w[j] = r.kinds[m.cell_kind[c]].placements[gi].syn.homeo.w_init_nA;
        if (S.kind == MCG_SYN_STC_CHARGE) m.i_stc_h[j] = S.h0;
      }
      if (S.kind == MCG_SYN_STC_CHARGE && G.size > 0) {
        // delayed-calcium queue: at most one entry per delivered event within
        // the delay window; start generous and let the engine grow it
        int64_t want = std::max<int64_t>(64, 8 * static_cast<int64_t>(G.size));
        const int64_t bound = cg_conns[cg] * (S.ca_delay + 1) + 8;
        want = std::min(want, std::max<int64_t>(bound, 16));
        int64_t cap = 16;
        while (cap < want) cap <<= 1;
        McgFifo F{};
        F.base = m.fifo_total;
        F.cap = static_cast<int32_t>(cap);
        m.fifo_total += cap;
        G.fifo = static_cast<int32_t>(m.fifos.size());
        m.fifos.push_back(F);
      }
      m.total_syn += G.size;
      if (S.kind == MCG_SYN_STC_CHARGE) m.stc_syn += G.size;
    }
  }

  tm.mark("fifos");
  // ---- sources (generate_source_events, engine.cpp:831-873) ----
  m.sources.resize(r.n_sources);
  for (int s = 0; s < r.n_sources; ++s) {
    const mcg_source& fs = r.sources[s];
    Source& S = m.sources[s];
    S.type = fs.type;
    if (fs.type == MCG_SRC_POISSON) {
      for (int i = 0; i + 2 < fs.n_values; i += 3) {
        S.t0.push_back(fs.values[i]);
        S.t1.push_back(fs.values[i + 1]);
        S.prob.push_back(fs.values[i + 2] * dt * 1e-3);
        S.a.push_back(ceil_steps(fs.values[i], dt));
        S.b.push_back(ceil_steps(fs.values[i + 1], dt));
      }
    } else if (fs.type == MCG_SRC_REGULAR) {
      S.r_t0 = fs.t0_ms;
      S.r_period = fs.period_ms;
      S.r_count = fs.count;
    } else {
      for (int i = 0; i < fs.n_values; ++i) S.steps.push_back(ceil_steps(fs.values[i], dt));
    }
  }

  // ---- probes (engine.cpp:393-403) ----
  m.probes.resize(r.n_probes);
  for (int i = 0; i < r.n_probes; ++i) {
    McgProbe& P = m.probes[i];
    P.gid = r.probe_gid[i];
    P.local = (P.gid >= g0 && P.gid < g1) ? static_cast<int32_t>(P.gid - g0) : -1;
    P.what = r.probe_what[i];
    P.comp = r.probe_comp[i];
    P.species = r.probe_species[i];
    P.group = r.probe_group[i];
    P.instance = r.probe_instance[i];
    P.every = r.probe_every[i] < 1 ? 1 : r.probe_every[i];
    P.out = 0;
  }

  tm.mark("sources + probes");
  // ---- totals ----
  for (int c = 0; c < nl; ++c) {
    const McgKind& K = m.kinds[m.cell_kind[c]];
    m.total_comps += K.n;
    m.species_comps += static_cast<int64_t>(K.n) * K.n_species;
    if (K.dyn == MCG_DYN_HH)
      for (int i = 0; i < K.n; ++i)
        if (m.k_g_na[K.arr + i] != 0.0) ++m.hh_comps;
  }
  tm.mark("totals");

}

}  // namespace mcg
