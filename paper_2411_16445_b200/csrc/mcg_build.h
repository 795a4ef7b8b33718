// mcg_build.h — host-side materialization of a recipe into the device layout.
//
// Restates Engine::Impl::build / build_kind / append_instance
// (engine.cpp:189-408) and discretize (morphology.cpp:67-143) in C++: the
// same expressions in the same order, so every constant the kernels consume
// is bitwise the value the reference computes.  The result is a set of flat
// host vectors that mcg_engine.cu uploads once.
#pragma once
#include <stdexcept>
#include <string>
#include <memory>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/mcg.h"
#include "mcg_model.h"

namespace mcg {

// std::allocator that default-initializes (no zero fill on resize): the
// build's large arrays are written completely, or filled by host threads
// (first touch in parallel), so the serial value-initialization of
// std::vector::resize would only cost page faults on one core
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept(std::is_nothrow_default_constructible<U>::value) {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};
template <class T>
using HVec = std::vector<T, NoInitAlloc<T>>;


struct Error : std::runtime_error {
  mcg_status code;
  Error(mcg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// CompartmentGrid (morphology.hpp:36-53)
struct Grid {
  std::vector<double> length, area, xs, volume;
  std::vector<int32_t> parent;
  std::vector<uint8_t> tag;
  std::vector<uint32_t> segment_of;
  double total_volume = 0;
  int size() const { return static_cast<int>(length.size()); }
};

Grid discretize(const mcg_kind& k);
int64_t ceil_steps(double t_ms, double dt_ms);

// reciprocal operand of mcg_div (mcg_device.cuh): RN(1/d), or 0 outside the
// range where the FMA-corrected quotient is proven correctly rounded
inline double mcg_recip(double d) {
  const double a = d < 0 ? -d : d;
  return (a >= 0x1p-200 && a <= 0x1p200) ? 1.0 / d : 0.0;
}

struct Source {
  int32_t type;
  std::vector<double> t0, t1, prob;   // poisson windows (prob = rate*dt*1e-3)
  std::vector<int64_t> a, b;           // poisson window step bounds
  std::vector<int64_t> steps;          // scripted: ceil_steps of each time
  double r_t0 = 0, r_period = 0;       // regular
  int64_t r_count = 0;
};

struct HostModel {
  double dt = 0;
  uint64_t seed = 0;
  int32_t rank = 0, world = 1;
  int32_t n_cells_global = 0;
  int32_t max_shard_cells = 0;  // largest shard of the partition (spike block capacity)
  uint32_t gid_begin = 0, gid_end = 0;  // local shard [begin, end)
  int64_t min_delay_steps = -1;

  // kinds
  std::vector<McgKind> kinds;
  std::vector<Grid> grids;
  std::vector<int32_t> k_parent;
  std::vector<int32_t> k_ch_idx;         // chain schedules (McgKind::ch_arr)
  std::vector<double> k_cap_dt, k_g_leak, k_g_leak_rhs, k_axial, k_g_na, k_g_k, k_cf, k_volume;
  std::vector<double> k_sp_cap_dt, k_sp_gs, k_sp_coupling, k_sp_init;
  std::vector<double> k_vf, k_vd;        // precomputed V elimination (per comp)
  std::vector<double> k_sp_f, k_sp_d;    // precomputed species elimination
  std::vector<double> k_vr, k_sp_r, k_rvol;  // mcg_recip of k_vd, k_sp_d, k_volume
  std::vector<double> k_sp_decay_tau;  // per kind species (for fast-forward)
  std::vector<int64_t> k_sp_off;       // per kind: offset into k_sp_decay_tau
  std::vector<McgSpec> specs;

  // local cells
  std::vector<int32_t> cell_kind;
  std::vector<int64_t> comp_off, sp_off, cg_off;
  std::vector<double> v, hh_m, hh_h, hh_n, species;
  std::vector<double> det_prev;
  std::vector<int32_t> armed;
  std::vector<int64_t> refr_until;
  std::vector<uint32_t> internal_seq;

  // synapse groups and instances
  std::vector<McgCellGroup> cgs;
  int64_t n_inst = 0;  // synapse instances (arrays left empty by the build are all zero)
  HVec<int32_t> i_comp;
  HVec<double> i_weight, i_kernel, i_stdp_pre, i_stdp_post, i_stdp_w, i_homeo_w;
  HVec<int64_t> i_stdp_last;
  HVec<double> i_stc_h, i_stc_z, i_stc_c, i_sps_abs;
  std::vector<McgFifo> fifos;
  int64_t fifo_total = 0;

  // edges with a local destination, sorted by (src_key, seq) -> rank
  HVec<int32_t> e_dst, e_group;
  HVec<uint32_t> e_inst;
  HVec<double> e_weight;
  HVec<uint32_t> e_src, e_seq;              // EventRec.src / seq of each edge (EventOrder)
  HVec<int32_t> e_comp;                     // static-charge edges: target compartment (else -1)
  HVec<double> e_wcf;                       // and weight * charge_factor[comp] (engine.cpp:457)
  HVec<int64_t> e_delay;
  std::vector<int64_t> out_begin, out_end;  // per global gid
  std::vector<int64_t> src_edge_off;        // per source CSR into src_edges
  std::vector<int64_t> src_edges;           // ranks
  int64_t max_delay_steps = 0;

  // connection resolution left to the device (build_model(..., defer_edges)):
  // the counts and offsets of pass 0 are here, the instance choice and the
  // edge records are not (e_* and src_edges empty, i_weight unset) until the
  // engine resolves them on the device (mcg_resolve.cuh)
  bool edges_deferred = false;
  int64_t n_edges = 0;                 // local edges (the length of every e_* array)
  std::vector<int64_t> cg_conn_off;    // per (cell, group): first local connection, by cg
  std::vector<uint8_t> cg_static;      // per (cell, group): static-charge placement
  std::vector<int32_t> cg_count;       // per (cell, group): pre-placed count (0: appended)
  std::vector<int32_t> cg_comp;        // per (cell, group): the placement's compartment
  std::vector<double> cg_cf;           // per (cell, group): charge factor of that compartment

  std::vector<Source> sources;
  std::vector<McgProbe> probes;

  // totals (stats)
  int64_t total_comps = 0, total_syn = 0, stc_syn = 0, hh_comps = 0, species_comps = 0;
};

// Eliminate a constant diagonal exactly as solve_tree does (tree_solver.cpp:
// 55-70): diag = cap + gs, += coupling (own, then children ascending), then
// leaves-to-root.  Writes f[i] (i >= 1) and the eliminated diagonal d[i].
// Returns false if the system is singular (the engine then runs the full
// solve, which reports the NumericError at the same step as the reference).
bool eliminate_constant(int n, const int32_t* parent, const double* cap, const double* gs,
                        const double* coupling, double* f, double* d);

// Chain schedule of a tree for the lockstep sweep (mcg_sweep.cuh): if only
// the root branches (into at most two chains), returns the padded chain length
// LP and fills idx (2 LP + 1 positions, -1 = padding) and a_first; else 0.
int chain_schedule(int n, const int32_t* parent, std::vector<int32_t>& idx, int& a_first);

// Chains of a tree for the warp-parallel general solve (mcg_solve_tree_warp):
// a chain runs from a node down while each node has exactly one child; the
// children of its bottom node start the chains of the next level.  Layout:
// [nch, maxlev, maxch, per chain (node offset, length, level, nchild,
// child chain ids by descending top index, -1 padded to maxch), nodes of
// every chain top to bottom].  Returns nch, or 0 (more than 32 chains, or a
// parent index not below its node).
int tree_chains(int n, const int32_t* parent, std::vector<int32_t>& out);

// Materialize; throws mcg::Error with the reference's messages.
// threads <= 0: build_threads() (MCG_BUILD_THREADS or the hardware threads)
// defer_edges: leave pass 1 (instances, edge records, source CSR) to the
// device when the recipe allows it (no STDP placement: its weights start from
// the resolved ones); m.edges_deferred says whether it did
void build_model(const mcg_recipe& r, const mcg_options& opt, HostModel& m, int threads = 0,
                 bool defer_edges = false);

// Shard assignment: contiguous gid ranges balanced by (compartments +
// synapse instances); identical on every rank.
void partition(const mcg_recipe& r, int world, std::vector<uint32_t>& bounds);

}  // namespace mcg
