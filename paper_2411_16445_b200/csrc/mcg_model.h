// mcg_model.h — the engine's data layout in HBM, shared by the host-side
// materialization (mcg_build.cpp) and the kernels (mcg_engine.cu).
//
// The reference keeps per-cell C++ objects (CellRT, SynGroupRT: engine.hpp
// :71-115) and per-kind constants (CellKindRT: engine.cpp:106-134).  Here the
// same state is flattened into structure-of-arrays device buffers:
//   * compartments: cell-major (a cell's compartments are contiguous), so the
//     warp that owns a cell reads them with coalesced loads;
//   * synapse instances: one SoA per field, grouped per (cell, group) in
//     instance order — the order every sequential fold of the reference uses;
//   * per-kind constants (matrix coefficients, capacities, rate constants) are
//     shared by all cells of a kind and stay L1/L2-resident.
// Constants that the reference recomputes every step from the same operands
// (cap/dt, exp(-dt/tau), sigma/sqrt(dt), ...) are computed once on the host
// with the identical expression, so they are bitwise the reference's values.
#pragma once
#include <stdint.h>

enum { MCG_DYN_NONE = 0, MCG_DYN_LIF = 1, MCG_DYN_LIF_EXACT = 2, MCG_DYN_HH = 3 };

// CellKindRT (engine.cpp:106-134) + the per-step hoisted constants
struct McgKind {
  int32_t n;              // compartments
  int32_t dyn;            // MCG_DYN_*
  int32_t detector_comp, noise_comp;
  int32_t has_detector, has_bg;
  int32_t n_species, sps_idx, prp_idx, prp_enabled, prp_comp;
  int32_t n_groups;       // placements
  int32_t spec0;          // first entry of this kind in the spec table
  int32_t n_stc_groups;
  int64_t arr;            // offset of this kind's per-compartment arrays
  int64_t sp_arr;         // offset of per-species per-compartment arrays
  int64_t ref_steps;
  double threshold;
  double v_rev, r_mem, v_reset;
  double i_bg, sig_bg;    // sig_bg = sigma_bg / sqrt(dt)        (engine.cpp:659)
  double bg_t0, bg_t1;    // quiet window
  double lif_exact_f;     // exp(-dt / tau_mem)                  (engine.cpp:671)
  double prp_theta_star, prp_rate;  // PrpSynthesisParams      (mechanisms.hpp:253)
  double e_na, e_k;
  // Constant-diagonal systems: the Hines elimination of the diagonal does not
  // depend on the state, so its factors f[i] = coupling[i]/diag[i] and the
  // eliminated diagonal d[i] are precomputed with solve_tree's own operation
  // sequence (tree_solver.cpp:55-70).  v_const: the LIF-cable V system when
  // no conductance synapse is active (gs = g_leak + 0.0); sp_const: species.
  int32_t v_const, sp_const;
  // chain schedule of the constant systems (mcg_sweep.cuh; mcg_build.cpp
  // chain_schedule): ch_lp > 0 when the tree is a "spider" (only the root
  // branches, at most two chains) and every eliminated diagonal is in the
  // reciprocal-quotient range.  Positions: chain A [0, ch_lp), chain B
  // [ch_lp, 2 ch_lp), leaf side padded, tops aligned; the root at 2 ch_lp.
  // k_ch_idx[ch_arr + pos] = node of the position (-1: padding).
  int32_t ch_lp, ch_afirst;
  int64_t ch_arr;
  // chains of the general (non-constant diagonal) V solve, one lane each
  // (mcg_solve_tree_warp; mcg_build.cpp tree_chains): gch_n chains (0: none,
  // the one-thread solve), the schedule at k_ch_idx[gch_arr]
  int32_t gch_n, gch_pad;
  int64_t gch_arr;
};

// SynSpec per kind placement (recipe.hpp:82-98) + hoisted constants
struct McgSpec {
  int32_t kind;           // MCG_SYN_*
  int32_t comp, count;
  int32_t pad;
  double f_decay;         // exp(-dt / tau_syn)                  (engine.cpp:582/601)
  double e_rev;
  // STDP (mechanisms.hpp:20-53)
  double tau_pre, tau_post, a_pre, a_post, wmax;
  // homeostasis (mechanisms.hpp:57-76)
  double dw_plus, dw_minus, h_wmax;
  // STC (mechanisms.hpp:175-246)
  double h0, tau_h, theta_p, theta_d, gamma_p, gamma_d, sigma;
  double f_int, tau_z, theta_tag;
  double cf;              // exp(-dt / tau_c)                    (engine.cpp:619)
  double nz1, nz2;        // sigma*sqrt(k/tau_h)*sqrt(dt), k=1,2 (mechanisms.hpp:226)
  double cpre_s, cpost_s; // c_pre*calcium_scale, c_post*calcium_scale
  int64_t ca_delay;       // stc_ca_delay_steps                  (engine.cpp:258-269)
  double r_tau_h, r_tau_z;  // mcg_recip(tau_h), mcg_recip(tau_z)
};

// one (cell, group) pair: SynGroupRT's location in the instance SoA
struct McgCellGroup {
  int64_t inst;           // first instance
  int32_t size;
  int32_t active_n;       // length of the active list (stored at inst in `active`)
  int32_t spec;           // index into the spec table
  int32_t fifo;           // internal (delayed-calcium) queue index, -1 if none
};

// delayed-calcium queue of one stc group (replaces the per-cell heap,
// engine.cpp:34-39/497-503/555-560: with a fixed delay per group the queue is
// already in (step, seq) order)
struct McgFifo {
  int64_t base;           // offset into fifo storage
  int64_t head, tail;     // monotonic counters
  int32_t cap;
  int32_t pad;
};

// probe (ProbeSpec + resolved group), recipe.hpp:173-181
struct McgProbe {
  uint32_t gid;
  int32_t local;          // local cell index, -1 if not on this shard
  int32_t what, comp, species, group, instance, every;
  int64_t out;            // write cursor base for the current call
};

// events: one 64-bit key per EventRec,  dst | (step - base) | rank
struct McgKeyLayout {
  int32_t rank_bits, step_bits, dst_bits;
  int32_t pad;
};

// edge table indexed by rank (edges sorted by (src_key, seq); engine.cpp:25-31)
// dst, group, instance, weight, delay in separate arrays (see McgDev)
