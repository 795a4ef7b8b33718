// mcg_device.cuh — device-side state view and the per-cell mechanism code.
//
// One warp owns one cell for a whole min-delay epoch (cells are independent
// inside an epoch: engine.cpp:913-942).  Work that the reference does as an
// order-dependent fold (event delivery, active-list conductance sums, the SPS
// fold, the Hines sweep) runs on lane 0 in the reference's order; work that
// is independent per synapse instance (STC early/late phase, kernel decay,
// STDP/homeostasis/STC post-spike hooks) runs across the 32 lanes.
//
// Mechanism ABI mapping (Arbor names -> reference code -> here):
//   init              Impl::build / append_instance   -> mcg_build.cpp
//   apply_events      apply_event  (engine.cpp:452)    -> mcg_apply_event
//   advance_state     step_cell §2 (engine.cpp:575)    -> mcg_advance_*
//   compute_currents  step_cell §2-3 (:578-664)        -> gsyn / rhs_current folds
//   post_event        post_event (engine.cpp:515)      -> mcg_post_event
#pragma once
#include <stdint.h>

#include "../../include/mcg.h"
#include "mcg_model.h"
#include "mcg_rng.h"

#define MCG_FULL 0xffffffffu
#define MCG_ERR_FLAG_SINGULAR 1
#define MCG_ERR_FLAG_FIFO 2
#define MCG_ERR_FLAG_ACTIVE 4
#define MCG_ERR_FLAG_SPIKES 8

// memo of one STC instance's noise pair (mcg_stc_noise); tag -1: empty
struct __align__(16) McgNzCache {
  long long tag;
  double z;
};

struct McgDev {
  double dt;
  uint64_t seed;
  // kinds
  const McgKind* kinds;
  const McgSpec* specs;
  const int32_t* k_parent;
  const int32_t* k_ch_idx;    // chain schedules (McgKind::ch_arr)
  const double *k_cap_dt, *k_g_leak, *k_g_leak_rhs, *k_axial, *k_g_na, *k_g_k, *k_cf, *k_volume;
  const double *k_sp_cap_dt, *k_sp_gs, *k_sp_coupling;
  // cells
  int32_t n_cells;
  uint32_t gid0;
  const int32_t* cell_kind;
  const int64_t *comp_off, *sp_off, *cg_off;
  double *v, *hh_m, *hh_h, *hh_n, *species, *det_prev;
  int32_t* armed;
  int64_t* refr_until;
  uint32_t* internal_seq;
  // per-compartment scratch (global fallback for cells too large for smem)
  double *s_gsyn, *s_gsyn_rhs, *s_rhs_cur, *s_diag, *s_rhs;
  double* s_r2;               // (1 + sp_max) x compartments
  const double *k_vf, *k_vd, *k_sp_f, *k_sp_d;
  const double *k_vr, *k_sp_r, *k_rvol;  // mcg_recip of k_vd, k_sp_d, k_volume
  int32_t sp_max;             // max species per kind
  int32_t smem_n;             // cells with n <= smem_n are staged in shared memory
  int32_t smem_stride;        // doubles per warp in dynamic shared memory
  // groups, instances
  McgCellGroup* cgs;
  McgFifo* fifos;
  int64_t* fifo_step;
  uint64_t* fifo_si;
  uint32_t* fifo_src;         // the originating event's src and weight, kept for
  double* fifo_w;             // checkpoints (the reference's internal EventRec copies them)
  const int32_t* i_comp;
  double *i_weight, *i_kernel;
  int32_t* i_active;
  double *i_stdp_pre, *i_stdp_post, *i_stdp_w;
  int64_t* i_stdp_last;
  double* i_homeo_w;
  double *i_stc_h, *i_stc_z, *i_stc_c, *i_sps_abs;
  McgNzCache* stc_nz;  // per STC instance: z1 of the last even step's noise pair
  // per-cell inboxes (mcg_events.cuh): incoming keys of this epoch (unsorted)
  // and the sorted pending list, double buffered; key = step << rank_bits | rank
  uint64_t* inc;
  int32_t* inc_n;
  int32_t inc_cap;
  uint64_t* pend;
  int32_t* pend_sel;
  int32_t* pend_off;
  int32_t* pend_n;
  int32_t pend_cap;
  int32_t rank_bits;
  const int64_t* ctl;       // [0] batch base step, [1] target step, [2] epoch length
  int32_t* abort;
  const int32_t* e_dst;
  const int32_t* e_group;
  const uint32_t* e_inst;
  const double* e_weight;
  const uint32_t* e_src;      // EventRec.src of each edge (gid, 0xFFFFFFFF for sources)
  const int32_t* e_comp;      // static-charge edges: compartment, w * cf (mcg_build.cpp)
  const double* e_wcf;
  const int64_t* e_delay;
  // spikes of this epoch: [cell][sp_cap]
  int32_t sp_cap;
  int32_t* sp_count;
  int64_t* sp_step;
  double* sp_t;
  // probes: per-cell CSR of probe indices, per-probe output
  const McgProbe* probes;
  const int32_t* probe_off;
  const int32_t* probe_idx;
  double* trace_buf;
  const int64_t* trace_base;  // per probe
  // status
  int32_t* err;
  unsigned long long* delivered;
  // optional per-cell RNG key override (mcg_set_cell_rng; k_point only):
  // cell c draws with key (cell_seed[c], cell_key_gid[c], ...) instead of
  // (seed, gid0 + c, ...): independent trials of one protocol in one engine
  const uint64_t* cell_seed;
  const uint32_t* cell_key_gid;
};

// x / d, bitwise IEEE division, from y = mcg_recip(d) = RN(1/d): with
// q = RN(x*y) and the exact remainder r = x - q*d (one FMA), RN(q + r*y) is the
// correctly rounded quotient (Markstein's theorem) as long as nothing under-
// or overflows, which the operand ranges below guarantee.  x == +-0 gives
// q = x*y, the IEEE signed zero of x/d.  Elsewhere (y == 0, tiny or huge x,
// inf, nan) it is the plain division.  Replaces a ~110-cycle dependent DDIV
// with three FP64 operations on the sweep critical paths.
// out of line: the rare paths keep their register pressure off the callers
__device__ __noinline__ double mcg_div_slow(double x, double d) { return __ddiv_rn(x, d); }

__device__ __forceinline__ double mcg_div(double x, double d, double y) {
  // the quotient is computed unconditionally (nothing on the dependent chain
  // waits for the range test); only the rare fallback is a branch
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(-q, d, x);
  double res = __fma_rn(r, y, q);
  const double ax = fabs(x);
  if (ax == 0.0) res = q;
  if (__builtin_expect(y == 0.0 || ax > 0x1p700 || (ax < 0x1p-700 && ax != 0.0), 0))
    res = mcg_div_slow(x, d);
  return res;
}

// a % b for a >= 0, b > 0: the 32-bit unsigned remainder when both fit (a
// short sequence instead of the 64-bit division routine; the queue counters
// and step numbers of any realistic run stay below 2^32)
__device__ __forceinline__ int64_t mcg_mod(int64_t a, int64_t b) {
  if (((static_cast<uint64_t>(a) | static_cast<uint64_t>(b)) >> 32) == 0)
    return static_cast<uint32_t>(a) % static_cast<uint32_t>(b);
  return a % b;
}

__device__ __forceinline__ unsigned mcg_lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// stdp_decay (mechanisms.hpp:35-38)
__device__ __forceinline__ void mcg_stdp_decay(double& pre, double& post, const McgSpec& S,
                                               double gap) {
  pre *= mcg_exp(-gap / S.tau_pre);
  post *= mcg_exp(-gap / S.tau_post);
}

// STC instance state of the addressed group: in global memory (slot0 < 0) or
// in the batch kernel's shared-memory copy, SoA with `stride` doubles per
// field (h, z, c, |h-h0|), instance i at slot0 + i
struct McgStcSm {
  double* base;
  int32_t stride, slot0;
};

// ---- apply_events (engine.cpp:452-513); lane 0 only -----------------------
__device__ void mcg_apply_event(const McgDev& D, const McgKind& K, int c, int64_t cg0,
                                double* V, int32_t group, uint32_t inst, double w, int etype,
                                bool refractory, int64_t s, McgStcSm R = McgStcSm{nullptr, 0, -1},
                                uint32_t src = 0) {
  McgCellGroup& G = D.cgs[cg0 + group];
  const McgSpec& S = D.specs[G.spec];
  const int64_t j = G.inst + inst;
  switch (S.kind) {
    case MCG_SYN_STATIC_CHARGE:
      if (!refractory && w != 0.0) {
        const int comp = D.i_comp[j];
        V[comp] += w * D.k_cf[K.arr + comp];
      }
      break;
    case MCG_SYN_STATIC_COND:
    case MCG_SYN_STATIC_CURRENT:
      if (w != 0.0) {
        if (D.i_kernel[j] == 0.0) {
          if (G.active_n >= G.size) atomicOr(D.err, MCG_ERR_FLAG_ACTIVE);
          else D.i_active[G.inst + G.active_n++] = static_cast<int32_t>(inst);
        }
        D.i_kernel[j] += w;
      }
      break;
    case MCG_SYN_STDP_COND: {
      double pre = D.i_stdp_pre[j], post = D.i_stdp_post[j];
      const double gap = double(s - D.i_stdp_last[j]) * D.dt;
      if (gap > 0) mcg_stdp_decay(pre, post, S, gap);
      D.i_stdp_last[j] = s;
      pre += S.a_pre;  // stdp_on_pre
      const double ww = D.i_stdp_w[j] + post;
      D.i_stdp_pre[j] = pre;
      D.i_stdp_post[j] = post;
      D.i_stdp_w[j] = ww;
      const double weff = fmin(fmax(ww, 0.0), S.wmax);
      if (weff != 0.0) {
        if (D.i_kernel[j] == 0.0) {
          if (G.active_n >= G.size) atomicOr(D.err, MCG_ERR_FLAG_ACTIVE);
          else D.i_active[G.inst + G.active_n++] = static_cast<int32_t>(inst);
        }
        D.i_kernel[j] += weff;
      }
      break;
    }
    case MCG_SYN_HOMEO_CURRENT: {
      const double hw = fmin(D.i_homeo_w[j] + S.dw_plus, S.h_wmax);
      D.i_homeo_w[j] = hw;
      if (hw != 0.0) {
        if (D.i_kernel[j] == 0.0) {
          if (G.active_n >= G.size) atomicOr(D.err, MCG_ERR_FLAG_ACTIVE);
          else D.i_active[G.inst + G.active_n++] = static_cast<int32_t>(inst);
        }
        D.i_kernel[j] += hw;
      }
      break;
    }
    case MCG_SYN_STC_CHARGE: {
      const bool sm = R.slot0 >= 0;
      const int32_t sl = R.slot0 + int32_t(inst);
      if (etype == 1) {
        if (sm) R.base[2 * R.stride + sl] += S.cpre_s;  // stc_on_pre_calcium
        else D.i_stc_c[j] += S.cpre_s;
      } else {
        // delayed calcium: internal event at s + delay, seq = internal_seq++
        McgFifo& F = D.fifos[G.fifo];
        if (F.tail - F.head >= F.cap) {
          atomicOr(D.err, MCG_ERR_FLAG_FIFO);
        } else {
          const int64_t slot = F.base + mcg_mod(F.tail, F.cap);
          D.fifo_step[slot] = s + S.ca_delay;
          D.fifo_si[slot] = (uint64_t(D.internal_seq[c]) << 32) | uint64_t(inst);
          D.fifo_src[slot] = src;
          D.fifo_w[slot] = w;
          ++F.tail;
        }
        ++D.internal_seq[c];
        if (!refractory) {
          const int comp = S.comp;  // every instance sits on the placement's compartment
          const double tw = sm ? R.base[sl] + S.h0 * R.base[R.stride + sl]
                               : D.i_stc_h[j] + S.h0 * D.i_stc_z[j];
          V[comp] += tw * w * D.k_cf[K.arr + comp];
        }
      }
      break;
    }
  }
}

// solve_tree (tree_solver.cpp:46-74), lane 0; returns false if singular
__device__ bool mcg_solve_tree(int n, const int32_t* par, const double* cap, const double* gs,
                               const double* coup, const double* rhs, double* v, double* diag,
                               double* r2) {
  for (int i = 0; i < n; ++i) {
    diag[i] = cap[i] + gs[i];
    r2[i] = cap[i] * v[i] + rhs[i];
  }
  for (int i = 1; i < n; ++i) {
    diag[i] += coup[i];
    diag[par[i]] += coup[i];
  }
  for (int i = n - 1; i >= 1; --i) {
    if (diag[i] <= 0.0) return false;
    const double f = coup[i] / diag[i];
    diag[par[i]] -= f * coup[i];
    r2[par[i]] += f * r2[i];
  }
  if (diag[0] <= 0.0) return false;
  v[0] = r2[0] / diag[0];
  for (int i = 1; i < n; ++i) v[i] = (r2[i] + coup[i] * v[par[i]]) / diag[i];
  return true;
}

// RN(1/d) when d is in the range where Markstein's quotient from it is exact
// (|d| in [2^-200, 2^200]); 0.0 otherwise, which sends mcg_div to IEEE division
__device__ __forceinline__ double mcg_rcp_or_zero(double d) {
  const double ad = fabs(d);
  return (ad >= 0x1p-200 && ad <= 0x1p200) ? __drcp_rn(d) : 0.0;
}

// solve_tree (tree_solver.cpp:46-74) with the reference's operations in the
// reference's order, arranged for one thread's latency: the elimination
// carries the node it last updated (a chain's next node, usually) in
// registers instead of a shared-memory round trip, every division is
// Markstein's quotient from RN(1/d) (mcg_div; IEEE division outside its
// proven range), and the substitution's reciprocals are formed during the
// elimination, off its dependent chain (stored over gs, which the caller no
// longer needs).  Returns false if singular, at the same node as the loop.
__device__ bool mcg_solve_tree_fast(int n, const int32_t* par, const double* cap, double* gs_y,
                                    const double* coup, const double* rhs, double* v, double* diag,
                                    double* r2) {
  for (int i = 0; i < n; ++i) {
    diag[i] = cap[i] + gs_y[i];
    r2[i] = cap[i] * v[i] + rhs[i];
  }
  for (int i = 1; i < n; ++i) {
    diag[i] += coup[i];
    diag[par[i]] += coup[i];
  }
  int cp = -1;  // node whose diag / r2 (every contribution so far) are in cd / cr only
  double cd = 0.0, cr = 0.0;
  for (int i = n - 1; i >= 1; --i) {
    double di, ri;
    if (i == cp) {
      di = cd;
      ri = cr;
      diag[i] = di;
      r2[i] = ri;
    } else {
      if (cp >= 0) {
        diag[cp] = cd;
        r2[cp] = cr;
      }
      di = diag[i];
      ri = r2[i];
    }
    if (di <= 0.0) return false;
    const double ci = coup[i];
    const double yi = mcg_rcp_or_zero(di);
    gs_y[i] = yi;
    const double f = mcg_div(ci, di, yi);
    const int p = par[i];
    double dp, rp;
    if (p == cp && cp != i) {  // still current in registers (also just stored)
      dp = cd;
      rp = cr;
    } else {
      dp = diag[p];
      rp = r2[p];
    }
    dp -= f * ci;  // diag[par[i]] -= f * coup[i]
    rp += f * ri;  // r2[par[i]] += f * r2[i]
    cp = p;
    cd = dp;
    cr = rp;
  }
  if (cp >= 0) {
    diag[cp] = cd;
    r2[cp] = cr;
  }
  if (diag[0] <= 0.0) return false;
  double vp = mcg_div(r2[0], diag[0], mcg_rcp_or_zero(diag[0]));
  v[0] = vp;
  for (int i = 1; i < n; ++i) {
    const int p = par[i];
    const double vpar = (p == i - 1) ? vp : v[p];
    vp = mcg_div(r2[i] + coup[i] * vpar, diag[i], gs_y[i]);
    v[i] = vp;
  }
  return true;
}

// solve_tree (tree_solver.cpp:46-74) by a whole warp, one lane per chain of
// the tree (mcg_build.cpp tree_chains; all 32 lanes call it).  Every node
// takes the reference's operations in the reference's order: its diagonal
// gathers cap + gs, its own coupling and its children's couplings in
// ascending child order (:55-62); in the elimination (:63-70) a node's
// children contribute in descending index order -- inside a chain the one
// child below it, at a chain's bottom the child chains' tops, gathered from
// their lanes by shuffles in that order -- before it is eliminated itself;
// the substitution (:71-73) runs top to bottom, a chain's top reading its
// parent from the level above.  What the loop serializes across branches
// runs side by side: the dependent chain is the deepest path of chains, not
// the node count.  Quotients as mcg_solve_tree_fast (Markstein from RN(1/d),
// reciprocals kept in gs_y for the substitution).  Returns false (on every
// lane) if a diagonal met during elimination is not positive.
__device__ bool mcg_solve_tree_warp(const int32_t* G, const int32_t* par, const double* cap, double* gs_y,
                                    const double* coup, const double* rhs, double* v, double* diag,
                                    double* r2, int lane) {
  const int nch = G[0], maxlev = G[1], maxch = G[2];
  const int rec = 4 + maxch;
  const int32_t* CH = G + 3;
  const int32_t* ND = CH + nch * rec;
  const bool on = lane < nch;
  int off = 0, len = 0, lev = -1, nchild = 0;
  if (on) {
    off = CH[lane * rec];
    len = CH[lane * rec + 1];
    lev = CH[lane * rec + 2];
    nchild = CH[lane * rec + 3];
  }
  // ---- diag and r2 of my chain's nodes
  for (int k = 0; k < len; ++k) {
    const int i = ND[off + k];
    double d = cap[i] + gs_y[i];
    if (i >= 1) d += coup[i];
    if (k + 1 < len) {
      d += coup[ND[off + k + 1]];
    } else {
      for (int q = nchild - 1; q >= 0; --q) {  // child chains, ascending top index
        const int cc = CH[lane * rec + 4 + q];
        d += coup[ND[CH[cc * rec]]];
      }
    }
    diag[i] = d;
    r2[i] = cap[i] * v[i] + rhs[i];
  }
  // ---- elimination, deepest chains first
  bool bad = false;
  double td = 0.0, tr = 0.0;  // my top's terms for its parent: f*coup, f*r2
  for (int L = maxlev; L >= 0; --L) {
    const bool act = lev == L;
    double cd = 0.0, cr = 0.0;
    if (act) {
      const int b = ND[off + len - 1];
      cd = diag[b];
      cr = r2[b];
    }
    for (int q = 0; q < maxch; ++q) {
      const bool take = act && q < nchild;
      const int src = take ? CH[lane * rec + 4 + q] : lane;
      const double a = __shfl_sync(0xffffffffu, td, src), c = __shfl_sync(0xffffffffu, tr, src);
      if (take) {
        cd -= a;  // diag[par[i]] -= f * coup[i]
        cr += c;  // r2[par[i]] += f * r2[i]
      }
    }
    if (act) {
      // the nodes below the top: each one's parent is the next one up
      int i = ND[off + len - 1];
      for (int k = len - 1; k >= 1; --k) {
        const int p = ND[off + k - 1];
        const double pd = diag[p], pr = r2[p], ci = coup[i];
        diag[i] = cd;
        r2[i] = cr;
        bad |= cd <= 0.0;
        const double yi = mcg_rcp_or_zero(cd);
        gs_y[i] = yi;
        const double f = mcg_div(ci, cd, yi);
        cd = pd - f * ci;
        cr = pr + f * cr;
        i = p;
      }
      // the top: the root is not eliminated; any other top's terms go to
      // its parent's lane
      diag[i] = cd;
      r2[i] = cr;
      if (i != 0) {
        bad |= cd <= 0.0;
        const double ci = coup[i];
        const double yi = mcg_rcp_or_zero(cd);
        gs_y[i] = yi;
        const double f = mcg_div(ci, cd, yi);
        td = f * ci;
        tr = f * cr;
      }
    }
    __syncwarp();
  }
  // ---- substitution, root chain first
  for (int L = 0; L <= maxlev; ++L) {
    if (lev == L) {
      // the top (the root, or a node whose parent the level above solved),
      // then the nodes below it, each from the one just solved
      int i = ND[off];
      double vp;
      if (i == 0) {
        bad |= diag[0] <= 0.0;
        vp = mcg_div(r2[0], diag[0], mcg_rcp_or_zero(diag[0]));
      } else {
        vp = mcg_div(r2[i] + coup[i] * v[par[i]], diag[i], gs_y[i]);
      }
      v[i] = vp;
      for (int k = 1; k < len; ++k) {
        i = ND[off + k];
        vp = mcg_div(r2[i] + coup[i] * vp, diag[i], gs_y[i]);
        v[i] = vp;
      }
    }
    __syncwarp();
  }
  return !__any_sync(0xffffffffu, bad);
}

// solve_tree with a precomputed constant elimination (McgKind::v_const /
// sp_const): the rhs sweep and back-substitution of tree_solver.cpp:55-73
// with f[i] = coupling[i]/diag[i] and the eliminated diagonal d[i] taken from
// mcg::eliminate_constant.  r2 must hold cap[i]*v[i] + rhs[i] on entry.
__device__ __forceinline__ void mcg_solve_const(int n, const int32_t* par, const double* coup,
                                                const double* f, const double* d, double* v,
                                                double* r2) {
  for (int i = n - 1; i >= 1; --i) r2[par[i]] += f[i] * r2[i];
  v[0] = r2[0] / d[0];
  for (int i = 1; i < n; ++i) v[i] = (r2[i] + coup[i] * v[par[i]]) / d[i];
}

// HH rates (engine.cpp:41-54) with the glibc-faithful exp
__device__ __forceinline__ double mcg_hh_am(double v) {
  const double x = v + 40.0;
  if (fabs(x) < 1e-7) return 1.0;
  return 0.1 * x / (1.0 - mcg_exp(-x / 10.0));
}
__device__ __forceinline__ double mcg_hh_bm(double v) { return 4.0 * mcg_exp(-(v + 65.0) / 18.0); }
__device__ __forceinline__ double mcg_hh_ah(double v) { return 0.07 * mcg_exp(-(v + 65.0) / 20.0); }
__device__ __forceinline__ double mcg_hh_bh(double v) {
  return 1.0 / (1.0 + mcg_exp(-(v + 35.0) / 10.0));
}
__device__ __forceinline__ double mcg_hh_an(double v) {
  const double x = v + 55.0;
  if (fabs(x) < 1e-7) return 0.1;
  return 0.01 * x / (1.0 - mcg_exp(-x / 10.0));
}
__device__ __forceinline__ double mcg_hh_bn(double v) {
  return 0.125 * mcg_exp(-(v + 65.0) / 80.0);
}

// STC early/late phase of one instance (mechanisms.hpp:213-242,
// engine.cpp:624-644) on values already in registers: h, z, calcium c and the
// |h - h0| last folded into the SPS pool (a).  Returns true when |h - h0|
// changed; `delta` is then the SPS increment at the placement's compartment.
// late: the cell has a PRP pool (prp = its value at that compartment).
struct McgStcVal {
  double h, z, c, a;
};

// plasticity noise draw of one STC instance (calcium above a threshold):
// normal_for(key, s) with the instance's key. Steps 2p and 2p + 1 draw the two
// normals of one Box-Muller pair, so the even step leaves z1 in the instance's
// McgNzCache entry for the odd one (a memo of a pure function of the key and
// the step: valid across restores and fast-forwards)
__device__ __noinline__ double mcg_stc_noise(McgNzCache* e, uint64_t seed, uint32_t gid, int gi,
                                             int i, int64_t s) {
  const uint64_t n = static_cast<uint64_t>(s);
  const long long pr = static_cast<long long>(n >> 1);
  if (n & 1u) {
    const McgNzCache c = *e;
    if (c.tag == pr) return c.z;
  }
  const mcg_key key = mcg_make_key(seed, gid, (2ull << 32) | uint64_t(gi), uint64_t(i));
  double z0, z1;
  mcg_normal_pair_for(&key, n, &z0, &z1);
  if (n & 1u) return z1;
  McgNzCache c;
  c.tag = pr;
  c.z = z1;
  *e = c;
  return z0;
}

// A synapse at rest — h exactly at its baseline, calcium above neither
// threshold, |h - h0| already folded as 0 — takes a step that only decays its
// calcium: stc_early_step adds exactly +0 to h (0.1*(h0 - h) = +0, no noise),
// |h - h0| = +0 equals the folded value, and stc_late_step (when it runs: a
// nonnegative tag threshold, finite PRP and f_int) adds a signed zero to z,
// which is never -0 (it starts at +0 and only changes by nonzero sums).
// the spec fields the test reads, loaded once per placement (a register copy:
// the spec table may live in global or shared memory)
struct McgStcRest {
  long long h0_bits;
  double theta_p, theta_d, cf;
  bool late_noop;  // stc_late_step at h == h0 adds a signed zero for any finite PRP
};

__device__ __forceinline__ McgStcRest mcg_stc_rest_of(const McgSpec& S) {
  McgStcRest r;
  r.h0_bits = __double_as_longlong(S.h0);
  r.theta_p = S.theta_p;
  r.theta_d = S.theta_d;
  r.cf = S.cf;
  r.late_noop = S.theta_tag >= 0.0 && fabs(S.f_int) <= 1.7976931348623157e308;
  return r;
}

__device__ __forceinline__ bool mcg_stc_at_rest(const McgStcRest& R, bool late, double prp, double h,
                                                double c, double a) {
  return __double_as_longlong(h) == R.h0_bits && !(c > R.theta_p) && !(c > R.theta_d) && a == 0.0 &&
         (!late || prp <= 0.0 || (R.late_noop && prp <= 1.7976931348623157e308));
}

__device__ __forceinline__ bool mcg_stc_step(const McgSpec& S, double dt, uint64_t seed,
                                             uint32_t gid, int gi, int i, int64_t s, bool late,
                                             double prp, double vol, double rvol, McgStcVal& v,
                                             double& delta, McgNzCache* nz) {
  double h = v.h;
  const bool up = v.c > S.theta_p, dn = v.c > S.theta_d;
  double nrm = 0.0;
  if (S.sigma != 0.0 && (up || dn)) nrm = mcg_stc_noise(nz, seed, gid, gi, i, s);
  // stc_early_step
  const int crossings = int(up) + int(dn);
  double d = 0.1 * (S.h0 - h);
  if (up) d += S.gamma_p * (10.0 - h);
  if (dn) d -= S.gamma_d * h;
  double dh = mcg_div(d, S.tau_h, S.r_tau_h) * dt;
  if (crossings > 0 && S.sigma != 0.0) dh += (crossings == 1 ? S.nz1 : S.nz2) * nrm;
  h += dh;
  const double na = fabs(h - S.h0);
  bool changed = false;
  if (na != v.a) {
    delta = mcg_div(na - v.a, vol, rvol);
    v.a = na;
    changed = true;
  }
  // stc_late_step
  if (late && !(prp <= 0.0)) {
    double dd = 0.0;
    if (h - S.h0 > S.theta_tag) dd += (1.0 - v.z);
    if (S.h0 - h > S.theta_tag) dd -= (v.z + 0.5);
    v.z += mcg_div(prp * S.f_int * dd * dt, S.tau_z, S.r_tau_z);
  }
  v.c *= S.cf;
  v.h = h;
  return changed;
}

// probe_value (engine.cpp:795-829)
__device__ double mcg_probe_value(const McgDev& D, const McgKind& K, int c, const McgProbe& P,
                                  const double* V, const double* SP,
                                  McgStcSm R = McgStcSm{nullptr, 0, -1}) {
  if (P.what == MCG_PROBE_VOLTAGE) return (K.dyn == MCG_DYN_NONE) ? 0.0 : V[P.comp];
  if (P.what == MCG_PROBE_SPECIES) return SP[int64_t(P.species) * K.n + P.comp];
  const McgCellGroup& G = D.cgs[D.cg_off[c] + P.group];
  const McgSpec& S = D.specs[G.spec];
  const int64_t j = G.inst + P.instance;
  if (S.kind == MCG_SYN_STC_CHARGE && R.slot0 >= 0) {
    const double* b = R.base + R.slot0 + P.instance;
    switch (P.what) {
      case MCG_PROBE_SYN_WEIGHT: return b[0] + S.h0 * b[R.stride];
      case MCG_PROBE_SYN_H: return b[0];
      case MCG_PROBE_SYN_Z: return b[R.stride];
      case MCG_PROBE_SYN_C: return b[2 * R.stride];
      default: break;
    }
  }
  switch (P.what) {
    case MCG_PROBE_SYN_WEIGHT:
      switch (S.kind) {
        case MCG_SYN_STDP_COND: return D.i_stdp_w[j];
        case MCG_SYN_HOMEO_CURRENT: return D.i_homeo_w[j];
        case MCG_SYN_STC_CHARGE: return D.i_stc_h[j] + S.h0 * D.i_stc_z[j];
        default: return D.i_weight[j];
      }
    case MCG_PROBE_SYN_H: return D.i_stc_h[j];
    case MCG_PROBE_SYN_Z: return D.i_stc_z[j];
    case MCG_PROBE_SYN_C: return D.i_stc_c[j];
    case MCG_PROBE_SYN_KERNEL: return D.i_kernel[j];
    default: return 0.0;
  }
}
