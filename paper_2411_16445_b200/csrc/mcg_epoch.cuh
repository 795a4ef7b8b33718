// mcg_epoch.cuh — shared helpers of the stepping kernels (warp sort, the
// per-cell shared-memory layout) and the fast-forward kernel
// (engine.cpp:947-1034), one warp per cell: the warp stages the cell's
// compartment state in shared memory, relaxes the STC synapses across lanes
// and solves the species systems on lanes 1..S concurrently.
#pragma once
#include "mcg_events.cuh"
#include "mcg_mech.cuh"

// ascending bitonic sort of a[0..n) by one warp, padding to the next power
// of two (<= capacity, itself a power of two) with ~0
__device__ __forceinline__ void mcg_warp_sort(uint64_t* a, int n, int lane) {
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + lane; i < m; i += 32) a[i] = ~0ull;
  __syncwarp();
  for (int k = 2; k <= m; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = lane; i < m; i += 32) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const uint64_t x = a[i], y = a[ixj];
          if (((i & k) == 0) ? (x > y) : (x < y)) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncwarp();
    }
}

struct McgCellMem {
  double *V, *SP, *HM, *HH, *HN;          // mutable compartment state
  double *gsyn, *gsyn_rhs, *rhs_cur;      // per-step accumulators
  double *diag, *r2;                      // solver scratch; r2 has (1 + sp_max) x n
};

__device__ __forceinline__ McgCellMem mcg_cell_mem(const McgDev& D, const McgKind& K, int c,
                                                   double* smem_warp) {
  McgCellMem M;
  const int n = K.n;
  const int64_t co = D.comp_off[c];
  if (smem_warp != nullptr && n <= D.smem_n) {
    const int m = D.smem_n;
    double* p = smem_warp;
    // V | SP | rhs_cur first: a LIF-only launch of the batch kernel keeps just
    // these (McgBatchArgs::comp_stride = (2 + sp_max) m, see setup_batch_kernel)
    M.V = p; p += m;
    M.SP = p; p += int64_t(D.sp_max) * m;
    M.rhs_cur = p; p += m;
    M.HM = p; p += m;
    M.HH = p; p += m;
    M.HN = p; p += m;
    M.gsyn = p; p += m;
    M.gsyn_rhs = p; p += m;
    M.diag = p; p += m;
    M.r2 = p;
  } else {
    M.V = D.v + co;
    M.SP = D.species + D.sp_off[c];
    M.HM = D.hh_m + co;
    M.HH = D.hh_h + co;
    M.HN = D.hh_n + co;
    M.gsyn = D.s_gsyn + co;
    M.gsyn_rhs = D.s_gsyn_rhs + co;
    M.rhs_cur = D.s_rhs_cur + co;
    M.diag = D.s_diag + co;
    M.r2 = D.s_r2 + co * (1 + D.sp_max);
  }
  return M;
}

// copy compartment state global <-> shared (no-op for global-resident cells)
__device__ __forceinline__ void mcg_stage(const McgDev& D, const McgKind& K, int c,
                                          const McgCellMem& M, bool load, int lane) {
  const int n = K.n;
  const int64_t co = D.comp_off[c];
  double* gv = D.v + co;
  if (M.V == gv) return;
  double* gs = D.species + D.sp_off[c];
  const int ns = K.n_species * n;
  for (int i = lane; i < n; i += 32) {
    if (load) M.V[i] = gv[i];
    else gv[i] = M.V[i];
  }
  // species are stored [sp][n] in both places, with stride n in global and
  // stride smem_n in shared memory
  for (int i = lane; i < ns; i += 32) {
    const int sp = i / n, k = i - sp * n;
    if (load) M.SP[sp * n + k] = gs[i];
    else gs[i] = M.SP[sp * n + k];
  }
  if (K.dyn == MCG_DYN_HH) {
    for (int i = lane; i < n; i += 32) {
      if (load) {
        M.HM[i] = D.hh_m[co + i];
        M.HH[i] = D.hh_h[co + i];
        M.HN[i] = D.hh_n[co + i];
      } else {
        D.hh_m[co + i] = M.HM[i];
        D.hh_h[co + i] = M.HH[i];
        D.hh_n[co + i] = M.HN[i];
      }
    }
  }
}

// one species system (engine.cpp:726-750 / 1003-1028); any single lane.
// cap: vol/dt (or vol/dtc); f, d: constant elimination for that cap.
__device__ __forceinline__ bool mcg_species_one(const McgDev& D, const McgKind& K, int sp,
                                                double* conc, double prod, const double* cap,
                                                const double* f, const double* d, double* r2,
                                                double* diag, double* rhs_scr) {
  const int n = K.n;
  const bool is_prp = sp == K.prp_idx;
  const int64_t ka = K.sp_arr + int64_t(sp) * n;
  if (n == 1) {
    const double cap0 = cap[ka];
    const double gse = D.k_sp_gs[ka];
    const double r = cap0 * conc[0] + (is_prp ? prod : 0.0);
    conc[0] = r / (cap0 + gse);
    return true;
  }
  const int pc = (is_prp && prod != 0.0) ? K.prp_comp : -1;
  if (f != nullptr) {
    const double* cp = cap + ka;
    for (int i = 0; i < n; ++i) r2[i] = cp[i] * conc[i] + (i == pc ? prod : 0.0);
    mcg_solve_const(n, D.k_parent + K.arr, D.k_sp_coupling + ka, f + ka, d + ka, conc, r2);
    return true;
  }
  for (int i = 0; i < n; ++i) rhs_scr[i] = (i == pc) ? prod : 0.0;
  return mcg_solve_tree(n, D.k_parent + K.arr, cap + ka, D.k_sp_gs + ka, D.k_sp_coupling + ka,
                        rhs_scr, conc, diag, r2);
}

// The constant-diagonal systems of one step, solved concurrently: lane 0 the
// LIF-cable V system (when v_sys), lane 1 + sp species sp (when the species
// systems are constant and n > 1).  Every active lane runs the same
// instruction stream on its own system, so the sweeps overlap instead of
// serializing as divergent paths.  Returns the species handled here.
__device__ __forceinline__ bool mcg_const_systems(const McgDev& D, const McgKind& K,
                                                  const McgCellMem& M, bool v_sys, bool hc,
                                                  const double* sp_cap, const double* sp_f,
                                                  const double* sp_d, int lane) {
  const int n = K.n;
  const bool sp_sys = n > 1 && K.sp_const && K.n_species > 0 && K.n_species < 32;
  double prod = 0.0;
  if (K.prp_enabled)
    prod = (M.SP[int64_t(K.sps_idx) * n + K.prp_comp] > K.prp_theta_star) ? K.prp_rate : 0.0;
  __syncwarp();  // prod is read before any species system is updated
  const int sp = lane - 1;
  const bool is_v = lane == 0 && v_sys;
  const bool is_sp = sp_sys && sp >= 0 && sp < K.n_species;
  if (is_v || is_sp) {
    const int64_t ka = K.sp_arr + int64_t(is_sp ? sp : 0) * n;
    double* x = is_v ? M.V : M.SP + int64_t(sp) * n;
    const double* cap = is_v ? D.k_cap_dt + K.arr : sp_cap + ka;
    const double* coup = is_v ? D.k_axial + K.arr : D.k_sp_coupling + ka;
    const double* f = is_v ? D.k_vf + K.arr : sp_f + ka;
    const double* d = is_v ? D.k_vd + K.arr : sp_d + ka;
    const double* glr = D.k_g_leak_rhs + K.arr;
    double* r2 = M.r2 + int64_t(is_v ? 0 : 1 + sp) * n;
    const int pc = (!is_v && sp == K.prp_idx && prod != 0.0) ? K.prp_comp : -1;
    for (int i = 0; i < n; ++i) {
      // V:       rhs = g_leak_rhs + 0.0 + (has_current ? rhs_current : 0.0)  (engine.cpp:683)
      // species: rhs = 0.0, or prod at the synthesis compartment           (engine.cpp:746-748)
      const double rhs = is_v ? (glr[i] + 0.0 + (hc ? M.rhs_cur[i] : 0.0))
                              : (i == pc ? prod : 0.0);
      r2[i] = cap[i] * x[i] + rhs;
    }
    mcg_solve_const(n, D.k_parent + K.arr, coup, f, d, x, r2);
  }
  return sp_sys;
}

// species not covered by mcg_const_systems: single-compartment closed forms
// (lanes 1 + sp) or, for singular systems, lane 0 with the full solver
__device__ __forceinline__ bool mcg_species_rest(const McgDev& D, const McgKind& K,
                                                 const McgCellMem& M, const double* cap,
                                                 int lane) {
  const int n = K.n;
  if (K.n_species == 0) return true;
  double prod = 0.0;
  if (K.prp_enabled)
    prod = (M.SP[int64_t(K.sps_idx) * n + K.prp_comp] > K.prp_theta_star) ? K.prp_rate : 0.0;
  __syncwarp();
  bool ok = true;
  if (n == 1) {
    const int sp = lane - 1;
    if (sp >= 0 && sp < K.n_species)
      ok = mcg_species_one(D, K, sp, M.SP + sp, prod, cap, nullptr, nullptr, M.r2, M.diag,
                           M.rhs_cur);
  } else if (lane == 0) {
    for (int sp = 0; sp < K.n_species; ++sp)
      ok &= mcg_species_one(D, K, sp, M.SP + int64_t(sp) * n, prod, cap, nullptr, nullptr,
                            M.r2 + int64_t(1 + sp) * n, M.diag, M.rhs_cur);
  }
  return ok;
}

// ---------------------------------------------------------------------------
// fast-forward (engine.cpp:947-1034): coarse STC relaxation + species solves
// ---------------------------------------------------------------------------

// Register-resident fast path of one cell's coarse steps, taken when the
// cell's STC synapses share one spec, number at most 32 * MCG_FF_K, and the
// SPS and PRP pools are different species (the common case: every network
// builder). Each lane keeps its synapses' h, z and folded |h - h0| in
// registers across all coarse steps; the SPS deltas go through shared memory
// and are folded by one lane per compartment, in instance order (the
// reference's order of the sps[comp] += delta updates for that compartment);
// the species systems are solved one lane each, with the eliminated value of
// a chain child and the parent's solution carried in registers and the
// divisions done by the reciprocal of the constant diagonal (mcg_div).
constexpr int MCG_FF_K = 8;
constexpr int MCG_FF_NMAX = 64;
constexpr int MCG_FF_SPMAX = 2;
// per-warp scratch (doubles): SPS deltas in per-compartment order, the
// constants of the species systems ({cap, f, d, 1/d, coupling} per
// compartment and species), parents and the compartments' delta offsets
constexpr int MCG_FF_SCR = 32 * MCG_FF_K + 5 * MCG_FF_SPMAX * MCG_FF_NMAX +
                           (2 * MCG_FF_NMAX + MCG_FF_NMAX + 1 + 3) / 4 + 1;

struct McgFfScr {
  double* dl;    // [32 K] deltas, grouped by compartment, slot order within
  double* sc;    // [SPMAX][n][5] cap, f, d, rd, coupling
  int16_t* par;  // [n]
  uint16_t* off; // [n + 1]
};

__device__ __forceinline__ McgFfScr mcg_ff_scr(double* p) {
  McgFfScr s;
  s.dl = p;
  s.sc = p + 32 * MCG_FF_K;
  s.par = reinterpret_cast<int16_t*>(s.sc + 5 * MCG_FF_SPMAX * MCG_FF_NMAX);
  s.off = reinterpret_cast<uint16_t*>(s.par + MCG_FF_NMAX);
  return s;
}

// one constant species system on one lane, mcg_solve_const's operation
// order: r2[par[i]] += f[i] * r2[i] for i = n-1 .. 1, then
// x[i] = (r2[i] + coup[i] * x[par[i]]) / d[i]. A child i of i - 1 is the last
// of its parent's children to add (children have larger indices), so its
// term and the parent's solution are carried in registers; only the other
// children go through r2 in shared memory, and r2[i - 1] is loaded one
// iteration ahead (a stored parent is never i - 1).
__device__ __forceinline__ void mcg_ff_solve(int n, const int16_t* __restrict__ par,
                                             const double* __restrict__ sc,
                                             double* __restrict__ x, double* __restrict__ r2) {
  bool cn = false;
  double fc = 0.0, rc = 0.0;
  double rn = r2[n - 1];
  for (int i = n - 1; i >= 1; --i) {
    double ri = rn;
    rn = r2[i - 1];
    const int p = par[i];
    const double fi = sc[5 * i + 1];
    if (cn) ri = ri + fc * rc;
    r2[i] = ri;
    if (p == i - 1) {
      cn = true;
      fc = fi;
      rc = ri;
    } else {
      r2[p] = r2[p] + fi * ri;
      cn = false;
    }
  }
  double r0 = rn;
  if (cn) r0 = r0 + fc * rc;
  double vp = mcg_div(r0, sc[2], sc[3]);
  x[0] = vp;
  for (int i = 1; i < n; ++i) {
    const int p = par[i];
    const double* e = sc + 5 * i;
    const double vpar = (p == i - 1) ? vp : x[p];
    vp = mcg_div(r2[i] + e[4] * vpar, e[2], e[3]);
    x[i] = vp;
  }
}

// The species systems of a cell of at most 32 compartments, one compartment
// per lane with its constants in registers, solved level by level: the
// elimination walks the tree's depths from the leaves up (a parent adds its
// children's f * r2 in decreasing child index, mcg_solve_const's order, in the
// round of their depth), the substitution from the root down. Every species
// rides on the same shuffles.
constexpr int MCG_FF_MAXCH = 4;

struct McgFfLanes {
  int depth, par, nch, ch[MCG_FF_MAXCH];
  uint32_t more[MCG_FF_MAXCH - 1];  // bit l of more[k-1]: depth l has a parent with > k children
  double cap[MCG_FF_SPMAX], f[MCG_FF_SPMAX], d[MCG_FF_SPMAX], rd[MCG_FF_SPMAX],
      coup[MCG_FF_SPMAX];
};

// false when some compartment has more than MCG_FF_MAXCH children
__device__ __forceinline__ bool mcg_ff_lanes_init(const McgDev& D, const McgKind& K,
                                                  const double* sp_cap_ff, const double* sp_f_ff,
                                                  const double* sp_d_ff, const double* sp_r_ff,
                                                  int lane, McgFfLanes& L, int& max_depth) {
  const int n = K.n;
  const int32_t* par = D.k_parent + K.arr;
  L.depth = 0;
  L.par = 0;
  L.nch = 0;
#pragma unroll
  for (int k = 0; k < MCG_FF_MAXCH; ++k) L.ch[k] = lane;
  if (lane < n) {
    L.par = lane > 0 ? par[lane] : 0;
    for (int p = lane; p > 0; p = par[p]) ++L.depth;
    // children in decreasing index: mcg_solve_const's order of their adds
    for (int j = n - 1; j > lane; --j)
      if (par[j] == lane) {
#pragma unroll
        for (int k = 0; k < MCG_FF_MAXCH; ++k)
          if (k == L.nch) L.ch[k] = j;
        ++L.nch;
      }
  }
  const bool ok = L.nch <= MCG_FF_MAXCH;
#pragma unroll
  for (int sp = 0; sp < MCG_FF_SPMAX; ++sp) {
    L.cap[sp] = L.f[sp] = L.coup[sp] = 0.0;
    L.d[sp] = L.rd[sp] = 1.0;
    if (lane < n && sp < K.n_species) {
      const int64_t ka = K.sp_arr + int64_t(sp) * n + lane;
      L.cap[sp] = sp_cap_ff[ka];
      L.f[sp] = sp_f_ff[ka];
      L.d[sp] = sp_d_ff[ka];
      L.rd[sp] = sp_r_ff[ka];
      L.coup[sp] = D.k_sp_coupling[ka];
    }
  }
  max_depth = __reduce_max_sync(MCG_FULL, L.depth);
#pragma unroll
  for (int k = 1; k < MCG_FF_MAXCH; ++k) {
    L.more[k - 1] = 0;
    for (int l = 1; l <= max_depth; ++l)
      if (__any_sync(MCG_FULL, lane < n && L.depth == l - 1 && L.nch > k))
        L.more[k - 1] |= 1u << l;
  }
  return __all_sync(MCG_FULL, ok);
}

// x / d by the reciprocal y (mcg_div) without its branch: bad marks the
// operands outside the proven range, which the caller redoes with IEEE division
__device__ __forceinline__ double mcg_div_nb(double x, double d, double y, bool& bad) {
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(-q, d, x);
  const double res = __fma_rn(r, y, q);
  const double ax = fabs(x);
  bad = y == 0.0 || ax > 0x1p700 || (ax < 0x1p-700 && ax != 0.0);
  return ax == 0.0 ? q : res;
}

__device__ __forceinline__ void mcg_ff_solve_lanes(const McgKind& K, const McgFfLanes& L,
                                                   int max_depth, double prod, double* SP,
                                                   int lane) {
  const int n = K.n;
  const int pc = prod != 0.0 ? K.prp_comp : -1;
  double x[MCG_FF_SPMAX], r[MCG_FF_SPMAX];
#pragma unroll
  for (int sp = 0; sp < MCG_FF_SPMAX; ++sp) {
    x[sp] = (lane < n && sp < K.n_species) ? SP[sp * n + lane] : 0.0;
    // r2 = cap * x + rhs (engine.cpp:1019-1025)
    r[sp] = L.cap[sp] * x[sp] + ((sp == K.prp_idx && lane == pc) ? prod : 0.0);
  }
  // elimination, leaves up: at depth l the parents (depth l - 1) pull f * r2
  // of their children
  for (int l = max_depth; l >= 1; --l) {
    double pr[MCG_FF_SPMAX];
#pragma unroll
    for (int sp = 0; sp < MCG_FF_SPMAX; ++sp) pr[sp] = L.f[sp] * r[sp];
    const bool gather = L.depth == l - 1;
    // pull k happens only where a parent has more than k children (more[k-1]),
    // which implies every earlier pull: one branch per level in the common case
#pragma unroll
    for (int k = 0; k < MCG_FF_MAXCH; ++k) {
      if (k > 0 && !((L.more[k > 0 ? k - 1 : 0] >> l) & 1u)) break;
      const bool take = gather && k < L.nch;
#pragma unroll
      for (int sp = 0; sp < MCG_FF_SPMAX; ++sp) {
        const double v = __shfl_sync(MCG_FULL, pr[sp], L.ch[k]);
        const double t = r[sp] + v;
        r[sp] = take ? t : r[sp];
      }
    }
  }
  // substitution, root down; operands outside the reciprocal division's proven
  // range (never seen in practice) send the whole sweep through mcg_div again
  bool bad = false;
#pragma unroll
  for (int sp = 0; sp < MCG_FF_SPMAX; ++sp) {
    bool b;
    const double q = mcg_div_nb(r[sp], L.d[sp], L.rd[sp], b);
    if (lane == 0) x[sp] = q;
    bad |= lane == 0 && b;
  }
  for (int l = 1; l <= max_depth; ++l) {
    const bool sel = L.depth == l;
#pragma unroll
    for (int sp = 0; sp < MCG_FF_SPMAX; ++sp) {
      const double xp = __shfl_sync(MCG_FULL, x[sp], L.par);
      bool b;
      const double q = mcg_div_nb(r[sp] + L.coup[sp] * xp, L.d[sp], L.rd[sp], b);
      x[sp] = sel ? q : x[sp];
      bad |= sel && b;
    }
  }
  if (__any_sync(MCG_FULL, bad)) {
#pragma unroll
    for (int sp = 0; sp < MCG_FF_SPMAX; ++sp)
      if (lane == 0) x[sp] = mcg_div(r[sp], L.d[sp], L.rd[sp]);
    for (int l = 1; l <= max_depth; ++l) {
#pragma unroll
      for (int sp = 0; sp < MCG_FF_SPMAX; ++sp) {
        const double xp = __shfl_sync(MCG_FULL, x[sp], L.par);
        if (L.depth == l) x[sp] = mcg_div(r[sp] + L.coup[sp] * xp, L.d[sp], L.rd[sp]);
      }
    }
  }
#pragma unroll
  for (int sp = 0; sp < MCG_FF_SPMAX; ++sp)
    if (lane < n && sp < K.n_species) SP[sp * n + lane] = x[sp];
}

// the cell's STC instance of concatenated slot s (group order, then instance)
__device__ __forceinline__ int64_t mcg_ff_inst(const McgDev& D, const McgKind& K, int64_t cg0,
                                               int s) {
  for (int gi = 0; gi < K.n_groups; ++gi) {
    const McgCellGroup G = D.cgs[cg0 + gi];
    if (D.specs[G.spec].kind != MCG_SYN_STC_CHARGE) continue;
    if (s < G.size) return G.inst + s;
    s -= G.size;
  }
  return -1;
}

__device__ __forceinline__ bool mcg_ff_cell_fast(const McgDev& D, const McgKind& K, int c,
                                              int64_t cg0, const McgCellMem& M, int spec,
                                              int nsyn, double fh, const double* sp_cap_ff,
                                              const double* sp_f_ff, const double* sp_d_ff,
                                              const double* sp_r_ff, double dtc,
                                              int64_t n_coarse, int lane, McgFfScr X) {
  const int n = K.n;
  const double* prp_base = (K.prp_idx >= 0) ? M.SP + int64_t(K.prp_idx) * n : nullptr;
  double* sps_base = (K.sps_idx >= 0) ? M.SP + int64_t(K.sps_idx) * n : nullptr;
  double h0 = 0.0, theta = 0.0, f_int = 0.0, tau_z = 1.0, rtz = 1.0;
  if (spec >= 0) {
    const McgSpec& S = D.specs[spec];
    h0 = S.h0;
    theta = S.theta_tag;
    f_int = S.f_int;
    tau_z = S.tau_z;
    rtz = S.r_tau_z;
  }
  // per-compartment delta offsets (a counting sort by lane 0)
  if (lane == 0) {
    for (int i = 0; i <= n; ++i) X.off[i] = 0;
    for (int s = 0; s < nsyn; ++s) X.off[D.i_comp[mcg_ff_inst(D, K, cg0, s)] + 1]++;
    for (int i = 0; i < n; ++i) X.off[i + 1] += X.off[i];
  }
  const bool sp_sys = n > 1 && K.sp_const && K.n_species > 0 && K.n_species < 32;
  const bool sp_fast = sp_sys && K.n_species <= MCG_FF_SPMAX;
  McgFfLanes LN;
  int max_depth = 0;
  const bool sp_lanes = sp_fast && n <= 32 &&
                        mcg_ff_lanes_init(D, K, sp_cap_ff, sp_f_ff, sp_d_ff, sp_r_ff, lane, LN,
                                          max_depth);
  if (sp_fast && !sp_lanes) {
    for (int e = lane; e < K.n_species * n; e += 32) {
      const int64_t ka = K.sp_arr + e;
      double* o = X.sc + 5 * e;
      o[0] = sp_cap_ff[ka];
      o[1] = sp_f_ff[ka];
      o[2] = sp_d_ff[ka];
      o[3] = sp_r_ff[ka];
      o[4] = D.k_sp_coupling[ka];
    }
    for (int i = lane; i < n; i += 32) X.par[i] = static_cast<int16_t>(D.k_parent[K.arr + i]);
  }
  __syncwarp();
  // per slot: h, z, the folded |h - h0| and (compartment | delta position << 8)
  double h[MCG_FF_K], z[MCG_FF_K], a[MCG_FF_K];
  int cp[MCG_FF_K];
#pragma unroll
  for (int k = 0; k < MCG_FF_K; ++k) {
    const int s = lane + 32 * k;
    h[k] = z[k] = a[k] = 0.0;
    cp[k] = 0;
    if (s < nsyn) {
      const int64_t j = mcg_ff_inst(D, K, cg0, s);
      h[k] = D.i_stc_h[j];
      z[k] = D.i_stc_z[j];
      a[k] = D.i_sps_abs[j];
      cp[k] = D.i_comp[j];
    }
  }
  const double* vol_k = D.k_volume + K.arr;
  const double* rvol_k = D.k_rvol + K.arr;
  // slot order within a compartment: slots of earlier k, then lower lanes
#pragma unroll
  for (int k = 0; k < MCG_FF_K; ++k) {
    const int s = lane + 32 * k;
    if (32 * k < nsyn) {
      const unsigned grp = __match_any_sync(MCG_FULL, s < nsyn ? cp[k] : -1);
      const int cmp = cp[k];
      if (s < nsyn) cp[k] = cmp | ((X.off[cmp] + __popc(grp & mcg_lanemask_lt())) << 8);
      __syncwarp();
      // advance each compartment's offset by its slots in this round
      if (s < nsyn && (grp & mcg_lanemask_lt()) == 0) X.off[cmp] += __popc(grp);
      __syncwarp();
    }
  }
  // restore the offsets (they now hold the compartments' ends)
  if (lane == 0) {
    for (int i = n; i > 0; --i) X.off[i] = X.off[i - 1];
    X.off[0] = 0;
  }
  const bool has_probe = D.probe_off[c] < D.probe_off[c + 1];
  bool ok = true;
  __syncwarp();
  for (int64_t q = 0; q < n_coarse; ++q) {
#pragma unroll
    for (int k = 0; k < MCG_FF_K; ++k) {
      const int s = lane + 32 * k;
      if (s < nsyn) {
        h[k] = h0 + (h[k] - h0) * fh;
        const double na = fabs(h[k] - h0);
        // an unchanged instance contributes -0.0, which leaves any sum as it is
        double dl = -0.0;
        if (na != a[k]) {
          dl = mcg_div(na - a[k], vol_k[cp[k] & 255], rvol_k[cp[k] & 255]);
          a[k] = na;
        }
        X.dl[cp[k] >> 8] = dl;
        if (prp_base) {
          const double prp = prp_base[cp[k] & 255];
          if (!(prp <= 0.0)) {
            double dd = 0.0;
            if (h[k] - h0 > theta) dd += (1.0 - z[k]);
            if (h0 - h[k] > theta) dd -= (z[k] + 0.5);
            z[k] += mcg_div(prp * f_int * dd * dtc, tau_z, rtz);
          }
        }
      }
    }
    __syncwarp();
    if (sps_base != nullptr && nsyn > 0) {
      // the compartment's sps += delta in slot order (engine.cpp:986-1000)
      for (int cc = lane; cc < n; cc += 32) {
        const int t0 = X.off[cc], t1 = X.off[cc + 1];
        if (t0 == t1) continue;
        double acc = sps_base[cc];
        int t = t0;
        if (t + 8 <= t1) {
          // the next eight deltas load while the current eight are added
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = X.dl[t + u];
          for (t += 8; t + 8 <= t1; t += 8) {
            double w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) w[u] = X.dl[t + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = w[u];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) acc += v[u];
        }
        for (; t < t1; ++t) acc += X.dl[t];
        sps_base[cc] = acc;
      }
      __syncwarp();
    }
    if (sp_lanes) {
      double prod = 0.0;
      if (K.prp_enabled)
        prod = (M.SP[int64_t(K.sps_idx) * n + K.prp_comp] > K.prp_theta_star) ? K.prp_rate : 0.0;
      mcg_ff_solve_lanes(K, LN, max_depth, prod, M.SP, lane);
    } else if (sp_fast) {
      double prod = 0.0;
      if (K.prp_enabled)
        prod = (M.SP[int64_t(K.sps_idx) * n + K.prp_comp] > K.prp_theta_star) ? K.prp_rate : 0.0;
      __syncwarp();
      // r2 = cap * x + rhs for every species, across lanes (engine.cpp:1019-1025)
      for (int e = lane; e < K.n_species * n; e += 32) {
        const int sp = e / n, i = e - sp * n;
        const int pc = (sp == K.prp_idx && prod != 0.0) ? K.prp_comp : -1;
        M.r2[int64_t(1 + sp) * n + i] = X.sc[5 * e] * M.SP[e] + (i == pc ? prod : 0.0);
      }
      __syncwarp();
      if (lane < K.n_species)
        mcg_ff_solve(n, X.par, X.sc + 5 * lane * n, M.SP + int64_t(lane) * n,
                     M.r2 + int64_t(1 + lane) * n);
    } else if (!mcg_const_systems(D, K, M, false, false, sp_cap_ff, sp_f_ff, sp_d_ff, lane)) {
      ok &= mcg_species_rest(D, K, M, sp_cap_ff, lane);
    }
    __syncwarp();
    if (has_probe) {
      // forced probe sample at step_ - 1 after the coarse step (engine.cpp:1031-1032)
#pragma unroll
      for (int k = 0; k < MCG_FF_K; ++k) {
        const int s = lane + 32 * k;
        if (s < nsyn) {
          const int64_t j = mcg_ff_inst(D, K, cg0, s);
          D.i_stc_h[j] = h[k];
          D.i_stc_z[j] = z[k];
        }
      }
      __syncwarp();
      if (lane == 0) {
        for (int qq = D.probe_off[c]; qq < D.probe_off[c + 1]; ++qq) {
          const int p = D.probe_idx[qq];
          D.trace_buf[D.trace_base[p] + q] = mcg_probe_value(D, K, c, D.probes[p], M.V, M.SP);
        }
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int k = 0; k < MCG_FF_K; ++k) {
    const int s = lane + 32 * k;
    if (s < nsyn) {
      const int64_t j = mcg_ff_inst(D, K, cg0, s);
      D.i_stc_h[j] = h[k];
      D.i_stc_z[j] = z[k];
      D.i_sps_abs[j] = a[k];
    }
  }
  return ok;
}

// the cells the register-resident path takes (mcg_ff_cell_fast): one STC
// spec, at most 32 * MCG_FF_K instances, SPS and PRP distinct species
__device__ __forceinline__ bool mcg_ff_fast_of(const McgDev& D, const McgKind& K, int64_t cg0,
                                               int& spec, int& nsyn) {
  spec = -1;
  nsyn = 0;
  bool uni = true;
  for (int gi = 0; gi < K.n_groups; ++gi) {
    const McgCellGroup G = D.cgs[cg0 + gi];
    if (D.specs[G.spec].kind != MCG_SYN_STC_CHARGE) continue;
    if (spec >= 0 && G.spec != spec) uni = false;
    spec = G.spec;
    nsyn += G.size;
  }
  const bool stc_seq = K.sps_idx >= 0 && K.sps_idx == K.prp_idx;
  return !stc_seq && uni && nsyn <= 32 * MCG_FF_K && K.n <= MCG_FF_NMAX;
}

// three 4-warp CTAs per SM (<= 168 registers): the 1,600 cells of config 3
// run in one wave
constexpr int MCG_FF_BLOCK = 128;
__global__ void __launch_bounds__(MCG_FF_BLOCK, 3) k_ff_fast(McgDev D, const double* fh_spec,
                                                 const double* sp_cap_ff, const double* sp_f_ff,
                                                 const double* sp_d_ff, const double* sp_r_ff,
                                                 double dtc, int64_t n_coarse) {
  extern __shared__ double mcg_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= D.n_cells) return;
  const McgKind& K = D.kinds[D.cell_kind[c]];
  const int64_t cg0 = D.cg_off[c];
  int spec, nsyn;
  if (!mcg_ff_fast_of(D, K, cg0, spec, nsyn)) return;
  // nothing in the cell changes over coarse steps: no STC synapse, species or probe
  if (nsyn == 0 && K.n_species == 0 && D.probe_off[c] == D.probe_off[c + 1]) return;
  const McgCellMem M = mcg_cell_mem(D, K, c, D.smem_stride ? mcg_smem + wib * D.smem_stride : nullptr);
  mcg_stage(D, K, c, M, true, lane);
  __syncwarp();
  double* scr = mcg_smem + (blockDim.x >> 5) * D.smem_stride + wib * MCG_FF_SCR;
  const bool ok = mcg_ff_cell_fast(D, K, c, cg0, M, spec, nsyn,
                                   spec >= 0 ? fh_spec[spec] : 0.0, sp_cap_ff, sp_f_ff, sp_d_ff,
                                   sp_r_ff, dtc, n_coarse, lane, mcg_ff_scr(scr));
  __syncwarp();
  mcg_stage(D, K, c, M, false, lane);
  const unsigned okm = __ballot_sync(MCG_FULL, ok);
  if (lane == 0 && okm != MCG_FULL) atomicOr(D.err, MCG_ERR_FLAG_SINGULAR);
}

// the other cells, with the general loop
__global__ void __launch_bounds__(128) k_ff(McgDev D, const double* fh_spec, const double* sp_cap_ff,
                                            const double* sp_f_ff, const double* sp_d_ff,
                                            const double* sp_r_ff, double dtc,
                                            int64_t n_coarse) {
  extern __shared__ double mcg_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= D.n_cells) return;
  const McgKind& K = D.kinds[D.cell_kind[c]];
  const int n = K.n;
  const int64_t cg0 = D.cg_off[c];
  {
    int spec, nsyn;
    if (mcg_ff_fast_of(D, K, cg0, spec, nsyn)) return;  // k_ff_fast's cell
  }
  const McgCellMem M = mcg_cell_mem(D, K, c, D.smem_stride ? mcg_smem + wib * D.smem_stride : nullptr);
  mcg_stage(D, K, c, M, true, lane);
  const double* prp_base = (K.prp_idx >= 0) ? M.SP + int64_t(K.prp_idx) * n : nullptr;
  double* sps_base = (K.sps_idx >= 0) ? M.SP + int64_t(K.sps_idx) * n : nullptr;
  const double* vol_k = D.k_volume + K.arr;
  const bool stc_seq = sps_base != nullptr && (const double*)sps_base == prp_base;
  bool ok = true;
  __syncwarp();
  for (int64_t q = 0; q < n_coarse; ++q) {
    for (int gi = 0; gi < K.n_groups; ++gi) {
      const McgCellGroup G = D.cgs[cg0 + gi];
      const McgSpec& S = D.specs[G.spec];
      if (S.kind != MCG_SYN_STC_CHARGE) continue;
      const double fh = fh_spec[G.spec];
      int acc_comp = -1;
      double acc = 0.0;
      const int step = stc_seq ? (G.size > 0 ? G.size : 1) : 32;
      for (int i0 = 0; i0 < G.size; i0 += step) {
        const int i = stc_seq ? i0 : i0 + lane;
        bool ch = false;
        double delta = 0.0;
        int comp = 0;
        if (i < G.size && (!stc_seq || lane == 0)) {
          const int iend = stc_seq ? G.size : i + 1;
          for (int ii = i; ii < iend; ++ii) {
            const int64_t j = G.inst + ii;
            const double h = S.h0 + (D.i_stc_h[j] - S.h0) * fh;
            double z = D.i_stc_z[j];
            const double na = fabs(h - S.h0);
            comp = D.i_comp[j];
            if (na != D.i_sps_abs[j]) {
              delta = (na - D.i_sps_abs[j]) / vol_k[comp];
              D.i_sps_abs[j] = na;
              ch = true;
              if (stc_seq && sps_base) sps_base[comp] += delta;
            }
            if (prp_base) {
              const double prp = prp_base[comp];
              if (!(prp <= 0.0)) {
                double dd = 0.0;
                if (h - S.h0 > S.theta_tag) dd += (1.0 - z);
                if (S.h0 - h > S.theta_tag) dd -= (z + 0.5);
                z += prp * S.f_int * dd * dtc / S.tau_z;
              }
            }
            D.i_stc_h[j] = h;
            D.i_stc_z[j] = z;
          }
        }
        if (!stc_seq) {
          unsigned mm = __ballot_sync(MCG_FULL, ch);
          if (sps_base) {
            while (mm) {
              const int l = __ffs(mm) - 1;
              mm &= mm - 1;
              const double dl = __shfl_sync(MCG_FULL, delta, l);
              const int cl = __shfl_sync(MCG_FULL, comp, l);
              if (lane == 0) {
                if (cl != acc_comp) {
                  if (acc_comp >= 0) sps_base[acc_comp] = acc;
                  acc_comp = cl;
                  acc = sps_base[cl];
                }
                acc += dl;
              }
            }
          }
        }
      }
      if (lane == 0 && acc_comp >= 0) sps_base[acc_comp] = acc;
      __syncwarp();
    }
    if (!mcg_const_systems(D, K, M, false, false, sp_cap_ff, sp_f_ff, sp_d_ff, lane))
      ok &= mcg_species_rest(D, K, M, sp_cap_ff, lane);
    __syncwarp();
    // forced probe sample at step_ - 1 after the coarse step (engine.cpp:1031-1032)
    if (lane == 0) {
      for (int qq = D.probe_off[c]; qq < D.probe_off[c + 1]; ++qq) {
        const int p = D.probe_idx[qq];
        D.trace_buf[D.trace_base[p] + q] = mcg_probe_value(D, K, c, D.probes[p], M.V, M.SP);
      }
    }
    __syncwarp();
  }
  mcg_stage(D, K, c, M, false, lane);
  const unsigned okm = __ballot_sync(MCG_FULL, ok);
  if (lane == 0 && okm != MCG_FULL) atomicOr(D.err, MCG_ERR_FLAG_SINGULAR);
}
