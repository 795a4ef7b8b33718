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
__global__ void __launch_bounds__(128) k_ff(McgDev D, const double* fh_spec, const double* sp_cap_ff,
                                            const double* sp_f_ff, const double* sp_d_ff,
                                            double dtc, int64_t n_coarse) {
  extern __shared__ double mcg_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= D.n_cells) return;
  const McgKind& K = D.kinds[D.cell_kind[c]];
  const int n = K.n;
  const int64_t cg0 = D.cg_off[c];
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
