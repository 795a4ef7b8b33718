// mcg_epoch.cuh — the epoch kernel (step_cell for every step of a min-delay
// epoch, engine.cpp:541-783) and the fast-forward kernel (engine.cpp:947-1034).
//
// One warp owns one cell.  At epoch start the warp stages the cell's
// compartment state (V, species, HH gates) and all per-compartment scratch in
// shared memory; every sequential sweep then runs on shared memory instead of
// chasing dependent global loads.  Independent sequential work runs on
// different lanes at once: lane 0 integrates V, lanes 1..S the species
// systems; HH gating is parallel over compartments; synapse mechanisms are
// parallel over instances with the reference's folds kept in order.
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
    M.V = p; p += m;
    M.SP = p; p += int64_t(D.sp_max) * m;
    M.HM = p; p += m;
    M.HH = p; p += m;
    M.HN = p; p += m;
    M.gsyn = p; p += m;
    M.gsyn_rhs = p; p += m;
    M.rhs_cur = p; p += m;
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

__global__ void __launch_bounds__(128) k_epoch(McgDev D, int32_t j) {
  extern __shared__ double mcg_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= D.n_cells || *D.abort) return;
  int64_t s0, s1;
  if (!mcg_epoch_bounds(D.ctl, j, s0, s1)) return;
  const McgKind& K = D.kinds[D.cell_kind[c]];
  const int n = K.n;
  const int64_t cg0 = D.cg_off[c];
  const uint32_t gid = D.gid0 + uint32_t(c);
  const bool is_lif = K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT;
  const McgCellMem M = mcg_cell_mem(D, K, c, D.smem_stride ? mcg_smem + wib * D.smem_stride : nullptr);
  mcg_stage(D, K, c, M, true, lane);
  double* V = M.V;
  const int32_t* par = D.k_parent + K.arr;
  const uint64_t rank_mask = (1ull << D.rank_bits) - 1;
  const double* prp_base = (K.prp_idx >= 0) ? M.SP + int64_t(K.prp_idx) * n : nullptr;
  double* sps_base = (K.sps_idx >= 0) ? M.SP + int64_t(K.sps_idx) * n : nullptr;
  const double* vol_k = D.k_volume + K.arr;
  const bool stc_seq = sps_base != nullptr && (const double*)sps_base == prp_base;
  const bool noise = is_lif && K.has_bg && K.sig_bg != 0.0;

  // ---- inbox: sort this epoch's incoming keys and merge them into the
  // pending list (the reference's per-epoch inbox sort, engine.cpp:917-925)
  int sel = D.pend_sel[c];
  const uint64_t* pend = D.pend + (int64_t(c) * 2 + sel) * D.pend_cap;
  int cur = D.pend_off[c], end = D.pend_n[c];
  {
    const int nin = D.inc_n[c];
    if (nin > 0) {
      uint64_t* in = D.inc + int64_t(c) * D.inc_cap;
      if (nin > 1) mcg_warp_sort(in, nin, lane);
      __syncwarp();
      uint64_t* out = D.pend + (int64_t(c) * 2 + (1 - sel)) * D.pend_cap;
      if (lane == 0) {
        int a = cur, b = 0, o = 0;
        while (a < end && b < nin) out[o++] = (pend[a] <= in[b]) ? pend[a++] : in[b++];
        while (a < end) out[o++] = pend[a++];
        while (b < nin) out[o++] = in[b++];
      }
      end = (end - cur) + nin;
      cur = 0;
      sel = 1 - sel;
      pend = out;
      __syncwarp();
    }
  }
  int64_t refr = D.refr_until[c];
  double det_prev = D.det_prev[c];
  int armed = D.armed[c];
  int nsp = 0;
  unsigned long long ndel = 0;
  bool ok = true;
  double nb = 0.0;  // this lane's background-noise draw for step (s0 + 32k + lane)
  __syncwarp();

  for (int64_t s = s0; s < s1; ++s) {
    const bool refractory = is_lif && s < refr;
    const int64_t so = s - s0;
    if (noise && (so & 31) == 0) {
      const int64_t sl = s + lane;
      if (sl < s1) {
        const mcg_key key = mcg_make_key(D.seed, gid, 1, 0);
        nb = mcg_normal_for(&key, static_cast<uint64_t>(sl));
      }
    }
    const double nrm_bg = noise ? __shfl_sync(MCG_FULL, nb, int(so & 31)) : 0.0;

    // ---- 1. deliver due events: inbox, then internal (engine.cpp:549-560)
    if (lane == 0) {
      while (cur < end) {
        const uint64_t key = pend[cur];
        const int64_t st = int64_t(key >> D.rank_bits);
        if (st > s) break;
        const int64_t r = int64_t(key & rank_mask);
        mcg_apply_event(D, K, c, cg0, V, D.e_group[r], D.e_inst[r], D.e_weight[r], 0, refractory,
                        s);
        ++cur;
        ++ndel;
      }
      if (K.n_stc_groups > 0) {
        for (;;) {
          int best = -1;
          uint64_t bseq = ~0ull;
          for (int gi = 0; gi < K.n_groups; ++gi) {
            const McgCellGroup& G = D.cgs[cg0 + gi];
            if (G.fifo < 0) continue;
            const McgFifo& F = D.fifos[G.fifo];
            if (F.head < F.tail) {
              const int64_t slot = F.base + (F.head % F.cap);
              if (D.fifo_step[slot] <= s) {
                const uint64_t seq = D.fifo_si[slot] >> 32;
                if (seq < bseq) {
                  bseq = seq;
                  best = gi;
                }
              }
            }
          }
          if (best < 0) break;
          McgFifo& F = D.fifos[D.cgs[cg0 + best].fifo];
          const uint64_t si = D.fifo_si[F.base + (F.head % F.cap)];
          ++F.head;
          mcg_apply_event(D, K, c, cg0, V, best, uint32_t(si & 0xffffffffu), 0.0, 1, refractory,
                          s);
        }
      }
    }
    // ---- 2. mechanisms and current accumulation (engine.cpp:562-664)
    const int nr = n > 1 ? n : 1;
    for (int i = lane; i < nr; i += 32) M.rhs_cur[i] = 0.0;
    bool has_gsyn = false, has_current = false;
    __syncwarp();
    for (int gi = 0; gi < K.n_groups; ++gi) {
      McgCellGroup* G = &D.cgs[cg0 + gi];
      const McgSpec& S = D.specs[G->spec];
      const int kind = S.kind;
      if (kind == MCG_SYN_STATIC_COND || kind == MCG_SYN_STDP_COND) {
        if (G->active_n == 0) continue;
        if (!has_gsyn) {
          for (int i = lane; i < n; i += 32) {
            M.gsyn[i] = 0.0;
            M.gsyn_rhs[i] = 0.0;
          }
          has_gsyn = true;
          __syncwarp();
        }
        mcg_decay_active(D, G, S.f_decay, true, M.gsyn, M.gsyn_rhs, S.e_rev, lane);
      } else if (kind == MCG_SYN_STATIC_CURRENT || kind == MCG_SYN_HOMEO_CURRENT) {
        if (G->active_n == 0) continue;
        if (mcg_decay_active(D, G, S.f_decay, false, M.rhs_cur, nullptr, 0.0, lane))
          has_current = true;
      } else if (kind == MCG_SYN_STC_CHARGE) {
        const int size = G->size;
        const int64_t ib = G->inst;
        if (stc_seq) {
          if (lane == 0)
            for (int i = 0; i < size; ++i) {
              const McgStcOut o = mcg_stc_instance(D, S, ib + i, gid, gi, i, s, prp_base, vol_k);
              if (o.changed) sps_base[o.comp] += o.delta;
            }
        } else {
          // the SPS fold (engine.cpp:634-641) in instance order, carried in a
          // register while consecutive instances hit the same compartment
          int acc_comp = -1;
          double acc = 0.0;
          for (int i0 = 0; i0 < size; i0 += 32) {
            const int i = i0 + lane;
            McgStcOut o{0.0, 0, false};
            if (i < size) o = mcg_stc_instance(D, S, ib + i, gid, gi, i, s, prp_base, vol_k);
            const double delta = o.delta;
            const int comp = o.comp;
            unsigned mm = __ballot_sync(MCG_FULL, o.changed);
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
          if (lane == 0 && acc_comp >= 0) sps_base[acc_comp] = acc;
        }
        __syncwarp();
      }
    }
    // background current (engine.cpp:652-664): warp-uniform decision
    {
      const double ts = double(s) * D.dt;
      const bool bg_gated = K.bg_t1 > K.bg_t0 && ts >= K.bg_t0 && ts < K.bg_t1;
      if (is_lif && K.has_bg && !bg_gated) {
        if (lane == 0) {
          double ib = K.i_bg;
          if (K.sig_bg != 0.0) ib += K.sig_bg * nrm_bg;
          M.rhs_cur[K.noise_comp] += ib;
        }
        has_current = true;
      }
    }
    __syncwarp();

    // ---- 3. continuous state update (engine.cpp:666-751)
    if (K.dyn == MCG_DYN_HH) {
      // gating at the pre-step voltage, parallel over compartments
      const double* gl = D.k_g_leak + K.arr;
      const double* glr = D.k_g_leak_rhs + K.arr;
      const double* gna_k = D.k_g_na + K.arr;
      const double* gk_k = D.k_g_k + K.arr;
      const double dt = D.dt;
      for (int i = lane; i < n; i += 32) {
        const double v = V[i];
        double gsum = gl[i];
        double grhs = glr[i];
        if (gna_k[i] != 0.0) {
          const double am = mcg_hh_am(v), bm = mcg_hh_bm(v);
          const double ah = mcg_hh_ah(v), bh = mcg_hh_bh(v);
          const double an = mcg_hh_an(v), bn = mcg_hh_bn(v);
          double m = M.HM[i], h = M.HH[i], nn = M.HN[i];
          m += (am / (am + bm) - m) * (1.0 - mcg_exp(-dt * (am + bm)));
          h += (ah / (ah + bh) - h) * (1.0 - mcg_exp(-dt * (ah + bh)));
          nn += (an / (an + bn) - nn) * (1.0 - mcg_exp(-dt * (an + bn)));
          M.HM[i] = m;
          M.HH[i] = h;
          M.HN[i] = nn;
          const double gna = gna_k[i] * m * m * m * h;
          const double gk = gk_k[i] * nn * nn * nn * nn;
          gsum += gna + gk;
          grhs += gna * K.e_na + gk * K.e_k;
        }
        M.gsyn[i] = gsum + (has_gsyn ? M.gsyn[i] : 0.0);
        M.gsyn_rhs[i] = grhs + (has_gsyn ? M.gsyn_rhs[i] : 0.0) + (has_current ? M.rhs_cur[i] : 0.0);
      }
      __syncwarp();
      if (lane == 0)
        ok &= mcg_solve_tree(n, par, D.k_cap_dt + K.arr, M.gsyn, D.k_axial + K.arr, M.gsyn_rhs, V,
                             M.diag, M.r2);
    } else if (lane == 0) {
      if (K.dyn == MCG_DYN_LIF_EXACT) {
        if (!refractory) {
          const double vinf = K.v_rev + K.r_mem * M.rhs_cur[0];
          V[0] = vinf + (V[0] - vinf) * K.lif_exact_f;
        }
      } else if (K.dyn == MCG_DYN_LIF && !refractory && (has_gsyn || !K.v_const)) {
        const double* gl = D.k_g_leak + K.arr;
        const double* glr = D.k_g_leak_rhs + K.arr;
        for (int i = 0; i < n; ++i) {
          const double gs = gl[i] + (has_gsyn ? M.gsyn[i] : 0.0);
          const double rr = glr[i] + (has_gsyn ? M.gsyn_rhs[i] : 0.0) +
                            (has_current ? M.rhs_cur[i] : 0.0);
          M.gsyn[i] = gs;
          M.gsyn_rhs[i] = rr;
        }
        ok &= mcg_solve_tree(n, par, D.k_cap_dt + K.arr, M.gsyn, D.k_axial + K.arr, M.gsyn_rhs,
                             V, M.diag, M.r2);
      }
    }
    // constant systems in parallel: V on lane 0 (LIF cable, no conductances),
    // species on lanes 1..S; then the species not covered there
    {
      const bool v_sys = K.dyn == MCG_DYN_LIF && !refractory && !has_gsyn && K.v_const != 0;
      if (!mcg_const_systems(D, K, M, v_sys, has_current, D.k_sp_cap_dt, D.k_sp_f, D.k_sp_d,
                             lane))
        ok &= mcg_species_rest(D, K, M, D.k_sp_cap_dt, lane);
    }
    __syncwarp();

    // ---- 4. spike detection, post-event hook, reset (engine.cpp:753-780)
    // lane 0 decides and broadcasts: the shuffle is the point after which the
    // reset below may overwrite V (all lanes reading V here would race with a
    // lane that already moved on to the reset)
    int fired = 0;
    double t_spike = 0.0;
    if (lane == 0 && K.has_detector && !refractory) {
      const double va = V[K.detector_comp];
      if (armed && det_prev < K.threshold && va >= K.threshold) {
        double f = (va > det_prev) ? (K.threshold - det_prev) / (va - det_prev) : 1.0;
        f = (f < 0.0) ? 0.0 : ((1.0 < f) ? 1.0 : f);  // std::clamp
        t_spike = (double(s) + f) * D.dt;
        fired = 1;
      }
    }
    fired = __shfl_sync(MCG_FULL, fired, 0);
    if (fired) {
      if (lane == 0) {
        if (nsp < D.sp_cap) {
          D.sp_step[int64_t(c) * D.sp_cap + nsp] = s;
          D.sp_t[int64_t(c) * D.sp_cap + nsp] = t_spike;
        } else {
          atomicOr(D.err, MCG_ERR_FLAG_SPIKES);
        }
      }
      ++nsp;
      mcg_post_event(D, K, cg0, s, lane);
      if (is_lif)
        for (int i = lane; i < n; i += 32) V[i] = K.v_reset;
      __syncwarp();
    }
    if (K.has_detector && !refractory) {
      if (fired) {
        if (is_lif) refr = s + 1 + K.ref_steps;
        else armed = 0;
      } else if (!armed && V[K.detector_comp] < K.threshold) {
        armed = 1;
      }
      det_prev = V[K.detector_comp];
    }
    // probes (engine.cpp:785-793)
    if (lane == 0) {
      for (int q = D.probe_off[c]; q < D.probe_off[c + 1]; ++q) {
        const int p = D.probe_idx[q];
        const McgProbe& P = D.probes[p];
        if ((s + 1) % P.every != 0) continue;
        const int64_t m0 = (D.ctl[3] + P.every) / P.every;  // ctl[3]: first step of the call
        D.trace_buf[D.trace_base[p] + ((s + 1) / P.every - m0)] =
            mcg_probe_value(D, K, c, P, V, M.SP);
      }
    }
    __syncwarp();
  }
  mcg_stage(D, K, c, M, false, lane);
  if (lane == 0) {
    D.pend_sel[c] = sel;
    D.pend_off[c] = cur;
    D.pend_n[c] = end;
    D.inc_n[c] = 0;
    D.sp_count[c] = nsp < D.sp_cap ? nsp : D.sp_cap;
    D.refr_until[c] = refr;
    D.det_prev[c] = det_prev;
    D.armed[c] = armed;
    if (ndel) atomicAdd(D.delivered, ndel);
  }
  const unsigned okm = __ballot_sync(MCG_FULL, ok);
  if (lane == 0 && okm != MCG_FULL) atomicOr(D.err, MCG_ERR_FLAG_SINGULAR);
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
