// mcg_batch.cuh — the persistent batch kernel: a whole batch of min-delay
// epochs (Engine::advance_to, engine.cpp:909-945) in one cooperative launch.
//
//   for each epoch j of the batch:
//     phase 1  expansion: source events of the epoch and the previous epoch's
//              spikes into the per-cell incoming buffers (mcg_events.cuh)
//     grid.sync
//     phase 2  every CTA steps its cell batches through the epoch
//     grid.sync
//
// Phase 2 maps threads to whatever each part of step_cell (engine.cpp:541-783)
// can use, with the cells' compartment state and all per-cell metadata staged
// in shared memory (no dependent global loads on the per-step critical path):
//   owner thread per cell   event delivery, SPS fold, background current,
//                           spike detection (the reference's ordered folds)
//   warp per cell           active-list kernel decay, post-spike hook, inbox merge
//   all threads             STC synapse updates of every cell of the batch,
//                           HH gating of every compartment of the batch
//   thread per system       the Hines sweeps: V and each species of every
//                           cell, all in one instruction stream
// Spikes are logged per CTA batch as chunks (epoch, batch, offset, count); the
// host restores the reference's (epoch, gid, step) order from the chunks.
#pragma once
#include <cooperative_groups.h>

#include "mcg_epoch.cuh"

struct McgBatchArgs {
  McgEv E;
  int32_t n_epochs;        // epochs in this launch
  int32_t cells_per_cta;   // C
  int32_t n_batches;       // ceil(n_cells / C)
  int32_t comp_stride;     // doubles of shared memory per cell for compartment state
  int32_t stc_max;         // max STC instances per cell
  int32_t n_stc_max;       // max STC groups per cell
  int32_t kind_doubles;    // shared memory for staged kind constants
  unsigned long long* phase;  // optional per-phase cycle totals (12)
  double* log_t;           // spike log of the launch
  uint32_t* log_gid;
  unsigned long long* log_n;
  int4* chunks;            // (epoch, batch, offset, count)
  unsigned long long* chunk_n;
};

// phase 1: sources of [s0, s1) + previous epoch's spikes (from the per-cell slots)
__device__ void mcg_expand(const McgEv& E, const McgDev& D, int32_t j, int64_t s0, int64_t s1,
                           int64_t max_len) {
  const int64_t len = s1 - s0;
  const int64_t nthr = int64_t(gridDim.x) * blockDim.x;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t ntask = int64_t(E.n_tasks) * max_len;
  for (int64_t t = tid; t < ntask; t += nthr) {
    const int64_t off = t % max_len;
    if (off >= len) continue;
    const McgSrcTask T = E.tasks[t / max_len];
    const int64_t e0 = E.src_edge_off[T.source], e1 = E.src_edge_off[T.source + 1];
    if (e1 == e0) continue;
    if (T.type == MCG_SRC_POISSON) {
      const int64_t s = s0 + off;
      if (s < T.a || s >= T.b) continue;
      const mcg_key key = mcg_make_key(E.seed, 0x100000000ull + uint64_t(T.source), 3, 0);
      if (!(mcg_uniform_for(&key, static_cast<uint64_t>(s)) < T.prob)) continue;
      for (int64_t k = e0; k < e1; ++k) {
        const int64_t r = E.src_edges[k];
        mcg_push(E, j, r, s + E.e_delay[r]);
      }
    } else if (off == 0) {
      if (T.type == MCG_SRC_SCRIPTED) {
        for (int64_t i = T.a; i < T.b; ++i) {
          const int64_t st = E.scripted_steps[i];
          if (st < s0 || st >= s1) continue;
          for (int64_t k = e0; k < e1; ++k) {
            const int64_t r = E.src_edges[k];
            mcg_push(E, j, r, st + E.e_delay[r]);
          }
        }
      } else if (T.r_period > 0) {
        int64_t k0 = static_cast<int64_t>(ceil((double(s0) * E.dt - T.r_t0) / T.r_period - 1e-9));
        if (k0 < 0) k0 = 0;
        for (int64_t kk = k0; kk < T.r_count; ++kk) {
          const int64_t st = static_cast<int64_t>(ceil((T.r_t0 + double(kk) * T.r_period) / E.dt - 1e-9));
          if (st >= s1) break;
          if (st < s0) continue;
          for (int64_t k = e0; k < e1; ++k) {
            const int64_t r = E.src_edges[k];
            mcg_push(E, j, r, st + E.e_delay[r]);
          }
        }
      }
    }
  }
  // spikes of the previous epoch, one warp per spiking cell
  const int lane = threadIdx.x & 31;
  const int64_t nw = nthr >> 5;
  for (int64_t c = tid >> 5; c < D.n_cells; c += nw) {
    const int k = D.sp_count[c];
    if (k == 0) continue;
    const uint32_t gid = D.gid0 + uint32_t(c);
    const int64_t e0 = E.out_begin[gid], e1 = E.out_end[gid];
    for (int q = 0; q < k; ++q) {
      const int64_t st = D.sp_step[c * D.sp_cap + q];
      for (int64_t r = e0 + lane; r < e1; r += 32) mcg_push(E, j, r, st + 1 + E.e_delay[r]);
    }
  }
}

// per-cell state kept in shared memory for the duration of an epoch
struct McgCellSm {
  int32_t kind, n, sel, cur, end;
  int32_t refractory, has_gsyn, has_current, fired, noise;
  int32_t nsp, armed, stc_off, stc_n, n_stc_seg, hh_off, hh_n, has_act;
  int32_t p0, p1;           // probe range
  int32_t kb, pad2;         // offset of the cell's staged kind constants (-1: global)
  int64_t refr;
  int64_t fifo_next;        // earliest queued delayed-calcium step (INT64_MAX if none)
  uint32_t iseq;
  uint32_t pad;
  unsigned long long ndel;
  double det_prev, prod;
};

// one STC group of a cell, in group order
struct McgSegSm {
  int64_t inst;
  int32_t gi, size, spec, comp;
};

// per-kind constants the sweeps read every step, staged in shared memory once
// per epoch (one copy per distinct kind of the batch).  Layout per kind of n
// compartments and S species (doubles):
//   cap_dt, g_leak, g_leak_rhs, axial, vf, vd, g_na, g_k            8 n
//   per species: sp_cap_dt, sp_gs, sp_coup, sp_f, sp_d               5 n S
// followed by the parent array (n int32, padded to doubles).
struct McgKindSm {
  const double *cap, *gl, *glr, *ax, *vf, *vd, *gna, *gk;
  const double *sp_cap, *sp_gs, *sp_coup, *sp_f, *sp_d;  // [sp * n + i]
  const int32_t* par;
};

__device__ __forceinline__ int mcg_kind_block_doubles(int n, int S) {
  return (8 + 5 * S) * n + (n + 1) / 2;
}

__device__ __forceinline__ McgKindSm mcg_kind_view(const double* p, int n, int S) {
  McgKindSm v;
  v.cap = p;
  v.gl = p + n;
  v.glr = p + 2 * n;
  v.ax = p + 3 * n;
  v.vf = p + 4 * n;
  v.vd = p + 5 * n;
  v.gna = p + 6 * n;
  v.gk = p + 7 * n;
  v.sp_cap = p + 8 * n;
  v.sp_gs = p + (8 + S) * n;
  v.sp_coup = p + (8 + 2 * S) * n;
  v.sp_f = p + (8 + 3 * S) * n;
  v.sp_d = p + (8 + 4 * S) * n;
  v.par = reinterpret_cast<const int32_t*>(p + (8 + 5 * S) * n);
  return v;
}

// copy kind K's constants into p (all threads of the CTA)
__device__ __forceinline__ void mcg_kind_stage(const McgDev& D, const McgKind& K, double* p) {
  const int n = K.n, S = K.n_species, T = blockDim.x;
  const double* src[8] = {D.k_cap_dt, D.k_g_leak, D.k_g_leak_rhs, D.k_axial,
                          D.k_vf,     D.k_vd,     D.k_g_na,       D.k_g_k};
  for (int i = threadIdx.x; i < 8 * n; i += T) p[i] = src[i / n][K.arr + i % n];
  const double* ssrc[5] = {D.k_sp_cap_dt, D.k_sp_gs, D.k_sp_coupling, D.k_sp_f, D.k_sp_d};
  for (int i = threadIdx.x; i < 5 * S * n; i += T) {
    const int a = i / (S * n), r = i % (S * n);
    p[8 * n + i] = ssrc[a][K.sp_arr + r];
  }
  int32_t* par = reinterpret_cast<int32_t*>(p + (8 + 5 * S) * n);
  for (int i = threadIdx.x; i < n; i += T) par[i] = D.k_parent[K.arr + i];
}

__device__ __forceinline__ McgKindSm mcg_kind_consts(const McgDev& D, const McgKind& K,
                                                     const double* ksm, int kb) {
  if (kb >= 0) return mcg_kind_view(ksm + kb, K.n, K.n_species);
  McgKindSm v;
  v.cap = D.k_cap_dt + K.arr;
  v.gl = D.k_g_leak + K.arr;
  v.glr = D.k_g_leak_rhs + K.arr;
  v.ax = D.k_axial + K.arr;
  v.vf = D.k_vf + K.arr;
  v.vd = D.k_vd + K.arr;
  v.gna = D.k_g_na + K.arr;
  v.gk = D.k_g_k + K.arr;
  v.sp_cap = D.k_sp_cap_dt + K.sp_arr;
  v.sp_gs = D.k_sp_gs + K.sp_arr;
  v.sp_coup = D.k_sp_coupling + K.sp_arr;
  v.sp_f = D.k_sp_f + K.sp_arr;
  v.sp_d = D.k_sp_d + K.sp_arr;
  v.par = D.k_parent + K.arr;
  return v;
}

// one species system from staged constants (engine.cpp:726-750)
__device__ __forceinline__ bool mcg_species_sys(int n, bool is_prp, int prp_comp, double prod,
                                                const double* cap, const double* gs,
                                                const double* coup, const double* f,
                                                const double* d, const int32_t* par, double* conc,
                                                double* r2, double* diag, double* rhs_scr) {
  if (n == 1) {
    const double r = cap[0] * conc[0] + (is_prp ? prod : 0.0);
    conc[0] = r / (cap[0] + gs[0]);
    return true;
  }
  const int pc = (is_prp && prod != 0.0) ? prp_comp : -1;
  if (f != nullptr) {
    for (int i = 0; i < n; ++i) r2[i] = cap[i] * conc[i] + (i == pc ? prod : 0.0);
    mcg_solve_const(n, par, coup, f, d, conc, r2);
    return true;
  }
  for (int i = 0; i < n; ++i) rhs_scr[i] = (i == pc) ? prod : 0.0;
  return mcg_solve_tree(n, par, cap, gs, coup, rhs_scr, conc, diag, r2);
}

__device__ __forceinline__ int64_t mcg_fifo_next(const McgDev& D, const McgKind& K, int64_t cg0) {
  int64_t nx = INT64_MAX;
  for (int gi = 0; gi < K.n_groups; ++gi) {
    const McgCellGroup& G = D.cgs[cg0 + gi];
    if (G.fifo < 0) continue;
    const McgFifo& F = D.fifos[G.fifo];
    if (F.head < F.tail) {
      const int64_t st = D.fifo_step[F.base + (F.head % F.cap)];
      if (st < nx) nx = st;
    }
  }
  return nx;
}

// one cell batch [c0, c0 + nc) through epoch [s0, s1)
__device__ void mcg_cell_batch(const McgDev& D, const McgBatchArgs& A, int32_t b, int32_t j,
                               int64_t s0, int64_t s1, double* smem, McgCellSm* cs,
                               double* nbuf, double* dbuf, uint32_t* fmask, McgSegSm* seg,
                               double* ksm) {
  const int tid = threadIdx.x;
  const int T = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = T >> 5;
  const int c0 = b * A.cells_per_cta;
  const int nc = min(A.cells_per_cta, D.n_cells - c0);
  const int S1 = 1 + D.sp_max;  // systems per cell
  const int m = D.smem_n;
  // optional per-phase cycle accounting (A.phase != nullptr)
  unsigned long long ph_last = clock64(), ph[12] = {0};
#define MCG_PH(i)                                     \
  do {                                                \
    if (A.phase && tid == 0) {                        \
      const unsigned long long t_ = clock64();        \
      ph[i] += t_ - ph_last;                          \
      ph_last = t_;                                   \
    }                                                 \
  } while (0)

  // ---- epoch entry: per-cell scalars and metadata
  if (tid < nc) {
    const int c = c0 + tid;
    McgCellSm& X = cs[tid];
    const McgKind& K = D.kinds[D.cell_kind[c]];
    X.kind = D.cell_kind[c];
    X.n = K.n;
    X.sel = D.pend_sel[c];
    X.cur = D.pend_off[c];
    X.end = D.pend_n[c];
    X.refr = D.refr_until[c];
    X.det_prev = D.det_prev[c];
    X.armed = D.armed[c];
    X.nsp = 0;
    X.ndel = 0;
    X.p0 = D.probe_off[c];
    X.p1 = D.probe_off[c + 1];
    const bool is_lif = K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT;
    X.noise = (is_lif && K.has_bg && K.sig_bg != 0.0) ? 1 : 0;
    const int64_t cg0 = D.cg_off[c];
    int ns = 0, tot = 0, act = 0;
    for (int gi = 0; gi < K.n_groups; ++gi) {
      const McgCellGroup& G = D.cgs[cg0 + gi];
      const McgSpec& S = D.specs[G.spec];
      if (S.kind == MCG_SYN_STATIC_COND || S.kind == MCG_SYN_STDP_COND ||
          S.kind == MCG_SYN_STATIC_CURRENT || S.kind == MCG_SYN_HOMEO_CURRENT)
        act = 1;
      if (S.kind != MCG_SYN_STC_CHARGE || ns >= A.n_stc_max) continue;
      McgSegSm& g = seg[tid * A.n_stc_max + ns];
      g.inst = G.inst;
      g.gi = gi;
      g.size = G.size;
      g.spec = G.spec;
      g.comp = S.comp;
      tot += G.size;
      ++ns;
    }
    X.has_act = act;
    X.n_stc_seg = ns;
    X.stc_n = tot;
    X.hh_n = (K.dyn == MCG_DYN_HH) ? K.n : 0;
    X.fifo_next = (K.n_stc_groups > 0) ? mcg_fifo_next(D, K, cg0) : INT64_MAX;
    X.iseq = D.internal_seq[c];
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0, hacc = 0, kacc = 0;
    for (int k = 0; k < nc; ++k) {
      cs[k].stc_off = acc;
      acc += cs[k].stc_n;
      cs[k].hh_off = hacc;
      hacc += cs[k].hh_n;
      // one staged copy per distinct kind of the batch
      cs[k].kb = -1;
      if (cs[k].n <= m) {
        for (int q = 0; q < k; ++q)
          if (cs[q].kind == cs[k].kind && cs[q].kb >= 0) {
            cs[k].kb = cs[q].kb;
            break;
          }
        if (cs[k].kb < 0) {
          const McgKind& K = D.kinds[cs[k].kind];
          cs[k].kb = kacc;
          kacc += mcg_kind_block_doubles(K.n, K.n_species);
        }
      }
    }
  }
  __syncthreads();
  for (int k = 0; k < nc; ++k) {
    if (cs[k].kb < 0) continue;
    bool first = true;
    for (int q = 0; q < k; ++q)
      if (cs[q].kb == cs[k].kb) first = false;
    if (first) mcg_kind_stage(D, D.kinds[cs[k].kind], ksm + cs[k].kb);
  }
  // stage compartment state (cells that fit; the rest use global memory)
  for (int k = 0; k < nc; ++k) {
    const int c = c0 + k;
    const McgKind& K = D.kinds[D.cell_kind[c]];
    if (K.n > m) continue;
    double* base = smem + int64_t(k) * A.comp_stride;
    const int n = K.n;
    const int64_t co = D.comp_off[c];
    for (int i = tid; i < n; i += T) base[i] = D.v[co + i];
    const double* gs = D.species + D.sp_off[c];
    for (int i = tid; i < K.n_species * n; i += T) base[m + i] = gs[i];
    if (K.dyn == MCG_DYN_HH)
      for (int i = tid; i < n; i += T) {
        base[(1 + D.sp_max) * m + i] = D.hh_m[co + i];
        base[(2 + D.sp_max) * m + i] = D.hh_h[co + i];
        base[(3 + D.sp_max) * m + i] = D.hh_n[co + i];
      }
  }
  __syncthreads();
  // inbox merge, warp per cell (the reference's per-epoch inbox sort)
  for (int k = warp; k < nc; k += nwarps) {
    const int c = c0 + k;
    const int nin = D.inc_n[c];
    if (nin == 0) continue;
    McgCellSm& X = cs[k];
    uint64_t* in = D.inc + int64_t(c) * D.inc_cap;
    if (nin > 1) mcg_warp_sort(in, nin, lane);
    __syncwarp();
    const uint64_t* pold = D.pend + (int64_t(c) * 2 + X.sel) * D.pend_cap;
    uint64_t* out = D.pend + (int64_t(c) * 2 + (1 - X.sel)) * D.pend_cap;
    if (lane == 0) {
      int a = X.cur, bb = 0, o = 0;
      const int e = X.end;
      while (a < e && bb < nin) out[o++] = (pold[a] <= in[bb]) ? pold[a++] : in[bb++];
      while (a < e) out[o++] = pold[a++];
      while (bb < nin) out[o++] = in[bb++];
      X.end = o;
      X.cur = 0;
      X.sel = 1 - X.sel;
    }
    __syncwarp();
  }
  __syncthreads();
  MCG_PH(9);
  const int stc_total = cs[nc - 1].stc_off + cs[nc - 1].stc_n;
  const int hh_total = cs[nc - 1].hh_off + cs[nc - 1].hh_n;

  const uint64_t rank_mask = (1ull << D.rank_bits) - 1;
  for (int64_t s = s0; s < s1; ++s) {
    const int64_t so = s - s0;
    // background-noise draws for the next 32 steps of every noisy cell
    if ((so & 31) == 0) {
      for (int q = tid; q < nc * 32; q += T) {
        const int k = q >> 5, l = q & 31;
        if (!cs[k].noise || s + l >= s1) continue;
        const mcg_key key = mcg_make_key(D.seed, D.gid0 + uint32_t(c0 + k), 1, 0);
        nbuf[q] = mcg_normal_for(&key, static_cast<uint64_t>(s + l));
      }
      __syncthreads();
      MCG_PH(0);
    }
    // ---- A. delivery (owner thread): inbox, then internal (engine.cpp:549-560)
    if (tid < nc) {
      const int c = c0 + tid;
      McgCellSm& X = cs[tid];
      const McgKind& K = D.kinds[X.kind];
      const bool is_lif = K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT;
      const bool refractory = is_lif && s < X.refr;
      X.refractory = refractory;
      double* V = (K.n <= m) ? smem + int64_t(tid) * A.comp_stride : D.v + D.comp_off[c];
      const int64_t cg0 = D.cg_off[c];
      int cur = X.cur;
      if (cur < X.end) {
        const uint64_t* pend = D.pend + (int64_t(c) * 2 + X.sel) * D.pend_cap;
        while (cur < X.end) {
          const uint64_t key = pend[cur];
          if (int64_t(key >> D.rank_bits) > s) break;
          const int64_t r = int64_t(key & rank_mask);
          mcg_apply_event(D, K, c, cg0, V, D.e_group[r], D.e_inst[r], D.e_weight[r], 0,
                          refractory, s);
          ++cur;
          ++X.ndel;
        }
        X.cur = cur;
      }
      if (K.n_stc_groups > 0) {
        const uint32_t iseq = D.internal_seq[c];
        if (iseq != X.iseq) {  // calcium was queued this step
          X.iseq = iseq;
          X.fifo_next = mcg_fifo_next(D, K, cg0);
        }
        if (X.fifo_next <= s) {
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
            mcg_apply_event(D, K, c, cg0, V, best, uint32_t(si & 0xffffffffu), 0.0, 1,
                            refractory, s);
          }
          X.fifo_next = mcg_fifo_next(D, K, cg0);
        }
      }
      X.has_gsyn = 0;
      X.has_current = 0;
      double* rc = (K.n <= m) ? V + (6 + D.sp_max) * m : D.s_rhs_cur + D.comp_off[c];
      const int nr = K.n > 1 ? K.n : 1;
      for (int i = 0; i < nr; ++i) rc[i] = 0.0;
    }
    __syncthreads();
    MCG_PH(1);

    // ---- B. active-list kernels (warp per cell, ordered folds, engine.cpp:578-616)
    for (int k = warp; k < nc; k += nwarps) {
      if (!cs[k].has_act) continue;
      const int c = c0 + k;
      const McgKind& K = D.kinds[cs[k].kind];
      const McgCellMem M = mcg_cell_mem(D, K, c, K.n <= m ? smem + int64_t(k) * A.comp_stride : nullptr);
      bool hg = false, hc = false;
      for (int gi = 0; gi < K.n_groups; ++gi) {
        McgCellGroup* G = &D.cgs[D.cg_off[c] + gi];
        const McgSpec& S = D.specs[G->spec];
        if (G->active_n == 0) continue;
        if (S.kind == MCG_SYN_STATIC_COND || S.kind == MCG_SYN_STDP_COND) {
          if (!hg) {
            for (int i = lane; i < K.n; i += 32) {
              M.gsyn[i] = 0.0;
              M.gsyn_rhs[i] = 0.0;
            }
            hg = true;
            __syncwarp();
          }
          mcg_decay_active(D, G, S.f_decay, true, M.gsyn, M.gsyn_rhs, S.e_rev, lane);
        } else if (S.kind == MCG_SYN_STATIC_CURRENT || S.kind == MCG_SYN_HOMEO_CURRENT) {
          if (mcg_decay_active(D, G, S.f_decay, false, M.rhs_cur, nullptr, 0.0, lane)) hc = true;
        }
      }
      if (lane == 0) {
        cs[k].has_gsyn = hg;
        cs[k].has_current = hc;
      }
    }
    // ---- C. STC synapses of every cell of the batch, one flat index space
    // (engine.cpp:617-646); changed flags as warp ballots for the fold
    for (int f0 = tid - lane; f0 < stc_total; f0 += T) {
      const int f = f0 + lane;
      bool changed = false;
      if (f < stc_total) {
        int lo = 0, hi = nc - 1;  // last cell with stc_off <= f
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (cs[mid].stc_off <= f) lo = mid;
          else hi = mid - 1;
        }
        const int k = lo, c = c0 + k;
        int li = f - cs[k].stc_off, q = 0;
        const McgSegSm* sg = seg + k * A.n_stc_max;
        while (li >= sg[q].size) li -= sg[q++].size;
        const McgKind& K = D.kinds[cs[k].kind];
        const double* SPb = (K.n <= m) ? smem + int64_t(k) * A.comp_stride + m
                                       : D.species + D.sp_off[c];
        const double* prp_base = (K.prp_idx >= 0) ? SPb + int64_t(K.prp_idx) * K.n : nullptr;
        const McgStcOut o = mcg_stc_instance(D, D.specs[sg[q].spec], sg[q].inst + li,
                                             D.gid0 + uint32_t(c), sg[q].gi, li, s, prp_base,
                                             D.k_volume + K.arr);
        dbuf[f] = o.delta;
        changed = o.changed;
      }
      const unsigned bal = __ballot_sync(MCG_FULL, changed);
      if (lane == 0) fmask[f0 >> 5] = bal;
    }
    __syncthreads();
    MCG_PH(2);

    // ---- D. SPS fold, synthesis trigger, background current (owner thread)
    if (tid < nc) {
      const int c = c0 + tid;
      McgCellSm& X = cs[tid];
      const McgKind& K = D.kinds[X.kind];
      const bool in_sm = K.n <= m;
      double* base = in_sm ? smem + int64_t(tid) * A.comp_stride : nullptr;
      double* SP = in_sm ? base + m : D.species + D.sp_off[c];
      if (K.sps_idx >= 0) {
        double* sps = SP + int64_t(K.sps_idx) * K.n;
        int f = X.stc_off;
        for (int q = 0; q < X.n_stc_seg; ++q) {
          const McgSegSm& g = seg[tid * A.n_stc_max + q];
          const int fe = f + g.size;
          // every instance of a placement sits on the placement's compartment
          double acc = sps[g.comp];
          while (f < fe) {
            const int w = f >> 5;
            uint32_t bits = fmask[w] >> (f & 31);
            const int lim = min(32 - (f & 31), fe - f);
            if (lim < 32) bits &= (1u << lim) - 1u;
            while (bits) {
              const int l = __ffs(bits) - 1;
              bits &= bits - 1;
              acc += dbuf[f + l];
            }
            f += lim;
          }
          sps[g.comp] = acc;
        }
      }
      X.prod = 0.0;
      if (K.prp_enabled)
        X.prod = (SP[int64_t(K.sps_idx) * K.n + K.prp_comp] > K.prp_theta_star) ? K.prp_rate : 0.0;
      const bool is_lif = K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT;
      const double ts = double(s) * D.dt;
      const bool bg_gated = K.bg_t1 > K.bg_t0 && ts >= K.bg_t0 && ts < K.bg_t1;
      if (is_lif && K.has_bg && !bg_gated) {
        double ib = K.i_bg;
        if (K.sig_bg != 0.0) ib += K.sig_bg * nbuf[tid * 32 + int(so & 31)];
        double* rc = in_sm ? base + (6 + D.sp_max) * m : D.s_rhs_cur + D.comp_off[c];
        rc[K.noise_comp] += ib;
        X.has_current = 1;
      }
    }
    __syncthreads();
    MCG_PH(3);

    // ---- E1. HH gating at the pre-step voltage, every compartment of the batch
    if (hh_total > 0) {
      for (int f = tid; f < hh_total; f += T) {
        int lo = 0, hi = nc - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (cs[mid].hh_off <= f) lo = mid;
          else hi = mid - 1;
        }
        const int k = lo, c = c0 + k;
        const McgKind& K = D.kinds[cs[k].kind];
        const McgCellMem M = mcg_cell_mem(D, K, c, K.n <= m ? smem + int64_t(k) * A.comp_stride : nullptr);
        const int i = f - cs[k].hh_off;
        const McgKindSm KS = mcg_kind_consts(D, K, ksm, cs[k].kb);
        const bool hg = cs[k].has_gsyn, hc = cs[k].has_current;
        const double v = M.V[i];
        double gsum = KS.gl[i];
        double grhs = KS.glr[i];
        const double gnak = KS.gna[i];
        if (gnak != 0.0) {
          const double am = mcg_hh_am(v), bm = mcg_hh_bm(v);
          const double ah = mcg_hh_ah(v), bh = mcg_hh_bh(v);
          const double an = mcg_hh_an(v), bn = mcg_hh_bn(v);
          double mm = M.HM[i], h = M.HH[i], nn = M.HN[i];
          mm += (am / (am + bm) - mm) * (1.0 - mcg_exp(-D.dt * (am + bm)));
          h += (ah / (ah + bh) - h) * (1.0 - mcg_exp(-D.dt * (ah + bh)));
          nn += (an / (an + bn) - nn) * (1.0 - mcg_exp(-D.dt * (an + bn)));
          M.HM[i] = mm;
          M.HH[i] = h;
          M.HN[i] = nn;
          const double gna = gnak * mm * mm * mm * h;
          const double gk = KS.gk[i] * nn * nn * nn * nn;
          gsum += gna + gk;
          grhs += gna * K.e_na + gk * K.e_k;
        }
        M.gsyn[i] = gsum + (hg ? M.gsyn[i] : 0.0);
        M.gsyn_rhs[i] = grhs + (hg ? M.gsyn_rhs[i] : 0.0) + (hc ? M.rhs_cur[i] : 0.0);
      }
      __syncthreads();
      MCG_PH(4);
    }

    // ---- E2. membrane and species systems: thread per (cell, system)
    for (int t = tid; t < nc * S1; t += T) {
      const int k = t / S1, sys = t - k * S1;
      const int c = c0 + k;
      const McgCellSm& X = cs[k];
      const McgKind& K = D.kinds[X.kind];
      const McgCellMem M = mcg_cell_mem(D, K, c, K.n <= m ? smem + int64_t(k) * A.comp_stride : nullptr);
      const McgKindSm KS = mcg_kind_consts(D, K, ksm, X.kb);
      const int n = K.n;
      const bool refractory = X.refractory;
      const bool hg = X.has_gsyn, hc = X.has_current;
      const int q = sys - 1;
      // constant-diagonal systems (LIF-cable V without conductances, species)
      // share one instruction stream across all cells and systems
      const bool v_sys = sys == 0 && K.dyn == MCG_DYN_LIF && !refractory && !hg && K.v_const;
      const bool s_sys = sys > 0 && q < K.n_species && n > 1 && K.sp_const;
      bool ok = true;
      if (v_sys || s_sys) {
        double* x = v_sys ? M.V : M.SP + int64_t(q) * n;
        const int qq = v_sys ? 0 : q;
        const double* cap = v_sys ? KS.cap : KS.sp_cap + qq * n;
        const double* coup = v_sys ? KS.ax : KS.sp_coup + qq * n;
        const double* f = v_sys ? KS.vf : KS.sp_f + qq * n;
        const double* d = v_sys ? KS.vd : KS.sp_d + qq * n;
        const double* glr = v_sys ? KS.glr : cap;
        const double* rc = v_sys ? M.rhs_cur : cap;
        double* r2 = M.r2 + int64_t(v_sys ? 0 : 1 + q) * n;
        const int pc = (!v_sys && q == K.prp_idx && X.prod != 0.0) ? K.prp_comp : -1;
        const double prod = X.prod;
        for (int i = 0; i < n; ++i) {
          // V:       rhs = g_leak_rhs + 0.0 + (has_current ? rhs_current : 0.0) (engine.cpp:683)
          // species: rhs = 0.0, or prod at the synthesis compartment          (engine.cpp:746-748)
          const double rhs = v_sys ? (glr[i] + 0.0 + (hc ? rc[i] : 0.0)) : (i == pc ? prod : 0.0);
          r2[i] = cap[i] * x[i] + rhs;
        }
        mcg_solve_const(n, KS.par, coup, f, d, x, r2);
      } else if (sys == 0) {
        if (K.dyn == MCG_DYN_LIF_EXACT) {
          if (!refractory) {
            const double vinf = K.v_rev + K.r_mem * M.rhs_cur[0];
            M.V[0] = vinf + (M.V[0] - vinf) * K.lif_exact_f;
          }
        } else if (K.dyn == MCG_DYN_LIF && !refractory) {
          for (int i = 0; i < n; ++i) {
            const double gs = KS.gl[i] + (hg ? M.gsyn[i] : 0.0);
            const double rr = KS.glr[i] + (hg ? M.gsyn_rhs[i] : 0.0) + (hc ? M.rhs_cur[i] : 0.0);
            M.gsyn[i] = gs;
            M.gsyn_rhs[i] = rr;
          }
          ok = mcg_solve_tree(n, KS.par, KS.cap, M.gsyn, KS.ax, M.gsyn_rhs, M.V, M.diag, M.r2);
        } else if (K.dyn == MCG_DYN_HH) {
          ok = mcg_solve_tree(n, KS.par, KS.cap, M.gsyn, KS.ax, M.gsyn_rhs, M.V, M.diag, M.r2);
        }
        // singular species systems need the full solver's scratch: run them
        // here, after V, in species order (never happens for valid recipes)
        if (n > 1 && !K.sp_const)
          for (int p = 0; p < K.n_species; ++p)
            ok &= mcg_species_sys(n, p == K.prp_idx, K.prp_comp, X.prod, KS.sp_cap + p * n,
                                  KS.sp_gs + p * n, KS.sp_coup + p * n, nullptr, nullptr, KS.par,
                                  M.SP + int64_t(p) * n, M.r2 + int64_t(1 + p) * n, M.diag,
                                  D.s_rhs + D.comp_off[c]);
      } else if (q < K.n_species && n == 1) {
        mcg_species_sys(1, q == K.prp_idx, K.prp_comp, X.prod, KS.sp_cap + q, KS.sp_gs + q,
                        KS.sp_coup + q, nullptr, nullptr, KS.par, M.SP + q, M.r2, M.diag,
                        M.rhs_cur);
      }
      if (!ok) atomicOr(D.err, MCG_ERR_FLAG_SINGULAR);
    }
    __syncthreads();
    MCG_PH(5);

    // ---- F. spike detection (engine.cpp:753-769)
    if (tid < nc) {
      const int c = c0 + tid;
      McgCellSm& X = cs[tid];
      const McgKind& K = D.kinds[X.kind];
      X.fired = 0;
      if (K.has_detector && !X.refractory) {
        const double* V = (K.n <= m) ? smem + int64_t(tid) * A.comp_stride : D.v + D.comp_off[c];
        const double va = V[K.detector_comp];
        if (X.armed && X.det_prev < K.threshold && va >= K.threshold) {
          double f = (va > X.det_prev) ? (K.threshold - X.det_prev) / (va - X.det_prev) : 1.0;
          f = (f < 0.0) ? 0.0 : ((1.0 < f) ? 1.0 : f);  // std::clamp
          X.fired = 1;
          if (X.nsp < D.sp_cap) {
            D.sp_step[int64_t(c) * D.sp_cap + X.nsp] = s;
            D.sp_t[int64_t(c) * D.sp_cap + X.nsp] = (double(s) + f) * D.dt;
          } else {
            atomicOr(D.err, MCG_ERR_FLAG_SPIKES);
          }
          ++X.nsp;
        }
      }
    }
    __syncthreads();
    MCG_PH(6);
    // post-event hook and LIF reset of the cells that fired (warp per cell)
    for (int k = warp; k < nc; k += nwarps) {
      if (!cs[k].fired) continue;
      const int c = c0 + k;
      const McgKind& K = D.kinds[cs[k].kind];
      mcg_post_event(D, K, D.cg_off[c], s, lane);
      if (K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT) {
        double* V = (K.n <= m) ? smem + int64_t(k) * A.comp_stride : D.v + D.comp_off[c];
        for (int i = lane; i < K.n; i += 32) V[i] = K.v_reset;
      }
    }
    __syncthreads();
    MCG_PH(7);
    // detector bookkeeping and probes (engine.cpp:770-793)
    if (tid < nc) {
      const int c = c0 + tid;
      McgCellSm& X = cs[tid];
      const McgKind& K = D.kinds[X.kind];
      const bool in_sm = K.n <= m;
      const double* V = in_sm ? smem + int64_t(tid) * A.comp_stride : D.v + D.comp_off[c];
      const bool is_lif = K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT;
      if (K.has_detector && !X.refractory) {
        if (X.fired) {
          if (is_lif) X.refr = s + 1 + K.ref_steps;
          else X.armed = 0;
        } else if (!X.armed && V[K.detector_comp] < K.threshold) {
          X.armed = 1;
        }
        X.det_prev = V[K.detector_comp];
      }
      for (int q = X.p0; q < X.p1; ++q) {
        const int p = D.probe_idx[q];
        const McgProbe& P = D.probes[p];
        if ((s + 1) % P.every != 0) continue;
        const int64_t m0 = (D.ctl[3] + P.every) / P.every;
        const double* SP = in_sm ? V + m : D.species + D.sp_off[c];
        D.trace_buf[D.trace_base[p] + ((s + 1) / P.every - m0)] = mcg_probe_value(D, K, c, P, V, SP);
      }
    }
    __syncthreads();
    MCG_PH(8);
  }

  // ---- epoch exit: write back state, log the batch's spikes as one chunk
  for (int k = 0; k < nc; ++k) {
    const int c = c0 + k;
    const McgKind& K = D.kinds[cs[k].kind];
    if (K.n > m) continue;
    const double* base = smem + int64_t(k) * A.comp_stride;
    const int n = K.n;
    const int64_t co = D.comp_off[c];
    for (int i = tid; i < n; i += T) D.v[co + i] = base[i];
    double* gs = D.species + D.sp_off[c];
    for (int i = tid; i < K.n_species * n; i += T) gs[i] = base[m + i];
    if (K.dyn == MCG_DYN_HH)
      for (int i = tid; i < n; i += T) {
        D.hh_m[co + i] = base[(1 + D.sp_max) * m + i];
        D.hh_h[co + i] = base[(2 + D.sp_max) * m + i];
        D.hh_n[co + i] = base[(3 + D.sp_max) * m + i];
      }
  }
  __shared__ int s_log_off;
  if (tid == 0) {
    int tot = 0;
    for (int k = 0; k < nc; ++k) tot += min(cs[k].nsp, D.sp_cap);
    s_log_off = -1;
    if (tot > 0) {
      const unsigned long long off = atomicAdd(A.log_n, static_cast<unsigned long long>(tot));
      const unsigned long long ci = atomicAdd(A.chunk_n, 1ull);
      A.chunks[ci] = make_int4(j, b, static_cast<int>(off), tot);
      s_log_off = static_cast<int>(off);
    }
  }
  __syncthreads();
  if (tid < nc) {
    const int c = c0 + tid;
    const McgCellSm& X = cs[tid];
    const int k = min(X.nsp, D.sp_cap);
    if (k > 0) {
      int before = 0;
      for (int q = 0; q < tid; ++q) before += min(cs[q].nsp, D.sp_cap);
      for (int i = 0; i < k; ++i) {
        A.log_t[s_log_off + before + i] = D.sp_t[int64_t(c) * D.sp_cap + i];
        A.log_gid[s_log_off + before + i] = D.gid0 + uint32_t(c);
      }
    }
    D.sp_count[c] = k;
    if (X.ndel) atomicAdd(D.delivered, X.ndel);
    D.pend_sel[c] = X.sel;
    D.pend_off[c] = X.cur;
    D.pend_n[c] = X.end;
    D.inc_n[c] = 0;
    D.refr_until[c] = X.refr;
    D.det_prev[c] = X.det_prev;
    D.armed[c] = X.armed;
  }
  __syncthreads();
  MCG_PH(10);
  if (A.phase && tid == 0)
    for (int i = 0; i < 12; ++i) atomicAdd(&A.phase[i], ph[i]);
#undef MCG_PH
}

__global__ void __launch_bounds__(512, 1) k_batch(McgDev D, McgBatchArgs A, int64_t max_len) {
  extern __shared__ double mcg_smem[];
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int C = A.cells_per_cta;
  // shared-memory carve-up: compartment blocks, noise draws, STC fold
  // deltas, per-cell scalars, STC segment table, changed-flag bitmask
  double* comp = mcg_smem;
  double* nbuf = comp + int64_t(C) * A.comp_stride;
  double* dbuf = nbuf + C * 32;
  double* ksm = dbuf + int64_t(C) * A.stc_max;
  McgCellSm* cs = reinterpret_cast<McgCellSm*>(ksm + A.kind_doubles);
  McgSegSm* seg = reinterpret_cast<McgSegSm*>(cs + C);
  uint32_t* fmask = reinterpret_cast<uint32_t*>(seg + C * A.n_stc_max);
  for (int32_t j = 0; j < A.n_epochs; ++j) {
    int64_t s0, s1;
    if (!mcg_epoch_bounds(D.ctl, j, s0, s1)) break;
    mcg_expand(A.E, D, j, s0, s1, max_len);
    grid.sync();
    if (*D.abort) break;
    for (int32_t b = blockIdx.x; b < A.n_batches; b += gridDim.x)
      mcg_cell_batch(D, A, b, j, s0, s1, comp, cs, nbuf, dbuf, fmask, seg, ksm);
    grid.sync();
  }
}
