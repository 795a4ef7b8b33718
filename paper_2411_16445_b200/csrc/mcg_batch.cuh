// mcg_batch.cuh — the persistent batch kernel: a whole batch of min-delay
// epochs (Engine::advance_to, engine.cpp:909-945) in one cooperative launch.
//
//   for each epoch j of the batch:
//     phase 1  expansion: source events of the epoch and the previous epoch's
//              spikes into the per-cell incoming buffers (mcg_events.cuh)
//     grid.sync
//     phase 2  every CTA steps its cell batch through the epoch
//     grid.sync
//
// Each CTA owns a batch of ~n_cells/148 cells.  When every batch has its own
// CTA ("resident" mode, the normal case) the batch's compartment state, kind
// constants and per-cell metadata are staged into shared memory once per
// launch and stay there for all epochs of the launch; otherwise each CTA
// stages and writes back a batch per epoch.  Phase 2 maps threads to whatever
// each part of step_cell (engine.cpp:541-783) can use:
//   owner thread per cell   event delivery, SPS fold, background current,
//                           spike detection (the reference's ordered folds)
//   warp per cell           active-list kernel decay, post-spike hook, inbox merge
//   all threads             STC synapse updates of every cell of the batch,
//                           HH gating, right-hand sides of the Hines systems
//   thread per system       the Hines sweeps: V and each species of every
//                           cell, all in one instruction stream
// Spikes are logged per CTA batch as chunks (epoch, batch, offset, count); the
// host restores the reference's (epoch, gid, step) order from the chunks.
#pragma once
#include <cooperative_groups.h>

#include "mcg_epoch.cuh"
#include "mcg_sweep.cuh"

#define MCG_NPHASE 24
#define MCG_LANE_INTS 10
#ifndef MCG_BATCH_THREADS
#define MCG_BATCH_THREADS 256
#endif

struct McgBatchArgs {
  McgEv E;
  int32_t n_epochs;        // epochs in this launch
  int32_t cells_per_cta;   // C
  int32_t n_batches;       // ceil(n_cells / C)
  int32_t comp_stride;     // doubles of shared memory per cell for compartment state
  int32_t stc_max;         // max STC instances per batch (shared-memory table size)
  int32_t n_stc_max;       // max STC groups per cell
  int32_t kind_doubles;    // shared memory for staged kind constants
  int32_t n_specs_sm;      // spec table staged in shared memory (0: read from global)
  int32_t stc_sm;          // STC instance state kept in shared memory (resident batches)
  int32_t ch_stride;       // doubles per cell of chain-sweep scratch ((1 + sp_max) x P_max; 0: none)
  int32_t ch_pmax;         // P_max = max over kinds of 2 ch_lp + 1
  int32_t ev_cap;          // staged-delivery event buffer entries (0: off)
  int32_t fmask_words;     // changed-flag words (fmask)
  int32_t nch_max;         // chain-sweep lanes of a batch (lane descriptor table rows)
  int32_t lean;            // LIF-only launch (compartment block V | SP | rhs_cur)
  int32_t act_max;         // one cell per CTA: phase-B scratch entries (0: warp path)
  unsigned long long* phase;  // optional per-phase cycle totals (MCG_NPHASE)
  double* log_t;           // spike log of the launch
  uint32_t* log_gid;
  unsigned long long* log_n;
  int4* chunks;            // (epoch, batch, offset, count)
  unsigned long long* chunk_n;
  int64_t* x_send;         // sharded: this rank's spikes of the epoch [count, (gid, step, t) x cap]
  int64_t x_cap;
  int32_t epoch_base;      // added to the launch's epoch index in the log chunks
  int32_t dbg;             // development trace (MCG_WARP_DBG: (cell + 1) << 8)
  int64_t dbg_s;
};

// phase 1: sources of [s0, s1) + previous epoch's spikes (from the per-cell slots)
__device__ void mcg_expand(const McgEv& E, const McgDev& D, int32_t j, int64_t s0, int64_t s1,
                           int64_t max_len) {
  const int64_t len = s1 - s0;
  const int64_t nthr = int64_t(gridDim.x) * blockDim.x;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  // Poisson windows: one warp per (window, step) task, lanes over the
  // source's out-edges; consecutive tasks on different CTAs (a burst of one
  // source's edges is spread over the grid instead of a few threads of CTA 0).
  // Windows that miss the epoch are skipped whole.
  const int64_t nw = nthr >> 5;
  const int64_t gw = int64_t(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  (void)max_len;
  const int64_t ntask = int64_t(E.n_poisson) * len;
  for (int64_t t = gw; t < ntask; t += nw) {
    int64_t q, off;
    if (((static_cast<uint64_t>(t) | static_cast<uint64_t>(len)) >> 32) == 0) {
      const uint32_t q32 = static_cast<uint32_t>(t) / static_cast<uint32_t>(len);
      q = q32;
      off = static_cast<uint32_t>(t) - q32 * static_cast<uint32_t>(len);
    } else {
      q = t / len;
      off = t - q * len;
    }
    const McgSrcTask T = E.tasks[q];
    const int64_t s = s0 + off;
    if (s < T.a || s >= T.b) {
      if (T.b <= s0 || T.a >= s1) {  // the window misses the epoch: this warp's
        const int64_t nxt = (q + 1) * len;  // next task in the following window
        t += ((nxt - t + nw - 1) / nw - 1) * nw;
      }
      continue;
    }
    const int64_t e0 = E.src_edge_off[T.source], e1 = E.src_edge_off[T.source + 1];
    if (e1 == e0) continue;
    int fire = 0;
    if (lane == 0) {
      const mcg_key key = mcg_make_key(E.seed, 0x100000000ull + uint64_t(T.source), 3, 0);
      fire = mcg_uniform_for(&key, static_cast<uint64_t>(s)) < T.prob ? 1 : 0;
    }
    if (!__shfl_sync(MCG_FULL, fire, 0)) continue;
    for (int64_t k = e0 + lane; k < e1; k += 32) {
      const int64_t r = E.src_edges[k];
      mcg_push(E, j, r, s + E.e_delay[r]);
    }
  }
  // regular and scripted sources: one warp per source
  for (int64_t q = E.n_poisson + gw; q < E.n_tasks; q += nw) {
    const McgSrcTask T = E.tasks[q];
    const int64_t e0 = E.src_edge_off[T.source], e1 = E.src_edge_off[T.source + 1];
    if (e1 == e0) continue;
    if (T.type == MCG_SRC_SCRIPTED) {
      for (int64_t i = T.a; i < T.b; ++i) {
        const int64_t st = E.scripted_steps[i];
        if (st < s0 || st >= s1) continue;
        for (int64_t k = e0 + lane; k < e1; k += 32) {
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
        for (int64_t k = e0 + lane; k < e1; k += 32) {
          const int64_t r = E.src_edges[k];
          mcg_push(E, j, r, st + E.e_delay[r]);
        }
      }
    }
  }
  // spikes of the previous epoch (engine.cpp:875-889: delivery at
  // step + 1 + delay), one warp per spike / spiking cell, lanes over out-edges
  if (E.x_recv != nullptr) {  // sharded: every rank's spikes, local out-edges only
    for (int r = 0; r < E.x_world; ++r) {
      const int64_t* blk = E.x_recv + r * E.x_block;
      const int64_t n = blk[0];
      for (int64_t w = tid >> 5; w < n; w += nw) {
        const uint32_t gid = static_cast<uint32_t>(blk[1 + 3 * w]);
        const int64_t st = blk[2 + 3 * w];
        const int64_t e0 = E.out_begin[gid], e1 = E.out_end[gid];
        for (int64_t q = e0 + lane; q < e1; q += 32) mcg_push(E, j, q, st + 1 + E.e_delay[q]);
      }
    }
    return;
  }
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

// per-cell state kept in shared memory while the batch is staged
struct McgCellSm {
  int32_t n, sel, cur, end;
  int32_t refractory, has_gsyn, has_current, fired, noise;
  int32_t nsp, armed, stc_off, stc_n, n_stc_seg, hh_off, hh_n, has_act;
  int32_t p0, p1;           // probe range
  int32_t kb;               // offset of the cell's staged kind constants (-1: global)
  int32_t lif;
  int32_t pad;
  int64_t refr;
  int64_t fifo_next;        // earliest queued delayed-calcium step (INT64_MAX if none)
  uint64_t nk;              // next pending inbox key (~0 if none)
  unsigned long long ndel;
  double det_prev, prod;
  // staged delivery (mcg_stage_events): the epoch's due events in shared memory
  int32_t fast;             // cell eligible for staged delivery (static per launch)
  int32_t staged;           // this epoch's events are staged
  int32_t ev_cur, ev_end;   // network events [ev_cur, ev_end) of the event buffer
  int32_t in_cur, in_end;   // delayed-calcium events [in_cur, in_end)
  uint32_t iseq;            // internal_seq (engine.cpp:499), resident copy
  int32_t pad2;
  uint8_t gk[8];            // per group: synapse kind
  int8_t gseg[8];           // per group: STC segment index (-1: none)
};

// one staged event (24 B): network events carry the weight (static charge:
// weight x charge factor, the product apply_event forms) and the target
// compartment; delayed-calcium events only their group and instance
struct McgEvSm {
  double w;
  uint32_t inst;            // | 0x80000000 when the raw weight is nonzero
  uint32_t src;             // EventRec.src (kept in delayed-calcium entries for checkpoints)
  uint16_t comp;
  uint8_t group;
  uint8_t so;               // step - s0
  uint32_t pad;
};

// one STC group of a cell, in group order
struct McgSegSm {
  int64_t inst;
  int32_t gi, size, spec, comp;
  int32_t start, pad;       // first instance's index within the cell's STC range
  double vol, rvol;         // volume of the placement's compartment, mcg_recip of it
  double cf;                // charge factor of the placement's compartment
  int64_t f_base, f_head, f_tail;  // delayed-calcium queue (McgFifo), resident copy
  int32_t f_cap, fifo;
  int32_t prp_sm;           // mcg_smem offset of the PRP value at comp (-1: global / none)
  int32_t late;             // the cell has a PRP pool (stc_late_step runs)
  int64_t ca_delay;         // spec fields the staged delivery reads (McgSpec copies,
  double h0, cpre_s;        // so the delivery chain stays in shared memory)
};

// per-kind constants the sweeps read every step, staged in shared memory once
// (one copy per distinct kind of the batch).  Layout per kind of n
// compartments and S species (doubles):
//   cap_dt, g_leak, g_leak_rhs, axial, vf, vd, vr, g_na, g_k        9 n
//   per species: sp_cap_dt, sp_gs, sp_coup, sp_f, sp_d, sp_r         6 n S
// followed by the parent array (n int32, padded to doubles) and a spare word.
struct McgKindSm {
  const double *cap, *gl, *glr, *ax, *vf, *vd, *vr, *gna, *gk;
  const double *sp_cap, *sp_gs, *sp_coup, *sp_f, *sp_d, *sp_r;  // [sp * n + i]
  const int32_t* par;
};

// + one spare word (mcg_sweep_const_sm), then the chain section when the kind
// has a chain schedule (lp > 0, P = 2 lp + 1 positions): the position -> node
// list (int32) and, per system (V, then each species), f | coup | d | y | cap |
// g_leak_rhs (V; 0 for species) in position order (mcg_sweep.cuh)
__host__ __device__ __forceinline__ int mcg_kind_block_doubles(int n, int S, int lp) {
  const int P = 2 * lp + 1;
  return (9 + 6 * S) * n + (n + 1) / 2 + 1 + (lp > 0 ? (P + 1) / 2 + 6 * (1 + S) * P : 0);
}
__host__ __device__ __forceinline__ int mcg_kind_chain_off(int n, int S) {  // doubles
  return (9 + 6 * S) * n + (n + 1) / 2 + 1;
}

__device__ __forceinline__ McgKindSm mcg_kind_view(const double* p, int n, int S) {
  McgKindSm v;
  v.cap = p;
  v.gl = p + n;
  v.glr = p + 2 * n;
  v.ax = p + 3 * n;
  v.vf = p + 4 * n;
  v.vd = p + 5 * n;
  v.vr = p + 6 * n;
  v.gna = p + 7 * n;
  v.gk = p + 8 * n;
  v.sp_cap = p + 9 * n;
  v.sp_gs = p + (9 + S) * n;
  v.sp_coup = p + (9 + 2 * S) * n;
  v.sp_f = p + (9 + 3 * S) * n;
  v.sp_d = p + (9 + 4 * S) * n;
  v.sp_r = p + (9 + 5 * S) * n;
  v.par = reinterpret_cast<const int32_t*>(p + (9 + 6 * S) * n);
  return v;
}

// copy kind K's constants into p (all threads of the CTA)
__device__ __forceinline__ void mcg_kind_stage(const McgDev& D, const McgKind& K, double* p) {
  const int n = K.n, S = K.n_species, T = blockDim.x;
  const double* src[9] = {D.k_cap_dt, D.k_g_leak, D.k_g_leak_rhs, D.k_axial, D.k_vf,
                          D.k_vd,     D.k_vr,     D.k_g_na,       D.k_g_k};
  for (int i = threadIdx.x; i < 9 * n; i += T) p[i] = src[i / n][K.arr + i % n];
  const double* ssrc[6] = {D.k_sp_cap_dt, D.k_sp_gs, D.k_sp_coupling,
                           D.k_sp_f,      D.k_sp_d,  D.k_sp_r};
  for (int i = threadIdx.x; i < 6 * S * n; i += T) {
    const int a = i / (S * n), r = i % (S * n);
    p[9 * n + i] = ssrc[a][K.sp_arr + r];
  }
  int32_t* par = reinterpret_cast<int32_t*>(p + (9 + 6 * S) * n);
  for (int i = threadIdx.x; i < n; i += T) par[i] = D.k_parent[K.arr + i];
  if (K.ch_lp > 0) {  // chain section (mcg_kind_block_doubles)
    const int P = 2 * K.ch_lp + 1;
    double* cb = p + mcg_kind_chain_off(n, S);
    int32_t* idx = reinterpret_cast<int32_t*>(cb);
    for (int i = threadIdx.x; i < P; i += T) idx[i] = D.k_ch_idx[K.ch_arr + i];
    double* sysb = cb + (P + 1) / 2;
    for (int i = threadIdx.x; i < (1 + S) * P; i += T) {
      const int sy = i / P, pos = i - sy * P;
      const int node = D.k_ch_idx[K.ch_arr + pos];
      double f = -0.0, c = 0.0, d = 1.0, y = 1.0, cp = 0.0, gl = 0.0;  // padding: exact identities
      if (node >= 0) {
        const int64_t o = (sy == 0) ? K.arr + node : K.sp_arr + int64_t(sy - 1) * n + node;
        f = (sy == 0) ? D.k_vf[o] : D.k_sp_f[o];
        c = (sy == 0) ? D.k_axial[o] : D.k_sp_coupling[o];
        d = (sy == 0) ? D.k_vd[o] : D.k_sp_d[o];
        y = (sy == 0) ? D.k_vr[o] : D.k_sp_r[o];
        cp = (sy == 0) ? D.k_cap_dt[o] : D.k_sp_cap_dt[o];
        gl = (sy == 0) ? D.k_g_leak_rhs[o] : 0.0;
      }
      double* q = sysb + sy * 6 * P;
      q[pos] = f;
      q[P + pos] = c;
      q[2 * P + pos] = d;
      q[3 * P + pos] = y;
      q[4 * P + pos] = cp;
      q[5 * P + pos] = gl;
    }
  }
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
  v.vr = D.k_vr + K.arr;
  v.gna = D.k_g_na + K.arr;
  v.gk = D.k_g_k + K.arr;
  v.sp_cap = D.k_sp_cap_dt + K.sp_arr;
  v.sp_gs = D.k_sp_gs + K.sp_arr;
  v.sp_coup = D.k_sp_coupling + K.sp_arr;
  v.sp_f = D.k_sp_f + K.sp_arr;
  v.sp_d = D.k_sp_d + K.sp_arr;
  v.sp_r = D.k_sp_r + K.sp_arr;
  v.par = D.k_parent + K.arr;
  return v;
}

// the dynamic shared memory of k_batch; the shared-memory-resident paths index
// it with 32-bit offsets so they compile to LDS/STS (a generic pointer that may
// point to either space costs a 64-bit generic load per access)
extern __shared__ double mcg_smem[];

// offsets (in doubles; par in int32 units) of one staged kind block
struct McgKindOff {
  int cap, gl, glr, ax, vf, vd, vr, gna, gk;
  int sp_cap, sp_gs, sp_coup, sp_f, sp_d, sp_r;  // + sp * n
  int par;
};

__device__ __forceinline__ McgKindOff mcg_kind_off(int o, int n, int S) {
  McgKindOff v;
  v.cap = o;
  v.gl = o + n;
  v.glr = o + 2 * n;
  v.ax = o + 3 * n;
  v.vf = o + 4 * n;
  v.vd = o + 5 * n;
  v.vr = o + 6 * n;
  v.gna = o + 7 * n;
  v.gk = o + 8 * n;
  v.sp_cap = o + 9 * n;
  v.sp_gs = o + (9 + S) * n;
  v.sp_coup = o + (9 + 2 * S) * n;
  v.sp_f = o + (9 + 3 * S) * n;
  v.sp_d = o + (9 + 4 * S) * n;
  v.sp_r = o + (9 + 5 * S) * n;
  v.par = 2 * (o + (9 + 6 * S) * n);
  return v;
}

// Constant-diagonal Hines solve (tree_solver.cpp:55-73 with the elimination
// factors f and eliminated diagonal d precomputed, y = mcg_recip(d)); r2 holds
// cap*x + rhs on entry, x receives the solution.  Operation order is the
// reference's: r2[par[i]] += f[i]*r2[i] for i = n-1..1, then
// x[i] = (r2[i] + coup[i]*x[par[i]]) / d[i] for i = 0..n-1.  Along unbranched
// runs (par[i] == i-1) the running value stays in a register, so each link of
// the dependency chain is a multiply-add pair (elimination) or a multiply-add
// plus mcg_div (substitution); everything else is prefetched one node ahead.
__device__ __forceinline__ void mcg_sweep_const(int n, const int32_t* par, const double* coup,
                                                const double* f, const double* d,
                                                const double* y, double* x, double* r2) {
  if (n == 1) {
    x[0] = mcg_div(r2[0], d[0], y[0]);
    return;
  }
  // elimination: cur = final r2 of node i; base = r2 of node i-1 before child i
  double cur = r2[n - 1];
  double base = r2[n - 2];
  int p = par[n - 1];
  double fi = f[n - 1];
  for (int i = n - 1; i >= 1; --i) {
    int pn = 0;
    double fn = 0.0, bn = 0.0;
    const bool more = i >= 2;
    if (more) {
      pn = par[i - 1];
      fn = f[i - 1];
    }
    const double t = fi * cur;
    if (p == i - 1) {
      if (more) bn = r2[i - 2];  // no store of this iteration touches node i-2
      cur = base + t;            // child i is node i-1's last (smallest) child
      r2[i - 1] = cur;
    } else {
      r2[p] = r2[p] + t;         // branch point p < i-1: partial sum in memory
      if (more) bn = r2[i - 2];  // after the store (p may be i-2)
      cur = base;                // node i-1 is complete (its children are > i)
    }
    p = pn;
    fi = fn;
    base = bn;
  }
  // back-substitution
  double vprev = mcg_div(r2[0], d[0], y[0]);
  x[0] = vprev;
  int p1 = par[1];
  double r1 = r2[1], c1 = coup[1], d1 = d[1], y1 = y[1];
  for (int i = 1; i < n; ++i) {
    int pn = 0;
    double rn = 0.0, cn = 0.0, dn = 1.0, yn = 0.0;
    if (i + 1 < n) {
      pn = par[i + 1];
      rn = r2[i + 1];
      cn = coup[i + 1];
      dn = d[i + 1];
      yn = y[i + 1];
    }
    const double vp = (p1 == i - 1) ? vprev : x[p1];
    vprev = mcg_div(r1 + c1 * vp, d1, y1);
    x[i] = vprev;
    p1 = pn;
    r1 = rn;
    c1 = cn;
    d1 = dn;
    y1 = yn;
  }
}

// right-hand side of a constant system on shared memory, four compartments'
// operands loaded ahead of their stores:
//   r2[i] = cap[i]*x[i] + (v ? (glr[i] + 0.0 + (rc >= 0 ? S[rc+i] : 0.0))
//                            : (i == pc ? prod : 0.0))
__device__ __forceinline__ void mcg_rhs_sm(int n, int cap, int x, int r2, bool v, int glr, int rc,
                                           int pc, double prod) {
  double* S = mcg_smem;
  const bool hc = rc >= 0;
  if (!v) glr = cap;  // any valid offset: the V-only operands are unused
  if (!hc) rc = cap;
  int i = 0;
  for (; i + 4 <= n; i += 4) {
    double c4[4], x4[4], g4[4], r4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c4[u] = S[cap + i + u];
      x4[u] = S[x + i + u];
      g4[u] = S[glr + i + u];
      r4[u] = S[rc + i + u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double rhs = v ? (g4[u] + 0.0 + (hc ? r4[u] : 0.0)) : (i + u == pc ? prod : 0.0);
      S[r2 + i + u] = c4[u] * x4[u] + rhs;
    }
  }
  for (; i < n; ++i) {
    const double rhs = v ? (S[glr + i] + 0.0 + (hc ? S[rc + i] : 0.0)) : (i == pc ? prod : 0.0);
    S[r2 + i] = S[cap + i] * S[x + i] + rhs;
  }
}

// mcg_sweep_const on shared memory: every operand an offset into mcg_smem.
// Operands of the next node are loaded unconditionally; at the ends of the
// sweeps that reads one element outside an array (r2[-1] or one past the
// end), which stays inside the carve-up (diag precedes r2; every kind block
// has one spare word, see mcg_kind_block_doubles) and is never used.
__device__ __forceinline__ void mcg_sweep_const_sm(int n, int par, int coup, int f, int d, int y,
                                                   int x, int r2) {
  double* S = mcg_smem;
  const int32_t* PI = reinterpret_cast<const int32_t*>(mcg_smem);
  if (n == 1) {
    S[x] = mcg_div(S[r2], S[d], S[y]);
    return;
  }
  // elimination: cur = final r2 of node i; base = r2 of node i-1 before child i
  double cur = S[r2 + n - 1];
  double base = S[r2 + n - 2];
  int p = PI[par + n - 1];
  double fi = S[f + n - 1];
#pragma unroll 1
  for (int i = n - 1; i >= 1; --i) {
    const int pn = PI[par + i - 1];
    const double fn = S[f + i - 1];
    const double t = fi * cur;
    const bool chain = p == i - 1;     // child i is node i-1's last (smallest) child
    if (!chain) S[r2 + p] += t;        // branch point p < i-1: partial sum in memory
    const double bn = S[r2 + i - 2];   // after that store (p may be i-2)
    cur = chain ? base + t : base;     // else node i-1 is complete (children > i)
    S[r2 + i - 1] = cur;
    p = pn;
    fi = fn;
    base = bn;
  }
  // back-substitution
  double vprev = mcg_div(S[r2], S[d], S[y]);
  S[x] = vprev;
  int p1 = PI[par + 1];
  double r1 = S[r2 + 1], c1 = S[coup + 1], d1 = S[d + 1], y1 = S[y + 1];
#pragma unroll 1
  for (int i = 1; i < n; ++i) {
    const int pn = PI[par + i + 1];
    const double rn = S[r2 + i + 1], cn = S[coup + i + 1], dn = S[d + i + 1], yn = S[y + i + 1];
    const double vp = (p1 == i - 1) ? vprev : S[x + p1];
    vprev = mcg_div(r1 + c1 * vp, d1, y1);
    S[x + i] = vprev;
    p1 = pn;
    r1 = rn;
    c1 = cn;
    d1 = dn;
    y1 = yn;
  }
}

// one species system from staged constants (engine.cpp:726-750), for the
// cases the constant stream does not cover
__device__ __forceinline__ bool mcg_species_sys(int n, bool is_prp, int prp_comp, double prod,
                                                const double* cap, const double* gs,
                                                const double* coup, const int32_t* par,
                                                double* conc, double* r2, double* diag,
                                                double* rhs_scr) {
  if (n == 1) {
    const double r = cap[0] * conc[0] + (is_prp ? prod : 0.0);
    conc[0] = r / (cap[0] + gs[0]);
    return true;
  }
  const int pc = (is_prp && prod != 0.0) ? prp_comp : -1;
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
      const int64_t st = D.fifo_step[F.base + mcg_mod(F.head, F.cap)];
      if (st < nx) nx = st;
    }
  }
  return nx;
}

// does system sys of a staged cell take the chain sweep this step
__device__ __forceinline__ bool mcg_chain_ok(const McgKind& K, const McgCellSm& X, int sys, int m) {
  if (K.ch_lp == 0 || K.n > m) return false;
  if (sys == 0) return K.dyn == MCG_DYN_LIF && !X.refractory && !X.has_gsyn && K.v_const;
  return sys - 1 < K.n_species && K.n > 1 && K.sp_const;
}

// shared-memory carve-up of one CTA (see k_batch)
struct McgBatchSm {
  double* comp;     // C x comp_stride: V | SP | HM HH HN | gsyn gsyn_rhs rhs_cur diag | r2
  double* nbuf;     // C x 32 background-noise draws
  double* dbuf;     // stc_max SPS fold deltas
  double* stc;      // stc_sm: 4 x stc_max STC state h | z | c | |h-h0| (SoA)
  double* abuf;     // act_max decayed kernels (kept) or -0.0 (dropped), phase B
  double* ksm;      // staged kind constants
  McgKind* kc;      // C kind records
  McgCellSm* cs;    // C cell records
  McgSegSm* seg;    // C x n_stc_max STC groups
  McgSpec* spec;    // staged spec table (n_specs_sm entries)
  uint32_t* floc;   // stc_max: (cell << 16) | group of each STC instance slot
  uint32_t* fmask;  // stc_max / 32 changed-flag words
  int* aidx;        // act_max instance index of each abuf entry
  McgEvSm* evb;     // staged events (ev_cap entries)
  int* lanes;       // nch_max x MCG_LANE_INTS static chain-lane descriptors
  int ksm_o;        // offset of ksm in mcg_smem (doubles)
  int chs_o;        // offset of the chain-sweep scratch (C x ch_stride doubles)
};

// the carve-up, derived from mcg_smem in every function that uses it (so the
// compiler sees shared-memory pointers, not generic ones)
__device__ __forceinline__ McgBatchSm mcg_batch_sm(const McgBatchArgs& A) {
  const int C = A.cells_per_cta;
  McgBatchSm B;
  B.comp = mcg_smem;
  B.nbuf = B.comp + C * A.comp_stride;
  B.dbuf = B.nbuf + C * 32;
  B.stc = B.dbuf + A.stc_max;
  B.abuf = B.stc + (A.stc_sm ? 4 * A.stc_max : 0);
  B.chs_o = C * A.comp_stride + C * 32 + A.stc_max + (A.stc_sm ? 4 * A.stc_max : 0) + A.act_max;
  B.ksm_o = B.chs_o + C * A.ch_stride;
  B.ksm = mcg_smem + B.ksm_o;
  B.kc = reinterpret_cast<McgKind*>(B.ksm + A.kind_doubles);
  B.cs = reinterpret_cast<McgCellSm*>(B.kc + C);
  B.seg = reinterpret_cast<McgSegSm*>(B.cs + C);
  B.spec = reinterpret_cast<McgSpec*>(B.seg + C * A.n_stc_max);
  B.floc = reinterpret_cast<uint32_t*>(B.spec + A.n_specs_sm);
  B.fmask = B.floc + A.stc_max;
  {
    B.aidx = reinterpret_cast<int*>(B.fmask + A.fmask_words);
    B.lanes = B.aidx + A.act_max;
    const uintptr_t e = reinterpret_cast<uintptr_t>(B.lanes + A.nch_max * MCG_LANE_INTS);
    B.evb = reinterpret_cast<McgEvSm*>((e + 15) & ~uintptr_t(15));
  }
  return B;
}

// optional per-phase cycle accounting (A.phase != nullptr), thread 0 of each
// CTA; the accumulators live in static shared memory (no registers held)
__shared__ unsigned long long mcg_ph_acc[MCG_NPHASE + 1];  // [MCG_NPHASE]: last stamp
#define MCG_PH(i)                                                  \
  do {                                                             \
    if (A.phase && threadIdx.x == 0) {                             \
      const unsigned long long t_ = clock64();                     \
      mcg_ph_acc[i] += t_ - mcg_ph_acc[MCG_NPHASE];                \
      mcg_ph_acc[MCG_NPHASE] = t_;                                 \
    }                                                              \
  } while (0)

__device__ __forceinline__ double* mcg_comp_block(const McgBatchArgs& A, const McgBatchSm& B,
                                                  int k) {
  return B.comp + k * A.comp_stride;
}

// where the STC state of cell k's group gi lives (shared-memory slot or global)
__device__ __forceinline__ McgStcSm mcg_stc_ref(const McgBatchArgs& A, const McgBatchSm& B, int k,
                                                int gi) {
  McgStcSm R{B.stc, A.stc_max, -1};
  if (!A.stc_sm) return R;
  const McgCellSm& X = B.cs[k];
  for (int q = 0; q < X.n_stc_seg; ++q) {
    const McgSegSm& g = B.seg[k * A.n_stc_max + q];
    if (g.gi == gi) R.slot0 = X.stc_off + g.start;
  }
  return R;
}

// post_event (engine.cpp:515-539) of cell k, one warp; STC calcium in the
// shared-memory copy when the batch keeps it there
__device__ __forceinline__ void mcg_post_event_b(const McgDev& D, const McgBatchArgs& A,
                                                 const McgBatchSm& B, const McgKind& K, int k,
                                                 int64_t cg0, int64_t s, int lane) {
  if (!A.stc_sm) {
    mcg_post_event(D, K, cg0, s, lane);
    return;
  }
  for (int gi = 0; gi < K.n_groups; ++gi) {
    const McgCellGroup G = D.cgs[cg0 + gi];
    const McgSpec& S = D.specs[G.spec];
    if (S.kind == MCG_SYN_STC_CHARGE) {
      const McgStcSm R = mcg_stc_ref(A, B, k, gi);
      for (int i = lane; i < G.size; i += 32) R.base[2 * R.stride + R.slot0 + i] += S.cpost_s;
    } else if (S.kind == MCG_SYN_STDP_COND) {
      for (int i = lane; i < G.size; i += 32) {
        const int64_t j = G.inst + i;
        double pre = D.i_stdp_pre[j], post = D.i_stdp_post[j];
        const double gap = double(s + 1 - D.i_stdp_last[j]) * D.dt;
        if (gap > 0) mcg_stdp_decay(pre, post, S, gap);
        D.i_stdp_last[j] = s + 1;
        post += S.a_post;  // stdp_on_post
        D.i_stdp_w[j] += pre;
        D.i_stdp_pre[j] = pre;
        D.i_stdp_post[j] = post;
      }
    } else if (S.kind == MCG_SYN_HOMEO_CURRENT) {
      for (int i = lane; i < G.size; i += 32) {
        const int64_t j = G.inst + i;
        D.i_homeo_w[j] = fmax(D.i_homeo_w[j] + S.dw_minus, 0.0);
      }
    }
  }
}

// staged delivery: queue metadata and internal_seq move between the global
// arrays (authoritative while a cell is not staged) and the cell's shared
// records (while it is)
__device__ __forceinline__ void mcg_unstage(const McgDev& D, const McgBatchArgs& A,
                                            const McgBatchSm& B, int k, int c) {
  McgCellSm& X = B.cs[k];
  for (int q = 0; q < X.n_stc_seg; ++q) {
    const McgSegSm& g = B.seg[k * A.n_stc_max + q];
    if (g.fifo < 0) continue;
    D.fifos[g.fifo].head = g.f_head;
    D.fifos[g.fifo].tail = g.f_tail;
  }
  D.internal_seq[c] = X.iseq;
  X.staged = 0;
}

// The epoch's due events of cell k, staged by its warp at the epoch's start
// (the reference's inbox and internal-heap pops of engine.cpp:549-560, with
// every global lookup done here in parallel instead of on the delivery chain):
// network events [cur, first step >= s1) of the sorted pending list with
// their edge payload resolved, then the delayed-calcium entries due before s1
// merged over the cell's STC groups in (step, seq) order (InternalOrder).
// Returns false (cell delivered from global memory this epoch) if the event
// buffer is full.
// ascending bitonic sort of one key per lane (~0 pads), by shuffles
__device__ __forceinline__ uint64_t mcg_warp_sort_reg(uint64_t v, int lane, int n) {
  // stages up to the smallest power of two >= n (the pads are the largest keys)
  for (int k = 2; k < 2 * n && k <= 32; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t p = __shfl_xor_sync(MCG_FULL, v, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      v = (lower == up) ? (v < p ? v : p) : (v < p ? p : v);
    }
  return v;
}

// regs: the pending list is exactly this epoch's sorted inbox, held one key
// per lane (rkey), its first rnd keys due (the merge loop's common case)
__device__ bool mcg_stage_events(const McgDev& D, const McgBatchArgs& A, const McgBatchSm& B,
                                 int k, int c, int64_t s0, int64_t s1, int lane, int* ev_top,
                                 bool regs = false, uint64_t rkey = 0, int rnd = 0) {
  McgCellSm& X = B.cs[k];
  const McgKind& K = B.kc[k];
  const uint64_t* pend = D.pend + (int64_t(c) * 2 + X.sel) * D.pend_cap;
  const uint64_t lim = uint64_t(s1) << D.rank_bits;
  int nd = rnd;
  if (!regs)
    for (int base = X.cur; base < X.end; base += 32) {
      const int i = base + lane;
      const unsigned bal = __ballot_sync(MCG_FULL, i < X.end && pend[i] < lim);
      nd += __popc(bal);
      if (bal != MCG_FULL) break;
    }
  if (!X.staged) {  // take the queue metadata over from global memory
    __syncwarp();
    if (lane == 0) {
      for (int q = 0; q < X.n_stc_seg; ++q) {
        McgSegSm& g = B.seg[k * A.n_stc_max + q];
        if (g.fifo < 0) continue;
        g.f_head = D.fifos[g.fifo].head;
        g.f_tail = D.fifos[g.fifo].tail;
      }
      X.iseq = D.internal_seq[c];
    }
    __syncwarp();
  }
  // delayed-calcium entries due in the epoch, per STC segment
  int ni = 0, nseg = 0;
  for (int q = 0; q < X.n_stc_seg; ++q) {
    const McgSegSm& g = B.seg[k * A.n_stc_max + q];
    if (g.fifo < 0) continue;
    int nq = 0;
    for (int64_t base = g.f_head; base < g.f_tail; base += 32) {
      const int64_t i = base + lane;
      const bool due = i < g.f_tail && D.fifo_step[g.f_base + mcg_mod(i, g.f_cap)] < s1;
      const unsigned bal = __ballot_sync(MCG_FULL, due);
      nq += __popc(bal);
      if (bal != MCG_FULL) break;
    }
    ni += nq;
    nseg += nq > 0 ? 1 : 0;
  }
  int beg = 0;
  if (lane == 0) beg = atomicAdd(ev_top, nd + ni);
  beg = __shfl_sync(MCG_FULL, beg, 0);
  if (beg + nd + ni > A.ev_cap) {
    __syncwarp();
    if (lane == 0) {
      if (X.staged) mcg_unstage(D, A, B, k, c);
      X.staged = 0;
      X.fifo_next = mcg_fifo_next(D, K, D.cg_off[c]);
      X.nk = (X.cur < X.end) ? pend[X.cur] : ~0ull;
    }
    __syncwarp();
    return false;
  }
  const uint64_t rank_mask = (1ull << D.rank_bits) - 1;
  for (int t = lane; t < nd; t += 32) {
    const uint64_t key = regs ? rkey : pend[X.cur + t];
    const int64_t r = int64_t(key & rank_mask);
    const int grp = D.e_group[r];
    const uint32_t inst = D.e_inst[r];
    const double w = D.e_weight[r];
    McgEvSm e;
    e.group = static_cast<uint8_t>(grp);
    e.so = static_cast<uint8_t>(int64_t(key >> D.rank_bits) - s0);
    e.comp = 0;
    e.w = w;
    if (X.gk[grp] == MCG_SYN_STATIC_CHARGE) {  // apply_event: V[comp] += w * cf[comp]
      e.comp = static_cast<uint16_t>(D.e_comp[r]);
      e.w = D.e_wcf[r];
    }
    e.inst = inst | (w != 0.0 ? 0x80000000u : 0u);
    e.src = D.e_src[r];
    e.pad = 0;
    B.evb[beg + t] = e;
  }
  // delayed calcium: one segment's entries in queue order, or a merge by seq
  int o = beg + nd;
  for (int q = 0; q < X.n_stc_seg; ++q) {
    McgSegSm& g = B.seg[k * A.n_stc_max + q];
    if (g.fifo < 0) continue;
    if (nseg <= 1) {
      int nq = 0;
      for (int64_t base = g.f_head; base < g.f_tail; base += 32) {
        const int64_t i = base + lane;
        const int64_t slot = g.f_base + mcg_mod(i, g.f_cap);
        const bool due = i < g.f_tail && D.fifo_step[slot] < s1;
        const unsigned bal = __ballot_sync(MCG_FULL, due);
        if (due) {
          McgEvSm e;
          e.w = 0.0;
          e.inst = uint32_t(D.fifo_si[slot] & 0xffffffffu);
          e.src = 0;
          e.pad = 0;
          e.comp = 0;
          e.group = static_cast<uint8_t>(g.gi);
          e.so = static_cast<uint8_t>(D.fifo_step[slot] - s0);
          B.evb[o + nq + __popc(bal & mcg_lanemask_lt())] = e;
        }
        nq += __popc(bal);
        if (bal != MCG_FULL) break;
      }
      o += nq;
      __syncwarp();
      if (lane == 0) g.f_head += nq;
      __syncwarp();
    }
  }
  if (nseg > 1 && lane == 0) {  // several groups due: pop in (step, seq) order
    for (;;) {
      int best = -1;
      int64_t bst = 0;
      uint64_t bseq = 0;
      for (int q = 0; q < X.n_stc_seg; ++q) {
        const McgSegSm& g = B.seg[k * A.n_stc_max + q];
        if (g.fifo < 0 || g.f_head >= g.f_tail) continue;
        const int64_t slot = g.f_base + mcg_mod(g.f_head, g.f_cap);
        const int64_t st = D.fifo_step[slot];
        if (st >= s1) continue;
        const uint64_t seq = D.fifo_si[slot] >> 32;
        if (best < 0 || st < bst || (st == bst && seq < bseq)) {
          best = q;
          bst = st;
          bseq = seq;
        }
      }
      if (best < 0) break;
      McgSegSm& g = B.seg[k * A.n_stc_max + best];
      const int64_t slot = g.f_base + mcg_mod(g.f_head, g.f_cap);
      McgEvSm e;
      e.w = 0.0;
      e.inst = uint32_t(D.fifo_si[slot] & 0xffffffffu);
          e.src = 0;
          e.pad = 0;
      e.comp = 0;
      e.group = static_cast<uint8_t>(g.gi);
      e.so = static_cast<uint8_t>(bst - s0);
      B.evb[o++] = e;
      ++g.f_head;
    }
  }
  __syncwarp();
  if (lane == 0) {
    X.ev_cur = beg;
    X.ev_end = beg + nd;
    X.in_cur = beg + nd;
    X.in_end = beg + nd + ni;
    X.cur += nd;
    X.nk = (X.cur < X.end) ? pend[X.cur] : ~0ull;
    X.staged = 1;
  }
  __syncwarp();
  return true;
}

// static part of every chain-sweep lane of batch b (mcg_ph_solve): lane t is
// (cell t / 2S1, system (t mod 2S1) / 2, side t mod 2); the per-step part
// (refractory / conductance state, currents, production) is added each step
__device__ void mcg_lanes_init(const McgDev& D, const McgBatchArgs& A, const McgBatchSm& B,
                               int nc) {
  const int S1 = 1 + D.sp_max, m = D.smem_n;
  for (int t = threadIdx.x; t < A.nch_max; t += blockDim.x) {
    int* L = B.lanes + t * MCG_LANE_INTS;
    const int k = t / (2 * S1), rem = t - k * 2 * S1, sys = rem >> 1;
    for (int i = 0; i < MCG_LANE_INTS; ++i) L[i] = 0;
    L[0] = -1;
    if (k >= nc) continue;
    const McgKind& K = B.kc[k];
    const McgCellSm& X = B.cs[k];
    const bool ok = K.ch_lp > 0 && K.n <= m &&
                    (sys == 0 ? (K.dyn == MCG_DYN_LIF && K.v_const)
                              : (sys - 1 < K.n_species && K.n > 1 && K.sp_const));
    const int n = K.n, P = 2 * K.ch_lp + 1;
    const int cho = B.ksm_o + X.kb + mcg_kind_chain_off(n, K.n_species);
    L[0] = k;
    L[1] = sys;
    L[2] = rem & 1;
    L[3] = K.ch_lp;
    L[4] = B.chs_o + k * A.ch_stride + sys * A.ch_pmax;
    L[5] = 2 * cho;
    L[6] = cho + (P + 1) / 2 + sys * 6 * P;
    L[7] = k * A.comp_stride + (sys == 0 ? 0 : m + (sys - 1) * n);
    L[8] = (ok ? 1 : 0) | (K.ch_afirst ? 2 : 0);
    L[9] = (sys > 0 && sys - 1 == K.prp_idx) ? K.prp_comp : -1;
  }
}

// kind blocks currently staged (offset, kind) per slot, kept across the
// batches of one launch (reset at launch start)
#define MCG_KSLOTS 16
__shared__ int mcg_kslot_off[MCG_KSLOTS];
__shared__ long long mcg_kslot_arr[MCG_KSLOTS];

// ---- staging: metadata, kind constants, compartment state of batch b
__device__ void mcg_batch_enter(const McgDev& D, const McgBatchArgs& A, int32_t b) {
  const McgBatchSm B = mcg_batch_sm(A);
  const int tid = threadIdx.x, T = blockDim.x;
  const int c0 = b * A.cells_per_cta;
  const int nc = min(A.cells_per_cta, D.n_cells - c0);
  const int m = D.smem_n;
  if (tid < nc) {
    const int c = c0 + tid;
    McgCellSm& X = B.cs[tid];
    B.kc[tid] = D.kinds[D.cell_kind[c]];
    const McgKind& K = B.kc[tid];
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
    X.lif = (K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT) ? 1 : 0;
    X.noise = (X.lif && K.has_bg && K.sig_bg != 0.0) ? 1 : 0;
    const int64_t cg0 = D.cg_off[c];
    int ns = 0, tot = 0, act = 0;
    for (int gi = 0; gi < K.n_groups; ++gi) {
      const McgCellGroup& G = D.cgs[cg0 + gi];
      const McgSpec& S = D.specs[G.spec];
      if (S.kind == MCG_SYN_STATIC_COND || S.kind == MCG_SYN_STDP_COND ||
          S.kind == MCG_SYN_STATIC_CURRENT || S.kind == MCG_SYN_HOMEO_CURRENT)
        act = 1;
      if (S.kind != MCG_SYN_STC_CHARGE || ns >= A.n_stc_max) continue;
      McgSegSm& g = B.seg[tid * A.n_stc_max + ns];
      g.inst = G.inst;
      g.gi = gi;
      g.size = G.size;
      g.spec = G.spec;
      g.comp = S.comp;
      g.start = tot;
      g.vol = D.k_volume[K.arr + S.comp];
      g.rvol = D.k_rvol[K.arr + S.comp];
      g.cf = D.k_cf[K.arr + S.comp];
      g.ca_delay = S.ca_delay;
      g.h0 = S.h0;
      g.cpre_s = S.cpre_s;
      g.late = K.prp_idx >= 0 ? 1 : 0;
      g.prp_sm = (K.prp_idx >= 0 && K.n <= m)
                     ? tid * A.comp_stride + m + K.prp_idx * K.n + S.comp : -1;
      g.fifo = G.fifo;
      if (G.fifo >= 0) {
        g.f_base = D.fifos[G.fifo].base;
        g.f_cap = D.fifos[G.fifo].cap;
      }
      tot += G.size;
      ++ns;
    }
    X.has_act = act;
    // staged delivery: static-charge and STC groups only, every STC group's
    // calcium delay at least an epoch (its queue entries due in an epoch exist
    // at the epoch's start), step offsets within an epoch fit a byte
    {
      int fast = (A.ev_cap > 0 && K.n <= m && K.n_groups <= 8 && D.ctl[2] <= 255) ? 1 : 0;
      for (int gi = 0; fast && gi < K.n_groups; ++gi) {
        const McgSpec& S = D.specs[D.cgs[cg0 + gi].spec];
        X.gk[gi] = static_cast<uint8_t>(S.kind);
        X.gseg[gi] = -1;
        if (S.kind == MCG_SYN_STC_CHARGE) {
          for (int q = 0; q < ns; ++q)
            if (B.seg[tid * A.n_stc_max + q].gi == gi) X.gseg[gi] = static_cast<int8_t>(q);
          if (X.gseg[gi] < 0 || S.ca_delay < D.ctl[2] || D.cgs[cg0 + gi].fifo < 0) fast = 0;
        } else if (S.kind != MCG_SYN_STATIC_CHARGE) {
          fast = 0;
        }
      }
      X.fast = fast;
      X.staged = 0;
    }
    X.n_stc_seg = ns;
    X.stc_n = tot;
    X.hh_n = (K.dyn == MCG_DYN_HH) ? K.n : 0;
    X.fifo_next = (K.n_stc_groups > 0) ? mcg_fifo_next(D, K, cg0) : INT64_MAX;
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0, hacc = 0, kacc = 0, nk = 0;
    long long karr[MCG_KSLOTS];
    int kbs[MCG_KSLOTS];
    for (int k = 0; k < nc; ++k) {
      B.cs[k].stc_off = acc;
      acc += B.cs[k].stc_n;
      B.cs[k].hh_off = hacc;
      hacc += B.cs[k].hh_n;
      // one staged copy per distinct kind of the batch
      B.cs[k].kb = -1;
      if (B.cs[k].n <= m) {
        for (int q = 0; q < nk; ++q)  // the batch's distinct kinds so far
          if (karr[q] == B.kc[k].arr) {
            B.cs[k].kb = kbs[q];
            break;
          }
        if (B.cs[k].kb < 0) {
          B.cs[k].kb = kacc;
          if (nk < MCG_KSLOTS) {
            karr[nk] = B.kc[k].arr;
            kbs[nk++] = kacc;
          }
          kacc += mcg_kind_block_doubles(B.kc[k].n, B.kc[k].n_species, B.kc[k].ch_lp);
        }
      }
    }
  }
  __syncthreads();
  // a kind block already holding the same kind (an earlier batch of this
  // launch, same offset) is not staged again
  int slot = 0;
  for (int k = 0; k < nc; ++k) {
    if (B.cs[k].kb < 0) continue;
    bool first = true;
    for (int q = 0; q < k; ++q)
      if (B.cs[q].kb == B.cs[k].kb) first = false;
    if (!first) continue;
    const bool have = slot < MCG_KSLOTS && mcg_kslot_off[slot] == B.cs[k].kb &&
                      mcg_kslot_arr[slot] == B.kc[k].arr;
    if (!have) mcg_kind_stage(D, B.kc[k], B.ksm + B.cs[k].kb);
    ++slot;
  }
  __syncthreads();
  if (tid == 0) {  // record what the kind blocks now hold
    int sl = 0;
    for (int k = 0; k < nc && sl < MCG_KSLOTS; ++k) {
      if (B.cs[k].kb < 0) continue;
      bool first = true;
      for (int q = 0; q < k; ++q)
        if (B.cs[q].kb == B.cs[k].kb) first = false;
      if (!first) continue;
      mcg_kslot_off[sl] = B.cs[k].kb;
      mcg_kslot_arr[sl] = B.kc[k].arr;
      ++sl;
    }
    for (; sl < MCG_KSLOTS; ++sl) mcg_kslot_off[sl] = -1;
  }
  // STC instance locator: slot f -> (cell, group), warp per cell
  for (int k = tid >> 5; k < nc; k += T >> 5) {
    const McgCellSm& X = B.cs[k];
    for (int q = 0; q < X.n_stc_seg; ++q) {
      const McgSegSm& g = B.seg[k * A.n_stc_max + q];
      for (int i = tid & 31; i < g.size; i += 32)
        B.floc[X.stc_off + g.start + i] = (uint32_t(k) << 16) | uint32_t(q);
    }
  }
  __syncthreads();
  if (A.stc_sm) {
    const int stc_total = B.cs[nc - 1].stc_off + B.cs[nc - 1].stc_n;
    const int S4 = A.stc_max;
    for (int f = tid; f < stc_total; f += T) {
      const uint32_t loc = B.floc[f];
      const int k = int(loc >> 16);
      const McgSegSm& g = B.seg[k * A.n_stc_max + int(loc & 0xffffu)];
      const int64_t j = g.inst + (f - B.cs[k].stc_off - g.start);
      B.stc[f] = D.i_stc_h[j];
      B.stc[S4 + f] = D.i_stc_z[j];
      B.stc[2 * S4 + f] = D.i_stc_c[j];
      B.stc[3 * S4 + f] = D.i_sps_abs[j];
    }
  }
  // compartment state (cells that fit; the rest use global memory), one flat
  // loop over (cell, V | species | HH slot) so all loads are in flight together
  {
    const int per = (1 + D.sp_max + 3) * m;
    for (int idx = tid; idx < nc * per; idx += T) {
      const int k = idx / per, r = idx - k * per;
      const McgKind& K = B.kc[k];
      const int n = K.n;
      if (n > m) continue;
      const int a = r / m, i = r - a * m;  // array a, compartment i
      if (i >= n) continue;
      double* base = mcg_comp_block(A, B, k);
      const int c = c0 + k;
      if (a == 0) {
        base[i] = D.v[D.comp_off[c] + i];
      } else if (a <= D.sp_max) {
        if (a - 1 < K.n_species) base[m + (a - 1) * n + i] = D.species[D.sp_off[c] + (a - 1) * n + i];
      } else if (K.dyn == MCG_DYN_HH) {
        const int h = a - 1 - D.sp_max;  // 0: m, 1: h, 2: n
        const double* src = h == 0 ? D.hh_m : (h == 1 ? D.hh_h : D.hh_n);
        base[(2 + D.sp_max + h) * m + i] = src[D.comp_off[c] + i];
      }
    }
  }
  if (A.nch_max > 0) mcg_lanes_init(D, A, B, nc);
  __syncthreads();
}

// ---- write-back of batch b (state that lives in shared memory while staged)
__device__ void mcg_batch_exit(const McgDev& D, const McgBatchArgs& A, int32_t b) {
  const McgBatchSm B = mcg_batch_sm(A);
  const int tid = threadIdx.x, T = blockDim.x;
  const int c0 = b * A.cells_per_cta;
  const int nc = min(A.cells_per_cta, D.n_cells - c0);
  const int m = D.smem_n;
  for (int k = 0; k < nc; ++k) {
    const int c = c0 + k;
    const McgKind& K = B.kc[k];
    if (K.n > m) continue;
    const double* base = mcg_comp_block(A, B, k);
    const int n = K.n;
    const int64_t co = D.comp_off[c];
    for (int i = tid; i < n; i += T) D.v[co + i] = base[i];
    double* gs = D.species + D.sp_off[c];
    for (int i = tid; i < K.n_species * n; i += T) gs[i] = base[m + i];
    if (K.dyn == MCG_DYN_HH)
      for (int i = tid; i < n; i += T) {
        D.hh_m[co + i] = base[(2 + D.sp_max) * m + i];
        D.hh_h[co + i] = base[(3 + D.sp_max) * m + i];
        D.hh_n[co + i] = base[(4 + D.sp_max) * m + i];
      }
  }
  if (A.stc_sm) {
    const int stc_total = B.cs[nc - 1].stc_off + B.cs[nc - 1].stc_n;
    const int S4 = A.stc_max;
    for (int f = tid; f < stc_total; f += T) {
      const uint32_t loc = B.floc[f];
      const int k = int(loc >> 16);
      const McgSegSm& g = B.seg[k * A.n_stc_max + int(loc & 0xffffu)];
      const int64_t j = g.inst + (f - B.cs[k].stc_off - g.start);
      D.i_stc_h[j] = B.stc[f];
      D.i_stc_z[j] = B.stc[S4 + f];
      D.i_stc_c[j] = B.stc[2 * S4 + f];
      D.i_sps_abs[j] = B.stc[3 * S4 + f];
    }
  }
  if (tid < nc) {
    const int c = c0 + tid;
    McgCellSm& X = B.cs[tid];
    if (X.staged) mcg_unstage(D, A, B, tid, c);
    if (X.ndel) atomicAdd(D.delivered, X.ndel);
    X.ndel = 0;
    D.refr_until[c] = X.refr;
    D.det_prev[c] = X.det_prev;
    D.armed[c] = X.armed;
  }
  __syncthreads();
}

// ---- E2: membrane and species systems of batch b (one step); out of line so
// its register allocation does not compete with the rest of the step loop
// the general V solves that a whole warp takes (mcg_solve_tree_warp): the
// systems mcg_ph_solve would otherwise give mcg_solve_tree_fast
__device__ __forceinline__ bool mcg_tree_warp_item(const McgKind& K, const McgCellSm& X, int sys) {
  if (sys != 0 || K.gch_n <= 0) return false;
  if (K.dyn == MCG_DYN_HH) return true;
  if (K.dyn == MCG_DYN_LIF) return !X.refractory && !(!X.has_gsyn && K.v_const);
  return false;
}

__device__ __noinline__ void mcg_ph_solve(const McgDev& D, const McgBatchArgs& A, int32_t b) {
  const McgBatchSm B = mcg_batch_sm(A);
  const int tid = threadIdx.x, T = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int c0 = b * A.cells_per_cta;
  const int nc = min(A.cells_per_cta, D.n_cells - c0);
  const int S1 = 1 + D.sp_max;
  const int m = D.smem_n;
  McgCellSm* cs = B.cs;
  const McgKind* kc = B.kc;
  // ---- E2a. chain-scheduled constant systems (mcg_sweep.cuh), one lane per
  // (cell, system, chain) on threads [0, split), beside the other systems
  // (thread per (cell, system)) on [split, T)
  const int nch = (A.ch_stride > 0) ? ((2 * S1 * nc + 31) & ~31) : 0;
  // LIF-only launches (A.lean): the other systems are point cells, one warp suffices
  const int split = nch > 0 ? (A.lean ? min(nch, T - 32) : min(256, T / 2)) : 0;
  // the other systems, one thread per (cell, system), spread over warps
  // first (item w + W l on lane l of the w-th warp of the range): a system's
  // solve is a serial chain whose branches and slow paths diverge between
  // cells, so items on separate warps run concurrently instead of taking
  // turns in one warp
  const int wr0 = split >> 5, nwr = (T - split) >> 5;
  // few items per warp: the general tree solves take a warp each instead of
  // a lane (the branches of a tree side by side)
  const bool warp_tree = nc * S1 <= 2 * nwr;
  if (tid < split) {
    for (int t = tid; t < nch; t += split) {
      McgChainLane L{};
      const int* LD = B.lanes + t * MCG_LANE_INTS;  // static part (mcg_lanes_init)
      const int k = LD[0];
      if (k >= 0 && (LD[8] & 1)) {
        const McgCellSm& X = cs[k];
        const int sys = LD[1];
        L.on = (sys != 0 || (!X.refractory && !X.has_gsyn)) ? 1 : 0;
        L.side = LD[2];
        L.lp = LD[3];
        L.r2c = LD[4];
        L.idx = LD[5];
        L.fc = LD[6];
        L.x = LD[7];
        L.a_first = (LD[8] >> 1) & 1;
        L.v = sys == 0;
        // right-hand sides (engine.cpp:683 / 746-748): V: g_leak_rhs + 0.0 +
        // rhs_current (if any current); species: production at the
        // synthesis compartment
        L.rc = (sys == 0 && X.has_current) ? k * A.comp_stride + (1 + D.sp_max) * m : -1;
        L.pc = (LD[9] >= 0 && X.prod != 0.0) ? LD[9] : -1;
        L.prod = X.prod;
      }
      MCG_PH(19);
      mcg_chain_lane(L);
      MCG_PH(20);
    }
  } else
  for (int t = (warp - wr0) + nwr * lane; split <= tid && t < nc * S1; t += nwr * 32) {
    const int k = t / S1, sys = t - k * S1;
    const int c = c0 + k;
    const McgCellSm& X = cs[k];
    const McgKind& K = kc[k];
    if (mcg_chain_ok(K, X, sys, m)) continue;
    if (warp_tree && mcg_tree_warp_item(K, X, sys)) continue;  // below
    const int n = K.n;
    const bool in_sm = n <= m;
    const McgCellMem M = mcg_cell_mem(D, K, c, in_sm ? mcg_comp_block(A, B, k) : nullptr);
    const McgKindSm KS = mcg_kind_consts(D, K, B.ksm, X.kb);
    const bool refractory = X.refractory;
    const bool hg = X.has_gsyn, hc = X.has_current;
    const int q = sys - 1;
    // constant-diagonal systems (LIF-cable V without conductances, species)
    // share one instruction stream across all cells and systems
    const bool v_sys = sys == 0 && K.dyn == MCG_DYN_LIF && !refractory && !hg && K.v_const;
    const bool s_sys = sys > 0 && q < K.n_species && n > 1 && K.sp_const;
    bool ok = true;
    if ((v_sys || s_sys) && in_sm) {
      const McgKindOff KO = mcg_kind_off(B.ksm_o + X.kb, n, K.n_species);
      const int bo = k * A.comp_stride, r2o = bo + (8 + D.sp_max) * m;
      // one call for V and species (operands selected first), so lanes with
      // different systems run the sweep in lockstep instead of serialized
      const int qn = v_sys ? 0 : q * n;
      const int x = v_sys ? bo : bo + m + qn, r2 = v_sys ? r2o : r2o + n + qn;
      // right-hand side (engine.cpp:683 / 746-748):
      //   V:       r2 = cap*v + (g_leak_rhs + 0.0 + (has_current ? rhs_cur : 0.0))
      //   species: r2 = cap*c + (prod at the synthesis compartment, else 0.0)
      const int pc = (!v_sys && q == K.prp_idx && X.prod != 0.0) ? K.prp_comp : -1;
      mcg_rhs_sm(n, v_sys ? KO.cap : KO.sp_cap + qn, x, r2, v_sys, KO.glr,
                 hc ? bo + (1 + D.sp_max) * m : -1, pc, X.prod);
      mcg_sweep_const_sm(n, KO.par, (v_sys ? KO.ax : KO.sp_coup) + qn,
                         (v_sys ? KO.vf : KO.sp_f) + qn, (v_sys ? KO.vd : KO.sp_d) + qn,
                         (v_sys ? KO.vr : KO.sp_r) + qn, x, r2);
    } else if (v_sys || s_sys) {
      double* x = v_sys ? M.V : M.SP + int64_t(q) * n;
      const int qq = v_sys ? 0 : q;
      const double* coup = v_sys ? KS.ax : KS.sp_coup + qq * n;
      const double* f = v_sys ? KS.vf : KS.sp_f + qq * n;
      const double* d = v_sys ? KS.vd : KS.sp_d + qq * n;
      const double* y = v_sys ? KS.vr : KS.sp_r + qq * n;
      double* r2 = M.r2 + int64_t(v_sys ? 0 : 1 + q) * n;
      {
        const double* cap = v_sys ? KS.cap : KS.sp_cap + qq * n;
        const int pc = (!v_sys && q == K.prp_idx && X.prod != 0.0) ? K.prp_comp : -1;
        for (int i = 0; i < n; ++i) {
          const double rhs = v_sys ? (KS.glr[i] + 0.0 + (hc ? M.rhs_cur[i] : 0.0))
                                   : (i == pc ? X.prod : 0.0);
          r2[i] = cap[i] * x[i] + rhs;
        }
      }
      mcg_sweep_const(n, KS.par, coup, f, d, y, x, r2);
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
        ok = mcg_solve_tree_fast(n, KS.par, KS.cap, M.gsyn, KS.ax, M.gsyn_rhs, M.V, M.diag, M.r2);
      } else if (K.dyn == MCG_DYN_HH) {
        // M.gsyn is rebuilt every step before the solve (phase E1 / B), so
        // the solve may keep its reciprocals there
        ok = mcg_solve_tree_fast(n, KS.par, KS.cap, M.gsyn, KS.ax, M.gsyn_rhs, M.V, M.diag, M.r2);
      }
      // singular species systems need the full solver's scratch: run them
      // here, after V, in species order (never happens for valid recipes)
      if (n > 1 && !K.sp_const)
        for (int p = 0; p < K.n_species; ++p)
          ok &= mcg_species_sys(n, p == K.prp_idx, K.prp_comp, X.prod, KS.sp_cap + p * n,
                                KS.sp_gs + p * n, KS.sp_coup + p * n, KS.par,
                                M.SP + int64_t(p) * n, M.r2 + int64_t(1 + p) * n, M.diag,
                                D.s_rhs + D.comp_off[c]);
    } else if (q < K.n_species && n == 1) {
      mcg_species_sys(1, q == K.prp_idx, K.prp_comp, X.prod, KS.sp_cap + q, KS.sp_gs + q,
                      KS.sp_coup + q, KS.par, M.SP + q, M.r2, M.diag, M.rhs_cur);
    }
    if (!ok) atomicOr(D.err, MCG_ERR_FLAG_SINGULAR);
  }
  if (warp_tree && split <= tid) {
    for (int t = warp - wr0; t < nc * S1; t += nwr) {  // warp-uniform items
      const int k = t / S1, sys = t - k * S1;
      const McgCellSm& X = cs[k];
      const McgKind& K = kc[k];
      if (mcg_chain_ok(K, X, sys, m) || !mcg_tree_warp_item(K, X, sys)) continue;
      const int c = c0 + k;
      const int n = K.n;
      const McgCellMem M = mcg_cell_mem(D, K, c, n <= m ? mcg_comp_block(A, B, k) : nullptr);
      const McgKindSm KS = mcg_kind_consts(D, K, B.ksm, X.kb);
      if (K.dyn == MCG_DYN_LIF) {
        const bool hg = X.has_gsyn, hc = X.has_current;
        for (int i = lane; i < n; i += 32) {
          const double gs = KS.gl[i] + (hg ? M.gsyn[i] : 0.0);
          const double rr = KS.glr[i] + (hg ? M.gsyn_rhs[i] : 0.0) + (hc ? M.rhs_cur[i] : 0.0);
          M.gsyn[i] = gs;
          M.gsyn_rhs[i] = rr;
        }
        __syncwarp();
      }
      bool ok = mcg_solve_tree_warp(D.k_ch_idx + K.gch_arr, KS.par, KS.cap, M.gsyn, KS.ax, M.gsyn_rhs, M.V,
                                    M.diag, M.r2, lane);
      if (lane == 0) {
        if (n > 1 && !K.sp_const)
          for (int p = 0; p < K.n_species; ++p)
            ok &= mcg_species_sys(n, p == K.prp_idx, K.prp_comp, X.prod, KS.sp_cap + p * n,
                                  KS.sp_gs + p * n, KS.sp_coup + p * n, KS.par,
                                  M.SP + int64_t(p) * n, M.r2 + int64_t(1 + p) * n, M.diag,
                                  D.s_rhs + D.comp_off[c]);
        if (!ok) atomicOr(D.err, MCG_ERR_FLAG_SINGULAR);
      }
      __syncwarp();
    }
  }
}

// ---- one epoch [s0, s1) of the staged batch b
__device__ void mcg_batch_epoch(const McgDev& D, const McgBatchArgs& A, int32_t b, int32_t j,
                                int64_t s0, int64_t s1) {
  const McgBatchSm B = mcg_batch_sm(A);
  const int tid = threadIdx.x;
  // the owner thread of cell k (the cells' serial chains: delivery, folds,
  // detection) is lane k / W of warp k % W: owners on different warps run
  // concurrently instead of taking turns inside one warp
  const int ko = (threadIdx.x >> 5) + (blockDim.x >> 5) * (threadIdx.x & 31);
  const int T = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = T >> 5;
  const int c0 = b * A.cells_per_cta;
  const int nc = min(A.cells_per_cta, D.n_cells - c0);
  const int m = D.smem_n;
  McgCellSm* cs = B.cs;
  const McgKind* kc = B.kc;
  const McgSpec* specs = A.n_specs_sm > 0 ? B.spec : D.specs;

  // inbox merge, warp per cell (the reference's per-epoch inbox sort), and
  // the staging of the epoch's due events
  __shared__ int s_ev_top;
  if (tid == 0) s_ev_top = 0;
  __syncthreads();
  for (int k = warp; k < nc; k += nwarps) {
    const int c = c0 + k;
    const int nin = D.inc_n[c];
    McgCellSm& X = cs[k];
    if (X.fast && X.cur >= X.end && nin <= 32) {
      // common case: nothing pending from earlier epochs and a small inbox,
      // sorted in registers and staged from them (pend gets the same keys)
      uint64_t key = ~0ull;
      int nd = 0;
      if (nin > 0) {
        const uint64_t* in = D.inc + int64_t(c) * D.inc_cap;
        key = mcg_warp_sort_reg(lane < nin ? in[lane] : ~0ull, lane, nin);
        const uint64_t lim = uint64_t(s1) << D.rank_bits;
        nd = __popc(__ballot_sync(MCG_FULL, lane < nin && key < lim));
        uint64_t* out = D.pend + (int64_t(c) * 2 + (1 - X.sel)) * D.pend_cap;
        if (lane < nin) out[lane] = key;
        __syncwarp();
        if (lane == 0) {
          X.end = nin;
          X.cur = 0;
          X.sel = 1 - X.sel;
        }
        __syncwarp();
      }
      mcg_stage_events(D, A, B, k, c, s0, s1, lane, &s_ev_top, true, key, nd);
      if (lane == 0) X.nsp = 0;
      continue;
    }
    if (nin > 0) {
      uint64_t* in = D.inc + int64_t(c) * D.inc_cap;
      if (nin > 1) mcg_warp_sort(in, nin, lane);
      __syncwarp();
      const uint64_t* pold = D.pend + (int64_t(c) * 2 + X.sel) * D.pend_cap;
      uint64_t* out = D.pend + (int64_t(c) * 2 + (1 - X.sel)) * D.pend_cap;
      if (X.cur >= X.end) {  // nothing pending from earlier epochs: copy
        for (int i = lane; i < nin; i += 32) out[i] = in[i];
        __syncwarp();
        if (lane == 0) {
          X.end = nin;
          X.cur = 0;
          X.sel = 1 - X.sel;
        }
      } else if (lane == 0) {
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
    if (X.fast) mcg_stage_events(D, A, B, k, c, s0, s1, lane, &s_ev_top);
    if (lane == 0) {
      if (!X.fast) X.nk = (X.cur < X.end) ? D.pend[(int64_t(c) * 2 + X.sel) * D.pend_cap + X.cur] : ~0ull;
      X.nsp = 0;
    }
  }
  __syncthreads();
  MCG_PH(10);
  const int stc_total = cs[nc - 1].stc_off + cs[nc - 1].stc_n;
  const int hh_total = cs[nc - 1].hh_off + cs[nc - 1].hh_n;
  const int stc_rounds = (stc_total + T - 1) / T;

  const uint64_t rank_mask = (1ull << D.rank_bits) - 1;
  for (int64_t s = s0; s < s1; ++s) {
    const int64_t so = s - s0;
    // background-noise draws for the next 32 steps of every noisy cell, one
    // Box-Muller pair per thread (normal_for, rng.cpp:67-78: step n uses pair
    // n >> 1 of threefry block n >> 2, element n & 1)
    if ((so & 31) == 0) {
      const int64_t w1 = min(s + 32, s1);
      for (int q = tid; q < nc * 17; q += T) {
        const int k = q / 17, pp = q - k * 17;
        if (!cs[k].noise) continue;
        const uint64_t pr = (uint64_t(s) >> 1) + uint64_t(pp);
        const int64_t n0 = int64_t(pr * 2);
        if (n0 + 1 < s || n0 >= w1) continue;
        const mcg_key key = mcg_make_key(D.seed, D.gid0 + uint32_t(c0 + k), 1, 0);
        uint64_t x[4];
        mcg_threefry(&key, pr >> 1, x);
        const unsigned h = unsigned(pr & 1u);
        const double u1 = ((double)(x[2 * h] >> 11) + 1.0) * MCG_2POW_M53;
        const double u2 = (double)(x[2 * h + 1] >> 11) * MCG_2POW_M53;
        double z0, z1;
        mcg_normal_pair(u1, u2, &z0, &z1);
        if (n0 >= s) B.nbuf[k * 32 + int(n0 - s)] = z0;
        if (n0 + 1 < w1) B.nbuf[k * 32 + int(n0 + 1 - s)] = z1;
      }
      __syncthreads();
      MCG_PH(0);
    }
    // ---- A. delivery (owner thread): inbox, then internal (engine.cpp:549-560)
    if (ko < nc) {
      const int c = c0 + ko;
      McgCellSm& X = cs[ko];
      const McgKind& K = kc[ko];
      const bool refractory = X.lif && s < X.refr;
      X.refractory = refractory;
      double* V = (K.n <= m) ? mcg_comp_block(A, B, ko) : D.v + D.comp_off[c];
      const int64_t cg0 = D.cg_off[c];
      const bool trace = (A.dbg >> 8) == c + 1 && s >= A.dbg_s && s <= A.dbg_s + 5;
      if (trace)
        printf("[k_batch] cell %d s %lld staged %d ev [%d,%d) in [%d,%d) V0 %.17g\n", c, (long long)s, X.staged,
               X.ev_cur, X.ev_end, X.in_cur, X.in_end, V[0]);
      if (X.staged) {
        // staged delivery (mcg_stage_events): network events, then delayed calcium
        const int S4 = A.stc_max;
        int e = X.ev_cur;
        while (e < X.ev_end && int(B.evb[e].so) == int(so)) {
          const McgEvSm E = B.evb[e];
          if (trace) printf("[k_batch]   ev so %d grp %d inst %u w %.17g\n", int(E.so), E.group, E.inst & 0x7fffffffu, E.w);
          const uint32_t inst = E.inst & 0x7fffffffu;
          if (X.gk[E.group] == MCG_SYN_STATIC_CHARGE) {
            if (!refractory && (E.inst >> 31)) V[E.comp] += E.w;  // w * cf[comp]
          } else {  // stc_charge, engine.cpp:493-510
            McgSegSm& g = B.seg[ko * A.n_stc_max + X.gseg[E.group]];
            if (g.f_tail - g.f_head >= g.f_cap) {
              atomicOr(D.err, MCG_ERR_FLAG_FIFO);
            } else {
              const int64_t slot = g.f_base + mcg_mod(g.f_tail, g.f_cap);
              D.fifo_step[slot] = s + g.ca_delay;
              D.fifo_si[slot] = (uint64_t(X.iseq) << 32) | uint64_t(inst);
              D.fifo_src[slot] = E.src;
              D.fifo_w[slot] = E.w;
              ++g.f_tail;
            }
            ++X.iseq;
            if (!refractory) {  // stc_total_weight: h + h0 * z
              double tw;
              if (A.stc_sm) {
                const int sl = X.stc_off + g.start + int(inst);
                tw = B.stc[sl] + g.h0 * B.stc[S4 + sl];
              } else {
                const int64_t j = g.inst + inst;
                tw = D.i_stc_h[j] + g.h0 * D.i_stc_z[j];
              }
              V[g.comp] += tw * E.w * g.cf;
            }
          }
          ++e;
          ++X.ndel;
        }
        X.ev_cur = e;
        int q = X.in_cur;
        while (q < X.in_end && int(B.evb[q].so) == int(so)) {
          const McgEvSm E = B.evb[q];
          const McgSegSm& g = B.seg[ko * A.n_stc_max + X.gseg[E.group]];
          if (A.stc_sm) B.stc[2 * S4 + X.stc_off + g.start + int(E.inst)] += g.cpre_s;
          else D.i_stc_c[g.inst + E.inst] += g.cpre_s;
          ++q;
        }
        X.in_cur = q;
      } else {
        uint64_t key = X.nk;
        if (int64_t(key >> D.rank_bits) <= s) {
          const uint64_t* pend = D.pend + (int64_t(c) * 2 + X.sel) * D.pend_cap;
          int cur = X.cur;
          while (int64_t(key >> D.rank_bits) <= s) {
            const int64_t r = int64_t(key & rank_mask);
            const int32_t grp = D.e_group[r];
            mcg_apply_event(D, K, c, cg0, V, grp, D.e_inst[r], D.e_weight[r], 0, refractory, s,
                            mcg_stc_ref(A, B, ko, grp), D.e_src[r]);
            ++cur;
            ++X.ndel;
            key = (cur < X.end) ? pend[cur] : ~0ull;
          }
          X.cur = cur;
          X.nk = key;
          // STC events queue delayed calcium (apply_event, engine.cpp:497-503)
          if (K.n_stc_groups > 0) X.fifo_next = mcg_fifo_next(D, K, cg0);
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
                const int64_t slot = F.base + mcg_mod(F.head, F.cap);
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
            const uint64_t si = D.fifo_si[F.base + mcg_mod(F.head, F.cap)];
            ++F.head;
            mcg_apply_event(D, K, c, cg0, V, best, uint32_t(si & 0xffffffffu), 0.0, 1,
                            refractory, s, mcg_stc_ref(A, B, ko, best));
          }
          X.fifo_next = mcg_fifo_next(D, K, cg0);
        }
      }
      X.has_gsyn = 0;
      X.has_current = 0;
      double* rc = (K.n <= m) ? V + (1 + D.sp_max) * m : D.s_rhs_cur + D.comp_off[c];
      const int nr = K.n > 1 ? K.n : 1;
      for (int i = 0; i < nr; ++i) rc[i] = 0.0;
    }
    MCG_PH(15);
    __syncthreads();
    MCG_PH(1);

    // ---- B. active-list kernels (warp per cell, ordered folds, engine.cpp:578-616)
    // One staged cell with long active lists (a neuron with many plastic
    // inputs, A.act_max > 0): every thread decays a share of the kernels, all
    // its loads in flight together, and leaves the kept value (or -0.0) and the
    // instance index in shared memory; warp 0 then compacts the lists and
    // folds them in list order while the other warps run phase C.  Each
    // group's entries start at a multiple of 32.
    const bool pb = A.act_max > 0 && nc == 1 && cs[0].has_act;
    if (pb) {
      const McgKind& K = kc[0];
      const int64_t cg0 = D.cg_off[c0];
      int off = 0;
      for (int gi = 0; gi < K.n_groups; ++gi) {
        McgCellGroup* G = &D.cgs[cg0 + gi];
        const McgSpec& S = specs[G->spec];
        const int na = G->active_n;
        const bool cond = S.kind == MCG_SYN_STATIC_COND || S.kind == MCG_SYN_STDP_COND;
        if (na == 0 || !(cond || S.kind == MCG_SYN_STATIC_CURRENT || S.kind == MCG_SYN_HOMEO_CURRENT))
          continue;
        const int64_t base = G->inst;
        const double f = S.f_decay;
        for (int a0 = 0; a0 < na; a0 += 4 * T) {
          int ii[4];
          double kk[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int a = a0 + u * T + tid;
            ii[u] = a < na ? D.i_active[base + a] : -1;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) kk[u] = ii[u] >= 0 ? D.i_kernel[base + ii[u]] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (ii[u] < 0) continue;
            double kv = kk[u] * f;
            if (cond ? (kv < 1e-30) : (fabs(kv) < 1e-30)) kv = 0.0;
            D.i_kernel[base + ii[u]] = kv;
            const int a = off + a0 + u * T + tid;
            B.abuf[a] = kv != 0.0 ? kv : -0.0;
            B.aidx[a] = ii[u];
          }
        }
        off += (na + 31) & ~31;
      }
      __syncthreads();
      if (warp == 0) {
        const McgCellMem M = mcg_cell_mem(D, K, c0, K.n <= m ? mcg_comp_block(A, B, 0) : nullptr);
        bool hg = false, hc = false;
        off = 0;
        for (int gi = 0; gi < K.n_groups; ++gi) {
          McgCellGroup* G = &D.cgs[cg0 + gi];
          const McgSpec& S = specs[G->spec];
          const int na = G->active_n;
          const bool cond = S.kind == MCG_SYN_STATIC_COND || S.kind == MCG_SYN_STDP_COND;
          if (na == 0 || !(cond || S.kind == MCG_SYN_STATIC_CURRENT || S.kind == MCG_SYN_HOMEO_CURRENT))
            continue;
          if (cond && !hg) {
            for (int i = lane; i < K.n; i += 32) {
              M.gsyn[i] = 0.0;
              M.gsyn_rhs[i] = 0.0;
            }
            hg = true;
            __syncwarp();
          }
          const int64_t base = G->inst;
          const double* v = B.abuf + off;
          // compaction: kept entries in list order
          int out = 0;
          for (int a0 = 0; a0 < na; a0 += 32) {
            const int a = a0 + lane;
            const bool keep = a < na && v[a] != 0.0;
            const unsigned mk = __ballot_sync(MCG_FULL, keep);
            if (keep) D.i_active[base + out + __popc(mk & mcg_lanemask_lt())] = B.aidx[off + a];
            out += __popc(mk);
          }
          // the fold: one dependent add per entry (-0.0 for dropped kernels, the
          // identity; a conductance's rhs term v * e_rev of a dropped kernel is
          // +-0.0, and the running sums, started at +0.0, are never -0.0)
          if (lane == 0) {
            double* acc = cond ? M.gsyn : M.rhs_cur;
            const int comp = S.comp;
            double r1 = acc[comp];
            if (cond) {
              const double erev = S.e_rev;
              double r2 = M.gsyn_rhs[comp];
              int i = 0;
              for (; i + 8 <= na; i += 8) {
                double x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = v[i + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  r1 += x[u];
                  r2 += x[u] * erev;
                }
              }
              for (; i < na; ++i) {
                r1 += v[i];
                r2 += v[i] * erev;
              }
              M.gsyn_rhs[comp] = r2;
            } else {
              int i = 0;
              for (; i + 8 <= na; i += 8) {
                double x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = v[i + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) r1 += x[u];
              }
              for (; i < na; ++i) r1 += v[i];
            }
            acc[comp] = r1;
            G->active_n = out;
          }
          if (!cond && out > 0) hc = true;
          off += (na + 31) & ~31;
          __syncwarp();
        }
        if (lane == 0) {
          cs[0].has_gsyn = hg;
          cs[0].has_current = hc;
        }
      }
    } else
    for (int k = warp; k < nc; k += nwarps) {
      if (!cs[k].has_act) continue;
      const int c = c0 + k;
      const McgKind& K = kc[k];
      const McgCellMem M = mcg_cell_mem(D, K, c, K.n <= m ? mcg_comp_block(A, B, k) : nullptr);
      bool hg = false, hc = false;
      for (int gi = 0; gi < K.n_groups; ++gi) {
        McgCellGroup* G = &D.cgs[D.cg_off[c] + gi];
        const McgSpec& S = specs[G->spec];
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
          mcg_decay_active(D, G, S.f_decay, true, M.gsyn, M.gsyn_rhs, S.e_rev, S.comp, lane);
        } else if (S.kind == MCG_SYN_STATIC_CURRENT || S.kind == MCG_SYN_HOMEO_CURRENT) {
          if (mcg_decay_active(D, G, S.f_decay, false, M.rhs_cur, nullptr, 0.0, S.comp, lane)) hc = true;
        }
      }
      if (lane == 0) {
        cs[k].has_gsyn = hg;
        cs[k].has_current = hc;
      }
    }
    MCG_PH(18);
    // ---- C. STC synapses of every cell of the batch, one flat index space
    // (engine.cpp:617-646), four instances per thread in flight; changed
    // flags as warp ballots for the fold
    if (A.stc_sm) {
      // state in shared memory: warp per cell, lanes over its instances, the
      // placement's constants (spec, PRP level, volume) loaded once per warp;
      // changed slots set their flag bit (fmask, cleared in phase A) and leave
      // their SPS delta at their own slot of dbuf
      const int S4 = A.stc_max;
      // few cells (a single neuron with many synapses): parts of each cell's
      // instances go to different warps (part p takes instances p*32 + lane, step 32 P)
      auto stc_cell = [&](int k, int i0, int istep) {
        const McgCellSm& X = cs[k];
        const int c = c0 + k;
        for (int q = 0; q < X.n_stc_seg; ++q) {
          const McgSegSm& g = B.seg[k * A.n_stc_max + q];
          const McgSpec& S = specs[g.spec];
          const McgStcRest R = mcg_stc_rest_of(S);
          const bool late = g.late;
          double prp = 0.0;
          if (late) {
            if (g.prp_sm >= 0) {
              prp = mcg_smem[g.prp_sm];
            } else {
              const McgKind& K = kc[k];
              prp = D.species[D.sp_off[c] + K.prp_idx * K.n + g.comp];
            }
          }
          const int fb = X.stc_off + g.start;
          for (int i = i0; i < g.size; i += istep) {
            const int f = fb + i;
            const double h = B.stc[f], cc = B.stc[2 * S4 + f], a = B.stc[3 * S4 + f];
            if (mcg_stc_at_rest(R, late, prp, h, cc, a)) {
              B.stc[2 * S4 + f] = cc * R.cf;  // the step reduces to the calcium decay
              B.dbuf[f] = -0.0;               // no SPS change (the additive identity)
              continue;
            }
            McgStcVal v{h, B.stc[S4 + f], cc, a};
            double delta = 0.0;
            const bool changed = mcg_stc_step(S, D.dt, D.seed, D.gid0 + uint32_t(c), g.gi, i, s,
                                              late, prp, g.vol, g.rvol, v, delta,
                                              D.stc_nz + g.inst + i);
            B.stc[f] = v.h;
            B.stc[S4 + f] = v.z;
            B.stc[2 * S4 + f] = v.c;
            B.stc[3 * S4 + f] = v.a;
            B.dbuf[f] = changed ? delta : -0.0;
          }
        }
      };
      // (warp 0 is folding phase B's kernels when pb)
      const int w0 = pb ? 1 : 0, nw = nwarps - w0;
      const int parts = max(1, nw / nc);
      if (parts == 1) {
        for (int k = warp - w0; k < nc; k += nw) if (k >= 0) stc_cell(k, lane, 32);
      } else {
        for (int it = warp - w0; it < nc * parts; it += nw) {
          if (it < 0) break;
          const int k = it / parts, part = it - k * parts;
          stc_cell(k, part * 32 + lane, 32 * parts);
        }
      }
    } else
    for (int r0 = 0; r0 < stc_rounds; r0 += 4) {
      McgStcVal v[4];
      int64_t jj[4];
      uint32_t loc[4];
      double dlt[4];
  #pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int f = (r0 + u) * T + tid;
        jj[u] = -1;
        if (r0 + u < stc_rounds && f < stc_total) {
          loc[u] = B.floc[f];
          const int k = int(loc[u] >> 16), q = int(loc[u] & 0xffffu);
          const McgSegSm& g = B.seg[k * A.n_stc_max + q];
          jj[u] = g.inst + (f - cs[k].stc_off - g.start);
          v[u].h = D.i_stc_h[jj[u]];
          v[u].c = D.i_stc_c[jj[u]];
          v[u].a = D.i_sps_abs[jj[u]];
        }
      }
  #pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (r0 + u >= stc_rounds) break;
        const int f = (r0 + u) * T + tid;
        bool changed = false;
        if (jj[u] >= 0) {
          const int k = int(loc[u] >> 16), q = int(loc[u] & 0xffffu);
          const McgSegSm& g = B.seg[k * A.n_stc_max + q];
          const McgKind& K = kc[k];
          const int c = c0 + k;
          const double* SPb = (K.n <= m) ? mcg_comp_block(A, B, k) + m : D.species + D.sp_off[c];
          const bool late = K.prp_idx >= 0;
          const double prp = late ? SPb[int64_t(K.prp_idx) * K.n + g.comp] : 0.0;
          const McgSpec& S = specs[g.spec];
          const McgStcRest R = mcg_stc_rest_of(S);
          if (mcg_stc_at_rest(R, late, prp, v[u].h, v[u].c, v[u].a)) {
            D.i_stc_c[jj[u]] = v[u].c * R.cf;  // the step reduces to the calcium decay
          } else {
            v[u].z = D.i_stc_z[jj[u]];
            double delta = 0.0;
            const int li = f - cs[k].stc_off - g.start;
            changed = mcg_stc_step(S, D.dt, D.seed, D.gid0 + uint32_t(c), g.gi, li, s, late, prp,
                                   g.vol, g.rvol, v[u], delta, D.stc_nz + jj[u]);
            dlt[u] = delta;
            D.i_stc_h[jj[u]] = v[u].h;
            D.i_stc_z[jj[u]] = v[u].z;
            D.i_stc_c[jj[u]] = v[u].c;
            if (changed) D.i_sps_abs[jj[u]] = v[u].a;
          }
        }
        if (jj[u] >= 0) B.dbuf[f] = changed ? dlt[u] : -0.0;
      }
    }
    MCG_PH(16);
    __syncthreads();
    MCG_PH(2);

    // ---- D. SPS fold, synthesis trigger, background current (owner thread)
    if (ko < nc) {
      const int c = c0 + ko;
      McgCellSm& X = cs[ko];
      const McgKind& K = kc[ko];
      const bool in_sm = K.n <= m;
      double* base = in_sm ? mcg_comp_block(A, B, ko) : nullptr;
      double* SP = in_sm ? base + m : D.species + D.sp_off[c];
      if (K.sps_idx >= 0) {
        double* sps = SP + int64_t(K.sps_idx) * K.n;
        int f = X.stc_off;
        for (int q = 0; q < X.n_stc_seg; ++q) {
          const McgSegSm& g = B.seg[ko * A.n_stc_max + q];
          const int fe = f + g.size;
          // every instance of a placement sits on the placement's compartment;
          // every slot holds its delta or -0.0 (unchanged: x + -0.0 == x for
          // every x), so the in-order fold is one dependent add per instance,
          // its loads issued eight ahead
          double acc = sps[g.comp];
          const double* d = B.dbuf + f;
          const int nseg = fe - f;
          int i = 0;
          for (; i + 8 <= nseg; i += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = d[i + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u];
          }
          for (; i < nseg; ++i) acc += d[i];
          f = fe;
          sps[g.comp] = acc;
        }
      }
      X.prod = 0.0;
      if (K.prp_enabled)
        X.prod = (SP[int64_t(K.sps_idx) * K.n + K.prp_comp] > K.prp_theta_star) ? K.prp_rate : 0.0;
      const double ts = double(s) * D.dt;
      const bool bg_gated = K.bg_t1 > K.bg_t0 && ts >= K.bg_t0 && ts < K.bg_t1;
      if (X.lif && K.has_bg && !bg_gated) {
        double ib = K.i_bg;
        if (K.sig_bg != 0.0) ib += K.sig_bg * B.nbuf[ko * 32 + int(so & 31)];
        double* rc = in_sm ? base + (1 + D.sp_max) * m : D.s_rhs_cur + D.comp_off[c];
        rc[K.noise_comp] += ib;
        X.has_current = 1;
      }
    }
    MCG_PH(17);
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
        const McgKind& K = kc[k];
        const McgCellMem M = mcg_cell_mem(D, K, c, K.n <= m ? mcg_comp_block(A, B, k) : nullptr);
        const int i = f - cs[k].hh_off;
        const McgKindSm KS = mcg_kind_consts(D, K, B.ksm, cs[k].kb);
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

    mcg_ph_solve(D, A, b);
    MCG_PH(5);
    __syncthreads();
    MCG_PH(6);

    // ---- F. spike detection (engine.cpp:753-769)
    if (ko < nc) {
      const int c = c0 + ko;
      McgCellSm& X = cs[ko];
      const McgKind& K = kc[ko];
      X.fired = 0;
      if (K.has_detector && !X.refractory) {
        const double* V = (K.n <= m) ? mcg_comp_block(A, B, ko) : D.v + D.comp_off[c];
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
    MCG_PH(7);
    // post-event hook and LIF reset of the cells that fired (warp per cell)
    for (int k = warp; k < nc; k += nwarps) {
      if (!cs[k].fired) continue;
      const int c = c0 + k;
      const McgKind& K = kc[k];
      mcg_post_event_b(D, A, B, K, k, D.cg_off[c], s, lane);
      if (cs[k].lif) {
        double* V = (K.n <= m) ? mcg_comp_block(A, B, k) : D.v + D.comp_off[c];
        for (int i = lane; i < K.n; i += 32) V[i] = K.v_reset;
      }
    }
    __syncthreads();
    MCG_PH(8);
    // detector bookkeeping and probes (engine.cpp:770-793)
    if (ko < nc) {
      const int c = c0 + ko;
      McgCellSm& X = cs[ko];
      const McgKind& K = kc[ko];
      const bool in_sm = K.n <= m;
      const double* V = in_sm ? mcg_comp_block(A, B, ko) : D.v + D.comp_off[c];
      if (K.has_detector && !X.refractory) {
        if (X.fired) {
          if (X.lif) X.refr = s + 1 + K.ref_steps;
          else X.armed = 0;
        } else if (!X.armed && V[K.detector_comp] < K.threshold) {
          X.armed = 1;
        }
        X.det_prev = V[K.detector_comp];
      }
      for (int q = X.p0; q < X.p1; ++q) {
        const int p = D.probe_idx[q];
        const McgProbe& Pr = D.probes[p];
        if (mcg_mod(s + 1, Pr.every) != 0) continue;
        const int64_t m0 = (D.ctl[3] + Pr.every) / Pr.every;
        const double* SP = in_sm ? V + m : D.species + D.sp_off[c];
        D.trace_buf[D.trace_base[p] + ((s + 1) / Pr.every - m0)] =
            mcg_probe_value(D, K, c, Pr, V, SP, mcg_stc_ref(A, B, ko, Pr.group));
      }
    }
    __syncthreads();
    MCG_PH(9);
  }

  // ---- epoch end: log the batch's spikes as one chunk, publish what the next
  // expansion reads (spike slots, inbox cursors)
  __shared__ int s_log_off;
  if (tid == 0) {
    int tot = 0;
    for (int k = 0; k < nc; ++k) tot += min(cs[k].nsp, D.sp_cap);
    s_log_off = -1;
    if (tot > 0) {
      const unsigned long long off = atomicAdd(A.log_n, static_cast<unsigned long long>(tot));
      const unsigned long long ci = atomicAdd(A.chunk_n, 1ull);
      A.chunks[ci] = make_int4(A.epoch_base + j, b, static_cast<int>(off), tot);
      s_log_off = static_cast<int>(off);
    }
  }
  __syncthreads();
  if (ko < nc) {
    const int c = c0 + ko;
    const McgCellSm& X = cs[ko];
    const int k = min(X.nsp, D.sp_cap);
    if (k > 0) {
      int before = 0;
      for (int q = 0; q < ko; ++q) before += min(cs[q].nsp, D.sp_cap);
      for (int i = 0; i < k; ++i) {
        A.log_t[s_log_off + before + i] = D.sp_t[int64_t(c) * D.sp_cap + i];
        A.log_gid[s_log_off + before + i] = D.gid0 + uint32_t(c);
      }
    }
    D.sp_count[c] = k;
    if (A.x_send != nullptr && k > 0) {  // sharded: publish for the caller's allgather
      const int64_t pos = static_cast<int64_t>(
          atomicAdd(reinterpret_cast<unsigned long long*>(A.x_send), static_cast<unsigned long long>(k)));
      if (pos + k > A.x_cap) {
        atomicOr(D.err, MCG_ERR_FLAG_SPIKES);
      } else {
        for (int i = 0; i < k; ++i) {
          A.x_send[1 + 3 * (pos + i)] = int64_t(D.gid0) + c;
          A.x_send[2 + 3 * (pos + i)] = D.sp_step[int64_t(c) * D.sp_cap + i];
          A.x_send[3 + 3 * (pos + i)] = __double_as_longlong(D.sp_t[int64_t(c) * D.sp_cap + i]);
        }
      }
    }
    D.pend_sel[c] = X.sel;
    D.pend_off[c] = X.cur;
    D.pend_n[c] = X.end;
    D.inc_n[c] = 0;
  }
  __syncthreads();
  MCG_PH(11);
}

__global__ void __launch_bounds__(MCG_BATCH_THREADS, 1) k_batch(const __grid_constant__ McgDev D,
                                                               const __grid_constant__ McgBatchArgs A,
                                                               int64_t max_len) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const McgBatchSm B = mcg_batch_sm(A);
  if (A.phase && threadIdx.x == 0) {
    for (int i = 0; i < MCG_NPHASE; ++i) mcg_ph_acc[i] = 0;
    mcg_ph_acc[MCG_NPHASE] = clock64();
  }
  if (threadIdx.x < MCG_KSLOTS) mcg_kslot_off[threadIdx.x] = -1;
  if (A.n_specs_sm > 0)
    for (int i = threadIdx.x; i < A.n_specs_sm; i += blockDim.x) B.spec[i] = D.specs[i];
  __syncthreads();
  // resident: every batch has its own CTA for the whole launch
  const bool resident = A.n_batches <= int(gridDim.x);
  const bool mine = int(blockIdx.x) < A.n_batches;
  if (resident && mine) mcg_batch_enter(D, A, blockIdx.x);
  MCG_PH(14);
  for (int32_t j = 0; j < A.n_epochs; ++j) {
    int64_t s0, s1;
    if (!mcg_epoch_bounds(D.ctl, j, s0, s1)) break;
    mcg_expand(A.E, D, j, s0, s1, max_len);
    MCG_PH(12);
    grid.sync();
    MCG_PH(13);
    if (*D.abort) break;
    if (resident) {
      if (mine) mcg_batch_epoch(D, A, blockIdx.x, j, s0, s1);
    } else {
      for (int32_t b = blockIdx.x; b < A.n_batches; b += gridDim.x) {
        mcg_batch_enter(D, A, b);
        mcg_batch_epoch(D, A, b, j, s0, s1);
        mcg_batch_exit(D, A, b);
      }
    }
    grid.sync();
    MCG_PH(13);
  }
  if (resident && mine) mcg_batch_exit(D, A, blockIdx.x);
  MCG_PH(14);
  if (A.phase && threadIdx.x == 0)
    for (int i = 0; i < MCG_NPHASE; ++i) {
      atomicAdd(&A.phase[i], mcg_ph_acc[i]);
      if (blockIdx.x == 0) atomicAdd(&A.phase[MCG_NPHASE + i], mcg_ph_acc[i]);  // CTA 0 alone
      atomicAdd(&A.phase[(2 + blockIdx.x) * MCG_NPHASE + i], mcg_ph_acc[i]);   // per CTA
    }
}
#undef MCG_PH
