// mcg_point.cuh — k_point: Engine::advance_to (engine.cpp:909-945) for
// networks of exact-LIF point cells without cell-to-cell connections, the
// shape of the single-synapse protocols (network.cpp:318-399, BASELINE
// config 1) and of any set of independent point neurons driven by sources.
//
// Without cell edges the reference runs the whole span as one epoch per
// call (engine.cpp:913-915) and step_cell (engine.cpp:541-783) is one long
// serial chain per cell.  On a GPU that chain's cost is the latency of each
// step's dependent fp64 operations, so here a cell's whole state lives in
// the registers of ONE thread for a whole epoch: V, the species pools (the
// n == 1 closed forms, engine.cpp:729-735), the STC synapses' h, z, c and
// folded |h - h0| (up to MCG_PT_STC instances), the detector, the refractory
// counter, the delayed-calcium queue cursors and the pending-event cursor.
// What can leave that chain is taken off it:
//   * the background-noise normals of the epoch (normal_for(key(seed, gid,
//     1, 0), s), rng.cpp:67-78) are drawn by the whole CTA into shared
//     memory before the serial run, one Box-Muller pair per thread at a time;
//   * network events arrive sorted in the cell's pending list (the same
//     expansion, inbox sort and merge as the other stepping kernels) and are
//     read one key ahead;
//   * the membrane's V_inf of step s + 1 is formed while step s runs.
// The plasticity noise (calcium above a threshold) is drawn on demand
// (mcg_stc_noise), as it is needed only during and shortly after stimulation.
// Every fp64 operation is the reference's, in its order (see mcg_warp.cuh
// for the phase-by-phase citations; the closed forms below cite theirs).
#pragma once
#include <cooperative_groups.h>

#include "mcg_batch.cuh"

#define MCG_PT_STC 4          // max STC instances per cell held in registers
#define MCG_PT_SP 4           // max species per cell held in registers
// k_point<NSTC, NSP> instances: <1, 2> (the protocol cells: one STC synapse,
// SPS + PRP) and <MCG_PT_STC, MCG_PT_SP>
#define MCG_PT_THREADS 128
#define MCG_PT_NB 4096        // background normals per epoch (>= epoch length)

struct McgPointArgs {
  McgEv E;
  int32_t n_epochs;
  int32_t epoch_base;
  double* log_t;              // spike log of the launch (as McgBatchArgs)
  uint32_t* log_gid;
  unsigned long long* log_n;
  int4* chunks;               // (epoch, cell, offset, count)
  unsigned long long* chunk_n;
};

// inbox of cell c (warp 0): sort this epoch's incoming keys and merge them
// into the pending list (the reference's per-epoch inbox sort,
// engine.cpp:916-925); cursors returned through shared memory
__device__ void mcg_pt_inbox(const McgDev& D, int c, int lane, int* cur_out) {
  int sel = D.pend_sel[c], cur = D.pend_off[c], end = D.pend_n[c];
  const int nin = D.inc_n[c];
  if (nin > 0) {
    uint64_t* in = D.inc + int64_t(c) * D.inc_cap;
    if (nin > 1) mcg_warp_sort(in, nin, lane);
    __syncwarp();
    const uint64_t* pold = D.pend + (int64_t(c) * 2 + sel) * D.pend_cap;
    uint64_t* out = D.pend + (int64_t(c) * 2 + (1 - sel)) * D.pend_cap;
    if (cur >= end) {
      for (int i = lane; i < nin; i += 32) out[i] = in[i];
      end = nin;
    } else {
      if (lane == 0) {
        int a = cur, b = 0, o = 0;
        while (a < end && b < nin) out[o++] = (pold[a] <= in[b]) ? pold[a++] : in[b++];
        while (a < end) out[o++] = pold[a++];
        while (b < nin) out[o++] = in[b++];
      }
      end = end - cur + nin;
    }
    cur = 0;
    sel = 1 - sel;
    __syncwarp();
  }
  if (lane == 0) {
    cur_out[0] = sel;
    cur_out[1] = cur;
    cur_out[2] = end;
  }
}

// one epoch [s0, s1) of cell c on this thread; nb = its background normals
template <int NSTC, int NSP>
__device__ void mcg_pt_run(const McgDev& D, const McgPointArgs& A, int c, int32_t j, int64_t s0,
                           int64_t s1, const double* nb, const int* pc) {
  const McgKind& Kg = D.kinds[D.cell_kind[c]];  // global copy: the rare probe path reads it
  const McgKind K = Kg;
  const uint32_t gid = D.gid0 + uint32_t(c);
  // RNG key of this cell: (seed, gid) unless overridden per cell (independent
  // trials in one engine, mcg_set_cell_rng)
  const uint64_t kseed = D.cell_seed ? D.cell_seed[c] : D.seed;
  const uint32_t kgid = D.cell_key_gid ? D.cell_key_gid[c] : gid;
  const int64_t cg0 = D.cg_off[c];
  // ---- state into registers
  double V = D.v[D.comp_off[c]];
  const int S = K.n_species;
  double sp[NSP], spc[NSP], spd[NSP], spr[NSP];
#pragma unroll
  for (int q = 0; q < NSP; ++q) {
    sp[q] = q < S ? D.species[D.sp_off[c] + q] : 0.0;
    if (q < S) {
      const int64_t ka = K.sp_arr + q;
      spc[q] = D.k_sp_cap_dt[ka];
      spd[q] = D.k_sp_cap_dt[ka] + D.k_sp_gs[ka];  // cap0 + gse (engine.cpp:734)
      spr[q] = __drcp_rn(spd[q]);
    } else {
      spc[q] = 0.0;
      spd[q] = spr[q] = 1.0;
    }
  }
  int64_t refr = D.refr_until[c];
  double det_prev = D.det_prev[c];
  int armed = D.armed[c];
  uint32_t iseq = D.internal_seq[c];
  uint32_t charge_groups = 0;  // bit gi: placement gi is static_charge
  int stc_gi = -1, stc_n = 0, stc_spec = 0, fifo = -1;
  int64_t stc_inst = 0;
  for (int gi = 0; gi < K.n_groups && gi < 8; ++gi) {
    const McgCellGroup Gr = D.cgs[cg0 + gi];
    const int kd = D.specs[Gr.spec].kind;
    if (kd == MCG_SYN_STATIC_CHARGE) charge_groups |= 1u << gi;
    if (kd == MCG_SYN_STC_CHARGE) {
      stc_gi = gi;
      stc_n = Gr.size;
      stc_inst = Gr.inst;
      stc_spec = Gr.spec;
      fifo = Gr.fifo;
    }
  }
  const McgSpec Sp = D.specs[stc_spec];
  const double cf0 = D.k_cf[K.arr];      // charge_factor[0]
  const double vol = D.k_volume[K.arr], rvol = D.k_rvol[K.arr];
  const bool late = K.prp_idx >= 0;
  McgStcVal st[NSTC];
#pragma unroll
  for (int i = 0; i < NSTC; ++i) {
    if (i < stc_n) {
      st[i] = McgStcVal{D.i_stc_h[stc_inst + i], D.i_stc_z[stc_inst + i], D.i_stc_c[stc_inst + i],
                        D.i_sps_abs[stc_inst + i]};
    } else {
      st[i] = McgStcVal{0.0, 0.0, 0.0, 0.0};
    }
  }
  int64_t f_base = 0, f_head = 0, f_tail = 0, next_due = INT64_MAX;
  int32_t f_cap = 1;
  if (fifo >= 0) {
    const McgFifo F = D.fifos[fifo];
    f_base = F.base;
    f_cap = F.cap;
    f_head = F.head;
    f_tail = F.tail;
    if (f_head < f_tail) next_due = D.fifo_step[f_base + mcg_mod(f_head, f_cap)];
  }
  // pending network events
  const int sel = pc[0];
  int cur = pc[1];
  const int end = pc[2];
  const uint64_t* pend = D.pend + (int64_t(c) * 2 + sel) * D.pend_cap;
  const int rb = D.rank_bits;
  const uint64_t rmask = (1ull << rb) - 1;
  uint64_t nk = cur < end ? pend[cur] : ~0ull;
  int64_t ndel = 0;
  // probes: next step s with (s + 1) a multiple of some probe's period
  const int p0 = D.probe_off[c], p1 = D.probe_off[c + 1];
  auto next_probe = [&](int64_t after) {  // smallest s >= after with a probe due
    int64_t best = INT64_MAX;
    for (int q = p0; q < p1; ++q) {
      const int64_t ev = D.probes[D.probe_idx[q]].every;
      const int64_t m = (after + 1 + ev - 1) / ev;  // ceil((after + 1) / ev)
      best = min(best, m * ev - 1);
    }
    return best;
  };
  int64_t s_probe = p0 < p1 ? next_probe(s0) : INT64_MAX;
  // the quiet window as a step interval [qa, qb): double(s) * dt is
  // nondecreasing in s, so {s : t0 <= s dt < t1} is contiguous; its ends are
  // found with the reference's own expression (engine.cpp:652-655)
  int64_t qa = s1, qb = s1;
  if (K.bg_t1 > K.bg_t0) {
    auto in_win = [&](int64_t q) {
      const double ts = double(q) * D.dt;
      return ts >= K.bg_t0 && ts < K.bg_t1;
    };
    auto first_ge = [&](double t) {  // first q >= s0 with double(q) * dt >= t
      int64_t lo = s0, hi = s1;
      while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (double(mid) * D.dt >= t) hi = mid;
        else lo = mid + 1;
      }
      return lo;
    };
    qa = first_ge(K.bg_t0);
    qb = first_ge(K.bg_t1);
    if (qa < s1 && !in_win(qa)) qa = qb = s1;  // defensive: empty window
  }
  const bool bg = K.has_bg != 0;
  const bool noisy = bg && K.sig_bg != 0.0;
  int nsp = 0;

  for (int64_t s = s0; s < s1; ++s) {
    const bool refractory = s < refr;
    // ---- 1. delivery (engine.cpp:549-560): network events, then delayed calcium
    while (int64_t(nk >> rb) <= s) {
      const int64_t r = int64_t(nk & rmask);
      const int grp = D.e_group[r];
      const double w = D.e_weight[r];
      if ((charge_groups >> grp) & 1u) {
        if (!refractory && w != 0.0) V += D.e_wcf[r];  // w * charge_factor[comp] (engine.cpp:455-460)
      } else {  // stc_charge, etype 0 (engine.cpp:497-510)
        const uint32_t inst = D.e_inst[r];
        if (f_tail - f_head >= f_cap) {
          atomicOr(D.err, MCG_ERR_FLAG_FIFO);
        } else {
          const int64_t slot = f_base + mcg_mod(f_tail, f_cap);
          D.fifo_step[slot] = s + Sp.ca_delay;
          D.fifo_si[slot] = (uint64_t(iseq) << 32) | uint64_t(inst);
          D.fifo_src[slot] = D.e_src[r];
          D.fifo_w[slot] = w;
          if (f_head == f_tail) next_due = s + Sp.ca_delay;
          ++f_tail;
        }
        ++iseq;
        if (!refractory) {
          double tw = 0.0;  // stc_total_weight: h + h0 * z
#pragma unroll
          for (int i = 0; i < NSTC; ++i)
            if (uint32_t(i) == inst) tw = st[i].h + Sp.h0 * st[i].z;
          V += tw * w * cf0;
        }
      }
      ++ndel;
      ++cur;
      nk = cur < end ? pend[cur] : ~0ull;
    }
    while (next_due <= s) {  // stc_on_pre_calcium (mechanisms.hpp:203-206)
      const int64_t slot = f_base + mcg_mod(f_head, f_cap);
      const uint32_t inst = uint32_t(D.fifo_si[slot] & 0xffffffffu);
      ++f_head;
#pragma unroll
      for (int i = 0; i < NSTC; ++i)
        if (uint32_t(i) == inst) st[i].c += Sp.cpre_s;
      next_due = f_head < f_tail ? D.fifo_step[f_base + mcg_mod(f_head, f_cap)] : INT64_MAX;
    }
    // ---- 2. STC synapses in instance order (engine.cpp:617-646), the SPS
    // fold inside the loop as the reference's
    {
      double prp = 0.0;  // PRP at the placement's compartment (the only one)
#pragma unroll
      for (int q = 0; q < NSP; ++q)
        if (late && q == K.prp_idx) prp = sp[q];
#pragma unroll
      for (int i = 0; i < NSTC; ++i) {
        if (i < stc_n) {
          double delta = 0.0;
          const bool changed = mcg_stc_step(Sp, D.dt, kseed, kgid, stc_gi, i, s, late, prp, vol, rvol, st[i],
                                            delta, D.stc_nz + stc_inst + i);
          if (changed && K.sps_idx >= 0) {
#pragma unroll
            for (int q = 0; q < NSP; ++q)
              if (q == K.sps_idx) sp[q] += delta;
          }
        }
      }
    }
    // ---- synthesis trigger (engine.cpp:721-725, mechanisms.hpp:264-266) and
    // background current (engine.cpp:652-664)
    double prod = 0.0;
    if (K.prp_enabled) {
      double spsv = 0.0;
#pragma unroll
      for (int q = 0; q < NSP; ++q)
        if (q == K.sps_idx) spsv = sp[q];
      prod = spsv > K.prp_theta_star ? K.prp_rate : 0.0;
    }
    double rc = 0.0;
    if (bg) {
      if (s < qa || s >= qb) {
        double ib = K.i_bg;
        if (noisy) ib += K.sig_bg * nb[s - s0];
        rc = 0.0 + ib;  // rhs_current[noise_comp] starts at 0.0
      }
    }
    // ---- 3. membrane, exact LIF (engine.cpp:666-673)
    if (!refractory) {
      const double vinf = K.v_rev + K.r_mem * rc;
      V = vinf + (V - vinf) * K.lif_exact_f;
    }
    // species closed forms (engine.cpp:729-735)
#pragma unroll
    for (int q = 0; q < NSP; ++q) {
      if (q < S) {
        const double r = spc[q] * sp[q] + (q == K.prp_idx ? prod : 0.0);
        sp[q] = mcg_div(r, spd[q], spr[q]);
      }
    }
    // ---- 4. detection, post-event hook, reset (engine.cpp:753-780)
    if (K.has_detector && !refractory) {
      bool fired = false;
      if (armed && det_prev < K.threshold && V >= K.threshold) {
        double f = (V > det_prev) ? (K.threshold - det_prev) / (V - det_prev) : 1.0;
        f = (f < 0.0) ? 0.0 : ((1.0 < f) ? 1.0 : f);  // std::clamp
        fired = true;
        if (nsp < D.sp_cap) {
          D.sp_step[int64_t(c) * D.sp_cap + nsp] = s;
          D.sp_t[int64_t(c) * D.sp_cap + nsp] = (double(s) + f) * D.dt;
        } else {
          atomicOr(D.err, MCG_ERR_FLAG_SPIKES);
        }
        ++nsp;
      }
      if (fired) {
#pragma unroll
        for (int i = 0; i < NSTC; ++i)  // stc_on_post (mechanisms.hpp:207-210)
          if (i < stc_n) st[i].c += Sp.cpost_s;
        V = K.v_reset;
        refr = s + 1 + K.ref_steps;
      } else if (!armed && V < K.threshold) {
        armed = 1;
      }
      det_prev = V;
    }
    // ---- probes (engine.cpp:785-829), on the post-step state
    if (s == s_probe) {
      for (int q = p0; q < p1; ++q) {
        const int p = D.probe_idx[q];
        const McgProbe& Pr = D.probes[p];
        if (mcg_mod(s + 1, Pr.every) != 0) continue;
        const int64_t m0 = (D.ctl[3] + Pr.every) / Pr.every;
        double val = 0.0;
        if (Pr.what == MCG_PROBE_VOLTAGE) {
          val = V;
        } else if (Pr.what == MCG_PROBE_SPECIES) {
#pragma unroll
          for (int r = 0; r < NSP; ++r)
            if (r == Pr.species) val = sp[r];
        } else if (Pr.group == stc_gi && Pr.what != MCG_PROBE_SYN_KERNEL) {
#pragma unroll
          for (int i = 0; i < NSTC; ++i)
            if (i == Pr.instance) {
              switch (Pr.what) {
                case MCG_PROBE_SYN_WEIGHT: val = st[i].h + Sp.h0 * st[i].z; break;
                case MCG_PROBE_SYN_H: val = st[i].h; break;
                case MCG_PROBE_SYN_Z: val = st[i].z; break;
                case MCG_PROBE_SYN_C: val = st[i].c; break;
                default: break;
              }
            }
        } else {
          val = mcg_probe_value(D, Kg, c, Pr, nullptr, nullptr);
        }
        D.trace_buf[D.trace_base[p] + ((s + 1) / Pr.every - m0)] = val;
      }
      s_probe = next_probe(s + 1);
    }
  }

  // ---- epoch end: state back, spikes as one log chunk, cursors
  D.v[D.comp_off[c]] = V;
#pragma unroll
  for (int q = 0; q < NSP; ++q)
    if (q < S) D.species[D.sp_off[c] + q] = sp[q];
#pragma unroll
  for (int i = 0; i < NSTC; ++i)
    if (i < stc_n) {
      D.i_stc_h[stc_inst + i] = st[i].h;
      D.i_stc_z[stc_inst + i] = st[i].z;
      D.i_stc_c[stc_inst + i] = st[i].c;
      D.i_sps_abs[stc_inst + i] = st[i].a;
    }
  D.refr_until[c] = refr;
  D.det_prev[c] = det_prev;
  D.armed[c] = armed;
  D.internal_seq[c] = iseq;
  if (fifo >= 0) {
    D.fifos[fifo].head = f_head;
    D.fifos[fifo].tail = f_tail;
  }
  const int nk_log = min(nsp, D.sp_cap);
  if (nk_log > 0) {
    const int off = static_cast<int>(atomicAdd(A.log_n, static_cast<unsigned long long>(nk_log)));
    const unsigned long long ci = atomicAdd(A.chunk_n, 1ull);
    A.chunks[ci] = make_int4(A.epoch_base + j, c, off, nk_log);
    for (int i = 0; i < nk_log; ++i) {
      A.log_t[off + i] = D.sp_t[int64_t(c) * D.sp_cap + i];
      A.log_gid[off + i] = gid;
    }
  }
  D.sp_count[c] = nk_log;
  D.pend_sel[c] = sel;
  D.pend_off[c] = cur;
  D.pend_n[c] = end;
  D.inc_n[c] = 0;
  if (ndel) atomicAdd(D.delivered, static_cast<unsigned long long>(ndel));
}

template <int NSTC, int NSP>
__global__ void __launch_bounds__(MCG_PT_THREADS, 1) k_point(const __grid_constant__ McgDev D,
                                                            const __grid_constant__ McgPointArgs A,
                                                            int64_t max_len) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double nb[MCG_PT_NB];
  __shared__ int pc[3];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int32_t j = 0; j < A.n_epochs; ++j) {
    int64_t s0, s1;
    if (!mcg_epoch_bounds(D.ctl, j, s0, s1)) break;
    mcg_expand(A.E, D, j, s0, s1, max_len);
    grid.sync();
    if (*D.abort) break;
    for (int c = blockIdx.x; c < D.n_cells; c += gridDim.x) {
      const McgKind& K = D.kinds[D.cell_kind[c]];
      // background normals of [s0, s1): step n takes half n & 1 of pair n >> 1,
      // pair p of Threefry block p >> 1 (rng.cpp:67-78)
      if (K.has_bg && K.sig_bg != 0.0) {
        const mcg_key key = mcg_make_key(D.cell_seed ? D.cell_seed[c] : D.seed,
                                         D.cell_key_gid ? D.cell_key_gid[c] : D.gid0 + uint32_t(c), 1, 0);
        const int64_t pa = s0 >> 1, pb = (s1 - 1) >> 1;
        for (int64_t pr = pa + tid; pr <= pb; pr += blockDim.x) {
          uint64_t x[4];
          mcg_threefry(&key, uint64_t(pr) >> 1, x);
          const unsigned h = unsigned(pr & 1);
          const double u1 = ((double)(x[2 * h] >> 11) + 1.0) * MCG_2POW_M53;
          const double u2 = (double)(x[2 * h + 1] >> 11) * MCG_2POW_M53;
          double z0, z1;
          mcg_normal_pair(u1, u2, &z0, &z1);
          const int64_t n0 = pr * 2;
          if (n0 >= s0) nb[n0 - s0] = z0;
          if (n0 + 1 < s1) nb[n0 + 1 - s0] = z1;
        }
      }
      if (tid < 32) mcg_pt_inbox(D, c, lane, pc);
      __syncthreads();
      if (tid == 0) mcg_pt_run<NSTC, NSP>(D, A, c, j, s0, s1, nb, pc);
      __syncthreads();
    }
    grid.sync();
  }
}
