// mcg_kernels.cuh — the per-epoch kernels.
//
//  k_source_fire    generate_source_events (engine.cpp:831-873): which sources
//                   fire at which steps of [s0, s1); Poisson draws on device.
//  k_spike_outdeg   size of the spike expansion (exchange, engine.cpp:875-889)
//  k_write_*        EventRec keys (dst | step | rank) for source firings and
//                   for the previous epoch's spikes
//  k_offsets        per-cell segment of the sorted keys (the segmented offsets
//                   of the delivery scan)
//  k_epoch          step_cell for every cell and every step of the epoch
//  k_spike_write    ordered compaction of the emitted spikes (gid, step order)
//  k_leftover       carry undelivered keys to the next epoch
//  k_ff_*           fast_forward_to (engine.cpp:947-1034)
#pragma once
#include "mcg_device.cuh"

// ---------------------------------------------------------------------------
// sources
// ---------------------------------------------------------------------------
struct McgSrcTask {
  int32_t source;
  int32_t type;        // MCG_SRC_*
  int32_t window;      // poisson window
  int32_t pad;
  int64_t a, b;        // poisson: window step bounds; scripted: [first,last) into steps
  double prob;         // poisson
  double r_t0, r_period;
  int64_t r_count;
};

struct McgSrcDev {
  const McgSrcTask* tasks;
  int32_t n_tasks;
  const int64_t* scripted_steps;
  const int64_t* src_edge_off;
  const int64_t* src_edges;
  int32_t* fire_src;
  int64_t* fire_step;
  int64_t fire_cap;
  unsigned long long* ctr;  // [0] n_fire, [1] n_src_events
  int32_t* err;
};

__device__ __forceinline__ void mcg_emit_fire(const McgSrcDev& S, int32_t src, int64_t st) {
  const unsigned long long k = atomicAdd(&S.ctr[0], 1ull);
  if (k < static_cast<unsigned long long>(S.fire_cap)) {
    S.fire_src[k] = src;
    S.fire_step[k] = st;
  } else {
    atomicOr(S.err, MCG_ERR_FLAG_SPIKES);
  }
  atomicAdd(&S.ctr[1],
            static_cast<unsigned long long>(S.src_edge_off[src + 1] - S.src_edge_off[src]));
}

__global__ void k_source_fire(McgSrcDev S, uint64_t seed, double dt, int64_t s0, int64_t s1) {
  const int64_t len = s1 - s0;
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= int64_t(S.n_tasks) * len) return;
  const McgSrcTask T = S.tasks[t / len];
  const int64_t off = t % len;
  if (S.src_edge_off[T.source + 1] == S.src_edge_off[T.source]) return;  // no edges
  if (T.type == MCG_SRC_POISSON) {
    const int64_t s = s0 + off;
    const int64_t a = T.a > s0 ? T.a : s0;
    const int64_t b = T.b < s1 ? T.b : s1;
    if (s < a || s >= b) return;
    const mcg_key key = mcg_make_key(seed, 0x100000000ull + uint64_t(T.source), 3, 0);
    if (mcg_uniform_for(&key, static_cast<uint64_t>(s)) < T.prob) mcg_emit_fire(S, T.source, s);
  } else if (off == 0) {
    if (T.type == MCG_SRC_SCRIPTED) {
      for (int64_t i = T.a; i < T.b; ++i) {
        const int64_t st = S.scripted_steps[i];
        if (st >= s0 && st < s1) mcg_emit_fire(S, T.source, st);
      }
    } else {  // regular
      if (T.r_period <= 0) return;
      int64_t k0 = static_cast<int64_t>(ceil((double(s0) * dt - T.r_t0) / T.r_period - 1e-9));
      if (k0 < 0) k0 = 0;
      for (int64_t kk = k0; kk < T.r_count; ++kk) {
        const int64_t st = static_cast<int64_t>(ceil((T.r_t0 + double(kk) * T.r_period) / dt - 1e-9));
        if (st >= s1) break;
        if (st >= s0) mcg_emit_fire(S, T.source, st);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// event keys
// ---------------------------------------------------------------------------
struct McgEvDev {
  uint64_t* keys;             // write buffer
  unsigned long long* wcur;   // write cursor
  int32_t rank_bits, step_bits;
  int64_t base;
  const int32_t* e_dst;
  const int64_t* e_delay;
  const int64_t* out_begin;   // per global gid
  const int64_t* out_end;
};

__device__ __forceinline__ uint64_t mcg_ev_key(const McgEvDev& E, int64_t rank, int64_t step) {
  return (uint64_t(uint32_t(E.e_dst[rank])) << (E.rank_bits + E.step_bits)) |
         (uint64_t(step - E.base) << E.rank_bits) | uint64_t(rank);
}

// warp per source firing: keys for all of the source's edges
__global__ void k_write_source_events(McgEvDev E, McgSrcDev S, int64_t n_fire) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= n_fire) return;
  const int32_t src = S.fire_src[w];
  const int64_t st = S.fire_step[w];
  const int64_t e0 = S.src_edge_off[src], e1 = S.src_edge_off[src + 1];
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(E.wcur, static_cast<unsigned long long>(e1 - e0));
  base = __shfl_sync(MCG_FULL, base, 0);
  for (int64_t k = e0 + lane; k < e1; k += 32) {
    const int64_t r = S.src_edges[k];
    E.keys[base + (k - e0)] = mcg_ev_key(E, r, st + E.e_delay[r]);
  }
}

// warp per emitted spike: keys for the spiking cell's out-edges with a local
// destination; delivery at em.step + 1 + delay (engine.cpp:881)
__global__ void k_write_spike_events(McgEvDev E, const uint32_t* sp_gid, const int64_t* sp_step,
                                     const unsigned long long* n_sp) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= static_cast<int64_t>(*n_sp)) return;
  const uint32_t gid = sp_gid[w];
  const int64_t st = sp_step[w];
  const int64_t e0 = E.out_begin[gid], e1 = E.out_end[gid];
  if (e1 <= e0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(E.wcur, static_cast<unsigned long long>(e1 - e0));
  base = __shfl_sync(MCG_FULL, base, 0);
  for (int64_t r = e0 + lane; r < e1; r += 32)
    E.keys[base + (r - e0)] = mcg_ev_key(E, r, st + 1 + E.e_delay[r]);
}

__global__ void k_spike_outdeg(const uint32_t* sp_gid, const unsigned long long* n_sp,
                               const int64_t* out_begin, const int64_t* out_end,
                               unsigned long long* acc) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(*n_sp)) return;
  const uint32_t g = sp_gid[i];
  const int64_t d = out_end[g] - out_begin[g];
  if (d > 0) atomicAdd(acc, static_cast<unsigned long long>(d));
}

// lower_bound of each cell's first key; cursor starts at the segment start
__global__ void k_offsets(const uint64_t* keys, int64_t n, int32_t n_cells, int32_t shift,
                          int64_t* ev_begin, int64_t* ev_cursor) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > n_cells) return;
  const uint64_t target = uint64_t(c) << shift;
  int64_t lo = 0, hi = n;
  if (c == n_cells) {
    lo = n;
  } else {
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1;
      else hi = mid;
    }
  }
  ev_begin[c] = lo;
  if (c < n_cells) ev_cursor[c] = lo;
}

// ---------------------------------------------------------------------------
// the epoch kernel: step_cell (engine.cpp:541-783) for s in [s0, s1)
// ---------------------------------------------------------------------------

// decay an active list, fold kept kernels in active-list order (engine.cpp:578-616)
__device__ __forceinline__ bool mcg_decay_active(const McgDev& D, McgCellGroup* G, double f,
                                                 bool cond, double* acc, double* acc2,
                                                 double erev, int lane) {
  const int na = G->active_n;
  const int64_t base = G->inst;
  int out = 0;
  for (int a0 = 0; a0 < na; a0 += 32) {
    const int a = a0 + lane;
    int i = 0, comp = 0;
    double kv = 0.0;
    bool keep = false;
    if (a < na) {
      i = D.i_active[base + a];
      const int64_t j = base + i;
      kv = D.i_kernel[j] * f;
      if (cond ? (kv < 1e-30) : (fabs(kv) < 1e-30)) kv = 0.0;
      D.i_kernel[j] = kv;
      keep = kv != 0.0;
      comp = D.i_comp[j];
    }
    const unsigned m = __ballot_sync(MCG_FULL, keep);
    __syncwarp();
    if (keep) D.i_active[base + out + __popc(m & mcg_lanemask_lt())] = i;
    unsigned mm = m;
    while (mm) {
      const int l = __ffs(mm) - 1;
      mm &= mm - 1;
      const double kl = __shfl_sync(MCG_FULL, kv, l);
      const int cl = __shfl_sync(MCG_FULL, comp, l);
      if (lane == 0) {
        acc[cl] += kl;
        if (cond) acc2[cl] += kl * erev;
      }
    }
    out += __popc(m);
  }
  __syncwarp();
  if (lane == 0) G->active_n = out;
  __syncwarp();
  return out > 0;
}

// post_event (engine.cpp:515-539): every synapse of the cell, lanes in parallel
__device__ __forceinline__ void mcg_post_event(const McgDev& D, const McgKind& K, int64_t cg0,
                                               int64_t s, int lane) {
  for (int gi = 0; gi < K.n_groups; ++gi) {
    const McgCellGroup G = D.cgs[cg0 + gi];
    const McgSpec& S = D.specs[G.spec];
    if (S.kind == MCG_SYN_STDP_COND) {
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
    } else if (S.kind == MCG_SYN_STC_CHARGE) {
      for (int i = lane; i < G.size; i += 32) D.i_stc_c[G.inst + i] += S.cpost_s;
    }
  }
}

// ---------------------------------------------------------------------------
// spike compaction and carry-over of undelivered events
// ---------------------------------------------------------------------------
__global__ void k_spike_write(McgDev D, const int64_t* sp_scan, uint32_t* ep_gid, int64_t* ep_step,
                              double* log_t, uint32_t* log_gid, unsigned long long* ctr_ep,
                              unsigned long long* ctr_log) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= D.n_cells) return;
  const int64_t base_log = static_cast<int64_t>(*ctr_log);
  const int k = D.sp_count[c];
  const int64_t o = sp_scan[c];
  for (int i = 0; i < k; ++i) {
    ep_gid[o + i] = D.gid0 + uint32_t(c);
    ep_step[o + i] = D.sp_step[int64_t(c) * D.sp_cap + i];
    log_t[base_log + o + i] = D.sp_t[int64_t(c) * D.sp_cap + i];
    log_gid[base_log + o + i] = D.gid0 + uint32_t(c);
  }
}

__global__ void k_spike_total(const int32_t* sp_count, const int64_t* sp_scan, int32_t n,
                              unsigned long long* ctr_ep, unsigned long long* ctr_log) {
  const int64_t tot = n > 0 ? sp_scan[n - 1] + sp_count[n - 1] : 0;
  *ctr_ep = static_cast<unsigned long long>(tot);
  *ctr_log += static_cast<unsigned long long>(tot);
}

__global__ void k_left_count(const int64_t* ev_begin, const int64_t* ev_cursor, int32_t n,
                             int64_t* left) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) left[c] = ev_begin[c + 1] - ev_cursor[c];
}

// warp per cell: copy the undelivered tail, rebased to the next epoch's base
__global__ void k_leftover(const uint64_t* keys, const int64_t* ev_begin, const int64_t* ev_cursor,
                           const int64_t* left_scan, int32_t n, uint64_t* out, uint64_t rebase) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= n) return;
  const int64_t a = ev_cursor[c], b = ev_begin[c + 1], o = left_scan[c];
  for (int64_t i = a + lane; i < b; i += 32) out[o + (i - a)] = keys[i] - rebase;
}

__global__ void k_left_total(const int64_t* left, const int64_t* left_scan, int32_t n,
                             unsigned long long* ctr) {
  *ctr = static_cast<unsigned long long>(n > 0 ? left_scan[n - 1] + left[n - 1] : 0);
}

// ---------------------------------------------------------------------------
// fast-forward (engine.cpp:947-1034)
// ---------------------------------------------------------------------------
__global__ void k_ff_pending(McgDev D, int32_t n_fifos, int32_t* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_fifos && D.fifos[i].head < D.fifos[i].tail) atomicOr(flag, 1);
}

// zero calcium, STDP traces, kernels and active lists (engine.cpp:961-969)
__global__ void k_ff_reset(McgDev D, int64_t n_cg) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n_cg) return;
  McgCellGroup& G = D.cgs[g];
  const McgSpec& S = D.specs[G.spec];
  for (int i = 0; i < G.size; ++i) {
    const int64_t j = G.inst + i;
    if (S.kind == MCG_SYN_STC_CHARGE) D.i_stc_c[j] = 0.0;
    if (S.kind == MCG_SYN_STDP_COND) {
      D.i_stdp_pre[j] = 0.0;
      D.i_stdp_post[j] = 0.0;
    }
    D.i_kernel[j] = 0.0;
  }
  G.active_n = 0;
}

