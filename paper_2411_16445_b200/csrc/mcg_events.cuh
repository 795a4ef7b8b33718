// mcg_events.cuh — device-resident event pipeline of the epoch loop.
//
// Replaces the reference's per-cell inboxes + std::sort + serial exchange
// (engine.cpp:831-889, 916-925) with:
//   k_inbox        generate_source_events for the epoch (Poisson draws on the
//                  device) and the spike exchange of the previous epoch: every
//                  EventRec becomes one 64-bit key  (delivery step << R) | rank
//                  appended to the destination cell's incoming buffer.  The
//                  rank orders edges by (src, seq) — EventOrder (:25-31) — with
//                  source edges (src = 0xFFFFFFFF) after all cell edges.
//   (k_epoch)      each cell's warp sorts its incoming keys and merges them
//                  into its pending list (mcg_epoch.cuh)
//   k_spike_write  ordered compaction of the epoch's spikes (gid, then step:
//                  the order exchange() appends them, :877-888) behind a CUB scan
// All epoch parameters are read from device memory, so a batch of epochs is
// one CUDA graph replayed without host round trips.  A buffer overflow sets
// `abort` (first epoch index + 1); every later kernel of the batch returns at
// entry, and the host grows the buffers and resumes at that epoch — the
// expansion only ever writes the incoming buffers, so no state is lost.
#pragma once
#include "mcg_device.cuh"

struct McgSrcTask {
  int32_t source;
  int32_t type;        // MCG_SRC_*
  int32_t window;      // poisson window
  int32_t pad;
  int64_t a, b;        // poisson: window step bounds; scripted: [first,last) into steps
  double prob;         // poisson: rate*dt*1e-3
  double r_t0, r_period;
  int64_t r_count;
};

struct McgEv {
  const McgSrcTask* tasks;
  int32_t n_tasks;
  const int64_t* scripted_steps;
  const int64_t* src_edge_off;
  const int64_t* src_edges;
  const int32_t* e_dst;
  const int64_t* e_delay;
  const int64_t* out_begin;   // per global gid
  const int64_t* out_end;
  uint64_t* inc;
  int32_t* inc_n;
  int32_t inc_cap;
  const int32_t* pend_off;
  const int32_t* pend_n;
  int32_t pend_cap;
  int32_t rank_bits;
  const int64_t* ctl;         // [0] batch base step, [1] target step, [2] epoch length
  int32_t* abort;
  const uint32_t* ep_gid;     // previous epoch's spikes (ordered)
  const int64_t* ep_step;
  const unsigned long long* ep_n;
  uint64_t seed;
  double dt;
};

// epoch j of the batch: [s0, s1); false if beyond the target
__device__ __forceinline__ bool mcg_epoch_bounds(const int64_t* ctl, int32_t j, int64_t& s0,
                                                 int64_t& s1) {
  s0 = ctl[0] + int64_t(j) * ctl[2];
  s1 = s0 + ctl[2];
  if (s1 > ctl[1]) s1 = ctl[1];
  return s0 < ctl[1];
}

__device__ __forceinline__ void mcg_push(const McgEv& E, int32_t j, int64_t rank, int64_t step) {
  const int32_t dst = E.e_dst[rank];
  const int32_t pos = atomicAdd(&E.inc_n[dst], 1);
  if (pos >= E.inc_cap || (E.pend_n[dst] - E.pend_off[dst]) + pos + 1 > E.pend_cap) {
    atomicCAS(E.abort, 0, j + 1);
    return;
  }
  E.inc[int64_t(dst) * E.inc_cap + pos] = (uint64_t(step) << E.rank_bits) | uint64_t(rank);
}

// source events for [s0, s1) (engine.cpp:831-873) and the previous epoch's
// spikes (engine.cpp:875-889: delivery at em.step + 1 + delay)
__global__ void k_inbox(McgEv E, int32_t j, int64_t max_len) {
  if (*E.abort) return;
  int64_t s0, s1;
  if (!mcg_epoch_bounds(E.ctl, j, s0, s1)) return;
  const int64_t len = s1 - s0;
  const int64_t nthr = int64_t(gridDim.x) * blockDim.x;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  // ---- sources: one thread per (task, step)
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
      } else if (T.r_period > 0) {  // regular
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
  // ---- spikes of the previous epoch: one warp per spike, lanes over out-edges
  const int lane = threadIdx.x & 31;
  const int64_t nw = nthr >> 5;
  const int64_t n_sp = static_cast<int64_t>(*E.ep_n);
  for (int64_t w = tid >> 5; w < n_sp; w += nw) {
    const uint32_t gid = E.ep_gid[w];
    const int64_t st = E.ep_step[w];
    const int64_t e0 = E.out_begin[gid], e1 = E.out_end[gid];
    for (int64_t r = e0 + lane; r < e1; r += 32) mcg_push(E, j, r, st + 1 + E.e_delay[r]);
  }
}

// ordered spike compaction: the epoch list (gid, step) feeds the next epoch's
// k_inbox, the batch log (t, gid) is copied to the host after the batch
__global__ void k_spike_write(const McgDev D, int32_t j, const int64_t* sp_scan, uint32_t* ep_gid,
                              int64_t* ep_step, double* log_t, uint32_t* log_gid,
                              const unsigned long long* log_n) {
  if (*D.abort) return;
  int64_t s0, s1;
  if (!mcg_epoch_bounds(D.ctl, j, s0, s1)) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= D.n_cells) return;
  const int k = D.sp_count[c];
  if (k == 0) return;
  const int64_t o = sp_scan[c];
  const int64_t base = static_cast<int64_t>(*log_n);
  for (int i = 0; i < k; ++i) {
    ep_gid[o + i] = D.gid0 + uint32_t(c);
    ep_step[o + i] = D.sp_step[int64_t(c) * D.sp_cap + i];
    log_t[base + o + i] = D.sp_t[int64_t(c) * D.sp_cap + i];
    log_gid[base + o + i] = D.gid0 + uint32_t(c);
  }
}

__global__ void k_spike_total(const McgDev D, int32_t j, const int64_t* sp_scan,
                              unsigned long long* ep_n, unsigned long long* log_n) {
  if (*D.abort) return;
  int64_t s0, s1;
  if (!mcg_epoch_bounds(D.ctl, j, s0, s1)) return;
  const int n = D.n_cells;
  const int64_t tot = n > 0 ? sp_scan[n - 1] + D.sp_count[n - 1] : 0;
  *ep_n = static_cast<unsigned long long>(tot);
  *log_n += static_cast<unsigned long long>(tot);
}

// after growing the inbox capacities: move each cell's pending keys into the
// new double buffer (selected half, from offset 0)
__global__ void k_pend_regrow(const uint64_t* old_pend, int32_t old_cap, uint64_t* new_pend,
                              int32_t new_cap, int32_t* pend_sel, int32_t* pend_off,
                              int32_t* pend_n, int32_t n_cells) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= n_cells) return;
  const int sel = pend_sel[c];
  const int a = pend_off[c], b = pend_n[c];
  const uint64_t* src = old_pend + (int64_t(c) * 2 + sel) * old_cap;
  uint64_t* dst = new_pend + (int64_t(c) * 2 + sel) * new_cap;
  for (int i = a + lane; i < b; i += 32) dst[i - a] = src[i];
  __syncwarp();
  if (lane == 0) {
    pend_off[c] = 0;
    pend_n[c] = b - a;
  }
}
