// mcg_events.cuh — device-resident event pipeline of the epoch loop.
//
// Replaces the reference's per-cell inboxes + std::sort + serial exchange
// (engine.cpp:831-889, 916-925): generate_source_events (Poisson draws on the
// device) and the spike exchange of the previous epoch turn every EventRec
// into one 64-bit key (delivery step << R) | rank appended to the destination
// cell's incoming buffer (mcg_expand, mcg_batch.cuh).  The rank orders edges
// by (src, seq) — EventOrder (:25-31) — with source edges (src = 0xFFFFFFFF)
// after all cell edges, so sorting keys restores the reference's delivery
// order; each cell sorts its incoming keys and merges them into its pending
// list at epoch entry.  An overflow sets `abort` (epoch index + 1); the batch
// kernel stops after that epoch's expansion and the host grows the buffers
// and resumes there — the expansion only writes the incoming buffers, so no
// state is lost.
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
  const McgSrcTask* tasks;    // Poisson windows first, then regular / scripted sources
  int32_t n_tasks;
  int32_t n_poisson;          // tasks [0, n_poisson) are Poisson windows
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
  uint64_t seed;
  double dt;
  // sharded mode: the previous epoch's spikes of all ranks (the caller's
  // allgather of every rank's send block), x_world blocks of x_block int64:
  // [count, (gid, step, t bits) x cap]; nullptr on a single shard (local spikes)
  const int64_t* x_recv;
  int32_t x_world;
  int64_t x_block;
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
