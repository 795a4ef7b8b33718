// mcg_resolve.cuh — connection resolution on the device (Impl::build,
// engine.cpp:357-391): the instance each connection lands on (append_instance
// for appended groups, select_target's SelectionCursor for pre-placed ones)
// and every local edge written into its slot of the rank order (EventOrder,
// engine.cpp:25-31: src key ascending, sources last, seq = connection index).
//
// The host's pass 0 (mcg_build.cpp) has already run the reference's checks in
// its order and counted; what is left is two stable orders of the connection
// list, both of which a stable radix sort by key gives directly:
//   * by (cell, group): the connections to one group in connection order.
//     Appended group: the instance is the connection's rank in that run
//     (append_instance, one new instance per connection).  Pre-placed group:
//     the cursor has advanced once per earlier ROUND_ROBIN connection to the
//     group (ROUND_ROBIN_HALT reads it, UNIVALENT returns 0 and has size 1),
//     so the instance is (earlier round-robin connections) % count.
//   * by src key: the rank of an edge is its position in that order; the
//     source bucket (key n_cells) sorted again by source id gives the
//     per-source CSR (src_edges), each source's edges in rank order.
// Every output equals the host's pass 1 bit for bit (tests/test_gpu_resolve.py).
#pragma once
#include <stdint.h>

namespace mcg_rs {

constexpr uint8_t kRoundRobin = MCG_POLICY_ROUND_ROBIN;
constexpr uint8_t kUnivalent = MCG_POLICY_UNIVALENT;

struct Conn {
  const uint8_t* from_source;
  const uint32_t* src;
  const uint32_t* dst;
  const int32_t* group;
  const uint8_t* policy;
  const double* weight;
  const double* delay_ms;
  int64_t n;
};

// sort keys: (cell, group) index and src key of every connection; connections
// to other ranks' cells sort last (key n_cg / n_cells + 1) and are dropped
__global__ void k_keys(Conn C, uint32_t g0, uint32_t g1, const int64_t* cg_off, uint32_t n_cg,
                       uint32_t n_cells, uint32_t* key_cg, uint32_t* key_src, uint32_t* val) {
  const int64_t ci = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ci >= C.n) return;
  const uint32_t dst = C.dst[ci];
  const bool local = dst >= g0 && dst < g1;
  key_cg[ci] = local ? uint32_t(cg_off[dst - g0] + C.group[ci]) : n_cg;
  key_src[ci] = !local ? n_cells + 1 : (C.from_source[ci] ? n_cells : C.src[ci]);
  val[ci] = uint32_t(ci);
}

// round-robin flags in (cell, group) order, for the cursor scan
__global__ void k_rr_flags(Conn C, const uint32_t* perm, int64_t n_local, int32_t* flag) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= C.n) return;
  flag[p] = (p < n_local && C.policy[perm[p]] == kRoundRobin) ? 1 : 0;
}

// instance of every local connection; appended instances take its weight
__global__ void k_instances(Conn C, const uint32_t* key_cg, const uint32_t* perm, int64_t n_local,
                            const int32_t* rr_scan, const int64_t* cg_conn_off, const int32_t* cg_count,
                            const McgCellGroup* cgs, uint32_t* inst_of, double* i_weight) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n_local) return;
  const uint32_t ci = perm[p], cg = key_cg[p];
  const int64_t s0 = cg_conn_off[cg];
  const int32_t count = cg_count[cg];
  uint32_t inst;
  if (count == 0) {
    inst = uint32_t(p - s0);
    i_weight[cgs[cg].inst + inst] = C.weight[ci];
  } else if (C.policy[ci] == kUnivalent) {
    inst = 0;
  } else {
    inst = uint32_t((rr_scan[p] - rr_scan[s0]) % count);
  }
  inst_of[ci] = inst;
}

struct Edges {
  int32_t *dst, *group, *comp;
  uint32_t *inst, *src, *seq;
  double *weight, *wcf;
  int64_t* delay;
};

// the edge at rank e: connection perm[e] (ceil_steps, engine.cpp:21-23, with
// the host build's operations; static-charge payload w * cf[comp],
// engine.cpp:455-459)
__global__ void k_edges(Conn C, const uint32_t* perm, int64_t ne, uint32_t g0, double dt,
                        const int64_t* cg_off, const uint8_t* cg_static, const int32_t* cg_comp,
                        const double* cg_cf, const uint32_t* inst_of, Edges E,
                        unsigned long long* max_delay, uint32_t* src_key, uint32_t* src_val, int64_t src0) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const uint32_t ci = perm[e];
  const int c = int(C.dst[ci] - g0);
  const int32_t gi = C.group[ci];
  const int64_t cg = cg_off[c] + gi;
  const double w = C.weight[ci];
  const bool from_src = C.from_source[ci] != 0;
  const int64_t d = int64_t(ceil(__dsub_rn(__ddiv_rn(C.delay_ms[ci], dt), 1e-9)));
  E.dst[e] = c;
  E.group[e] = gi;
  E.inst[e] = inst_of[ci];
  E.weight[e] = w;
  E.delay[e] = d;
  E.src[e] = from_src ? 0xFFFFFFFFu : C.src[ci];
  E.seq[e] = ci;
  if (cg_static[cg]) {
    E.comp[e] = cg_comp[cg];
    E.wcf[e] = __dmul_rn(w, cg_cf[cg]);
  } else {
    E.comp[e] = -1;
    E.wcf[e] = 0.0;
  }
  atomicMax(max_delay, static_cast<unsigned long long>(d));
  if (from_src) {  // the source bucket, re-sorted by source id for the CSR
    src_key[e - src0] = C.src[ci];
    src_val[e - src0] = uint32_t(e);
  }
}

__global__ void k_u32_to_i64(const uint32_t* a, int64_t n, int64_t* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i];
}

// worst-case inbox occupancy per destination (Engine::size_inboxes_for_worst_case):
// cell edges carry `per_cell` events per epoch, source edges their source's
__global__ void k_worst_cell(const int32_t* e_dst, const uint32_t* e_src, const int64_t* e_delay, int64_t ne,
                             int64_t per, int64_t L, unsigned long long* inc, unsigned long long* pend) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne || e_src[e] == 0xFFFFFFFFu) return;
  const int c = e_dst[e];
  const int64_t d = e_delay[e];
  atomicAdd(inc + c, static_cast<unsigned long long>(per));
  atomicAdd(pend + c, static_cast<unsigned long long>(per * ((d + L - 1) / L + 1)));
}
__global__ void k_worst_src(const int32_t* e_dst, const int64_t* e_delay, const int64_t* src_edges,
                            const int64_t* per_k, int64_t nk, int64_t L, unsigned long long* inc,
                            unsigned long long* pend) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nk) return;
  const int64_t e = src_edges[k];
  const int c = e_dst[e];
  const int64_t d = e_delay[e], per = per_k[k];
  atomicAdd(inc + c, static_cast<unsigned long long>(per));
  atomicAdd(pend + c, static_cast<unsigned long long>(per * ((d + L - 1) / L + 1)));
}

inline unsigned blocks(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }

}  // namespace mcg_rs
