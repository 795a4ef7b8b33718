// mcg_warp.cuh — the warp-group kernel k_warp: Engine::advance_to
// (engine.cpp:909-945) for networks of LIF cells with charge-type synapses
// (static_charge, stc_charge), the class of every consolidation network
// (network.cpp:426-598; BASELINE configs 1, 3, 4, 5).
//
// Cells are independent inside a min-delay epoch (engine.cpp:913-942), so a
// group of G cells belongs to ONE warp for the whole epoch and runs all of
// step_cell (engine.cpp:541-783) with nothing but __syncwarp between phases:
//   lane k < G        cell k's ordered folds: event delivery, delayed calcium,
//                     the SPS fold, background current, detection, probes
//   lanes over items  the cell group's active STC synapses (below), the
//                     post-spike hook, inbox sorts, noise draws
//   lane per system   the Hines sweeps: (cell, V or species, chain side) on
//                     2 (1 + S) lanes per cell (mcg_sweep.cuh), point cells'
//                     closed forms on the same lanes
// There is no CTA-wide barrier inside an epoch: every warp advances at its own
// pace and the SM interleaves the warps' latency-bound chains.  The grid
// barrier remains once per expansion and once per epoch (mcg_expand's inboxes).
//
// Lazy calcium.  A resting STC synapse (h bitwise at h0, |h - h0| folded as 0,
// calcium above neither threshold, a finite PRP level) takes a step that only
// decays its calcium, c *= exp(-dt/tau_c) (mcg_stc_at_rest).  While nothing
// touches it, k such steps are k sequential multiplications by the same
// constant, so the synapse is not visited at all: it keeps (c, t) = its
// calcium just before the STC update of step t, and whoever touches it next
// (delayed calcium, the post-spike hook, a probe, the end of advance_to)
// first applies the s - t multiplications one by one (mcg_decay_steps), which
// are exactly the reference's roundings.  Only synapses that are not at rest
// are in the per-cell active mask and run the full update every step; one
// leaves the mask when its update leaves it at rest again.  This needs the
// thresholds >= 0 and 0 <= cf <= 1 (a resting calcium stays below them) and
// a late step that is a no-op at rest (McgStcRest::late_noop); otherwise every
// synapse stays in the mask.
#pragma once
#include <cooperative_groups.h>

#include "mcg_batch.cuh"

#define MCG_WG_MAX 8  // cells per warp group
#define MCG_WPH_N 16   // phase-timing slots (MCG_PHASE_TIMING)

// optional per-phase cycle accounting: lane 0 of each warp, one row per warp
__shared__ unsigned long long mcg_wph[8][MCG_WPH_N + 1];
#define WPH(i)                                                      \
  do {                                                              \
    if (A.phase && lane == 0) {                                     \
      const unsigned long long t_ = clock64();                      \
      unsigned long long* r_ = mcg_wph[threadIdx.x >> 5];           \
      r_[i] += t_ - r_[MCG_WPH_N];                                  \
      r_[MCG_WPH_N] = t_;                                           \
    }                                                               \
  } while (0)
#define MCG_MW_MAX 32  // STC mask words per cell (<= 1024 STC instances)

struct McgWarpArgs {
  McgEv E;
  int32_t n_epochs;      // epochs in this launch
  int32_t G;             // cells per group
  int32_t n_groups;      // groups (cell g + k * n_groups, k < G: strided)
  int32_t resident;      // every warp owns at most one group: staged for the launch
  int32_t m;             // compartments per cell block (smem_n)
  int32_t S;             // species per cell block (sp_max)
  int32_t P;             // chain positions per system (0: no chain kinds)
  int32_t MW;            // STC mask words per cell
  int32_t cell_doubles;  // (2 + S) m: V | SP (stride n) | rhs_current
  int32_t ev_cap;        // staged network events per warp
  int32_t warp_doubles;  // per-warp region of the dynamic shared memory
  int32_t kind_doubles;  // staged kind blocks (mcg_kind_block_doubles each)
  int32_t n_kinds;
  int32_t n_specs_sm;
  int32_t lazy;          // lazy calcium on
  int32_t cu_every;      // epochs between catch-ups of the resting calcium
  unsigned long long* phase;  // optional per-phase cycle totals (MCG_PHASE_TIMING)
  int32_t dbg;           // development switches (MCG_WARP_DBG)
  int64_t dbg_s;         // first traced step (MCG_WARP_DBG_S)
  const int32_t* kb_off;  // per kind: offset of its staged block (doubles)
  uint32_t* stc_mask;    // per cell MW words: STC instances updated every step
  int64_t* stc_t;        // per STC instance: step of its lazily kept calcium
  double* log_t;         // spike log of the launch (as McgBatchArgs)
  uint32_t* log_gid;
  unsigned long long* log_n;
  int4* chunks;          // (epoch, group, offset, count)
  unsigned long long* chunk_n;
  int64_t* x_send;       // sharded export (as McgBatchArgs)
  int64_t x_cap;
  int32_t epoch_base;    // added to the launch's epoch index in the log chunks
  int32_t no_abort;      // inboxes sized for the worst case: no expansion can overflow
};

// one staged network event of the epoch (the pending list's head, with the
// edge payload resolved): static charge carries w * cf[comp] and comp
struct McgWEv {
  double w;
  uint32_t inst;
  uint32_t src;
  uint16_t comp;
  uint8_t group;
  uint8_t nz;            // raw weight nonzero
  int32_t so;            // step - s0
};

// per cell of a warp group (shared memory); lane k owns cell k's record
struct McgWCell {
  int64_t stc_inst;      // first STC instance (global index)
  int64_t f_base, f_head, f_tail;  // delayed-calcium queue (McgFifo), resident copy
  int64_t refr;          // refractory_until
  int64_t next_due;      // step of the queue's head entry (INT64_MAX: empty)
  int64_t ca_delay;
  uint64_t nk;           // next pending key (unstaged delivery)
  double det_prev;
  double vol, rvol, cf;  // of the STC placement's compartment
  double h0, cpre_s, cpost_s, ccf;  // STC spec fields on the delivery / post chains
  double prod;
  double rc_val;         // rhs_current at noise_comp this step (0.0 + I_bg); others are 0.0
  double sp_den, sp_rden;  // n == 1 species closed form: cap + gs, its reciprocal (per lane)
  int32_t c;             // local cell index (-1: empty slot)
  int32_t kind;
  int32_t sel, cur, end; // pending list: buffer half, cursor, end
  int32_t ev_cur, ev_end;
  int32_t staged;
  int32_t nsp;
  int32_t stc_n, stc_comp, stc_spec, stc_gi, fifo, f_cap;
  uint32_t iseq;
  int32_t armed, lif, noise, fired, refractory, has_current, n_groups;
  int32_t probe0, probe1;  // the cell's probe range (D.probe_off), read once per entry
  int32_t prp_off;       // mcg_smem offset of PRP at the STC compartment (-1: no pool)
  int32_t sps_off;       // mcg_smem offset of SPS at the STC compartment (-1: none)
  int32_t base;          // mcg_smem offset of the cell block
  int32_t late;          // stc_late_step runs (the kind has a PRP pool)
  int32_t pad;
  uint8_t gk[8];         // synapse kind per group
};

// shared-memory carve-up of one warp (offsets in doubles into mcg_smem)
struct McgWarpSm {
  int cells;   // G cell blocks
  int r2c;     // G x (1 + S) x P chain scratch
  int nb;      // G x 32 background-noise draws
  int db;      // 32 SPS deltas of one STC round
  int ic;      // 32 int32: cell slot of each item of the round
  int ev;      // ev_cap McgWEv
  int rec;     // G McgWCell
  int mask;    // G x MW uint32
  int mbar;    // mbarrier of the warp's bulk (TMA) staging copies + its phase word
};

__host__ __device__ __forceinline__ int mcg_warp_region_doubles(int G, int m, int S, int P, int MW,
                                                                int ev_cap) {
  const int rec = (int(sizeof(McgWCell)) + 7) / 8;
  const int d = G * (2 + S) * m + G * (1 + S) * P + G * 32 + 32 + 16 + ev_cap * 3 + G * rec +
                (G * MW + 1) / 2 + 2 + 2;
  return (d + 1) & ~1;  // even: 16-byte aligned warp regions (bulk copies)
}

__device__ __forceinline__ McgWarpSm mcg_warp_sm(const McgWarpArgs& A, int w) {
  McgWarpSm R;
  const int base0 = (A.kind_doubles + (A.n_kinds * int(sizeof(McgKind)) + 7) / 8 +
                     (A.n_specs_sm * int(sizeof(McgSpec)) + 7) / 8 + 1) & ~1;  // 16-byte aligned
  const int b = base0 + w * A.warp_doubles;
  R.cells = b;
  R.r2c = R.cells + A.G * A.cell_doubles;
  R.nb = R.r2c + A.G * (1 + A.S) * A.P;
  R.db = R.nb + A.G * 32;
  R.ic = R.db + 32;
  R.ev = R.ic + 16;
  R.rec = R.ev + A.ev_cap * 3;
  R.mask = R.rec + A.G * ((int(sizeof(McgWCell)) + 7) / 8);
  R.mbar = R.mask + (A.G * A.MW + 1) / 2 + 2;
  return R;
}

// ---- bulk (TMA) copies of a group's compartment blocks ----------------------
// cp.async.bulk moves a cell's V block and its species blocks (contiguous in
// global memory and in the cell's shared-memory block) as one transfer each,
// completing on the warp's mbarrier; blocks whose addresses or sizes are not
// 16-byte multiples take the element-wise path
__device__ __forceinline__ uint32_t mcg_sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ bool mcg_bulk_ok(const void* g, const void* sm, int bytes) {
  return bytes > 0 && (bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0 && (mcg_sa(sm) & 15) == 0;
}
__device__ __forceinline__ void mcg_mbar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mcg_mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mcg_mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mcg_bulk_load(void* sm, const void* g, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          mcg_sa(sm)),
      "l"(g), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mcg_bulk_store(void* g, const void* sm, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(g), "r"(mcg_sa(sm)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ McgKind* mcg_warp_kinds(const McgWarpArgs& A) {
  return reinterpret_cast<McgKind*>(mcg_smem + A.kind_doubles);
}
__device__ __forceinline__ const McgSpec* mcg_warp_specs(const McgDev& D, const McgWarpArgs& A) {
  if (A.n_specs_sm == 0) return D.specs;
  return reinterpret_cast<const McgSpec*>(mcg_smem + A.kind_doubles +
                                          (A.n_kinds * int(sizeof(McgKind)) + 7) / 8);
}

// k sequential at-rest steps of a calcium value (c *= cf, the reference's
// per-step rounding); a zero stays zero
__device__ __forceinline__ double mcg_decay_steps(double c, double cf, int64_t k) {
  while (k >= 4 && c != 0.0) {
    c *= cf;
    c *= cf;
    c *= cf;
    c *= cf;
    k -= 4;
  }
  while (k > 0 && c != 0.0) {
    c *= cf;
    --k;
  }
  return c;
}

// n-th (0-based) set bit of x
__device__ __forceinline__ int mcg_nth_bit(uint32_t x, int n) {
  return __fns(x, 0, n + 1);
}

// ---- group entry: cell records, compartment state, STC masks ---------------
__device__ void mcg_wg_enter(const McgDev& D, const McgWarpArgs& A, const McgWarpSm& W, int g,
                             int lane) {
  const McgKind* kinds = mcg_warp_kinds(A);
  const McgSpec* specs = mcg_warp_specs(D, A);
  McgWCell* R = reinterpret_cast<McgWCell*>(mcg_smem + W.rec);
  const int m = A.m;
  if (lane < A.G) {
    McgWCell& X = R[lane];
    const int c = g + lane * A.n_groups;
    X.c = c < D.n_cells ? c : -1;
    X.base = W.cells + lane * A.cell_doubles;
    if (X.c >= 0) {
      const int kind = D.cell_kind[c];
      const McgKind& K = kinds[kind];
      X.kind = kind;
      X.sel = D.pend_sel[c];
      X.cur = D.pend_off[c];
      X.end = D.pend_n[c];
      X.refr = D.refr_until[c];
      X.det_prev = D.det_prev[c];
      X.armed = D.armed[c];
      X.iseq = D.internal_seq[c];
      X.lif = (K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT) ? 1 : 0;
      X.noise = (X.lif && K.has_bg && K.sig_bg != 0.0) ? 1 : 0;
      X.n_groups = K.n_groups;
      X.stc_n = 0;
      X.fifo = -1;
      X.prp_off = X.sps_off = -1;
      X.late = K.prp_idx >= 0 ? 1 : 0;
      X.nsp = 0;
      X.staged = 0;
      X.next_due = INT64_MAX;
      X.probe0 = D.probe_off[c];
      X.probe1 = D.probe_off[c + 1];
      const int64_t cg0 = D.cg_off[c];
      for (int gi = 0; gi < K.n_groups && gi < 8; ++gi) {
        const McgCellGroup Gr = D.cgs[cg0 + gi];
        const McgSpec& S = specs[Gr.spec];
        X.gk[gi] = static_cast<uint8_t>(S.kind);
        if (S.kind != MCG_SYN_STC_CHARGE) continue;
        X.stc_inst = Gr.inst;
        X.stc_n = Gr.size;
        X.stc_comp = S.comp;
        X.stc_spec = Gr.spec;
        X.stc_gi = gi;
        X.fifo = Gr.fifo;
        X.ca_delay = S.ca_delay;
        X.h0 = S.h0;
        X.cpre_s = S.cpre_s;
        X.cpost_s = S.cpost_s;
        X.ccf = S.cf;
        X.vol = D.k_volume[K.arr + S.comp];
        X.rvol = D.k_rvol[K.arr + S.comp];
        X.cf = D.k_cf[K.arr + S.comp];
        if (K.prp_idx >= 0) X.prp_off = X.base + m + K.prp_idx * K.n + S.comp;
        if (K.sps_idx >= 0) X.sps_off = X.base + m + K.sps_idx * K.n + S.comp;
      }
      if (X.fifo >= 0) {
        const McgFifo F = D.fifos[X.fifo];
        X.f_base = F.base;
        X.f_cap = F.cap;
        X.f_head = F.head;
        X.f_tail = F.tail;
        if (F.head < F.tail) X.next_due = D.fifo_step[F.base + mcg_mod(F.head, F.cap)];
      }
    }
  }
  __syncwarp();
  WPH(14);  // cell records done (the rest of the entry counts as "groups")
  // compartment state: a cell's V block and its species blocks are
  // contiguous in global memory and in its shared-memory block, so each is one
  // bulk (TMA) copy when 16-byte aligned; the rest go element by element
  // (cp.async), every load in flight at once
  const uint32_t bar = mcg_sa(mcg_smem + W.mbar);
  uint32_t* bphase = reinterpret_cast<uint32_t*>(mcg_smem + W.mbar + 1);
  uint32_t tx = 0;
  uint32_t bulk_mask = 0;  // bit 2k: cell k's V block by bulk copy, bit 2k + 1: its species
  for (int k = 0; k < A.G; ++k) {
    const int c = R[k].c;
    if (c < 0) continue;
    const McgKind& K = kinds[R[k].kind];
    const int n = K.n;
    if (mcg_bulk_ok(D.v + D.comp_off[c], mcg_smem + R[k].base, n * 8)) {
      bulk_mask |= 1u << (2 * k);
      tx += uint32_t(n) * 8u;
    }
    if (K.n_species > 0 &&
        mcg_bulk_ok(D.species + D.sp_off[c], mcg_smem + R[k].base + m, K.n_species * n * 8)) {
      bulk_mask |= 2u << (2 * k);
      tx += uint32_t(K.n_species * n) * 8u;
    }
  }
  if (tx > 0) {
    if (lane == 0) mcg_mbar_expect(bar, tx);
    __syncwarp();
    if (lane < A.G && R[lane].c >= 0) {
      const int c = R[lane].c;
      const McgKind& K = kinds[R[lane].kind];
      if (bulk_mask & (1u << (2 * lane)))
        mcg_bulk_load(mcg_smem + R[lane].base, D.v + D.comp_off[c], uint32_t(K.n) * 8u, bar);
      if (bulk_mask & (2u << (2 * lane)))
        mcg_bulk_load(mcg_smem + R[lane].base + m, D.species + D.sp_off[c], uint32_t(K.n_species * K.n) * 8u,
                      bar);
    }
  }
  // the blocks that are not bulk-copied, element by element, cell by cell
  for (int k = 0; k < A.G; ++k) {
    const int c = R[k].c;
    if (c < 0) continue;
    const McgKind& K = kinds[R[k].kind];
    const int n = K.n;
    const int nb = (bulk_mask & (1u << (2 * k)) ? 0 : n) + (bulk_mask & (2u << (2 * k)) ? 0 : K.n_species * n);
    for (int e = lane; e < nb; e += 32) {
      // e < n_v: V element e (when V is element-wise); then the species
      const bool v_el = !(bulk_mask & (1u << (2 * k)));
      const int nv = v_el ? n : 0;
      const bool is_v = e < nv;
      const int j = is_v ? e : e - nv;  // species: offset in the (species x n) block
      const double* src = is_v ? D.v + D.comp_off[c] + j : D.species + D.sp_off[c] + j;
      double* dst = mcg_smem + R[k].base + (is_v ? j : m + j);
      const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src) : "memory");
    }
  }
  uint32_t* MK = reinterpret_cast<uint32_t*>(mcg_smem + W.mask);
  for (int idx = lane; idx < A.G * A.MW; idx += 32) {
    const int k = idx / A.MW, w = idx - k * A.MW;
    const int c = R[k].c;
    MK[idx] = (c >= 0 && w * 32 < R[k].stc_n) ? A.stc_mask[int64_t(c) * A.MW + w] : 0u;
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  if (tx > 0) {
    const uint32_t ph = *bphase;
    mcg_mbar_wait(bar, ph & 1u);
    __syncwarp();
    if (lane == 0) *bphase = ph + 1;
  }
  __syncwarp();
}

// ---- group exit: state back to global memory --------------------------------
__device__ void mcg_wg_exit(const McgDev& D, const McgWarpArgs& A, const McgWarpSm& W, int lane) {
  const McgKind* kinds = mcg_warp_kinds(A);
  McgWCell* R = reinterpret_cast<McgWCell*>(mcg_smem + W.rec);
  const int m = A.m;
  // blocks that entered by bulk copy leave by bulk copy (the shared-memory
  // writes of the epoch made visible to the async proxy first); the rest
  // element by element
  uint32_t bulk_mask = 0;
  for (int k = 0; k < A.G; ++k) {
    const int c = R[k].c;
    if (c < 0) continue;
    const McgKind& K = kinds[R[k].kind];
    const int n = K.n;
    if (mcg_bulk_ok(D.v + D.comp_off[c], mcg_smem + R[k].base, n * 8)) bulk_mask |= 1u << (2 * k);
    if (K.n_species > 0 &&
        mcg_bulk_ok(D.species + D.sp_off[c], mcg_smem + R[k].base + m, K.n_species * n * 8))
      bulk_mask |= 2u << (2 * k);
  }
  if (bulk_mask) {
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    if (lane < A.G && R[lane].c >= 0) {
      const int c = R[lane].c;
      const McgKind& K = kinds[R[lane].kind];
      if (bulk_mask & (1u << (2 * lane)))
        mcg_bulk_store(D.v + D.comp_off[c], mcg_smem + R[lane].base, uint32_t(K.n) * 8u);
      if (bulk_mask & (2u << (2 * lane)))
        mcg_bulk_store(D.species + D.sp_off[c], mcg_smem + R[lane].base + m, uint32_t(K.n_species * K.n) * 8u);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      // the shared-memory blocks are reused by the next group: wait until the
      // copies have read them (their global writes complete before the
      // grid barrier: the wait_group at the end of the warp's epoch)
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
  }
  for (int k = 0; k < A.G; ++k) {
    const int c = R[k].c;
    if (c < 0) continue;
    const McgKind& K = kinds[R[k].kind];
    const int n = K.n;
    const bool v_el = !(bulk_mask & (1u << (2 * k)));
    const int nv = v_el ? n : 0;
    const int nb = nv + (bulk_mask & (2u << (2 * k)) ? 0 : K.n_species * n);
    for (int e = lane; e < nb; e += 32) {
      const bool is_v = e < nv;
      const int j = is_v ? e : e - nv;
      const double v = mcg_smem[R[k].base + (is_v ? j : m + j)];
      if (is_v) D.v[D.comp_off[c] + j] = v;
      else D.species[D.sp_off[c] + j] = v;
    }
  }
  const uint32_t* MK = reinterpret_cast<const uint32_t*>(mcg_smem + W.mask);
  for (int idx = lane; idx < A.G * A.MW; idx += 32) {
    const int k = idx / A.MW, w = idx - k * A.MW;
    const int c = R[k].c;
    if (c >= 0 && w * 32 < R[k].stc_n) A.stc_mask[int64_t(c) * A.MW + w] = MK[idx];
  }
  if (lane < A.G && R[lane].c >= 0) {
    const McgWCell& X = R[lane];
    const int c = X.c;
    D.refr_until[c] = X.refr;
    D.det_prev[c] = X.det_prev;
    D.armed[c] = X.armed;
    D.internal_seq[c] = X.iseq;
    if (X.fifo >= 0) {
      D.fifos[X.fifo].head = X.f_head;
      D.fifos[X.fifo].tail = X.f_tail;
    }
  }
  __syncwarp();
}

// calcium delivered to STC instance i of cell record X at step s (before the
// step's STC update): stc_on_pre_calcium / stc_on_post_calcium with the lazy
// decay applied first; a synapse the calcium lifts above a threshold joins
// the active mask
__device__ __forceinline__ void mcg_wg_calcium(const McgDev& D, const McgWarpArgs& A,
                                               const McgSpec& S, const McgWCell& X, uint32_t* mk,
                                               int i, int64_t t_now, double add) {
  const int64_t j = X.stc_inst + i;
  const uint32_t bit = 1u << (i & 31);
  if (A.lazy && !(mk[i >> 5] & bit)) {
    double c = mcg_decay_steps(D.i_stc_c[j], X.ccf, t_now - A.stc_t[j]);
    c += add;
    D.i_stc_c[j] = c;
    A.stc_t[j] = t_now;
    if (c > S.theta_p || c > S.theta_d) {
      mk[i >> 5] |= bit;
      if (A.dbg & 4) A.stc_t[j] = -1;
    }
    if ((A.dbg & 4) && i >= X.stc_n) printf("[k_warp] BAD calcium inst %d >= %d cell %d\n", i, X.stc_n, X.c);
  } else {
    D.i_stc_c[j] += add;
  }
}

// ---- epoch entry of cell slot k (whole warp): inbox sort and merge into the
// pending list (the reference's per-epoch inbox sort, engine.cpp:916-925),
// then the epoch's due network events staged into the warp's event buffer
// with their edge payload resolved
__device__ void mcg_wg_inbox(const McgDev& D, const McgWarpArgs& A, const McgWarpSm& W, int k,
                             int64_t s0, int64_t s1, int lane, int& ev_top) {
  McgWCell* R = reinterpret_cast<McgWCell*>(mcg_smem + W.rec);
  McgWCell& X = R[k];
  const int c = X.c;
  const int nin = D.inc_n[c];
  const uint64_t lim = uint64_t(s1) << D.rank_bits;
  if (lane == 0 && (A.dbg >> 8) == c + 1 && s0 >= A.dbg_s - 12 && s0 <= A.dbg_s + 5) {
    printf("[k_warp] inbox cell %d s0 %lld nin %d cur %d end %d sel %d:", c, (long long)s0, nin, X.cur, X.end, X.sel);
    for (int i = 0; i < nin && i < 8; ++i)
      printf(" %lld", (long long)(D.inc[int64_t(c) * D.inc_cap + i] >> D.rank_bits));
    printf("\n");
  }
  bool regs = false;
  uint64_t key = ~0ull;
  int nd = 0;
  if (X.cur >= X.end && nin <= 32) {
    // nothing pending from earlier epochs and a small inbox: sorted in
    // registers, staged from them (pend gets the same keys)
    if (nin > 0) {
      const uint64_t* in = D.inc + int64_t(c) * D.inc_cap;
      key = mcg_warp_sort_reg(lane < nin ? in[lane] : ~0ull, lane, nin);
      nd = __popc(__ballot_sync(MCG_FULL, lane < nin && key < lim));
      uint64_t* out = D.pend + (int64_t(c) * 2 + (1 - X.sel)) * D.pend_cap;
      if (lane < nin) out[lane] = key;
      __syncwarp();
      if (lane == 0) {
        X.end = nin;
        X.cur = 0;
        X.sel = 1 - X.sel;
      }
    }
    regs = true;
  } else if (nin > 0) {
    uint64_t* in = D.inc + int64_t(c) * D.inc_cap;
    if (nin > 1) mcg_warp_sort(in, nin, lane);
    __syncwarp();
    const uint64_t* pold = D.pend + (int64_t(c) * 2 + X.sel) * D.pend_cap;
    uint64_t* out = D.pend + (int64_t(c) * 2 + (1 - X.sel)) * D.pend_cap;
    if (X.cur >= X.end) {
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
  }
  __syncwarp();
  const uint64_t* pend = D.pend + (int64_t(c) * 2 + X.sel) * D.pend_cap;
  if (!regs) {
    for (int base = X.cur; base < X.end; base += 32) {
      const int i = base + lane;
      const unsigned bal = __ballot_sync(MCG_FULL, i < X.end && pend[i] < lim);
      nd += __popc(bal);
      if (bal != MCG_FULL) break;
    }
  }
  const int cur0 = X.cur, end0 = X.end;
  __syncwarp();
  if (ev_top + nd > A.ev_cap) {  // no room: this cell delivers from the pending list
    if (lane == 0) {
      X.staged = 0;
      X.nk = (cur0 < end0) ? pend[cur0] : ~0ull;
    }
    __syncwarp();
    return;
  }
  McgWEv* EV = reinterpret_cast<McgWEv*>(mcg_smem + W.ev);
  const uint64_t rank_mask = (1ull << D.rank_bits) - 1;
  for (int t = lane; t < nd; t += 32) {
    const uint64_t kk = regs ? key : pend[cur0 + t];
    const int64_t r = int64_t(kk & rank_mask);
    const int grp = D.e_group[r];
    const double w = D.e_weight[r];
    McgWEv e;
    e.group = static_cast<uint8_t>(grp);
    e.so = static_cast<int32_t>(int64_t(kk >> D.rank_bits) - s0);
    e.inst = D.e_inst[r];
    e.src = D.e_src[r];
    e.nz = w != 0.0 ? 1 : 0;
    e.comp = 0;
    e.w = w;
    if (X.gk[grp] == MCG_SYN_STATIC_CHARGE) {  // apply_event: V[comp] += w * cf[comp]
      e.comp = static_cast<uint16_t>(D.e_comp[r]);
      e.w = D.e_wcf[r];
    } else if (!(A.dbg & 1)) {  // the delivery reads h and z of the target: warm the line
      const int64_t j = X.stc_inst + e.inst;
      asm volatile("prefetch.global.L1 [%0];" ::"l"(D.i_stc_h + j));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(D.i_stc_z + j));
    }
    EV[ev_top + t] = e;
  }
  __syncwarp();
  if (lane == 0) {
    X.ev_cur = ev_top;
    X.ev_end = ev_top + nd;
    X.cur = cur0 + nd;
    X.nk = (X.cur < X.end) ? pend[X.cur] : ~0ull;
    X.staged = 1;
  }
  ev_top += nd;
  __syncwarp();
}

// ---- one epoch [s0, s1) of the warp's group g ------------------------------
__device__ void mcg_wg_epoch(const McgDev& D, const McgWarpArgs& A, const McgWarpSm& W, int g,
                             int32_t j, int64_t s0, int64_t s1, int lane) {
  const McgKind* kinds = mcg_warp_kinds(A);
  const McgSpec* specs = mcg_warp_specs(D, A);
  McgWCell* R = reinterpret_cast<McgWCell*>(mcg_smem + W.rec);
  uint32_t* MK = reinterpret_cast<uint32_t*>(mcg_smem + W.mask);
  McgWEv* EV = reinterpret_cast<McgWEv*>(mcg_smem + W.ev);
  double* S_ = mcg_smem;
  const int G = A.G, m = A.m, S1 = 1 + A.S;
  const bool mine = lane < G && R[lane].c >= 0;

  // inbox merge and staging, cell by cell (only cells with something pending
  // or arriving do any work)
  {
    int ev_top = 0;
    const int cc = lane < G ? R[lane].c : -1;
    const bool busy = cc >= 0 && (D.inc_n[cc] > 0 || R[lane].cur < R[lane].end);
    unsigned todo = __ballot_sync(MCG_FULL, busy);
    if (lane < G && cc >= 0 && !busy) {
      R[lane].staged = 1;  // nothing due: an empty staged range
      R[lane].ev_cur = R[lane].ev_end = 0;
      R[lane].nk = ~0ull;
    }
    __syncwarp();
    while (todo) {
      const int k = __ffs(todo) - 1;
      todo &= todo - 1;
      mcg_wg_inbox(D, A, W, k, s0, s1, lane, ev_top);
    }
    if (mine) R[lane].nsp = 0;
  }
  WPH(15);  // inbox merge and staging done
  // resting synapses' calcium brought to s0 every cu_every epochs, so that a
  // catch-up inside an epoch (delayed calcium, the post-spike hook) spans at
  // most cu_every epochs of multiplications
  if (A.lazy && j % A.cu_every == 0) {
    for (int k = 0; k < G; ++k) {
      const McgWCell& X = R[k];
      if (X.c < 0 || X.stc_n == 0) continue;
      const uint32_t* mk = MK + k * A.MW;
      for (int i0 = 0; i0 < X.stc_n; i0 += 128) {
        double cv[4];
        int64_t tv[4];
        bool lz[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * 32 + lane;
          lz[u] = i < X.stc_n && !(mk[i >> 5] & (1u << (i & 31)));
          if (lz[u]) {
            tv[u] = A.stc_t[X.stc_inst + i];
            cv[u] = D.i_stc_c[X.stc_inst + i];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * 32 + lane;
          if (lz[u] && tv[u] < s0) {
            D.i_stc_c[X.stc_inst + i] = mcg_decay_steps(cv[u], X.ccf, s0 - tv[u]);
            A.stc_t[X.stc_inst + i] = s0;
          }
        }
      }
    }
    __syncwarp();
  }
  // per-lane constants of this epoch: the n == 1 species closed form's
  // denominator cap + gs (engine.cpp:738) and its reciprocal
  const int sys_k = lane / (2 * S1), sys_rem = lane - sys_k * 2 * S1, sys = sys_rem >> 1,
            side = sys_rem & 1;
  double sp_den = 1.0, sp_rden = 1.0;
  const bool sys_lane = sys_k < G && R[sys_k].c >= 0;
  int sys_n = 0;
  if (sys_lane) {
    const McgKind& K = kinds[R[sys_k].kind];
    sys_n = K.n;
    if (sys > 0 && sys - 1 < K.n_species && K.n == 1) {
      const int64_t ka = K.sp_arr + (sys - 1);
      sp_den = D.k_sp_cap_dt[ka] + D.k_sp_gs[ka];
      sp_rden = __drcp_rn(sp_den);
    }
  }
  // this lane's chain-sweep descriptor (mcg_sweep.cuh), static through the
  // epoch; the step fills in on / current / production
  McgChainLane Lst{};
  Lst.rc_node = -2;
  int lane_noise = -2, lane_prp = -1, lane_prp_comp = -1;
  if (sys_lane && sys < S1) {
    const McgWCell& X = R[sys_k];
    const McgKind& K = kinds[X.kind];
    const bool ok = K.ch_lp > 0 && (sys == 0 ? (K.dyn == MCG_DYN_LIF && K.v_const)
                                             : (sys - 1 < K.n_species && K.n > 1 && K.sp_const));
    if (ok) {
      const int n = K.n, Pk = 2 * K.ch_lp + 1;
      const int cho = A.kb_off[X.kind] + mcg_kind_chain_off(n, K.n_species);
      Lst.side = side;
      Lst.lp = K.ch_lp;
      Lst.r2c = W.r2c + sys_k * S1 * A.P + sys * A.P;
      Lst.idx = 2 * cho;
      Lst.fc = cho + (Pk + 1) / 2 + sys * 6 * Pk;
      Lst.x = X.base + (sys == 0 ? 0 : m + (sys - 1) * n);
      Lst.a_first = K.ch_afirst;
      Lst.v = sys == 0;
      Lst.rc = -1;
      lane_noise = K.noise_comp;
      lane_prp = K.prp_idx;
      lane_prp_comp = K.prp_comp;
    }
  }
  __syncwarp();
  WPH(0);

  for (int64_t s = s0; s < s1; ++s) {
    const int64_t so = s - s0;
    // ---- background-noise draws for the next 32 steps (normal_for,
    // rng.cpp:67-78: step n uses pair n >> 1 of threefry block n >> 2)
    if ((so & 31) == 0) {
      // only the pairs that cover [s, w1): one round of tasks for a short epoch
      const int64_t w1 = min(s + 32, s1);
      const int np = int(((w1 - 1) >> 1) - (s >> 1)) + 1;
      for (int q = lane; q < G * np; q += 32) {
        const int k = q / np, pp = q - k * np;
        if (R[k].c < 0 || !R[k].noise) continue;
        const uint64_t pr = (uint64_t(s) >> 1) + uint64_t(pp);
        const int64_t n0 = int64_t(pr * 2);
        const mcg_key key = mcg_make_key(D.seed, D.gid0 + uint32_t(R[k].c), 1, 0);
        uint64_t x[4];
        mcg_threefry(&key, pr >> 1, x);
        const unsigned h = unsigned(pr & 1u);
        const double u1 = ((double)(x[2 * h] >> 11) + 1.0) * MCG_2POW_M53;
        const double u2 = (double)(x[2 * h + 1] >> 11) * MCG_2POW_M53;
        double z0, z1;
        mcg_normal_pair(u1, u2, &z0, &z1);
        if (n0 >= s) S_[W.nb + k * 32 + int(n0 - s)] = z0;
        if (n0 + 1 < w1) S_[W.nb + k * 32 + int(n0 + 1 - s)] = z1;
      }
    }
    // rhs_current (engine.cpp:575): k_warp's kinds carry no current synapse,
    // so the buffer is zero but for the background current at noise_comp,
    // kept in a register (McgWCell::rc_val, McgChainLane::rc_node / rc_val)
    __syncwarp();
    WPH(1);
    // ---- A. delivery (engine.cpp:549-560): the inbox in (step, src, seq)
    // order, then the delayed calcium in (step, seq) order
    if (mine) {
      McgWCell& X = R[lane];
      const McgKind& K = kinds[X.kind];
      const bool refractory = X.lif && s < X.refr;
      X.refractory = refractory;
      X.has_current = 0;
      X.rc_val = 0.0;
      double* V = S_ + X.base;
      auto stc_event = [&](uint32_t inst, double w, uint32_t src) {
        // apply_event, stc_charge etype 0 (engine.cpp:497-510)
        if (X.f_tail - X.f_head >= X.f_cap) {
          atomicOr(D.err, MCG_ERR_FLAG_FIFO);
        } else {
          const int64_t slot = X.f_base + mcg_mod(X.f_tail, X.f_cap);
          D.fifo_step[slot] = s + X.ca_delay;
          D.fifo_si[slot] = (uint64_t(X.iseq) << 32) | uint64_t(inst);
          D.fifo_src[slot] = src;
          D.fifo_w[slot] = w;
          if (X.f_head == X.f_tail) X.next_due = s + X.ca_delay;
          ++X.f_tail;
        }
        ++X.iseq;
        if (!refractory) {  // stc_total_weight: h + h0 * z
          const int64_t jj = X.stc_inst + inst;
          const double tw = (A.dbg & 2) ? __ldcg(D.i_stc_h + jj) + X.h0 * __ldcg(D.i_stc_z + jj)
                                        : D.i_stc_h[jj] + X.h0 * D.i_stc_z[jj];
          V[X.stc_comp] += tw * w * X.cf;
        }
      };
      const bool trace = (A.dbg >> 8) == X.c + 1 && s >= A.dbg_s && s <= A.dbg_s + 5;
      if (trace)
        printf("[k_warp] cell %d s %lld staged %d ev [%d,%d) nk %llx cur %d end %d refr %d V0 %.17g Vb %.17g nd %lld\n", X.c,
               (long long)s, X.staged, X.ev_cur, X.ev_end, (unsigned long long)X.nk, X.cur, X.end,
               int(refractory), V[0], V[X.stc_comp], (long long)X.next_due);
      if (X.staged) {
        int e = X.ev_cur;
        while (e < X.ev_end && EV[e].so == int(so)) {
          const McgWEv E = EV[e];
          if (trace)
            printf("[k_warp]   ev so %d grp %d inst %u w %.17g comp %d gk %d\n", E.so, E.group, E.inst, E.w,
                   E.comp, X.gk[E.group]);
          if (X.gk[E.group] == MCG_SYN_STATIC_CHARGE) {
            if (!refractory && E.nz) V[E.comp] += E.w;  // w * cf[comp]
          } else {
            stc_event(E.inst, E.w, E.src);
          }
          ++e;
        }
        X.ev_cur = e;
      } else {
        uint64_t key = X.nk;
        if (int64_t(key >> D.rank_bits) <= s) {
          const uint64_t* pend = D.pend + (int64_t(X.c) * 2 + X.sel) * D.pend_cap;
          const uint64_t rank_mask = (1ull << D.rank_bits) - 1;
          int cur = X.cur;
          while (int64_t(key >> D.rank_bits) <= s) {
            const int64_t r = int64_t(key & rank_mask);
            const int grp = D.e_group[r];
            const double w = D.e_weight[r];
            if (X.gk[grp] == MCG_SYN_STATIC_CHARGE) {
              if (!refractory && w != 0.0) V[D.e_comp[r]] += D.e_wcf[r];
            } else {
              stc_event(D.e_inst[r], w, D.e_src[r]);
            }
            ++cur;
            key = (cur < X.end) ? pend[cur] : ~0ull;
          }
          X.cur = cur;
          X.nk = key;
        }
      }
      if (X.next_due <= s) {  // delayed calcium (stc_on_pre_calcium)
        const McgSpec& Sp = specs[X.stc_spec];
        uint32_t* mk = MK + lane * A.MW;
        while (X.next_due <= s) {
          const int64_t slot = X.f_base + mcg_mod(X.f_head, X.f_cap);
          const uint32_t inst = uint32_t(D.fifo_si[slot] & 0xffffffffu);
          ++X.f_head;
          mcg_wg_calcium(D, A, Sp, X, mk, int(inst), s, X.cpre_s);
          X.next_due = (X.f_head < X.f_tail) ? D.fifo_step[X.f_base + mcg_mod(X.f_head, X.f_cap)]
                                             : INT64_MAX;
        }
      }
      (void)K;
    }
    __syncwarp();
    WPH(2);
    // ---- B. STC synapses (engine.cpp:617-646): the active ones.  A PRP level
    // that is not finite ends every lazy synapse's rest (rare path).
    if (A.lazy) {
      bool wake = false;
      if (mine && R[lane].stc_n > 0 && R[lane].late && R[lane].prp_off >= 0) {
        const double prp = S_[R[lane].prp_off];
        wake = !(prp <= 0.0) && !(prp <= 1.7976931348623157e308);
      }
      unsigned wk = __ballot_sync(MCG_FULL, wake);
      while (wk) {
        const int k = __ffs(wk) - 1;
        wk &= wk - 1;
        const McgWCell& X = R[k];
        uint32_t* mk = MK + k * A.MW;
        for (int i = lane; i < X.stc_n; i += 32) {
          const int64_t jj = X.stc_inst + i;
          const bool lazy = !(mk[i >> 5] & (1u << (i & 31)));
          if (lazy) {
            D.i_stc_c[jj] = mcg_decay_steps(D.i_stc_c[jj], X.ccf, s - A.stc_t[jj]);
            A.stc_t[jj] = s;
          }
        }
        __syncwarp();
        for (int w = lane; w * 32 < X.stc_n; w += 32) {
          const int rem = X.stc_n - w * 32;
          mk[w] = rem >= 32 ? MCG_FULL : ((1u << rem) - 1u);
        }
        __syncwarp();
      }
    }
    {
      const int npairs = G * A.MW;
      for (int p0 = 0; p0 < npairs; p0 += 32) {
        const int p = p0 + lane;
        const uint32_t bits = p < npairs ? MK[p] : 0u;
        const int cnt = __popc(bits);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(MCG_FULL, incl, o);
          if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(MCG_FULL, incl, 31);
        for (int r0 = 0; r0 < total; r0 += 32) {
          const int q = r0 + lane;
          // the pair holding item q: the first lane whose inclusive count > q
          int lo = 0;
#pragma unroll
          for (int step = 16; step >= 1; step >>= 1) {
            const int v = __shfl_sync(MCG_FULL, incl, lo + step - 1);
            if (v <= q) lo += step;
          }
          const int pl = lo;  // lane (pair) index
          const uint32_t pb = __shfl_sync(MCG_FULL, bits, pl & 31);
          const int pex = __shfl_sync(MCG_FULL, incl - cnt, pl & 31);
          bool changed = false;
          int kslot = -1;
          double delta = 0.0;
          if (q < total) {
            const int pp = p0 + pl;
            const int k = pp / A.MW, w = pp - k * A.MW;
            const int i = w * 32 + mcg_nth_bit(pb, q - pex);
            kslot = k;
            const McgWCell& X = R[k];
            const McgSpec& Sp = specs[X.stc_spec];
            const int64_t jj = X.stc_inst + i;
            if ((A.dbg & 4) && A.lazy && A.stc_t[jj] != -1)
              printf("[k_warp] STALE active synapse cell %d inst %d s %lld t %lld\n", X.c, i, (long long)s,
                     (long long)A.stc_t[jj]);
            McgStcVal v{D.i_stc_h[jj], D.i_stc_z[jj], D.i_stc_c[jj], D.i_sps_abs[jj]};
            const double prp = (X.late && X.prp_off >= 0) ? S_[X.prp_off] : 0.0;
            changed = mcg_stc_step(Sp, D.dt, D.seed, D.gid0 + uint32_t(X.c), X.stc_gi, i, s,
                                   X.late != 0, prp, X.vol, X.rvol, v, delta, D.stc_nz + jj);
            D.i_stc_h[jj] = v.h;
            D.i_stc_z[jj] = v.z;
            D.i_stc_c[jj] = v.c;
            if (changed) D.i_sps_abs[jj] = v.a;
            if (A.lazy) {
              const McgStcRest Rr = mcg_stc_rest_of(Sp);
              if (__double_as_longlong(v.h) == Rr.h0_bits && !(v.c > Rr.theta_p) &&
                  !(v.c > Rr.theta_d) && v.a == 0.0) {
                A.stc_t[jj] = s + 1;  // at rest from the next step on
                atomicAnd(&MK[pp], ~(1u << (i & 31)));
              }
            }
          }
          // an unchanged item contributes -0.0, the identity of fp64 addition
          // (x + -0.0 == x for every x, signed zeros and NaN included)
          S_[W.db + lane] = changed ? delta : -0.0;
          const unsigned chg = __ballot_sync(MCG_FULL, changed);
          // SPS fold of this round's changed items, cell by cell in instance
          // order (engine.cpp:634-641).  The round's items are cell-major, so
          // cell slot k's are one lane range: its lane adds the deltas from
          // its first to its last changed item, unconditionally (independent
          // loads, one dependent add per item)
          unsigned myl = 0;
          if (chg) {
            for (int k = 0; k < G; ++k) {
              const unsigned b = __ballot_sync(MCG_FULL, changed && kslot == k);
              if (lane == k) myl = b;
            }
          }
          __syncwarp();
          if (myl && R[lane].sps_off >= 0) {
            const int la = __ffs(myl) - 1, lb = 32 - __clz(myl);
            double acc = S_[R[lane].sps_off];
            const double* db = S_ + W.db;
#pragma unroll 4
            for (int l = la; l < lb; ++l) acc += db[l];
            S_[R[lane].sps_off] = acc;
          }
          __syncwarp();
        }
      }
    }
    WPH(3);
    // ---- C. synthesis trigger and background current (engine.cpp:652-664,
    // 721-725)
    if (mine) {
      McgWCell& X = R[lane];
      const McgKind& K = kinds[X.kind];
      const double* SP = S_ + X.base + m;
      X.prod = 0.0;
      if (K.prp_enabled)
        X.prod = (SP[int64_t(K.sps_idx) * K.n + K.prp_comp] > K.prp_theta_star) ? K.prp_rate : 0.0;
      const double ts = double(s) * D.dt;
      const bool bg_gated = K.bg_t1 > K.bg_t0 && ts >= K.bg_t0 && ts < K.bg_t1;
      if (X.lif && K.has_bg && !bg_gated) {
        double ib = K.i_bg;
        if (K.sig_bg != 0.0) ib += K.sig_bg * S_[W.nb + lane * 32 + int(so & 31)];
        X.rc_val = 0.0 + ib;  // the zero-filled rhs_current plus ib
        X.has_current = 1;
      }
    }
    __syncwarp();
    WPH(4);
    // ---- D. membrane and species systems: (cell, system, chain side) lanes
    {
      McgChainLane L = Lst;  // static part (epoch entry)
      int kind = -1;
      if (Lst.lp > 0) {
        const McgWCell& X = R[sys_k];
        kind = X.kind;
        L.on = (sys != 0 || !X.refractory) ? 1 : 0;
        L.rc_node = (sys == 0 && X.has_current) ? lane_noise : -2;
        L.rc_val = X.rc_val;
        L.pc = (sys > 0 && sys - 1 == lane_prp && X.prod != 0.0) ? lane_prp_comp : -1;
        L.prod = X.prod;
      } else if (sys_lane && sys < S1) {
        kind = R[sys_k].kind;
      }
      mcg_chain_lane<false>(L);
      WPH(12);
      // single-compartment systems on their side-0 lanes
      if (sys_lane && sys < S1 && side == 0 && sys_n == 1) {
        const McgWCell& X = R[sys_k];
        const McgKind& K = kinds[kind];
        double* V = S_ + X.base;
        const double rc0 = X.rc_val;  // rhs_current[0] (noise_comp == 0 for n == 1)
        if (sys == 0) {
          if (K.dyn == MCG_DYN_LIF_EXACT) {
            if (!X.refractory) {  // engine.cpp:667-673
              const double vinf = K.v_rev + K.r_mem * rc0;
              V[0] = vinf + (V[0] - vinf) * K.lif_exact_f;
            }
          } else if (K.dyn == MCG_DYN_LIF && !X.refractory) {  // cable, n == 1
            const double rhs = D.k_g_leak_rhs[K.arr] + 0.0 + (X.has_current ? rc0 : 0.0);
            const double r2 = D.k_cap_dt[K.arr] * V[0] + rhs;
            V[0] = mcg_div(r2, D.k_vd[K.arr], D.k_vr[K.arr]);
          }
        } else if (sys - 1 < K.n_species) {  // engine.cpp:736-740
          const int q = sys - 1;
          double* conc = S_ + X.base + m + q;
          const double r = D.k_sp_cap_dt[K.sp_arr + q] * conc[0] + (q == K.prp_idx ? X.prod : 0.0);
          conc[0] = mcg_div(r, sp_den, sp_rden);
        }
      }
    }
    __syncwarp();
    WPH(5);
    if (mine && (A.dbg >> 8) == R[lane].c + 1 && s >= A.dbg_s && s <= A.dbg_s + 5)
      printf("[k_warp] cell %d s %lld after solve V0 %.17g Vb %.17g hc %d rc %.17g\n", R[lane].c, (long long)s,
             S_[R[lane].base], S_[R[lane].base + R[lane].stc_comp], R[lane].has_current,
             R[lane].rc_val);
    // ---- E. spike detection (engine.cpp:753-769)
    if (mine) {
      McgWCell& X = R[lane];
      const McgKind& K = kinds[X.kind];
      X.fired = 0;
      if (K.has_detector && !X.refractory) {
        const double va = S_[X.base + K.detector_comp];
        if (X.armed && X.det_prev < K.threshold && va >= K.threshold) {
          double f = (va > X.det_prev) ? (K.threshold - X.det_prev) / (va - X.det_prev) : 1.0;
          f = (f < 0.0) ? 0.0 : ((1.0 < f) ? 1.0 : f);  // std::clamp
          X.fired = 1;
          if (X.nsp < D.sp_cap) {
            D.sp_step[int64_t(X.c) * D.sp_cap + X.nsp] = s;
            D.sp_t[int64_t(X.c) * D.sp_cap + X.nsp] = (double(s) + f) * D.dt;
          } else {
            atomicOr(D.err, MCG_ERR_FLAG_SPIKES);
          }
          ++X.nsp;
        }
      }
    }
    {
      unsigned fired = __ballot_sync(MCG_FULL, mine && R[lane].fired);
      while (fired) {
        const int k = __ffs(fired) - 1;
        fired &= fired - 1;
        const McgWCell& X = R[k];
        const McgKind& K = kinds[X.kind];
        // post_event (engine.cpp:515-539): STC c += c_post * scale, every
        // instance; resting ones first take their lazy decay through step s
        if (X.stc_n > 0) {
          const McgSpec& Sp = specs[X.stc_spec];
          uint32_t* mk = MK + k * A.MW;
          for (int i0 = 0; i0 < X.stc_n; i0 += 32) {
            const int i = i0 + lane;
            bool wake = false;
            if (i < X.stc_n) {
              const int64_t jj = X.stc_inst + i;
              const bool lazy = A.lazy && !(mk[i >> 5] & (1u << (i & 31)));
              if (lazy) {
                double c = mcg_decay_steps(D.i_stc_c[jj], X.ccf, s + 1 - A.stc_t[jj]);
                c += X.cpost_s;
                D.i_stc_c[jj] = c;
                A.stc_t[jj] = s + 1;
                wake = c > Sp.theta_p || c > Sp.theta_d;
                if (wake && (A.dbg & 4)) A.stc_t[jj] = -1;
              } else {
                D.i_stc_c[jj] += X.cpost_s;
              }
            }
            const unsigned wb = __ballot_sync(MCG_FULL, wake);
            if (lane == 0 && wb) mk[i0 >> 5] |= wb;
          }
        }
        if (X.lif)  // LIF reset: every compartment (engine.cpp:770-772)
          for (int i = lane; i < K.n; i += 32) S_[X.base + i] = K.v_reset;
        __syncwarp();
      }
    }
    WPH(6);
    // ---- F. detector bookkeeping and probes (engine.cpp:770-793)
    if (mine) {
      McgWCell& X = R[lane];
      const McgKind& K = kinds[X.kind];
      const double* V = S_ + X.base;
      if (K.has_detector && !X.refractory) {
        if (X.fired) {
          if (X.lif) X.refr = s + 1 + K.ref_steps;
          else X.armed = 0;
        } else if (!X.armed && V[K.detector_comp] < K.threshold) {
          X.armed = 1;
        }
        X.det_prev = V[K.detector_comp];
      }
      const int p0 = X.probe0, p1 = X.probe1;
      for (int q = p0; q < p1; ++q) {
        const int p = D.probe_idx[q];
        const McgProbe& Pr = D.probes[p];
        if (mcg_mod(s + 1, Pr.every) != 0) continue;
        const int64_t m0 = (D.ctl[3] + Pr.every) / Pr.every;
        double val;
        if (Pr.what == MCG_PROBE_SYN_C && Pr.group == X.stc_gi && X.stc_n > 0 && A.lazy &&
            !(MK[lane * A.MW + (Pr.instance >> 5)] & (1u << (Pr.instance & 31)))) {
          const int64_t jj = X.stc_inst + Pr.instance;  // the lazily kept calcium, as of now
          val = mcg_decay_steps(D.i_stc_c[jj], X.ccf, s + 1 - A.stc_t[jj]);
        } else {
          val = mcg_probe_value(D, K, X.c, Pr, V, V + m);
        }
        D.trace_buf[D.trace_base[p] + ((s + 1) / Pr.every - m0)] = val;
      }
    }
    __syncwarp();
    WPH(7);
  }

  // ---- epoch end: the group's spikes as one log chunk, what the next
  // expansion reads (spike slots, inbox cursors)
  const int nk = mine ? min(R[lane].nsp, D.sp_cap) : 0;
  int before = nk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(MCG_FULL, before, o);
    if (lane >= o) before += v;
  }
  const int tot = __shfl_sync(MCG_FULL, before, 31);
  before -= nk;
  int off = 0;
  if (tot > 0) {
    if (lane == 0) {
      off = static_cast<int>(atomicAdd(A.log_n, static_cast<unsigned long long>(tot)));
      const unsigned long long ci = atomicAdd(A.chunk_n, 1ull);
      A.chunks[ci] = make_int4(A.epoch_base + j, g, off, tot);
    }
    off = __shfl_sync(MCG_FULL, off, 0);
  }
  if (mine) {
    McgWCell& X = R[lane];
    const int c = X.c;
    for (int i = 0; i < nk; ++i) {
      A.log_t[off + before + i] = D.sp_t[int64_t(c) * D.sp_cap + i];
      A.log_gid[off + before + i] = D.gid0 + uint32_t(c);
    }
    D.sp_count[c] = nk;
    if (A.x_send != nullptr && nk > 0) {  // sharded: publish for the caller's allgather
      const int64_t pos = static_cast<int64_t>(
          atomicAdd(reinterpret_cast<unsigned long long*>(A.x_send), static_cast<unsigned long long>(nk)));
      if (pos + nk > A.x_cap) {
        atomicOr(D.err, MCG_ERR_FLAG_SPIKES);
      } else {
        for (int i = 0; i < nk; ++i) {
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
  __syncwarp();
  WPH(8);
}

__global__ void __launch_bounds__(256, 1) k_warp(const __grid_constant__ McgDev D,
                                                 const __grid_constant__ McgWarpArgs A,
                                                 int64_t max_len) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // kind blocks, kind records and the spec table, once per launch
  for (int k = 0; k < A.n_kinds; ++k)
    if (A.kb_off[k] >= 0) mcg_kind_stage(D, D.kinds[k], mcg_smem + A.kb_off[k]);
  {
    McgKind* kc = mcg_warp_kinds(A);
    for (int k = threadIdx.x; k < A.n_kinds; k += blockDim.x) kc[k] = D.kinds[k];
    if (A.n_specs_sm > 0) {
      McgSpec* sp = const_cast<McgSpec*>(mcg_warp_specs(D, A));
      for (int i = threadIdx.x; i < A.n_specs_sm; i += blockDim.x) sp[i] = D.specs[i];
    }
  }
  if (A.phase && lane == 0) {
    for (int i = 0; i < MCG_WPH_N; ++i) mcg_wph[w][i] = 0;
    mcg_wph[w][MCG_WPH_N] = clock64();
  }
  __syncthreads();
  const McgWarpSm W = mcg_warp_sm(A, w);
  if (lane == 0) {  // the warp's bulk-copy mbarrier, phase 0
    mcg_mbar_init(mcg_sa(mcg_smem + W.mbar));
    *reinterpret_cast<uint32_t*>(mcg_smem + W.mbar + 1) = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const int gw = w * gridDim.x + blockIdx.x;  // consecutive groups on different SMs
  const int nw = gridDim.x * (blockDim.x >> 5);
  if (A.resident && gw < A.n_groups) mcg_wg_enter(D, A, W, gw, lane);
  for (int32_t j = 0; j < A.n_epochs; ++j) {
    int64_t s0, s1;
    if (!mcg_epoch_bounds(D.ctl, j, s0, s1)) break;
    WPH(11);
    mcg_expand(A.E, D, j, s0, s1, max_len);
    WPH(10);
    grid.sync();
    WPH(11);
    // the overflow flag, read by every warp after the barrier, costs ~5 us
    // per epoch (one contended line); unneeded when overflow is impossible
    if (!A.no_abort && *D.abort) break;
    WPH(13);
    for (int g = gw; g < A.n_groups; g += nw) {
      if (!A.resident) mcg_wg_enter(D, A, W, g, lane);
      WPH(9);
      mcg_wg_epoch(D, A, W, g, j, s0, s1, lane);
      if (!A.resident) mcg_wg_exit(D, A, W, lane);
      WPH(9);
    }
    // the warp's bulk stores of this epoch complete before the barrier (the
    // next epoch's bulk loads, other kernels, the host read them)
    if (!A.resident && lane < A.G) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    grid.sync();
  }
  if (A.resident && gw < A.n_groups) mcg_wg_exit(D, A, W, lane);
  if (lane < A.G) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  WPH(9);
  if (A.phase && lane == 0 && gw < A.n_groups)
    for (int i = 0; i < MCG_WPH_N; ++i) {
      atomicAdd(&A.phase[i], mcg_wph[w][i]);
      atomicMax(&A.phase[MCG_WPH_N + i], mcg_wph[w][i]);
    }
}

// ---- lazy-calcium bookkeeping of the STC instances, warp per cell ----------
// init: every instance not at rest (or all, without lazy calcium) goes into
// the active mask; the others keep their calcium as of step `now`
__global__ void k_lazy_init(McgDev D, uint32_t* mask, int64_t* stc_t, int32_t MW, int32_t lazy,
                            int64_t now) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= D.n_cells) return;
  const McgKind K = D.kinds[D.cell_kind[c]];
  const int64_t cg0 = D.cg_off[c];
  for (int gi = 0; gi < K.n_groups; ++gi) {
    const McgCellGroup Gr = D.cgs[cg0 + gi];
    const McgSpec& S = D.specs[Gr.spec];
    if (S.kind != MCG_SYN_STC_CHARGE) continue;
    const McgStcRest Rr = mcg_stc_rest_of(S);
    for (int i0 = 0; i0 < Gr.size; i0 += 32) {
      const int i = i0 + lane;
      bool act = false;
      if (i < Gr.size) {
        const int64_t j = Gr.inst + i;
        const double h = D.i_stc_h[j], cc = D.i_stc_c[j], a = D.i_sps_abs[j];
        act = !lazy || !(__double_as_longlong(h) == Rr.h0_bits && !(cc > Rr.theta_p) &&
                         !(cc > Rr.theta_d) && a == 0.0);
        stc_t[j] = now;
      }
      if (act && i < Gr.size && lazy == 2) stc_t[Gr.inst + i] = -1;
      const unsigned b = __ballot_sync(MCG_FULL, act);
      if (lane == 0 && (i0 >> 5) < MW) mask[int64_t(c) * MW + (i0 >> 5)] = b;
    }
    break;  // one STC placement per kind (k_warp's eligibility)
  }
}

// flush: every resting instance's calcium brought to step `now`
__global__ void k_lazy_flush(McgDev D, const uint32_t* mask, const int64_t* stc_t, int32_t MW,
                             int64_t now) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= D.n_cells) return;
  const McgKind K = D.kinds[D.cell_kind[c]];
  const int64_t cg0 = D.cg_off[c];
  for (int gi = 0; gi < K.n_groups; ++gi) {
    const McgCellGroup Gr = D.cgs[cg0 + gi];
    const McgSpec& S = D.specs[Gr.spec];
    if (S.kind != MCG_SYN_STC_CHARGE) continue;
    for (int i = lane; i < Gr.size; i += 32) {
      if (mask[int64_t(c) * MW + (i >> 5)] & (1u << (i & 31))) continue;
      const int64_t j = Gr.inst + i;
      D.i_stc_c[j] = mcg_decay_steps(D.i_stc_c[j], S.cf, now - stc_t[j]);
    }
    break;
  }
}
