// mcg_engine.cu — host orchestration of the B200 engine and the C ABI
// (include/mcg.h).
//
// Engine::advance_to (engine.cpp:909-945) runs as launches of the persistent
// cooperative batch kernel k_batch (mcg_batch.cuh): up to kBatch min-delay
// epochs per launch, each epoch = spike/source expansion into per-cell
// inboxes, grid barrier, every CTA steps its cells through the epoch, grid
// barrier.  Epoch bounds live in device memory; the host synchronizes once per
// launch (spike log chunks, overflow/abort flags).  All state stays resident
// in HBM; cell state, spikes and traces are copied to the host only when
// asked (the lazily-synced mirror of engine.hpp).
#include <cub/cub.cuh>  // mcg_er_connect's scan
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is dlopen'ed (NcclApi)

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>
#include <unordered_map>

#include "mcg_batch.cuh"
#include "mcg_warp.cuh"
#include "mcg_point.cuh"
#include "mcg_protocols.cuh"
#include "mcg_checkpoint.h"
#include "mcg_build.h"
#include "mcg_resolve.cuh"

static void layout_digest(const mcg::HostModel& m, uint64_t out[4]);

namespace mcg {

namespace {

thread_local std::string g_last_error;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(MCG_ERR_CUDA, std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  // allocations from the device's memory pool, which keeps freed memory (its
  // release threshold is raised at engine creation): constructing an engine
  // does not map fresh memory.  Complete before use on any stream; freed
  // only when the device is idle.
  void release() {
    if (p) {
      cudaDeviceSynchronize();
      cudaFreeAsync(p, 0);
      cudaStreamSynchronize(0);
    }
    p = nullptr;
  }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) {
      CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), 0));
      CK(cudaStreamSynchronize(0));
    }
  }
  template <class Al>
  void upload(const std::vector<T, Al>& v, cudaStream_t st) {
    alloc(std::max<size_t>(v.size(), 1));
    if (!v.empty())
      CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  }
  void zero(cudaStream_t st) {
    if (p) CK(cudaMemsetAsync(p, 0, n * sizeof(T), st));
  }
};

int bits_for(uint64_t v) {  // bits needed to represent values in [0, v]
  int b = 1;
  while (b < 63 && (v >> b) != 0) ++b;
  return b;
}

// device counters, mirrored to pinned host memory once per batch
enum { C_EP_SPK = 0, C_LOG = 1, C_DELIVERED = 2, C_N = 4 };

// anything still undelivered: queued keys, unexpanded spikes with local
// fan-out, or delayed calcium (the fast-forward guard, engine.cpp:958-960)
// fast-forward guard (engine.cpp:958-960): which cells hold undelivered
// events -- pending or incoming inbox entries, queued delayed calcium, or
// events the last epoch's spikes will deliver (expanded at the next epoch's
// entry here, already in the targets' inboxes in the reference)
__global__ void k_pending(McgDev D, const int64_t* out_begin, const int64_t* out_end,
                          const int32_t* e_dst, int32_t* cell_flag) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= D.n_cells) return;
  bool p = D.pend_n[i] > D.pend_off[i] || D.inc_n[i] > 0;
  const McgKind& K = D.kinds[D.cell_kind[i]];
  for (int gi = 0; gi < K.n_groups; ++gi) {
    const int32_t f = D.cgs[D.cg_off[i] + gi].fifo;
    if (f >= 0 && D.fifos[f].head < D.fifos[f].tail) p = true;
  }
  if (p) cell_flag[i] = 1;
  if (D.sp_count[i] > 0) {
    const uint32_t g = D.gid0 + uint32_t(i);
    for (int64_t r = out_begin[g]; r < out_end[g]; ++r) cell_flag[e_dst[r]] = 1;
  }
}

}  // namespace

// NCCL, loaded at run time by the first engine that shards through it (a
// single-GPU build never needs libnccl; with torch in the process its
// bundled libnccl.so.2 is the one found)
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  void load() {
    if (h) return;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    if (!h) throw Error(MCG_ERR_CUDA, std::string("nccl: cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* n) {
      void* f = dlsym(h, n);
      if (!f) throw Error(MCG_ERR_CUDA, std::string("nccl: missing symbol ") + n);
      return f;
    };
    get_unique_id = reinterpret_cast<decltype(get_unique_id)>(sym("ncclGetUniqueId"));
    comm_init_rank = reinterpret_cast<decltype(comm_init_rank)>(sym("ncclCommInitRank"));
    all_gather = reinterpret_cast<decltype(all_gather)>(sym("ncclAllGather"));
    comm_destroy = reinterpret_cast<decltype(comm_destroy)>(sym("ncclCommDestroy"));
    error_string = reinterpret_cast<decltype(error_string)>(sym("ncclGetErrorString"));
  }
  void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(MCG_ERR_CUDA, std::string("nccl: ") + what + ": " + error_string(r));
  }
};
NcclApi& nccl_api() {
  static NcclApi api;
  api.load();
  return api;
}

// the epoch's gathered spikes (every rank's send block) appended to the
// global spike log as (s0, gid, step, t bits); the host orders each epoch by
// (gid, step), Impl::exchange's order (engine.cpp:877-888)
__global__ void k_collect_recv(const int64_t* recv, int32_t world, int64_t block, const int64_t* ctl,
                               int64_t* glog, unsigned long long* glog_n, int64_t cap, int32_t* err) {
  const int64_t s0 = ctl[0];
  for (int r = 0; r < world; ++r) {
    const int64_t* b = recv + r * block;
    const int64_t n = b[0];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long pos = atomicAdd(glog_n, 1ull);
      if (static_cast<int64_t>(pos) >= cap) {
        atomicOr(err, MCG_ERR_FLAG_SPIKES);
        continue;
      }
      glog[4 * pos] = s0;
      glog[4 * pos + 1] = b[1 + 3 * i];
      glog[4 * pos + 2] = b[2 + 3 * i];
      glog[4 * pos + 3] = b[3 + 3 * i];
    }
  }
}

struct Engine {
  HostModel m;
  cudaStream_t st = nullptr;
  int device = 0;
  int64_t step = 0;
  int64_t L = 1;              // epoch length (min_delay_steps, or free_epoch without cell edges)
  static constexpr int kSmemMaxComps = 96;  // cells up to this size live in shared memory
  static constexpr int kBlock = 128;        // fast-forward: 4 warps = 4 cells per block
  static constexpr int kBatch = 32;         // epochs per batch-kernel launch

  // device model
  DBuf<McgKind> d_kinds;
  DBuf<McgSpec> d_specs;
  DBuf<int32_t> d_k_parent, d_k_ch_idx;
  DBuf<double> d_k_cap_dt, d_k_g_leak, d_k_g_leak_rhs, d_k_axial, d_k_g_na, d_k_g_k, d_k_cf,
      d_k_volume, d_k_sp_cap_dt, d_k_sp_gs, d_k_sp_coupling, d_k_vf, d_k_vd, d_k_sp_f, d_k_sp_d, d_k_vr, d_k_sp_r, d_k_rvol;
  DBuf<int32_t> d_cell_kind;
  DBuf<int64_t> d_comp_off, d_sp_off, d_cg_off;
  DBuf<double> d_v, d_hh_m, d_hh_h, d_hh_n, d_species, d_det_prev;
  DBuf<int32_t> d_armed;
  DBuf<int64_t> d_refr;
  DBuf<uint32_t> d_iseq;
  DBuf<double> d_s_gsyn, d_s_gsyn_rhs, d_s_rhs_cur, d_s_diag, d_s_rhs, d_s_r2;
  int32_t sp_max = 0, smem_n = 0, smem_stride = 0;
  size_t smem_bytes = 0;
  DBuf<McgCellGroup> d_cgs;
  DBuf<McgFifo> d_fifos;
  DBuf<int64_t> d_fifo_step;
  DBuf<uint64_t> d_fifo_si;
  DBuf<uint32_t> d_fifo_src;
  DBuf<double> d_fifo_w;
  DBuf<int32_t> d_i_comp, d_i_active;
  DBuf<double> d_i_weight, d_i_kernel, d_i_stdp_pre, d_i_stdp_post, d_i_stdp_w, d_i_homeo_w,
      d_i_stc_h, d_i_stc_z, d_i_stc_c, d_i_sps_abs;
  DBuf<McgNzCache> d_stc_nz;
  DBuf<int64_t> d_i_stdp_last;
  // edges
  DBuf<int32_t> d_e_dst, d_e_group;
  DBuf<uint32_t> d_e_inst;
  DBuf<double> d_e_weight;
  DBuf<uint32_t> d_e_src;
  DBuf<int32_t> d_e_comp;
  DBuf<double> d_e_wcf;
  DBuf<int64_t> d_e_delay, d_out_begin, d_out_end, d_src_edge_off, d_src_edges;
  DBuf<uint32_t> d_e_seq;  // device-resolved edges only: their seq, for the host copy
  bool host_edges = true;  // m.e_* hold the edge records (else only the device does)
  int32_t rank_bits = 1;
  // sources
  DBuf<McgSrcTask> d_tasks;
  DBuf<int64_t> d_scripted;
  int32_t n_tasks = 0, n_poisson = 0;
  // inboxes
  DBuf<uint64_t> d_inc, d_pend;
  DBuf<int32_t> d_inc_n, d_pend_sel, d_pend_off, d_pend_n;
  int32_t inc_cap = 32, pend_cap = 64;
  // epoch control
  DBuf<int64_t> d_ctl;
  int64_t* h_ctl = nullptr;
  DBuf<int32_t> d_abort;
  // spikes
  int32_t sp_cap = 1;
  DBuf<int32_t> d_sp_count;
  DBuf<int64_t> d_sp_step;
  DBuf<double> d_sp_t;
  DBuf<double> d_log_t;       // batch log
  DBuf<uint32_t> d_log_gid;
  // probes
  DBuf<McgProbe> d_probes;
  DBuf<int32_t> d_probe_off, d_probe_idx;
  DBuf<double> d_trace;
  DBuf<int64_t> d_trace_base;
  std::vector<int64_t> probe_base_host;
  int64_t probe_total = 0;
  std::vector<std::vector<std::pair<double, double>>> traces;
  // status
  DBuf<unsigned long long> d_ctr;
  DBuf<int32_t> d_err;
  unsigned long long* h_ctr = nullptr;
  int32_t* h_err = nullptr;
  int32_t* h_abort = nullptr;
  // host spike mirror
  std::vector<double> spk_t;
  std::vector<uint32_t> spk_gid;
  // persistent batch kernel (cell batches per CTA)
  static constexpr int kBatchThreads = MCG_BATCH_THREADS;
  int32_t bc_cells = 1, bc_batches = 1, bc_grid = 1, bc_stc_max = 1, bc_nstc_max = 1;
  int32_t bc_ch_pmax = 0, bc_ch_stride = 0;
  int32_t bc_ev_cap = 0, bc_fmask_words = 0;
  int32_t bc_stride = 0;  // doubles per staged cell's compartment block
  int32_t bc_nch_max = 0;  // chain-sweep lane descriptors per batch
  int32_t bc_lean = 0;
  int32_t bc_act_max = 0;
  int bc_carve = 100;  // shared-memory carveout (percent) this engine's batch kernel needs
  int32_t bc_kind_doubles = 0, bc_specs_sm = 0, bc_stc_sm = 0;
  size_t bc_smem = 0;
  DBuf<int4> d_chunks;
  DBuf<unsigned long long> d_chunk_n;
  // warp-group kernel (mcg_warp.cuh) for LIF networks with charge-type synapses
  bool use_warp = false;
  int32_t wg_G = 1, wg_groups = 1, wg_warps = 1, wg_grid = 1, wg_resident = 0, wg_P = 0, wg_MW = 1;
  int32_t wg_ev_cap = 0, wg_warp_doubles = 0, wg_kind_doubles = 0, wg_specs_sm = 0, wg_lazy = 0;
  size_t wg_smem = 0;
  int32_t wg_no_abort = 0;
  DBuf<int32_t> d_kb_off;
  DBuf<uint32_t> d_stc_mask;
  DBuf<int64_t> d_stc_t;
  bool lazy_valid = false;  // active masks and calcium stamps match the state
  // register-resident kernel for independent point cells (mcg_point.cuh)
  bool use_point = false;
  bool pt_small = false;  // every cell fits k_point<1, 2>
  DBuf<uint64_t> d_cell_seed;      // per-cell RNG key override (mcg_set_cell_rng)
  DBuf<uint32_t> d_cell_key_gid;
  int32_t pt_grid = 1;
  bool lazy_dirty = false;  // resting synapses' calcium lags `step` (k_warp ran since the last flush)
  cudaEvent_t evk0 = nullptr, evk1 = nullptr;
  // MCG_PHASE_TIMING=1: per-phase cycle totals of the batch kernel, printed
  // to stderr after every advance_to (development instrumentation)
  bool phase_timing = std::getenv("MCG_PHASE_TIMING") != nullptr;
  DBuf<unsigned long long> d_phase;

  void print_phases(int64_t call_steps = 0) {
    if (!phase_timing || !d_phase.p) return;
    if (use_warp) {
      unsigned long long ph[2 * MCG_WPH_N];
      CK(cudaMemcpy(ph, d_phase.p, sizeof(ph), cudaMemcpyDeviceToHost));
      const double warps = std::min<double>(wg_groups, double(wg_grid) * wg_warps);
      std::fprintf(stderr, "k_warp phase us/step/warp (mean | max warp), steps=%lld warps=%.0f:",
                   (long long)call_steps, warps);
      static const char* nm[MCG_WPH_N] = {"epoch_in", "noise", "deliver", "stc", "trigger", "solve",
                                          "detect_post", "probes", "epoch_out", "groups", "expand", "gsync",
                                          "solve_chain", "abort_chk", "enter_rec", "inbox"};
      for (int i = 0; i < MCG_WPH_N; ++i)
        std::fprintf(stderr, " %s %.3f|%.3f", nm[i], ph[i] / warps / 1965.0 / std::max<int64_t>(call_steps, 1),
                     ph[MCG_WPH_N + i] / 1965.0 / std::max<int64_t>(call_steps, 1));
      std::fprintf(stderr, "\n");
      d_phase.zero(st);
      return;
    }
    unsigned long long ph[2 * MCG_NPHASE];
    CK(cudaMemcpy(ph, d_phase.p, sizeof(ph), cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "phase cycles (sum over CTAs):");
    for (int i = 0; i < MCG_NPHASE; ++i) std::fprintf(stderr, " %d:%llu", i, ph[i]);
    std::fprintf(stderr, "  steps=%lld batches=%d\nphase cycles (CTA 0):", (long long)stats.steps, bc_batches);
    for (int i = 0; i < MCG_NPHASE; ++i) std::fprintf(stderr, " %d:%llu", i, ph[MCG_NPHASE + i]);
    std::fprintf(stderr, "  steps=%lld batches=1\n", (long long)stats.steps);
    // per CTA: work cycles (everything but the grid-sync wait, phase 13)
    std::vector<unsigned long long> pc(size_t(bc_grid) * MCG_NPHASE);
    CK(cudaMemcpy(pc.data(), d_phase.p + 2 * MCG_NPHASE, pc.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<std::pair<double, int>> w;
    for (int b = 0; b < bc_grid; ++b) {
      double t = 0;
      for (int i = 0; i < MCG_NPHASE; ++i)
        if (i != 13) t += double(pc[size_t(b) * MCG_NPHASE + i]);
      w.emplace_back(t, b);
    }
    std::sort(w.rbegin(), w.rend());
    std::fprintf(stderr, "per-CTA work cycles: max %.4g (CTA %d) median %.4g min %.4g (CTA %d)\n", w[0].first,
                 w[0].second, w[w.size() / 2].first, w.back().first, w.back().second);
    for (int r = 0; r < 3 && r < int(w.size()); ++r) {
      std::fprintf(stderr, "  CTA %d:", w[r].second);
      for (int i = 0; i < MCG_NPHASE; ++i)
        std::fprintf(stderr, " %d:%.3g", i, double(pc[size_t(w[r].second) * MCG_NPHASE + i]));
      std::fprintf(stderr, "\n");
    }
    d_phase.zero(st);  // per advance_to call
  }
  // stats
  mcg_stats stats{};
  bool timing = false;
  cudaEvent_t eva = nullptr, evb = nullptr;

  McgDev dev{};

  ~Engine() {
    if (nccl_comm) nccl_api().comm_destroy(static_cast<ncclComm_t>(nccl_comm));
    if (h_ctl_ring) cudaFreeHost(h_ctl_ring);
    if (h_ctr) cudaFreeHost(h_ctr);
    if (h_err) cudaFreeHost(h_err);
    if (h_abort) cudaFreeHost(h_abort);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (eva) cudaEventDestroy(eva);
    if (evb) cudaEventDestroy(evb);
    if (evk0) cudaEventDestroy(evk0);
    if (evk1) cudaEventDestroy(evk1);
    if (st) cudaStreamDestroy(st);
  }

  // geometry of the persistent batch kernel: ~n_cells/148 cells per CTA,
  // capped by shared memory; grid = co-resident CTAs
  void setup_batch_kernel() {
    const int nl = n_local();
    int dev_sms = 148;
    CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device));
    std::vector<int> stc_n(nl, 0);
    int cell_stc_max = 0;
    bc_nstc_max = 1;
    for (int c = 0; c < nl; ++c) {
      const McgKind& K = m.kinds[m.cell_kind[c]];
      int tot = 0, ng = 0;
      for (int gi = 0; gi < K.n_groups; ++gi) {
        const McgCellGroup& G = m.cgs[m.cg_off[c] + gi];
        if (m.specs[G.spec].kind != MCG_SYN_STC_CHARGE) continue;
        tot += G.size;
        ++ng;
      }
      stc_n[c] = tot;
      cell_stc_max = std::max(cell_stc_max, tot);
      bc_nstc_max = std::max(bc_nstc_max, ng);
    }
    if (bc_nstc_max > 0xffff) throw Error(MCG_ERR_ENGINE, "too many STC placements per kind");
    // compartment block per staged cell: the full layout (mcg_cell_mem), or just
    // V | SP | rhs_cur when every staged kind is a LIF with only charge-type
    // synapses and its cable systems take the chain sweep (no HH gates,
    // conductances or solver scratch are ever touched)
    bool lean = !std::getenv("MCG_FULL_BLOCK");
    for (size_t ki = 0; ki < m.kinds.size() && lean; ++ki) {
      const McgKind& K = m.kinds[ki];
      if (K.n > smem_n) continue;
      if (K.dyn != MCG_DYN_LIF && K.dyn != MCG_DYN_LIF_EXACT) lean = false;
      if (K.n > 1 && !(K.ch_lp > 0 && K.v_const && (K.n_species == 0 || K.sp_const))) lean = false;
      for (int gi = 0; gi < K.n_groups && lean; ++gi) {
        const int kd = m.specs[K.spec0 + gi].kind;
        if (kd != MCG_SYN_STATIC_CHARGE && kd != MCG_SYN_STC_CHARGE) lean = false;
      }
    }
    bc_stride = lean ? (2 + sp_max) * smem_n : smem_stride;
    bc_lean = lean ? 1 : 0;
    // per cell: compartment block, noise draws, kind and cell records, STC
    // segments, and (upper bound) its STC slots in the fold/locator tables
    // chain-sweep scratch: (1 + sp_max) systems x P_max positions per cell
    bc_ch_pmax = 0;
    for (const McgKind& K : m.kinds)
      if (K.n <= smem_n && K.ch_lp > 0) bc_ch_pmax = std::max(bc_ch_pmax, 2 * K.ch_lp + 1);
    bc_ch_stride = bc_ch_pmax > 0 ? (1 + sp_max) * bc_ch_pmax : 0;
    const size_t per_cell = size_t(bc_stride) * 8 + 32 * 8 + sizeof(McgKind) + sizeof(McgCellSm) +
                            size_t(bc_nstc_max) * sizeof(McgSegSm) + size_t(cell_stc_max) * 12 +
                            size_t(bc_ch_stride) * 8;
    // staged kind constants (McgKindSm): one block per distinct kind of a batch
    size_t kb_max = 0;
    for (const McgKind& K : m.kinds)
      if (K.n <= smem_n)
        kb_max = std::max<size_t>(kb_max, mcg_kind_block_doubles(K.n, K.n_species, K.ch_lp));
    // the spec table, when small, is staged once per launch
    bc_specs_sm = m.specs.size() * sizeof(McgSpec) <= 16 * 1024 ? static_cast<int32_t>(m.specs.size()) : 0;
    const size_t fixed = size_t(bc_specs_sm) * sizeof(McgSpec) + 2048;
    const size_t budget = 200 * 1024;
    // one staged kind block per distinct kind of a batch: at most min(C, kinds)
    const size_t nkinds = std::max<size_t>(m.kinds.size(), 1);
    int c_max = 1;
    while (c_max < 0xffff &&
           fixed + size_t(c_max + 1) * per_cell + std::min<size_t>(c_max + 1, nkinds) * kb_max * 8 <= budget)
      ++c_max;
    bc_cells = std::clamp((nl + dev_sms - 1) / std::max(dev_sms, 1), 1, std::min(c_max, 0xffff));
    // test hook: cap the batch size (forces per-epoch batch staging on small nets)
    if (const char* cap = std::getenv("MCG_MAX_CELLS_PER_CTA")) bc_cells = std::max(1, std::min(bc_cells, std::atoi(cap)));
    bc_batches = std::max(1, (nl + bc_cells - 1) / bc_cells);
    // STC slots of the fullest batch
    bc_stc_max = 1;
    for (int b = 0; b < bc_batches; ++b) {
      int tot = 0;
      for (int c = b * bc_cells; c < std::min(nl, (b + 1) * bc_cells); ++c) tot += stc_n[c];
      bc_stc_max = std::max(bc_stc_max, tot);
    }
    bc_kind_doubles = static_cast<int32_t>(std::min<size_t>(bc_cells, m.kinds.size()) * kb_max);
    // fold-flag words: one per 32 slots of every 512-thread round
    const size_t fmask_words = size_t((bc_stc_max + kBatchThreads - 1) / kBatchThreads) * (kBatchThreads / 32) + 1;
    bc_nch_max = bc_ch_stride > 0 ? (2 * (1 + sp_max) * bc_cells + 31) / 32 * 32 : 0;
    bc_smem = size_t(bc_nch_max) * MCG_LANE_INTS * 4 + 16 +
              size_t(bc_cells) * (size_t(bc_stride) * 8 + 32 * 8 + sizeof(McgKind) + sizeof(McgCellSm) +
                                  size_t(bc_nstc_max) * sizeof(McgSegSm) + size_t(bc_ch_stride) * 8) +
              size_t(bc_stc_max) * (8 + 4) + size_t(bc_kind_doubles) * 8 +
              size_t(bc_specs_sm) * sizeof(McgSpec) + fmask_words * 4 + 64;
    // resident batches (one per CTA) keep their STC state in shared memory too
    int smem_optin = 0;
    CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    bc_stc_sm = (bc_batches <= dev_sms && stc_n.size() > 0 &&
                 bc_smem + size_t(bc_stc_max) * 32 <= size_t(smem_optin) - 1024)
                    ? 1 : 0;
    if (std::getenv("MCG_NO_STC_SM")) bc_stc_sm = 0;
    if (bc_stc_sm) bc_smem += size_t(bc_stc_max) * 32;
    bc_fmask_words = static_cast<int32_t>(fmask_words);
    // one cell per CTA: phase B's scratch (decayed kernel | instance index per
    // active-list entry, groups padded to 32) when the lists are long enough
    // to be worth spreading over the CTA
    bc_act_max = 0;
    if (bc_cells == 1 && !std::getenv("MCG_NO_PAR_ACTIVE")) {
      int amax = 0;
      for (int c = 0; c < nl; ++c) {
        const McgKind& K = m.kinds[m.cell_kind[c]];
        int tot = 0;
        for (int gi = 0; gi < K.n_groups; ++gi) {
          const McgCellGroup& G = m.cgs[m.cg_off[c] + gi];
          const int kd = m.specs[G.spec].kind;
          if (kd == MCG_SYN_STATIC_COND || kd == MCG_SYN_STDP_COND || kd == MCG_SYN_STATIC_CURRENT ||
              kd == MCG_SYN_HOMEO_CURRENT)
            tot += (G.size + 31) & ~31;
        }
        amax = std::max(amax, tot);
      }
      if (amax >= 256 && bc_smem + size_t(amax) * 12 + 64 <= size_t(smem_optin) - 4096) bc_act_max = amax;
      bc_smem += size_t(bc_act_max) * 12;
    }
    // staged delivery: the epoch's due events of the resident batch in shared
    // memory (mcg_stage_events), in whatever the opt-in limit leaves
    bc_ev_cap = 0;
    if (!std::getenv("MCG_NO_STAGED_EVENTS")) {
      const size_t lim = size_t(smem_optin) - 4096;  // static shared memory of the kernel
      const size_t left = lim > bc_smem + 32 ? lim - bc_smem - 32 : 0;
      bc_ev_cap = static_cast<int32_t>(std::min<size_t>(left / sizeof(McgEvSm), 4096));
      if (bc_ev_cap < 64) bc_ev_cap = 0;
      if (bc_ev_cap > 0) bc_smem += size_t(bc_ev_cap) * sizeof(McgEvSm) + 16;
    }
    CK(cudaFuncSetAttribute(k_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(bc_smem)));
    // leave the rest of the unified L1/shared array to L1 (STC state streams through it)
    bc_carve = std::min(100, static_cast<int>((bc_smem * 100 + 228 * 1024 - 1) / (228 * 1024)) + 5);
    const int carve = bc_carve;
    CK(cudaFuncSetAttribute(k_batch, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_batch, kBatchThreads, bc_smem));
    if (occ < 1) throw Error(MCG_ERR_CUDA, "batch kernel does not fit on an SM");
    // few batches but many sources: widen towards one CTA per SM, since the
    // CTAs without a batch still expand source events (a single neuron with
    // 1000 Poisson inputs); with few sources every extra CTA only adds to the
    // grid barriers (one synapse on one neuron: config 1)
    const int64_t want = std::min<int64_t>(dev_sms, (static_cast<int64_t>(m.sources.size()) + 3) / 4);
    bc_grid = static_cast<int>(std::min<int64_t>(std::max<int64_t>(bc_batches, want),
                                                 int64_t(occ) * dev_sms));
    if (bc_stc_sm && bc_grid < bc_batches) throw Error(MCG_ERR_CUDA, "batch kernel: not resident");
    d_chunks.alloc(size_t(kBatch) * bc_batches + 1);
    d_chunk_n.alloc(1);
    d_chunk_n.zero(st);
    if (!evk0) CK(cudaEventCreate(&evk0));
    if (!evk1) CK(cudaEventCreate(&evk1));
  }

  int32_t n_local() const { return static_cast<int32_t>(m.cell_kind.size()); }

  // k_warp (mcg_warp.cuh) runs networks whose every kind is a LIF cell small
  // enough for shared memory, cable kinds with constant, chain-scheduled V and
  // species systems, and at most one STC placement plus static-charge ones:
  // every consolidation network.  Everything else runs on k_batch.
  bool warp_eligible(std::string* why) const {
    auto no = [&](const char* w) {
      if (why) *why = w;
      return false;
    };
    if (std::getenv("MCG_NO_WARP")) return no("MCG_NO_WARP");
    const int nl = n_local();
    if (nl == 0) return no("no local cells");
    if (sp_max > 15) return no("more than 15 species");
    std::vector<char> used(m.kinds.size(), 0);
    for (int c = 0; c < nl; ++c) used[m.cell_kind[c]] = 1;
    for (size_t ki = 0; ki < m.kinds.size(); ++ki) {
      if (!used[ki]) continue;
      const McgKind& K = m.kinds[ki];
      if (K.n > smem_n || K.n > 0xffff) return no("kind too large for shared memory");
      if (K.dyn == MCG_DYN_LIF_EXACT) {
        if (K.n != 1) return no("exact LIF with several compartments");
      } else if (K.dyn == MCG_DYN_LIF) {
        if (!K.v_const) return no("LIF cable without a constant V system");
        if (K.n > 1 && (K.ch_lp == 0 || (K.n_species > 0 && !K.sp_const)))
          return no("cable kind without a chain schedule");
      } else {
        return no("membrane is not LIF");
      }
      if (K.n_groups > 8) return no("more than 8 placements");
      int n_stc = 0;
      for (int gi = 0; gi < K.n_groups; ++gi) {
        const int kd = m.specs[K.spec0 + gi].kind;
        if (kd == MCG_SYN_STC_CHARGE) ++n_stc;
        else if (kd != MCG_SYN_STATIC_CHARGE) return no("synapse kind other than charge / STC");
      }
      if (n_stc > 1) return no("more than one STC placement");
    }
    for (int c = 0; c < nl; ++c) {
      const McgKind& K = m.kinds[m.cell_kind[c]];
      for (int gi = 0; gi < K.n_groups; ++gi) {
        const McgCellGroup& G = m.cgs[m.cg_off[c] + gi];
        if (m.specs[G.spec].kind != MCG_SYN_STC_CHARGE) continue;
        if (G.size > 32 * MCG_MW_MAX) return no("more than 1024 STC synapses on a cell");
        if (G.fifo < 0) return no("STC group without a delayed-calcium queue");
      }
    }
    return true;
  }

  void setup_warp_kernel() {
    use_warp = false;
    std::string why;
    if (!warp_eligible(&why)) {
      if (std::getenv("MCG_VERBOSE")) std::fprintf(stderr, "engine: k_batch (%s)\n", why.c_str());
      return;
    }
    const int nl = n_local();
    int dev_sms = 148, smem_optin = 0;
    CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    // kind blocks (mcg_kind_block_doubles), one per kind
    std::vector<int32_t> kb(m.kinds.size(), -1);
    int kd = 0, pmax = 0;
    for (size_t ki = 0; ki < m.kinds.size(); ++ki) {
      const McgKind& K = m.kinds[ki];
      if (K.n > smem_n) continue;
      kb[ki] = kd;
      kd += mcg_kind_block_doubles(K.n, K.n_species, K.ch_lp);
      if (K.ch_lp > 0) pmax = std::max(pmax, 2 * K.ch_lp + 1);
    }
    int stc_max = 0;
    bool lazy = !std::getenv("MCG_NO_LAZY");
    for (int c = 0; c < nl; ++c) {
      const McgKind& K = m.kinds[m.cell_kind[c]];
      for (int gi = 0; gi < K.n_groups; ++gi) {
        const McgCellGroup& G = m.cgs[m.cg_off[c] + gi];
        if (m.specs[G.spec].kind == MCG_SYN_STC_CHARGE) stc_max = std::max(stc_max, G.size);
      }
    }
    // lazy calcium needs a resting calcium to stay below the thresholds and a
    // late step that is a no-op at rest (mcg_warp.cuh)
    for (const McgSpec& S : m.specs) {
      if (S.kind != MCG_SYN_STC_CHARGE) continue;
      if (!(S.theta_p >= 0.0 && S.theta_d >= 0.0 && S.cf >= 0.0 && S.cf <= 1.0 && S.theta_tag >= 0.0 &&
            std::fabs(S.f_int) <= 1.7976931348623157e308))
        lazy = false;
    }
    wg_lazy = lazy ? 1 : 0;
    wg_kind_doubles = kd;
    wg_P = pmax;
    wg_MW = std::max(1, (stc_max + 31) / 32);
    const int S = sp_max;
    // every cell of a group has 2 (1 + S) system lanes (mcg_wg_epoch phase D)
    const int g_max = std::max(1, std::min(MCG_WG_MAX, 32 / (2 * (1 + S))));
    wg_specs_sm = m.specs.size() * sizeof(McgSpec) <= 16 * 1024 ? static_cast<int32_t>(m.specs.size()) : 0;
    wg_ev_cap = 128;
    if (const char* ev = std::getenv("MCG_WARP_EVCAP")) wg_ev_cap = std::max(0, std::atoi(ev));
    const size_t fixed = size_t(wg_kind_doubles) * 8 + ((m.kinds.size() * sizeof(McgKind) + 7) / 8) * 8 +
                        ((size_t(wg_specs_sm) * sizeof(McgSpec) + 7) / 8) * 8;
    const size_t lim = size_t(smem_optin) - 2048;
    auto warps_fit = [&](int g) {  // warps per CTA that fit the shared memory with groups of g
      const size_t wd = size_t(mcg_warp_region_doubles(g, smem_n, S, wg_P, wg_MW, wg_ev_cap)) * 8;
      return fixed + wd > lim ? 0 : static_cast<int>(std::min<size_t>(8, (lim - fixed) / wd));
    };
    // group size: each warp's step is a latency-bound chain whose length
    // hardly depends on G, so more, smaller groups put more warps on each SM
    // (config 3: G = 2 runs 10-15 % faster than G = 5); the smallest G >= 2
    // that keeps every group resident, else the largest (fewer groups to
    // stage per epoch)
    wg_G = g_max;
    for (int g = std::min(2, g_max); g <= g_max; ++g)
      if ((nl + g - 1) / g <= dev_sms * warps_fit(g)) {
        wg_G = g;
        break;
      }
    if (const char* gv = std::getenv("MCG_WARP_G")) wg_G = std::clamp(std::atoi(gv), 1, g_max);
    wg_groups = (nl + wg_G - 1) / wg_G;
    wg_warp_doubles = mcg_warp_region_doubles(wg_G, smem_n, S, wg_P, wg_MW, wg_ev_cap);
    if (fixed + size_t(wg_warp_doubles) * 8 > lim) {
      if (std::getenv("MCG_VERBOSE")) std::fprintf(stderr, "engine: k_batch (warp region too large)\n");
      return;
    }
    const int max_warps = static_cast<int>(std::min<size_t>(8, (lim - fixed) / (size_t(wg_warp_doubles) * 8)));
    // resident when every group has its own warp: spread over the SMs
    if (wg_groups <= dev_sms * max_warps) {
      wg_resident = 1;
      wg_grid = std::min(dev_sms, wg_groups);
      wg_warps = (wg_groups + wg_grid - 1) / wg_grid;
    } else {
      wg_resident = 0;
      wg_grid = dev_sms;
      wg_warps = max_warps;
    }
    // test hooks: fewer warps / CTAs (forces per-epoch group staging on small nets)
    if (const char* wv = std::getenv("MCG_WARP_WARPS")) wg_warps = std::clamp(std::atoi(wv), 1, max_warps);
    if (const char* gv = std::getenv("MCG_WARP_GRID")) wg_grid = std::clamp(std::atoi(gv), 1, dev_sms);
    wg_resident = wg_groups <= wg_grid * wg_warps ? 1 : 0;
    wg_smem = fixed + size_t(wg_warps) * wg_warp_doubles * 8 + 64;
    CK(cudaFuncSetAttribute(k_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(wg_smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_warp, wg_warps * 32, wg_smem));
    if (occ < 1) {
      if (std::getenv("MCG_VERBOSE")) std::fprintf(stderr, "engine: k_batch (k_warp does not fit)\n");
      return;
    }
    wg_grid = std::min(wg_grid, occ * dev_sms);
    if (wg_resident && wg_groups > wg_grid * wg_warps) wg_resident = 0;
    d_kb_off.upload(kb, st);
    d_stc_mask.alloc(size_t(std::max(nl, 1)) * wg_MW);
    d_stc_mask.zero(st);
    d_stc_t.alloc(std::max<size_t>(m.i_stc_h.size(), 1));
    d_chunks.alloc(size_t(kBatch) * std::max(bc_batches, wg_groups) + 1);
    use_warp = true;
    lazy_valid = false;
    lazy_dirty = false;
    // inboxes sized so that no epoch's expansion can overflow them: the
    // kernel then skips the per-epoch overflow check (up to 1/4 of the free
    // device memory, at most 8 GiB)
    {
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      wg_no_abort = (!std::getenv("MCG_WARP_ABORT_CHECK") &&
                     size_inboxes_for_worst_case(std::min(fr / 4, size_t(8) << 30))) ? 1 : 0;
    }
    if (std::getenv("MCG_VERBOSE"))
      std::fprintf(stderr, "engine: k_warp G=%d groups=%d grid=%d warps=%d resident=%d P=%d MW=%d lazy=%d smem=%zu "
                   "no_abort=%d inc_cap=%d pend_cap=%d\n",
                   wg_G, wg_groups, wg_grid, wg_warps, wg_resident, wg_P, wg_MW, wg_lazy, wg_smem, wg_no_abort,
                   inc_cap, pend_cap);
  }

  // k_point (mcg_point.cuh) runs networks of exact-LIF point cells with
  // charge-type synapses and no cell-to-cell connections (one epoch spans the
  // whole call in the reference, engine.cpp:913-915): one thread carries a
  // cell's state in registers through the epoch, one CTA per cell.
  bool point_eligible(int dev_sms, std::string* why) const {
    auto no = [&](const char* w) {
      if (why) *why = w;
      return false;
    };
    if (std::getenv("MCG_NO_POINT")) return no("MCG_NO_POINT");
    if (m.world != 1) return no("sharded");
    if (m.min_delay_steps > 0) return no("cell-to-cell connections");
    if (L > MCG_PT_NB) return no("epoch longer than the noise buffer");
    const int nl = n_local();
    if (nl == 0 || nl > dev_sms) return no("cell count outside 1..#SMs");
    for (int c = 0; c < nl; ++c) {
      const McgKind& K = m.kinds[m.cell_kind[c]];
      if (K.dyn != MCG_DYN_LIF_EXACT || K.n != 1) return no("not an exact-LIF point cell");
      if (K.n_species > MCG_PT_SP) return no("too many species");
      if (K.n_groups > 8) return no("more than 8 placements");
      int n_stc = 0;
      for (int gi = 0; gi < K.n_groups; ++gi) {
        const McgCellGroup& G = m.cgs[m.cg_off[c] + gi];
        const int kd = m.specs[G.spec].kind;
        if (kd == MCG_SYN_STC_CHARGE) {
          ++n_stc;
          if (G.size > MCG_PT_STC) return no("too many STC synapses on a point cell");
          if (G.size > 0 && G.fifo < 0) return no("STC group without a delayed-calcium queue");
        } else if (kd != MCG_SYN_STATIC_CHARGE) {
          return no("synapse kind other than charge / STC");
        }
      }
      if (n_stc > 1) return no("more than one STC placement");
    }
    return true;
  }

  void setup_point_kernel() {
    use_point = false;
    int dev_sms = 148;
    CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device));
    std::string why;
    if (!point_eligible(dev_sms, &why)) {
      if (std::getenv("MCG_VERBOSE")) std::fprintf(stderr, "engine: no k_point (%s)\n", why.c_str());
      return;
    }
    pt_grid = n_local();
    pt_small = true;
    for (int c = 0; c < pt_grid; ++c) {
      const McgKind& K = m.kinds[m.cell_kind[c]];
      if (K.n_species > 2) pt_small = false;
      for (int gi = 0; gi < K.n_groups; ++gi) {
        const McgCellGroup& G = m.cgs[m.cg_off[c] + gi];
        if (m.specs[G.spec].kind == MCG_SYN_STC_CHARGE && G.size > 1) pt_small = false;
      }
    }
    d_chunks.alloc(size_t(kBatch) * std::max<int64_t>(std::max(bc_batches, wg_groups), pt_grid) + 1);
    use_point = true;
    use_warp = false;  // no lazy calcium: the synapses' calcium is stepped in registers
    if (std::getenv("MCG_VERBOSE")) std::fprintf(stderr, "engine: k_point grid=%d L=%lld\n", pt_grid, (long long)L);
  }

  // lazy calcium (mcg_warp.cuh): masks and stamps from the current state
  void lazy_init() {
    if (!use_warp || lazy_valid) return;
    const int nl = n_local();
    refresh_dev();
    const int dbg = std::getenv("MCG_WARP_DBG") ? std::atoi(std::getenv("MCG_WARP_DBG")) : 0;
    k_lazy_init<<<(nl * 32 + 255) / 256, 256, 0, st>>>(dev, d_stc_mask.p, d_stc_t.p, wg_MW,
                                                        (wg_lazy && (dbg & 4)) ? 2 : wg_lazy, step);
    CK(cudaGetLastError());
    stats.kernel_launches += 1;
    lazy_valid = true;
    lazy_dirty = false;
  }
  // every resting synapse's calcium brought to `step` (before the host reads
  // or rewrites STC state)
  void ensure_flushed() {
    if (!use_warp || !lazy_dirty) return;
    const int nl = n_local();
    refresh_dev();
    k_lazy_flush<<<(nl * 32 + 255) / 256, 256, 0, st>>>(dev, d_stc_mask.p, d_stc_t.p, wg_MW, step);
    CK(cudaGetLastError());
    stats.kernel_launches += 1;
    lazy_dirty = false;
    lazy_valid = false;  // stamps are stale now; the next advance re-derives them
  }

  void init(const mcg_recipe& r, const mcg_options& opt) {
    device = opt.device;
    CK(cudaSetDevice(device));
    {  // keep freed device memory in the pool (DBuf allocations)
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
    }
    const auto t0 = std::chrono::steady_clock::now();
    build_model(r, opt, m, 0, !std::getenv("MCG_HOST_RESOLVE"));
    {
      // grow the device pool once to about the engine's size: the uploads
      // below are then served from memory the pool already holds instead of
      // mapping it allocation by allocation (config 5: 1.3 s -> 0.15 s of
      // uploads for the first engine of a process)
      const size_t ne = size_t(m.n_edges), ni = size_t(m.n_inst), nc = m.v.size() + m.species.size();
      // (device-resolved edges: plus the resolution's transient buffers)
      const size_t est = ne * (m.edges_deferred ? 128 : 56) + ni * 112 + nc * 80 + size_t(m.fifo_total) * 32 +
                         (size_t(64) << 20);
      // skipped when the pool already holds that much free (an earlier
      // engine's memory): a second growth would map memory the pool has
      size_t have = 0;
      {
        cudaMemPool_t pool;
        uint64_t reserved = 0, used = 0;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
          have = size_t(reserved - used);
        cudaGetLastError();
      }
      void* p = nullptr;
      if (have >= est) {
      } else if (cudaMallocAsync(&p, est, 0) == cudaSuccess) {
        cudaFreeAsync(p, 0);
        cudaStreamSynchronize(0);
      } else {
        cudaGetLastError();  // not fatal: the uploads allocate as they go
      }
    }
    const auto t1 = std::chrono::steady_clock::now();
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaMallocHost(&h_ctr, C_N * sizeof(unsigned long long)));
    CK(cudaMallocHost(&h_err, sizeof(int32_t)));
    CK(cudaMallocHost(&h_abort, sizeof(int32_t)));
    CK(cudaMallocHost(&h_ctl, 4 * sizeof(int64_t)));
    CK(cudaEventCreate(&eva));
    CK(cudaEventCreate(&evb));
    const int nl = n_local();
    // epoch length: min delay (cells independent within it, engine.cpp:913-915)
    const int64_t free_epoch = std::clamp<int64_t>((int64_t(1) << 22) / std::max(nl, 1), 16, 4096);
    L = m.min_delay_steps > 0 ? m.min_delay_steps : free_epoch;
    // spikes per cell per epoch: at most one per (ref_steps + 1) steps (LIF)
    // or every other step (HH hysteresis)
    sp_cap = 1;
    for (const McgKind& K : m.kinds) {
      int64_t b = 0;
      if (K.dyn == MCG_DYN_LIF || K.dyn == MCG_DYN_LIF_EXACT) b = (L + K.ref_steps) / (K.ref_steps + 1);
      else if (K.dyn == MCG_DYN_HH) b = (L + 1) / 2;
      sp_cap = static_cast<int32_t>(std::max<int64_t>(sp_cap, std::min<int64_t>(b, L)));
    }
    const int64_t ne = m.n_edges;
    rank_bits = bits_for(static_cast<uint64_t>(std::max<int64_t>(ne, 1)));
    if (rank_bits > 30) throw Error(MCG_ERR_ENGINE, "too many local edges for the event key");

    d_kinds.upload(m.kinds, st);
    d_specs.upload(m.specs, st);
    d_k_parent.upload(m.k_parent, st);
    d_k_ch_idx.upload(m.k_ch_idx, st);
    d_k_cap_dt.upload(m.k_cap_dt, st);
    d_k_g_leak.upload(m.k_g_leak, st);
    d_k_g_leak_rhs.upload(m.k_g_leak_rhs, st);
    d_k_axial.upload(m.k_axial, st);
    d_k_g_na.upload(m.k_g_na, st);
    d_k_g_k.upload(m.k_g_k, st);
    d_k_cf.upload(m.k_cf, st);
    d_k_volume.upload(m.k_volume, st);
    d_k_sp_cap_dt.upload(m.k_sp_cap_dt, st);
    d_k_sp_gs.upload(m.k_sp_gs, st);
    d_k_sp_coupling.upload(m.k_sp_coupling, st);
    d_k_vf.upload(m.k_vf, st);
    d_k_vd.upload(m.k_vd, st);
    d_k_sp_f.upload(m.k_sp_f, st);
    d_k_sp_d.upload(m.k_sp_d, st);
    d_k_vr.upload(m.k_vr, st);
    d_k_sp_r.upload(m.k_sp_r, st);
    d_k_rvol.upload(m.k_rvol, st);
    d_cell_kind.upload(m.cell_kind, st);
    d_comp_off.upload(m.comp_off, st);
    d_sp_off.upload(m.sp_off, st);
    d_cg_off.upload(m.cg_off, st);
    d_v.upload(m.v, st);
    d_hh_m.upload(m.hh_m, st);
    d_hh_h.upload(m.hh_h, st);
    d_hh_n.upload(m.hh_n, st);
    d_species.upload(m.species, st);
    d_det_prev.upload(m.det_prev, st);
    d_armed.upload(m.armed, st);
    d_refr.upload(m.refr_until, st);
    d_iseq.upload(m.internal_seq, st);
    const size_t nc = std::max<size_t>(m.v.size(), 1) + 1;
    d_s_gsyn.alloc(nc);
    d_s_gsyn_rhs.alloc(nc);
    d_s_rhs_cur.alloc(nc);
    d_s_diag.alloc(nc);
    d_s_rhs.alloc(nc);
    for (const McgKind& K : m.kinds) {
      sp_max = std::max(sp_max, K.n_species);
      if (K.n <= kSmemMaxComps) smem_n = std::max(smem_n, K.n);
    }
    d_s_r2.alloc(nc * (1 + sp_max));
    smem_stride = (9 + 2 * sp_max) * smem_n;
    smem_bytes = static_cast<size_t>(smem_stride) * sizeof(double) * (kBlock / 32);
    CK(cudaFuncSetAttribute(k_ff, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem_bytes)));
    d_cgs.upload(m.cgs, st);
    d_fifos.upload(m.fifos, st);
    d_fifo_step.alloc(std::max<int64_t>(m.fifo_total, 1));
    d_fifo_si.alloc(std::max<int64_t>(m.fifo_total, 1));
    d_fifo_src.alloc(std::max<int64_t>(m.fifo_total, 1));
    d_fifo_w.alloc(std::max<int64_t>(m.fifo_total, 1));
    d_i_comp.upload(m.i_comp, st);
    d_i_active.alloc(std::max<size_t>(m.i_comp.size(), 1));
    // instance arrays the build left empty start all zero: fill on the device
    auto up_or_zero = [&](auto& d, const auto& h) {
      if (!h.empty()) {
        d.upload(h, st);
      } else {
        d.alloc(std::max<size_t>(size_t(m.n_inst), 1));
        d.zero(st);
      }
    };
    up_or_zero(d_i_weight, m.i_weight);
    up_or_zero(d_i_kernel, m.i_kernel);
    up_or_zero(d_i_stdp_pre, m.i_stdp_pre);
    up_or_zero(d_i_stdp_post, m.i_stdp_post);
    up_or_zero(d_i_stdp_w, m.i_stdp_w);
    up_or_zero(d_i_stdp_last, m.i_stdp_last);
    up_or_zero(d_i_homeo_w, m.i_homeo_w);
    up_or_zero(d_i_stc_h, m.i_stc_h);
    up_or_zero(d_i_stc_z, m.i_stc_z);
    up_or_zero(d_i_stc_c, m.i_stc_c);
    up_or_zero(d_i_sps_abs, m.i_sps_abs);
    d_stc_nz.alloc(std::max<size_t>(m.i_stc_h.size(), 1));
    if (d_stc_nz.p)
      CK(cudaMemsetAsync(d_stc_nz.p, 0xff, d_stc_nz.n * sizeof(McgNzCache), st));  // tag -1
    if (m.edges_deferred) {
      resolve_edges(r);
    } else {
      d_e_dst.upload(m.e_dst, st);
      d_e_group.upload(m.e_group, st);
      d_e_inst.upload(m.e_inst, st);
      d_e_weight.upload(m.e_weight, st);
      d_e_src.upload(m.e_src, st);
      d_e_comp.upload(m.e_comp, st);
      d_e_wcf.upload(m.e_wcf, st);
      d_e_delay.upload(m.e_delay, st);
      d_src_edges.upload(m.src_edges, st);
    }
    d_out_begin.upload(m.out_begin, st);
    d_out_end.upload(m.out_end, st);
    d_src_edge_off.upload(m.src_edge_off, st);

    // source tasks: one per Poisson window, one per regular/scripted source
    std::vector<McgSrcTask> tasks;
    std::vector<int64_t> scripted;
    for (size_t s = 0; s < m.sources.size(); ++s) {
      const Source& S = m.sources[s];
      McgSrcTask T{};
      T.source = static_cast<int32_t>(s);
      T.type = S.type;
      if (S.type == MCG_SRC_POISSON) {
        for (size_t w = 0; w < S.prob.size(); ++w) {
          T.window = static_cast<int32_t>(w);
          T.a = S.a[w];
          T.b = S.b[w];
          T.prob = S.prob[w];
          tasks.push_back(T);
        }
      } else if (S.type == MCG_SRC_REGULAR) {
        T.r_t0 = S.r_t0;
        T.r_period = S.r_period;
        T.r_count = S.r_count;
        tasks.push_back(T);
      } else {
        T.a = static_cast<int64_t>(scripted.size());
        for (int64_t x : S.steps) scripted.push_back(x);
        T.b = static_cast<int64_t>(scripted.size());
        tasks.push_back(T);
      }
    }
    // Poisson windows first (expanded per (window, step)), then the sources
    // expanded once per epoch; the expansion's push order is irrelevant (the
    // inbox sort orders the keys)
    std::stable_partition(tasks.begin(), tasks.end(),
                          [](const McgSrcTask& T) { return T.type == MCG_SRC_POISSON; });
    n_tasks = static_cast<int32_t>(tasks.size());
    n_poisson = 0;
    for (const McgSrcTask& T : tasks) n_poisson += T.type == MCG_SRC_POISSON ? 1 : 0;
    d_tasks.upload(tasks, st);
    d_scripted.upload(scripted, st);

    // inboxes, sized from the mean in-degree; grown on overflow
    {
      const double per_cell = double(ne) / std::max(nl, 1);
      while (inc_cap < 4 * per_cell && inc_cap < (1 << 20)) inc_cap <<= 1;
      pend_cap = 2 * inc_cap;
    }
    alloc_inboxes();
    d_ctl.alloc(4);
    d_abort.alloc(1);
    d_abort.zero(st);

    const size_t slots = static_cast<size_t>(std::max(nl, 1)) * sp_cap;
    d_sp_count.alloc(std::max(nl, 1));
    d_sp_count.zero(st);
    d_sp_step.alloc(slots);
    d_sp_t.alloc(slots);
    d_log_t.alloc(slots * kBatch);
    d_log_gid.alloc(slots * kBatch);

    // probes: per-cell CSR over local probes
    std::vector<int32_t> poff(nl + 1, 0), pidx;
    for (const auto& P : m.probes)
      if (P.local >= 0) ++poff[P.local + 1];
    for (int c = 0; c < nl; ++c) poff[c + 1] += poff[c];
    pidx.resize(poff[nl]);
    {
      std::vector<int32_t> fill(poff.begin(), poff.end() - 1);
      for (size_t p = 0; p < m.probes.size(); ++p)
        if (m.probes[p].local >= 0) pidx[fill[m.probes[p].local]++] = static_cast<int32_t>(p);
    }
    d_probes.upload(m.probes, st);
    d_probe_off.upload(poff, st);
    d_probe_idx.upload(pidx, st);
    d_trace.alloc(1);
    d_trace_base.alloc(std::max<size_t>(m.probes.size(), 1));
    traces.assign(m.probes.size(), {});

    d_ctr.alloc(C_N);
    d_ctr.zero(st);
    d_err.alloc(1);
    d_err.zero(st);
    CK(cudaStreamSynchronize(st));

    stats.total_comps = m.total_comps;
    stats.total_synapses = m.total_syn;
    stats.stc_synapses = m.stc_syn;
    stats.hh_comps = m.hh_comps;
    stats.species_comps = m.species_comps;
    const auto t2 = std::chrono::steady_clock::now();
    setup_batch_kernel();
    setup_warp_kernel();
    setup_point_kernel();
    refresh_dev();
    if (std::getenv("MCG_PROFILE_BUILD")) {
      const auto t3 = std::chrono::steady_clock::now();
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "engine: build_model %.2f ms, uploads %.2f ms, batch setup %.2f ms\n",
                   ms(t0, t1), ms(t1, t2), ms(t2, t3));
    }
  }

  void alloc_inboxes() {
    const size_t nl = static_cast<size_t>(std::max(n_local(), 1));
    d_inc.alloc(nl * inc_cap);
    d_pend.alloc(nl * 2 * pend_cap);
    d_inc_n.alloc(nl);
    d_inc_n.zero(st);
    d_pend_sel.alloc(nl);
    d_pend_sel.zero(st);
    d_pend_off.alloc(nl);
    d_pend_off.zero(st);
    d_pend_n.alloc(nl);
    d_pend_n.zero(st);
  }

  // double both inbox capacities, keeping the pending keys
  void grow_inboxes() {
    const int nl = n_local();
    const int32_t old_pend = pend_cap;
    DBuf<uint64_t> np;
    inc_cap *= 2;
    pend_cap *= 2;
    np.alloc(static_cast<size_t>(std::max(nl, 1)) * 2 * pend_cap);
    if (nl > 0)
      k_pend_regrow<<<(nl * 32 + 127) / 128, 128, 0, st>>>(d_pend.p, old_pend, np.p, pend_cap,
                                                           d_pend_sel.p, d_pend_off.p,
                                                           d_pend_n.p, nl);
    CK(cudaStreamSynchronize(st));
    std::swap(d_pend.p, np.p);
    std::swap(d_pend.n, np.n);
    d_inc.alloc(static_cast<size_t>(std::max(nl, 1)) * inc_cap);
    d_inc_n.zero(st);
  }

  void refresh_dev() {
    McgDev& D = dev;
    D.dt = m.dt;
    D.seed = m.seed;
    D.kinds = d_kinds.p;
    D.specs = d_specs.p;
    D.k_parent = d_k_parent.p;
    D.k_ch_idx = d_k_ch_idx.p;
    D.k_cap_dt = d_k_cap_dt.p;
    D.k_g_leak = d_k_g_leak.p;
    D.k_g_leak_rhs = d_k_g_leak_rhs.p;
    D.k_axial = d_k_axial.p;
    D.k_g_na = d_k_g_na.p;
    D.k_g_k = d_k_g_k.p;
    D.k_cf = d_k_cf.p;
    D.k_volume = d_k_volume.p;
    D.k_sp_cap_dt = d_k_sp_cap_dt.p;
    D.k_sp_gs = d_k_sp_gs.p;
    D.k_sp_coupling = d_k_sp_coupling.p;
    D.n_cells = n_local();
    D.gid0 = m.gid_begin;
    D.cell_kind = d_cell_kind.p;
    D.comp_off = d_comp_off.p;
    D.sp_off = d_sp_off.p;
    D.cg_off = d_cg_off.p;
    D.v = d_v.p;
    D.hh_m = d_hh_m.p;
    D.hh_h = d_hh_h.p;
    D.hh_n = d_hh_n.p;
    D.species = d_species.p;
    D.det_prev = d_det_prev.p;
    D.armed = d_armed.p;
    D.refr_until = d_refr.p;
    D.internal_seq = d_iseq.p;
    D.s_gsyn = d_s_gsyn.p;
    D.s_gsyn_rhs = d_s_gsyn_rhs.p;
    D.s_rhs_cur = d_s_rhs_cur.p;
    D.s_diag = d_s_diag.p;
    D.s_rhs = d_s_rhs.p;
    D.s_r2 = d_s_r2.p;
    D.k_vf = d_k_vf.p;
    D.k_vd = d_k_vd.p;
    D.k_sp_f = d_k_sp_f.p;
    D.k_sp_d = d_k_sp_d.p;
    D.k_vr = d_k_vr.p;
    D.k_sp_r = d_k_sp_r.p;
    D.k_rvol = d_k_rvol.p;
    D.sp_max = sp_max;
    D.smem_n = smem_n;
    D.smem_stride = smem_stride;
    D.cgs = d_cgs.p;
    D.fifos = d_fifos.p;
    D.fifo_step = d_fifo_step.p;
    D.fifo_si = d_fifo_si.p;
    D.fifo_src = d_fifo_src.p;
    D.fifo_w = d_fifo_w.p;
    D.i_comp = d_i_comp.p;
    D.i_weight = d_i_weight.p;
    D.i_kernel = d_i_kernel.p;
    D.i_active = d_i_active.p;
    D.i_stdp_pre = d_i_stdp_pre.p;
    D.i_stdp_post = d_i_stdp_post.p;
    D.i_stdp_w = d_i_stdp_w.p;
    D.i_stdp_last = d_i_stdp_last.p;
    D.i_homeo_w = d_i_homeo_w.p;
    D.i_stc_h = d_i_stc_h.p;
    D.stc_nz = d_stc_nz.p;
    D.i_stc_z = d_i_stc_z.p;
    D.i_stc_c = d_i_stc_c.p;
    D.i_sps_abs = d_i_sps_abs.p;
    D.inc = d_inc.p;
    D.inc_n = d_inc_n.p;
    D.inc_cap = inc_cap;
    D.pend = d_pend.p;
    D.pend_sel = d_pend_sel.p;
    D.pend_off = d_pend_off.p;
    D.pend_n = d_pend_n.p;
    D.pend_cap = pend_cap;
    D.rank_bits = rank_bits;
    D.ctl = d_ctl.p;
    D.abort = d_abort.p;
    D.e_dst = d_e_dst.p;
    D.e_group = d_e_group.p;
    D.e_inst = d_e_inst.p;
    D.e_weight = d_e_weight.p;
    D.e_src = d_e_src.p;
    D.e_comp = d_e_comp.p;
    D.e_wcf = d_e_wcf.p;
    D.e_delay = d_e_delay.p;
    D.sp_cap = sp_cap;
    D.sp_count = d_sp_count.p;
    D.sp_step = d_sp_step.p;
    D.sp_t = d_sp_t.p;
    D.probes = d_probes.p;
    D.probe_off = d_probe_off.p;
    D.probe_idx = d_probe_idx.p;
    D.trace_buf = d_trace.p;
    D.trace_base = d_trace_base.p;
    D.err = d_err.p;
    D.delivered = d_ctr.p + C_DELIVERED;
    D.cell_seed = d_cell_seed.n ? d_cell_seed.p : nullptr;
    D.cell_key_gid = d_cell_key_gid.n ? d_cell_key_gid.p : nullptr;
  }

  McgEv ev_dev() {
    McgEv E{};
    E.tasks = d_tasks.p;
    E.n_tasks = n_tasks;
    E.n_poisson = n_poisson;
    E.scripted_steps = d_scripted.p;
    E.src_edge_off = d_src_edge_off.p;
    E.src_edges = d_src_edges.p;
    E.e_dst = d_e_dst.p;
    E.e_delay = d_e_delay.p;
    E.out_begin = d_out_begin.p;
    E.out_end = d_out_end.p;
    E.inc = d_inc.p;
    E.inc_n = d_inc_n.p;
    E.inc_cap = inc_cap;
    E.pend_off = d_pend_off.p;
    E.pend_n = d_pend_n.p;
    E.pend_cap = pend_cap;
    E.rank_bits = rank_bits;
    E.ctl = d_ctl.p;
    E.abort = d_abort.p;
    E.seed = m.seed;
    E.dt = m.dt;
    return E;
  }

  void check_err() {
    if (*h_err == 0) return;
    const int e = *h_err;
    *h_err = 0;
    CK(cudaMemsetAsync(d_err.p, 0, sizeof(int32_t), st));
    if (e & MCG_ERR_FLAG_SINGULAR) throw Error(MCG_ERR_NUMERIC, "tree solve: singular system");
    if (e & MCG_ERR_FLAG_FIFO) throw Error(MCG_ERR_ENGINE, "internal event queue overflow");
    if (e & MCG_ERR_FLAG_ACTIVE) throw Error(MCG_ERR_ENGINE, "active synapse list overflow");
    if (e & MCG_ERR_FLAG_SPIKES) throw Error(MCG_ERR_ENGINE, "spike buffer overflow");
  }

  void sync_counters_raw() {
    CK(cudaMemcpyAsync(h_ctr, d_ctr.p, C_N * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_err, d_err.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_abort, d_abort.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    stats.events_delivered = static_cast<int64_t>(h_ctr[C_DELIVERED]);
  }

  // spike log of one launch: chunks (epoch, batch, offset, count) -> the
  // reference's order (epoch, then gid, then step; engine.cpp:877-888)
  void drain_chunks() {
    unsigned long long nch = 0;
    CK(cudaMemcpyAsync(&nch, d_chunk_n.p, sizeof(nch), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t n = static_cast<int64_t>(h_ctr[C_LOG]);
    if (nch == 0 || n == 0) {
      CK(cudaMemsetAsync(d_chunk_n.p, 0, sizeof(unsigned long long), st));
      CK(cudaMemsetAsync(d_ctr.p + C_LOG, 0, sizeof(unsigned long long), st));
      h_ctr[C_LOG] = 0;
      return;
    }
    std::vector<int4> ch(nch);
    std::vector<double> lt(n);
    std::vector<uint32_t> lg(n);
    CK(cudaMemcpyAsync(ch.data(), d_chunks.p, nch * sizeof(int4), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(lt.data(), d_log_t.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(lg.data(), d_log_gid.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemsetAsync(d_chunk_n.p, 0, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(d_ctr.p + C_LOG, 0, sizeof(unsigned long long), st));
    CK(cudaStreamSynchronize(st));
    h_ctr[C_LOG] = 0;
    std::sort(ch.begin(), ch.end(), [](const int4& a, const int4& b) {
      return a.x != b.x ? a.x < b.x : a.y < b.y;
    });
    if (use_warp) {
      // k_warp's groups hold strided gids: within an epoch, order by gid (a
      // cell's spikes are contiguous and in step order, so a stable sort)
      size_t a = 0;
      std::vector<int64_t> idx;
      while (a < ch.size()) {
        size_t b = a;
        idx.clear();
        while (b < ch.size() && ch[b].x == ch[a].x) {
          for (int i = 0; i < ch[b].w; ++i) idx.push_back(ch[b].z + i);
          ++b;
        }
        std::stable_sort(idx.begin(), idx.end(), [&](int64_t u, int64_t v) { return lg[u] < lg[v]; });
        for (int64_t q : idx) {
          spk_t.push_back(lt[q]);
          spk_gid.push_back(lg[q]);
        }
        a = b;
      }
    } else {
      for (const int4& q : ch)
        for (int i = 0; i < q.w; ++i) {
          spk_t.push_back(lt[q.z + i]);
          spk_gid.push_back(lg[q.z + i]);
        }
    }
  }

  // one persistent launch: up to kBatch epochs from `step` towards `target`
  // sharded operation (world > 1): the caller's exchange buffers
  int64_t* x_send = nullptr;
  int64_t* x_recv = nullptr;
  int64_t x_cap = 0;
  int32_t x_world = 0;

  int64_t shard_spike_cap() const { return int64_t(std::max(n_local(), 1)) * sp_cap; }

  // ---- the exchange inside the library (mcg_shard_init_nccl) --------------
  void* nccl_comm = nullptr;
  DBuf<int64_t> d_xs, d_xr;          // this rank's send block, all ranks' blocks
  DBuf<int64_t> d_ctl_ring;          // epoch control of each launch of a batch
  int64_t* h_ctl_ring = nullptr;
  DBuf<int64_t> d_glog;              // gathered spikes of a batch: (s0, gid, step, t bits)
  DBuf<unsigned long long> d_glog_n;
  std::vector<double> gspk_t;        // the global spike list (every rank's spikes)
  std::vector<uint32_t> gspk_gid;
  bool async_ok = false;             // inboxes sized so that no expansion can overflow

  // connection resolution on the device (mcg_resolve.cuh) after the host's
  // pass 0 (build_model(..., defer_edges)): d_e_*, d_src_edges and the
  // appended instances' weights in d_i_weight; the host keeps src_edges and
  // max_delay_steps, and gets the edge records only when it needs them
  // (ensure_host_edges: checkpoints)
  void resolve_edges(const mcg_recipe& r) {
    using namespace mcg_rs;
    const int64_t nconn = r.n_connections, ne = m.n_edges;
    const int64_t n_cg = static_cast<int64_t>(m.cgs.size());
    if (nconn >= (int64_t(1) << 32) || n_cg >= (int64_t(1) << 31))
      throw Error(MCG_ERR_ENGINE, "resolve: connection list too long for 32-bit keys");
    const uint32_t g0 = m.gid_begin, g1 = m.gid_end;
    // the connection list, as the recipe holds it
    DBuf<uint8_t> from_src, policy;
    DBuf<uint32_t> src, dst;
    DBuf<int32_t> group;
    DBuf<double> weight, delay;
    auto up = [&](auto& d, const auto* h) {
      d.alloc(size_t(std::max<int64_t>(nconn, 1)));
      CK(cudaMemcpyAsync(d.p, h, size_t(nconn) * sizeof(*h), cudaMemcpyHostToDevice, st));
    };
    up(from_src, r.conn_from_source);
    up(policy, r.conn_policy);
    up(src, r.conn_src);
    up(dst, r.conn_dst);
    up(group, r.conn_group);
    up(weight, r.conn_weight);
    up(delay, r.conn_delay_ms);
    const Conn C{from_src.p, src.p, dst.p, group.p, policy.p, weight.p, delay.p, nconn};
    DBuf<int64_t> cg_conn_off, cg_off_l;
    DBuf<int32_t> cg_count, cg_comp;
    DBuf<uint8_t> cg_static;
    DBuf<double> cg_cf;
    DBuf<McgCellGroup> cgs;
    cg_conn_off.upload(m.cg_conn_off, st);
    cg_off_l.upload(m.cg_off, st);
    cg_count.upload(m.cg_count, st);
    cg_comp.upload(m.cg_comp, st);
    cg_static.upload(m.cg_static, st);
    cg_cf.upload(m.cg_cf, st);
    cgs.upload(m.cgs, st);
    // keys, then the two stable orders
    const size_t nc = size_t(nconn);
    DBuf<uint32_t> key_cg, key_src, val, key_s, perm1, perm2, inst_of;
    key_cg.alloc(nc);
    key_src.alloc(nc);
    val.alloc(nc);
    key_s.alloc(nc);
    perm1.alloc(nc);
    perm2.alloc(nc);
    inst_of.alloc(nc);
    k_keys<<<blocks(nconn), 256, 0, st>>>(C, g0, g1, cg_off_l.p, uint32_t(n_cg), uint32_t(r.n_cells), key_cg.p,
                                         key_src.p, val.p);
    CK(cudaGetLastError());
    DBuf<uint8_t> tmp;
    auto sort = [&](const uint32_t* k_in, uint32_t* k_out, const uint32_t* v_in, uint32_t* v_out, int64_t n,
                    uint64_t max_key) {
      size_t tb = 0;
      const int bits = bits_for(max_key);
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, v_in, v_out, n, 0, bits, st));
      if (tb > tmp.n) tmp.alloc(tb);
      CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k_in, k_out, v_in, v_out, n, 0, bits, st));
    };
    sort(key_cg.p, key_s.p, val.p, perm1.p, nconn, uint64_t(n_cg));
    {
      DBuf<int32_t> flag, scan;
      flag.alloc(nc);
      scan.alloc(nc);
      k_rr_flags<<<blocks(nconn), 256, 0, st>>>(C, perm1.p, ne, flag.p);
      size_t tb = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.p, scan.p, nconn, st));
      if (tb > tmp.n) tmp.alloc(tb);
      CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.p, scan.p, nconn, st));
      k_instances<<<blocks(ne), 256, 0, st>>>(C, key_s.p, perm1.p, ne, scan.p, cg_conn_off.p, cg_count.p,
                                              cgs.p, inst_of.p, d_i_weight.p);
      CK(cudaGetLastError());
    }
    sort(key_src.p, key_s.p, val.p, perm2.p, nconn, uint64_t(r.n_cells) + 1);
    // the edge records, in rank order
    const size_t nes = size_t(std::max<int64_t>(ne, 1));
    d_e_dst.alloc(nes);
    d_e_group.alloc(nes);
    d_e_inst.alloc(nes);
    d_e_weight.alloc(nes);
    d_e_src.alloc(nes);
    d_e_comp.alloc(nes);
    d_e_wcf.alloc(nes);
    d_e_delay.alloc(nes);
    const int64_t n_se = static_cast<int64_t>(m.src_edges.size()), src0 = ne - n_se;
    DBuf<uint32_t> skey, sval, skey_s, sval_s;
    DBuf<unsigned long long> maxd;
    skey.alloc(size_t(std::max<int64_t>(n_se, 1)));
    sval.alloc(size_t(std::max<int64_t>(n_se, 1)));
    maxd.alloc(1);
    maxd.zero(st);
    const Edges E{d_e_dst.p, d_e_group.p, d_e_comp.p, d_e_inst.p, d_e_src.p, nullptr, d_e_weight.p, d_e_wcf.p,
                  d_e_delay.p};
    d_e_seq.alloc(nes);
    Edges E2 = E;
    E2.seq = d_e_seq.p;
    k_edges<<<blocks(ne), 256, 0, st>>>(C, perm2.p, ne, g0, m.dt, cg_off_l.p, cg_static.p, cg_comp.p, cg_cf.p,
                                        inst_of.p, E2, maxd.p, skey.p, sval.p, src0);
    CK(cudaGetLastError());
    // per-source CSR of the source bucket: each source's edges in rank order
    d_src_edges.alloc(size_t(std::max<int64_t>(n_se, 1)));
    if (n_se > 0) {
      skey_s.alloc(size_t(n_se));
      sval_s.alloc(size_t(n_se));
      sort(skey.p, skey_s.p, sval.p, sval_s.p, n_se, uint64_t(std::max(r.n_sources, 1)));
      k_u32_to_i64<<<blocks(n_se), 256, 0, st>>>(sval_s.p, n_se, d_src_edges.p);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(m.src_edges.data(), d_src_edges.p, size_t(n_se) * sizeof(int64_t),
                         cudaMemcpyDeviceToHost, st));
    }
    unsigned long long md = 0;
    CK(cudaMemcpyAsync(&md, maxd.p, sizeof(md), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    m.max_delay_steps = static_cast<int64_t>(md);
    host_edges = false;
  }

  // the layout digest of mcg_build_digest from this engine's own layout (the
  // device-resolved edges and instance weights when the build deferred them)
  void layout_digest(uint64_t out[4]) {
    ensure_host_edges();
    HostModel c = m;
    const auto w = download(d_i_weight, size_t(m.n_inst));
    c.i_weight.assign(w.begin(), w.end());
    ::layout_digest(c, out);
  }

  // the edge records and appended weights on the host (after resolve_edges)
  void ensure_host_edges() {
    if (host_edges) return;
    const size_t ne = size_t(m.n_edges);
    auto get = [&](auto& h, const auto& d) {
      h.resize(ne);
      if (ne) CK(cudaMemcpyAsync(h.data(), d.p, ne * sizeof(h[0]), cudaMemcpyDeviceToHost, st));
    };
    get(m.e_dst, d_e_dst);
    get(m.e_group, d_e_group);
    get(m.e_inst, d_e_inst);
    get(m.e_weight, d_e_weight);
    get(m.e_src, d_e_src);
    get(m.e_seq, d_e_seq);
    get(m.e_comp, d_e_comp);
    get(m.e_wcf, d_e_wcf);
    get(m.e_delay, d_e_delay);
    CK(cudaStreamSynchronize(st));
    host_edges = true;
  }

  // inbox capacities that no epoch can exceed: per destination, every in-edge
  // delivers at most sp_cap (cell edges) or, from a source, one event per step
  // (Poisson) or per scheduled time (regular / scripted, which may share a
  // step) events per epoch, and an event waits at most ceil(delay / L) + 1
  // epochs in the pending list; false (and nothing changed) above the budget
  bool size_inboxes_for_worst_case(size_t budget_bytes) {
    const int nl = n_local();
    std::vector<int64_t> inc(std::max(nl, 1), 0), pend(std::max(nl, 1), 0);
    if (!host_edges) {  // the same counts on the device
      using namespace mcg_rs;
      DBuf<unsigned long long> di, dp;
      di.alloc(inc.size());
      dp.alloc(pend.size());
      di.zero(st);
      dp.zero(st);
      k_worst_cell<<<blocks(std::max<int64_t>(m.n_edges, 1)), 256, 0, st>>>(d_e_dst.p, d_e_src.p, d_e_delay.p,
                                                                            m.n_edges, sp_cap, L, di.p, dp.p);
      std::vector<int64_t> per_k(m.src_edges.size());
      for (size_t q = 0; q < m.sources.size(); ++q) {
        const Source& S = m.sources[q];
        const int64_t per = S.type == MCG_SRC_POISSON ? L
                            : S.type == MCG_SRC_REGULAR ? std::max<int64_t>(S.r_count, 0)
                                                        : static_cast<int64_t>(S.steps.size());
        for (int64_t k = m.src_edge_off[q]; k < m.src_edge_off[q + 1]; ++k) per_k[size_t(k)] = per;
      }
      DBuf<int64_t> dk;
      if (!per_k.empty()) {
        dk.upload(per_k, st);
        k_worst_src<<<blocks(int64_t(per_k.size())), 256, 0, st>>>(d_e_dst.p, d_e_delay.p, d_src_edges.p, dk.p,
                                                                   int64_t(per_k.size()), L, di.p, dp.p);
      }
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(inc.data(), di.p, inc.size() * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(pend.data(), dp.p, pend.size() * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    auto add = [&](size_t r, int64_t per) {
      const int c = m.e_dst[r];
      if (c < 0) return;
      const int64_t d = m.e_delay[r];
      inc[c] += per;
      pend[c] += per * ((d + L - 1) / L + 1);
    };
    for (size_t r = 0; r < m.e_dst.size(); ++r)
      if (m.e_src[r] != 0xFFFFFFFFu) add(r, sp_cap);
    for (size_t q = 0; host_edges && q < m.sources.size(); ++q) {
      const Source& S = m.sources[q];
      const int64_t per = S.type == MCG_SRC_POISSON ? L
                          : S.type == MCG_SRC_REGULAR ? std::max<int64_t>(S.r_count, 0)
                                                      : static_cast<int64_t>(S.steps.size());
      for (int64_t k = m.src_edge_off[q]; k < m.src_edge_off[q + 1]; ++k) add(size_t(m.src_edges[k]), per);
    }
    const int64_t mi = *std::max_element(inc.begin(), inc.end());
    const int64_t mp = *std::max_element(pend.begin(), pend.end());
    int64_t ic = 32, pc = 64;
    while (ic < mi + 1) ic <<= 1;
    while (pc < mp + 1) pc <<= 1;
    if (ic > (int64_t(1) << 24) || pc > (int64_t(1) << 24)) return false;
    const size_t bytes = size_t(std::max(nl, 1)) * size_t(ic + 2 * pc) * 8;
    if (bytes > budget_bytes) return false;
    if (ic > inc_cap || pc > pend_cap) {
      // move the pending keys into the larger buffers (as grow_inboxes)
      while (pend_cap < pc || inc_cap < ic) {
        if (inc_cap < ic && pend_cap < pc) grow_inboxes();
        else if (inc_cap < ic) {
          inc_cap *= 2;
          d_inc.alloc(static_cast<size_t>(std::max(nl, 1)) * inc_cap);
          d_inc_n.zero(st);
        } else {
          const int32_t keep = inc_cap;
          grow_inboxes();
          inc_cap = keep;
          d_inc.alloc(static_cast<size_t>(std::max(nl, 1)) * inc_cap);
          d_inc_n.zero(st);
        }
      }
    }
    return true;
  }

  void init_nccl(const uint8_t* id) {
    if (m.world < 1) throw Error(MCG_ERR_ARGUMENT, "nccl: world < 1");
    NcclApi& api = nccl_api();
    CK(cudaSetDevice(device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    api.check(api.comm_init_rank(&comm, m.world, uid, m.rank), "ncclCommInitRank");
    nccl_comm = comm;
    // a common block capacity: every rank's spikes per epoch are at most its
    // cell count times sp_cap, sp_cap depends only on the kinds and L, and the
    // partition (hence the largest shard) is the same on every rank
    const int64_t cap = int64_t(std::max(m.max_shard_cells, 1)) * sp_cap;
    const int64_t block = 1 + 3 * cap;
    d_xs.alloc(size_t(block));
    d_xs.zero(st);
    d_xr.alloc(size_t(block) * m.world);
    d_xr.zero(st);
    x_send = d_xs.p;
    x_recv = d_xr.p;
    x_cap = cap;
    x_world = m.world;
    d_ctl_ring.alloc(4 * kBatch);
    if (!h_ctl_ring) CK(cudaMallocHost(&h_ctl_ring, 4 * kBatch * sizeof(int64_t)));
    d_glog.alloc(size_t(4) * kBatch * size_t(std::max(m.n_cells_global, 1)) * sp_cap);
    d_glog_n.alloc(1);
    d_glog_n.zero(st);
    async_ok = size_inboxes_for_worst_case(size_t(16) << 30) && !std::getenv("MCG_SHARD_SYNC");
    refresh_dev();
    CK(cudaStreamSynchronize(st));
  }

  // the gathered spikes of the batch, epoch by epoch in (gid, step) order
  void drain_glog() {
    unsigned long long n = 0;
    CK(cudaMemcpyAsync(&n, d_glog_n.p, sizeof(n), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (n == 0) return;
    std::vector<int64_t> g(4 * n);
    CK(cudaMemcpyAsync(g.data(), d_glog.p, g.size() * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemsetAsync(d_glog_n.p, 0, sizeof(unsigned long long), st));
    CK(cudaStreamSynchronize(st));
    std::vector<int64_t> idx(n);
    for (size_t i = 0; i < n; ++i) idx[i] = int64_t(i);
    std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
      for (int k = 0; k < 3; ++k)
        if (g[4 * a + k] != g[4 * b + k]) return g[4 * a + k] < g[4 * b + k];
      return false;
    });
    for (int64_t i : idx) {
      double t;
      std::memcpy(&t, &g[4 * i + 3], 8);
      gspk_t.push_back(t);
      gspk_gid.push_back(static_cast<uint32_t>(g[4 * i + 1]));
    }
  }

  // sharded advance with the exchange on the engine's stream: per epoch one
  // stepping launch, ncclAllGather of the spike blocks, the gathered spikes
  // appended to the global log; the host waits once per batch of kBatch
  // epochs (or per epoch when the inboxes could overflow)
  void shard_advance(double t_ms) {
    if (!nccl_comm) throw Error(MCG_ERR_ENGINE, "sharded engine: mcg_shard_init_nccl first");
    invalidate_mirror();
    const int64_t target = ceil_steps(t_ms, m.dt);
    if (step >= target) return;
    const int64_t a = step;
    probes_begin(a, target, false, 0);
    lazy_init();
    refresh_dev();
    NcclApi& api = nccl_api();
    const int64_t block = 1 + 3 * x_cap;
    CK(cudaEventRecord(eva, st));
    while (step < target) {
      const int64_t n_ep = async_ok ? std::min<int64_t>(kBatch, (target - step + L - 1) / L) : 1;
      int64_t s = step;
      for (int64_t e = 0; e < n_ep; ++e) {
        int64_t* hc = h_ctl_ring + 4 * e;
        hc[0] = s;
        hc[1] = target;
        hc[2] = L;
        hc[3] = a;
        s = std::min<int64_t>(s + L, target);
      }
      CK(cudaMemcpyAsync(d_ctl_ring.p, h_ctl_ring, 4 * n_ep * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      for (int64_t e = 0; e < n_ep; ++e) {
        launch_epoch_kernel(1, d_ctl_ring.p + 4 * e, static_cast<int32_t>(e));
        api.check(api.all_gather(x_send, x_recv, size_t(block), ncclInt64,
                                 static_cast<ncclComm_t>(nccl_comm), st), "ncclAllGather");
        k_collect_recv<<<1, 256, 0, st>>>(x_recv, x_world, block, d_ctl_ring.p + 4 * e, d_glog.p,
                                          d_glog_n.p, int64_t(d_glog.n / 4), d_err.p);
        stats.kernel_launches += 2;
      }
      sync_counters_raw();
      if (*h_abort) throw Error(MCG_ERR_ENGINE, "sharded engine: inbox overflow");
      stats.epochs += n_ep;
      stats.epoch_kernel_launches += n_ep;
      stats.steps += s - step;
      drain_chunks();
      drain_glog();
      step = s;
      check_err();
    }
    CK(cudaEventRecord(evb, st));
    CK(cudaEventSynchronize(evb));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, eva, evb));
    stats.advance_ms += ms;
    stats.advance_calls += 1;
    probes_end(a, target, false, 0, 1);
  }

  // one launch of the stepping kernel (k_warp or k_batch) over `planned`
  // epochs described by the device control block `ctl`
  void launch_epoch_kernel(int64_t planned, const int64_t* ctl, int32_t epoch_base = 0) {
    const bool sharded = x_send != nullptr;
    refresh_dev();
    McgBatchArgs A{};
    A.E = ev_dev();
    if (sharded) {
      CK(cudaMemsetAsync(x_send, 0, sizeof(int64_t), st));
      A.E.x_recv = x_recv;
      A.E.x_world = x_world;
      A.E.x_block = 1 + 3 * x_cap;
      A.x_send = x_send;
      A.x_cap = x_cap;
    }
    A.n_epochs = static_cast<int32_t>(planned);
    A.E.ctl = ctl;
    McgDev Dv = dev;
    Dv.ctl = ctl;
    int64_t max_len = L;
    if (use_point) {
      McgPointArgs P{};
      P.E = A.E;
      P.n_epochs = A.n_epochs;
      P.epoch_base = epoch_base;
      P.log_t = d_log_t.p;
      P.log_gid = d_log_gid.p;
      P.log_n = d_ctr.p + C_LOG;
      P.chunks = d_chunks.p;
      P.chunk_n = d_chunk_n.p;
      void* pargs[] = {&Dv, &P, &max_len};
      CK(cudaEventRecord(evk0, st));
      void* fn = pt_small ? reinterpret_cast<void*>(k_point<1, 2>)
                          : reinterpret_cast<void*>(k_point<MCG_PT_STC, MCG_PT_SP>);
      CK(cudaLaunchCooperativeKernel(fn, pt_grid, MCG_PT_THREADS, pargs, 0, st));
    } else if (use_warp) {
      McgWarpArgs W{};
      W.E = A.E;
      W.n_epochs = A.n_epochs;
      W.G = wg_G;
      W.n_groups = wg_groups;
      W.resident = wg_resident;
      W.m = smem_n;
      W.S = sp_max;
      W.P = wg_P;
      W.MW = wg_MW;
      W.cell_doubles = (2 + sp_max) * smem_n;
      W.ev_cap = wg_ev_cap;
      W.warp_doubles = wg_warp_doubles;
      W.kind_doubles = wg_kind_doubles;
      W.n_kinds = static_cast<int32_t>(m.kinds.size());
      W.n_specs_sm = wg_specs_sm;
      W.lazy = wg_lazy;
      W.cu_every = static_cast<int32_t>(std::max<int64_t>(1, 48 / std::max<int64_t>(L, 1)));
      if (phase_timing) {
        if (!d_phase.p) {
          d_phase.alloc(size_t(2 + std::max(bc_grid, wg_grid)) * MCG_NPHASE);
          d_phase.zero(st);
        }
        W.phase = d_phase.p;
      }
      W.dbg = std::getenv("MCG_WARP_DBG") ? std::atoi(std::getenv("MCG_WARP_DBG")) : 0;
      W.dbg_s = std::getenv("MCG_WARP_DBG_S") ? std::atoll(std::getenv("MCG_WARP_DBG_S")) : 30;
      W.kb_off = d_kb_off.p;
      W.stc_mask = d_stc_mask.p;
      W.stc_t = d_stc_t.p;
      W.log_t = d_log_t.p;
      W.log_gid = d_log_gid.p;
      W.log_n = d_ctr.p + C_LOG;
      W.chunks = d_chunks.p;
      W.chunk_n = d_chunk_n.p;
      W.x_send = A.x_send;
      W.x_cap = A.x_cap;
      W.epoch_base = epoch_base;
      W.no_abort = wg_no_abort;
      void* wargs[] = {&Dv, &W, &max_len};
      CK(cudaEventRecord(evk0, st));
      CK(cudaFuncSetAttribute(k_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(wg_smem)));
      CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_warp), wg_grid, wg_warps * 32, wargs,
                                     wg_smem, st));
      if (wg_lazy) lazy_dirty = true;
    } else {
    A.cells_per_cta = bc_cells;
    A.n_batches = bc_batches;
    A.comp_stride = bc_stride;
    A.stc_max = bc_stc_max;
    A.n_stc_max = bc_nstc_max;
    A.kind_doubles = bc_kind_doubles;
    A.n_specs_sm = bc_specs_sm;
    A.stc_sm = bc_stc_sm;
    A.ch_stride = bc_ch_stride;
    A.ch_pmax = bc_ch_pmax;
    A.ev_cap = bc_ev_cap;
    A.nch_max = bc_nch_max;
    A.lean = bc_lean;
    A.act_max = bc_act_max;
    A.fmask_words = bc_fmask_words;
    if (phase_timing) {
      if (!d_phase.p) {
        d_phase.alloc(size_t(2 + bc_grid) * MCG_NPHASE);
        d_phase.zero(st);
      }
      A.phase = d_phase.p;
    }
    A.log_t = d_log_t.p;
    A.log_gid = d_log_gid.p;
    A.log_n = d_ctr.p + C_LOG;
    A.chunks = d_chunks.p;
    A.chunk_n = d_chunk_n.p;
    A.epoch_base = epoch_base;
    A.dbg = std::getenv("MCG_WARP_DBG") ? std::atoi(std::getenv("MCG_WARP_DBG")) : 0;
    A.dbg_s = std::getenv("MCG_WARP_DBG_S") ? std::atoll(std::getenv("MCG_WARP_DBG_S")) : 30;
    void* args[] = {&Dv, &A, &max_len};
    CK(cudaEventRecord(evk0, st));
    // the kernel attributes are process-global and another engine in this
    // process (a shard, a second network) may have set its own: restate ours
    CK(cudaFuncSetAttribute(k_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(bc_smem)));
    CK(cudaFuncSetAttribute(k_batch, cudaFuncAttributePreferredSharedMemoryCarveout, bc_carve));
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_batch), bc_grid, kBatchThreads, args,
                                   bc_smem, st));
    }
  }

  void run_batch(int64_t target, int64_t call_first) {
    h_ctl[0] = step;
    h_ctl[1] = target;
    h_ctl[2] = L;
    h_ctl[3] = call_first;
    CK(cudaMemcpyAsync(d_ctl.p, h_ctl, 4 * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    const bool sharded = x_send != nullptr;
    // sharded: one epoch per launch, the exchange happens between launches
    const int64_t planned = sharded ? 1 : std::min<int64_t>(kBatch, (target - step + L - 1) / L);
    launch_epoch_kernel(planned, d_ctl.p);
    CK(cudaEventRecord(evk1, st));
    sync_counters_raw();
    const int32_t ab = *h_abort;
    const int64_t done = ab ? ab - 1 : planned;
    {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, evk0, evk1));
      stats.epoch_kernel_ms += ms;
    }
    stats.epochs += done;
    stats.epoch_kernel_launches += 1;
    stats.kernel_launches += 1;
    stats.steps += std::min<int64_t>(step + done * L, target) - step;
    drain_chunks();
    step = std::min<int64_t>(step + done * L, target);
    check_err();
    if (ab) {
      // an inbox overflowed while expanding epoch `done`: grow and resume there
      *h_abort = 0;
      d_abort.zero(st);
      grow_inboxes();
      refresh_dev();
    }
  }

  // probe sample slots for steps [a, b) (or n_forced forced samples)
  void probes_begin(int64_t a, int64_t b, bool forced, int64_t n_forced) {
    std::vector<int64_t> base(m.probes.size(), 0);
    int64_t tot = 0;
    for (size_t p = 0; p < m.probes.size(); ++p) {
      const McgProbe& P = m.probes[p];
      base[p] = tot;
      if (P.local < 0) continue;
      int64_t cnt;
      if (forced) {
        cnt = n_forced;
      } else {
        const int64_t m0 = (a + P.every) / P.every, m1 = b / P.every;
        cnt = m1 >= m0 ? m1 - m0 + 1 : 0;
      }
      tot += cnt;
    }
    if (static_cast<size_t>(tot) > d_trace.n) d_trace.alloc(static_cast<size_t>(tot) * 2);
    if (!m.probes.empty())
      CK(cudaMemcpyAsync(d_trace_base.p, base.data(), base.size() * sizeof(int64_t),
                         cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    probe_base_host = base;
    probe_total = tot;
    dev.trace_buf = d_trace.p;
  }

  void probes_end(int64_t a, int64_t b, bool forced, int64_t n_forced, int64_t per) {
    if (probe_total == 0) return;
    std::vector<double> buf(probe_total);
    CK(cudaMemcpyAsync(buf.data(), d_trace.p, probe_total * sizeof(double), cudaMemcpyDeviceToHost,
                       st));
    CK(cudaStreamSynchronize(st));
    for (size_t p = 0; p < m.probes.size(); ++p) {
      const McgProbe& P = m.probes[p];
      if (P.local < 0) continue;
      const int64_t o = probe_base_host[p];
      if (forced) {
        for (int64_t q = 0; q < n_forced; ++q) {
          const int64_t s = a + (q + 1) * per - 1;  // sample_probes(cell, step_-1, true)
          traces[p].emplace_back((double(s) + 1.0) * m.dt, buf[o + q]);
        }
      } else {
        const int64_t m0 = (a + P.every) / P.every, m1 = b / P.every;
        for (int64_t mm = m0; mm <= m1; ++mm) {
          const int64_t s = mm * P.every - 1;
          traces[p].emplace_back((double(s) + 1.0) * m.dt, buf[o + (mm - m0)]);
        }
      }
    }
  }

  // one min-delay epoch towards t_ms (sharded epoch loop, engine.cpp:913-942):
  // expands the imported spikes, steps the epoch, exports this rank's spikes
  void run_epoch(double t_ms) {
    invalidate_mirror();
    if (x_send == nullptr) throw Error(MCG_ERR_ENGINE, "sharded engine: exchange buffers not set");
    const int64_t target = ceil_steps(t_ms, m.dt);
    if (step >= target) return;
    const int64_t a = step, b = std::min<int64_t>(target, step + L);
    probes_begin(a, b, false, 0);
    lazy_init();
    refresh_dev();
    CK(cudaEventRecord(eva, st));
    while (step < b) run_batch(b, a);
    CK(cudaEventRecord(evb, st));
    CK(cudaEventSynchronize(evb));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, eva, evb));
    stats.advance_ms += ms;
    stats.advance_calls += 1;
    probes_end(a, b, false, 0, 1);
  }

  void advance_to(double t_ms) {
    invalidate_mirror();
    if (m.world > 1)
      throw Error(MCG_ERR_ENGINE, "sharded engine: drive it with mcg_shard_run_epoch + an exchange");
    const int64_t target = ceil_steps(t_ms, m.dt);
    if (step >= target) return;
    const int64_t a = step;
    probes_begin(a, target, false, 0);
    lazy_init();
    refresh_dev();
    CK(cudaEventRecord(eva, st));
    while (step < target) run_batch(target, a);
    CK(cudaEventRecord(evb, st));
    CK(cudaEventSynchronize(evb));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, eva, evb));
    stats.advance_ms += ms;
    stats.advance_calls += 1;
    print_phases(target - a);
    probes_end(a, target, false, 0, 1);
  }

  void fast_forward_to(double t_ms, double coarse_dt_ms) {
    invalidate_mirror();
    // a shard cannot decide the reference's pending-spike guard alone: the
    // other ranks' spikes of the last epoch (x_recv) are not expanded yet, and
    // the guard's reset-before-throw order runs over the global gid range
    if (m.world > 1)
      throw Error(MCG_ERR_ENGINE, "fast-forward: not supported for a sharded engine");
    const double dt = m.dt;
    const int64_t per = static_cast<int64_t>(std::llround(coarse_dt_ms / dt));
    if (per < 1 || std::fabs(double(per) * dt - coarse_dt_ms) > 1e-9 * coarse_dt_ms)
      throw Error(MCG_ERR_ENGINE, "fast-forward: coarse dt must be a multiple of dt");
    const int64_t target = ceil_steps(t_ms, dt);
    if ((target - step) % per != 0)
      throw Error(MCG_ERR_ENGINE, "fast-forward: span must be a multiple of coarse dt");
    ensure_flushed();
    lazy_valid = false;
    const int nl = n_local();
    const int nf = static_cast<int>(m.fifos.size());
    refresh_dev();
    (void)nf;
    DBuf<int32_t> flag;
    flag.alloc(std::max(nl, 1));
    flag.zero(st);
    if (nl > 0)
      k_pending<<<static_cast<unsigned>((nl + 255) / 256), 256, 0, st>>>(
          dev, d_out_begin.p, d_out_end.p, d_e_dst.p, flag.p);
    std::vector<int32_t> hflag(std::max(nl, 1), 0);
    CK(cudaMemcpyAsync(hflag.data(), flag.p, hflag.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int first = nl;
    for (int c = 0; c < nl; ++c)
      if (hflag[c]) {
        first = c;
        break;
      }
    // the reference resets each cell's calcium, STDP traces and kernels as it
    // walks the cells and throws at the first one with undelivered events:
    // the cells before it are reset (engine.cpp:958-969)
    const int64_t ncg = first < nl ? m.cg_off[first] : static_cast<int64_t>(m.cgs.size());
    if (ncg > 0) {
      k_ff_reset<<<static_cast<unsigned>((ncg + 127) / 128), 128, 0, st>>>(dev, ncg);
      stats.kernel_launches += 1;
    }
    if (first < nl) {
      CK(cudaStreamSynchronize(st));
      throw Error(MCG_ERR_ENGINE, "fast-forward: pending undelivered spikes");
    }
    const int64_t n_coarse = (target - step) / per;
    if (n_coarse <= 0) return;
    const double dtc = coarse_dt_ms;
    std::vector<double> fh(m.specs.size(), 0.0);
    for (size_t i = 0; i < m.specs.size(); ++i) fh[i] = std::exp(-0.1 * dtc / m.specs[i].tau_h);
    // species systems at the coarse step: cap = vol/dtc (engine.cpp:1019-1025),
    // eliminated once with solve_tree's operation order
    std::vector<double> cap_ff(m.k_sp_cap_dt.size()), f_ff(cap_ff.size()), d_ff(cap_ff.size()),
        r_ff(cap_ff.size(), 0.0);
    std::vector<McgKind> kinds_ff = m.kinds;
    for (size_t k = 0; k < m.kinds.size(); ++k) {
      McgKind& K = kinds_ff[k];
      for (int s = 0; s < K.n_species; ++s) {
        const int64_t o = K.sp_arr + int64_t(s) * K.n;
        for (int i = 0; i < K.n; ++i) cap_ff[o + i] = m.grids[k].volume[i] / dtc;
        if (K.n > 1 && !eliminate_constant(K.n, m.grids[k].parent.data(), cap_ff.data() + o,
                                           m.k_sp_gs.data() + o, m.k_sp_coupling.data() + o,
                                           f_ff.data() + o, d_ff.data() + o))
          K.sp_const = 0;
        for (int i = 0; i < K.n; ++i) r_ff[o + i] = mcg_recip(d_ff[o + i]);
      }
    }
    DBuf<double> d_fh, d_cap_ff, d_f_ff, d_d_ff, d_r_ff;
    DBuf<McgKind> d_kinds_ff;
    d_fh.upload(fh, st);
    d_cap_ff.upload(cap_ff, st);
    d_f_ff.upload(f_ff, st);
    d_d_ff.upload(d_ff, st);
    d_r_ff.upload(r_ff, st);
    d_kinds_ff.upload(kinds_ff, st);
    probes_begin(step, target, true, n_coarse);
    refresh_dev();
    if (nl > 0) {
      McgDev dff = dev;
      dff.kinds = d_kinds_ff.p;
      // register-resident cells, then the rest (mcg_ff_fast_of splits them)
      const size_t ff_smem = (smem_bytes / (kBlock / 32) + sizeof(double) * MCG_FF_SCR) *
                             (MCG_FF_BLOCK / 32);
      CK(cudaFuncSetAttribute(k_ff_fast, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(ff_smem)));
      k_ff_fast<<<(nl * 32 + MCG_FF_BLOCK - 1) / MCG_FF_BLOCK, MCG_FF_BLOCK, ff_smem, st>>>(
          dff, d_fh.p, d_cap_ff.p, d_f_ff.p, d_d_ff.p, d_r_ff.p, dtc, n_coarse);
      CK(cudaFuncSetAttribute(k_ff, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem_bytes)));
      k_ff<<<(nl * 32 + kBlock - 1) / kBlock, kBlock, smem_bytes, st>>>(
          dff, d_fh.p, d_cap_ff.p, d_f_ff.p, d_d_ff.p, d_r_ff.p, dtc, n_coarse);
      stats.kernel_launches += 1;
      stats.kernel_launches += 1;
    }
    const int64_t a = step;
    step = target;
    sync_counters_raw();
    check_err();
    probes_end(a, target, true, n_coarse, per);
  }

  void sync_spikes() {}  // the host mirror is filled after every batch

  void clear_spikes() {
    spk_t.clear();
    spk_gid.clear();
  }

  int local_of(uint32_t gid) const {
    if (gid < m.gid_begin || gid >= m.gid_end)
      throw Error(MCG_ERR_ARGUMENT, "gid not on this shard");
    return static_cast<int>(gid - m.gid_begin);
  }

  // host mirror of the state arrays cell(gid) reads: the first
  // read of a field after the device state changed downloads the whole array
  // once; later reads (the other cells) are host copies.  Writes go through
  // to the device and keep a valid mirror current.
  std::vector<std::vector<unsigned char>> mirror = std::vector<std::vector<unsigned char>>(32);
  std::vector<char> mirror_ok = std::vector<char>(32, 0);
  void invalidate_mirror() { std::fill(mirror_ok.begin(), mirror_ok.end(), 0); }

  template <class T>
  void mirrored_field(int field, void* out, const DBuf<T>& b, int64_t off, int64_t count,
                      bool write, const void* in) {
    if (count <= 0) return;
    if (field < 0 || field >= 32) return copy_field(out, b.p, off, count, write, in);
    std::vector<unsigned char>& h = mirror[field];
    if (write) {
      copy_field(out, b.p, off, count, true, in);
      if (mirror_ok[field]) std::memcpy(h.data() + off * sizeof(T), in, count * sizeof(T));
      return;
    }
    if (!mirror_ok[field]) {
      h.resize(b.n * sizeof(T));
      if (b.n) {
        CK(cudaMemcpyAsync(h.data(), b.p, b.n * sizeof(T), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      }
      mirror_ok[field] = 1;
    }
    std::memcpy(out, h.data() + off * sizeof(T), count * sizeof(T));
  }

  template <class T>
  void copy_field(void* out, const T* base, int64_t off, int64_t count, bool write,
                  const void* in) {
    if (count <= 0) return;
    if (write)
      CK(cudaMemcpyAsync(const_cast<T*>(base) + off, in, count * sizeof(T), cudaMemcpyHostToDevice,
                         st));
    else
      CK(cudaMemcpyAsync(out, base + off, count * sizeof(T), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }

  void state_io(int field, uint32_t gid, int index, int64_t off, int64_t count, void* out,
                const void* in, bool write) {
    const int c = local_of(gid);
    ensure_flushed();
    if (write) lazy_valid = false;
    const McgKind& K = m.kinds[m.cell_kind[c]];
    const int64_t co = m.comp_off[c];
    auto comp_range = [&](int64_t lim) {
      if (off < 0 || count < 0 || off + count > lim) throw Error(MCG_ERR_ARGUMENT, "range out of bounds");
    };
    switch (field) {
      case MCG_FIELD_V: comp_range(K.n); return mirrored_field(field, out, d_v, co + off, count, write, in);
      case MCG_FIELD_HH_M: comp_range(K.n); return mirrored_field(field, out, d_hh_m, co + off, count, write, in);
      case MCG_FIELD_HH_H: comp_range(K.n); return mirrored_field(field, out, d_hh_h, co + off, count, write, in);
      case MCG_FIELD_HH_N: comp_range(K.n); return mirrored_field(field, out, d_hh_n, co + off, count, write, in);
      case MCG_FIELD_SPECIES:
        if (index < 0 || index >= K.n_species) throw Error(MCG_ERR_ARGUMENT, "species index");
        comp_range(K.n);
        return mirrored_field(field, out, d_species, m.sp_off[c] + int64_t(index) * K.n + off, count, write, in);
      case MCG_FIELD_DETECTOR_PREV_V: return mirrored_field(field, out, d_det_prev, c, 1, write, in);
      case MCG_FIELD_REFRACTORY_UNTIL: return mirrored_field(field, out, d_refr, c, 1, write, in);
      case MCG_FIELD_DETECTOR_ARMED: {
        int32_t a = 0;
        if (write) {
          a = static_cast<int32_t>(*static_cast<const int64_t*>(in));
          return copy_field<int32_t>(nullptr, d_armed.p, c, 1, true, &a);
        }
        copy_field(&a, d_armed.p, c, 1, false, nullptr);
        *static_cast<int64_t*>(out) = a;
        return;
      }
      case MCG_FIELD_INTERNAL_SEQ: {
        uint32_t a = 0;
        if (write) {
          a = static_cast<uint32_t>(*static_cast<const int64_t*>(in));
          return copy_field<uint32_t>(nullptr, d_iseq.p, c, 1, true, &a);
        }
        copy_field(&a, d_iseq.p, c, 1, false, nullptr);
        *static_cast<int64_t*>(out) = a;
        return;
      }
      default: break;
    }
    if (index < 0 || index >= K.n_groups) throw Error(MCG_ERR_ARGUMENT, "group index");
    const McgCellGroup& G = m.cgs[m.cg_off[c] + index];
    comp_range(G.size);
    const int64_t j = G.inst + off;
    switch (field) {
      case MCG_FIELD_SYN_COMP: return mirrored_field(field, out, d_i_comp, j, count, write, in);
      case MCG_FIELD_SYN_WEIGHT: return mirrored_field(field, out, d_i_weight, j, count, write, in);
      case MCG_FIELD_SYN_KERNEL: return mirrored_field(field, out, d_i_kernel, j, count, write, in);
      case MCG_FIELD_STDP_A_PRE: return mirrored_field(field, out, d_i_stdp_pre, j, count, write, in);
      case MCG_FIELD_STDP_A_POST: return mirrored_field(field, out, d_i_stdp_post, j, count, write, in);
      case MCG_FIELD_STDP_W: return mirrored_field(field, out, d_i_stdp_w, j, count, write, in);
      case MCG_FIELD_STDP_LAST: return mirrored_field(field, out, d_i_stdp_last, j, count, write, in);
      case MCG_FIELD_HOMEO_W: return mirrored_field(field, out, d_i_homeo_w, j, count, write, in);
      case MCG_FIELD_STC_H: return mirrored_field(field, out, d_i_stc_h, j, count, write, in);
      case MCG_FIELD_STC_Z: return mirrored_field(field, out, d_i_stc_z, j, count, write, in);
      case MCG_FIELD_STC_C: return mirrored_field(field, out, d_i_stc_c, j, count, write, in);
      case MCG_FIELD_STC_SPS_ABS: return mirrored_field(field, out, d_i_sps_abs, j, count, write, in);
      default: throw Error(MCG_ERR_ARGUMENT, "unknown field");
    }
  }

  // ---- checkpoints (engine.cpp:1036-1325) ----------------------------------
  template <class T>
  std::vector<T> download(const DBuf<T>& b, size_t n) {
    std::vector<T> h(n);
    if (n) CK(cudaMemcpyAsync(h.data(), b.p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    return h;
  }
  template <class T, class Al>
  void upload_to(DBuf<T>& b, const std::vector<T, Al>& h) {
    if (!h.empty()) CK(cudaMemcpyAsync(b.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  }

  // Engine::make_checkpoint (engine.cpp:1150-1233).  The pending inbox of a
  // cell is what the reference holds after its last exchange: the unconsumed
  // sorted events, then the events the last epoch's spikes pushed (Impl::
  // exchange, :875-889: cells in gid order, spikes in step order, out-edges in
  // seq order), which this engine expands only at the next epoch's start.
  std::vector<uint8_t> make_checkpoint() {
    if (m.world > 1) throw Error(MCG_ERR_ENGINE, "checkpoint: not supported for a sharded engine");
    ensure_flushed();
    ensure_host_edges();
    const int nl = n_local();
    const size_t nv = m.v.size(), nsp = m.species.size(), ni = m.i_comp.size();
    const auto v = download(d_v, nv), hm = download(d_hh_m, nv), hh = download(d_hh_h, nv),
               hn = download(d_hh_n, nv), sp = download(d_species, nsp),
               det = download(d_det_prev, size_t(nl));
    const auto armed = download(d_armed, size_t(nl));
    const auto refr = download(d_refr, size_t(nl));
    const auto iseq = download(d_iseq, size_t(nl));
    const auto ker = download(d_i_kernel, ni), wgt = download(d_i_weight, ni),
               spre = download(d_i_stdp_pre, ni), spost = download(d_i_stdp_post, ni),
               sw = download(d_i_stdp_w, ni), hw = download(d_i_homeo_w, ni),
               sh = download(d_i_stc_h, ni), sz = download(d_i_stc_z, ni), sc = download(d_i_stc_c, ni),
               sa = download(d_i_sps_abs, ni);
    const auto slast = download(d_i_stdp_last, ni);
    const auto pend = download(d_pend, size_t(std::max(nl, 1)) * 2 * pend_cap);
    const auto psel = download(d_pend_sel, size_t(nl)), poff = download(d_pend_off, size_t(nl)),
               pn = download(d_pend_n, size_t(nl));
    const auto fifos = download(d_fifos, m.fifos.size());
    const size_t nf = size_t(std::max<int64_t>(m.fifo_total, 1));
    const auto fstep = download(d_fifo_step, nf);
    const auto fsi = download(d_fifo_si, nf);
    const auto fsrc = download(d_fifo_src, nf);
    const auto fw = download(d_fifo_w, nf);
    const auto spc = download(d_sp_count, size_t(nl));
    const auto sps = download(d_sp_step, size_t(std::max(nl, 1)) * sp_cap);
    CK(cudaStreamSynchronize(st));

    // the last epoch's exchange, per destination
    std::vector<std::vector<CkEvent>> extra(nl);
    for (int c = 0; c < nl; ++c) {
      const uint32_t gid = m.gid_begin + uint32_t(c);
      for (int q = 0; q < spc[c] && q < sp_cap; ++q) {
        const int64_t st0 = sps[size_t(c) * sp_cap + q];
        for (int64_t r = m.out_begin[gid]; r < m.out_end[gid]; ++r)
          extra[m.e_dst[r]].push_back(CkEvent{st0 + 1 + m.e_delay[r], gid, m.e_seq[r],
                                              uint16_t(m.e_group[r]), 0, m.e_inst[r], m.e_weight[r]});
      }
    }
    const uint64_t mask = (1ull << rank_bits) - 1;
    Ckpt ck;
    ck.u64["meta/step"] = {static_cast<uint64_t>(step)};
    ck.f64["meta/dt_ms"] = {m.dt};
    for (int c = 0; c < nl; ++c) {
      const McgKind& K = m.kinds[m.cell_kind[c]];
      const int n = K.n;
      const int64_t co = m.comp_off[c];
      const std::string pre = "cell/" + std::to_string(m.gid_begin + uint32_t(c)) + "/";
      if (K.dyn != MCG_DYN_NONE) ck.f64[pre + "v"].assign(v.begin() + co, v.begin() + co + n);
      ck.f64[pre + "det"] = {det[c]};
      ck.u64[pre + "flags"] = {static_cast<uint64_t>(refr[c]), armed[c] ? 1ull : 0ull, uint64_t(iseq[c])};
      for (int q = 0; q < K.n_species; ++q) {
        const int64_t o = m.sp_off[c] + int64_t(q) * n;
        ck.f64[pre + "species/" + std::to_string(q)].assign(sp.begin() + o, sp.begin() + o + n);
      }
      if (K.dyn == MCG_DYN_HH) {
        ck.f64[pre + "hh_m"].assign(hm.begin() + co, hm.begin() + co + n);
        ck.f64[pre + "hh_h"].assign(hh.begin() + co, hh.begin() + co + n);
        ck.f64[pre + "hh_n"].assign(hn.begin() + co, hn.begin() + co + n);
      }
      std::vector<CkEvent> internal;
      for (int gi = 0; gi < K.n_groups; ++gi) {
        const McgCellGroup& G = m.cgs[m.cg_off[c] + gi];
        const McgSpec& S = m.specs[G.spec];
        const std::string gp = pre + "g" + std::to_string(gi) + "/";
        const int64_t a = G.inst, b = G.inst + G.size;
        ck.f64[gp + "kernel"].assign(ker.begin() + a, ker.begin() + b);
        ck.f64[gp + "weight"].assign(wgt.begin() + a, wgt.begin() + b);
        if (G.size > 0 && S.kind == MCG_SYN_STDP_COND) {
          ck.f64[gp + "stdp_a_pre"].assign(spre.begin() + a, spre.begin() + b);
          ck.f64[gp + "stdp_a_post"].assign(spost.begin() + a, spost.begin() + b);
          ck.f64[gp + "stdp_w"].assign(sw.begin() + a, sw.begin() + b);
          std::vector<uint64_t> ls(G.size);
          for (int i = 0; i < G.size; ++i) ls[i] = static_cast<uint64_t>(slast[a + i]);
          ck.u64[gp + "stdp_last"] = ls;
        }
        if (G.size > 0 && S.kind == MCG_SYN_HOMEO_CURRENT)
          ck.f64[gp + "homeo_w"].assign(hw.begin() + a, hw.begin() + b);
        if (G.size > 0 && S.kind == MCG_SYN_STC_CHARGE) {
          ck.f64[gp + "stc_h"].assign(sh.begin() + a, sh.begin() + b);
          ck.f64[gp + "stc_z"].assign(sz.begin() + a, sz.begin() + b);
          ck.f64[gp + "stc_c"].assign(sc.begin() + a, sc.begin() + b);
          ck.f64[gp + "stc_sps"].assign(sa.begin() + a, sa.begin() + b);
        }
        if (G.fifo >= 0) {  // delayed-calcium queue -> internal events
          const McgFifo& F = fifos[G.fifo];
          for (int64_t h = F.head; h < F.tail; ++h) {
            const int64_t slot = F.base + (h % F.cap);
            internal.push_back(CkEvent{fstep[slot], fsrc[slot], uint32_t(fsi[slot] >> 32), uint16_t(gi), 1,
                                       uint32_t(fsi[slot] & 0xffffffffu), fw[slot]});
          }
        }
      }
      std::vector<CkEvent> inbox;
      const uint64_t* pl = pend.data() + (size_t(c) * 2 + psel[c]) * pend_cap;
      for (int i = poff[c]; i < pn[c]; ++i) {
        const int64_t r = int64_t(pl[i] & mask);
        inbox.push_back(CkEvent{int64_t(pl[i] >> rank_bits), m.e_src[r], m.e_seq[r],
                                uint16_t(m.e_group[r]), 0, m.e_inst[r], m.e_weight[r]});
      }
      inbox.insert(inbox.end(), extra[c].begin(), extra[c].end());
      std::sort(internal.begin(), internal.end(), [](const CkEvent& x, const CkEvent& y) {
        if (x.step != y.step) return x.step < y.step;
        return x.seq < y.seq;
      });
      ck_pack(ck, pre + "inbox", inbox);
      ck_pack(ck, pre + "internal", internal);
    }
    return ck_serialize(ck);
  }

  // Checkpoint::deserialize + Engine::restore (engine.cpp:1095-1140, 1235-1325)
  void restore(const uint8_t* bytes, size_t size) {
    ensure_flushed();  // a rejected checkpoint leaves the current state whole
    ensure_host_edges();
    lazy_valid = false;
    invalidate_mirror();
    if (m.world > 1) throw Error(MCG_ERR_ENGINE, "checkpoint: not supported for a sharded engine");
    const Ckpt ck = ck_deserialize(bytes, size);
    auto getf = [&](const std::string& n) -> const std::vector<double>& {
      auto it = ck.f64.find(n);
      if (it == ck.f64.end()) throw Error(MCG_ERR_ENGINE, "checkpoint: missing " + n);
      return it->second;
    };
    auto getu = [&](const std::string& n) -> const std::vector<uint64_t>& {
      auto it = ck.u64.find(n);
      if (it == ck.u64.end()) throw Error(MCG_ERR_ENGINE, "checkpoint: missing " + n);
      return it->second;
    };
    auto sized = [](const std::vector<double>& a, size_t n) -> const std::vector<double>& {
      if (a.size() != n) throw Error(MCG_ERR_ENGINE, "checkpoint: state size mismatch");
      return a;
    };
    const auto& dtv = getf("meta/dt_ms");
    if (dtv.empty() || std::fabs(dtv[0] - m.dt) > 1e-15) throw Error(MCG_ERR_ENGINE, "checkpoint: dt mismatch");
    const auto& stv = getu("meta/step");
    if (stv.empty()) throw Error(MCG_ERR_ENGINE, "checkpoint: missing meta/step");
    const int nl = n_local();
    const size_t nv = m.v.size(), nsp = m.species.size(), ni = m.i_comp.size();
    auto v = download(d_v, nv), hm = download(d_hh_m, nv), hh = download(d_hh_h, nv),
         hn = download(d_hh_n, nv), sp = download(d_species, nsp), det = download(d_det_prev, size_t(nl));
    auto armed = download(d_armed, size_t(nl));
    auto refr = download(d_refr, size_t(nl));
    auto iseq = download(d_iseq, size_t(nl));
    auto ker = download(d_i_kernel, ni), wgt = download(d_i_weight, ni), spre = download(d_i_stdp_pre, ni),
         spost = download(d_i_stdp_post, ni), sw = download(d_i_stdp_w, ni), hw = download(d_i_homeo_w, ni),
         sh = download(d_i_stc_h, ni), sz = download(d_i_stc_z, ni), sc = download(d_i_stc_c, ni),
         sa = download(d_i_sps_abs, ni);
    auto slast = download(d_i_stdp_last, ni);
    auto act = download(d_i_active, std::max<size_t>(ni, 1));
    auto cgs = download(d_cgs, m.cgs.size());
    auto fifos = download(d_fifos, m.fifos.size());
    const size_t nf = size_t(std::max<int64_t>(m.fifo_total, 1));
    std::vector<int64_t> fstep(nf, 0);
    std::vector<uint64_t> fsi(nf, 0);
    std::vector<uint32_t> fsrc(nf, 0);
    std::vector<double> fw(nf, 0.0);
    CK(cudaStreamSynchronize(st));
    // (src, seq) -> edge rank: EventRec identity of a pending network event
    std::unordered_map<uint64_t, int64_t> rank_of;
    rank_of.reserve(m.e_src.size() * 2);
    for (size_t r = 0; r < m.e_src.size(); ++r) rank_of[(uint64_t(m.e_src[r]) << 32) | m.e_seq[r]] = int64_t(r);
    std::vector<std::vector<uint64_t>> keys(nl);
    int64_t kmax = 0;
    for (int c = 0; c < nl; ++c) {
      const McgKind& K = m.kinds[m.cell_kind[c]];
      const int n = K.n;
      const int64_t co = m.comp_off[c];
      const std::string pre = "cell/" + std::to_string(m.gid_begin + uint32_t(c)) + "/";
      if (K.dyn != MCG_DYN_NONE) {
        const auto& a = sized(getf(pre + "v"), n);
        std::copy(a.begin(), a.end(), v.begin() + co);
      }
      const auto& dv = getf(pre + "det");
      if (dv.empty()) throw Error(MCG_ERR_ENGINE, "checkpoint: state size mismatch");
      det[c] = dv[0];
      const auto& fl = getu(pre + "flags");
      if (fl.size() < 3) throw Error(MCG_ERR_ENGINE, "checkpoint: state size mismatch");
      refr[c] = static_cast<int64_t>(fl[0]);
      armed[c] = fl[1] != 0 ? 1 : 0;
      iseq[c] = static_cast<uint32_t>(fl[2]);
      for (int q = 0; q < K.n_species; ++q) {
        const auto& a = sized(getf(pre + "species/" + std::to_string(q)), n);
        std::copy(a.begin(), a.end(), sp.begin() + m.sp_off[c] + int64_t(q) * n);
      }
      if (K.dyn == MCG_DYN_HH) {
        std::copy(sized(getf(pre + "hh_m"), n).begin(), sized(getf(pre + "hh_m"), n).end(), hm.begin() + co);
        std::copy(sized(getf(pre + "hh_h"), n).begin(), sized(getf(pre + "hh_h"), n).end(), hh.begin() + co);
        std::copy(sized(getf(pre + "hh_n"), n).begin(), sized(getf(pre + "hh_n"), n).end(), hn.begin() + co);
      }
      for (int gi = 0; gi < K.n_groups; ++gi) {
        McgCellGroup& G = cgs[m.cg_off[c] + gi];
        const McgSpec& S = m.specs[G.spec];
        const std::string gp = pre + "g" + std::to_string(gi) + "/";
        const int64_t a = G.inst;
        const auto& kk = sized(getf(gp + "kernel"), G.size);
        const auto& ww = sized(getf(gp + "weight"), G.size);
        std::copy(kk.begin(), kk.end(), ker.begin() + a);
        std::copy(ww.begin(), ww.end(), wgt.begin() + a);
        if (S.kind == MCG_SYN_STATIC_COND || S.kind == MCG_SYN_STDP_COND ||
            S.kind == MCG_SYN_STATIC_CURRENT || S.kind == MCG_SYN_HOMEO_CURRENT) {
          int na = 0;  // active list in instance order (engine.cpp:1262-1264)
          for (int i = 0; i < G.size; ++i)
            if (kk[i] != 0.0) act[a + na++] = i;
          G.active_n = na;
        }
        if (G.size > 0 && S.kind == MCG_SYN_STDP_COND) {
          const auto& x = sized(getf(gp + "stdp_a_pre"), G.size);
          const auto& y = sized(getf(gp + "stdp_a_post"), G.size);
          const auto& z = sized(getf(gp + "stdp_w"), G.size);
          const auto& l = getu(gp + "stdp_last");
          if (l.size() != size_t(G.size)) throw Error(MCG_ERR_ENGINE, "checkpoint: state size mismatch");
          for (int i = 0; i < G.size; ++i) {
            spre[a + i] = x[i];
            spost[a + i] = y[i];
            sw[a + i] = z[i];
            slast[a + i] = static_cast<int64_t>(l[i]);
          }
        }
        if (G.size > 0 && S.kind == MCG_SYN_HOMEO_CURRENT) {
          const auto& x = sized(getf(gp + "homeo_w"), G.size);
          std::copy(x.begin(), x.end(), hw.begin() + a);
        }
        if (G.size > 0 && S.kind == MCG_SYN_STC_CHARGE) {
          const auto& x = sized(getf(gp + "stc_h"), G.size);
          const auto& y = sized(getf(gp + "stc_z"), G.size);
          const auto& z = sized(getf(gp + "stc_c"), G.size);
          const auto& q = sized(getf(gp + "stc_sps"), G.size);
          std::copy(x.begin(), x.end(), sh.begin() + a);
          std::copy(y.begin(), y.end(), sz.begin() + a);
          std::copy(z.begin(), z.end(), sc.begin() + a);
          std::copy(q.begin(), q.end(), sa.begin() + a);
        }
        if (G.fifo >= 0) fifos[G.fifo].head = fifos[G.fifo].tail = 0;
      }
      // pending network events -> sorted keys
      for (const CkEvent& e : ck_unpack(getu(pre + "inbox_meta"), getf(pre + "inbox_w"))) {
        auto it = rank_of.find((uint64_t(e.src) << 32) | e.seq);
        if (it == rank_of.end() || e.etype != 0) throw Error(MCG_ERR_ENGINE, "checkpoint: event does not match the recipe");
        const int64_t r = it->second;
        if (m.e_dst[r] != c || m.e_group[r] != e.group || m.e_inst[r] != e.instance ||
            std::memcmp(&m.e_weight[r], &e.weight, 8) != 0 || e.step < 0)
          throw Error(MCG_ERR_ENGINE, "checkpoint: event does not match the recipe");
        keys[c].push_back((uint64_t(e.step) << rank_bits) | uint64_t(r));
      }
      std::sort(keys[c].begin(), keys[c].end());
      kmax = std::max<int64_t>(kmax, int64_t(keys[c].size()));
      // delayed calcium -> the groups' queues, in (step, seq) order
      std::vector<CkEvent> internal = ck_unpack(getu(pre + "internal_meta"), getf(pre + "internal_w"));
      std::sort(internal.begin(), internal.end(), [](const CkEvent& x, const CkEvent& y) {
        if (x.step != y.step) return x.step < y.step;
        return x.seq < y.seq;
      });
      for (const CkEvent& e : internal) {
        if (e.group >= K.n_groups || e.etype != 1) throw Error(MCG_ERR_ENGINE, "checkpoint: event does not match the recipe");
        const McgCellGroup& G = cgs[m.cg_off[c] + e.group];
        if (G.fifo < 0) throw Error(MCG_ERR_ENGINE, "checkpoint: event does not match the recipe");
        McgFifo& F = fifos[G.fifo];
        if (F.tail - F.head >= F.cap) throw Error(MCG_ERR_ENGINE, "internal event queue overflow");
        const int64_t slot = F.base + (F.tail % F.cap);
        fstep[slot] = e.step;
        fsi[slot] = (uint64_t(e.seq) << 32) | e.instance;
        fsrc[slot] = e.src;
        fw[slot] = e.weight;
        ++F.tail;
      }
    }
    while (kmax > pend_cap) grow_inboxes();
    std::vector<uint64_t> pend(size_t(std::max(nl, 1)) * 2 * pend_cap, 0);
    std::vector<int32_t> psel(nl, 0), poff(nl, 0), pn(nl, 0);
    for (int c = 0; c < nl; ++c) {
      std::copy(keys[c].begin(), keys[c].end(), pend.begin() + size_t(c) * 2 * pend_cap);
      pn[c] = static_cast<int32_t>(keys[c].size());
    }
    upload_to(d_v, v);
    upload_to(d_hh_m, hm);
    upload_to(d_hh_h, hh);
    upload_to(d_hh_n, hn);
    upload_to(d_species, sp);
    upload_to(d_det_prev, det);
    upload_to(d_armed, armed);
    upload_to(d_refr, refr);
    upload_to(d_iseq, iseq);
    upload_to(d_i_kernel, ker);
    upload_to(d_i_weight, wgt);
    upload_to(d_i_stdp_pre, spre);
    upload_to(d_i_stdp_post, spost);
    upload_to(d_i_stdp_w, sw);
    upload_to(d_i_stdp_last, slast);
    upload_to(d_i_homeo_w, hw);
    upload_to(d_i_stc_h, sh);
    upload_to(d_i_stc_z, sz);
    upload_to(d_i_stc_c, sc);
    upload_to(d_i_sps_abs, sa);
    upload_to(d_i_active, act);
    upload_to(d_cgs, cgs);
    upload_to(d_fifos, fifos);
    upload_to(d_fifo_step, fstep);
    upload_to(d_fifo_si, fsi);
    upload_to(d_fifo_src, fsrc);
    upload_to(d_fifo_w, fw);
    upload_to(d_pend, pend);
    upload_to(d_pend_sel, psel);
    upload_to(d_pend_off, poff);
    upload_to(d_pend_n, pn);
    d_inc_n.zero(st);
    d_sp_count.zero(st);
    CK(cudaStreamSynchronize(st));
    step = static_cast<int64_t>(stv[0]);
    refresh_dev();
  }
};

}  // namespace mcg

struct mcg_engine {
  mcg::Engine e;
};

namespace {
template <class F>
mcg_status guarded(F&& f) {
  try {
    f();
    return MCG_OK;
  } catch (const mcg::Error& e) {
    mcg::g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    mcg::g_last_error = e.what();
    return MCG_ERR_ARGUMENT;
  }
}
}  // namespace

extern "C" {

int32_t mcg_abi_version(void) { return MCG_ABI_VERSION; }
const char* mcg_last_error(void) { return mcg::g_last_error.c_str(); }

mcg_status mcg_create(const mcg_recipe* recipe, const mcg_options* opt, mcg_engine** out) {
  return guarded([&] {
    if (!recipe || !opt || !out) throw mcg::Error(MCG_ERR_ARGUMENT, "null argument");
    *out = nullptr;
    if (!(opt->dt_ms > 0)) throw mcg::Error(MCG_ERR_ENGINE, "dt must be positive");
    if (opt->world < 1 || opt->rank < 0 || opt->rank >= opt->world)
      throw mcg::Error(MCG_ERR_ARGUMENT, "invalid rank/world");
    auto h = std::make_unique<mcg_engine>();
    h->e.init(*recipe, *opt);
    *out = h.release();
  });
}

void mcg_destroy(mcg_engine* eng) { delete eng; }

double mcg_time_ms(const mcg_engine* eng) { return double(eng->e.step) * eng->e.m.dt; }
double mcg_dt_ms(const mcg_engine* eng) { return eng->e.m.dt; }
int64_t mcg_step(const mcg_engine* eng) { return eng->e.step; }
int32_t mcg_num_cells(const mcg_engine* eng) { return eng->e.m.n_cells_global; }
int64_t mcg_min_delay_steps(const mcg_engine* eng) { return eng->e.m.min_delay_steps; }

mcg_status mcg_advance_to(mcg_engine* eng, double t_ms) {
  return guarded([&] { eng->e.advance_to(t_ms); });
}
mcg_status mcg_fast_forward_to(mcg_engine* eng, double t_ms, double coarse_dt_ms) {
  return guarded([&] { eng->e.fast_forward_to(t_ms, coarse_dt_ms); });
}

int64_t mcg_num_spikes(mcg_engine* eng) {
  int64_t n = -1;
  guarded([&] {
    eng->e.sync_spikes();
    n = static_cast<int64_t>(eng->e.spk_t.size());
  });
  return n;
}
mcg_status mcg_get_spikes(mcg_engine* eng, int64_t first, int64_t count, double* t_ms,
                          uint32_t* gid) {
  return guarded([&] {
    eng->e.sync_spikes();
    const int64_t n = static_cast<int64_t>(eng->e.spk_t.size());
    if (first < 0 || count < 0 || first + count > n)
      throw mcg::Error(MCG_ERR_ARGUMENT, "spike range out of bounds");
    std::memcpy(t_ms, eng->e.spk_t.data() + first, count * sizeof(double));
    std::memcpy(gid, eng->e.spk_gid.data() + first, count * sizeof(uint32_t));
  });
}
mcg_status mcg_clear_spikes(mcg_engine* eng) { return guarded([&] { eng->e.clear_spikes(); }); }

int64_t mcg_trace_len(mcg_engine* eng, int32_t probe) {
  if (probe < 0 || probe >= static_cast<int32_t>(eng->e.traces.size())) return -1;
  return static_cast<int64_t>(eng->e.traces[probe].size());
}
mcg_status mcg_get_trace(mcg_engine* eng, int32_t probe, double* t_ms, double* value) {
  return guarded([&] {
    if (probe < 0 || probe >= static_cast<int32_t>(eng->e.traces.size()))
      throw mcg::Error(MCG_ERR_ARGUMENT, "probe index out of range");
    const auto& tr = eng->e.traces[probe];
    for (size_t i = 0; i < tr.size(); ++i) {
      t_ms[i] = tr[i].first;
      value[i] = tr[i].second;
    }
  });
}

int32_t mcg_cell_ncomp(const mcg_engine* eng, uint32_t gid) {
  const auto& E = eng->e;
  if (gid < E.m.gid_begin || gid >= E.m.gid_end) return -1;
  return E.m.kinds[E.m.cell_kind[gid - E.m.gid_begin]].n;
}
int32_t mcg_cell_ngroups(const mcg_engine* eng, uint32_t gid) {
  const auto& E = eng->e;
  if (gid < E.m.gid_begin || gid >= E.m.gid_end) return -1;
  return E.m.kinds[E.m.cell_kind[gid - E.m.gid_begin]].n_groups;
}
int64_t mcg_group_size(const mcg_engine* eng, uint32_t gid, int32_t group) {
  const auto& E = eng->e;
  if (gid < E.m.gid_begin || gid >= E.m.gid_end) return -1;
  const int c = static_cast<int>(gid - E.m.gid_begin);
  const auto& K = E.m.kinds[E.m.cell_kind[c]];
  if (group < 0 || group >= K.n_groups) return -1;
  return E.m.cgs[E.m.cg_off[c] + group].size;
}
int32_t mcg_cell_parent(const mcg_engine* eng, uint32_t gid, int32_t comp) {
  const auto& E = eng->e;
  if (gid < E.m.gid_begin || gid >= E.m.gid_end) return -2;
  const auto& K = E.m.kinds[E.m.cell_kind[gid - E.m.gid_begin]];
  if (comp < 0 || comp >= K.n) return -2;
  return E.m.k_parent[K.arr + comp];
}

mcg_status mcg_checkpoint(mcg_engine* eng, uint8_t* buf, int64_t cap, int64_t* size) {
  return guarded([&] {
    if (!eng || !size) throw mcg::Error(MCG_ERR_ARGUMENT, "checkpoint: null argument");
    const std::vector<uint8_t> b = eng->e.make_checkpoint();
    *size = static_cast<int64_t>(b.size());
    if (buf) {
      if (cap < *size) throw mcg::Error(MCG_ERR_ARGUMENT, "checkpoint: buffer too small");
      std::memcpy(buf, b.data(), b.size());
    }
  });
}

mcg_status mcg_restore(mcg_engine* eng, const uint8_t* buf, int64_t size) {
  return guarded([&] {
    if (!eng || (!buf && size > 0) || size < 0) throw mcg::Error(MCG_ERR_ARGUMENT, "restore: null argument");
    eng->e.restore(buf, static_cast<size_t>(size));
  });
}

mcg_status mcg_read_state(mcg_engine* eng, int32_t field, uint32_t gid, int32_t index,
                          int64_t offset, int64_t count, void* out) {
  return guarded([&] { eng->e.state_io(field, gid, index, offset, count, out, nullptr, false); });
}
mcg_status mcg_write_state(mcg_engine* eng, int32_t field, uint32_t gid, int32_t index,
                           int64_t offset, int64_t count, const void* in) {
  return guarded([&] { eng->e.state_io(field, gid, index, offset, count, nullptr, in, true); });
}

mcg_status mcg_get_stats(mcg_engine* eng, mcg_stats* out) {
  return guarded([&] {
    eng->e.sync_counters_raw();
    eng->e.stats.events_delivered = static_cast<int64_t>(eng->e.h_ctr[mcg::C_DELIVERED]);
    eng->e.stats.stepping_kernel = eng->e.use_point ? 2 : (eng->e.use_warp ? 1 : 0);
    eng->e.stats.edges_on_device = eng->e.m.edges_deferred ? 1 : 0;
    *out = eng->e.stats;
  });
}
mcg_status mcg_set_cell_rng(mcg_engine* eng, const uint64_t* seeds, const uint32_t* key_gids) {
  return guarded([&] {
    mcg::Engine& E = eng->e;
    if (!E.use_point)
      throw mcg::Error(MCG_ERR_ENGINE, "per-cell RNG keys need the point-cell kernel (k_point)");
    const int nl = E.n_local();
    std::vector<uint64_t> sd(seeds, seeds + nl);
    std::vector<uint32_t> kg(key_gids, key_gids + nl);
    E.d_cell_seed.upload(sd, E.st);
    E.d_cell_key_gid.upload(kg, E.st);
    E.refresh_dev();
    mcg::cuda_check(cudaStreamSynchronize(E.st), "cudaStreamSynchronize");
  });
}

mcg_status mcg_set_timing(mcg_engine* eng, int32_t enabled) {
  return guarded([&] { eng->e.timing = enabled != 0; });
}

int64_t mcg_shard_spike_cap(const mcg_engine* eng) { return eng ? eng->e.shard_spike_cap() : 0; }

uint32_t mcg_shard_gid_begin(const mcg_engine* eng) { return eng ? eng->e.m.gid_begin : 0; }

uint32_t mcg_shard_gid_end(const mcg_engine* eng) { return eng ? eng->e.m.gid_end : 0; }

mcg_status mcg_shard_set_buffers(mcg_engine* eng, int64_t* send, int64_t* recv, int64_t block_cap,
                                 int32_t world) {
  return guarded([&] {
    if (!eng || !send || !recv || world < 1)
      throw mcg::Error(MCG_ERR_ARGUMENT, "shard buffers: null pointer or world < 1");
    mcg::Engine* E = &eng->e;
    if (block_cap < E->shard_spike_cap())
      throw mcg::Error(MCG_ERR_ARGUMENT, "shard buffers: block capacity below mcg_shard_spike_cap");
    E->x_send = send;
    E->x_recv = recv;
    E->x_cap = block_cap;
    E->x_world = world;
  });
}

mcg_status mcg_partition(const mcg_recipe* recipe, int32_t world, uint32_t* bounds) {
  return guarded([&] {
    if (!recipe || !bounds || world < 1)
      throw mcg::Error(MCG_ERR_ARGUMENT, "partition: null pointer or world < 1");
    std::vector<uint32_t> b;
    mcg::partition(*recipe, world, b);
    std::copy(b.begin(), b.end(), bounds);
  });
}

extern "C++" {
// FNV-1a over the runtime layout: edge records, instances, CSRs, groups, queues
static void layout_digest(const mcg::HostModel& m, uint64_t out[4]) {
  uint64_t h = 1469598103934665603ull;  // FNV-1a over the layout
  auto mix = [&](uint64_t x) {
    h ^= x;
    h *= 1099511628211ull;
  };
  auto mixd = [&](double x) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    mix(b);
  };
  for (size_t i = 0; i < m.e_dst.size(); ++i) {
    mix(uint64_t(m.e_dst[i]));
    mix(uint64_t(m.e_group[i]));
    mix(m.e_inst[i]);
    mix(m.e_src[i]);
    mix(m.e_seq[i]);
    mix(uint64_t(m.e_delay[i]));
    mix(uint64_t(int64_t(m.e_comp[i])));
    mixd(m.e_weight[i]);
    mixd(m.e_wcf[i]);
  }
  for (size_t i = 0; i < m.i_comp.size(); ++i) {
    mix(uint64_t(m.i_comp[i]));
    mixd(m.i_weight[i]);
    mixd(m.i_stc_h[i]);
  }
  for (double x : m.i_stdp_w) mixd(x);
  for (double x : m.i_homeo_w) mixd(x);
  for (int64_t x : m.src_edge_off) mix(uint64_t(x));
  for (int64_t x : m.src_edges) mix(uint64_t(x));
  for (int64_t x : m.out_begin) mix(uint64_t(x));
  for (int64_t x : m.out_end) mix(uint64_t(x));
  for (const McgCellGroup& G : m.cgs) {
    mix(uint64_t(G.inst));
    mix(uint64_t(G.size));
    mix(uint64_t(int64_t(G.fifo)));
  }
  for (const McgFifo& F : m.fifos) {
    mix(uint64_t(F.base));
    mix(uint64_t(F.cap));
  }
  mix(uint64_t(m.min_delay_steps));
  mix(uint64_t(m.max_delay_steps));
  out[0] = h;
  out[1] = m.e_dst.size();
  out[2] = uint64_t(m.n_inst);
  out[3] = uint64_t(m.min_delay_steps);
}
}  // extern "C++"

mcg_status mcg_build_digest(const mcg_recipe* recipe, const mcg_options* opt, int32_t threads,
                            uint64_t out[4]) {
  return guarded([&] {
    if (!recipe || !opt || !out) throw mcg::Error(MCG_ERR_ARGUMENT, "build_digest: null pointer");
    mcg::HostModel m;
    mcg::build_model(*recipe, *opt, m, threads);
    layout_digest(m, out);
  });
}

mcg_status mcg_engine_layout_digest(mcg_engine* eng, uint64_t out[4]) {
  return guarded([&] {
    if (!eng || !out) throw mcg::Error(MCG_ERR_ARGUMENT, "engine_layout_digest: null pointer");
    eng->e.layout_digest(out);
  });
}

mcg_status mcg_shard_run_epoch(mcg_engine* eng, double t_ms) {
  return guarded([&] { eng->e.run_epoch(t_ms); });
}

mcg_status mcg_nccl_unique_id(uint8_t* id) {
  return guarded([&] {
    if (!id) throw mcg::Error(MCG_ERR_ARGUMENT, "nccl: null id");
    mcg::NcclApi& api = mcg::nccl_api();
    ncclUniqueId uid;
    api.check(api.get_unique_id(&uid), "ncclGetUniqueId");
    std::memcpy(id, &uid, sizeof(uid));
  });
}

mcg_status mcg_shard_init_nccl(mcg_engine* eng, const uint8_t* id) {
  return guarded([&] {
    if (!eng || !id) throw mcg::Error(MCG_ERR_ARGUMENT, "nccl: null pointer");
    eng->e.init_nccl(id);
  });
}

mcg_status mcg_shard_advance_to(mcg_engine* eng, double t_ms) {
  return guarded([&] { eng->e.shard_advance(t_ms); });
}

int64_t mcg_shard_num_global_spikes(const mcg_engine* eng) {
  return eng ? static_cast<int64_t>(eng->e.gspk_t.size()) : 0;
}

mcg_status mcg_shard_get_global_spikes(mcg_engine* eng, int64_t first, int64_t count, double* t_ms,
                                       uint32_t* gid) {
  return guarded([&] {
    const mcg::Engine& E = eng->e;
    if (first < 0 || count < 0 || first + count > static_cast<int64_t>(E.gspk_t.size()))
      throw mcg::Error(MCG_ERR_ARGUMENT, "spike range out of bounds");
    for (int64_t i = 0; i < count; ++i) {
      if (t_ms) t_ms[i] = E.gspk_t[first + i];
      if (gid) gid[i] = E.gspk_gid[first + i];
    }
  });
}

}  // extern "C"

// ---- device numerics self-test ------------------------------------------------
__global__ void k_device_math(int32_t func, const double* in, int64_t n, mcg_key key, uint64_t n0,
                              double* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s, c;
  switch (func) {
    case MCG_MATH_EXP: out[i] = mcg_exp(in[i]); break;
    case MCG_MATH_LOG: out[i] = mcg_log(in[i]); break;
    case MCG_MATH_SIN: mcg_sincos(in[i], &s, &c); out[i] = s; break;
    case MCG_MATH_COS: mcg_sincos(in[i], &s, &c); out[i] = c; break;
    case MCG_MATH_UNIFORM_FOR: out[i] = mcg_uniform_for(&key, n0 + uint64_t(i)); break;
    case MCG_MATH_NORMAL_FOR: out[i] = mcg_normal_for(&key, n0 + uint64_t(i)); break;
    default: out[i] = 0.0;
  }
}

extern "C" mcg_status mcg_device_math(int32_t device, int32_t func, const double* in, int64_t n,
                                      const uint64_t key[4], uint64_t n0, double* out) {
  return guarded([&] {
    using mcg::cuda_check;
    CK(cudaSetDevice(device));
    if (n <= 0) return;
    double *din = nullptr, *dout = nullptr;
    CK(cudaMalloc(&din, n * sizeof(double)));
    CK(cudaMalloc(&dout, n * sizeof(double)));
    if (in) CK(cudaMemcpy(din, in, n * sizeof(double), cudaMemcpyHostToDevice));
    mcg_key k = mcg_make_key(key ? key[0] : 0, key ? key[1] : 0, key ? key[2] : 0,
                             key ? key[3] : 0);
    k_device_math<<<static_cast<unsigned>((n + 255) / 256), 256>>>(func, din, n, k, n0, dout);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, dout, n * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(din);
    cudaFree(dout);
  });
}

// ---- Erdos-Renyi connectivity on the device ---------------------------------------
// thread t covers pair indices [t*64, t*64+64) of the row-major (i, j) space
// restricted to rows [r0, r1); pass 1 counts, pass 2 writes in order.
#define MCG_ER_CHUNK 64
__global__ void k_er(uint64_t seed, uint32_t n, double p, uint64_t k0, uint64_t k1,
                     int64_t* counts, const int64_t* offs, uint32_t* src, uint32_t* dst) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t a = k0 + t * MCG_ER_CHUNK;
  if (a >= k1) return;
  const uint64_t b = a + MCG_ER_CHUNK < k1 ? a + MCG_ER_CHUNK : k1;
  const mcg_key key = mcg_make_key(seed, 0, 17, 0);
  int64_t c = 0, o = offs ? offs[t] : 0;
  uint64_t x[4];
  uint64_t blk = ~0ull;
  uint32_t i = uint32_t(a / n), j = uint32_t(a - uint64_t(i) * n);  // (i, j) of pair k, stepped
  for (uint64_t k = a; k < b; ++k, ++j) {
    if (j == n) {
      j = 0;
      ++i;
    }
    if ((k >> 2) != blk) {
      blk = k >> 2;
      mcg_threefry(&key, blk, x);
    }
    if (i == j) continue;
    const double u = (double)(x[k & 3u] >> 11) * MCG_2POW_M53;
    if (u < p) {
      if (src) {
        src[o + c] = i;
        dst[o + c] = j;
      }
      ++c;
    }
  }
  if (!offs) counts[t] = c;
}

extern "C" mcg_status mcg_er_connect(int32_t device, uint64_t seed, uint32_t n, double p,
                                     uint32_t src_begin, uint32_t src_end, uint32_t* src,
                                     uint32_t* dst, int64_t* count) {
  return guarded([&] {
    using mcg::cuda_check;
    CK(cudaSetDevice(device));
    const uint64_t k0 = uint64_t(src_begin) * n, k1 = uint64_t(src_end) * n;
    if (k1 <= k0) {
      *count = 0;
      return;
    }
    const uint64_t nthr = (k1 - k0 + MCG_ER_CHUNK - 1) / MCG_ER_CHUNK;
    int64_t *d_cnt = nullptr, *d_off = nullptr;
    CK(cudaMalloc(&d_cnt, nthr * sizeof(int64_t)));
    CK(cudaMalloc(&d_off, nthr * sizeof(int64_t)));
    const unsigned blocks = static_cast<unsigned>((nthr + 255) / 256);
    k_er<<<blocks, 256>>>(seed, n, p, k0, k1, d_cnt, nullptr, nullptr, nullptr);
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, d_cnt, d_off, static_cast<int64_t>(nthr)));
    void* tmp = nullptr;
    CK(cudaMalloc(&tmp, tb));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, d_cnt, d_off, static_cast<int64_t>(nthr)));
    int64_t last_off = 0, last_cnt = 0;
    CK(cudaMemcpy(&last_off, d_off + nthr - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&last_cnt, d_cnt + nthr - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
    const int64_t total = last_off + last_cnt;
    if (src && dst && total > 0) {
      if (*count < total) throw mcg::Error(MCG_ERR_ARGUMENT, "er_connect: output too small");
      uint32_t *d_src = nullptr, *d_dst = nullptr;
      CK(cudaMalloc(&d_src, total * sizeof(uint32_t)));
      CK(cudaMalloc(&d_dst, total * sizeof(uint32_t)));
      k_er<<<blocks, 256>>>(seed, n, p, k0, k1, d_cnt, d_off, d_src, d_dst);
      CK(cudaMemcpy(src, d_src, total * sizeof(uint32_t), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(dst, d_dst, total * sizeof(uint32_t), cudaMemcpyDeviceToHost));
      cudaFree(d_src);
      cudaFree(d_dst);
    }
    cudaFree(tmp);
    cudaFree(d_cnt);
    cudaFree(d_off);
    *count = total;
  });
}

// ---- standalone protocol drivers (mcg_protocols.cuh) ------------------------------
namespace {
// the calcium jump schedule of gb_pairing_trial (mechanisms.cpp:46-58), sorted
// with the same std::sort call; returns n_steps (:60-61)
int64_t gb_schedule(const mcg_gb_params& p, double delta_t_ms, const mcg_gb_protocol& proto,
                    std::vector<std::pair<int64_t, double>>& jumps) {
  const double dt = proto.dt_ms;
  const auto step_of = [dt](double t) { return static_cast<int64_t>(std::ceil(t / dt - 1e-9)); };
  jumps.clear();
  jumps.reserve(2 * proto.n_pairs);
  const double t0 = 100.0 + std::max(0.0, -delta_t_ms);
  for (int k = 0; k < proto.n_pairs; ++k) {
    const double t_pre = t0 + k * proto.period_ms;
    jumps.emplace_back(step_of(t_pre + p.t_c_delay_ms), p.c_pre);
    jumps.emplace_back(step_of(t_pre + delta_t_ms), p.c_post);
  }
  std::sort(jumps.begin(), jumps.end(),
            [](const auto& a, const auto& b) { return a.first < b.first; });
  return step_of(t0 + proto.n_pairs * proto.period_ms + proto.settle_ms);
}
}  // namespace

extern "C" mcg_status mcg_gb_trials(int32_t device, const mcg_gb_params* p, const double* deltas,
                                    int32_t n_deltas, const mcg_gb_protocol* proto, double* w0,
                                    double* wf) {
  return guarded([&] {
    using mcg::cuda_check;
    if (!p || !proto || (n_deltas > 0 && (!deltas || !w0 || !wf)))
      throw mcg::Error(MCG_ERR_ARGUMENT, "gb_trials: null argument");
    if (n_deltas <= 0 || proto->trials <= 0) return;
    if (!(proto->dt_ms > 0)) throw mcg::Error(MCG_ERR_ARGUMENT, "gb_trials: dt must be positive");
    CK(cudaSetDevice(device));
    std::vector<int64_t> jstep, nsteps(n_deltas);
    std::vector<double> jamt;
    std::vector<int32_t> joff(n_deltas + 1, 0);
    std::vector<std::pair<int64_t, double>> jumps;
    for (int d = 0; d < n_deltas; ++d) {
      nsteps[d] = gb_schedule(*p, deltas[d], *proto, jumps);
      for (const auto& j : jumps) {
        jstep.push_back(j.first);
        jamt.push_back(j.second);
      }
      joff[d + 1] = static_cast<int32_t>(jstep.size());
    }
    McgGbDev P{};
    P.tau_w = p->tau_w_ms;
    P.w_star = p->w_star;
    P.gamma_p = p->gamma_p;
    P.gamma_d = p->gamma_d;
    P.theta_p = p->theta_p;
    P.theta_d = p->theta_d;
    P.sigma = p->sigma_pl;
    P.r_tau_w = mcg::mcg_recip(p->tau_w_ms);
    P.cdecay = std::exp(-proto->dt_ms / p->tau_c_ms);
    P.nz1 = p->sigma_pl * std::sqrt(double(1) / p->tau_w_ms) * std::sqrt(proto->dt_ms);
    P.nz2 = p->sigma_pl * std::sqrt(double(2) / p->tau_w_ms) * std::sqrt(proto->dt_ms);
    P.dt = proto->dt_ms;
    P.seed = proto->seed;
    P.trials = proto->trials;
    P.n_deltas = n_deltas;
    const int64_t nt = int64_t(proto->trials) * n_deltas;
    mcg::DBuf<int64_t> d_js, d_ns;
    mcg::DBuf<double> d_ja, d_w0, d_wf;
    mcg::DBuf<int32_t> d_jo;
    d_js.upload(jstep, 0);
    d_ja.upload(jamt, 0);
    d_jo.upload(joff, 0);
    d_ns.upload(nsteps, 0);
    d_w0.alloc(nt);
    d_wf.alloc(nt);
    k_gb_trials<<<static_cast<unsigned>((nt + 127) / 128), 128>>>(P, d_js.p, d_ja.p, d_jo.p, d_ns.p,
                                                                   d_w0.p, d_wf.p);
    CK(cudaGetLastError());
    CK(cudaMemcpy(w0, d_w0.p, nt * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(wf, d_wf.p, nt * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

extern "C" mcg_status mcg_gb_dp_curve(int32_t device, const mcg_gb_params* p, const double* deltas,
                                      int32_t n_deltas, const mcg_gb_protocol* proto,
                                      mcg_gb_point* out) {
  if (!proto || !out || n_deltas < 0) {
    mcg::g_last_error = "gb_dp_curve: null argument";
    return MCG_ERR_ARGUMENT;
  }
  const int T = proto->trials;
  std::vector<double> w0(size_t(std::max(T, 0)) * std::max(n_deltas, 0)), wf(w0.size());
  const mcg_status st = mcg_gb_trials(device, p, deltas, n_deltas, proto, w0.data(), wf.data());
  if (st != MCG_OK) return st;
  // gb_dp_curve's reductions (mechanisms.cpp:99-116) and mean_ci (analysis.cpp:82-94)
  for (int d = 0; d < n_deltas; ++d) {
    std::vector<double> change(T);
    double sum_w0 = 0, sum_wf = 0;
    for (int tr = 0; tr < T; ++tr) {
      const double a = w0[size_t(d) * T + tr], b = wf[size_t(d) * T + tr];
      change[tr] = b - a;
      sum_w0 += a;
      sum_wf += b;
    }
    double mean = 0, half = 0;
    if (T > 0) {
      for (double s : change) mean += s;
      mean /= T;
      if (T >= 2) {
        double var = 0;
        for (double s : change) var += (s - mean) * (s - mean);
        var /= (T - 1);
        half = 1.959963984540054 * std::sqrt(var / T);
      }
    }
    mcg_gb_point& pt = out[d];
    pt.delta_t_ms = deltas[d];
    pt.mean_initial = sum_w0 / T;
    pt.mean_final = sum_wf / T;
    pt.mean_change = mean;
    pt.change_ci_half = half;
    pt.ratio = pt.mean_initial != 0 ? pt.mean_final / pt.mean_initial : 0.0;
  }
  return MCG_OK;
}

extern "C" mcg_status mcg_stdp_window(int32_t device, const mcg_stdp_params* p,
                                      const double* deltas, int32_t n, int32_t n_pairs,
                                      double period_ms, double* out) {
  return guarded([&] {
    using mcg::cuda_check;
    if (!p || (n > 0 && (!deltas || !out))) throw mcg::Error(MCG_ERR_ARGUMENT, "stdp_window: null argument");
    if (n <= 0) return;
    CK(cudaSetDevice(device));
    // the pairing events of stdp_window (mechanisms.cpp:12-24), stable-sorted
    struct Ev {
      double t;
      bool pre;
    };
    std::vector<double> et;
    std::vector<uint8_t> ep;
    std::vector<int32_t> eo(n + 1, 0);
    for (int i = 0; i < n; ++i) {
      const double delta_t_ms = deltas[i];
      std::vector<Ev> events;
      events.reserve(2 * n_pairs);
      const double t0 = std::max(0.0, -delta_t_ms);
      for (int k = 0; k < n_pairs; ++k) {
        events.push_back({t0 + k * period_ms, true});
        events.push_back({t0 + k * period_ms + delta_t_ms, false});
      }
      std::stable_sort(events.begin(), events.end(), [](const Ev& a, const Ev& b) { return a.t < b.t; });
      for (const Ev& e : events) {
        et.push_back(e.t);
        ep.push_back(e.pre ? 1 : 0);
      }
      eo[i + 1] = static_cast<int32_t>(et.size());
    }
    McgStdpDev P{p->tau_pre_ms, p->tau_post_ms, p->a_pre_uS, p->a_post_uS, p->w0_uS, n, n_pairs};
    mcg::DBuf<double> d_t, d_out;
    mcg::DBuf<uint8_t> d_p;
    mcg::DBuf<int32_t> d_o;
    d_t.upload(et, 0);
    d_p.upload(ep, 0);
    d_o.upload(eo, 0);
    d_out.alloc(n);
    k_stdp_window<<<(n + 127) / 128, 128>>>(P, d_t.p, d_p.p, d_o.p, d_out.p);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, d_out.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  });
}
