/* mcg.h — C ABI of the B200 cable-cell integration engine.
 *
 * This is the drop-in boundary for the reference's per-timestep integration
 * loop.  The reference exposes that loop as the in-process C++ class
 * mcsim::Engine (/root/reference/proj/include/mcsim/engine.hpp:126-167,
 * pimpl Engine::Impl at src/engine.cpp:149-185), constructed from a
 * declarative mcsim::Recipe (include/mcsim/recipe.hpp:24-189).  Every entry
 * point below replaces one member of that class; the mapping is listed per
 * function.  A C++ maintainer binds it by forwarding Engine's members to these
 * calls (INTEGRATION.md shows the shim); Python binds it with ctypes
 * (paper_2411_16445_b200/engine.py).
 *
 * Conventions: plain pointers and sizes only; every call returns an
 * mcg_status; on failure mcg_last_error() returns the same message text the
 * reference's exception carries (e.g. "configuration: dt exceeds a connection
 * delay", "fast-forward: pending undelivered spikes").  All device memory is
 * owned by the engine.  Units follow units.hpp: ms, mV, nA, uS, nF, um.
 */
#ifndef MCG_H
#define MCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCG_ABI_VERSION 1

typedef int32_t mcg_status;
enum {
  MCG_OK = 0,
  MCG_ERR_ENGINE = 1,     /* mcsim::EngineError     (engine.hpp:16-18)      */
  MCG_ERR_NUMERIC = 2,    /* mcsim::NumericError    (tree_solver.hpp:11-13) */
  MCG_ERR_TARGETING = 3,  /* mcsim::TargetingError  (recipe.hpp:138-140)    */
  MCG_ERR_MORPHOLOGY = 4, /* mcsim::MorphologyError (morphology.hpp:55-57)  */
  MCG_ERR_CUDA = 5,       /* device failure (no reference equivalent)       */
  MCG_ERR_ARGUMENT = 6    /* invalid argument to this ABI                   */
};

/* ---- recipe: flat mirror of recipe.hpp (field order preserved) -------- */

enum { MCG_MEMBRANE_NONE = 0, MCG_MEMBRANE_LIF = 1, MCG_MEMBRANE_HH = 2 };

typedef struct { /* LifMembrane, recipe.hpp:24-42 */
  double tau_mem_ms, r_mem_MOhm, v_rev_mV, v_reset_mV, v_thresh_mV, t_ref_ms;
  double r_axial_ohm_m, i_bg_nA, sigma_bg_nA_sqrt_ms, bg_quiet_t0_ms, bg_quiet_t1_ms;
  int32_t noise_comp, detector_comp, exact;
} mcg_lif;

typedef struct { /* HhMembrane, recipe.hpp:45-57 */
  double c_m, r_axial_ohm_m, g_leak, e_leak_mV, g_na, e_na_mV, g_k, e_k_mV;
  double v_init_mV, threshold_mV;
  int32_t detector_comp;
} mcg_hh;

typedef struct { /* SpeciesSpec (name resolved by the host layer) */
  double diffusivity, decay_tau_ms, init;
} mcg_species;

typedef struct { /* StdpParams, mechanisms.hpp:20-27 */
  double tau_pre_ms, tau_post_ms, a_pre_uS, a_post_uS, w0_uS, wmax_uS;
} mcg_stdp_params;

typedef struct { /* HomeostasisParams, mechanisms.hpp:57-63 */
  double dw_plus_nA, dw_minus_nA, w_init_nA, wmax_nA, w_varying_nA;
} mcg_homeo_params;

typedef struct { /* StcParams, mechanisms.hpp:175-194 */
  double h0_mV, tau_h_ms, tau_c_ms, gamma_p, gamma_d, theta_p, theta_d, sigma_pl_mV;
  double c_pre, c_post, t_c_delay_ms, tau_z_ms, f_int, theta_tag_mV;
  double tau_p_ms, p_max, theta_pro_mV;
} mcg_stc_params;

enum { /* SynKind, recipe.hpp:73-80 */
  MCG_SYN_STATIC_CHARGE = 0,
  MCG_SYN_STATIC_COND = 1,
  MCG_SYN_STATIC_CURRENT = 2,
  MCG_SYN_STDP_COND = 3,
  MCG_SYN_HOMEO_CURRENT = 4,
  MCG_SYN_STC_CHARGE = 5
};

typedef struct { /* SynSpec, recipe.hpp:82-90 */
  int32_t kind;
  double tau_syn_ms, e_rev_mV;
  mcg_stdp_params stdp;
  mcg_homeo_params homeo;
  mcg_stc_params stc;
  double calcium_scale;
} mcg_syn_spec;

typedef struct { /* PlacementSpec (label resolved by the host layer) */
  mcg_syn_spec syn;
  int32_t comp, count;
} mcg_placement;

enum { /* Region, morphology.hpp:12-19 */
  MCG_REGION_SOMA = 0, MCG_REGION_APICAL = 1, MCG_REGION_BASAL = 2,
  MCG_REGION_SPINE_NECK = 3, MCG_REGION_SPINE_HEAD = 4, MCG_REGION_GENERIC = 5
};

typedef struct { /* CellKindSpec, recipe.hpp:105-114 */
  int32_t n_segments;            /* Segment list (morphology.hpp:26-32)    */
  const int32_t* seg_parent;     /* -1 for the root                        */
  const double* seg_length_um;
  const double* seg_radius_um;
  const uint8_t* seg_tag;        /* MCG_REGION_*                           */
  const double* seg_parent_pos;
  double target_compartment_um;
  int32_t membrane;              /* MCG_MEMBRANE_*                          */
  mcg_lif lif;
  mcg_hh hh;
  int32_t n_species;
  const mcg_species* species;
  int32_t sps_idx, prp_idx;      /* species named sps_species/prp_species, -1 */
  int32_t n_placements;
  const mcg_placement* placements;
  int32_t prp_enabled, prp_comp; /* PrpUnitSpec                              */
} mcg_kind;

enum { MCG_SRC_POISSON = 0, MCG_SRC_REGULAR = 1, MCG_SRC_SCRIPTED = 2 };

typedef struct { /* SourceSpec variant, recipe.hpp:118-134 */
  int32_t type;
  int32_t n_values;     /* poisson: 3*windows (t0,t1,rate_hz); scripted: times */
  const double* values;
  double t0_ms, period_ms; /* regular */
  int64_t count;           /* regular */
} mcg_source;

enum { MCG_POLICY_UNIVALENT = 0, MCG_POLICY_ROUND_ROBIN = 1, MCG_POLICY_ROUND_ROBIN_HALT = 2 };

enum { /* ProbeWhat, recipe.hpp:163-171 */
  MCG_PROBE_VOLTAGE = 0, MCG_PROBE_SPECIES = 1, MCG_PROBE_SYN_WEIGHT = 2,
  MCG_PROBE_SYN_H = 3, MCG_PROBE_SYN_Z = 4, MCG_PROBE_SYN_C = 5, MCG_PROBE_SYN_KERNEL = 6
};

typedef struct { /* Recipe, recipe.hpp:183-189, connections/probes as SoA */
  int32_t n_kinds;
  const mcg_kind* kinds;
  int32_t n_cells;
  const uint32_t* cell_kind;
  int32_t n_sources;
  const mcg_source* sources;
  int64_t n_connections;          /* ConnectionSpec, recipe.hpp:151-159 */
  const uint8_t* conn_from_source;
  const uint32_t* conn_src;
  const uint32_t* conn_dst;
  const int32_t* conn_group;      /* label resolved to placement index; -1 = not found */
  const uint8_t* conn_policy;     /* MCG_POLICY_* */
  const double* conn_weight;
  const double* conn_delay_ms;
  int32_t n_probes;               /* ProbeSpec, recipe.hpp:173-181 */
  const uint32_t* probe_gid;
  const uint8_t* probe_what;      /* MCG_PROBE_* */
  const int32_t* probe_comp;
  const int32_t* probe_species;
  const int32_t* probe_group;     /* label resolved; -1 when the label is empty */
  const int32_t* probe_instance;
  const int32_t* probe_every;
  /* optional (0 / NULL allowed): the label text of each connection, so an
     unresolved label (conn_group -1) is reported with the reference's message
     "connection label '<label>' not found" (engine.cpp:367-369) */
  int32_t n_labels;
  const char* const* labels;
  const int32_t* conn_label;      /* index into labels per connection */
} mcg_recipe;

typedef struct { /* EngineOptions, engine.hpp:37-41, plus placement */
  double dt_ms;
  uint64_t seed;
  int32_t workers;    /* accepted for ABI parity; results never depend on it */
  int32_t device;     /* CUDA device ordinal                                  */
  int32_t rank;       /* this process's shard (0 for single-GPU)             */
  int32_t world;      /* number of shards (1 for single-GPU)                 */
} mcg_options;

typedef struct mcg_engine mcg_engine;

/* ---- lifecycle --------------------------------------------------------- */

/* Engine(const Recipe&, const EngineOptions&)  engine.cpp:893-899, Impl::build :312-408 */
mcg_status mcg_create(const mcg_recipe* recipe, const mcg_options* opt, mcg_engine** out);
/* ~Engine()  engine.cpp:901 */
void mcg_destroy(mcg_engine* eng);
/* message of the last failed call on this thread (exception what()) */
const char* mcg_last_error(void);
int32_t mcg_abi_version(void);

/* ---- time -------------------------------------------------------------- */

double mcg_time_ms(const mcg_engine* eng);   /* Engine::time_ms  engine.cpp:903 */
double mcg_dt_ms(const mcg_engine* eng);     /* Engine::dt_ms    engine.hpp:132 */
int64_t mcg_step(const mcg_engine* eng);     /* Engine::step     engine.hpp:133 */
int32_t mcg_num_cells(const mcg_engine* eng);/* Engine::num_cells engine.hpp:147 */
int64_t mcg_min_delay_steps(const mcg_engine* eng); /* Impl::min_delay_steps :156 */

/* Engine::advance_to  engine.cpp:909-945 (epoch loop: sources, delivery,
 * step_cell for every cell, spike exchange) */
mcg_status mcg_advance_to(mcg_engine* eng, double t_ms);
/* Engine::fast_forward_to  engine.cpp:947-1034 */
mcg_status mcg_fast_forward_to(mcg_engine* eng, double t_ms, double coarse_dt_ms);

/* ---- observables --------------------------------------------------------- */

/* Engine::spikes / clear_spikes  engine.hpp:144-145.  Records are in the
 * reference's order: epoch, then gid, then step. */
int64_t mcg_num_spikes(mcg_engine* eng);
mcg_status mcg_get_spikes(mcg_engine* eng, int64_t first, int64_t count, double* t_ms,
                          uint32_t* gid);
mcg_status mcg_clear_spikes(mcg_engine* eng);

/* Engine::traces  engine.hpp:153-155: probe i's (t_ms, value) samples */
int64_t mcg_trace_len(mcg_engine* eng, int32_t probe);
mcg_status mcg_get_trace(mcg_engine* eng, int32_t probe, double* t_ms, double* value);

/* Engine::cell(gid) / grid_of(gid) mirrors (engine.hpp:148-150, CellRT :89-115,
 * SynGroupRT :71-85).  `index` is the species index for MCG_FIELD_SPECIES and
 * the group index for per-synapse fields; count elements from `offset`. */
enum {
  MCG_FIELD_V = 0,            /* f64[ncomp]   CellRT::v_mV                  */
  MCG_FIELD_SPECIES = 1,      /* f64[ncomp]   CellRT::species[index]        */
  MCG_FIELD_HH_M = 2,         /* f64[ncomp]                                 */
  MCG_FIELD_HH_H = 3,
  MCG_FIELD_HH_N = 4,
  MCG_FIELD_DETECTOR_PREV_V = 5, /* f64[1]                                  */
  MCG_FIELD_REFRACTORY_UNTIL = 6, /* i64[1]                                 */
  MCG_FIELD_DETECTOR_ARMED = 7,   /* i64[1]                                 */
  MCG_FIELD_SYN_COMP = 8,     /* i32[size]   SynGroupRT::comp               */
  MCG_FIELD_SYN_WEIGHT = 9,   /* f64[size]   SynGroupRT::weight             */
  MCG_FIELD_SYN_KERNEL = 10,  /* f64[size]   SynGroupRT::kernel             */
  MCG_FIELD_STDP_A_PRE = 11,  /* f64[size]   StdpState::a_pre               */
  MCG_FIELD_STDP_A_POST = 12,
  MCG_FIELD_STDP_W = 13,
  MCG_FIELD_STDP_LAST = 14,   /* i64[size]   SynGroupRT::stdp_last_step     */
  MCG_FIELD_HOMEO_W = 15,     /* f64[size]   HomeostasisState::w            */
  MCG_FIELD_STC_H = 16,       /* f64[size]   StcState::h                    */
  MCG_FIELD_STC_Z = 17,
  MCG_FIELD_STC_C = 18,
  MCG_FIELD_STC_SPS_ABS = 19, /* f64[size]   SynGroupRT::sps_abs            */
  MCG_FIELD_INTERNAL_SEQ = 20 /* i64[1]      CellRT::internal_seq           */
};
int32_t mcg_cell_ncomp(const mcg_engine* eng, uint32_t gid);
int32_t mcg_cell_ngroups(const mcg_engine* eng, uint32_t gid);
int64_t mcg_group_size(const mcg_engine* eng, uint32_t gid, int32_t group);
int32_t mcg_cell_parent(const mcg_engine* eng, uint32_t gid, int32_t comp);
mcg_status mcg_read_state(mcg_engine* eng, int32_t field, uint32_t gid, int32_t index,
                          int64_t offset, int64_t count, void* out);
mcg_status mcg_write_state(mcg_engine* eng, int32_t field, uint32_t gid, int32_t index,
                           int64_t offset, int64_t count, const void* in);

/* ---- sharded epoch loop (world > 1) ---------------------------------------
 * The reference's epoch loop (engine.cpp:913-942) with cells partitioned over
 * ranks (contiguous gid ranges balanced by compartments + synapses; each rank
 * owns its cells and their incoming synapses).  Per epoch the caller runs
 *   mcg_shard_run_epoch     expands the spikes in `recv` (all ranks' send
 *                           blocks of the previous epoch) through this rank's
 *                           incoming edges, steps one min-delay epoch towards
 *                           t_ms, writes this rank's spikes into `send`
 *   allgather(send -> recv) e.g. ncclAllGather / torch.distributed
 * Blocks are int64[1 + 3*block_cap] = [count, (gid, step, t) x block_cap]
 * (t: the interpolated spike time's IEEE bits; every rank can rebuild the
 * global spike list, epoch by epoch, sorted by (gid, step)), the
 * same block_cap on every rank (>= mcg_shard_spike_cap of every rank); `recv`
 * holds `world` blocks in rank order and must be zero-initialised before the
 * first epoch.  Both are device pointers; the engine synchronizes its stream
 * before returning.  Replaces Impl::exchange (engine.cpp:875-889). */
int64_t mcg_shard_spike_cap(const mcg_engine* eng);   /* max local spikes per epoch */
uint32_t mcg_shard_gid_begin(const mcg_engine* eng);  /* local gid range [begin, end) */
uint32_t mcg_shard_gid_end(const mcg_engine* eng);
mcg_status mcg_shard_set_buffers(mcg_engine* eng, int64_t* send, int64_t* recv, int64_t block_cap,
                                 int32_t world);
mcg_status mcg_shard_run_epoch(mcg_engine* eng, double t_ms);
/* The same loop with the exchange inside the library: mcg_shard_init_nccl
 * creates an NCCL communicator of mcg_options.world ranks (this engine is
 * mcg_options.rank) from an id made by mcg_nccl_unique_id on one rank and
 * shared by the caller (any transport), and allocates the blocks on the
 * engine's device.  mcg_shard_advance_to then runs every epoch up to t_ms as
 * one stepping launch + ncclAllGather on the engine's stream, with one host
 * wait per 32 epochs (inboxes are sized so that no epoch can overflow them;
 * MCG_SHARD_SYNC=1 waits every epoch).  Every rank keeps the global spike
 * list (all ranks' spikes, the reference's (epoch, gid, step) order);
 * mcg_num_spikes / mcg_get_spikes keep returning this rank's own spikes.
 * libnccl.so.2 is loaded at run time (dlopen).  Replaces the worker pool's
 * barrier + Impl::exchange (engine.cpp:926-942, 875-889). */
mcg_status mcg_nccl_unique_id(uint8_t id[128]);
mcg_status mcg_shard_init_nccl(mcg_engine* eng, const uint8_t id[128]);
mcg_status mcg_shard_advance_to(mcg_engine* eng, double t_ms);
int64_t mcg_shard_num_global_spikes(const mcg_engine* eng);
mcg_status mcg_shard_get_global_spikes(mcg_engine* eng, int64_t first, int64_t count, double* t_ms,
                                       uint32_t* gid);
/* the shard bounds mcg_create uses for (recipe, world): rank r owns gids
 * [bounds[r], bounds[r+1]); bounds has world + 1 entries.  Host only (no GPU). */
mcg_status mcg_partition(const mcg_recipe* recipe, int32_t world, uint32_t* bounds);
/* Host only (no GPU): run the recipe -> runtime build (Impl::build,
 * engine.cpp:189-408) with `threads` host threads (<= 0: the default) and
 * return a digest of the resulting layout (edges in rank order, instances,
 * CSR, queues): out = {FNV-1a hash, edges, instances, min_delay_steps}.
 * Errors are the build's (the reference's messages, first failing connection
 * first).  Used to check that the threaded build is independent of the
 * thread count. */
mcg_status mcg_build_digest(const mcg_recipe* recipe, const mcg_options* opt, int32_t threads,
                            uint64_t out[4]);

/* The same digest from a constructed engine's own layout: the edge records
 * and instances its build resolved (on the device for recipes without STDP
 * placements: mcg_resolve.cuh, engine.cpp:357-391).  Equal to
 * mcg_build_digest of the same recipe and options.  Host-side check only
 * (downloads the edge records). */
mcg_status mcg_engine_layout_digest(mcg_engine* eng, uint64_t out[4]);

/* ---- instrumentation (bench.py) -------------------------------------------- */

typedef struct {
  int64_t epochs;             /* epochs run since creation                    */
  int64_t steps;              /* fine steps advanced                          */
  int64_t kernel_launches;    /* device kernel launches issued by the engine  */
  int64_t events_delivered;   /* EventRecs consumed by apply_event            */
  double epoch_kernel_ms;     /* summed CUDA-event time of the epoch kernel   */
  int64_t epoch_kernel_launches;
  int64_t total_comps;        /* sum of compartments over local cells         */
  int64_t total_synapses;     /* synapse instances over local cells           */
  int64_t stc_synapses;
  int64_t hh_comps;           /* compartments carrying HH channels            */
  int64_t species_comps;      /* sum over cells of species x compartments     */
  double advance_ms;          /* CUDA-event time of advance_to calls (engine stream) */
  int64_t advance_calls;
  int32_t stepping_kernel;    /* 0: k_batch, 1: k_warp, 2: k_point (mcg_engine.cu) */
  int32_t edges_on_device;    /* 1: connections resolved on the device (mcg_resolve.cuh) */
} mcg_stats;
mcg_status mcg_get_stats(mcg_engine* eng, mcg_stats* out);
/* enable/disable CUDA-event timing of the epoch kernel (adds one event pair per epoch) */
mcg_status mcg_set_timing(mcg_engine* eng, int32_t enabled);
/* Independent trials in one engine (the stc-protocols experiment,
 * experiments.cpp:262-289, runs run_stc_protocol(cfg, p, t) for t < trials,
 * each an Engine with seed cfg.seed + t and one cell, gid 0): cell c of this
 * engine draws its random numbers with the key (seeds[c], key_gids[c], ...)
 * instead of (options.seed, c, ...).  seeds / key_gids have one entry per
 * cell.  Only for the point-cell kernel (k_point): MCG_ERR_ENGINE otherwise.
 * Not part of mcsim::Engine; protocols.run_stc_protocols uses it. */
mcg_status mcg_set_cell_rng(mcg_engine* eng, const uint64_t* seeds, const uint32_t* key_gids);

/* ---- device numerics (differential tests of the glibc-faithful ports) ---- */

enum { MCG_MATH_EXP = 0, MCG_MATH_LOG = 1, MCG_MATH_SIN = 2, MCG_MATH_COS = 3,
       MCG_MATH_UNIFORM_FOR = 4, MCG_MATH_NORMAL_FOR = 5 };
/* out[i] = f(in[i]) evaluated on the device.  For the RNG functions in[] is
 * ignored and out[i] = uniform_for/normal_for(key, n0 + i) (rng.cpp:67-84). */
mcg_status mcg_device_math(int32_t device, int32_t func, const double* in, int64_t n,
                           const uint64_t key[4], uint64_t n0, double* out);

/* ---- host libm pin (bitwise parity precondition) ----------------------- */

/* Checks that the libm.so.6 mapped into this process is the glibc build the
 * device ports were written against (build-id 0d9969fe…, glibc 2.39-0ubuntu8.5),
 * that the CPU has FMA + AVX2 (glibc's ifunc then selects the FMA variants the
 * ports follow), and that the host build of the ports agrees bit for bit with
 * the live exp/log/sincos on `samples` pseudo-random arguments per range
 * (<= 0: 20000).  The reference's libm calls (engine.cpp:44-54, :582-719,
 * rng.cpp:62-64) produce the engine's results only when this returns MCG_OK.
 * A one-line report is written to report[0..cap). */
mcg_status mcg_libm_check(int64_t samples, char* report, int64_t cap);

/* ---- recipe materialization on the device --------- */

/* Directed Erdos-Renyi sample of er_connected (network.cpp:34-39):
 * pair (i, j), i != j, is connected iff uniform_for(key(seed,0,17,0), i*n+j) < p.
 * Pairs are produced in the reference builder's loop order (i outer, j inner,
 * network.cpp:548-550) for sources i in [src_begin, src_end).  Call with
 * src == NULL to get the count in *count; then with arrays of that size. */
mcg_status mcg_er_connect(int32_t device, uint64_t seed, uint32_t n, double p, uint32_t src_begin,
                          uint32_t src_end, uint32_t* src, uint32_t* dst, int64_t* count);

/* ---- checkpoints ----------------------------------- */

/* Engine::make_checkpoint + Checkpoint::serialize (engine.cpp:1070-1093,
 * 1150-1233): the engine's state as MCSCKPT1 bytes, byte-identical to the
 * reference's for the same run.  buf == NULL: *size only. */
mcg_status mcg_checkpoint(mcg_engine* eng, uint8_t* buf, int64_t cap, int64_t* size);
/* Checkpoint::deserialize + Engine::restore (engine.cpp:1095-1140, 1235-1325);
 * accepts the reference's checkpoints (same validation and messages). */
mcg_status mcg_restore(mcg_engine* eng, const uint8_t* buf, int64_t size);

/* ---- standalone protocol drivers ------------------- */

/* GbParams (mechanisms.hpp:80-92), field order as the reference's aggregate */
typedef struct {
  double tau_w_ms, w_star, gamma_p, gamma_d, theta_p, theta_d, sigma_pl, tau_c_ms;
  double c_pre, c_post, t_c_delay_ms;
} mcg_gb_params;
/* GbPairingProtocol (mechanisms.hpp:276-283) */
typedef struct {
  int32_t n_pairs;
  int32_t trials;
  double period_ms, settle_ms, dt_ms;
  uint64_t seed;
} mcg_gb_protocol;
/* GbCurvePoint (mechanisms.hpp:285-292) */
typedef struct {
  double delta_t_ms, mean_initial, mean_final, mean_change, change_ci_half, ratio;
} mcg_gb_point;
/* Every pairing trial of gb_pairing_trial (mechanisms.cpp:40-90) on the device,
 * one thread per (delta, trial): w0[d * trials + t] and wf[...] are the initial
 * and final weights of trial t at deltas[d] (delta_index = d). */
mcg_status mcg_gb_trials(int32_t device, const mcg_gb_params* p, const double* deltas,
                         int32_t n_deltas, const mcg_gb_protocol* proto, double* w0, double* wf);
/* gb_dp_curve (mechanisms.cpp:92-119): the trials on the device, the per-delta
 * means and confidence intervals (mean_ci, analysis.cpp:82-94) on the host in
 * the reference's summation order. */
mcg_status mcg_gb_dp_curve(int32_t device, const mcg_gb_params* p, const double* deltas,
                           int32_t n_deltas, const mcg_gb_protocol* proto, mcg_gb_point* out);
/* stdp_window (mechanisms.cpp:9-38) for n deltas, one thread per delta:
 * out[i] = weight change per pair at deltas[i]. */
mcg_status mcg_stdp_window(int32_t device, const mcg_stdp_params* p, const double* deltas,
                           int32_t n, int32_t n_pairs, double period_ms, double* out);

#ifdef __cplusplus
}
#endif
#endif /* MCG_H */
