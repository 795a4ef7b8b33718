"""ctypes mirror of include/mcg.h (the engine's C ABI).

Every structure here is field-for-field the C declaration; the library is
`paper_2411_16445_b200/libmcg.so`, built in-tree by `_build.py` for sm_100a.
There is no fallback: if the library is missing, `lib()` raises.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCG_LIB") or os.path.join(_HERE, "libmcg.so")

# status codes
MCG_OK = 0
MCG_ERR_ENGINE = 1
MCG_ERR_NUMERIC = 2
MCG_ERR_TARGETING = 3
MCG_ERR_MORPHOLOGY = 4
MCG_ERR_CUDA = 5
MCG_ERR_ARGUMENT = 6


class mcg_lif(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "tau_mem_ms", "r_mem_MOhm", "v_rev_mV", "v_reset_mV", "v_thresh_mV", "t_ref_ms",
        "r_axial_ohm_m", "i_bg_nA", "sigma_bg_nA_sqrt_ms", "bg_quiet_t0_ms", "bg_quiet_t1_ms")] + [
        ("noise_comp", C.c_int32), ("detector_comp", C.c_int32), ("exact", C.c_int32)]


class mcg_hh(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "c_m", "r_axial_ohm_m", "g_leak", "e_leak_mV", "g_na", "e_na_mV", "g_k", "e_k_mV",
        "v_init_mV", "threshold_mV")] + [("detector_comp", C.c_int32)]


class mcg_species(C.Structure):
    _fields_ = [("diffusivity", C.c_double), ("decay_tau_ms", C.c_double), ("init", C.c_double)]


class mcg_stdp_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "tau_pre_ms", "tau_post_ms", "a_pre_uS", "a_post_uS", "w0_uS", "wmax_uS")]


class mcg_homeo_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "dw_plus_nA", "dw_minus_nA", "w_init_nA", "wmax_nA", "w_varying_nA")]


STC_FIELDS = ("h0_mV", "tau_h_ms", "tau_c_ms", "gamma_p", "gamma_d", "theta_p", "theta_d",
              "sigma_pl_mV", "c_pre", "c_post", "t_c_delay_ms", "tau_z_ms", "f_int",
              "theta_tag_mV", "tau_p_ms", "p_max", "theta_pro_mV")


class mcg_stc_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in STC_FIELDS]


class mcg_syn_spec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("tau_syn_ms", C.c_double), ("e_rev_mV", C.c_double),
                ("stdp", mcg_stdp_params), ("homeo", mcg_homeo_params), ("stc", mcg_stc_params),
                ("calcium_scale", C.c_double)]


class mcg_placement(C.Structure):
    _fields_ = [("syn", mcg_syn_spec), ("comp", C.c_int32), ("count", C.c_int32)]


class mcg_kind(C.Structure):
    _fields_ = [("n_segments", C.c_int32), ("seg_parent", C.POINTER(C.c_int32)),
                ("seg_length_um", C.POINTER(C.c_double)), ("seg_radius_um", C.POINTER(C.c_double)),
                ("seg_tag", C.POINTER(C.c_uint8)), ("seg_parent_pos", C.POINTER(C.c_double)),
                ("target_compartment_um", C.c_double), ("membrane", C.c_int32),
                ("lif", mcg_lif), ("hh", mcg_hh), ("n_species", C.c_int32),
                ("species", C.POINTER(mcg_species)), ("sps_idx", C.c_int32),
                ("prp_idx", C.c_int32), ("n_placements", C.c_int32),
                ("placements", C.POINTER(mcg_placement)), ("prp_enabled", C.c_int32),
                ("prp_comp", C.c_int32)]


class mcg_source(C.Structure):
    _fields_ = [("type", C.c_int32), ("n_values", C.c_int32), ("values", C.POINTER(C.c_double)),
                ("t0_ms", C.c_double), ("period_ms", C.c_double), ("count", C.c_int64)]


class mcg_recipe(C.Structure):
    _fields_ = [("n_kinds", C.c_int32), ("kinds", C.POINTER(mcg_kind)),
                ("n_cells", C.c_int32), ("cell_kind", C.POINTER(C.c_uint32)),
                ("n_sources", C.c_int32), ("sources", C.POINTER(mcg_source)),
                ("n_connections", C.c_int64),
                ("conn_from_source", C.POINTER(C.c_uint8)), ("conn_src", C.POINTER(C.c_uint32)),
                ("conn_dst", C.POINTER(C.c_uint32)), ("conn_group", C.POINTER(C.c_int32)),
                ("conn_policy", C.POINTER(C.c_uint8)), ("conn_weight", C.POINTER(C.c_double)),
                ("conn_delay_ms", C.POINTER(C.c_double)),
                ("n_probes", C.c_int32), ("probe_gid", C.POINTER(C.c_uint32)),
                ("probe_what", C.POINTER(C.c_uint8)), ("probe_comp", C.POINTER(C.c_int32)),
                ("probe_species", C.POINTER(C.c_int32)), ("probe_group", C.POINTER(C.c_int32)),
                ("probe_instance", C.POINTER(C.c_int32)), ("probe_every", C.POINTER(C.c_int32)),
                ("n_labels", C.c_int32), ("labels", C.POINTER(C.c_char_p)),
                ("conn_label", C.POINTER(C.c_int32))]


class mcg_options(C.Structure):
    _fields_ = [("dt_ms", C.c_double), ("seed", C.c_uint64), ("workers", C.c_int32),
                ("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32)]


class mcg_stats(C.Structure):
    _fields_ = [("epochs", C.c_int64), ("steps", C.c_int64), ("kernel_launches", C.c_int64),
                ("events_delivered", C.c_int64), ("epoch_kernel_ms", C.c_double),
                ("epoch_kernel_launches", C.c_int64), ("total_comps", C.c_int64),
                ("total_synapses", C.c_int64), ("stc_synapses", C.c_int64),
                ("hh_comps", C.c_int64), ("species_comps", C.c_int64),
                ("advance_ms", C.c_double), ("advance_calls", C.c_int64),
                ("stepping_kernel", C.c_int32), ("edges_on_device", C.c_int32)]


class mcg_gb_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("tau_w_ms", "w_star", "gamma_p", "gamma_d", "theta_p",
                                          "theta_d", "sigma_pl", "tau_c_ms", "c_pre", "c_post",
                                          "t_c_delay_ms")]


class mcg_gb_protocol(C.Structure):
    _fields_ = [("n_pairs", C.c_int32), ("trials", C.c_int32), ("period_ms", C.c_double),
                ("settle_ms", C.c_double), ("dt_ms", C.c_double), ("seed", C.c_uint64)]


class mcg_gb_point(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("delta_t_ms", "mean_initial", "mean_final",
                                          "mean_change", "change_ci_half", "ratio")]


# field ids (mcg.h)
FIELD = dict(v=0, species=1, hh_m=2, hh_h=3, hh_n=4, detector_prev_v=5, refractory_until=6,
             detector_armed=7, syn_comp=8, syn_weight=9, syn_kernel=10, stdp_a_pre=11,
             stdp_a_post=12, stdp_w=13, stdp_last=14, homeo_w=15, stc_h=16, stc_z=17, stc_c=18,
             stc_sps_abs=19, internal_seq=20)

# every symbol include/mcg.h declares (checked by tests/test_abi.py)
EXPORTS = ("mcg_create", "mcg_destroy", "mcg_last_error", "mcg_abi_version", "mcg_time_ms",
           "mcg_dt_ms", "mcg_step", "mcg_num_cells", "mcg_min_delay_steps", "mcg_advance_to",
           "mcg_fast_forward_to", "mcg_num_spikes", "mcg_get_spikes", "mcg_clear_spikes",
           "mcg_trace_len", "mcg_get_trace", "mcg_cell_ncomp", "mcg_cell_ngroups",
           "mcg_group_size", "mcg_cell_parent", "mcg_read_state", "mcg_write_state",
           "mcg_get_stats", "mcg_set_timing", "mcg_device_math",
           "mcg_er_connect", "mcg_build_digest", "mcg_engine_layout_digest", "mcg_set_cell_rng", "mcg_shard_spike_cap", "mcg_shard_gid_begin", "mcg_shard_gid_end",
           "mcg_shard_set_buffers", "mcg_shard_run_epoch", "mcg_partition",
           "mcg_gb_trials", "mcg_gb_dp_curve", "mcg_stdp_window", "mcg_checkpoint", "mcg_restore",
           "mcg_libm_check", "mcg_nccl_unique_id", "mcg_shard_init_nccl", "mcg_shard_advance_to",
           "mcg_shard_num_global_spikes", "mcg_shard_get_global_spikes")

_lib = None


def _declare(L):
    P = C.POINTER
    eng = C.c_void_p
    sig = {
        "mcg_create": (C.c_int32, [P(mcg_recipe), P(mcg_options), P(C.c_void_p)]),
        "mcg_destroy": (None, [eng]),
        "mcg_last_error": (C.c_char_p, []),
        "mcg_abi_version": (C.c_int32, []),
        "mcg_time_ms": (C.c_double, [eng]),
        "mcg_dt_ms": (C.c_double, [eng]),
        "mcg_step": (C.c_int64, [eng]),
        "mcg_num_cells": (C.c_int32, [eng]),
        "mcg_min_delay_steps": (C.c_int64, [eng]),
        "mcg_advance_to": (C.c_int32, [eng, C.c_double]),
        "mcg_fast_forward_to": (C.c_int32, [eng, C.c_double, C.c_double]),
        "mcg_num_spikes": (C.c_int64, [eng]),
        "mcg_get_spikes": (C.c_int32, [eng, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
        "mcg_clear_spikes": (C.c_int32, [eng]),
        "mcg_trace_len": (C.c_int64, [eng, C.c_int32]),
        "mcg_get_trace": (C.c_int32, [eng, C.c_int32, C.c_void_p, C.c_void_p]),
        "mcg_cell_ncomp": (C.c_int32, [eng, C.c_uint32]),
        "mcg_cell_ngroups": (C.c_int32, [eng, C.c_uint32]),
        "mcg_group_size": (C.c_int64, [eng, C.c_uint32, C.c_int32]),
        "mcg_cell_parent": (C.c_int32, [eng, C.c_uint32, C.c_int32]),
        "mcg_read_state": (C.c_int32, [eng, C.c_int32, C.c_uint32, C.c_int32, C.c_int64,
                                       C.c_int64, C.c_void_p]),
        "mcg_write_state": (C.c_int32, [eng, C.c_int32, C.c_uint32, C.c_int32, C.c_int64,
                                        C.c_int64, C.c_void_p]),
        "mcg_get_stats": (C.c_int32, [eng, P(mcg_stats)]),
        "mcg_set_timing": (C.c_int32, [eng, C.c_int32]),
        "mcg_device_math": (C.c_int32, [C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                        C.c_void_p, C.c_uint64, C.c_void_p]),
        "mcg_er_connect": (C.c_int32, [C.c_int32, C.c_uint64, C.c_uint32, C.c_double,
                                       C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                       P(C.c_int64)]),
        "mcg_shard_spike_cap": (C.c_int64, [eng]),
        "mcg_shard_gid_begin": (C.c_uint32, [eng]),
        "mcg_shard_gid_end": (C.c_uint32, [eng]),
        "mcg_shard_set_buffers": (C.c_int32, [eng, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32]),
        "mcg_shard_run_epoch": (C.c_int32, [eng, C.c_double]),
        "mcg_partition": (C.c_int32, [P(mcg_recipe), C.c_int32, C.c_void_p]),
        "mcg_build_digest": (C.c_int32, [P(mcg_recipe), P(mcg_options), C.c_int32, C.c_void_p]),
        "mcg_engine_layout_digest": (C.c_int32, [C.c_void_p, C.c_void_p]),
        "mcg_set_cell_rng": (C.c_int32, [eng, C.c_void_p, C.c_void_p]),
        "mcg_nccl_unique_id": (C.c_int32, [C.c_void_p]),
        "mcg_shard_init_nccl": (C.c_int32, [eng, C.c_void_p]),
        "mcg_shard_advance_to": (C.c_int32, [eng, C.c_double]),
        "mcg_shard_num_global_spikes": (C.c_int64, [eng]),
        "mcg_shard_get_global_spikes": (C.c_int32, [eng, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
        "mcg_checkpoint": (C.c_int32, [eng, C.c_void_p, C.c_int64, P(C.c_int64)]),
        "mcg_restore": (C.c_int32, [eng, C.c_void_p, C.c_int64]),
        "mcg_libm_check": (C.c_int32, [C.c_int64, C.c_char_p, C.c_int64]),
        "mcg_gb_trials": (C.c_int32, [C.c_int32, P(mcg_gb_params), C.c_void_p, C.c_int32,
                                      P(mcg_gb_protocol), C.c_void_p, C.c_void_p]),
        "mcg_gb_dp_curve": (C.c_int32, [C.c_int32, P(mcg_gb_params), C.c_void_p, C.c_int32,
                                        P(mcg_gb_protocol), C.c_void_p]),
        "mcg_stdp_window": (C.c_int32, [C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                        C.c_double, C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def lib():
    """The loaded engine library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} missing: build it with `python -m paper_2411_16445_b200._build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def libm_check(samples: int = 20000):
    """(ok, report): is this host's libm the glibc build the device ports
    follow (mcg_libm_check in include/mcg.h)?  Bitwise parity with a reference
    running on this host needs ok."""
    buf = C.create_string_buffer(512)
    st = lib().mcg_libm_check(samples, buf, len(buf))
    return st == 0, buf.value.decode()
