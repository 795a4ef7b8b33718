"""TEST INFRASTRUCTURE — the parity oracle, never part of the product path.

ctypes access to the UNMODIFIED reference simulator (mcsim, compiled from
/root/reference/proj/src by oracle/build_ref.sh into oracle/_ref/) through
oracle/ref_shim.cpp.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs may import this module.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libmcsim_ref.so")

import sys  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
from paper_2411_16445_b200 import _abi as A  # noqa: E402  (struct mirrors only)


class ref_consolidation_cfg(C.Structure):  # network.hpp:152-196
    _fields_ = [("n_cells", C.c_int32), ("n_exc", C.c_int32), ("p_conn", C.c_double),
                ("pattern", C.c_int32), ("seed", C.c_uint64), ("workers", C.c_int32),
                ("dt_ms", C.c_double), ("multi_compartment", C.c_int32),
                ("cell_size", C.c_int32), ("dend_size", C.c_int32), ("d_p", C.c_double),
                ("d_sps", C.c_double), ("stc", A.mcg_stc_params), ("in_vivo_factor", C.c_double)] + [
        (n, C.c_double) for n in (
            "tau_mem_ms", "r_mem_MOhm", "v_rev_mV", "v_reset_mV", "v_thresh_mV", "t_ref_ms",
            "i_bg_nA", "sigma_bg_nA_sqrt_ms", "w_rec_scale", "w_ei_mV", "w_ie_mV", "w_ii_mV",
            "delay_ms")] + [("n_stim_sources", C.c_int32)] + [
        (n, C.c_double) for n in (
            "t_learn_ms", "learn_duration_ms", "learn_rate_hz", "recall_duration_ms",
            "recall_rate_hz", "w_stim_mV", "coarse_dt_ms")]


class ref_busyring_cfg(C.Structure):  # bench.hpp:20-34
    _fields_ = [("n_cells", C.c_int32), ("ring_size", C.c_int32), ("random_per_cell", C.c_int32),
                ("delay_ms", C.c_double), ("ring_weight_uS", C.c_double),
                ("tau_syn_ms", C.c_double), ("tree_depth", C.c_int32),
                ("stdp_on_random", C.c_int32), ("stdp", A.mcg_stdp_params),
                ("duration_ms", C.c_double), ("dt_ms", C.c_double), ("seed", C.c_uint64),
                ("workers", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run oracle/build_ref.sh")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        vp = C.c_void_p
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_default_consolidation": (None, [P(ref_consolidation_cfg)]),
            "ref_default_busyring": (None, [P(ref_busyring_cfg)]),
            "ref_default_stc_params": (None, [P(A.mcg_stc_params)]),
            "ref_build_consolidation": (C.c_int, [P(ref_consolidation_cfg), C.c_int, P(vp)]),
            "ref_build_busyring": (C.c_int, [P(ref_busyring_cfg), P(vp)]),
            "ref_calibrate_ring_weight": (C.c_double, [P(ref_busyring_cfg)]),
            "ref_recipe_from_flat": (C.c_int, [P(A.mcg_recipe), P(vp)]),
            "ref_recipe_view": (P(A.mcg_recipe), [vp]),
            "ref_recipe_label": (C.c_char_p, [vp, C.c_int, C.c_int]),
            "ref_recipe_c_morpho": (C.c_double, [vp]),
            "ref_recipe_destroy": (None, [vp]),
            "ref_engine_create": (C.c_int, [P(A.mcg_recipe), C.c_double, C.c_uint64, C.c_int,
                                            P(vp)]),
            "ref_engine_destroy": (None, [vp]),
            "ref_advance_to": (C.c_int, [vp, C.c_double]),
            "ref_fast_forward_to": (C.c_int, [vp, C.c_double, C.c_double]),
            "ref_step": (C.c_int64, [vp]),
            "ref_time_ms": (C.c_double, [vp]),
            "ref_num_spikes": (C.c_int64, [vp]),
            "ref_get_spikes": (None, [vp, vp, vp]),
            "ref_clear_spikes": (None, [vp]),
            "ref_trace_len": (C.c_int64, [vp, C.c_int]),
            "ref_get_trace": (None, [vp, C.c_int, vp, vp]),
            "ref_cell_ncomp": (C.c_int32, [vp, C.c_uint32]),
            "ref_cell_ngroups": (C.c_int32, [vp, C.c_uint32]),
            "ref_group_size": (C.c_int64, [vp, C.c_uint32, C.c_int32]),
            "ref_cell_parent": (C.c_int32, [vp, C.c_uint32, C.c_int32]),
            "ref_read_state": (C.c_int, [vp, C.c_int, C.c_uint32, C.c_int, C.c_int64, C.c_int64,
                                         vp]),
            "ref_threefry": (None, [P(C.c_uint64), P(C.c_uint64), P(C.c_uint64)]),
            "ref_uniform_for": (C.c_double, [P(C.c_uint64), C.c_uint64]),
            "ref_normal_for": (C.c_double, [P(C.c_uint64), C.c_uint64]),
            "ref_er_connected": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_double]),
            "ref_solve_tree": (C.c_int, [C.c_int, vp, vp, vp, vp, vp, vp]),
            "ref_discretize": (C.c_int, [P(A.mcg_kind), C.c_int, vp, vp, vp, vp, vp]),
            "ref_run_stc_protocol": (C.c_int, [C.c_int, C.c_uint64, P(C.c_double),
                                               P(C.c_double), P(C.c_double)]),
            "ref_gb_pairing_trial": (C.c_double, [P(A.mcg_gb_params), C.c_double,
                                                  P(A.mcg_gb_protocol), C.c_uint64, C.c_uint64,
                                                  P(C.c_double)]),
            "ref_gb_dp_curve": (C.c_int, [P(A.mcg_gb_params), vp, C.c_int, P(A.mcg_gb_protocol),
                                          vp]),
            "ref_stdp_window": (C.c_double, [P(A.mcg_stdp_params), C.c_double, C.c_int,
                                             C.c_double]),
            "ref_make_checkpoint": (C.c_int, [vp, vp, C.c_int64, P(C.c_int64)]),
            "ref_write_v": (C.c_int, [vp, C.c_uint32, vp, C.c_int64]),
            "ref_restore": (C.c_int, [vp, vp, C.c_int64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _chk(st):
    if st != 0:
        raise RefError(st, lib().ref_last_error().decode())


def default_consolidation(**kw) -> ref_consolidation_cfg:
    c = ref_consolidation_cfg()
    lib().ref_default_consolidation(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def default_busyring(**kw) -> ref_busyring_cfg:
    c = ref_busyring_cfg()
    lib().ref_default_busyring(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class RefRecipe:
    """A recipe built by the reference's own builder, exported flat (mcg.h)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def consolidation(cls, cfg: ref_consolidation_cfg, eight_hour=False):
        h = C.c_void_p()
        _chk(lib().ref_build_consolidation(C.byref(cfg), 1 if eight_hour else 0, C.byref(h)))
        return cls(h)

    @classmethod
    def busyring(cls, cfg: ref_busyring_cfg):
        h = C.c_void_p()
        _chk(lib().ref_build_busyring(C.byref(cfg), C.byref(h)))
        return cls(h)

    @classmethod
    def from_flat(cls, view):
        h = C.c_void_p()
        _chk(lib().ref_recipe_from_flat(C.byref(view), C.byref(h)))
        return cls(h)

    @property
    def view(self):
        return lib().ref_recipe_view(self._h).contents

    def label(self, kind, placement):
        return lib().ref_recipe_label(self._h, kind, placement).decode()

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_recipe_destroy(self._h)
            self._h = None


class RefEngine:
    """The reference's mcsim::Engine driven through the shim."""

    def __init__(self, view, dt_ms, seed, workers=1):
        self._view = view
        h = C.c_void_p()
        _chk(lib().ref_engine_create(C.byref(view), dt_ms, seed, workers, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_engine_destroy(self._h)
            self._h = None

    def advance_to(self, t):
        _chk(lib().ref_advance_to(self._h, t))

    def fast_forward_to(self, t, c):
        _chk(lib().ref_fast_forward_to(self._h, t, c))

    def step(self):
        return lib().ref_step(self._h)

    def time_ms(self):
        return lib().ref_time_ms(self._h)

    def spike_arrays(self):
        n = lib().ref_num_spikes(self._h)
        t = np.empty(n, np.float64)
        g = np.empty(n, np.uint32)
        if n:
            lib().ref_get_spikes(self._h, t.ctypes.data, g.ctypes.data)
        return t, g

    def clear_spikes(self):
        lib().ref_clear_spikes(self._h)

    def write_v(self, gid, values):
        a = np.ascontiguousarray(values, np.float64)
        _chk(lib().ref_write_v(self._h, gid, a.ctypes.data, a.size))

    def make_checkpoint(self) -> bytes:
        n = C.c_int64()
        _chk(lib().ref_make_checkpoint(self._h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * max(n.value, 1))()
        _chk(lib().ref_make_checkpoint(self._h, buf, n.value, C.byref(n)))
        return bytes(buf)[:n.value]

    def restore(self, data: bytes):
        buf = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(bytes(data) or b"\0")
        _chk(lib().ref_restore(self._h, buf, len(data)))

    def trace_arrays(self, p):
        n = lib().ref_trace_len(self._h, p)
        t = np.empty(n, np.float64)
        v = np.empty(n, np.float64)
        if n:
            lib().ref_get_trace(self._h, p, t.ctypes.data, v.ctypes.data)
        return t, v

    def ncomp(self, gid):
        return lib().ref_cell_ncomp(self._h, gid)

    def ngroups(self, gid):
        return lib().ref_cell_ngroups(self._h, gid)

    def group_size(self, gid, g):
        return lib().ref_group_size(self._h, gid, g)

    def read(self, field, gid, index=0, count=None, dtype=np.float64):
        fid = A.FIELD[field]
        if count is None:
            if fid in (0, 1, 2, 3, 4):
                count = self.ncomp(gid)
            elif fid in (5, 6, 7, 20):
                count = 1
            else:
                count = self.group_size(gid, index)
        out = np.empty(count, dtype)
        if count:
            _chk(lib().ref_read_state(self._h, fid, gid, index, 0, count, out.ctypes.data))
        return out


def key_arr(k):
    return (C.c_uint64 * 4)(*[int(x) & (2**64 - 1) for x in k])


def threefry(key, ctr):
    out = (C.c_uint64 * 4)()
    lib().ref_threefry(key_arr(key), key_arr(ctr), out)
    return list(out)


def uniform_for(key, n):
    return lib().ref_uniform_for(key_arr(key), n)


def normal_for(key, n):
    return lib().ref_normal_for(key_arr(key), n)


def er_connected(seed, src, dst, n, p):
    return bool(lib().ref_er_connected(seed, src, dst, n, p))


def solve_tree(parent, cap, g, coupling, rhs, v):
    parent = np.ascontiguousarray(parent, np.int32)
    arrs = [np.ascontiguousarray(a, np.float64) for a in (cap, g, coupling, rhs)]
    v = np.array(v, np.float64)
    _chk(lib().ref_solve_tree(len(parent), parent.ctypes.data, *[a.ctypes.data for a in arrs],
                              v.ctypes.data))
    return v


def run_stc_protocol(proto, trial):
    h, z, p = C.c_double(), C.c_double(), C.c_double()
    _chk(lib().ref_run_stc_protocol(proto, trial, C.byref(h), C.byref(z), C.byref(p)))
    return h.value, z.value, p.value


# ---- protocol drivers (mechanisms.cpp:9-119), the reference's own functions
def _gb_structs(p, proto):
    from dataclasses import fields
    from paper_2411_16445_b200.protocols import GbParams
    cp = A.mcg_gb_params(*[float(getattr(p, f.name)) for f in fields(GbParams)])
    cq = A.mcg_gb_protocol(int(proto.n_pairs), int(proto.trials), float(proto.period_ms),
                           float(proto.settle_ms), float(proto.dt_ms), int(proto.seed))
    return cp, cq


def gb_pairing_trial(p, delta_t_ms, proto, trial, delta_index=0):
    """(final w, w0) of the reference's gb_pairing_trial."""
    cp, cq = _gb_structs(p, proto)
    w0 = C.c_double()
    wf = lib().ref_gb_pairing_trial(C.byref(cp), float(delta_t_ms), C.byref(cq), trial,
                                    delta_index, C.byref(w0))
    return wf, w0.value


def gb_dp_curve(p, deltas, proto):
    """The reference's gb_dp_curve as a list of 6-tuples (GbCurvePoint fields)."""
    cp, cq = _gb_structs(p, proto)
    d = np.ascontiguousarray(deltas, np.float64)
    out = (A.mcg_gb_point * max(d.size, 1))()
    _chk(lib().ref_gb_dp_curve(C.byref(cp), d.ctypes.data, d.size, C.byref(cq), out))
    return [tuple(getattr(out[i], f) for f, _ in A.mcg_gb_point._fields_) for i in range(d.size)]


def stdp_window(delta_t_ms, p=None, n_pairs=60, period_ms=1000.0):
    from paper_2411_16445_b200.recipe import StdpParams
    p = p or StdpParams()
    cp = A.mcg_stdp_params(p.tau_pre_ms, p.tau_post_ms, p.a_pre_uS, p.a_post_uS, p.w0_uS,
                           p.wmax_uS)
    return lib().ref_stdp_window(C.byref(cp), float(delta_t_ms), int(n_pairs), float(period_ms))


# the reference's CSV writers (csvio.cpp) run as a small executable built from
# its own sources (oracle/ref_csv.cpp): in-process iostreams of the statically
# linked C++ runtime of libmcsim_ref.so do not survive inside Python
CSV_EXE = os.path.join(os.path.dirname(LIB_PATH), "ref_csv")


def _ref_csv(kind, path, a, b, b_dtype):
    import subprocess
    import tempfile
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, b_dtype)
    with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as f:
        f.write(np.int64(a.size).tobytes() + a.tobytes() + b.tobytes())
        name = f.name
    try:
        subprocess.run([CSV_EXE, kind, name, path], check=True)
    finally:
        os.unlink(name)


def write_spikes_csv(path, t_s, gid):
    _ref_csv("spikes", path, t_s, gid, np.uint32)


def write_trace_csv(path, t_s, v):
    _ref_csv("trace", path, t_s, v, np.float64)
