"""Field-by-field comparison of two flat recipes (include/mcg.h mcg_recipe)."""
import numpy as np

from paper_2411_16445_b200 import _abi as A


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def _struct_dict(s):
    out = {}
    for f, t in s._fields_:
        v = getattr(s, f)
        if hasattr(v, "_fields_"):
            out[f] = _struct_dict(v)
        elif not hasattr(t, "contents"):
            out[f] = v
    return out


def assert_recipes_equal(a, b):
    assert a.n_kinds == b.n_kinds
    assert a.n_cells == b.n_cells
    np.testing.assert_array_equal(_arr(a.cell_kind, a.n_cells, np.uint32),
                                  _arr(b.cell_kind, b.n_cells, np.uint32))
    for k in range(a.n_kinds):
        ka, kb = a.kinds[k], b.kinds[k]
        assert ka.n_segments == kb.n_segments, f"kind {k}"
        for f, dt in (("seg_parent", np.int32), ("seg_length_um", np.float64),
                      ("seg_radius_um", np.float64), ("seg_tag", np.uint8),
                      ("seg_parent_pos", np.float64)):
            np.testing.assert_array_equal(_arr(getattr(ka, f), ka.n_segments, dt),
                                          _arr(getattr(kb, f), kb.n_segments, dt),
                                          err_msg=f"kind {k} {f}")
        for f in ("target_compartment_um", "membrane", "n_species", "sps_idx", "prp_idx",
                  "n_placements", "prp_enabled", "prp_comp"):
            assert getattr(ka, f) == getattr(kb, f), f"kind {k} {f}"
        if ka.membrane == 1:
            assert _struct_dict(ka.lif) == _struct_dict(kb.lif), f"kind {k} lif"
        if ka.membrane == 2:
            assert _struct_dict(ka.hh) == _struct_dict(kb.hh), f"kind {k} hh"
        for s in range(ka.n_species):
            assert _struct_dict(ka.species[s]) == _struct_dict(kb.species[s]), f"kind {k} sp {s}"
        for p in range(ka.n_placements):
            assert _struct_dict(ka.placements[p]) == _struct_dict(kb.placements[p]), \
                f"kind {k} placement {p}"
    assert a.n_sources == b.n_sources
    for s in range(a.n_sources):
        sa, sb = a.sources[s], b.sources[s]
        assert (sa.type, sa.n_values) == (sb.type, sb.n_values), f"source {s}"
        np.testing.assert_array_equal(_arr(sa.values, sa.n_values, np.float64),
                                      _arr(sb.values, sb.n_values, np.float64))
        assert (sa.t0_ms, sa.period_ms, sa.count) == (sb.t0_ms, sb.period_ms, sb.count)
    assert a.n_connections == b.n_connections
    n = a.n_connections
    for f, dt in (("conn_from_source", np.uint8), ("conn_src", np.uint32), ("conn_dst", np.uint32),
                  ("conn_group", np.int32), ("conn_policy", np.uint8),
                  ("conn_weight", np.float64), ("conn_delay_ms", np.float64)):
        np.testing.assert_array_equal(_arr(getattr(a, f), n, dt), _arr(getattr(b, f), n, dt),
                                      err_msg=f)
    assert a.n_probes == b.n_probes
