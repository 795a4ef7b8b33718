"""Engine — Python mirror of mcsim::Engine (engine.hpp:126-167) over the C ABI.

    eng = Engine(recipe, EngineOptions(dt_ms=0.5, seed=1))
    eng.advance_to(1000.0)
    eng.spikes()            # [SpikeRecord(t_ms, gid)] in the reference's order
    eng.cell(3).v_mV        # lazily read from HBM
    eng.fast_forward_to(t, coarse_dt_ms)

Every call goes through include/mcg.h into the sm_100a library; errors come
back as the reference's exception types with the reference's messages.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _abi as A
from .recipe import (EngineError, FlatRecipe, MorphologyError, NumericError, Recipe,
                     TargetingError)


@dataclass
class EngineOptions:  # engine.hpp:37-41
    dt_ms: float = 0.025
    seed: int = 0
    workers: int = 1


@dataclass
class SpikeRecord:  # engine.hpp:20-23
    t_ms: float
    gid: int


_ERR = {A.MCG_ERR_ENGINE: EngineError, A.MCG_ERR_NUMERIC: NumericError,
        A.MCG_ERR_TARGETING: TargetingError, A.MCG_ERR_MORPHOLOGY: MorphologyError}


def _check(status: int):
    if status != A.MCG_OK:
        msg = A.lib().mcg_last_error().decode()
        raise _ERR.get(status, RuntimeError)(msg)


class Checkpoint:
    """The reference's Checkpoint (engine.hpp:107-124): named f64 / u64 arrays,
    serialized as MCSCKPT1 (engine.cpp:1070-1148)."""

    MAGIC = b"MCSCKPT1"

    def __init__(self, data: bytes = b""):
        self.data = bytes(data)

    def serialize(self) -> bytes:
        return self.data

    @staticmethod
    def deserialize(data: bytes) -> Tuple[dict, dict]:
        """(f64, u64) name -> array, with the reference's validation and
        messages (EngineError)."""
        import struct
        d = bytes(data)
        if len(d) < 16 or d[:8] != Checkpoint.MAGIC:
            raise EngineError("checkpoint: bad magic")
        pos = 8

        def take(n):
            nonlocal pos
            if pos + n > len(d):
                raise EngineError("checkpoint: truncated")
            out = d[pos:pos + n]
            pos += n
            return out
        if struct.unpack("<I", take(4))[0] != 1:
            raise EngineError("checkpoint: version mismatch")
        if struct.unpack("<I", take(4))[0] != 0x01020304:
            raise EngineError("checkpoint: endianness mismatch")
        f64, u64 = {}, {}
        while pos < len(d):
            nlen = struct.unpack("<I", take(4))[0]
            name = take(nlen).decode()
            if pos >= len(d):
                raise EngineError("checkpoint: truncated")
            typ = d[pos]
            pos += 1
            count = struct.unpack("<Q", take(8))[0]
            if count > (len(d) - pos) // 8:
                raise EngineError("checkpoint: corrupted length header")
            raw = take(8 * count)
            # a repeated name keeps its first record (the reference emplaces)
            if typ == 0:
                f64.setdefault(name, np.frombuffer(raw, "<f8").copy())
            elif typ == 1:
                u64.setdefault(name, np.frombuffer(raw, "<u8").copy())
            else:
                raise EngineError("checkpoint: unknown record type")
        return f64, u64

    def save(self, path: str) -> None:  # Checkpoint::save (engine.cpp:1134-1140)
        with open(path, "wb") as f:
            f.write(self.data)

    @staticmethod
    def load(path: str) -> "Checkpoint":
        try:
            with open(path, "rb") as f:
                data = f.read()
        except OSError:
            raise EngineError("checkpoint: cannot open " + path)
        Checkpoint.deserialize(data)
        return Checkpoint(data)


class GroupView:
    """SynGroupRT mirror (engine.hpp:71-85): per-instance arrays read on access."""

    def __init__(self, eng: "Engine", gid: int, index: int, label: str):
        self._e, self._gid, self._i, self.label = eng, gid, index, label

    def size(self) -> int:
        return int(A.lib().mcg_group_size(self._e._h, self._gid, self._i))

    def _read(self, field: str, dtype) -> np.ndarray:
        n = self.size()
        out = np.empty(n, dtype)
        if n:
            _check(A.lib().mcg_read_state(self._e._h, A.FIELD[field], self._gid, self._i, 0, n,
                                          out.ctypes.data_as(C.c_void_p)))
        return out

    comp = property(lambda s: s._read("syn_comp", np.int32))
    weight = property(lambda s: s._read("syn_weight", np.float64))
    kernel = property(lambda s: s._read("syn_kernel", np.float64))
    stdp_a_pre = property(lambda s: s._read("stdp_a_pre", np.float64))
    stdp_a_post = property(lambda s: s._read("stdp_a_post", np.float64))
    stdp_w = property(lambda s: s._read("stdp_w", np.float64))
    stdp_last_step = property(lambda s: s._read("stdp_last", np.int64))
    homeo_w = property(lambda s: s._read("homeo_w", np.float64))
    stc_h = property(lambda s: s._read("stc_h", np.float64))
    stc_z = property(lambda s: s._read("stc_z", np.float64))
    stc_c = property(lambda s: s._read("stc_c", np.float64))
    sps_abs = property(lambda s: s._read("stc_sps_abs", np.float64))


class CellView:
    """CellRT mirror (engine.hpp:89-115), synced lazily from device state."""

    def __init__(self, eng: "Engine", gid: int):
        self._e, self.gid = eng, gid
        L = A.lib()
        self.ncomp = int(L.mcg_cell_ncomp(eng._h, gid))
        if self.ncomp < 0:
            raise EngineError("gid not on this shard")
        kind = eng._kind_of(gid)
        labels = [p.label for p in kind.placements] if kind is not None else []
        ng = int(L.mcg_cell_ngroups(eng._h, gid))
        self.groups = [GroupView(eng, gid, i, labels[i] if i < len(labels) else "")
                       for i in range(ng)]
        self._kind = kind

    def _comp(self, field: str, index: int = 0) -> np.ndarray:
        out = np.empty(self.ncomp, np.float64)
        _check(A.lib().mcg_read_state(self._e._h, A.FIELD[field], self.gid, index, 0, self.ncomp,
                                      out.ctypes.data_as(C.c_void_p)))
        return out

    def _scalar(self, field: str, dtype):
        out = np.empty(1, dtype)
        _check(A.lib().mcg_read_state(self._e._h, A.FIELD[field], self.gid, 0, 0, 1,
                                      out.ctypes.data_as(C.c_void_p)))
        return out[0]

    @property
    def v_mV(self) -> np.ndarray:
        return self._comp("v")

    @property
    def species(self) -> List[np.ndarray]:
        n = len(self._kind.species) if self._kind is not None else 0
        return [self._comp("species", i) for i in range(n)]

    hh_m = property(lambda s: s._comp("hh_m"))
    hh_h = property(lambda s: s._comp("hh_h"))
    hh_n = property(lambda s: s._comp("hh_n"))
    detector_prev_v = property(lambda s: float(s._scalar("detector_prev_v", np.float64)))
    refractory_until = property(lambda s: int(s._scalar("refractory_until", np.int64)))
    detector_armed = property(lambda s: bool(s._scalar("detector_armed", np.int64)))
    internal_seq = property(lambda s: int(s._scalar("internal_seq", np.int64)))

    def find_group(self, label: str) -> int:
        for i, g in enumerate(self.groups):
            if g.label == label:
                return i
        return -1

    def set_v(self, values):
        a = np.ascontiguousarray(values, np.float64)
        _check(A.lib().mcg_write_state(self._e._h, A.FIELD["v"], self.gid, 0, 0, len(a),
                                       a.ctypes.data_as(C.c_void_p)))


class Engine:
    """B200 engine with mcsim::Engine's public surface."""

    def __init__(self, recipe, options: EngineOptions = EngineOptions(), *, device: int = 0,
                 rank: int = 0, world: int = 1):
        L = A.lib()
        if isinstance(recipe, Recipe):
            self._flat = recipe.flatten()
            self._recipe: Optional[Recipe] = recipe
            view = self._flat.view
        elif isinstance(recipe, FlatRecipe):
            self._flat, self._recipe, view = recipe, recipe.recipe, recipe.view
        else:  # a raw mcg_recipe (e.g. exported by the reference's builders)
            self._flat, self._recipe, view = recipe, None, recipe
        opt = A.mcg_options(float(options.dt_ms), int(options.seed) & (2**64 - 1),
                            int(options.workers), int(device), int(rank), int(world))
        h = C.c_void_p()
        _check(L.mcg_create(C.byref(view), C.byref(opt), C.byref(h)))
        self._h = h
        self.options = options

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            A.lib().mcg_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    def _kind_of(self, gid: int):
        if self._recipe is None:
            return None
        return self._recipe.kinds[int(self._recipe.cell_kind[gid])]

    # ---- time ----
    def time_ms(self) -> float:
        return float(A.lib().mcg_time_ms(self._h))

    def dt_ms(self) -> float:
        return float(A.lib().mcg_dt_ms(self._h))

    def step(self) -> int:
        return int(A.lib().mcg_step(self._h))

    def num_cells(self) -> int:
        return int(A.lib().mcg_num_cells(self._h))

    def min_delay_steps(self) -> int:
        return int(A.lib().mcg_min_delay_steps(self._h))

    def advance_to(self, t_ms: float):
        _check(A.lib().mcg_advance_to(self._h, float(t_ms)))

    def fast_forward_to(self, t_ms: float, coarse_dt_ms: float):
        _check(A.lib().mcg_fast_forward_to(self._h, float(t_ms), float(coarse_dt_ms)))

    # ---- observables ----
    def spike_arrays(self) -> Tuple[np.ndarray, np.ndarray]:
        L = A.lib()
        n = int(L.mcg_num_spikes(self._h))
        if n < 0:
            _check(A.MCG_ERR_CUDA)
        t = np.empty(n, np.float64)
        g = np.empty(n, np.uint32)
        if n:
            _check(L.mcg_get_spikes(self._h, 0, n, t.ctypes.data_as(C.c_void_p),
                                    g.ctypes.data_as(C.c_void_p)))
        return t, g

    def make_checkpoint(self) -> "Checkpoint":
        """Engine::make_checkpoint (engine.cpp:1150-1233): MCSCKPT1 bytes,
        identical to the reference engine's at the same point of the same run."""
        L = A.lib()
        n = C.c_int64()
        _check(L.mcg_checkpoint(self._h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * max(n.value, 1))()
        _check(L.mcg_checkpoint(self._h, buf, n.value, C.byref(n)))
        return Checkpoint(bytes(buf)[:n.value])

    def restore(self, ck: "Checkpoint") -> None:
        """Engine::restore (engine.cpp:1235-1325); takes the reference's
        checkpoints as well."""
        data = ck.data if isinstance(ck, Checkpoint) else bytes(ck)
        buf = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(data or b"\0")
        _check(A.lib().mcg_restore(self._h, buf, len(data)))

    def write_spikes_csv(self, path: str) -> None:
        """spikes.csv of the run so far: times in seconds (t_ms * 1e-3, as the
        reference's drivers convert, network.cpp:104), rows by (t, gid),
        %.17g (csvio.cpp:58-69)."""
        from .csvio import write_spikes_csv
        t, g = self.spike_arrays()
        write_spikes_csv(path, t * 1e-3, g)

    def write_trace_csv(self, probe: int, path: str) -> None:
        """One probe's trace as time_s,value (csvio.cpp:34-39), t_ms * 1e-3."""
        from .csvio import write_trace_csv
        t, v = self.trace_arrays(probe)
        write_trace_csv(path, t * 1e-3, v)

    def spikes(self) -> List[SpikeRecord]:
        t, g = self.spike_arrays()
        return [SpikeRecord(float(a), int(b)) for a, b in zip(t, g)]

    def clear_spikes(self):
        _check(A.lib().mcg_clear_spikes(self._h))

    def cell(self, gid: int) -> CellView:
        return CellView(self, int(gid))

    def trace_arrays(self, probe: int) -> Tuple[np.ndarray, np.ndarray]:
        L = A.lib()
        n = int(L.mcg_trace_len(self._h, probe))
        if n < 0:
            raise IndexError("probe index out of range")
        t = np.empty(n, np.float64)
        v = np.empty(n, np.float64)
        if n:
            _check(L.mcg_get_trace(self._h, probe, t.ctypes.data_as(C.c_void_p),
                                   v.ctypes.data_as(C.c_void_p)))
        return t, v

    def traces(self) -> List[List[Tuple[float, float]]]:
        out = []
        p = 0
        while True:
            n = int(A.lib().mcg_trace_len(self._h, p))
            if n < 0:
                break
            t, v = self.trace_arrays(p)
            out.append(list(zip(t.tolist(), v.tolist())))
            p += 1
        return out

    def stats(self) -> dict:
        s = A.mcg_stats()
        _check(A.lib().mcg_get_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in A.mcg_stats._fields_}

    def set_timing(self, enabled: bool):
        _check(A.lib().mcg_set_timing(self._h, 1 if enabled else 0))

    def set_cell_rng(self, seeds, key_gids):
        """Per-cell RNG keys (mcg_set_cell_rng): cell c draws with (seeds[c],
        key_gids[c]) instead of (options.seed, c) -- independent trials of a
        single-cell protocol in one engine (point-cell kernel only)."""
        sd = np.ascontiguousarray(seeds, dtype=np.uint64)
        kg = np.ascontiguousarray(key_gids, dtype=np.uint32)
        if len(sd) != self.num_cells() or len(kg) != self.num_cells():
            raise ValueError("set_cell_rng: one seed and one key gid per cell")
        _check(A.lib().mcg_set_cell_rng(self._h, sd.ctypes.data_as(C.c_void_p), kg.ctypes.data_as(C.c_void_p)))

    # ---- sharded epoch loop (include/mcg.h; driven by shard.ShardedEngine) ----
    def shard_spike_cap(self) -> int:
        return int(A.lib().mcg_shard_spike_cap(self._h))

    def gid_range(self) -> Tuple[int, int]:
        L = A.lib()
        return int(L.mcg_shard_gid_begin(self._h)), int(L.mcg_shard_gid_end(self._h))

    def set_exchange_buffers(self, send_ptr: int, recv_ptr: int, block_cap: int, world: int):
        _check(A.lib().mcg_shard_set_buffers(self._h, C.c_void_p(send_ptr), C.c_void_p(recv_ptr),
                                             int(block_cap), int(world)))

    def run_epoch(self, t_ms: float):
        _check(A.lib().mcg_shard_run_epoch(self._h, float(t_ms)))

    # ---- the exchange inside the library (NCCL on the engine's stream) ----
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(A.lib().mcg_nccl_unique_id(buf))
        return bytes(buf)

    def init_nccl(self, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid)[:128].ljust(128, b"\0"))
        _check(A.lib().mcg_shard_init_nccl(self._h, buf))

    def shard_advance_to(self, t_ms: float):
        _check(A.lib().mcg_shard_advance_to(self._h, float(t_ms)))

    def global_spike_arrays(self) -> Tuple[np.ndarray, np.ndarray]:
        """Every rank's spikes (the reference's (epoch, gid, step) order)."""
        n = int(A.lib().mcg_shard_num_global_spikes(self._h))
        t = np.empty(n, np.float64)
        g = np.empty(n, np.uint32)
        if n:
            _check(A.lib().mcg_shard_get_global_spikes(self._h, 0, n, t.ctypes.data_as(C.c_void_p),
                                                       g.ctypes.data_as(C.c_void_p)))
        return t, g
