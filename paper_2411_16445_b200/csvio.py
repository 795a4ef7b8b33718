"""The reference's CSV outputs (proj/src/csvio.cpp), byte for byte.

spikes.csv is the bit-exact parity artefact of a network run:
rows sorted by (time, gid) (csvio.cpp:58-69), times in seconds, every double
printed with %.17g (format_double, csvio.cpp:12-16).
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np


def format_double(v: float) -> str:  # csvio.cpp:12-16 (snprintf "%.17g")
    return "%.17g" % float(v)


def write_spikes_csv(path: str, t_s: Sequence[float], gid: Sequence[int]) -> None:
    """csvio.cpp:58-69: header time_s,cell_id; rows ordered by (t, gid)."""
    t = np.asarray(t_s, dtype=np.float64)
    g = np.asarray(gid, dtype=np.uint32)
    order = np.lexsort((g, t))
    with open(path, "w", newline="\n") as f:
        f.write("time_s,cell_id\n")
        f.writelines(f"{format_double(t[i])},{int(g[i])}\n" for i in order)


def read_spikes_csv(path: str) -> Tuple[np.ndarray, np.ndarray]:  # csvio.cpp:71-88
    with open(path) as f:
        head = f.readline()
        if not head.startswith("time_s,cell_id"):
            raise RuntimeError(f"{path}: expected 'time_s,cell_id' header")
        t, g = [], []
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            if "," not in line:
                raise RuntimeError(f"{path}: malformed row")
            a, b = line.split(",", 1)
            t.append(float(a))
            g.append(int(b))
    return np.array(t, dtype=np.float64), np.array(g, dtype=np.uint32)


def write_trace_csv(path: str, t_s: Sequence[float], value: Sequence[float]) -> None:
    """csvio.cpp:34-39: header time_s,value."""
    with open(path, "w", newline="\n") as f:
        f.write("time_s,value\n")
        f.writelines(f"{format_double(a)},{format_double(b)}\n" for a, b in zip(t_s, value))


def read_trace_csv(path: str) -> Tuple[np.ndarray, np.ndarray]:  # csvio.cpp:41-56
    with open(path) as f:
        head = f.readline()
        if not head.startswith("time_s,value"):
            raise RuntimeError(f"{path}: expected 'time_s,value' header")
        t, v = [], []
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            if "," not in line:
                raise RuntimeError(f"{path}: malformed row")
            a, b = line.split(",", 1)
            t.append(float(a))
            v.append(float(b))
    return np.array(t, dtype=np.float64), np.array(v, dtype=np.float64)
