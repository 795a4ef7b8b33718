"""tools/scaling.py: the reference's scaling_efficiency (bench.cpp:227-240)
applied to bench.py's weak-scaled lines (work rate R(n) = n value(n))."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, pts):
    files = []
    for n, v in pts.items():
        p = tmp_path / f"b{n}.json"
        p.write_text(json.dumps({"metric": "m", "n_gpus": n, "value": v}) + "\n")
        files.append(str(p))
    ref = tmp_path / "ref.json"  # reference-arm lines are ignored
    ref.write_text(json.dumps({"impl": "reference", "n_gpus": 1, "value": 1e9}) + "\n")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "scaling.py"), *files, str(ref)],
                         capture_output=True, text=True, check=True).stdout
    rows = {}
    for line in out.splitlines()[1:]:
        n, v, e, ep = line.split()
        rows[int(n)] = (float(v), float(e), float(ep))
    return rows


def test_perfect_weak_scaling_is_one(tmp_path):
    rows = _run(tmp_path, {1: 40.0, 2: 40.0, 4: 40.0, 8: 40.0})
    assert all(abs(e - 1.0) < 1e-9 and abs(ep - 1.0) < 1e-9 for _, e, ep in rows.values())


def test_efficiency_is_value_ratio(tmp_path):
    rows = _run(tmp_path, {1: 40.0, 2: 30.0, 8: 10.0})
    assert abs(rows[2][1] - 0.75) < 1e-9 and abs(rows[8][1] - 0.25) < 1e-9
    # n0 = 1: eps' == eps
    assert all(abs(e - ep) < 1e-12 for _, e, ep in rows.values())
