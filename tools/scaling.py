"""Scaling efficiency of bench.py lines at several GPU counts, with the
reference's formula (scaling_efficiency, bench.cpp:227-240):
    eps(n)  = t(n0) / (t(n) * n)          ("as printed")
    eps'(n) = t(n0) * n0 / (t(n) * n)     ("normalized")
where t(n) is the wall time of a FIXED amount of work on n units.  bench.py's
N > 1 lines are weak-scaled (2000 N cells over N GPUs, value = whole-network
sim-s/wall-s), so the work rate is R(n) = n * value(n) config-3 network-seconds
per wall second and t(n) = W / R(n) for any fixed W: eps(n) = R(n) / (n R(n0)),
eps'(n) = n0 R(n) / (n R(n0)); with n0 = 1 both are value(n) / value(1).

  python tools/scaling.py BENCH_N1.json BENCH_N2.json ...   (one JSON line each;
  files holding a list of lines work too)"""
import json
import sys


def lines(path):
    with open(path) as f:
        txt = f.read().strip()
    try:
        d = json.loads(txt)
        return d if isinstance(d, list) else [d]
    except json.JSONDecodeError:
        return [json.loads(l) for l in txt.splitlines() if l.startswith("{")]


def main(paths):
    pts = {}
    for p in paths:
        for d in lines(p):
            if "value" in d and "n_gpus" in d and d.get("impl") != "reference":
                pts[int(d["n_gpus"])] = float(d["value"])
    if not pts:
        print("no bench lines")
        return 1
    n0 = min(pts)
    rate = {n: n * v for n, v in pts.items()}
    print(f"{'N':>3} {'sim-s/wall-s':>13} {'eps':>7} {'eps_prime':>9}")
    for n in sorted(pts):
        eps = rate[n] / (n * rate[n0])
        print(f"{n:>3} {pts[n]:13.3f} {eps:7.3f} {n0 * eps:9.3f}")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
