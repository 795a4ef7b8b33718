import sys, time
sys.path.insert(0, "/root/repo")
from paper_2411_16445_b200 import network as N
N.uniform_stream((1, 0, 0, 0), 0, 4)
for _ in range(2):
    t = time.perf_counter(); s, d = N.er_pairs(1, 100000, 0.002); print("er_pairs", time.perf_counter() - t, len(s), flush=True)
