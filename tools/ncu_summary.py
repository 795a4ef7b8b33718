"""Summarize an ncu report: key metrics + top source lines by stall samples."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:70s} {v[i]:>14s} {u[i]}")
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
cur = hdr = None
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        hdr = None
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].strip():
        continue
    try:
        samp = float(r[4] or 0)
        inst = float(r[7] or 0)
    except ValueError:
        continue
    k = (cur, r[0])
    agg[k][0] += samp
    agg[k][1] += inst
    if r[1].strip():
        agg[k][2] = r[1].strip()[:90]
ts = sum(x[0] for x in agg.values()) or 1
ti = sum(x[1] for x in agg.values()) or 1
print(f"\nsamples {ts:.0f}  warp-instructions {ti:.0f}")
for k, x in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:>5s} samp {100 * x[0] / ts:5.1f}% inst {100 * x[1] / ti:5.1f}%  {x[2]}")
