"""Summaries of one GPU profiling session (tools/gpu_profile.sh) -> profiles/.

  python tools/make_profiles.py r01
writes profiles/<tag>_bench.json, <tag>_launches.md, <tag>_k_batch_ncu.md and
profiles/batch_kernel_dram.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(PROF, exist_ok=True)

# ---- bench line
bench = None
with open(os.path.join(OUT, "bench.json")) as f:
    for line in f:
        line = line.strip()
        if line.startswith("{"):
            bench = json.loads(line)
with open(os.path.join(PROF, f"{tag}_bench.json"), "w") as f:
    json.dump(bench, f, indent=1)

# ---- launch list (ncu --metrics gpu__time_duration.sum, same bench command)
rows = [r for r in csv.reader(open(os.path.join(OUT, "launches.csv")))
        if r and not r[0].startswith("==")]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
per = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r[ui], 1e-6)
    per[r[ki].split("(")[0]].append(v * scale)
tot = sum(sum(v) for v in per.values())
with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
    f.write(f"# {tag}: kernel launch list of `bench.py --steps 2 --warmup 3 --no-cpu-baseline`\n\n")
    f.write("ncu `--metrics gpu__time_duration.sum --clock-control none` (cold cache, serialized:\n"
            "absolute times are not bench values; the share is what matters).\n\n")
    f.write("| kernel | launches | total ms | mean ms | share |\n|---|---:|---:|---:|---:|\n")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"| `{k}` | {len(v)} | {sum(v):.3f} | {sum(v)/len(v):.4f} | {100*sum(v)/tot:.1f}% |\n")

# ---- full capture of one k_batch launch
rep = os.path.join(OUT, "batch_full.ncu-rep")
def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
def metric(name):
    return (v[h.index(name)], u[h.index(name)]) if name in h else (None, None)
def to_bytes(val, unit):
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val.replace(",", "")) * mul
rd = to_bytes(*metric("dram__bytes_read.sum"))
wr = to_bytes(*metric("dram__bytes_write.sum"))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct"]
summary = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "30"],
                         capture_output=True, text=True).stdout
with open(os.path.join(PROF, f"{tag}_k_batch_ncu.md"), "w") as f:
    f.write(f"# {tag}: `ncu --set full --import-source on -k regex:k_batch -s 20 -c 1` of bench.py\n\n")
    f.write("One launch of the persistent batch kernel (32 min-delay epochs = 192 fine steps of the\n"
            "config-3 network, during the timed region).  Cold-cache replay.\n\n")
    f.write("| metric | value | unit |\n|---|---:|---|\n")
    for k in keys:
        val, un = metric(k)
        if val is not None:
            f.write(f"| `{k}` | {val} | {un} |\n")
    f.write("\n## Stall samples / instructions by source line\n\n```\n" + summary + "```\n")
with open(os.path.join(PROF, "batch_kernel_dram.json"), "w") as f:
    json.dump({"kernel": "k_batch", "tag": tag, "dram_bytes_per_launch": rd + wr,
               "dram_read": rd, "dram_write": wr, "fine_steps_in_launch": 192,
               "source": f"profiles/{tag}_k_batch_ncu.md"}, f, indent=1)
print(open(os.path.join(PROF, f"{tag}_launches.md")).read())
