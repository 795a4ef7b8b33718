"""One ncu report -> markdown summary for profiles/: key counters, warp-stall
reasons (per issue-active cycle) and the top source lines by stall samples.
  python tools/ncu_md.py gpurun_out/x.ncu-rep "title" "context line" > profiles/x.md"""
import csv, io, os, subprocess, sys
rep, title = sys.argv[1], sys.argv[2]
ctx = sys.argv[3] if len(sys.argv) > 3 else ""
here = os.path.dirname(os.path.abspath(__file__))
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
h, u, v = raw[0], raw[1], raw[2]
print(f"# {title}\n")
if ctx:
    print(ctx + "\n")
print(f"Source: `ncu --set full --clock-control none --import-source on` ({os.path.basename(rep)}), "
      "read with `tools/ncu_md.py`.\n")
print("| counter | value | unit |\n|---|---:|---|")
for w in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed",
          "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
          "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]:
    if w in h:
        i = h.index(w)
        print(f"| `{w}` | {v[i]} | {u[i]} |")
print("\nWarp stalls per issue-active cycle (`smsp__average_warps_issue_stalled_*_per_issue_active.ratio`, > 0.05):\n")
print("| reason | ratio |\n|---|---:|")
rs = []
for i, k in enumerate(h):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            x = float(v[i])
        except ValueError:
            continue
        if x > 0.05:
            rs.append((x, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
for x, k in sorted(rs, reverse=True):
    print(f"| {k} | {x:.2f} |")
print("\nTop source lines by warp-stall samples:\n\n```")
out = subprocess.run([sys.executable, os.path.join(here, "ncu_summary.py"), rep, "25"], capture_output=True,
                     text=True).stdout
print("\n".join(l for l in out.splitlines() if ".cuh:" in l or ".h:" in l or ".hpp:" in l or l.startswith("samples")))
print("```")
