"""Round-2 summaries of tools/gpu_session_r02.sh's outputs -> profiles/:
r02_bench.json, r02_bench_reference.json, r02_launches.md, r02_k_warp_ncu.md
(+ k_warp_dram.json, read by bench.py for roofline.traffic),
r02_k_warp_config5_ncu.md, r02_k_point_config1_ncu.md, r02_timings.md."""
import collections, csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"


def last_json(path):
    with open(path) as f:
        return json.loads([l for l in f if l.startswith("{")][-1])


json.dump(last_json(os.path.join(OUT, "bench.json")), open(os.path.join(PROF, f"{tag}_bench.json"), "w"), indent=1)
json.dump(last_json(os.path.join(OUT, "bench_ref.json")), open(os.path.join(PROF, f"{tag}_bench_reference.json"), "w"),
          indent=1)

rows = [r for r in csv.reader(open(os.path.join(OUT, "launches.csv"))) if r and not r[0].startswith("==")]
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
    f.write(f"# {tag}: kernel launch list of `bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other`\n\n")
    f.write("ncu `--metrics gpu__time_duration.sum --clock-control none` (cold cache, serialized:\n"
            "absolute times are not bench values; the share is what matters).\n\n")
    f.write("| kernel | launches | total ms | mean ms | share |\n|---|---:|---:|---:|---:|\n")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"| `{k}` | {len(v)} | {sum(v):.3f} | {sum(v)/len(v):.4f} | {100*sum(v)/tot:.1f}% |\n")

md = os.path.join(ROOT, "tools", "ncu_md.py")


def summary(rep, out, title, ctx):
    txt = subprocess.run([sys.executable, md, os.path.join(OUT, rep), title, ctx], capture_output=True, text=True).stdout
    open(os.path.join(PROF, out), "w").write(txt)
    return txt


summary("warp_full.ncu-rep", f"{tag}_k_warp_ncu.md", f"{tag}: k_warp in bench.py (config 3)",
        "`ncu --set full -k regex:k_warp -s 20 -c 1` of `bench.py --steps 2 --warmup 3 --no-cpu-baseline "
        "--no-other`: one launch of 32 min-delay epochs = 192 fine steps of config 3 (t = 3.1-3.2 s, "
        "spontaneous). Algorithmic bytes per launch: 18.8 MB x 192 = 3.61 GB.")
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", os.path.join(OUT, "warp_full.ncu-rep"), "--page", "raw",
                                                  "--csv"], capture_output=True, text=True).stdout)))
h, u, v = raw[0], raw[1], raw[2]
mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(v[h.index("dram__bytes_read.sum")]) * mul[u[h.index("dram__bytes_read.sum")]]
wr = float(v[h.index("dram__bytes_write.sum")]) * mul[u[h.index("dram__bytes_write.sum")]]
json.dump({"kernel": "k_warp", "tag": tag, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
           "fine_steps_in_launch": 192, "source": f"profiles/{tag}_k_warp_ncu.md"},
          open(os.path.join(PROF, "k_warp_dram.json"), "w"), indent=1)
summary("c5_warp.ncu-rep", f"{tag}_k_warp_config5_ncu.md", f"{tag}: k_warp at config 5",
        "Config 5 (N = 100,000, 80k MC x 48 comps, p = 0.002, 12.8 M STC synapses), launch 2 of "
        "tools/prof_c5.py (T0=100): 2 epochs = 8 fine steps, non-resident (148 CTAs x 8 warps walk "
        "20,000 groups per epoch). Algorithmic bytes: 1.006 GB per fine step.")
summary("pt.ncu-rep", f"{tag}_k_point_config1_ncu.md", f"{tag}: k_point at config 1",
        "Config 1 (STET protocol, one exact-LIF point cell, one STC synapse), the first launch of "
        "tools/prof_point.py (T_END=8000 ms: 40,000 fine steps at dt 0.2 ms, before the stimulus). One CTA; "
        "thread 0 runs the serial chain, the other 127 threads draw the epoch's noise and then wait.")
lines = []
for fn in ("config1.txt", "setup.txt"):
    p = os.path.join(OUT, fn)
    if os.path.exists(p):
        lines.append(f"## {fn}\n\n```\n" + open(p).read().strip() + "\n```\n")
open(os.path.join(PROF, f"{tag}_timings.md"), "w").write(
    f"# {tag}: wall-clock timings from tools/gpu_session_r02.sh\n\n`tools/config1_time.py` (each protocol "
    "through the B200 engine and the reference, oracle/_ref, one core) and `tools/setup_time.py` (config 5: "
    "recipe + engine construction).\n\n" + "\n".join(lines))
print(open(os.path.join(PROF, f"{tag}_launches.md")).read())
