"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys, collections
rows = csv.reader(open(sys.argv[1]))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, hdr, tot = None, None, collections.Counter()
stalls = collections.defaultdict(collections.Counter)
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or not r[0].isdigit(): continue
    d = dict(zip(hdr[2:], r[2:]))  # skip the two source columns' duplicate names
    try: s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError: continue
    key = (cur, int(r[0]), r[1][:90])
    tot[key] += s
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try: stalls[key][k[6:]] += int(v or 0)
            except ValueError: pass
allv = sum(tot.values())
print("total samples", allv)
for key, s in tot.most_common(n_top):
    top = ", ".join(f"{k}:{v}" for k, v in stalls[key].most_common(3) if v)
    print(f"{100*s/allv:5.1f}% {key[0]}:{key[1]}  {key[2]}  [{top}]")
