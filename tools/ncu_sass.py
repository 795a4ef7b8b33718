"""SASS rows (with stall samples) under given source lines: ncu_sass.py csv file.cuh L0 L1"""
import csv, sys, collections
rows = csv.reader(open(sys.argv[1]))
fn, l0, l1 = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cur, hdr, on = None, None, False
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    if r[0].isdigit():
        on = cur == fn and l0 <= int(r[0]) <= l1
        if on: print(f"--- {r[0]}: {r[1][:100]}")
        continue
    if on and len(r) > 4:
        d = dict(zip(hdr[2:], r[2:]))
        st = collections.Counter({k[6:]: int(v or 0) for k, v in d.items()
                                  if k.startswith("stall_") and "Not Issued" not in k and (v or "0").isdigit()})
        top = " ".join(f"{k}:{v}" for k, v in st.most_common(2) if v)
        print(f"   {r[3][:60]:60s} s={d.get('Warp Stall Sampling (All Samples)','')} ex={d.get('Instructions Executed','')} {top}")
