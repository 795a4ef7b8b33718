"""Opcode histogram per source line from `nvdisasm -g` output: sass_lines.py file.sass name.cuh L0 L1"""
import re, sys, collections
lines = open(sys.argv[1]).read().split("\n")
fn, l0, l1 = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cur = None
cnt = collections.defaultdict(collections.Counter)
for l in lines:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", l)
    if m and cur:
        cnt[cur][m.group(2)] += 1
for key in sorted(cnt):
    if key[0] == fn and l0 <= key[1] <= l1:
        print(key[1], dict(cnt[key].most_common(10)))
