"""Attribute ncu per-SASS stall samples / executed instructions to source lines.
usage: python tools/line_attrib.py <nvdisasm -gi output> <kernel mangled name> <ncu sass csv> [file-filter]"""
import csv
import os
import re
import sys
from collections import defaultdict

dis, kern, src = sys.argv[1], sys.argv[2], sys.argv[3]
filt = sys.argv[4] if len(sys.argv) > 4 else "eval_fast.cu"
off2line = {}
cur = None
inside = False
for ln in open(dis):
    if ln.startswith("//----") and ".text." in ln:
        inside = kern in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
    if m:
        f, l, rest = m.group(1), int(m.group(2)), m.group(3)
        mi = re.findall(r'inlined at "([^"]+)", line (\d+)', rest)
        chain = [(f, l)] + [(a, int(b)) for a, b in mi]
        pick = next(((a, b) for a, b in chain if filt in a), chain[-1])
        cur = pick
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src)))
h = rows[1]
ia, iex, ismp = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = None
ex, sm = defaultdict(float), defaultdict(float)
tot_e = tot_s = 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    a = int(r[ia], 16)
    base = a if base is None else base
    key = off2line.get(a - base, ("?", 0))
    e, s = float(r[iex] or 0), float(r[ismp] or 0)
    ex[key] += e
    sm[key] += s
    tot_e += e
    tot_s += s
srcl = {}
try:
    for i, t in enumerate(open(os.environ.get("PJ_SRC") or [k[0] for k in ex if filt in k[0]][0]), 1):
        srcl[i] = t.strip()
except Exception:
    pass
print(f"{'line':>5s} {'exec%':>6s} {'stall%':>6s}  source")
for k in sorted(ex, key=lambda k: -sm[k])[:40]:
    print(f"{k[1]:5d} {100 * ex[k] / tot_e:6.2f} {100 * sm[k] / tot_s:6.2f}  {srcl.get(k[1], k[0])[:100] if filt in k[0] else k[0]}")
