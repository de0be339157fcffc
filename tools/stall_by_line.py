"""Per-source-line stall breakdown (long_sb / short_sb / wait / math) from an ncu SASS source dump.
usage: python tools/stall_by_line.py <nvdisasm -gi> <kernel> <sass csv> [top] [source-file substring]"""
import csv
import re
import sys
from collections import defaultdict

dis, kern, src = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
srcpat = sys.argv[5] if len(sys.argv) > 5 else "eval_fast"
off2line, cur, inside = {}, None, False
for ln in open(dis):
    if ln.startswith("//----") and ".text." in ln:
        inside = kern in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
    if m:
        chain = [(m.group(1), int(m.group(2)))] + [(a, int(b)) for a, b in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))]
        cur = next(((a, b) for a, b in chain if srcpat in a), chain[-1])
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src)))
h = rows[1]
cols = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_math", "stall_barrier", "stall_mio",
        "stall_branch_resolving", "Instructions Executed"]
idx = [h.index(c) for c in cols]
ia = h.index("Address")
agg = defaultdict(lambda: [0.0] * len(cols))
tot = [0.0] * len(cols)
base = None
for r in rows[2:]:
    if len(r) < len(h):
        continue
    a = int(r[ia], 16)
    base = a if base is None else base
    k = off2line.get(a - base, ("?", 0))[1]
    for i, c in enumerate(idx):
        v = float(r[c] or 0)
        agg[k][i] += v
        tot[i] += v
src_lines = {i: t.strip() for i, t in enumerate(open([f for f, _ in off2line.values() if srcpat in f][0]), 1)}
print("totals:", {c: int(t) for c, t in zip(cols, tot)})
for ci, c in enumerate(cols[:5] + cols[-1:]):
    ci = cols.index(c)
    print(f"--- {c}")
    for k in sorted(agg, key=lambda k: -agg[k][ci])[:top]:
        print(f"  {k:4d} {100 * agg[k][ci] / max(tot[ci], 1):5.1f}%  {src_lines.get(k, '')[:90]}")
