"""Shared-memory wavefronts (total and excessive = bank conflicts) per source line of one kernel,
from an ncu --set full capture (--import-source on) and the object the kernel was built from.

    python tools/smem_by_line.py <report.ncu-rep> <object.o> <kernel substring> <source substring> [top]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, obj, kern, srcpat = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 12
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, check=True, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-gi", os.path.join(td, cub)], capture_output=True, text=True).stdout
off2line, cur, inside, srcfile = {}, None, False, None
for ln in dis.split("\n"):
    if ln.startswith("//----") and ".text." in ln:
        inside = kern in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
    if m:
        chain = [(m.group(1), int(m.group(2)))] + [(a, int(b)) for a, b in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))]
        cur = next(((a, b) for a, b in chain if srcpat in a), chain[-1])
        if srcpat in cur[0]:
            srcfile = cur[0]
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
cols = ["L1 Wavefronts Shared Excessive", "L1 Wavefronts Shared", "Instructions Executed",
        "Warp Stall Sampling (All Samples)"]
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
    k = off2line.get(a - base, 0)
    for i, c in enumerate(idx):
        v = float(r[c] or 0)
        agg[k][i] += v
        tot[i] += v
print("totals:", {c: f"{t:.4g}" for c, t in zip(cols, tot)})
src = open(srcfile).read().split("\n") if srcfile and os.path.exists(srcfile) else []
for k in sorted(agg, key=lambda k: -agg[k][1])[:top]:
    v = agg[k]
    if v[1] == 0:
        break
    s = src[k - 1].strip()[:80] if 0 < k <= len(src) else ""
    print(f"line {k:4d}  wavefronts {v[1]:.3g}  excessive {v[0]:.3g} ({100 * v[0] / max(v[1], 1):.0f}%)  {s}")
