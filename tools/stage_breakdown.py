"""Per-stage breakdown of the fused fast dd kernel from an ncu --set full capture (SURVEY.md §8d:
"per fused kernel with a per-stage breakdown"): warp samples (time), executed warp instructions
and FP64 thread instructions attributed to source lines, grouped by the stage markers of
csrc/eval_fast.cu ("// ---- stage ...").

usage: python tools/stage_breakdown.py <report.ncu-rep> <out prefix> [kernel-substring]"""
import csv
import io
import json
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1201_0499_b200", "csrc", "eval_fast.cu")
OBJ = os.path.join(ROOT, "paper_1201_0499_b200", "_build", "eval_fast.cu.o")

rep, out = sys.argv[1], sys.argv[2]
kname = sys.argv[3] if len(sys.argv) > 3 else "fast_kernelILi8ELi32ELb1E"

# stage boundaries from the source markers
lines = open(SRC).read().split("\n")
marks = []
for i, ln in enumerate(lines, 1):
    m = re.search(r"// ---- (stages? [^:;(]*)", ln)
    if m:
        marks.append((i, m.group(1).strip()))
first_stage = marks[0][0]


def stage_of(line):
    name = "tile setup (points, tables, schedule prefetch)"
    for i, nm in marks:
        if line >= i:
            name = nm
    if line < first_stage:
        name = "tile setup (points, tables, schedule prefetch)"
    return name


with tempfile.TemporaryDirectory() as td:
    subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-xelf", "all", OBJ], cwd=td, check=True, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "-gi", os.path.join(td, cub)], capture_output=True,
                         text=True, check=True).stdout
off2line, cur, inside = {}, None, False
for ln in dis.split("\n"):
    if ln.startswith("//----") and ".text." in ln:
        inside = kname in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', ln)
    if m:
        chain = [(m.group(1), int(m.group(2)))] + [(a, int(b)) for a, b in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))]
        cur = next(((a, b) for a, b in chain if "eval_fast" in a), chain[-1])[1]
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                        text=True).stdout
rows = list(csv.reader(io.StringIO(csvtxt)))
h = rows[1]
ia, isrc = h.index("Address"), h.index("Source")
isamp, iinst = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ith = h.index("Thread Instructions Executed")
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
base = None
for r in rows[2:]:
    if len(r) < len(h):
        continue
    a = int(r[ia], 16)
    base = a if base is None else base
    st = stage_of(off2line.get(a - base, 0))
    agg[st][0] += float(r[isamp] or 0)
    agg[st][1] += float(r[iinst] or 0)
    op = r[isrc].strip().split()
    o = (op[1] if op and op[0].startswith("@") else (op[0] if op else "")).split(".")[0]
    if o in ("DFMA", "DADD", "DMUL"):
        agg[st][2] += float(r[ith] or 0)
tot = [sum(v[i] for v in agg.values()) for i in range(3)]
res = {st: {"time_share": v[0] / tot[0], "instr_share": v[1] / tot[1], "fp64_share": v[2] / max(tot[2], 1)}
       for st, v in agg.items()}
json.dump(res, open(out + ".json", "w"), indent=1)
with open(out + ".md", "w") as fh:
    fh.write(f"# per-stage breakdown of `{kname}` (`{os.path.basename(rep)}`)\n\n")
    fh.write("| stage | time (warp samples) | warp instructions | FP64 instructions |\n|---|---|---|---|\n")
    for st, v in sorted(res.items(), key=lambda kv: -kv[1]["time_share"]):
        fh.write(f"| {st} | {100 * v['time_share']:.1f}% | {100 * v['instr_share']:.1f}% | {100 * v['fp64_share']:.1f}% |\n")
print(open(out + ".md").read())
