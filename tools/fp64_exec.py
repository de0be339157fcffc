"""Executed FP64 work of a kernel from an ncu SASS source dump (thread-level instruction
counts): DFMA / DADD / DMUL totals and the hardware FP64 rate 2*DFMA + DADD + DMUL per second
(the instruction-level counterpart of bench.py's algorithmic roofline.achieved).

usage: python tools/fp64_exec.py <sass.csv> <duration_s> [points]"""
import csv
import json
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
dur = float(sys.argv[2])
pts = int(sys.argv[3]) if len(sys.argv) > 3 else 0
h = rows[1]
isrc, ith = h.index("Source"), h.index("Predicated-On Thread Instructions Executed")
cnt = defaultdict(float)
for r in rows[2:]:
    if len(r) < len(h):
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    base = o.split(".")[0]
    if base in ("DFMA", "DADD", "DMUL"):
        cnt[base] += float(r[ith] or 0)
flops = 2 * cnt["DFMA"] + cnt["DADD"] + cnt["DMUL"]
res = {k: cnt[k] for k in ("DFMA", "DADD", "DMUL")}
res["hw_fp64_flops"] = flops
res["hw_fp64_tflops"] = flops / dur / 1e12
if pts:
    res["fp64_instr_per_eval"] = (cnt["DFMA"] + cnt["DADD"] + cnt["DMUL"]) / pts
    res["hw_flops_per_eval"] = flops / pts
print(json.dumps(res, indent=1))
