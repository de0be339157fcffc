"""Aggregate an ncu source-page SASS dump (--page source --csv --print-source sass) by opcode:
executed warp instructions and stall samples. usage: python tools/sass_mix.py dump.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iex, isrc, ismp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
cnt, smp = defaultdict(float), defaultdict(float)
tot = tots = 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    x = float(r[iex] or 0)
    s = float(r[ismp] or 0)
    cnt[o] += x
    smp[o] += s
    tot += x
    tots += s
print(f"{'op':10s} {'exec%':>7s} {'stall%':>7s}")
for o in sorted(cnt, key=lambda o: -cnt[o])[:25]:
    print(f"{o:10s} {100 * cnt[o] / tot:7.2f} {100 * smp[o] / tots:7.2f}")
