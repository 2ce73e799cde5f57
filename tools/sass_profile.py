#!/usr/bin/env python
"""Summarise an ncu SASS source page (CSV): instructions per unit of work by opcode and the
stall samples by 50-instruction block.  usage: sass_profile.py src.csv units [block]"""
import collections
import csv
import re
import sys

path, units = sys.argv[1], float(sys.argv[2])
blk_n = int(sys.argv[3]) if len(sys.argv) > 3 else 50
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = [r for r in csv.DictReader(lines[start:]) if r["Address"].startswith("0x")]
seen, uniq = set(), []
for r in rows:           # some ncu versions print the listing twice
    if r["Address"] in seen:
        break
    seen.add(r["Address"])
    uniq.append(r)
rows = uniq
ins, st = collections.Counter(), collections.Counter()
tot = stot = 0
blocks = collections.OrderedDict()
for i, r in enumerate(rows):
    src = re.sub(r"^@!?U?P\w+\s+", "", r["Source"].strip())
    op = src.split()[0].split(".")[0] if src else "?"
    n = int(r["Instructions Executed"] or 0)
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    ins[op] += n; st[op] += s; tot += n; stot += s
    b = blocks.setdefault(i // blk_n, [0, 0, collections.Counter()])
    b[0] += n; b[1] += s; b[2][op] += n
print(f"{len(rows)} SASS lines, {tot / units:.1f} warp-instr per unit, {stot} stall samples")
for op, n in ins.most_common(25):
    print(f"  {op:10s} {n / units:8.1f}  stall {100 * st[op] / max(stot, 1):5.1f}%")
print("blocks:")
for b, (n, s, c) in blocks.items():
    if n / units > 0.5 or s > 0.01 * stot:
        print(f"  {b * blk_n:5d} {n / units:7.1f} instr  stall {100 * s / max(stot, 1):5.1f}%  "
              + " ".join(f"{k}:{v / units:.0f}" for k, v in c.most_common(5)))
