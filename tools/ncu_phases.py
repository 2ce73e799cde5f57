#!/usr/bin/env python
"""Stall-sample share and warp instructions per code region of one kernel from an ncu report's
SASS source page (`ncu -i rep --page source --csv --print-source sass`).  Regions are given as
`name:lo-hi` address offsets (hex, relative to the kernel's first instruction); without them the
kernel is cut at its barriers.

usage: ncu_phases.py source.csv [name:lo-hi ...]"""
import collections
import csv
import sys


def main(path, specs):
    rows = list(csv.reader(open(path)))
    h, data = rows[1], []
    for r in rows[2:]:  # the first kernel block only (a multi-kernel export repeats the header)
        if not r or r[0] in ("Kernel Name", "Address"):
            break
        data.append(r)
    ia, isrc = h.index("Address"), h.index("Source")
    iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    idx = {c: h.index(c) for c in stalls}
    f = lambda x: float(x) if x not in ("", "n/a") else 0.0  # noqa: E731
    base = int(data[0][ia], 16)
    tot = sum(f(r[iss]) for r in data) or 1.0
    if specs:
        segs = []
        for s in specs:
            name, rng = s.split(":")
            lo, hi = rng.split("-")
            segs.append((int(lo, 16), int(hi, 16), name))
    else:
        cuts = [0] + [int(r[ia], 16) - base for r in data if "BAR.SYNC" in r[isrc]] + [1 << 40]
        segs = [(cuts[i], cuts[i + 1], f"region{i}") for i in range(len(cuts) - 1)]
    print(f"{rows[0][1][:90]}: {tot:.0f} stall samples, "
          f"{sum(f(r[iex]) for r in data) / 1e6:.1f} M warp instructions")
    for lo, hi, name in segs:
        s = ex = 0.0
        c = collections.Counter()
        for r in data:
            a = int(r[ia], 16) - base
            if lo <= a < hi:
                s += f(r[iss])
                ex += f(r[iex])
                for k in stalls:
                    c[k] += f(r[idx[k]])
        if s:
            top = ", ".join(f"{k[6:]} {v / s * 100:.0f}%" for k, v in c.most_common(5))
            print(f"  {name:20s} [{lo:05x}, {min(hi, 0xfffff):05x}) {s / tot * 100:5.1f}% of samples, "
                  f"{ex / 1e6:7.1f} M warp inst | {top}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
