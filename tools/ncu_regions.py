"""Stall samples of an ncu source page (--page source --csv) by code region: the straight-line
ranges between CALL / RET / barrier instructions (the out-of-line product functions show up as
the ranges ending in RET).  Used to read the latency-path profiles (profiles/README.md).

    ncu -i rep.ncu-rep --page source --csv > src.csv; python tools/ncu_regions.py src.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
isrc = h.index("Source")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
idx = {r: h.index(r) for r in reasons}
start = 0
acc = collections.Counter()
for n, r in enumerate(data):
    for k, i in idx.items():
        try:
            acc[k] += int(r[i] or 0)
        except ValueError:
            pass
    src = r[isrc]
    if any(m in src for m in ("CALL", "RET", "BAR.SYNC", "ATOMG", "EXIT")):
        tot = sum(acc.values())
        if tot >= 20:
            top = ", ".join(f"{k[6:]} {v}" for k, v in acc.most_common(4))
            print(f"{start:5d}-{n:5d} {tot:5d}  {top}  | {src.strip()[:40]}")
        acc = collections.Counter()
        start = n + 1
