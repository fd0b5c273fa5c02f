#!/usr/bin/env python
"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel:
total ms, launches, share. Usage: python tools/launch_summary.py launches.csv [skip_first_n]"""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for i, r in enumerate(rows[1:]):
    if i < skip or len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(r[iu], 1e-6)
    full = r[ik].replace("(anonymous namespace)", "anon").replace("<unnamed>", "anon").replace("void ", "")
    base = full.split("(")[0]
    name = base.split("<")[0].split("::")[-1] + ("<" + base.split("<", 1)[1] if "<" in base else "")
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.1f} ms over {sum(cnt.values())} launches")
for k, v in tot.most_common(25):
    print(f"{v:10.2f} ms {100 * v / T:5.1f}% {cnt[k]:6d}  {k[:110]}")
