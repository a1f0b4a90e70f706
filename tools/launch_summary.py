#!/usr/bin/env python3
"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list.  usage: tools/launch_summary.py launches.csv"""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
acc = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    n = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("lvx::", "")
    v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(r[ui], 1e-3)
    a = acc.setdefault(n, [0, 0.0]); a[0] += 1; a[1] += v
tot = sum(a[1] for a in acc.values())
nf = acc.get("k_scan", [1])[0]
print(f"frames captured: {nf}; total kernel time per frame: {tot / nf:.1f} us (cold-cache, serialised by the profiler)")
for n, a in sorted(acc.items(), key=lambda x: -x[1][1]):
    print(f"{n[:44]:44s} n={a[0]:4d} total={a[1] / 1e3:9.3f} ms  per-frame={a[1] / nf:9.1f} us  share={100 * a[1] / tot:5.1f}%")
