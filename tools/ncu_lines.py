#!/usr/bin/env python3
"""Per-source-line summary of an ncu report: samples, instructions, avg active threads.
usage: tools/ncu_lines.py report.ncu-rep [top_n] [kernel_substr]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ksel = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fpath = func = None; hdr = None
acc = collections.OrderedDict()
for row in rows:
    if not row: continue
    if row[0] == "File Path": fpath = row[1].split("/")[-1]; continue
    if row[0] == "Function Name": func = row[1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or len(row) < 10: continue
    if ksel and ksel not in (func or ""): continue
    if row[2] != "-":  # sass row
        continue
    try:
        ln = int(row[0])
    except ValueError:
        continue
    i_s = hdr.index("# Samples"); i_i = hdr.index("Instructions Executed"); i_t = hdr.index("Thread Instructions Executed")
    k = (func.split("(")[0].split("::")[-1], fpath, ln)
    a = acc.setdefault(k, [0, 0, 0, row[1].strip()[:110]])
    a[0] += int(row[i_s] or 0); a[1] += int(row[i_i] or 0); a[2] += int(row[i_t] or 0)
by_k = collections.defaultdict(lambda: [0, 0])
for (kn, f, ln), a in acc.items():
    by_k[kn][0] += a[0]; by_k[kn][1] += a[1]
for kn, (S, I) in by_k.items():
    print(f"== {kn}: samples {S} inst {I}")
    items = [(k, a) for k, a in acc.items() if k[0] == kn]
    items.sort(key=lambda x: -x[1][0])
    for (kn2, f, ln), a in items[:topn]:
        thr = a[2] / a[1] if a[1] else 0
        print(f"{100*a[0]/max(S,1):5.1f}%smp {100*a[1]/max(I,1):5.1f}%inst thr={thr:4.1f} {f}:{ln:4d} {a[3]}")

# optional region summary: env NCU_REGIONS="name:file:lo-hi,..."
import os
reg = os.environ.get("NCU_REGIONS")
if reg:
    for kn, (S, I) in by_k.items():
        print(f"== regions of {kn}")
        tot_s = tot_i = 0
        for spec in reg.split(","):
            name, f, rng = spec.split(":"); lo, hi = map(int, rng.split("-"))
            s = sum(a[0] for k, a in acc.items() if k[0] == kn and k[1] == f and lo <= k[2] <= hi)
            i = sum(a[1] for k, a in acc.items() if k[0] == kn and k[1] == f and lo <= k[2] <= hi)
            t = sum(a[2] for k, a in acc.items() if k[0] == kn and k[1] == f and lo <= k[2] <= hi)
            tot_s += s; tot_i += i
            print(f"{100*s/max(S,1):5.1f}%smp {100*i/max(I,1):5.1f}%inst thr={t/max(i,1):4.1f}  {name}")
        print(f"{100*tot_s/max(S,1):5.1f}%smp {100*tot_i/max(I,1):5.1f}%inst covered")
