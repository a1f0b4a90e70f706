#!/usr/bin/env python3
"""One-line-per-kernel summary of an `ncu --set full` report (first launch of every kernel) and the
per-launch DRAM traffic as JSON.   usage: tools/ncu_summary.py report.ncu-rep [traffic.json workload]"""
import csv, io, json, re, subprocess, sys
M = [("time_ms", "gpu__time_duration.sum"), ("dR_MB", "dram__bytes_read.sum"), ("dW_MB", "dram__bytes_write.sum"),
     ("L2hit", "lts__t_sector_hit_rate.pct"), ("L1hit", "l1tex__t_sector_hit_rate.pct"),
     ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active"), ("regs", "launch__registers_per_thread"),
     ("sm%", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
     ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
     ("inst_M", "smsp__inst_executed.sum"), ("thr/inst", "smsp__thread_inst_executed_per_inst_executed.ratio"),
     ("fp64%", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
     ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active")]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(m for _, m in M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
def scale(name, val, unit):
    v = float(val.replace(",", "")) if val not in ("", "n/a") else float("nan")
    if name == "time_ms":
        v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3, "nsecond": 1e-6}.get(unit, 1.0)
    if name in ("dR_MB", "dW_MB"):
        v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
    if name == "inst_M":
        v *= 1e-6
    return v
import os
try:
    PEAK = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
    PEAK_SRC = "MEASURED_PEAKS.json hbm_gbs"
except Exception:
    PEAK, PEAK_SRC = 6650.0, "fallback of B200_PROFILING.md"
seen, traffic = set(), {}
print(f"# DRAM GB/s = (dram bytes read + written) / kernel time; frac = that over the HBM peak of {PEAK:.0f} GB/s ({PEAK_SRC})")
print(f"{'kernel':34s}" + "".join(f"{n:>9s}" for n, _ in M) + f"{'DRAM GB/s':>11s}{'frac':>7s}")
for r in rows[2:]:
    d = dict(zip(h, r)); u = dict(zip(h, units))
    k = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("lvx::", "")
    k = re.sub(r"<.*", "", k)
    if k in seen:
        continue
    seen.add(k)
    vals = {n: scale(n, d.get(m, ""), u.get(m, "")) for n, m in M}
    gbs = (vals["dR_MB"] + vals["dW_MB"]) / max(vals["time_ms"], 1e-9)      # MB / ms = GB/s
    print(f"{k:34s}" + "".join(f"{vals[n]:9.2f}" for n, _ in M) + f"{gbs:11.1f}{gbs / PEAK:7.3f}")
    traffic[k] = int((vals["dR_MB"] + vals["dW_MB"]) * 1e6)
if len(sys.argv) > 3:
    path, wl = sys.argv[2], sys.argv[3]
    try:
        j = json.load(open(path))
    except Exception:
        j = {}
    j[wl] = traffic
    import glob, hashlib, os
    hsh = hashlib.sha256()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for f in sorted(glob.glob(os.path.join(root, "paper_2510_09081_b200", "csrc", "*.cu*"))):
        hsh.update(open(f, "rb").read())
    j.setdefault("_csrc_sha16", {})[wl] = hsh.hexdigest()[:16]     # bench.py refuses the numbers on other sources
    j["_source"] = "ncu --set full --clock-control none, first launch of each kernel in bench.py --workload <w> --steps 1 --warmup 3 --pipeline 1; see profiles/*_ncu_full_*_summary.txt"
    json.dump(j, open(path, "w"), indent=1)
