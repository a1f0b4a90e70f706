#!/usr/bin/env python3
"""Per-kernel digest of the SASS in liblvx_b200.so (cuobjdump): instruction count, registers, local-memory and
shared-memory bytes, and the instruction classes the design claims rest on -- RED vs ATOM (fire-and-forget vs
returning atomics), LDG/STG widths (128/64-bit vector access), LDL/STL (spills / local arrays), DFMA/DADD/DMUL
(f64 arithmetic), SHFL / VOTE / REDUX / MATCH (warp collectives), BAR.
usage: tools/sass_digest.py [lib.so] > profiles/<tag>_sass_digest.txt"""
import collections, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2510_09081_b200", "liblvx_b200.so")
res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
usage = {}
cur = None
for line in res.splitlines():
    m = re.match(r"\s*Function (\S+):", line)
    if m:
        cur = m.group(1); continue
    if cur and "REG:" in line:
        usage[cur] = dict(re.findall(r"(REG|STACK|SHARED|LOCAL):(\d+)", line)); cur = None
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1); kern[cur] = collections.Counter(); continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
    if cur and m:
        op = m.group(1)
        c = kern[cur]
        c["inst"] += 1
        base = op.split(".")[0]
        if base in ("RED", "REDG"): c["RED" + (".64" if ".64" in op else "")] += 1
        elif base in ("ATOM", "ATOMG"): c["ATOM" + (".64" if ".64" in op else "")] += 1
        elif base == "ATOMS": c["ATOMS"] += 1
        elif base == "LDG": c["LDG." + ("128" if ".128" in op else "64" if ".64" in op else "u8/16" if (".U8" in op or ".U16" in op or ".S8" in op or ".S16" in op) else "32")] += 1
        elif base == "STG": c["STG." + ("128" if ".128" in op else "64" if ".64" in op else "u8/16" if (".U8" in op or ".U16" in op) else "32")] += 1
        elif base in ("LDL", "STL"): c[base] += 1
        elif base in ("LDS", "STS"): c[base] += 1
        elif base in ("DFMA", "DADD", "DMUL", "DSETP", "MUFU"): c[base] += 1
        elif base in ("SHFL", "VOTE", "VOTEU", "REDUX", "MATCH", "BAR", "WARPSYNC"): c[base.replace("VOTEU", "VOTE")] += 1
cols = ["inst", "RED", "RED.64", "ATOM", "ATOM.64", "ATOMS", "LDG.128", "LDG.64", "LDG.32", "LDG.u8/16", "STG.128", "STG.64", "STG.32",
        "STG.u8/16", "LDL", "STL", "LDS", "STS", "DFMA", "DADD", "DMUL", "MUFU", "SHFL", "VOTE", "REDUX", "MATCH", "BAR"]
def short(n):
    out = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    out = re.sub(r"\(.*", "", out).replace("void ", "").replace("lvx::", "")
    return out
print(f"SASS digest of {os.path.basename(lib)} (sm_100a; cuobjdump -sass / -res-usage); columns = static instruction counts")
print(f"{'kernel':34s} {'regs':>4s} {'stack':>5s} {'smem':>6s} " + " ".join(f"{c:>7s}" for c in cols))
for k, c in kern.items():
    u = usage.get(k, {})
    print(f"{short(k)[:34]:34s} {u.get('REG', '?'):>4s} {u.get('STACK', '?'):>5s} {u.get('SHARED', '?'):>6s} " +
          " ".join(f"{c.get(col, 0):7d}" for col in cols))
