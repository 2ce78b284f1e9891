"""Executed-instruction and stall-sample mix by SASS opcode of an .ncu-rep (source page).
usage: python tools/ncu_sass.py REP [--top N]   (prints per-opcode executed warp instructions,
their share, stall samples, and L1 shared-memory wavefronts / excess)"""
import csv, re, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
iW, iX = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive")
agg = defaultdict(lambda: [0, 0, 0, 0])
for r in rows[2:]:
    if len(r) <= iX:
        continue
    src = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip())
    op = src.split(" ")[0].split(".")[0] if src else "?"
    a = agg[op]
    a[0] += int(r[iE] or 0); a[1] += int(r[iS] or 0); a[2] += int(r[iW] or 0); a[3] += int(r[iX] or 0)
te = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total executed warp instructions {te}, stall samples {ts}")
print(f"{'op':14s} {'executed':>12s} {'share':>6s} {'stall%':>6s} {'smem_wf':>10s} {'excess':>10s}")
for op, (e, s, w, x) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{op:14s} {e:12d} {100*e/te:5.1f}% {100*s/ts:5.1f}% {w:10d} {x:10d}")
