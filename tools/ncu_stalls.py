"""Top SASS lines per stall reason of an .ncu-rep: python tools/ncu_stalls.py rep.ncu-rep [reason ...]"""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
iS = h.index("Source")
reasons = sys.argv[2:] or ["stall_long_sb", "stall_wait", "stall_short_sb", "stall_math", "stall_branch_resolving"]
for rs in reasons:
    i = h.index(rs)
    tot = sum(int(r[i]) for r in data) or 1
    print(f"== {rs}: {tot} samples")
    for r in sorted(data, key=lambda r: -int(r[i]))[:8]:
        print(f"   {100*int(r[i])/tot:5.1f}%  {r[0][-5:]}  {r[iS][:90]}")
