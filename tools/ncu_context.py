"""Print SASS context around the top stall-sample instructions of an .ncu-rep."""
import csv, subprocess, sys
rep = sys.argv[1]; ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 4; before = int(sys.argv[3]) if len(sys.argv) > 3 else 8
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]; d = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iSrc = h.index("Source")
tot = sum(int(r[iS]) for r in d)
order = sorted(range(len(d)), key=lambda k: -int(d[k][iS]))[:ntop]
for k in order:
    print(f"---- {d[k][0][-5:]} {d[k][iS]} samples ({100*int(d[k][iS])/tot:.1f}%)")
    for r in d[max(0, k - before):k + 2]:
        print(f"  {r[0][-5:]} {r[iS]:>6s} {r[iSrc][:100]}")
