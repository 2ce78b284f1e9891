"""Summarise an .ncu-rep: key throughput metrics, stall reasons, top SASS lines, opcode mix."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__grid_size", "smsp__cycles_active.avg"]
for k in want:
    if k in h:
        i = h.index(k); print(f"{k:60s} {v[i]:>20s} {u[i]}")
st = []
for i, a in enumerate(h):
    if a.startswith("smsp__average_warps_issue_stalled_") and a.endswith("_per_issue_active.ratio"):
        try: st.append((float(v[i].replace(",", "")), a.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError: pass
print("stalls (warps per issue):", ", ".join(f"{n}={x:.2f}" for x, n in sorted(st, reverse=True)[:10]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]; data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed"); iSrc = h.index("Source")
tot_e = sum(int(r[iE]) for r in data); tot_s = sum(int(r[iS]) for r in data)
print("sass lines", len(data), "instr executed", tot_e, "samples", tot_s)
for r in sorted(data, key=lambda r: -int(r[iS]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  {r[0][-5:]} samp={r[iS]:>6s} exec={r[iE]:>9s}  {r[iSrc][:80]}")
c = Counter()
for r in data:
    t = r[iSrc].split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    c[op.split(".")[0]] += int(r[iE])
print("opcode mix %:", ", ".join(f"{k}={100*x/tot_e:.1f}" for k, x in c.most_common(22)))
