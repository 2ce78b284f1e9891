"""Round profile summaries for profiles/: ncu --set full reports -> <tag>_ncu_<prec>.md and
<tag>_traffic.json; launch-list csv -> <tag>_launches.md.
usage: python tools/profile_summary.py TAG LAUNCHES_CSV Q16_REP FP32_REP"""
import collections, csv, json, re, subprocess, sys
from pathlib import Path

tag, launches, reps = sys.argv[1], sys.argv[2], {"q16": sys.argv[3], "fp32": sys.argv[4]}
root = Path(__file__).resolve().parents[1]
prof = root / "profiles"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]
traffic = {}
for prec, rep in reps.items():
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    d, u = dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    tb = sum(float(d[k].replace(",", "")) * scale.get(u[k], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    traffic[prec] = int(tb)
    traffic[prec + "_ms"] = float(d["gpu__time_duration.sum"])
    mix = subprocess.run([sys.executable, str(root / "tools/ncu_sass.py"), rep, "--top", "20"],
                         capture_output=True, text=True).stdout
    lines = [f"# ncu --set full: {d['Kernel Name'][:80]} 512^3 ({tag})", "",
             f"Command: `ncu --set full --clock-control none --import-source on -k regex:fluid_interior -s 2 -c 1 "
             f"python tools/prof_step.py 512 {prec} 4` after a plain run of the same command (launch 2 = the "
             f"no-stats variant, the bench hot path).", "", "```"]
    lines += [f"{k:62s} {d.get(k)} {u.get(k, '')}" for k in KEYS]
    lines += ["```", "", "```", mix.rstrip(), "```", ""]
    (prof / f"{tag}_ncu_{prec}.md").write_text("\n".join(lines))
traffic["source"] = (f"ncu --set full ({tag}_ncu_q16.md, {tag}_ncu_fp32.md): dram__bytes_read.sum + "
                     "dram__bytes_write.sum per fluid_interior launch, 512^3, no-stats variants")
(prof / f"{tag}_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
h = next(r for r in rows if "Kernel Name" in r)
iK, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows:
    if r is h or r[iK] == "Kernel Name":
        continue
    v = float(r[iV].replace(",", ""))
    ms = v / 1e6 if r[iU] in ("ns", "nsecond") else (v / 1e3 if r[iU] in ("us", "usecond") else v)
    a = agg.setdefault(re.sub(r"\(.*", "", r[iK]).replace("void ", "").replace("hlbm::", ""), [0, 0.0])
    a[0] += 1
    a[1] += ms
tot = sum(a[1] for a in agg.values()) or 1
out = [f"# {tag} launch list: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv "
       "python bench.py --steps 2 --warmup 3`", "",
       "Per-launch times are cold-cache and serialised (compare shares, not absolutes).  Setup kernels",
       "(init_modes, fill_ghosts) run outside the timed region; inside it every step is one `fluid_interior`",
       "launch: STATS=0 in the device-timed loops, STATS=1 in `Solver.step(1)` of the e2e leg.  Template",
       "arguments: <Q16, FORCE, SPECIAL, DITHER, STATS, QMODE, STAGES, NB, LAT>.", "",
       "| launches | total ms | share | avg us | kernel |", "|---|---|---|---|---|"]
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"| {n} | {ms:.3f} | {100 * ms / tot:.1f}% | {1000 * ms / n:.1f} | `{k}` |")
(prof / f"{tag}_launches.md").write_text("\n".join(out) + "\n")
print("wrote", tag, traffic)
