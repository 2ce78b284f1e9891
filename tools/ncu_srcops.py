"""Executed SASS instructions per CUDA source line, by opcode (needs -lineinfo + --import-source).
usage: python tools/ncu_srcops.py REP [--per N] [--top K] [--fp]
   --per N: divide counts by N (e.g. warp-planes per launch); --fp: include FP32/FP32x2 opcodes"""
import collections, csv, re, subprocess, sys

rep = sys.argv[1]
per = float(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1.0
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
with_fp = "--fp" in sys.argv
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, key, iE = None, None, None
agg = collections.defaultdict(collections.Counter)
src = {}
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        iE = r.index("Instructions Executed")
        continue
    if iE is None or len(r) <= iE:
        continue
    if r[0]:
        key = (fname, r[0])
        src[key] = r[1].strip()
        continue
    if not r[2].startswith("0x") or r[iE] in ("", "-"):
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[3].strip()).split(" ")[0].split(".")[0]
    agg[key][op] += int(r[iE])
skip = set() if with_fp else {"FADD2", "FFMA2", "FMUL2", "FADD", "FFMA", "FMUL", "MUFU"}
tot = collections.Counter({k: sum(v for o, v in c.items() if o not in skip) for k, c in agg.items()})
for k, n in tot.most_common(top):
    ops = ", ".join(f"{o}:{v / per:.1f}" for o, v in agg[k].most_common(5) if o not in skip)
    print(f"{n / per:7.1f}  {k[0]}:{k[1]:5s} {src.get(k, '')[:58]:58s} | {ops}")
