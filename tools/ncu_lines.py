"""Per-CUDA-source-line stall samples / instructions of an .ncu-rep (needs -lineinfo + --import-source)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; fname = None; res = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8 or r[0] == "": continue
    try: res.append((int(r[4]), int(r[7]), fname, r[0], r[1][:90]))
    except ValueError: pass
tot = sum(x[0] for x in res) or 1; tote = sum(x[1] for x in res) or 1
print("total samples", tot, "instr", tote)
for s, e, f, ln, src in sorted(res, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*s/tot:5.1f}% {100*e/tote:5.1f}%i {f}:{ln} {src}")
