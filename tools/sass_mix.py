"""Static SASS opcode mix of one kernel in an object/.so: python tools/sass_mix.py OBJ NAME_SUBSTRING [OPS...]"""
import re, subprocess, sys
from collections import Counter
obj, key = sys.argv[1], sys.argv[2]
ops = sys.argv[3:]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if key not in name:
        continue
    c = Counter()
    for m in re.finditer(r"/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f):
        c[m.group(1)] += 1
    tot = sum(c.values())
    sel = ops or [k for k, _ in c.most_common(12)]
    print(name[:90], "total", tot, " ".join(f"{k}={c[k]}" for k in sel))
