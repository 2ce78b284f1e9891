import sys, subprocess
code = '''
import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import step as ostep
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
shape = tuple(int(v) for v in sys.argv[1].split(",")); steps = int(sys.argv[2])
rho, mom, st = ostep.random_state(shape, seed=1, drho=0.05, umax=0.05, sneq=0.005)
with Solver(SimGrid(shape), SolverConfig(nu=0.02)) as s:
    s.set_moments(rho, mom, st)
    s.step(steps)
print("ok")
'''
for shape, steps in [("16,16,16", 2), ("16,16,16", 3), ("20,30,68", 1), ("16,16,68", 1), ("16,30,16", 1), ("20,16,16", 1), ("20,16,16", 2)]:
    r = subprocess.run([sys.executable, "-c", code, shape, str(steps)], capture_output=True, text=True, timeout=120)
    print(shape, steps, (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:150], flush=True)
