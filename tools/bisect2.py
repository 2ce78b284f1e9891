import sys, subprocess
code = '''
import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import sphere_mask
dims = tuple(int(v) for v in sys.argv[1].split(",")); prec = sys.argv[2]; xseg = int(sys.argv[3]); dither = sys.argv[4] == "1"; bcx = sys.argv[5]
m = sphere_mask(dims, (dims[0]//4, dims[1]//2, dims[2]//2), min(dims)//8)
bc = {"x": (bcx, "outflow") if bcx == "inflow" else ("periodic", "periodic"), "y": ("periodic", "periodic"), "z": ("periodic", "periodic")}
cfg = SolverConfig(nu=1e-4, bc=bc, u_in=(0.1, 0, 0), precision=prec, xseg=xseg, quant=QuantSpec(dither=dither))
with Solver(SimGrid(dims, m), cfg) as s:
    s.init_modes(np.array([[0, 0, 0, 0.1, 0, 0, np.pi / 2]]))
    s.step(3)
print("ok")
'''
cases = [("64,64,64","q16",0,0,"inflow"), ("64,64,64","q16",0,0,"periodic"), ("64,64,64","q16",0,1,"inflow"),
         ("128,128,128","q16",0,0,"inflow"), ("512,256,256","q16",128,1,"inflow"), ("512,256,256","q16",128,0,"periodic"),
         ("512,256,256","q16",128,0,"inflow"), ("64,64,64","fp32",0,0,"inflow")]
for dims, prec, xseg, dith, bcx in cases:
    r = subprocess.run([sys.executable, "-c", code, dims, prec, str(xseg), str(dith), bcx], capture_output=True, text=True, timeout=120)
    print(dims, prec, xseg, dith, bcx, (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:120], flush=True)
