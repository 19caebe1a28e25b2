import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import swr_inputs as si
from oracle import oracle
from paper_1503_02564_b200 import SWR
def rel(a, b): return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
cases = [
  ("NT=1000 N=6", si.Problem(a0=-6, b0=6, T=0.5, dx=0.02, dt=5e-4, N=6, potential=si.POT_VX, transmission=si.TC_S02)),
  ("NT=700 N=5 robin", si.Problem(a0=-6, b0=6, T=0.35, dx=0.02, dt=5e-4, N=5, potential=si.POT_VX, transmission=si.TC_ROBIN, robin_p=19.0)),
  ("NT=30 N=3", si.Problem(a0=-6, b0=6, T=0.03, dx=0.02, dt=1e-3, N=3, potential=si.POT_VX, transmission=si.TC_S02)),
  ("N=2 Nj odd", si.Problem(a0=-6, b0=6, T=0.1, dx=0.04, dt=1e-3, N=2, potential=si.POT_VX, transmission=si.TC_S02)),
]
for name, p in cases:
    arr = si.inputs(p)
    x = p.nodes(); arr["u0"] = np.exp(-(x + 1) ** 2 + 3j * x)
    t0 = time.time(); ro = oracle.Oracle(p, arr).solve(); t1 = time.time()
    s = SWR(p, arr); st, uT, rg = s.solve()
    print(name, "Nj", p.Nj, "NT", p.NT, "iters", rg["iterations"], ro["iterations"], "err %.2e" % rel(uT, ro["uT"]), "st", st, ro["status"], "oracle %.1fs" % (t1 - t0), flush=True)
