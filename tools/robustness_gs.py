import sys, time
sys.path.insert(0, '.')
import numpy as np, torch, dataclasses
import swr_inputs as si
from oracle import oracle
from paper_1503_02564_b200 import SWR
def rel(a, b): return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
base = si.Problem(a0=-6, b0=6, T=0.35, dx=0.02, dt=5e-4, N=5, potential=si.POT_VX, transmission=si.TC_ROBIN, robin_p=19.0)
for gs in (1, 2):
  for tmode in (None,):
    p = dataclasses.replace(base, gs_passes=gs)
    arr = si.inputs(p)
    x = p.nodes(); arr["u0"] = np.exp(-(x + 1) ** 2 + 3j * x)
    ro = oracle.Oracle(p, arr).solve()
    s = SWR(p, arr); st, uT, rg = s.solve()
    h_o = np.array(ro["history"]); h_g = np.array(rg["history"])
    n = min(len(h_o), len(h_g))
    d = np.abs(h_o[:n] - h_g[:n]) / h_o[0]
    first = int(np.argmax(d > 1e-8)) if (d > 1e-8).any() else -1
    print("gs", gs, "iters", rg["iterations"], ro["iterations"], "err %.2e" % rel(uT, ro["uT"]), "first hist divergence >1e-8 at", first, "res at end", h_o[-1], h_g[-1], flush=True)
