"""Table 6 Pade rows with the fixed point for two coefficient readings (SWR_PADE_CLASSIC)."""
import sys, os
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
for m in (20, 50, 100):
    out = []
    for kry in (si.KRY_FIXED_POINT, si.KRY_GMRES, si.KRY_BICGSTAB):
        p = si.config("C2", N=2, g0_random=True, krylov=kry, transmission=si.TC_S22, pade_m=m)
        s = SWR(p, si.inputs(p)); s.build(); st, uT, r = s.solve(); torch.cuda.synchronize()
        out.append(r["iterations"] if st == 0 else f"st{st}")
        del s
    print(os.environ.get("SWR_PADE_THETA", "classic" if os.environ.get("SWR_PADE_CLASSIC") else "midpoint"), m, out, flush=True)
