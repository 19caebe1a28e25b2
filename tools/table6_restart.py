"""Table 6, Robin p = 5 and Pade m = 20 with GMRES: iteration counts against the restart length."""
import sys
sys.path.insert(0, '.')
import torch
import swr_inputs as si
from paper_1503_02564_b200 import SWR
for name, kw in (("Robin p=5", dict(transmission=si.TC_ROBIN, robin_p=5.0)),
                 ("S2^{2,20}", dict(transmission=si.TC_S22, pade_m=20)), ("S0^2", dict(transmission=si.TC_S02))):
    out = []
    for restart in (30, 100, 300, 1000):
        p = si.config("C2", N=2, g0_random=True, krylov=si.KRY_GMRES, restart=restart, **kw)
        s = SWR(p, si.inputs(p)); s.build(); st, uT, r = s.solve(); torch.cuda.synchronize()
        out.append((restart, r["iterations"] if st == 0 else f"st{st}"))
        del s
    print(name, out, flush=True)
